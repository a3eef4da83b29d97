"""paper_2006_10226_b200 — B200-native (sm_100a) QNN pre-quantized operator hot path.

arXiv 2006.10226, "Efficient Execution of Quantized Deep Learning Models: A
Compiler Approach": the lowered qnn.conv2d / qnn.dense (four-term zero-point
algebra, Eq. 3, with the fixed-point requantize of Eq. 5 fused into the
epilogue), depthwise conv, standalone requantize and quantize/dequantize.

The compute lives in ``libqnn.so`` (CUDA for sm_100a, C ABI in
``include/qnn.h``); ``qnn`` is the ctypes binding.
"""
from . import qnn  # noqa: F401
from .qnn import (PackedConv2d, PackedDense, QnnError, lib, qnn_add, qnn_conv2d, qnn_dense,  # noqa: F401
                  qnn_depthwise_conv2d, qnn_dequantize, qnn_dequantize_host, qnn_derive_multiplier, qnn_pool2d,
                  qnn_quantize, qnn_quantize_host, qnn_requantize)
