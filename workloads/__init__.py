"""Seeded synthetic inputs and workload shape tables.

Shared by the tests, the bench and smoke(); used to feed BOTH the oracle and
the CUDA path the same bytes.  This package holds none of the method's
arithmetic: no convolution, no zero-point algebra, no requantize — only
random-number generation (numpy PCG64, ``default_rng(seed)``) and shape tables
(derived from torchvision model definitions; the paper
lists no shapes).  See DESIGN.md "Input recipe".
"""
from .gen import (ConvCase, DenseCase, conv_case, dense_case, rand_q, rng,  # noqa: F401
                  calibrated_out_scale)
from .shapes import (ConvShape, resnet50_convs, resnet50_fc, mobilenet_v2_convs,  # noqa: F401
                     inception_v3_convs, resnet50_unique)
