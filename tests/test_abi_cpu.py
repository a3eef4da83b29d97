"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/qnn.h declares, and its host-only logic (fixed-point multiplier
derivation, argument validation, plan sizing) behaves — no kernel launches."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def qlib():
    from paper_2006_10226_b200 import build
    build.build()
    from paper_2006_10226_b200 import qnn
    return qnn


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "qnn.h")).read()
    return sorted(set(re.findall(r"QNN_API\s+[\w\s\*]*?\b(qnn_\w+)\s*\(", src)))


def test_header_declares_abi():
    syms = _declared_symbols()
    assert len(syms) == 23
    for s in ("qnn_conv2d", "qnn_depthwise_conv2d", "qnn_dense", "qnn_requantize", "qnn_quantize", "qnn_dequantize",
              "qnn_quantize_host", "qnn_dequantize_host"):
        assert s in syms


def test_library_exports_every_declared_symbol(qlib):
    L = qlib.lib()
    for s in _declared_symbols():
        assert hasattr(L, s), s
    assert sorted(qlib.EXPORTED) == _declared_symbols()


def test_library_is_sm100a_only(qlib):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", qlib.LIB_PATH], capture_output=True, text=True)
    archs = set(re.findall(r"sm_\d+a?", out.stdout))
    assert archs == {"sm_100a"}, archs


def test_sass_uses_tcgen05_and_tma(qlib):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", qlib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCIMMA" in out          # tcgen05.mma.kind::i8
    assert "UTMALDG.4D.IM2COL" in out  # TMA im2col loads
    assert "LDTM" in out             # tcgen05.ld TMEM -> registers


def test_derive_multiplier_matches_oracle(qlib, orc):
    g = np.random.default_rng(5)
    ms = list(np.exp(g.uniform(-40, 20, size=3000))) + [0.5, 1.0, 0.25, 0.1, 1 / 3, 0.5 + 2 ** -32, 1 - 2 ** -40,
                                                         5e-324, 2.2250738585072014e-308]
    for m in ms:
        assert qlib.qnn_derive_multiplier(float(m)) == orc.derive_multiplier(float(m)), m
    for bad in (0.0, -2.0, float("nan"), float("inf")):
        with pytest.raises(qlib.QnnError):
            qlib.qnn_derive_multiplier(bad)


def test_status_strings(qlib):
    L = qlib.lib()
    for code, name in qlib.STATUS.items():
        assert L.qnn_status_string(code).decode() == name


def _desc(qlib, **kw):
    d = qlib.Conv2dDesc()
    base = dict(N=1, H=8, W=8, C=16, K=16, R=3, S=3, stride_h=1, stride_w=1, pad_t=1, pad_l=1, pad_b=1, pad_r=1,
                dil_h=1, dil_w=1, groups=1, in_cstride=0, out_cstride=0)
    base.update(kw)
    for k, v in base.items():
        setattr(d, k, v)
    d.input_dtype = kw.get("input_dtype", qlib.QNN_U8)
    d.kernel_dtype = kw.get("kernel_dtype", qlib.QNN_S8)
    d.input_zero_point = kw.get("input_zero_point", 128)
    d.kernel_zero_point = kw.get("kernel_zero_point", 0)
    d.input_scale = kw.get("input_scale", 0.5)
    sc = (ctypes.c_float * 1)(0.01)
    d.kernel_scales = ctypes.cast(sc, ctypes.POINTER(ctypes.c_float))
    d.num_kernel_scales = 1
    d._keep = sc
    return d


def _size(qlib, d, o=None):
    n = ctypes.c_size_t()
    st = qlib.lib().qnn_conv2d_prepack_size(ctypes.byref(d), ctypes.byref(o) if o else None, ctypes.byref(n))
    return st, n.value


def test_plan_sizes_and_validation(qlib):
    o = qlib.output_params(4.0, 128, "u8")
    st, n = _size(qlib, _desc(qlib), o)
    assert st == 0 and n > 0
    # packed weights dominate: Kpad(32) * 9 taps * Cw(32) bytes at least
    assert n >= 32 * 9 * 32
    cases = [
        (dict(N=0), 1),                         # empty batch is an invalid shape
        (dict(stride_h=0), 1),
        (dict(input_zero_point=300), 1),        # zp outside u8
        (dict(kernel_zero_point=-129), 1),      # zp outside s8
        (dict(groups=2), 2),                    # grouped (non-depthwise) conv: unsupported
        (dict(input_scale=0.0), 1),
        (dict(input_scale=float("nan")), 1),
        (dict(R=9, pad_t=0, pad_b=0, H=4), 1),  # filter larger than padded input
        (dict(C=8192, R=3, S=3), 2),            # KK*255*255 >= 2^31 (reading R10)
        (dict(in_cstride=8), 1),                # channel pitch smaller than C
    ]
    for kw, want in cases:
        st, _ = _size(qlib, _desc(qlib, **kw), o)
        assert st == want, (kw, st)
    # output params validation
    for bad in (qlib.output_params(0.0, 0), qlib.output_params(1.0, 300), qlib.output_params(1.0, 0, "s8", act_min=10, act_max=5)):
        st, _ = _size(qlib, _desc(qlib), bad)
        assert st == 1
    assert _size(qlib, _desc(qlib), qlib.output_params(1.0, 0, "s32"))[0] == 2   # s32 via NULL params only
    # depthwise plans are valid
    assert _size(qlib, _desc(qlib, groups=16), o)[0] == 0


def test_requantize_validation_before_launch(qlib):
    L = qlib.lib()
    shp = (ctypes.c_int64 * 2)(4, 3)
    sc1 = (ctypes.c_float * 1)(0.5)
    sc2 = (ctypes.c_float * 2)(0.5, 0.25)
    dummy = ctypes.c_void_p(16)
    # wrong per-channel length along axis 1 (3 != 2)
    assert L.qnn_requantize(dummy, 2, dummy, 1, shp, 2, 1, sc2, 2, 0, 1.0, 0, 0, None) == 1
    # zp out of range
    assert L.qnn_requantize(dummy, 2, dummy, 1, shp, 2, -1, sc1, 1, 0, 1.0, 256, 0, None) == 1
    # bad axis
    assert L.qnn_requantize(dummy, 2, dummy, 1, shp, 2, 5, sc1, 1, 0, 1.0, 0, 0, None) == 1
    # m >= 2^30 is unsupported (reading R15)
    big = (ctypes.c_float * 1)(2.0 ** 31)
    assert L.qnn_requantize(dummy, 2, dummy, 1, shp, 2, -1, big, 1, 0, 1.0, 0, 0, None) == 2
    # quantize needs an 8-bit output
    zp = (ctypes.c_int32 * 1)(0)
    assert L.qnn_quantize(dummy, dummy, 2, shp, 2, -1, sc1, zp, 1, None) == 2
    # empty tensors enqueue nothing and succeed
    z = (ctypes.c_int64 * 1)(0)
    assert L.qnn_requantize(None, 2, None, 1, z, 1, -1, sc1, 1, 0, 1.0, 0, 0, None) == 0


def test_no_cpu_fallback_without_library(qlib, tmp_path, monkeypatch):
    """The binding raises if libqnn.so is absent (no silent fallback)."""
    import paper_2006_10226_b200.qnn as q
    monkeypatch.setattr(q, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(q, "_lib", None)
    monkeypatch.delenv("QNN_AUTOBUILD", raising=False)
    with pytest.raises(q.QnnError):
        q.lib()


def test_legalize_rejects_non_u8_weights():
    """The Legalize applies to u8 weights only; the dtype check happens in the
    binding before any launch, so it is testable without a GPU."""
    import torch

    from paper_2006_10226_b200.qnn import QnnError, legalize_s8_weights
    with pytest.raises(QnnError):
        legalize_s8_weights(torch.zeros(4, 1, 1, 16, dtype=torch.int8), 0)
