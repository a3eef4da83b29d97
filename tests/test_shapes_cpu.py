"""Pins the workload shape tables (`workloads/shapes.py`) to
something other than themselves: torchvision's model definitions of the
paper's three evaluation models (Table 2).  Every Conv2d of the
torchvision model is recorded with a forward hook on one image, and the
multiset of (C, K, H, W, R, S, stride, pad, groups) must equal the table's.
Also pins the analytic weight count `tools/fp_baseline.py` reports (SURVEY
§8f row f3: int8 weights are exactly 1/4 of fp32)."""
import sys
import os

import pytest
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from workloads.shapes import inception_v3_convs, mobilenet_v2_convs, resnet50_convs, resnet50_fc  # noqa: E402

tv = pytest.importorskip("torchvision")


def _torch_convs(model, hw):
    rec = []

    def hook(mod, inp, out):
        x = inp[0]
        p = mod.padding
        rec.append((mod.in_channels, mod.out_channels, x.shape[2], x.shape[3], mod.kernel_size[0],
                    mod.kernel_size[1], tuple(mod.stride), (p[0], p[1], p[0], p[1]), mod.groups))

    hs = [m.register_forward_hook(hook) for m in model.modules() if isinstance(m, torch.nn.Conv2d)]
    with torch.no_grad():
        model.eval()(torch.zeros(1, 3, hw, hw))
    for h in hs:
        h.remove()
    return sorted(rec)


def _table(convs):
    return sorted((c.C, c.K, c.H, c.W, c.R, c.S, tuple(c.stride), tuple(c.pad), c.groups) for c in convs)


def test_resnet50_shapes_match_torchvision():
    assert _table(resnet50_convs()) == _torch_convs(tv.models.resnet50(), 224)


def test_mobilenet_v2_shapes_match_torchvision():
    assert _table(mobilenet_v2_convs()) == _torch_convs(tv.models.mobilenet_v2(), 224)


def test_inception_v3_shapes_match_torchvision():
    m = tv.models.inception_v3(init_weights=False, aux_logits=False)
    assert _table(inception_v3_convs()) == _torch_convs(m, 299)


def test_resnet50_weight_count_and_int8_ratio():
    m = tv.models.resnet50()
    n_tv = sum(p.numel() for p in m.parameters() if p.dim() > 1)     # conv + fc weights, no BN / bias
    fin, fout = resnet50_fc()
    n = sum(c.K * (c.C // c.groups) * c.R * c.S for c in resnet50_convs()) + fin * fout
    assert n == n_tv == 25_502_912
    assert 4 * n == sum(p.numel() * p.element_size() for p in m.parameters() if p.dim() > 1)


def test_footprint_liveness_planner():
    """tools/fp_baseline.py's buffer-liveness peak on a hand-checked chain:
    a(u8 x100) -> b(u8 x50) -> c(s32 x10) -> a.  a stays live across the whole sequence (it is
    rewritten last), so the peak is at the middle call: 100 + 50 + 40 bytes; as fp32 every
    element takes 4 bytes: 400 + 200 + 40."""
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import fp_baseline as fb
    tr = fb._Trace()
    a, b = torch.zeros(100, dtype=torch.uint8), torch.zeros(50, dtype=torch.uint8)
    c = torch.zeros(10, dtype=torch.int32)
    f = tr.wrap(lambda *x, **k: None)
    f(a, out=b)
    f(b, out=c)
    f(c, out=a)
    assert tr.peak_live() == 190 and tr.peak_live(as_fp32=True) == 640
    assert tr.peak_live(exclude={a.untyped_storage().data_ptr()}) == 90


def test_fp_baseline_bn_folding_preserves_the_forward():
    """tools/fp_baseline.py folds BN into the convs of the cuDNN comparison arm (row f2); the
    folded model must compute the same function (fp32 rounding only) and contain no BN."""
    import copy

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import fp_baseline as fb
    torch.manual_seed(0)
    m = tv.models.resnet50().eval()
    for mod in m.modules():
        if isinstance(mod, torch.nn.BatchNorm2d):
            mod.running_mean.uniform_(-0.5, 0.5)
            mod.running_var.uniform_(0.5, 2.0)
            mod.weight.data.uniform_(0.5, 1.5)
            mod.bias.data.uniform_(-0.2, 0.2)
    f = fb._fold_bn(copy.deepcopy(m))
    assert not any(isinstance(q, torch.nn.BatchNorm2d) for q in f.modules())
    x = torch.randn(2, 3, 224, 224)
    with torch.no_grad():
        y0, y1 = m(x), f(x)
    assert (y0 - y1).abs().max().item() <= 1e-5 * max(1.0, y0.abs().max().item())
