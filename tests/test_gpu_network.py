"""End-to-end parity of the full ResNet-50 forward (convs + max pool +
residual qnn.add + global average pool + fc) on the GPU vs the oracle composition, bit-exact
logits, at batch 2 (the oracle runs the same ops one by one on the CPU)."""
import os
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.mark.parametrize("fused", [True, False], ids=["fused_residual", "separate_add"])
def test_resnet50_full_forward_matches_oracle(fused):
    import bench
    m = bench.resnet50_full_model(2, seed=6100, fused=fused)
    net = bench.GpuResNet50Full(m, torch.device("cuda"))
    net.step()
    torch.cuda.synchronize()
    got = net.logits.cpu().numpy()
    want = bench.oracle_full_forward(m, 2)
    assert got.shape == want.shape
    assert np.array_equal(got.view(np.int32), want.view(np.int32))
    # the forward is not degenerate: logits vary across classes and images
    assert np.unique(got).size > 100 and not np.array_equal(got[0], got[1])


@pytest.mark.parametrize("world", [2, 4, 8])
def test_bench_shards_concatenate_to_one_gpu_output(world):
    """SURVEY §8e test T3 on the CUDA path: configs[4]'s batch split over `world` ranks with
    bench.shard_model (each shard planned and launched at its own batch, as rank r would run
    it) reproduces the 1-GPU output bit for bit.  The ranks are run one after another on this
    GPU: the sharded path has no collective, so nothing waits on another rank."""
    import bench
    from paper_2006_10226_b200.sharding import shard_range
    G = 40
    gm = bench.resnet50_model(G)
    dev = torch.device("cuda")
    full = bench.GpuResNet50(gm, dev)
    full.step()
    torch.cuda.synchronize()
    want_logits = full.fc_out.cpu().numpy()
    want_last = full.stack.outs["layer4.2.conv3"].cpu().numpy()
    got_logits, got_last = [], []
    for r in range(world):
        lo, hi = shard_range(G, r, world)
        net = bench.GpuResNet50(bench.shard_model(gm, lo, hi), dev)
        net.step()
        torch.cuda.synchronize()
        got_logits.append(net.fc_out.cpu().numpy())
        got_last.append(net.stack.outs["layer4.2.conv3"].cpu().numpy())
    assert np.array_equal(np.concatenate(got_logits), want_logits)
    assert np.array_equal(np.concatenate(got_last), want_last)
    # and the full forward (glue ops) shards the same way
    fm = bench.resnet50_full_model(G)
    ffull = bench.GpuResNet50Full(fm, dev)
    ffull.step()
    torch.cuda.synchronize()
    parts = []
    for r in range(world):
        lo, hi = shard_range(G, r, world)
        n = bench.GpuResNet50Full(bench.shard_full_model(fm, lo, hi), dev)
        n.step()
        torch.cuda.synchronize()
        parts.append(n.logits.cpu().numpy())
    assert np.array_equal(np.concatenate(parts).view(np.int32), ffull.logits.cpu().numpy().view(np.int32))


def test_inception_v3_full_forward_matches_oracle():
    """configs[4]'s second network as a true forward: 94 convs whose branch
    outputs land in channel slices of the concat buffers (out_cstride), stem and reduction max
    pools, branch average pools, global average pool, fc, dequantize -- bit-exact logits, and
    every intermediate buffer equal, vs the oracle running the same ops one by one."""
    import bench
    m = bench.inception_v3_full_model(2, seed=7100)
    net = bench.GpuInceptionV3(m, torch.device("cuda"))
    for b in net.buf.values():
        b.fill_(0xA5)                     # sentinel: a channel slice left unwritten shows up below
    net.step()
    torch.cuda.synchronize()
    want_logits, want_acc, want_buf = bench.oracle_inception_forward(m, 2, with_buffers=True)
    for name, b in want_buf.items():
        assert np.array_equal(net.buf[name].cpu().numpy(), b), name
    assert np.array_equal(net.fc_out.cpu().numpy(), want_acc.astype(np.int32))
    got = net.logits.cpu().numpy()
    # int32 -> fp32 dequantize: BJ:north_star allows 1 ulp (fl32(s * fl32(q - zp)) rounds twice)
    ulps = np.abs(got.view(np.int32).astype(np.int64) - want_logits.view(np.int32).astype(np.int64))
    assert ulps.max() <= 1
    assert np.unique(got).size > 100 and not np.array_equal(got[0], got[1])


def test_inception_v3_shards_concatenate():
    import bench
    from paper_2006_10226_b200.sharding import shard_range
    G, world = 6, 2
    m = bench.inception_v3_full_model(G, seed=7200)
    dev = torch.device("cuda")
    full = bench.GpuInceptionV3(m, dev)
    full.step()
    torch.cuda.synchronize()
    parts = []
    for r in range(world):
        lo, hi = shard_range(G, r, world)
        n = bench.GpuInceptionV3(bench.shard_inception(m, lo, hi), dev)
        n.step()
        torch.cuda.synchronize()
        parts.append(n.logits.cpu().numpy())
    assert np.array_equal(np.concatenate(parts).view(np.int32), full.logits.cpu().numpy().view(np.int32))
