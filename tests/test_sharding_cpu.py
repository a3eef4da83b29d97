"""Multi-process (gloo, world_size 2) coverage of the N>1 path on CPU: batch
sharding is a partition, per-shard results concatenate to the full result
(images are independent: SURVEY §8e), and timing takes the max over ranks.
The CUDA kernels are not involved (no GPU here); the per-shard compute uses
the oracle, which is allowed in tests."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2006_10226_b200.sharding import max_over_ranks, shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 256, 257):
        for world in (1, 2, 3, 8):
            got = [shard_range(n, r, world) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == n
            for (a, b), (c, d) in zip(got, got[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in got]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as orc
    from workloads import gen
    case = gen.conv_case(11, 5, 8, 7, 7, 8, 3, 3, (1, 1), (1, 1, 1, 1))
    lo, hi = shard_range(case.A.shape[0], rank, world)
    sub = np.ascontiguousarray(case.nchw()[lo:hi])
    y = orc.qnn_conv2d(sub, case.oihw(), case.zp_A, case.zp_W, case.s_A, case.s_W, case.bias, case.out_params(),
                       case.stride, case.pad)
    # gather shards (test-only: the bench has no data-path collective)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([y.shape[0]]))
    maxn = int(max(s.item() for s in sizes))
    pad = np.zeros((maxn,) + y.shape[1:], y.dtype)
    pad[:y.shape[0]] = y
    bufs = [torch.zeros(pad.shape, dtype=torch.uint8) for _ in range(world)]
    dist.all_gather(bufs, torch.from_numpy(pad))
    t = max_over_ranks(1.0 + rank, dist)
    if rank == 0:
        full = np.concatenate([b.numpy()[:int(s.item())] for b, s in zip(bufs, sizes)])
        ref = orc.qnn_conv2d(case.nchw(), case.oihw(), case.zp_A, case.zp_W, case.s_A, case.s_W, case.bias,
                             case.out_params(), case.stride, case.pad)
        out["equal"] = bool(np.array_equal(full, ref))
        out["tmax"] = t
    dist.destroy_process_group()


def test_two_rank_gloo_shards_concatenate_to_full_batch():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out["equal"] is True
    assert out["tmax"] == 2.0


def test_bench_reference_arm_runs_on_cpu():
    """`bench.py --impl reference` (the oracle arm) prints one JSON line with the contract keys."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "impl", "cpu_baseline", "e2e", "higher_is_better", "config"):
        assert k in line
    assert line["impl"] == "reference" and line["value"] > 0


def test_bench_gpus2_spawns_two_ranks_on_cpu():
    """`bench.py --gpus 2` without torchrun launches the two ranks itself (127.0.0.1); with the
    reference arm (no GPU needed) rank 0 prints exactly one JSON line and rank 1 exits 0."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=900, cwd=root,
                       env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    assert json.loads(lines[0])["n_gpus"] == 2


def test_bench_rejects_world_gpus_mismatch():
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "4",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300, cwd=root,
                       env=env)
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr


def test_shard_model_partitions_the_batch():
    import bench
    gm = bench.resnet50_model(7)
    parts = [bench.shard_model(gm, *shard_range(7, r, 3)) for r in range(3)]
    assert np.array_equal(np.concatenate([p["image"] for p in parts]), gm["image"])
    assert np.array_equal(np.concatenate([p["fc"]["A"] for p in parts]), gm["fc"]["A"])
    for k in gm["fresh"]:
        assert np.array_equal(np.concatenate([p["fresh"][k] for p in parts]), gm["fresh"][k])
    for p in parts:
        n = p["image"].shape[0]
        assert all(sp.N == n for sp in p["specs"])
        assert p["weights"] is gm["weights"]      # replicated, not re-drawn
