"""GPU parity: qnn.dense (tcgen05 GEMM + fused requantize) vs the oracle."""
import numpy as np
import pytest

from gpu_helpers import gpu_dense, mismatch_report, oracle_dense
from workloads import gen
import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,K,adt,wdt,zpW,odt,pc", [
    (1, 1000, 2048, "u8", "s8", 0, "u8", True),        # ResNet-50 fc at batch 1
    (64, 1000, 2048, "u8", "s8", 0, "s8", True),
    (512, 512, 512, "u8", "s8", 0, "u8", True),        # config 4 smallest
    (300, 200, 96, "s8", "s8", 0, "s32", True),
    (129, 257, 160, "u8", "u8", 100, "u8", False),     # u8 x u8, zp_W != 0, ragged
    (1024, 1024, 1024, "u8", "s8", 0, "u8", True),
])
def test_dense_full(M, N, K, adt, wdt, zpW, odt, pc):
    for mode in ("upward", "tonearest"):
        case = gen.dense_case(M * 7 + N, M, N, K, adt, wdt, zp_W=zpW, per_channel=pc, out_dtype=odt, rounding=mode)
        _, _, y = gpu_dense(case)
        got, want = y.cpu().numpy(), oracle_dense(case)
        assert np.array_equal(got, want), mismatch_report(got, want)


@pytest.mark.parametrize("n", [2048, 4096, 8192])
def test_dense_large_sampled(n):
    """config 4 sizes: full launch, 4096 sampled outputs vs the oracle."""
    case = gen.dense_case(3000 + n, n, n, n)
    _, _, y = gpu_dense(case)
    got = y.cpu().numpy().reshape(-1)
    idx = np.random.default_rng(n).choice(got.size, 4096, replace=False)
    idx[:4] = [0, got.size - 1, n - 1, got.size - n]
    acc = orc.dense_acc_at(case.A, case.W, case.zp_A, case.zp_W, idx, case.bias)
    o = case.out_params()
    M, S = orc.conv_multipliers(case.s_A, case.s_W, o["scale"], n)
    k = idx % n
    want = np.array([orc.requantize_acc(acc[i:i + 1], M[k[i]:k[i] + 1], S[k[i]:k[i] + 1], o["dtype"],
                                        o["zero_point"], o["rounding"], o["relu"], axis=0)[0] for i in range(idx.size)])
    assert np.array_equal(got[idx], want)


@pytest.mark.parametrize("n,wdt,zpW,mode", [(4096, "u8", 119, "tonearest"), (8192, "u8", 140, "upward"),
                                            (3000, "s8", -3, "tonearest")])
def test_dense_large_sampled_zpW(n, wdt, zpW, mode):
    """configs[3] with asymmetric weights (zp_W != 0: the Term-3 row sums of the activations)
    and both rounding modes, incl. a size that is not a multiple of the tile (3000)."""
    case = gen.dense_case(6000 + n, n, n, n, "u8", wdt, zp_W=zpW, per_channel=False, rounding=mode)
    _, _, y = gpu_dense(case)
    got = y.cpu().numpy().reshape(-1)
    idx = np.random.default_rng(n + 1).choice(got.size, 4096, replace=False)
    idx[:4] = [0, got.size - 1, n - 1, got.size - n]
    acc = orc.dense_acc_at(case.A, case.W, case.zp_A, case.zp_W, idx, case.bias)
    o = case.out_params()
    M, S = orc.conv_multipliers(case.s_A, case.s_W, o["scale"], n)
    k = idx % n
    Mk = np.broadcast_to(M, (n,)) if np.size(M) == 1 else M
    Sk = np.broadcast_to(S, (n,)) if np.size(S) == 1 else S
    want = np.array([orc.requantize_acc(acc[i:i + 1], Mk[k[i]:k[i] + 1], Sk[k[i]:k[i] + 1], o["dtype"],
                                        o["zero_point"], o["rounding"], o["relu"], axis=0)[0] for i in range(idx.size)])
    assert np.array_equal(got[idx], want)
