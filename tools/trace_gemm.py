"""Run one conv layer with QNN_GEMM_TRACE and print CTA 0's pipeline timeline (profiling aid)."""
import os, sys, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
buf = torch.zeros(16384, dtype=torch.int64, device="cuda")  # slots < 16384
os.environ["QNN_GEMM_TRACE"] = str(buf.data_ptr())
from tools.bench_layers import conv_layer  # noqa
from workloads.shapes import resnet50_unique
name, batch = sys.argv[1], int(sys.argv[2])
c = [x for x in resnet50_unique() if x.name == name][0]
fn, macs, by = conv_layer(c, batch)
fn(); torch.cuda.synchronize(); buf.zero_(); fn(); torch.cuda.synchronize()
t = buf.cpu().numpy()
t0 = t[6000]
def rel(a): return (a[a > 0] - t0)
prod, mma, es, ew, ee = rel(t[0:2048]), rel(t[2048:4096]), rel(t[4096:4608]), rel(t[5120:5632]), rel(t[4608:5120])
print(name, batch, "prologue", t[6001] - t0, "total", t[6002] - t0)
print("producer kb issue (first 12):", prod[:12].tolist(), "n", prod.size)
print("mma kb start (first 12):", mma[:12].tolist(), "n", mma.size)
print("producer dt median", np.median(np.diff(prod)) if prod.size > 2 else None, "mma dt median", np.median(np.diff(mma)) if mma.size > 2 else None)
print("epi tile: start/tfull/done (first 8):", list(zip(es[:8].tolist(), ew[:8].tolist(), ee[:8].tolist())))
print("epi per tile: wait", np.median(ew - es[:ew.size]) if ew.size else None, "work", np.median(ee - ew[:ee.size]) if ee.size else None, "tile period", np.median(np.diff(es)) if es.size > 2 else None)
pre, post = t[6100:6164], t[6200:6264]
m = (pre > 0) & (post > 0)
print("mma: before-commit rel to kb start:", (pre[m][:10] - t[2048+1:2048+11][:m.sum()]).tolist() if m.sum() else None)
print("commit cost:", (post[m] - pre[m])[:16].tolist())
pw0, pw1, pi = t[6300:6556], t[0:256], t[6600:6856]
n = int(((pw0 > 0) & (pi > 0)).sum())
print("producer: wait(empty) cost:", (pw1[:n] - pw0[:n])[:16].tolist())
print("producer: issue cost      :", (pi[:n] - pw1[:n])[:16].tolist())
if n > 1:
    print("producer: loop overhead   :", (pw0[1:n] - pi[:n-1])[:16].tolist())
ep = t[12000:12000 + 8 * 60].reshape(60, 8)
print("epilogue warp0 'two' path: tmem-loaded, store-buffer-free, chunkA, chunkB  (rel. to tfull wake)")
for i in range(0, 40, 2):
    if ep[i, 0] > 0:
        w = t[5120 + i]
        print(i, [int(x - w) if x > 0 else None for x in ep[i, :4]])
mw0, mw1 = t[6900:7156], t[2048:2048+256]
n2 = int((mw0 > 0).sum())
print("mma: wait(full) cost:", (mw1[:n2] - mw0[:n2])[:20].tolist())
print("load latency (issue->mma start):", (mw1[:min(n, n2)] - pi[:min(n, n2)])[:20].tolist())
def r(a): return (a.astype(np.int64) - t0) * (a > 0)
m0, m1, m2 = r(t[7200:7300]), r(t[7300:7400]), r(t[7400:7500])
rel = t[7500:7500 + 1600].reshape(100, 16)
relmax = np.where(rel > 0, rel - t0, 0).max(axis=1)
ew = r(t[5120:5220])
print("tile | mma wait tempty start/end | commit tfull | last epi release (max over warps) | epi tfull wake")
for i in range(4, 14):
    print(i, m0[i], m1[i], m2[i], relmax[i - 2] if i >= 2 else None, ew[i])
for i in (4, 5, 6):
    row = rel[i]
    print("tile", i, "tfull wake(w0)", ew[i], "release per warp:", [int(x - t0) if x > 0 else None for x in row])
wk = t[9200:9200 + 1600].reshape(100, 16); en = t[10900:10900 + 1600].reshape(100, 16)
for i in (4, 5, 6):
    print("tile", i, "wake:", [int(x - t0) if x > 0 else None for x in wk[i]])
    print("       end :", [int(x - t0) if x > 0 else None for x in en[i]])
# a_rows: MMA issue time per stage (stage start -> all its MMAs issued)
st, iss = t[2048:2048 + 64], t[6100:6164]
m = (st > 0) & (iss > 0)
if m.sum():
    print("a_rows MMA issue cycles per stage:", (iss[m] - st[m])[:20].tolist())
