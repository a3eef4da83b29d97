#!/usr/bin/env python
"""Round-2 ncu evidence -> profiles/ (run here, on the reports tools/profile_r02.sh brought back).

* r02_launches_step.csv / r02_launches_summary.txt: one step of the benched conv stack
  (quantize, 53 conv, fc, dequantize) and one step of the full network, from the ncu launch
  list of the bench command (cold-cache, serialised: compare SHARES with the live breakdown);
* r02_ncu_<layer>.txt: the `--set full` details page of one GEMM launch per layer, plus the
  tensor-pipe counters and the utilisation they imply (see the note at the top of each file);
* gemm_traffic.json: mean DRAM bytes per GEMM launch of the stack step (bench.py roofline.traffic).
"""
from __future__ import annotations

import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUN = os.environ.get("R02_RUN") or os.path.join(ROOT, "gpurun_out", "r02prof")
OUT = os.path.join(ROOT, "profiles")
sys.path.insert(0, os.path.join(ROOT, "tools"))
from summarize_profiles import load_launches, short  # noqa: E402

MAC_PER_CLK_SM = 8183      # profiles/mma_peak.json: tcgen05.mma kind::i8 128x256x32 issue rate
LAYER_MACS = {}            # filled from workloads.shapes


def steps(L):
    isq = lambda n: "quantize" in n and "dequantize" not in n and "requantize" not in n
    out = []
    for qi, x in enumerate(L):
        if isq(x["name"]):
            di = next((j for j in range(qi, len(L)) if "dequantize" in L[j]["name"]), None)
            if di is not None:
                out.append(L[qi:di + 1])
    return out


def summarize_step(step, tag, title):
    tot = sum(x.get("gpu__time_duration.sum", 0) for x in step)
    with open(os.path.join(OUT, f"r02_launches_{tag}.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["idx", "kernel", "duration_ns", "dram_read_bytes", "dram_write_bytes"])
        for i, x in enumerate(step):
            w.writerow([i, short(x["name"]), int(x.get("gpu__time_duration.sum", 0)),
                        int(x.get("dram__bytes_read.sum", 0)), int(x.get("dram__bytes_write.sum", 0))])
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for x in step:
        a = agg[short(x["name"])]
        a[0] += 1
        a[1] += x.get("gpu__time_duration.sum", 0)
        a[2] += x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0)
    lines = [title, f"step launches: {len(step)}   summed kernel time: {tot / 1e3:.1f} us", "",
             f"{'kernel':62s} {'n':>4s} {'time_us':>10s} {'share':>7s} {'dram_MB':>9s}"]
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k:62s} {n:4d} {t / 1e3:10.1f} {t / tot:7.3f} {b / 1e6:9.1f}")
    gemm = [x for x in step if "qnn_gemm_i8_kernel" in x["name"] or "qnn_gemm_t_kernel" in x["name"]]
    per_launch = sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in gemm) / max(1, len(gemm))
    lines += ["", f"GEMM launches: {len(gemm)}; mean DRAM traffic per launch {per_launch / 1e6:.2f} MB; "
                  f"GEMM share of step {sum(x.get('gpu__time_duration.sum', 0) for x in gemm) / tot:.3f}"]
    return lines, per_launch, len(gemm)


def layer_macs():
    sys.path.insert(0, ROOT)
    from workloads.shapes import resnet50_unique
    for c in resnet50_unique():
        P = (c.H + c.pad[0] + c.pad[2] - c.R) // c.stride[0] + 1
        Q = (c.W + c.pad[1] + c.pad[3] - c.S) // c.stride[1] + 1
        LAYER_MACS[c.name] = 256 * P * Q * c.K * c.R * c.S * c.C


def layer_report(name):
    rep = os.path.join(RUN, f"prof_{name}.ncu-rep")
    if not os.path.exists(rep):
        return None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
    d = {k: (v, scale.get(u, 1)) for k, u, v in zip(rr[0], rr[1], rr[2])}
    g = lambda k: next((v[0] for kk, v in d.items() if kk == k or kk.endswith("." + k) or kk.endswith(k)), "")
    sc = lambda k: next((v[1] for kk, v in d.items() if kk == k or kk.endswith("." + k) or kk.endswith(k)), 1)
    def num(k):
        try:
            return float(g(k).replace(",", "")) * sc(k)
        except ValueError:   # 'no data'
            return float("nan")
    t_us = num("gpu__time_duration.sum")
    cyc = num("sm__cycles_elapsed.avg")
    nmma = num("sm__inst_executed_pipe_tensor_subpipe_imma.sum")
    macs = LAYER_MACS[name]
    util = macs / (148 * cyc * MAC_PER_CLK_SM)
    dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    det = []
    for r in rows[1:]:
        dd = dict(zip(h, r))
        det.append(f"{dd.get('Section Name', '')[:34]:34s} {dd.get('Metric Name', '')[:48]:48s} "
                   f"{dd.get('Metric Value', '')} {dd.get('Metric Unit', '')}")
    plain = open(os.path.join(RUN, f"plain_{name}.log")).read().strip().splitlines()[-1]
    hdr = [f"ResNet-50 b256 {name}: ncu --set full --clock-control none --import-source on -k regex:qnn_gemm -s 3 -c 1",
           f"  python tools/bench_layers.py --suite resnet50 --batch 256 --only {name} --reps 3",
           f"kernel: {g('Kernel Name') or d.get('Kernel Name', '')}",
           f"live (no profiler, L2 flushed, CUDA events): {plain}", "",
           "Tensor-pipe evidence (this launch, ncu clocks):",
           f"  gpu__time_duration.sum                          {t_us:10.2f} us",
           f"  sm__cycles_elapsed.avg                          {cyc:10.0f} cycles/SM",
           f"  sm__inst_executed_pipe_tensor_subpipe_imma.sum  {nmma:10.0f} UTCIMMA (+ commits) warp instructions",
           f"  sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg {num('sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg'):10.0f}",
           f"  algorithmic MACs                                {macs:.4g}",
           f"  tensor utilisation = MACs / (148 SMs x cycles x {MAC_PER_CLK_SM} MAC/clk/SM) = {util:.3f}",
           f"  DRAM bytes {dram / 1e6:.1f} MB -> {dram / t_us / 1e3:.0f} GB/s",
           "  (the *_realtime cycle counters advance a fixed count per MMA instruction -- 256 per",
           "   128x256x32 in gemm_t, 512 per instruction in the pixel-major kernel -- on a clock that is",
           "   not the SM clock, so their pct_of_peak figure (round 1's '1.15%') is not a utilisation;",
           "   the MAC-based figure above is)", ""]
    open(os.path.join(OUT, f"r02_ncu_{name}.txt"), "w").write("\n".join(hdr + det) + "\n")
    return dict(layer=name, t_us=t_us, util=round(util, 3), dram_MB=round(dram / 1e6, 1), utcimma_inst=nmma,
                regs=g("launch__registers_per_thread"))


def main():
    L = load_launches(os.path.join(RUN, "launches.csv"))
    S = steps(L)
    stack = next(s for s in S if len(s) == 56)
    full = [s for s in S if len(s) > 56]
    cmd = "python bench.py --steps 2 --warmup 3 --no-cpu-baseline --breakdown-steps 1 --no-inception"
    note = (f"ncu launch list of `{cmd}` (--metrics gpu__time_duration.sum,dram__bytes_read.sum,"
            "dram__bytes_write.sum --clock-control none); cold-cache and serialised: compare SHARES, not absolutes.")
    l1, per_launch, ng = summarize_step(stack, "step", "conv stack step (the bench's `value`): " + note)
    lines = l1
    if full:
        l2, _, _ = summarize_step(full[-1], "full_network", "full-network step (`full_network`): " + note)
        lines += ["", ""] + l2
    open(os.path.join(OUT, "r02_launches_summary.txt"), "w").write("\n".join(lines) + "\n")
    json.dump({"batch": 256, "bytes_per_launch": per_launch, "launches": ng,
               "source": "profiles/r02_launches_step.csv (dram__bytes_read.sum + dram__bytes_write.sum, ncu)"},
              open(os.path.join(OUT, "gemm_traffic.json"), "w"), indent=1)
    print("\n".join(lines))
    layer_macs()
    res = [r for r in (layer_report(n) for n in ("layer1.0.conv2", "layer3.1.conv2", "layer1.0.conv3", "conv1")) if r]
    json.dump(res, open(os.path.join(OUT, "r02_tensor_pipe.json"), "w"), indent=1)
    for r in res:
        print(r)


if __name__ == "__main__":
    main()
