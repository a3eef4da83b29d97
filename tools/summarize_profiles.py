#!/usr/bin/env python
"""Summarise the round's ncu captures into profiles/ (committed evidence).

Inputs (gpurun_out/): launches.csv (ncu launch list of `bench.py --steps 2`),
prof_top.ncu-rep (ncu --set full of the top GEMM launch), bench_plain.log.
Outputs (profiles/): rNN_launches_step.csv (one step's kernels, cold-cache
serialised durations), rNN_launches_summary.txt (per-kernel share of the step),
rNN_top_kernel_ncu.txt, gemm_traffic.json (DRAM bytes per GEMM launch, read by
bench.py for roofline.traffic), rNN_bench.json.
"""
from __future__ import annotations

import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUN = os.path.join(ROOT, "gpurun_out")
OUT = os.path.join(ROOT, "profiles")


def load_launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    by_id = defaultdict(dict)
    for r in rows[hi + 1:]:
        d = dict(zip(h, r))
        if not d.get("ID"):
            continue
        k = int(d["ID"])
        by_id[k]["name"] = d["Kernel Name"]
        v = d["Metric Value"].replace(",", "")
        by_id[k][d["Metric Name"]] = float(v) if v else 0.0
    return [by_id[k] for k in sorted(by_id)]


def short(name):
    n = name.split("(")[0]
    for p in ("void ", "qnn::"):
        n = n.replace(p, "")
    return n[:60]


def main(rnd="r01"):
    os.makedirs(OUT, exist_ok=True)
    L = load_launches(os.path.join(RUN, "launches.csv"))
    # the last complete step: from the last quantize launch to the following dequantize
    isq = lambda n: "quantize" in n and "dequantize" not in n and "requantize" not in n
    qidx = [i for i, x in enumerate(L) if isq(x["name"])]
    step = None
    for qi in reversed(qidx):
        di = next((j for j in range(qi, len(L)) if "dequantize" in L[j]["name"]), None)
        if di is not None:
            step = L[qi:di + 1]
            break
    assert step, "no complete step found"
    with open(os.path.join(OUT, f"{rnd}_launches_step.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["idx", "kernel", "duration_ns", "dram_read_bytes", "dram_write_bytes"])
        for i, x in enumerate(step):
            w.writerow([i, short(x["name"]), int(x.get("gpu__time_duration.sum", 0)),
                        int(x.get("dram__bytes_read.sum", 0)), int(x.get("dram__bytes_write.sum", 0))])
    tot = sum(x.get("gpu__time_duration.sum", 0) for x in step)
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for x in step:
        a = agg[short(x["name"])]
        a[0] += 1
        a[1] += x.get("gpu__time_duration.sum", 0)
        a[2] += x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0)
    lines = [f"ncu launch list of `python bench.py --steps 2 --warmup 3 --no-cpu-baseline --breakdown-steps 1`",
             "(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none);",
             "one step = last quantize .. dequantize sequence; durations are cold-cache and serialised, so",
             "compare SHARES with the bench's live breakdown, not absolutes.", "",
             f"step launches: {len(step)}   summed kernel time: {tot / 1e3:.1f} us", "",
             f"{'kernel':62s} {'n':>4s} {'time_us':>10s} {'share':>7s} {'dram_MB':>9s}"]
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k:62s} {n:4d} {t / 1e3:10.1f} {t / tot:7.3f} {b / 1e6:9.1f}")
    gemm = [x for x in step if "qnn_gemm_i8_kernel" in x["name"] or "qnn_gemm_t_kernel" in x["name"]]
    per_launch = sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in gemm) / max(1, len(gemm))
    lines.append("")
    lines.append(f"GEMM launches: {len(gemm)}; mean DRAM traffic per launch {per_launch / 1e6:.2f} MB; "
                 f"GEMM share of step {sum(x.get('gpu__time_duration.sum', 0) for x in gemm) / tot:.3f}")
    open(os.path.join(OUT, f"{rnd}_launches_summary.txt"), "w").write("\n".join(lines) + "\n")
    json.dump({"batch": 256, "bytes_per_launch": per_launch, "launches": len(gemm),
               "source": f"profiles/{rnd}_launches_step.csv (dram__bytes_read.sum + dram__bytes_write.sum, ncu)"},
              open(os.path.join(OUT, "gemm_traffic.json"), "w"), indent=1)
    print("\n".join(lines))

    rep = os.path.join(RUN, "prof_top.ncu-rep")
    if os.path.exists(rep):
        out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        h = rows[0]
        keep = []
        for r in rows[1:]:
            d = dict(zip(h, r))
            keep.append(f"{d.get('Section Name', '')[:34]:34s} {d.get('Metric Name', '')[:48]:48s} "
                        f"{d.get('Metric Value', '')} {d.get('Metric Unit', '')}")
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rr = list(csv.reader(raw.splitlines()))
        d = dict(zip(rr[0], rr[2] if len(rr) > 2 else rr[1]))
        want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                "sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg",
                "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
        keep.append("")
        for k in want:
            for kk in d:
                if kk.endswith(k) or kk == k:
                    keep.append(f"raw {kk} = {d[kk]}")
        hdr = ["ncu --set full --clock-control none --import-source on -k regex:qnn_gemm -s 3 -c 1",
               "python tools/bench_layers.py --suite resnet50 --batch 256 --only layer1.0.conv3 --reps 3", ""]
        open(os.path.join(OUT, f"{rnd}_top_kernel_ncu.txt"), "w").write("\n".join(hdr + keep) + "\n")
    bp = os.path.join(RUN, "bench_plain.log")
    if os.path.exists(bp):
        line = [l for l in open(bp).read().splitlines() if l.startswith("{")][-1]
        json.dump(json.loads(line), open(os.path.join(OUT, f"{rnd}_bench.json"), "w"), indent=1)




def summarize_bw(rnd="r01"):
    """Depthwise / requantize / quantize / dequantize launches: ncu duration and DRAM bytes,
    matched in order to the bench_layers rows (algorithmic bytes from the layer shapes)."""
    import statistics as stt
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = peaks.get("hbm_gbs", 6552.3)
    lines = [f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
             f"dram__throughput.avg.pct_of_peak_sustained_elapsed (cold L2 per launch) of",
             "`tools/bench_layers.py --suite mobilenet --batch 128` and `--suite requant`;",
             "GB/s = ALGORITHMIC bytes (bench_layers row) / ncu duration; peak = measured HBM "
             f"{hbm:.0f} GB/s. DRAM bytes < algorithmic where the output is still in L2 at kernel end.", "",
             f"{'op':34s} {'kernel':28s} {'us':>8s} {'alg_MB':>8s} {'GB/s':>8s} {'frac':>6s} {'dram_MB':>8s}"]
    for csvf, logf, pick in (("bw_launches.csv", "bw_plain.log", lambda n: ".dw" in n),
                             ("rq_launches.csv", "rq_plain.log", lambda n: True)):
        pc, pl_ = os.path.join(RUN, csvf), os.path.join(RUN, logf)
        if not (os.path.exists(pc) and os.path.exists(pl_)):
            continue
        L = load_launches(pc)
        groups = []
        for x in L:
            key = short(x["name"])
            if groups and groups[-1][0] == key and len(groups[-1][1]) < 6:
                groups[-1][1].append(x)
            else:
                groups.append((key, [x]))
        rows = [json.loads(l) for l in open(pl_).read().splitlines() if l.startswith("{")]
        rows = [r for r in rows if pick(r["name"])]
        for (key, xs), r in zip(groups, rows):
            us = stt.median(x.get("gpu__time_duration.sum", 0) for x in xs) / 1e3
            dram = stt.median(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in xs)
            alg = r["gbs"] * r["ms"] * 1e6   # bytes
            gbs = alg / (us * 1e3) if us else 0.0
            lines.append(f"{r['name']:34s} {key[:28]:28s} {us:8.1f} {alg / 1e6:8.1f} {gbs:8.0f} {gbs / hbm:6.3f} "
                         f"{dram / 1e6:8.1f}")
    open(os.path.join(OUT, f"{rnd}_bandwidth_ops_ncu.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
    summarize_bw(sys.argv[1] if len(sys.argv) > 1 else "r01")
