#!/bin/bash
# A/B per-layer timing: default env (A) vs "$1" env assignment (B, e.g. QNN_NO_AROWS=1), interleaved twice
set -u
ENVB=$1; shift
mkdir -p gpurun_out
for r in 1 2; do
  python tools/bench_layers.py "$@" --json gpurun_out/ab_A$r.json > /dev/null 2>&1
  env $ENVB python tools/bench_layers.py "$@" --json gpurun_out/ab_B$r.json > /dev/null 2>&1
done
python - <<'PY'
import json
def load(f): return {x['name']: x['ms'] for x in json.load(open(f))}
A1, A2, B1, B2 = (load(f"gpurun_out/ab_{k}.json") for k in ("A1", "A2", "B1", "B2"))
ta = tb = 0
for k in A1:
    a = (A1[k] + A2[k]) / 2 * 1e3; b = (B1[k] + B2[k]) / 2 * 1e3
    ta += a; tb += b
    print(f"{k:40s} A {a:8.1f}  B {b:8.1f}  B/A {b / a:5.3f}")
print(f"{'TOTAL':40s} A {ta:8.1f}  B {tb:8.1f}  B/A {tb / ta:5.3f}")
PY
