#!/bin/bash
# End-of-round check (run under gpurun): smoke(), the whole GPU suite, the default bench line,
# and the ncu launch list of the same bench command (profiles refresh).
set -u
OUT=gpurun_out/final
mkdir -p $OUT
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke OK')" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python -m pytest tests/ -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo "bench rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --breakdown-steps 1 --no-inception"
$CMD > $OUT/launch_cmd_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -c 2000 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1; echo "launches rc=$?"
