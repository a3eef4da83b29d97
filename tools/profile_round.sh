#!/bin/bash
# Round profiling (run under gpurun): plain bench, ncu launch list of the same command, one
# ncu --set full capture of the top GEMM launch (a ResNet-50 b256 layer), and ncu DRAM
# counters for the bandwidth-bound ops (depthwise, requantize, quantize, dequantize).
set -u
OUT=gpurun_out
python bench.py --steps 20 --warmup 3 > $OUT/bench_plain.log 2>&1; echo "bench rc=$?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --breakdown-steps 1 > $OUT/bench_ncu_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 600 --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --breakdown-steps 1 \
  > $OUT/ncu_launches.log 2>&1; echo "launches rc=$?"
python tools/bench_layers.py --suite resnet50 --batch 256 --only layer1.0.conv3 --reps 3 > $OUT/top_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qnn_gemm -s 3 -c 1 -o $OUT/prof_top -f \
  python tools/bench_layers.py --suite resnet50 --batch 256 --only layer1.0.conv3 --reps 3 > $OUT/ncu_top.log 2>&1
echo "top rc=$?"
# bandwidth-bound ops: DRAM bytes and duration per launch (cache control all: cold L2)
python tools/bench_layers.py --suite mobilenet --batch 128 --reps 3 > $OUT/bw_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
  -k regex:"dw3_tma|depthwise|requantize|quantize|dequantize" --csv --log-file $OUT/bw_launches.csv \
  python tools/bench_layers.py --suite mobilenet --batch 128 --reps 3 > $OUT/ncu_bw.log 2>&1
python tools/bench_layers.py --suite requant --reps 3 > $OUT/rq_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
  -k regex:"requantize|quantize|dequantize" --csv --log-file $OUT/rq_launches.csv \
  python tools/bench_layers.py --suite requant --reps 3 > $OUT/ncu_rq.log 2>&1
echo "bw rc=$?"
