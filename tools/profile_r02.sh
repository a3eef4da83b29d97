#!/bin/bash
# Round-2 profiling (run under gpurun, one GPU): plain bench, the ncu launch list of the same
# command, and one ncu --set full capture (+ tensor-pipe counters) per named ResNet-50 b256 layer.
# Usage: tools/profile_r02.sh [layer ...]
set -u
OUT=gpurun_out/r02prof
mkdir -p $OUT
LAYERS=${@:-layer1.0.conv2 layer3.1.conv2 layer1.0.conv3 conv1}
TP=sm__ops_path_tensor_op_imma_src_int8.sum,sm__inst_executed_pipe_tensor_subpipe_imma.sum,sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg,sm__cycles_elapsed.avg,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --breakdown-steps 1 --no-inception"
$CMD > $OUT/launch_cmd_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 2000 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1; echo "launches rc=$?"
for L in $LAYERS; do
  python tools/bench_layers.py --suite resnet50 --batch 256 --only $L --reps 3 > $OUT/plain_$L.log 2>&1 || { echo "$L plain failed"; continue; }
  timeout 600 ncu --set full --metrics $TP --clock-control none --import-source on -k regex:qnn_gemm -s 3 -c 1 \
    -o $OUT/prof_$L -f python tools/bench_layers.py --suite resnet50 --batch 256 --only $L --reps 3 > $OUT/ncu_$L.log 2>&1
  echo "$L rc=$?"
done
