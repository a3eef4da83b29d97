#!/bin/bash
# time layers under the QNN_GEMM_DEBUG knobs (profiling only; outputs are garbage with knobs set)
for L in layer1.0.conv3 layer1.0.conv2 layer1.0.conv1 layer3.1.conv2; do
  for D in 0 1 2 3 4 8 16 19 23 31; do
    echo -n "$L dbg=$D "; QNN_GEMM_DEBUG=$D python tools/bench_layers.py --suite resnet50 --batch 256 --only $L --reps 5 2>&1 | tail -1
  done
done
