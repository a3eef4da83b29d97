#!/bin/bash
# time layers under the QNN_GEMM_DEBUG knobs with the instrumented build (profiling only; outputs are
# garbage with knobs set): 2 no stores, 4 no A loads, 8 no MMAs, 16 no TMEM loads
export QNN_LIB=${QNN_LIB:-paper_2006_10226_b200/libqnn_instr.so}
for L in ${LAYERS:-layer1.0.conv3 layer1.0.conv2}; do
  for D in 0 2 4 8 16 18 6 14 30; do
    echo -n "$L dbg=$D "; QNN_GEMM_DEBUG=$D python tools/bench_layers.py --suite resnet50 --batch 256 --only $L --reps 20 2>&1 | tail -1
  done
done
