#!/bin/bash
# Per-layer timing of alternative in-tree builds / env knobs (run under gpurun):
#   tools/ab_variants.sh "<layer> ..." "<label>=<env assignments>" ...
# e.g. tools/ab_variants.sh "layer1.0.conv3" "new=" "old=QNN_LIB=paper_2006_10226_b200/libqnn_old.so"
set -u
LAYERS=$1; shift
for L in $LAYERS; do
  for V in "$@"; do
    label=${V%%=*}; envs=${V#*=}
    ms=$(env $envs python tools/bench_layers.py --suite resnet50 --batch ${BATCH:-256} --only $L --reps ${REPS:-20} 2>/dev/null \
         | python -c "import sys,json; print(' '.join(str(json.loads(l)['ms']) for l in sys.stdin if l.startswith('{')))")
    echo "$L $label $ms"
  done
done
