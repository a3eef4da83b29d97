# run under gpurun: bench for each lib variant; prints value + per-layer json to gpurun_out
tag=$1; shift
for V in "$@"; do
  label=${V%%=*}; envs=${V#*=}
  env $envs python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_$label.json 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('gpurun_out/${tag}_$label.json') if l.startswith('{')][-1]); print('$label', d['value'], d['full_network']['value'], d['inception_v3']['value'])"
done
