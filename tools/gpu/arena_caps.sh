# usage: bash tools/gpu/arena_caps.sh <config> caps...  -- K6 throughput vs the first-pass block-list capacity
cfg=$1; shift
for cap in "$@"; do
  MP_ARENA_CAP=$cap timeout 300 python bench.py --mode arena --config $cfg --steps 5 > gpurun_out/a.json 2>gpurun_out/a.err
  python -c "import json;d=json.load(open('gpurun_out/a.json'));print('$cfg cap=$cap', '%.3g'%d['value'], d['unit'], {k:v for k,v in d.items() if 'ms' in k})" || tail -3 gpurun_out/a.err
done
