# usage: bash tools/gpu/arena_var.sh <config> libs...  -- K6 throughput per tuning build (MP_LIB)
cfg=$1; shift
for lib in "$@"; do
  MP_LIB=$lib timeout 300 python bench.py --mode arena --config $cfg --steps 5 > gpurun_out/a.json 2>gpurun_out/a.err
  python -c "import json;d=json.load(open('gpurun_out/a.json'));print('$cfg $lib', '%.3g'%d['value'])" || tail -3 gpurun_out/a.err
done
