# usage: bash tools/gpu/variants.sh <config> "ENV=.. ENV2=.." "ENV=.." ...  -- bench one config under env variants
cfg=$1; shift
for v in "$@"; do
  env $v timeout 300 python bench.py --config $cfg --steps ${STEPS:-100} --warmup 10 --no-cpu-baseline > gpurun_out/v.json 2>gpurun_out/v.err
  python -c "import json;d=json.load(open('gpurun_out/v.json'));print('$cfg [$v]', round(d['ms_per_step']*1000,2),'us', 'frac', round(d['roofline']['frac'],4), 'clk', d['clocks']['sm_mhz'])" || tail -3 gpurun_out/v.err
done
