# usage: bash tools/gpu/e2e_pack.sh <config>  -- e2e plans/s with and without the 16-bit order packing
cfg=${1:-c2}
for rep in 1 2; do
for v in "MP_NO_PACK16=1" "X=1"; do
  env $v timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/e.json 2>gpurun_out/e.err
  python -c "import json;d=json.load(open('gpurun_out/e.json'));e=d['e2e'];print('$cfg [$v]', '%.3g'%e['value'], 'plans/s', round(d['config']['candidates_per_gpu']/e['value']*1e3,3), 'ms/step; device', round(d['ms_per_step']*1e3,1), 'us')" || tail -3 gpurun_out/e.err
done
done
