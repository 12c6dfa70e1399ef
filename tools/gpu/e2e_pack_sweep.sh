# usage: bash tools/gpu/e2e_pack_sweep.sh <config> "ENV ..." ...  -- e2e plans/s per env variant
cfg=$1; shift
nproc; 
for v in "$@"; do
  env $v timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 100 > gpurun_out/e.json 2>gpurun_out/e.err
  python -c "import json;d=json.load(open('gpurun_out/e.json'));e=d['e2e'];print('$cfg [$v]', '%.3g'%e['value'], round(d['config']['candidates_per_gpu']/e['value']*1e3,3), 'ms/step')" || tail -3 gpurun_out/e.err
done
