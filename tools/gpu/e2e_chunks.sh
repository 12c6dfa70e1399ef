# usage: bash tools/gpu/e2e_chunks.sh <config> -- e2e plans/s of the host-buffer call vs MP_PIPE_CHUNKS
cfg=${1:-c2}
for rep in 1 2; do
for ch in 1 2 4 8; do
  MP_PIPE_CHUNKS=$ch timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/e.json 2>gpurun_out/e.err
  python -c "import json;d=json.load(open('gpurun_out/e.json'));e=d['e2e'];print('$cfg chunks=$ch', round(e['value']), 'plans/s', round(d['config']['candidates_per_gpu']/e['value']*1e3,3), 'ms/step; torch h2d', round(e['torch_pinned_h2d_gbs'],1), 'GB/s')" || tail -3 gpurun_out/e.err
done
done
