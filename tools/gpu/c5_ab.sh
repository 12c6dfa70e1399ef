# usage: bash tools/gpu/c5_ab.sh -- C5 parity subset, then the default bench line twice (no CPU leg)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "partitioned or c5 or wide or 24bit or large" 2>&1 | tail -2
for i in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab_$i.json 2> gpurun_out/ab_$i.err
  python -c "import json;d=json.load(open('gpurun_out/ab_$i.json'));print('c5', round(d['ms_per_step']*1000,2),'us', '%.4g'%d['value'], 'frac', round(d['roofline']['frac'],4), 'kern_us', d['roofline'].get('kernel_us'), 'clk', d['clocks']['sm_mhz'])" || tail -5 gpurun_out/ab_$i.err
done
