# usage: VARIANTS="old" bash tools/gpu/c5_ab.sh -- C5 parity subset, then the default bench line
# for the in-tree library and each lib/variants/<name>.so, alternating (no CPU leg)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "partitioned or c5 or wide or 24bit or large" 2>&1 | tail -2
for i in 1 2; do
  for v in cur $VARIANTS; do
    if [ $v = cur ]; then L=""; else L="paper_2210_12924_b200/lib/variants/$v.so"; fi
    MP_LIB=${L:-paper_2210_12924_b200/lib/libmemplan_b200.so} timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
    python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print('$v', round(d['ms_per_step']*1000,2),'us', '%.4g'%d['value'], 'frac', round(d['roofline']['frac'],4), 'clk', d['clocks']['sm_mhz'])" || tail -5 gpurun_out/ab_$v.err
  done
done
