# usage: VARIANTS="base" bash tools/gpu/arena_ab.sh -- K6 parity, then the arena bench (first
# fit) for the in-tree library and each lib/variants/<name>.so
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_arena.py tests/test_gpu_parity.py -x -q -k "arena or baseline or sink_counts" 2>&1 | tail -2
for c in c2 c3 c4; do
    for v in cur $VARIANTS; do
      if [ $v = cur ]; then L=paper_2210_12924_b200/lib/libmemplan_b200.so; else L=paper_2210_12924_b200/lib/variants/$v.so; fi
      MP_LIB=$L timeout 300 python bench.py --mode arena --config $c --steps 5 --no-cpu-baseline > gpurun_out/aab.json 2> gpurun_out/aab.err
      python -c "import json;d=json.load(open('gpurun_out/aab.json'));print('$c', '$v', round(d['ms_per_step'],3),'ms', '%.4g'%d['value'])" || tail -3 gpurun_out/aab.err
  done
done
