# usage: bash tools/gpu/place_quick.sh  -- K5 throughput at C2/C3/C4
for c in c2 c3 c4; do
  timeout 300 python bench.py --mode place --config $c --steps 3 --place-batch 2048 > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "import json;d=json.load(open('gpurun_out/p.json'));print('$c', '%.3g'%d['value'], d['unit'], 'single ms %.2f'%d['single_problem_ms'])" || tail -3 gpurun_out/p.err
done
