# usage: bash tools/gpu/place_ab.sh -- K5 parity (placement + plans), then the place bench at C2/C3/C4
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_placement.py tests/test_gpu_plans.py -x -q 2>&1 | tail -2
for c in c2 c3 c4; do
  timeout 600 python bench.py --mode place --config $c --steps 5 --no-cpu-baseline > gpurun_out/pab_$c.json 2> gpurun_out/pab_$c.err
  python -c "import json;d=json.load(open('gpurun_out/pab_$c.json'));print('$c', '%.4g'%d['value'], d['unit'], 'one', d.get('single_problem_ms'))" || tail -3 gpurun_out/pab_$c.err
done
