# usage: bash tools/gpu/quick.sh [tests] [c2] [c5] [c3] [c4]  -- quick GPU checks; outputs under gpurun_out/
mkdir -p gpurun_out
for a in "$@"; do
  case $a in
    tests) timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 ;;
    c2|c3|c4|c5)
      timeout 300 python bench.py --config $a --steps ${STEPS:-100} --warmup 10 --no-cpu-baseline \
        > gpurun_out/q_$a.json 2>gpurun_out/q_$a.err
      python -c "import json;d=json.load(open('gpurun_out/q_$a.json'));print('$a', round(d['ms_per_step']*1000,2),'us', '%.3g'%d['value'], 'frac', round(d['roofline']['frac'],4), 'clk', d['clocks']['sm_mhz'])" || tail -5 gpurun_out/q_$a.err ;;
  esac
done
