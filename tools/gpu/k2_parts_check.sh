# K2 sorted-tile count + partitioned scorer checks, then the lines they feed
timeout 1200 python -m pytest tests -x -q -m gpu -k "pair or pinned or c5 or partitioned or large or wide or shard or lp or validation or golden or edge_cases or plans" 2>&1 | tail -3
bash tools/gpu/quick.sh c5
MP_PARTS_NO_DEFER=1 bash tools/gpu/quick.sh c5
for c in c3 c5; do timeout 600 python bench.py --mode pairs --config $c --steps 10 > gpurun_out/pairs_$c.json 2> gpurun_out/pairs_$c.err; python -c "import json;d=json.load(open('gpurun_out/pairs_$c.json'));print('$c pairs', d['pairs_ms'], 'ms', '%.3g'%d['value'], d['roofline']['frac'])" || tail -3 gpurun_out/pairs_$c.err; done
