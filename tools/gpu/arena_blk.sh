# usage: bash tools/gpu/arena_blk.sh <config>  -- K6 with the edge->block index off / on / automatic
cfg=${1:-c2}
for b in 0 1 auto; do
  if [ $b = auto ]; then unset MP_ARENA_BLK; else export MP_ARENA_BLK=$b; fi
  timeout 300 python bench.py --mode arena --config $cfg --steps 5 > gpurun_out/a.json 2>gpurun_out/a.err
  python -c "import json;d=json.load(open('gpurun_out/a.json'));print('$cfg blk=$b', '%.3g'%d['value'], d['unit'])" || tail -3 gpurun_out/a.err
done
unset MP_ARENA_BLK
