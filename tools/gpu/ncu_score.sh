# usage: bash tools/gpu/ncu_score.sh <config> <tag>   -- one ncu --set full capture of the fused scorer
cfg=${1:-c2}; tag=${2:-x}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score -s 5 -c 1 \
  -o gpurun_out/score_${cfg}_${tag} python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_${cfg}_${tag}.log 2>&1; tail -3 gpurun_out/ncu_${cfg}_${tag}.log
