# usage: bash tools/gpu/multirank_check.sh -- the N>1 bench path (2 and 4 ranks) on a one-GPU box over gloo
for n in 2 4; do
  MP_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29500 + n)) bench.py --gpus $n --steps 20 --warmup 3 \
    --no-cpu-baseline > gpurun_out/mr_$n.json 2> gpurun_out/mr_$n.err
  echo "rc=$? n=$n"; tail -c 600 gpurun_out/mr_$n.json; tail -3 gpurun_out/mr_$n.err
  MP_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29600 + n)) bench.py --impl reference --gpus $n --steps 2 --warmup 1 \
    > gpurun_out/mrr_$n.json 2> gpurun_out/mrr_$n.err
  echo "ref rc=$? n=$n"; tail -c 300 gpurun_out/mrr_$n.json
done
# the row-sharded pair sweep / validation (K2/K4) at N = 2 over gloo
MP_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29701 bench.py --mode pairs --config c3 --gpus 2 --steps 5 \
  > gpurun_out/mrp_2.json 2> gpurun_out/mrp_2.err
echo "pairs rc=$?"; tail -c 400 gpurun_out/mrp_2.json; tail -3 gpurun_out/mrp_2.err
