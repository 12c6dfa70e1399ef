O=gpurun_out/ev; mkdir -p $O
for c in c3 c4; do python bench.py --config $c --steps 50 --warmup 5 > $O/bench_$c.json 2> $O/bench_$c.err; done
