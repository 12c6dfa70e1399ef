# Round-2 state check: gpu tests, default bench (C5 with cpu_baseline), reference arm, C2 line.
O=gpurun_out/st; mkdir -p $O
nproc > $O/nproc.txt; lscpu | grep -i "model name" >> $O/nproc.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; tail -3 $O/gpu_tests.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; cat $O/bench.json
timeout 600 python bench.py --impl reference > $O/ref.json 2> $O/ref.err; cat $O/ref.json
timeout 300 python bench.py --config c2 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err; cat $O/bench_c2.json
