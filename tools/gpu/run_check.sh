set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b_c2.json 2>gpurun_out/b_c2.err; tail -2 gpurun_out/b_c2.err; cat gpurun_out/b_c2.json
timeout 300 python bench.py --config c5 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b_c5.json 2>gpurun_out/b_c5.err; tail -2 gpurun_out/b_c5.err; cat gpurun_out/b_c5.json
