timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "partitioned or c5 or wide or 24bit" 2>&1 | tail -2
bash tools/gpu/quick.sh c5
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:score_parts -s 5 -c 1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "dram__|gpu__time" 
