# Refresh the K6 lines + capture after an arena change (outputs under gpurun_out/ev/).
O=gpurun_out/ev; mkdir -p $O
python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1; tail -1 $O/gpu_tests.log
for c in c2 c3 c4; do python bench.py --mode arena --config $c --steps 5 > $O/arena_$c.json 2> $O/arena_$c.err; done
ncu --set full --clock-control none --import-source on -k regex:arena -s 0 -c 1 -o $O/ncu_c2_arena python bench.py --mode arena --steps 1 > /dev/null 2>&1
ls $O | wc -l
