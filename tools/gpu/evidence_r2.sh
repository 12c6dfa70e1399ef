# Round-2 evidence: smoke, GPU tests, bench lines (all modes), reference arm, launch list, ncu.
# usage: bash tools/gpu/evidence_r2.sh   (outputs under gpurun_out/ev2/)
O=${EV:-gpurun_out/ev2}; mkdir -p $O
nproc > $O/host.txt; lscpu | grep -i "model name" >> $O/host.txt; nvidia-smi -L >> $O/host.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1500 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1; tail -1 $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --impl reference > $O/ref_c5.json 2> $O/ref_c5.err
for c in c2 c3 c4; do timeout 600 python bench.py --config $c --steps 100 --warmup 10 > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 600 python bench.py --impl reference --config c2 > $O/ref_c2.json 2> $O/ref_c2.err
for c in c2 c3; do timeout 600 python bench.py --mode plan --config $c --steps 5 > $O/plan_$c.json 2> $O/plan_$c.err; done
timeout 900 python bench.py --mode plan --config c5 --steps 2 --warmup 3 > $O/plan_c5.json 2> $O/plan_c5.err
timeout 600 python tools/gpu/big_place.py > $O/big_place_c5.txt 2>&1
for c in c2 c3 c5; do timeout 600 python bench.py --mode pairs --config $c --steps 10 > $O/pairs_$c.json 2> $O/pairs_$c.err; done
for c in c2 c3 c4; do timeout 600 python bench.py --mode place --config $c --steps 5 --place-batch 2048 > $O/place_$c.json 2> $O/place_$c.err; done
for c in c2 c3 c4; do timeout 600 python bench.py --mode joint --config $c --steps 3 > $O/joint_$c.json 2> $O/joint_$c.err; done
for c in c2 c3 c4; do timeout 600 python bench.py --mode arena --config $c --steps 5 > $O/arena_$c.json 2> $O/arena_$c.err; done
for c in c2 c3; do timeout 600 python bench.py --mode lp --config $c --steps 3 > $O/lp_$c.json 2> $O/lp_$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c5.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv python bench.py --config c2 --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score -s 5 -c 1 -o $O/ncu_c5_score python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score -s 5 -c 1 -o $O/ncu_c2_score python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score -s 5 -c 1 -o $O/ncu_c4_score python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:count_sorted -s 2 -c 1 -o $O/ncu_c5_pairs_count python bench.py --mode pairs --config c5 --steps 2 > /dev/null 2>&1
ls -la $O
