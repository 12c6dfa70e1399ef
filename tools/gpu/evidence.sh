# Round evidence: smoke, bench lines (all modes), reference arm, launch list, ncu captures.
# usage: bash tools/gpu/evidence.sh   (outputs under gpurun_out/ev/)
set -x
O=gpurun_out/ev; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1; tail -1 $O/gpu_tests.log
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --impl reference > $O/ref_c2.json 2> $O/ref_c2.err
for c in c3 c4; do python bench.py --config $c --steps 50 --warmup 5 > $O/bench_$c.json 2> $O/bench_$c.err; done
python bench.py --config c5 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
for c in c2 c3 c5; do python bench.py --mode pairs --config $c --steps 10 > $O/pairs_$c.json 2> $O/pairs_$c.err; done
for c in c2 c3 c4; do python bench.py --mode place --config $c --steps 5 --place-batch 2048 > $O/place_$c.json 2> $O/place_$c.err; done
for c in c2 c3 c4; do python bench.py --mode joint --config $c --steps 3 > $O/joint_$c.json 2> $O/joint_$c.err; done
for c in c2 c3 c4; do python bench.py --mode arena --config $c --steps 5 > $O/arena_$c.json 2> $O/arena_$c.err; done
for c in c2 c3; do python bench.py --mode lp --config $c --steps 3 > $O/lp_$c.json 2> $O/lp_$c.err; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_c2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:score -s 5 -c 1 -o $O/ncu_c2_score python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:place -s 3 -c 1 -o $O/ncu_c2_place python bench.py --mode place --steps 1 --place-batch 2048 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:arena -s 0 -c 1 -o $O/ncu_c2_arena python bench.py --mode arena --steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:lp_write -s 1 -c 1 -o $O/ncu_c3_lp python bench.py --mode lp --config c3 --steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:score -s 5 -c 1 -o $O/ncu_c5_score python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la $O
