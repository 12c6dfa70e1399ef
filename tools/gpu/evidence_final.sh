# Final evidence after the last scorer change: smoke, GPU tests, default bench line (C5, with the
# reference on the host cores), the reference arm, C2-C4 lines, C5 launch list and ncu capture.
# usage: bash tools/gpu/evidence_final.sh   (outputs under gpurun_out/evf/)
O=${EV:-gpurun_out/evf}; mkdir -p $O
nproc > $O/host.txt; lscpu | grep -i "model name" >> $O/host.txt; nvidia-smi -L >> $O/host.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1500 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1; tail -1 $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --impl reference > $O/ref_c5.json 2> $O/ref_c5.err
for c in c2 c3 c4; do timeout 600 python bench.py --config $c --steps 100 --warmup 10 > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c5.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score -s 5 -c 1 -o $O/ncu_c5_score python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la $O
