# Final C5 evidence: default bench line (with the reference on the host cores), reference arm,
# launch list and one ncu --set full capture of the scorer
O=gpurun_out/fin; mkdir -p $O
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --impl reference > $O/ref_c5.json 2> $O/ref_c5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c5.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score -s 5 -c 1 -o $O/ncu_c5_score python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls $O
