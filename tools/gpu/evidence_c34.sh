# ncu captures of the scorer at C3/C4 (for roofline.traffic), then their bench lines.
O=gpurun_out/ev; mkdir -p $O
for c in c3 c4; do
  ncu --set full --clock-control none --import-source on -k regex:score -s 5 -c 1 -o $O/ncu_${c}_score python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
ls $O/*.ncu-rep
