# K2 sorted-count test + kPartsU variants of the C5 scorer (tools/build_variants.py u2/u8)
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "sorted_tile" 2>&1 | tail -3
for v in default u2 u8 pf; do
  if [ $v = default ]; then unset MP_LIB; else export MP_LIB=$PWD/paper_2210_12924_b200/lib/variants/$v.so; fi
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', d['ms_per_step'], d['roofline']['frac'], d['parity_rows']['ok'])"
done
