set -x
for v in default u4 u1; do
  if [ $v = default ]; then unset MP_LIB; else export MP_LIB=$PWD/paper_2210_12924_b200/lib/variants/$v.so; fi
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', d['ms_per_step'], d['roofline']['frac'], d['parity_rows']['ok'])"
done
unset MP_LIB
MP_SCORE_NO_PARTS=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('scratch', d['ms_per_step'], d['roofline']['frac'])"
