# C2/C3 register-slot scorer variants (tools/build_variants.py sn/sn6/sn4: node records in smem)
for v in default sn sn6 sn4; do
  if [ $v = default ]; then unset MP_LIB; else export MP_LIB=$PWD/paper_2210_12924_b200/lib/variants/$v.so; fi
  for c in c2 c3; do
    timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v $c', round(d['ms_per_step']*1000,2), round(d['roofline']['frac'],4), d['parity_rows']['ok'])"
  done
done
