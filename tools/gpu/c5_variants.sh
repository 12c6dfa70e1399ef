# C5 scorer A/B: default vs MP_PARTS_NO_DEFER, plus the parts parity tests
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "large or partitioned or c5 or wide or stamp or 24bit" 2>&1 | tail -3
bash tools/gpu/quick.sh c5
MP_PARTS_NO_DEFER=1 bash tools/gpu/quick.sh c5
