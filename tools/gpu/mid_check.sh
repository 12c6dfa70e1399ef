# mid32 scorer (C4: 32-bit scan inputs, 64-bit sums) parity + A/B
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "model or cap or random_orders or edge_cases or host_scoring or device_scoring" 2>&1 | tail -3
bash tools/gpu/quick.sh c4
MP_SCORE_NO_MID=1 bash tools/gpu/quick.sh c4
