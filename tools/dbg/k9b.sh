python tools/apply_probe.py --rhs 10 2>&1 | tail -1
PHM_K9_TWO_SIDED=2 python tools/apply_probe.py --rhs 64 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -q -p no:cacheprovider -x -k "block_rhs or multi_rhs or k9 or graph_replay or golden or clustered or amplitude" 2>&1 | tail -1
PHM_K9_TWO_SIDED=2 ncu --set full --import-source on --clock-control none -k regex:k_near_mrhs3 --launch-skip 2 -c 1 -o gpurun_out/r2/k9b_m10 -f python tools/apply_probe.py --rhs 10 --steps 2 > /dev/null 2>&1
python bench.py --config c5 --steps 4 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5', d['value'], d['kernels'].get('coupling'), d['kernels'].get('near_mrhs'))"
