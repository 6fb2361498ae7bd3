python tools/apply_probe.py 2>&1 | tail -1
python tools/apply_probe.py --rhs 10 2>&1 | tail -1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3', d['value'], d['mvm'])"
python bench.py --config c5 --steps 4 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5', d['value'], d['kernels'].get('coupling'), d['kernels'].get('near_mrhs'))"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "coupling or block_rhs or multi_rhs or h2_snapshot" 2>&1 | tail -1
