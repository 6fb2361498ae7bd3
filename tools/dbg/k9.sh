python tools/apply_probe.py --rhs 64 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "block_rhs or multi_rhs or k9 or graph_replay" 2>&1 | tail -1
timeout 2000 python tools/shard_probe.py --config c4 --n-shards 8 --ranks 0 --steps 4 2>/dev/null | tail -1
