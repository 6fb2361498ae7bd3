#!/usr/bin/env bash
# Runs bench.py for every configuration (C3 with the CPU baseline) and keeps
# the JSON lines under gpurun_out/ (run under gpurun from the repo root).
set -u
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/all_c3.json 2> gpurun_out/all_c3.err
for c in c1 c2 c5; do
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/all_$c.json 2> gpurun_out/all_$c.err
done
for f in gpurun_out/all_c*.json; do
  python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],2), round(d['e2e']['value'],2), round(d['roofline']['frac'],3), d['clocks'])"
done
