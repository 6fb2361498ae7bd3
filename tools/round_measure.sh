#!/usr/bin/env bash
# One GPU session of round measurements (run under gpurun from the repo root):
# the GPU test suite (with the parity report), every bench configuration,
# the reference arm, the launch list and ncu --set full captures of the top
# kernels of the C3 step and of the standalone MVM. Outputs in gpurun_out/<tag>/.
set -u
tag=${1:-r02}
out=gpurun_out/$tag
mkdir -p $out
PHM_PARITY_REPORT=$out/parity_vs_reference.json timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/gputest.log 2>&1
echo "gpu tests rc=$?"; tail -2 $out/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; tail -1 $out/smoke.log
python bench.py --steps 20 --warmup 5 > $out/bench_c3.json 2> $out/bench_c3.err
for c in c1 c2 c5; do
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_$c.json 2> $out/bench_$c.err
done
python bench.py --impl reference --steps 20 --warmup 5 > $out/ref_c3.json 2> $out/ref_c3.err
for f in $out/bench_c*.json $out/ref_c3.json; do
  python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],3), d.get('e2e',{}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('mvm') or {}).get('frac_of_hbm'), (d.get('clocks') or {}).get('reasons'))"
done
python tools/apply_probe.py > $out/apply_probe.json 2>&1
python tools/apply_probe.py --rhs 10 > $out/apply_probe_m10.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/c3_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $out/c3_launches.log 2>&1
for k in k_near_tma k_coupling_mma k_class_inst_pf; do
  ncu --set full --import-source on --clock-control none -k "regex:${k}\b" -c 1 -o $out/c3_full_$k -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $out/c3_full_$k.log 2>&1
done
for k in k_near_gemv_lean k_coupling_mma; do
  ncu --set full --import-source on --clock-control none -k "regex:${k}\b" --launch-skip 3 -c 1 -o $out/apply_full_$k -f \
    python tools/apply_probe.py --steps 2 > $out/apply_full_$k.log 2>&1
done
for k in k_near_mrhs3 k_coupling_mma; do
  ncu --set full --import-source on --clock-control none -k "regex:${k}\b" --launch-skip 3 -c 1 -o $out/apply_m10_full_$k -f \
    python tools/apply_probe.py --rhs 10 --steps 2 > $out/apply_m10_full_$k.log 2>&1
done
# keep what comes back under gpurun's 64 MiB: summaries of every capture, the
# captures themselves only when small
for r in $out/*.ncu-rep; do
  python profiles/summarize_full.py $r > ${r%.ncu-rep}_summary.txt 2>&1
  ncu -i $r --page source --csv --print-source sass > ${r%.ncu-rep}_sass.csv 2>/dev/null
  python - "${r%.ncu-rep}_sass.csv" > ${r%.ncu-rep}_hot.txt <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
i = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[i]) for r in data if r[i].isdigit())
print("warp stall samples", tot)
for r in sorted(data, key=lambda r: -int(r[i]) if r[i].isdigit() else 0)[:25]:
    print(r[i], r[0][-6:], r[1].strip()[:90])
PY
  rm -f ${r%.ncu-rep}_sass.csv
  [ $(stat -c %s $r) -gt 6000000 ] && rm -f $r
done
# per-rank cost of the sharded step (C3 at 2/4/8 shards; C4 rank 0 of 8)
timeout 900 python tools/shard_probe.py --n-shards 2 4 8 --ranks 0 -1 > $out/shard_probe_c3.txt 2>&1
timeout 1500 python tools/shard_probe.py --config c4 --n-shards 8 --ranks 0 --steps 5 > $out/shard_probe_c4.txt 2>&1
du -sh $out
echo done
