#!/usr/bin/env bash
# Profiles one bench configuration on the GPU box (run under gpurun from the
# repo root). Writes into gpurun_out/<tag>_*: the plain bench line (run first,
# without a profiler), the ncu launch list of the same command, and one
# `--set full` capture per listed kernel.
#   tools/profile_round.sh r01 c3 "k_near_tma k_coupling_mma k_class_inst"
set -euo pipefail
tag=${1:-r01}
cfg=${2:-c3}
kernels=${3:-"k_near_tma k_coupling_mma k_class_inst"}
out=gpurun_out
mkdir -p "$out"
python bench.py --config "$cfg" --steps 5 --warmup 3 > "$out/${tag}_${cfg}_bench.json" 2> "$out/${tag}_${cfg}_bench.err"
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$out/${tag}_${cfg}_launches.csv" \
  python bench.py --config "$cfg" --steps 3 --warmup 3 > "$out/${tag}_${cfg}_launches.log" 2>&1
for k in $kernels; do
  ncu --set full --import-source on --clock-control none -k "regex:${k}" -c 1 \
    -o "$out/${tag}_${cfg}_full_${k}" -f \
    python bench.py --config "$cfg" --steps 1 --warmup 3 > "$out/${tag}_${cfg}_full_${k}.log" 2>&1
done
echo done
