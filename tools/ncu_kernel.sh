#!/usr/bin/env bash
# One ncu --set full capture of one kernel of a command, reduced to a summary
# row and a SASS hot-spot list (run under gpurun from the repo root).
#   tools/ncu_kernel.sh <out_prefix> <kernel_regex> <launch_skip> -- <command...>
set -u
pre=$1; k=$2; skip=$3; shift 4
mkdir -p "$(dirname "$pre")"
ncu --set full --import-source on --clock-control none -k "regex:${k}" --launch-skip "$skip" -c 1 -o "$pre" -f "$@" > "$pre.log" 2>&1
python profiles/summarize_full.py "$pre.ncu-rep" > "${pre}_summary.txt" 2>&1
ncu -i "$pre.ncu-rep" --page details --csv > "${pre}_details.csv" 2>/dev/null
ncu -i "$pre.ncu-rep" --page source --csv --print-source sass > "${pre}_sass.csv" 2>/dev/null
python - "${pre}_sass.csv" > "${pre}_hot.txt" <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1] if "Warp Stall Sampling (All Samples)" in rows[1] else rows[0]
data = rows[rows.index(hdr) + 1:]
i = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[i]) for r in data if r[i].isdigit())
print("warp stall samples", tot)
for r in sorted(data, key=lambda r: -int(r[i]) if r[i].isdigit() else 0)[:40]:
    print(r[i], r[0][-6:], r[1].strip()[:100])
PY
rm -f "${pre}_sass.csv"
[ "$(stat -c %s "$pre.ncu-rep")" -gt 8000000 ] && rm -f "$pre.ncu-rep"
exit 0
