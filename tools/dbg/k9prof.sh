mkdir -p gpurun_out/r2
PHM_K9_TWO_SIDED=2 python tools/apply_probe.py --rhs 64 2>&1 | tail -1
for r in 10 64; do
PHM_K9_TWO_SIDED=2 ncu --set full --import-source on --clock-control none -k regex:k_near_mrhs3 --launch-skip 2 -c 1 -o gpurun_out/r2/k9_m$r -f python tools/apply_probe.py --rhs $r --steps 2 > gpurun_out/r2/ncu_k9_m$r.log 2>&1
done
echo done
