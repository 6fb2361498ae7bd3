mkdir -p gpurun_out/r2
ncu --set full --import-source on --clock-control none -k regex:k_coupling_mma --launch-skip 3 -c 1 -o gpurun_out/r2/apply_coupling2 -f python tools/apply_probe.py --steps 2 > gpurun_out/r2/ncu_apply_coupling2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_coupling_mma --launch-skip 3 -c 1 -o gpurun_out/r2/apply_coupling2_m10 -f python tools/apply_probe.py --rhs 10 --steps 2 > gpurun_out/r2/ncu_apply_coupling2_m10.log 2>&1
echo done
