mkdir -p gpurun_out/r2
python tools/apply_probe.py > gpurun_out/r2/apply_probe.json 2>&1; tail -1 gpurun_out/r2/apply_probe.json
PHM_APPLY_OVERLAP=0 python tools/apply_probe.py > gpurun_out/r2/apply_probe_serial.json 2>&1; tail -1 gpurun_out/r2/apply_probe_serial.json
ncu --set full --import-source on --clock-control none -k regex:k_coupling_mma --launch-skip 3 -c 1 -o gpurun_out/r2/apply_coupling -f python tools/apply_probe.py --steps 2 > gpurun_out/r2/ncu_apply_coupling.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_near_tma_apply --launch-skip 3 -c 1 -o gpurun_out/r2/apply_near -f python tools/apply_probe.py --steps 2 > gpurun_out/r2/ncu_apply_near.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/apply_launches.csv python tools/apply_probe.py --steps 3 > /dev/null 2>&1
echo done
