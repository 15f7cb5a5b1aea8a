set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:time_stage_fused -s 1 -c 1 -o gpurun_out/ts28 -f python tools/prof_apply.py --iters 3 > gpurun_out/ts28_ncu.log 2>&1; tail -3 gpurun_out/ts28_ncu.log
ncu -i gpurun_out/ts28.ncu-rep --page source --csv --print-source sass > gpurun_out/ts28_source.csv 2>/dev/null
ncu -i gpurun_out/ts28.ncu-rep --page raw --csv > gpurun_out/ts28_raw.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/ts28_source.csv 30
