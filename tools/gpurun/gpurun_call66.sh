set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:time_filter_dmma -s 1 -c 1 -o gpurun_out/tf66 -f python tools/prof_apply.py --iters 3 > gpurun_out/tf66_ncu.log 2>&1; tail -2 gpurun_out/tf66_ncu.log
ncu -i gpurun_out/tf66.ncu-rep --page source --csv --print-source sass > gpurun_out/tf66_source.csv 2>/dev/null
ncu -i gpurun_out/tf66.ncu-rep --page raw --csv > gpurun_out/tf66_raw.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/tf66_source.csv 14
