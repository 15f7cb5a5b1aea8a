set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_dmma -s 2 -c 1 -o gpurun_out/sten27 -f python tools/prof_apply.py --iters 3 > gpurun_out/sten27_ncu.log 2>&1; tail -3 gpurun_out/sten27_ncu.log
ncu -i gpurun_out/sten27.ncu-rep --page source --csv --print-source sass > gpurun_out/sten27_source.csv 2>/dev/null
ncu -i gpurun_out/sten27.ncu-rep --page raw --csv > gpurun_out/sten27_raw.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/sten27_source.csv 30
