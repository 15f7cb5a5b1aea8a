set -x
mkdir -p gpurun_out
RX_NE=64 RX_NET=128 RX_P=2 RX_STORE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:reaction_ws -s 30 -c 1 -o gpurun_out/rx56 -f python tools/time_reaction.py --one paper_2311_17500_b200/lib/libmonoiga_b200.so > gpurun_out/rx56_ncu.log 2>&1; tail -2 gpurun_out/rx56_ncu.log
ncu -i gpurun_out/rx56.ncu-rep --page source --csv --print-source sass > gpurun_out/rx56_source.csv 2>/dev/null
ncu -i gpurun_out/rx56.ncu-rep --page raw --csv > gpurun_out/rx56_raw.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/rx56_source.csv 14
