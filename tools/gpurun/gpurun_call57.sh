set -x
mkdir -p gpurun_out
RX_NET=24 RX_STORE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:reaction_ws -s 20 -c 1 -o gpurun_out/rx57 -f python tools/time_reaction.py --one paper_2311_17500_b200/lib/libmonoiga_b200.so > gpurun_out/rx57_ncu.log 2>&1; tail -2 gpurun_out/rx57_ncu.log
ncu -i gpurun_out/rx57.ncu-rep --page source --csv --print-source sass > gpurun_out/rx57_source.csv 2>/dev/null
ncu -i gpurun_out/rx57.ncu-rep --page raw --csv > gpurun_out/rx57_raw.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/rx57_source.csv 6
