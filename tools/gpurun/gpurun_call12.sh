set -x
mkdir -p gpurun_out
# reaction kernel (fused mode) source-level profile at 96^3 x 24
RX_NET=24 RX_STORE=0 timeout 600 python tools/time_reaction.py paper_2311_17500_b200/lib/libmonoiga_b200.so > gpurun_out/rx12_time.log 2>&1; cat gpurun_out/rx12_time.log
RX_NET=24 RX_STORE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:reaction_tile -s 30 -c 1 -o gpurun_out/rx12 -f python tools/time_reaction.py --one paper_2311_17500_b200/lib/libmonoiga_b200.so > gpurun_out/rx12_ncu.log 2>&1; tail -3 gpurun_out/rx12_ncu.log
ncu -i gpurun_out/rx12.ncu-rep --page source --csv --print-source sass > gpurun_out/rx12_source.csv 2>/dev/null
ncu -i gpurun_out/rx12.ncu-rep --page raw --csv > gpurun_out/rx12_raw.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/rx12_source.csv 40
ls -la gpurun_out/rx12*
