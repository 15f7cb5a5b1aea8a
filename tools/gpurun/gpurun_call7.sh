set -x
mkdir -p gpurun_out
timeout 600 python tools/time_variants.py paper_2311_17500_b200/lib/libmonoiga_b200.so varlib/sten_noprefetch.so varlib/sten_nonpersist.so > gpurun_out/variants7.log 2>&1; cat gpurun_out/variants7.log
timeout 600 python tools/time_krylov.py paper_2311_17500_b200/lib/libmonoiga_b200.so > gpurun_out/krylov7.log 2>&1; cat gpurun_out/krylov7.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:stencil_dmma -s 1 -c 1 --csv python tools/time_variants.py --one varlib/sten_noprefetch.so > gpurun_out/ncu_sten_nopf.csv 2>&1; grep -E "dram|duration" gpurun_out/ncu_sten_nopf.csv | tail -3
timeout 600 python tools/profile_cfg1.py > gpurun_out/cfg1_warm2.log 2>&1; head -30 gpurun_out/cfg1_warm2.log
