set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest4.log 2>&1; tail -8 gpurun_out/gputest4.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"sub_reduce|dots_partial|dots_final|scale_div|comb" --csv --log-file gpurun_out/krylov_r02b.csv python tools/prof_krylov.py 24 > gpurun_out/ncu_krylov2.log 2>&1; tail -1 gpurun_out/ncu_krylov2.log
TV_REACTION=1 timeout 600 python tools/time_variants.py paper_2311_17500_b200/lib/libmonoiga_b200.so > gpurun_out/variants4.log 2>&1; cat gpurun_out/variants4.log
