# reaction pipeline check: correctness (variant B tests), timing vs the serial schedule, cfg-1 profile
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_lifting.py tests/test_gpu_sharded_local.py tests/test_fixed_point.py tests/test_mapped.py -m gpu -q -p no:cacheprovider > gpurun_out/gputest3.log 2>&1; tail -5 gpurun_out/gputest3.log
TV_REACTION=1 timeout 600 python tools/time_variants.py paper_2311_17500_b200/lib/libmonoiga_b200.so varlib/rx_serial.so varlib/rx_nobal.so > gpurun_out/variants3.log 2>&1; cat gpurun_out/variants3.log
TV_REACTION=1 TV_NE=64 TV_NET=256 timeout 600 python tools/time_variants.py paper_2311_17500_b200/lib/libmonoiga_b200.so varlib/rx_serial.so >> gpurun_out/variants3.log 2>&1; tail -2 gpurun_out/variants3.log
RX_STORE=1 RX_NE=64 RX_NET=128 RX_P=2 timeout 600 python tools/time_reaction.py paper_2311_17500_b200/lib/libmonoiga_b200.so varlib/rx_serial.so >> gpurun_out/variants3.log 2>&1; tail -2 gpurun_out/variants3.log
timeout 300 python -m cProfile -o gpurun_out/cfg1.prof tools/solve_cfg.py --cfg 1 > gpurun_out/cfg1.log 2>&1; tail -1 gpurun_out/cfg1.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"sub_reduce|dots_partial|dots_final|scale_div|comb" --csv --log-file gpurun_out/krylov_r02.csv python tools/prof_krylov.py 24 > gpurun_out/ncu_krylov.log 2>&1; tail -2 gpurun_out/ncu_krylov.log
