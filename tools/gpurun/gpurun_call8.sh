set -x
mkdir -p gpurun_out
timeout 600 python tools/profile_cfg1.py > gpurun_out/cfg1_warm3.log 2>&1; head -12 gpurun_out/cfg1_warm3.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest8.log 2>&1; tail -4 gpurun_out/gputest8.log; grep -E "FAILED|Error" gpurun_out/gputest8.log | head
timeout 300 python tools/time_krylov.py paper_2311_17500_b200/lib/libmonoiga_b200.so > gpurun_out/krylov8.log 2>&1; cat gpurun_out/krylov8.log
