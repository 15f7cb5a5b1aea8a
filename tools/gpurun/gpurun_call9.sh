set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_fixed_point.py tests/test_lifting.py tests/test_mapped.py tests/test_gpu_sharded_fixed_point.py -m gpu -q -p no:cacheprovider > gpurun_out/gputest9.log 2>&1; tail -4 gpurun_out/gputest9.log; grep FAILED gpurun_out/gputest9.log | head
timeout 600 python tools/profile_cfg1.py > gpurun_out/cfg1_warm4.log 2>&1; head -3 gpurun_out/cfg1_warm4.log
