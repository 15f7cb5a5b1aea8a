set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded_local.py tests/test_mapped.py -m gpu -q -p no:cacheprovider -x > gpurun_out/gputest26.log 2>&1; tail -3 gpurun_out/gputest26.log
timeout 900 python tools/time_variants.py paper_2311_17500_b200/lib/libmonoiga_b200.so varlib/sten_coupled.so 2>&1 | tail -4
TV_NE=64 TV_NET=128 TV_P=2 timeout 900 python tools/time_variants.py paper_2311_17500_b200/lib/libmonoiga_b200.so varlib/sten_coupled.so 2>&1 | tail -4
