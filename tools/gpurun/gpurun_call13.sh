set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_lifting.py tests/test_gpu_sharded_local.py tests/test_mapped.py -m gpu -q -p no:cacheprovider -x > gpurun_out/gputest13.log 2>&1; tail -5 gpurun_out/gputest13.log
for ws in 0 1; do
MI_RX_WS=$ws RX_STORE=0 timeout 600 python tools/time_reaction.py paper_2311_17500_b200/lib/libmonoiga_b200.so 2>&1 | tail -2
done
MI_RX_WS=1 RX_NE=64 RX_NET=256 RX_STORE=0 timeout 600 python tools/time_reaction.py paper_2311_17500_b200/lib/libmonoiga_b200.so 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -x -k "cfg4 or cfg5" > gpurun_out/gputest13b.log 2>&1; tail -5 gpurun_out/gputest13b.log
