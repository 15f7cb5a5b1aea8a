set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_lifting.py tests/test_mapped.py -m gpu -q -p no:cacheprovider -x > gpurun_out/gputest15.log 2>&1; tail -3 gpurun_out/gputest15.log
RX_STORE=0 timeout 900 python tools/time_reaction.py paper_2311_17500_b200/lib/libmonoiga_b200.so varlib/rxws_nounroll.so 2>&1 | grep op_reaction
RX_NE=64 RX_NET=256 RX_STORE=0 timeout 600 python tools/time_reaction.py paper_2311_17500_b200/lib/libmonoiga_b200.so 2>&1 | grep op_reaction
