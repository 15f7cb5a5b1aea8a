RX_NE=64 RX_NET=128 RX_P=2 RX_STORE=1 timeout 600 python tools/time_reaction.py varlib/npp1.so paper_2311_17500_b200/lib/libmonoiga_b200.so 2>&1 | grep op_reaction
RX_NE=48 RX_NET=96 RX_P=3 RX_STORE=1 timeout 600 python tools/time_reaction.py paper_2311_17500_b200/lib/libmonoiga_b200.so 2>&1 | grep op_reaction
timeout 900 python -m pytest tests/test_gpu_reaction_ws.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
