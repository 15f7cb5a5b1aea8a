L=paper_2311_17500_b200/lib/libmonoiga_b200.so
timeout 900 python -m pytest tests/test_gpu_reaction_ws.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
RX_NE=64 RX_NET=128 RX_P=2 RX_STORE=1 timeout 600 python tools/time_reaction.py $L varlib/st9.so 2>&1 | grep op_reaction
