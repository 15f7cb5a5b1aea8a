timeout 900 python -m pytest tests/test_gpu_reaction_ws.py tests/test_gpu_parity.py tests/test_lifting.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
L=paper_2311_17500_b200/lib/libmonoiga_b200.so
RX_STORE=0 timeout 600 python tools/time_reaction.py $L 2>&1 | grep op_reaction
RX_NE=64 RX_NET=256 RX_STORE=0 timeout 600 python tools/time_reaction.py $L 2>&1 | grep op_reaction
RX_NE=64 RX_NET=128 RX_P=2 RX_STORE=1 timeout 600 python tools/time_reaction.py $L 2>&1 | grep op_reaction
RX_NE=64 RX_NET=128 RX_P=2 RX_STORE=0 timeout 600 python tools/time_reaction.py $L 2>&1 | grep op_reaction
RX_NE=48 RX_NET=96 RX_P=3 RX_STORE=1 timeout 600 python tools/time_reaction.py $L 2>&1 | grep op_reaction
