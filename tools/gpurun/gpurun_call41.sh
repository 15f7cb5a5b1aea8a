L=paper_2311_17500_b200/lib/libmonoiga_b200.so
RX_NE=64 RX_NET=128 RX_P=2 RX_STORE=0 timeout 600 python tools/time_reaction.py $L 2>&1 | grep op_reaction
RX_STORE=0 timeout 600 python tools/time_reaction.py $L 2>&1 | grep op_reaction
timeout 900 python tools/solve_cfg.py --cfg 3 2>&1 | tail -4 | cut -c1-600
