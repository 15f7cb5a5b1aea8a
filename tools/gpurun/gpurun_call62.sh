RX_STORE=0 timeout 900 python tools/time_reaction.py paper_2311_17500_b200/lib/libmonoiga_b200.so varlib/rc216.so varlib/rc224.so 2>&1 | grep op_reaction
