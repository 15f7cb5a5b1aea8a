L=paper_2311_17500_b200/lib/libmonoiga_b200.so
RX_STORE=0 timeout 900 python tools/time_reaction.py $L varlib/rx_p3only.so $L varlib/rx_p3only.so 2>&1 | grep op_reaction
