RX_STORE=0 timeout 900 python tools/time_reaction.py varlib/rxskew600.so varlib/rxskew1200.so varlib/rxskew2000.so 2>&1 | grep op_reaction
