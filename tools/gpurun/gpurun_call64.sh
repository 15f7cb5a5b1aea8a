timeout 900 python tools/time_variants.py paper_2311_17500_b200/lib/libmonoiga_b200.so varlib/tsabl1.so varlib/tsabl2.so 2>&1 | grep apply
