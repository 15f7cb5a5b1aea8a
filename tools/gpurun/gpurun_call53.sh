timeout 900 python -m pytest tests/test_gpu_fold.py tests/test_gpu_parity.py tests/test_gpu_sharded_local.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 900 python tools/time_variants.py paper_2311_17500_b200/lib/libmonoiga_b200.so varlib/cg1.so varlib/cg2p4.so 2>&1 | grep apply
TV_NE=64 TV_NET=128 TV_P=2 timeout 900 python tools/time_variants.py paper_2311_17500_b200/lib/libmonoiga_b200.so varlib/cg1.so 2>&1 | grep apply
TV_NE=64 TV_NET=256 TV_P=3 timeout 900 python tools/time_variants.py paper_2311_17500_b200/lib/libmonoiga_b200.so varlib/cg1.so 2>&1 | grep apply
