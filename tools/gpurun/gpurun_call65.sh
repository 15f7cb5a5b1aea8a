timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded_local.py tests/test_lifting.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -6
timeout 900 python tools/time_variants.py paper_2311_17500_b200/lib/libmonoiga_b200.so varlib/nofuse.so 2>&1 | grep apply
TV_NE=64 TV_NET=128 TV_P=2 timeout 900 python tools/time_variants.py paper_2311_17500_b200/lib/libmonoiga_b200.so varlib/nofuse.so 2>&1 | grep apply
