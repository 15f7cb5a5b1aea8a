set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded_local.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 900 python tools/time_variants.py paper_2311_17500_b200/lib/libmonoiga_b200.so varlib/noz.so 2>&1 | grep apply
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:stencil_dmma -s 2 -c 1 python tools/prof_apply.py --iters 3 2>&1 | grep -E "dram__|gpu__time" 
