set -x
mkdir -p gpurun_out
timeout 600 python tools/time_variants.py paper_2311_17500_b200/lib/libmonoiga_b200.so varlib/sten_nonpersist.so > gpurun_out/variants5.log 2>&1; cat gpurun_out/variants5.log
timeout 600 python tools/time_krylov.py paper_2311_17500_b200/lib/libmonoiga_b200.so varlib/kb592_ku1.so varlib/kb296_ku1.so varlib/kb592_ku2.so varlib/kb296_ku4.so > gpurun_out/krylov5.log 2>&1; cat gpurun_out/krylov5.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gputest5.log 2>&1; tail -4 gpurun_out/gputest5.log
