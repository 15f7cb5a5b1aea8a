# round-2 GPU check: smoke, GPU tests (without the full-size module), bench, ablation timing, ncu
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r02.log 2>&1; tail -2 gpurun_out/smoke_r02.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_fullsize.py > gpurun_out/gputest2.log 2>&1; tail -15 gpurun_out/gputest2.log
timeout 300 python tools/time_variants.py paper_2311_17500_b200/lib/libmonoiga_b200.so varlib/unfused.so > gpurun_out/variants2.log 2>&1; cat gpurun_out/variants2.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; tail -c 600 gpurun_out/bench_r02a.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --skip-extras > gpurun_out/ncu_launch.log 2>&1; tail -2 gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_dmma -s 2 -c 1 -o gpurun_out/sten_r02 -f python tools/prof_apply.py --iters 3 > gpurun_out/ncu_sten.log 2>&1; tail -2 gpurun_out/ncu_sten.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:reaction_tile -s 40 -c 1 -o gpurun_out/rx_r02 -f python tools/prof_apply.py --reaction --iters 2 > gpurun_out/ncu_rx.log 2>&1; tail -2 gpurun_out/ncu_rx.log
