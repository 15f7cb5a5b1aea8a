# bench + the profiles of the round: launch list, ncu --set full of the top kernels, Krylov, warm cfg-1 host profile
set -x
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; tail -c 400 gpurun_out/bench_r02b.json
timeout 600 python tools/profile_cfg1.py > gpurun_out/cfg1_warm.log 2>&1; head -40 gpurun_out/cfg1_warm.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --skip-extras > gpurun_out/ncu_launch.log 2>&1; tail -1 gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_dmma -s 2 -c 1 -o gpurun_out/sten_r02 -f python tools/prof_apply.py --iters 3 > gpurun_out/ncu_sten.log 2>&1; tail -1 gpurun_out/ncu_sten.log
timeout 900 ncu --set full --clock-control none -k regex:"time_filter|time_stage|mode_fold" -s 8 -c 8 -o gpurun_out/fd_r02 -f python tools/prof_apply.py --iters 3 > gpurun_out/ncu_fd.log 2>&1; tail -1 gpurun_out/ncu_fd.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"sub_reduce|dots_partial|dots_final|scale_div|comb" --csv --log-file gpurun_out/krylov_r02c.csv python tools/prof_krylov.py 24 > gpurun_out/ncu_krylov3.log 2>&1; tail -1 gpurun_out/ncu_krylov3.log
