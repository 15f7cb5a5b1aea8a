set -x
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gputest50.log 2>&1; tail -4 gpurun_out/gputest50.log; grep -E "FAILED|ERROR" gpurun_out/gputest50.log | head
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench50.log 2> gpurun_out/bench50.err; tail -c 600 gpurun_out/bench50.log; tail -3 gpurun_out/bench50.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --skip-extras > gpurun_out/bench50_short.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches50.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --skip-extras > gpurun_out/ncu50.log 2>&1; tail -2 gpurun_out/ncu50.log
