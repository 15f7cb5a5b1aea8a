set -x
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gputest24.log 2>&1; tail -5 gpurun_out/gputest24.log; grep -E "FAILED|ERROR" gpurun_out/gputest24.log | head
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench24.log 2> gpurun_out/bench24.err; tail -c 1500 gpurun_out/bench24.log; tail -5 gpurun_out/bench24.err
