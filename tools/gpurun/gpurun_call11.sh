set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gputest11.log 2>&1; tail -5 gpurun_out/gputest11.log; grep -E "FAILED|ERROR" gpurun_out/gputest11.log | head
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench11.log 2> gpurun_out/bench11.err; tail -c 6000 gpurun_out/bench11.log; tail -5 gpurun_out/bench11.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench11_ref.log 2>&1; tail -c 1500 gpurun_out/bench11_ref.log
