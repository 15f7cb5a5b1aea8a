set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "from_host or gmres_matches" > gpurun_out/gputest10.log 2>&1; tail -3 gpurun_out/gputest10.log
timeout 600 python tools/time_e2e.py > gpurun_out/e2e10.log 2>&1; cat gpurun_out/e2e10.log
