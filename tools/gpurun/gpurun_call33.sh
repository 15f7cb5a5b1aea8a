set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "to_host or from_host" 2>&1 | tail -3
timeout 900 python tools/time_e2e.py 2>&1 | tail -8
