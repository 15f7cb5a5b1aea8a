set -x
mkdir -p gpurun_out
(PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_fullsize.py 4 2 > gpurun_out/fullsize_gen.log 2>&1; cp tests/golden/fullsize_cfg4.npz tests/golden/fullsize_cfg2.npz gpurun_out/ 2>/dev/null) &
GEN=$!
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect tests/test_gpu_fullsize.py > gpurun_out/gputest1.log 2>&1
tail -3 gpurun_out/gputest1.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "cfg3 or 3]" > gpurun_out/gputest_fs3.log 2>&1
tail -3 gpurun_out/gputest_fs3.log
wait $GEN
tail -5 gpurun_out/fullsize_gen.log
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider > gpurun_out/gputest_fs.log 2>&1
tail -5 gpurun_out/gputest_fs.log
timeout 2400 python tools/ref_cpu.py > gpurun_out/ref_cpu.log 2>&1; cp profiles/r02_ref_cpu.json gpurun_out/ 2>/dev/null
tail -3 gpurun_out/ref_cpu.log
