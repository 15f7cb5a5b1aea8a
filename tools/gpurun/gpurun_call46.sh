timeout 900 python -m pytest tests/test_mapped.py tests/test_theta.py tests/test_lowrank.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
python tools/prof_mapped_setup.py 2>&1 | cut -c1-150 | head -22
