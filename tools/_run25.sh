python -m pytest tests/test_gpu_big.py tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -6
python tools/prof_fit.py c4 --reps 3 2>&1 | tail -1
python tools/prof_fit.py c2 --reps 3 2>&1 | tail -1
python tools/prof_fit.py c3 --reps 3 2>&1 | tail -1
