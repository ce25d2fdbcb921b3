python -m pytest tests/test_gpu_big.py -m gpu -x -q 2>&1 | tail -4
python tools/prof_fit.py c3 --reps 3 2>&1 | tail -1
FFCA_LIB=$PWD/paper_2101_08563_b200/libffca_x_noincr.so python tools/prof_fit.py c3 --reps 3 2>&1 | tail -1
