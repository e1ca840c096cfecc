python -m pytest tests -m gpu -q -x -k "compat" 2>&1 | tail -2
python tools/compat_bench.py --q 10000 100000 --reps 3
