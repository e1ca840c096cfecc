python -m pytest tests/test_compat_gpu.py tests/test_compat_sim_replay.py -q -x 2>&1 | tail -3
