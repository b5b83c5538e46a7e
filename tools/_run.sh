python -m pytest tests/test_gpu_bfs.py -m gpu -x -q -k "sequential or modes or dispatch or small" > gpurun_out/s9_pytest_seq.log 2>&1; tail -15 gpurun_out/s9_pytest_seq.log
