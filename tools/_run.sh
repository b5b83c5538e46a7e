python -m pytest tests/test_gpu_bfs.py tests/test_gpu_configs.py -m gpu -x -q > gpurun_out/s12_pytest.log 2>&1; tail -3 gpurun_out/s12_pytest.log
