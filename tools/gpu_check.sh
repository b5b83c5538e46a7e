#!/bin/bash
# quick GPU iteration: build must already succeed locally; run fast tests + level traces
timeout 900 python -m pytest tests -x -q -m "gpu and not slow" --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python tools/level_trace.py --roots 1 2>&1 | tail -9
timeout 300 python tools/level_trace.py --scale 26 --roots 1 2>&1 | tail -9
