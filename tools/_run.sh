P=paper_2012_10026_b200
RB_LIB=$P/lib_spec.so python -m pytest tests/test_gpu_bfs.py -m gpu -x -q > gpurun_out/s14_pytest_spec.log 2>&1; tail -3 gpurun_out/s14_pytest_spec.log
tools/ab.sh "--scale 26 --steps 3 --warmup 3" 2 nospec:RB_LIB=$P/lib_nospec.so spec:RB_LIB=$P/lib_spec.so specbig:RB_LIB=$P/lib_specbig.so
tools/ab.sh "--graph chunglu --scale 24 --steps 3 --warmup 3" 1 nospec:RB_LIB=$P/lib_nospec.so spec:RB_LIB=$P/lib_spec.so specbig:RB_LIB=$P/lib_specbig.so
tools/ab.sh "--scale 22 --steps 3 --warmup 3" 2 nospec:RB_LIB=$P/lib_nospec.so spec:RB_LIB=$P/lib_spec.so specbig:RB_LIB=$P/lib_specbig.so
