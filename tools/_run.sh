P=paper_2012_10026_b200
RB_LIB=$P/lib_cn0.so python -m pytest tests/test_gpu_bfs.py -m gpu -x -q > gpurun_out/s6_pytest_cn.log 2>&1; tail -3 gpurun_out/s6_pytest_cn.log
tools/ab.sh "--scale 26 --steps 3 --warmup 3" 2 base:RB_LIB=$P/lib_base.so cnoff:RB_LIB=$P/lib_cnoff.so cn22:RB_LIB=$P/lib_cn22.so cn0:RB_LIB=$P/lib_cn0.so > gpurun_out/s6_ab3.txt 2>&1
cat gpurun_out/s6_ab3.txt
RB_LIB=$P/lib_cn0.so python tools/td_phases.py --scale 26 --index 23 56 > gpurun_out/s6_tdph_cn0.txt 2>&1
tools/ab.sh "--graph chunglu --scale 24 --steps 3 --warmup 3" 1 base:RB_LIB=$P/lib_base.so cnoff:RB_LIB=$P/lib_cnoff.so cn0:RB_LIB=$P/lib_cn0.so > gpurun_out/s6_ab3_cl.txt 2>&1
cat gpurun_out/s6_ab3_cl.txt
