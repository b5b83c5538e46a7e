P=paper_2012_10026_b200
RB_LIB=$P/lib_scanall.so python -m pytest tests/test_gpu_bfs.py tests/test_gpu_chunglu.py -m gpu -x -q > gpurun_out/s8_pytest_scanall.log 2>&1; tail -3 gpurun_out/s8_pytest_scanall.log
for v in scan; do
RB_LIB=$P/lib_$v.so python bench.py --steps 3 --warmup 3 --no-cpu-baseline --validate-roots 64 --dump-levels gpurun_out/s8_lv_s26_$v.json > gpurun_out/s8_b_s26_$v.json 2>&1
RB_LIB=$P/lib_$v.so python bench.py --graph chunglu --scale 24 --steps 3 --warmup 3 --no-cpu-baseline --validate-roots 64 --dump-levels gpurun_out/s8_lv_cl_$v.json > gpurun_out/s8_b_cl_$v.json 2>&1
done
python tools/level_classes.py gpurun_out/s8_lv_s26_scan.json gpurun_out/s8_lv_cl_scan.json
tools/ab.sh "--scale 26 --steps 3 --warmup 3" 1 noscan:RB_LIB=$P/lib_noscan.so scan:RB_LIB=$P/lib_scan.so
tools/ab.sh "--graph chunglu --scale 24 --steps 3 --warmup 3" 1 noscan:RB_LIB=$P/lib_noscan.so scan:RB_LIB=$P/lib_scan.so
tools/ab.sh "--scale 22 --steps 3 --warmup 3" 1 noscan:RB_LIB=$P/lib_noscan.so scan:RB_LIB=$P/lib_scan.so
