P=paper_2012_10026_b200
for n in librcmbfs_b200 lib_nopar lib_nored lib_probecg lib_noprobe; do
  echo "== $n"; RB_LIB=$P/$n.so python tools/td_phases.py --scale 26 --index 23 2>&1 | grep -A3 "L2 BT"
done > gpurun_out/s7_td_diag.txt 2>&1
cat gpurun_out/s7_td_diag.txt
