P=paper_2012_10026_b200
for v in notail tail; do for i in 0 23; do echo "== $v $i"; RB_LIB=$P/lib_$v.so python tools/one_root.py --scale 26 --index $i 2>&1 | tail -10; done; done
