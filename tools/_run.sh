P=paper_2012_10026_b200
tools/ab.sh "--scale 26 --steps 3 --warmup 3" 2 nopf:RB_LIB=$P/lib_nopf.so pf:RB_LIB=$P/lib_pf.so pf2:RB_LIB=$P/lib_pf2.so
tools/ab.sh "--graph chunglu --scale 24 --steps 3 --warmup 3" 1 nopf:RB_LIB=$P/lib_nopf.so pf2:RB_LIB=$P/lib_pf2.so
