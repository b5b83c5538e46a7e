#!/bin/bash
# mean / hmean per-root device time over 64 roots (L2 flushed), Chung-Lu 2^$1 (default 24)
S=${1:-24}
timeout 600 python tools/level_trace.py --graph chunglu --scale $S --roots 64 --flush --brief 2>&1 | grep root | python3 -c "
import sys,re
t=[float(re.search(r': ([0-9.]+) us',l).group(1)) for l in sys.stdin]
print('n',len(t),'mean %.1f'%(sum(t)/len(t)),'max %.1f'%max(t),'hmean-time %.1f'%(len(t)/sum(1/x for x in t)))"
