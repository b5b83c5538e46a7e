#!/bin/bash
# A/B timing of library variants on one box: ab.sh "<bench args>" rounds name=ENV... 
# e.g. tools/ab.sh "--scale 26" 3 base:RB_LIB=paper_2012_10026_b200/lib_base.so new:
args=$1; rounds=$2; shift 2
for r in $(seq $rounds); do
  for v in "$@"; do
    name=${v%%:*}; envs=${v#*:}
    out=$(env $envs timeout 600 python bench.py $args --no-cpu-baseline --validate-roots 0 2>/dev/null)
    echo "$name $(echo "$out" | python -c 'import json,sys;d=json.loads(sys.stdin.read());r=d["roofline"]["by_direction"];print("%.1f GTEPS %.1f us  TD %.1f us BU %.1f us" % (d["value"], d["ms_per_step"]*1e3, r["top_down"]["seconds"]/d["steps"]*1e6, r["bottom_up"]["seconds"]/d["steps"]*1e6))')"
  done
done
