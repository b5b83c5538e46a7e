#!/bin/bash
# A/B timing of library variants / env knobs on one box:
#   tools/ab.sh "<bench args>" rounds name:ENV=.. name2:ENV=..
# e.g. tools/ab.sh "--scale 26" 3 base:RB_LIB=paper_2012_10026_b200/lib_base.so new:
args=$1; rounds=$2; shift 2
for r in $(seq $rounds); do
  for v in "$@"; do
    name=${v%%:*}; envs=${v#*:}
    out=$(env $envs timeout 900 python bench.py $args --no-cpu-baseline --validate-roots 0 2>/dev/null)
    echo "$name $(echo "$out" | python -c 'import json,sys
d=json.loads(sys.stdin.read()); r=d["roofline"]["by_direction"]; n=d["config"]["roots"]
print("%.1f GTEPS %.1f us/root  TD %.1f BU %.1f us/root  frac TD %.3f BU %.3f  e2e %.1f" % (d["value"], d["ms_per_root_mean"]*1e3,
      r["top_down"]["seconds"]/n*1e6, r["bottom_up"]["seconds"]/n*1e6, r["top_down"]["frac"], r["bottom_up"]["frac"], d["e2e"]["value"]))')"
  done
done
