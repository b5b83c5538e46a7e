#!/bin/bash
# Round-2 evidence: bench lines (+ the per-level data roofline.by_direction is
# computed from) for s26 / s22 / Chung-Lu 2^24, the ncu launch list (time +
# DRAM bytes per kernel, preprocessing included) of an s26 bench run, per-level
# `ncu --set full` captures (one launch per level) of an s26 root whose big
# level is bottom-up (index 25), one whose big level is a deferred top-down
# (index 7) and a Chung-Lu root, and one whole-kernel `--set full` capture.
set -u
O=gpurun_out/prof2
mkdir -p $O
timeout 900 python bench.py --steps 5 --warmup 3 --dump-levels $O/levels_s26.json > $O/bench_s26.json 2> $O/bench_s26.err; echo bench_s26=$?
timeout 900 python bench.py --scale 22 --steps 5 --warmup 3 --dump-levels $O/levels_s22.json > $O/bench_s22.json 2> $O/bench_s22.err; echo bench_s22=$?
timeout 900 python bench.py --graph chunglu --scale 24 --steps 5 --warmup 3 --dump-levels $O/levels_cl24.json > $O/bench_cl24.json 2> $O/bench_cl24.err; echo bench_cl24=$?
P="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --validate-roots 0 --profile-roots 2"
timeout 600 $P > /dev/null 2>&1 && timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -c 800 --csv --log-file $O/launches_s26.csv $P > $O/ncu_launch.log 2>&1; echo launches=$?
tools/profile_levels.sh s26_bu25 --scale 26 --index 25
tools/profile_levels.sh s26_td7 --scale 26 --index 7
tools/profile_levels.sh cl24_i0 --graph chunglu --scale 24 --index 0
F="python bench.py --profile-roots 1 --no-cpu-baseline --validate-roots 0"
timeout 600 $F > /dev/null 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k regex:bfs_persistent \
  -s 1 -c 1 -o $O/full_s26 $F > $O/ncu_full_s26.log 2>&1; echo full_s26=$?
