#!/bin/bash
# Per-level ncu evidence (verdict r1 item 3): one launch per level
# (RB_LEVELS_PER_LAUNCH=1) for one root, `ncu --set full` of every level's
# bfs_persistent launch.  Usage: tools/profile_levels.sh <name> <one_root args>
# Outputs gpurun_out/prof/levels_<name>.{txt,ncu-rep}.
set -u
name=$1; shift
O=gpurun_out/prof; mkdir -p $O
RB_LEVELS_PER_LAUNCH=1 timeout 600 python tools/one_root.py --no-warmup "$@" > $O/levels_$name.txt 2>&1 && \
RB_LEVELS_PER_LAUNCH=1 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:bfs_persistent \
  -o $O/levels_$name python tools/one_root.py --no-warmup "$@" > $O/levels_${name}_ncu.log 2>&1
echo "levels_$name=$?"
