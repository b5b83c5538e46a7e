#!/bin/bash
# Round-2 evidence: bench lines (+ the per-level data roofline.by_direction is
# computed from) for s26 / s22 / Chung-Lu 2^24, the ncu launch list (time +
# DRAM bytes per kernel, preprocessing included) of an s26 bench run, per-level
# `ncu --set full` captures (one launch per level) of an s26 root whose big
# level is bottom-up (index 25), one whose big level is a deferred top-down
# (index 7) and a Chung-Lu root, and one whole-kernel `--set full` capture.
# Reports are summarised on the box (JSON / CSV) and deleted: gpurun returns
# at most 64 MiB.   usage: tools/profile_round2.sh [benches|launches|levels|full]...
set -u
O=gpurun_out/prof2
mkdir -p $O
summ() {  # rep name command
  python tools/ncu_summary.py full "$1.ncu-rep" "$3" "$2" > "$1.json" 2> /dev/null
  ncu -i "$1.ncu-rep" --page raw --csv > "$1_raw.csv" 2> /dev/null
  ncu -i "$1.ncu-rep" --page source --csv --print-source cuda > "$1_source.csv" 2> /dev/null
  gzip -f "$1_raw.csv" "$1_source.csv"
  rm -f "$1.ncu-rep"
}
for what in "$@"; do
case $what in
benches)
timeout 900 python bench.py --steps 5 --warmup 3 --dump-levels $O/levels_s26.json > $O/bench_s26.json 2> $O/bench_s26.err; echo bench_s26=$?
timeout 900 python bench.py --scale 22 --steps 5 --warmup 3 --dump-levels $O/levels_s22.json > $O/bench_s22.json 2> $O/bench_s22.err; echo bench_s22=$?
timeout 900 python bench.py --graph chunglu --scale 24 --steps 5 --warmup 3 --dump-levels $O/levels_cl24.json > $O/bench_cl24.json 2> $O/bench_cl24.err; echo bench_cl24=$?
;;
launches)
P="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --validate-roots 0 --profile-roots 2"
timeout 600 $P > /dev/null 2>&1 && timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -c 800 --csv --log-file $O/launches_s26.csv $P > $O/ncu_launch.log 2>&1; echo launches=$?
gzip -f $O/launches_s26.csv
;;
levels)
for spec in "s26_bu25:--scale 26 --index 25" "s26_td7:--scale 26 --index 7" "cl24_i0:--graph chunglu --scale 24 --index 0"; do
  name=${spec%%:*}; args=${spec#*:}
  RB_LEVELS_PER_LAUNCH=1 timeout 600 python tools/one_root.py --no-warmup $args > $O/levels_$name.txt 2>&1 && \
  RB_LEVELS_PER_LAUNCH=1 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:bfs_persistent \
    -o $O/levels_$name python tools/one_root.py --no-warmup $args > $O/levels_${name}_ncu.log 2>&1
  echo levels_$name=$?
  summ $O/levels_$name $name "RB_LEVELS_PER_LAUNCH=1 ncu --set full -k regex:bfs_persistent python tools/one_root.py --no-warmup $args"
done
;;
full)
F="python bench.py --profile-roots 1 --no-cpu-baseline --validate-roots 0"
timeout 600 $F > /dev/null 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k regex:bfs_persistent \
  -s 1 -c 1 -o $O/full_s26 $F > $O/ncu_full_s26.log 2>&1; echo full_s26=$?
summ $O/full_s26 kronecker-s26-ef16-rcm-bfs "ncu --set full -k regex:bfs_persistent -s 1 -c 1 $F"
;;
esac
done
du -sh $O
