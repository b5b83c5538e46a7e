#!/bin/bash
# Round-end evidence: bench lines (s22 headline, s26, Chung-Lu), the ncu launch
# list of the s22 bench, and one `ncu --set full` capture of bfs_persistent per
# config (the timed root after one warm-up).  Outputs under gpurun_out/prof/.
set -u
O=gpurun_out/prof
mkdir -p $O
timeout 900 python bench.py > $O/bench_s22.json 2> $O/bench_s22.err; echo bench_s22=$?
timeout 1200 python bench.py --scale 26 > $O/bench_s26.json 2> $O/bench_s26.err; echo bench_s26=$?
timeout 1200 python bench.py --graph chunglu --scale 24 > $O/bench_cl24.json 2> $O/bench_cl24.err; echo bench_cl24=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_s22.csv \
  python bench.py --steps 4 --warmup 3 --no-cpu-baseline --validate-roots 0 > $O/ncu_launch.log 2>&1; echo launches=$?
for cfg in "s22:--scale 22" "s26:--scale 26" "cl24:--graph chunglu --scale 24"; do
  name=${cfg%%:*}; args=${cfg#*:}
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:bfs_persistent -s 1 -c 1 \
    -o $O/full_$name python bench.py $args --profile-roots 1 --no-cpu-baseline --validate-roots 0 \
    > $O/ncu_full_$name.log 2>&1; echo full_$name=$?
done
