bash tools/profile_round2.sh benches launches levels full
(time python bench.py --impl reference --steps 2 --warmup 1) > gpurun_out/prof2/bench_reference_s26.json 2> gpurun_out/prof2/bench_reference_s26.err; echo ref=$?
tail -4 gpurun_out/prof2/bench_reference_s26.err
