python bench.py --steps 5 --warmup 3 > gpurun_out/s10_bench.json 2> gpurun_out/s10_bench.err; echo rc=$?
python -c "
import json; d=json.load(open('gpurun_out/s10_bench.json')); print(d['value'], d['e2e']['value'], d['clocks'], d['gpu_launches'], d['roofline']['frac'])"
tail -3 gpurun_out/s10_bench.err
