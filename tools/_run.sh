timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/s15_pytest_full.log 2>&1; echo pytest=$?; tail -2 gpurun_out/s15_pytest_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s15_smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/s15_smoke.log
python bench.py --steps 5 --warmup 3 > gpurun_out/s15_bench_s26.json 2> gpurun_out/s15_bench_s26.err; echo bench=$?
python bench.py --scale 22 --steps 5 --warmup 3 > gpurun_out/s15_bench_s22.json 2>/dev/null
python bench.py --graph chunglu --scale 24 --steps 5 --warmup 3 > gpurun_out/s15_bench_cl24.json 2>/dev/null
python -c "
import json
for c in ('s26','s22','cl24'):
    d=json.load(open('gpurun_out/s15_bench_%s.json'%c)); print(c, round(d['value'],1), round(d['e2e']['value'],1), d['roofline']['frac'], d['clocks'], d['validation']['passed'])"
