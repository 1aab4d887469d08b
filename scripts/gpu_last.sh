# last check of the session's final build: a GPU-test subset, smoke, the
# default bench line (C3) and C2
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_switches.py -q -m gpu > gpurun_out/last_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/last_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/last_smoke.log
python bench.py > gpurun_out/last_bench_c3.json 2> gpurun_out/last_bench_c3.err
python bench.py --config C2 > gpurun_out/last_bench_c2.json 2> gpurun_out/last_bench_c2.err
tail -n 3 gpurun_out/last_tests.log; tail -n 1 gpurun_out/last_smoke.log
for c in c3 c2; do python -c "import json; d=json.loads(open('gpurun_out/last_bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['value'],1), (d.get('e2e') or {}).get('value'), round(d['roofline']['frac'],3), d['config'].get('k_in_per_system'), d['clocks'])"; done
