# full GPU pass after a kernel change: GPU suite, smoke, bench lines C3
# (default), C2, C4.   bash scripts/gpu_full.sh TAG
TAG=${1:-full}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
python bench.py > gpurun_out/${TAG}_bench_c3.json 2> gpurun_out/${TAG}_bench_c3.err
python bench.py --config C2 > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err
python bench.py --config C4 > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err
tail -3 gpurun_out/${TAG}_gpu_tests.log; tail -1 gpurun_out/${TAG}_smoke.log
for c in c3 c2 c4; do python -c "import json,sys; d=json.loads(open('gpurun_out/${TAG}_bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['value'], d['e2e']['value'], d['roofline']['frac'], d['config'].get('k_in_per_system'))"; done
