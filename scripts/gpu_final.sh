# round-end pass of the second session: GPU suite, smoke, the default bench
# line (C3) and C2 / C4 / C5, the ncu launch list of the default bench command
# and the C3 cycle-end probe launch list.   bash scripts/gpu_final.sh TAG
TAG=${1:-fin}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
python bench.py > gpurun_out/${TAG}_bench_c3.json 2> gpurun_out/${TAG}_bench_c3.err
python bench.py --config C2 > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err
python bench.py --config C4 > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err
python bench.py --config C5 --no-e2e > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-traffic --no-cpu --no-e2e > gpurun_out/${TAG}_ncu.log 2>&1
python scripts/launch_summary.py gpurun_out/${TAG}_launches.csv gpurun_out/${TAG}_launches_summary.txt
bash scripts/ncu_cycle_end.sh ${TAG}_ce C3
tail -n 3 gpurun_out/${TAG}_gpu_tests.log; tail -n 1 gpurun_out/${TAG}_smoke.log
for c in c3 c2 c4 c5; do python -c "import json; d=json.loads(open('gpurun_out/${TAG}_bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['value'],1), (d.get('e2e') or {}).get('value'), round(d['roofline']['frac'],3), d['config'].get('k_in_per_system'), d['clocks'])"; done
head -12 gpurun_out/${TAG}_launches_summary.txt; cat gpurun_out/${TAG}_ce_summary.txt
