# One GPU-box pass: full GPU suite, smoke, the default bench line, and the ncu
# launch list of the same bench command (kernel shares; cold, serialised).
# Usage (on the box): bash scripts/round_end_check.sh TAG
TAG=${1:-run}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-traffic --no-cpu --no-e2e > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu.log
tail -3 gpurun_out/${TAG}_gpu_tests.log; tail -1 gpurun_out/${TAG}_smoke.log; tail -c 600 gpurun_out/${TAG}_bench.json
