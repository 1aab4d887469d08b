# per-solve setup cost after caching the device-memory query per sequence:
# C3 bench under RBICG_TIMING (setup lines), plain C3 bench, a test subset
mkdir -p gpurun_out
RBICG_TIMING=1 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-traffic > gpurun_out/su_c3_timing.json 2> gpurun_out/su_c3_timing.err
python bench.py > gpurun_out/su_bench_c3.json 2> gpurun_out/su_bench_c3.err
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "c1_sequence or c4_small or full_size_k_matched or c4_sweep or own_chain or repeated" > gpurun_out/su_tests.log 2>&1; echo "rc=$?" >> gpurun_out/su_tests.log
grep "rbicg setup\|rbicg timing" gpurun_out/su_c3_timing.err | tail -12
python -c "import json; d=json.loads(open('gpurun_out/su_bench_c3.json').read().strip().splitlines()[-1]); print('c3', round(d['value'],1), d['e2e']['value'], d['config']['k_in_per_system'], d['config']['step_ms'], d['config']['iterations_per_system'])"
tail -n 3 gpurun_out/su_tests.log
