mkdir -p gpurun_out
bash scripts/ncu_cycle_end.sh c4g C4
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "projection or c4_small or fast_pencil or c4_sweep or own_chain or irka" > gpurun_out/c4g_parity.log 2>&1; echo "rc=$?" >> gpurun_out/c4g_parity.log
cat gpurun_out/c4g_summary.txt; tail -n 3 gpurun_out/c4g_parity.log
