bash scripts/gram_forms.sh gf1 > gpurun_out/gf1.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "projection or c1_sequence or c4_small or fast_pencil or repeated or full_size_k_matched or c4_sweep or own_chain" > gpurun_out/gf1_parity.log 2>&1; echo "rc=$?" >> gpurun_out/gf1_parity.log
cat gpurun_out/gf1.txt; tail -3 gpurun_out/gf1_parity.log
