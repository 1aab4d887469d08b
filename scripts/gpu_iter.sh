# one GPU iteration on the cycle-end kernels: ncu --set full of the pencil
# Gram and the C~^*C Gram (C3 probe), the SpMM register-cap variants, and the
# parity tests of the cycle end.   bash scripts/gpu_iter.sh TAG
TAG=${1:-it}
mkdir -p gpurun_out
for kn in k_gram_mma k_gram_cc_mma; do
  RBICG_SYNC_CYCLE=1 ncu --set full --import-source on --clock-control none --kernel-name regex:"^$kn" \
    --launch-skip 0 --launch-count 1 -o gpurun_out/${TAG}_ncu_$kn -f \
    python scripts/cycle_end_probe.py C3 > gpurun_out/${TAG}_ncu_$kn.log 2>&1
done
bash scripts/spmm_minb.sh ${TAG}_spmm > gpurun_out/${TAG}_spmm.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "projection or c1_sequence or c4_small or fast_pencil or repeated or full_size_k_matched or c4_sweep or own_chain" > gpurun_out/${TAG}_parity.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_parity.log
cat gpurun_out/${TAG}_spmm.txt; tail -3 gpurun_out/${TAG}_parity.log
