# Cycle-end diagnosis on one GPU box: per-phase trace of one general-case cycle
# end (C2, C3; synchronised phases, RBICG_TRACE) and ncu --set full of the
# pencil Gram and the C~^*C Gram on C3.   bash scripts/ce_diag.sh TAG
TAG=${1:-ced}
mkdir -p gpurun_out
for c in C2 C3; do
  RBICG_SYNC_CYCLE=1 RBICG_TRACE=1 python scripts/cycle_end_probe.py $c > gpurun_out/${TAG}_trace_$c.log 2>&1
done
for kn in k_gram_mma k_gram_cc k_spmm_rows; do
  RBICG_SYNC_CYCLE=1 ncu --set full --import-source on --clock-control none --kernel-name regex:"^$kn" \
    --launch-skip 0 --launch-count 1 -o gpurun_out/${TAG}_ncu_$kn -f \
    python scripts/cycle_end_probe.py C3 > gpurun_out/${TAG}_ncu_$kn.log 2>&1
done
tail -n 30 gpurun_out/${TAG}_trace_C2.log gpurun_out/${TAG}_trace_C3.log
