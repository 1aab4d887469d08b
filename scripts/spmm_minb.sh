# k_spmm_rows register-cap variants (RBICG_SPMM_MINB = 1..4) on one C3
# general-case cycle end: ncu launch list (time, DRAM bytes) per variant.
# bash scripts/spmm_minb.sh TAG
TAG=${1:-spmm}
mkdir -p gpurun_out
for mb in 1 2 3 4; do
  RBICG_SPMM_MINB=$mb RBICG_SYNC_CYCLE=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --kernel-name regex:"k_spmm|k_gram" --csv \
    --log-file gpurun_out/${TAG}_mb$mb.csv python scripts/cycle_end_probe.py C3 > gpurun_out/${TAG}_mb$mb.log 2>&1
  python scripts/launch_summary.py gpurun_out/${TAG}_mb$mb.csv gpurun_out/${TAG}_mb${mb}_summary.txt
  echo "== MINB=$mb"; cat gpurun_out/${TAG}_mb${mb}_summary.txt
done
