# pencil-Gram forms on one C3 general-case cycle-end probe: the default (2-D
# warp grid, k_gram_mma2) and the flat tile ranges (RBICG_GRAM_FLAT=1,
# k_gram_mma); ncu launch lists.  bash scripts/gram_forms.sh TAG
TAG=${1:-gf}
mkdir -p gpurun_out
for v in default RBICG_GRAM_FLAT; do
  case $v in default) e="";; *) e="$v=1";; esac
  env $e RBICG_SYNC_CYCLE=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --kernel-name regex:"k_gram|k_spmm" --csv \
    --log-file gpurun_out/${TAG}_$v.csv python scripts/cycle_end_probe.py C3 > gpurun_out/${TAG}_$v.log 2>&1
  python scripts/launch_summary.py gpurun_out/${TAG}_$v.csv gpurun_out/${TAG}_${v}_summary.txt
  echo "== $v"; cat gpurun_out/${TAG}_${v}_summary.txt
done
