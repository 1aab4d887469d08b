mkdir -p gpurun_out
for e in "" RBICG_GRAM_CC_FFMA=1 RBICG_GRAM_FLAT=1 RBICG_SPMM_MINB=1; do
  echo "== [$e]"; env $e RBICG_FUSED=0 python scripts/debug_overlap_resid.py 2>&1 | grep -v Warn
done > gpurun_out/dbg_resid.txt 2>&1
cat gpurun_out/dbg_resid.txt
