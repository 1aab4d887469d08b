# diagnosis of the forced-overlap NCCL test with the round-2 session-1 kernel
# forms, then the full GPU pass (no -x), smoke and the bench lines.
TAG=${1:-full}
mkdir -p gpurun_out
RBICG_GRAM_CC_FFMA=1 RBICG_GRAM_FLAT=1 RBICG_SPMM_MINB=1 python -m pytest tests/test_gpu_dist.py -q -m gpu -k "forced_overlap_in_graph" > gpurun_out/${TAG}_old_forms.log 2>&1
python -m pytest tests/test_gpu_dist.py -q -m gpu -k "forced_overlap_in_graph" > gpurun_out/${TAG}_new_forms.log 2>&1
tail -3 gpurun_out/${TAG}_old_forms.log gpurun_out/${TAG}_new_forms.log
bash scripts/gpu_full.sh ${TAG}
