# ncu launch list (time, DRAM bytes) of the cycle-end kernels of one C3
# general-case cycle end in stream order: bash scripts/ncu_cycle_end.sh TAG [CFG]
TAG=${1:-ce}; CFG=${2:-C3}
mkdir -p gpurun_out
RBICG_SYNC_CYCLE=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --kernel-name regex:"k_gram|k_gemm|k_spmm|k_resid|k_step7|k_init2" --csv \
  --log-file gpurun_out/${TAG}_launches.csv python scripts/cycle_end_probe.py $CFG > gpurun_out/${TAG}.log 2>&1
python scripts/launch_summary.py gpurun_out/${TAG}_launches.csv gpurun_out/${TAG}_summary.txt
