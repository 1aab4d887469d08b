set -x
mkdir -p gpurun_out
bash scripts/ncu_cycle_end.sh ce2_c3 C3
bash scripts/ncu_cycle_end.sh ce2_c4 C4
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64peak scripts/ubench/fp64peak.cu && /tmp/fp64peak > gpurun_out/fp64peak.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/ce2_parity.log 2>&1; echo "rc=$?" >> gpurun_out/ce2_parity.log
cat gpurun_out/ce2_c3_summary.txt gpurun_out/ce2_c4_summary.txt gpurun_out/fp64peak.txt; tail -3 gpurun_out/ce2_parity.log
