set -x
for k in 1 10; do
  ncu --set full --import-source on --clock-control none --kernel-name regex:"^k_pass" --launch-skip 4 --launch-count 2 -o gpurun_out/ncu_c3_k$k -f python scripts/kernel_traffic.py C3 $k > gpurun_out/ncu_c3_k$k.log 2>&1
done
ncu --set full --import-source on --clock-control none --kernel-name regex:"^k_fused" --launch-skip 4 --launch-count 1 -o gpurun_out/ncu_c3_k0 -f python scripts/kernel_traffic.py C3 0 > gpurun_out/ncu_c3_k0.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name regex:"^k_pass" --launch-skip 4 --launch-count 2 -o gpurun_out/ncu_c4_k8 -f python scripts/kernel_traffic.py C4 8 > gpurun_out/ncu_c4_k8.log 2>&1
