mkdir -p gpurun_out
RBICG_SYNC_CYCLE=1 ncu --set full --import-source on --clock-control none --kernel-name regex:"^k_gram_mma2" \
  --launch-skip 0 --launch-count 2 -o gpurun_out/g2_ncu -f python scripts/cycle_end_probe.py C3 > gpurun_out/g2_ncu.log 2>&1
ncu -i gpurun_out/g2_ncu.ncu-rep --page raw --csv > gpurun_out/g2_raw.csv 2>/dev/null
echo done
