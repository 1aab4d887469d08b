# steady-state cycle-end phase times: the C2 / C3 bench under RBICG_TIMING
# (per-solve phase times) and RBICG_TRACE (synchronised per-phase totals of
# the cycle-end worker; the loop keeps running beside it).
mkdir -p gpurun_out
for c in C2 C3; do
  RBICG_TIMING=1 python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu --no-traffic > gpurun_out/tr_timing_$c.json 2> gpurun_out/tr_timing_$c.err
  RBICG_TRACE=1 python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu --no-traffic > gpurun_out/tr_trace_$c.json 2> gpurun_out/tr_trace_$c.err
done
tail -n 40 gpurun_out/tr_trace_C2.err; tail -n 12 gpurun_out/tr_timing_C2.err
