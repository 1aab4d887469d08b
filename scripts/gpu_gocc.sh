# overlap experiment: pencil-Gram CTAs per SM capped (RBICG_GRAM_OCC) and the
# side-stream SM cap (RBICG_SIDE_SMS), C2 and C3 bench lines
mkdir -p gpurun_out
for c in C2 C3; do for v in "" "RBICG_GRAM_OCC=1" "RBICG_GRAM_OCC=1 RBICG_SIDE_SMS=0" "RBICG_GRAM_OCC=2 RBICG_SIDE_SMS=0"; do
  env $v python bench.py --config $c --steps 4 --warmup 3 --no-e2e --no-cpu --no-traffic > gpurun_out/go.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/go.json').read().strip().splitlines()[-1]); print('$c', '[$v]', round(d['value']), d['config']['k_in_per_system'], d['config']['iterations_per_system'], round(d['config']['cycle_end_ms']), round(d['config']['loop_ms']))"
done; done
