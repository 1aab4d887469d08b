# side-stream SM cap sweep (RBICG_SIDE_SMS) on the C2 / C3 bench lines
mkdir -p gpurun_out
for c in C2 C3; do for v in def 0 74 49; do
  if [ $v = def ]; then e=""; else e="RBICG_SIDE_SMS=$v"; fi
  env $e python bench.py --config $c --steps 4 --warmup 3 --no-e2e --no-cpu --no-traffic > gpurun_out/ss_${c}_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ss_${c}_$v.json').read().strip().splitlines()[-1]); print('$c', '$v', round(d['value']), d['config']['k_in_per_system'], d['config']['iterations_per_system'])"
done; done
