# A/B of the stencil CG config: p.q fused into the lane-range SpMV (default) vs a separate pass
for round in 1 2; do
for f in 1 0; do
  LILAC_B200_LRC_DOT=$f python bench.py --config stencil --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -n 1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('fused_dot=$f', round(l['value'],2), 'CG it/s', round(l['ms_per_step'],3), 'ms/step', 'verify', json.dumps(l.get('verify'))[:200])"
done
done
