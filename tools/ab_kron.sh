# A/B of the Kronecker-22 PageRank config: fused update (default) vs SpMV + update kernels
for round in 1 2; do
for f in 1 0; do
  LILAC_B200_PAGERANK_FUSED=$f python bench.py --config kron --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -n 1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('fused=$f', round(l['value'],1), 'GFLOP/s', round(l['ms_per_step']*1e3,1), 'us/step', 'verify', json.dumps(l.get('verify'))[:160])"
done
done
