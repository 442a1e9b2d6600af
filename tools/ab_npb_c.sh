# A/B of library variants on the NPB C CG rate: base then each variant, twice
for round in 1 2; do
for v in base "$@"; do
  if [ $v = base ]; then L=; else L=variants/$v/liblilac_b200.so; fi
  LILAC_B200_LIB=$L python bench.py --config npb_c --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --no-scaling-model --no-verify 2>/dev/null | tail -n 1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$v', round(l['value'],1), round(l['spmv']['ms']*1e3,1))"
done
done
