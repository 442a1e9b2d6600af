# A/B of library variants on the Parboil JDS config: cold-L2 and warm kernel times
for round in 1 2; do
for v in base "$@"; do
  if [ $v = base ]; then L=; else L=variants/$v/liblilac_b200.so; fi
  LILAC_B200_LIB=$L python bench.py --config parboil --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -n 1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); s=l['spmv']; print('$v', 'cold us', round(s['ms_cold']*1e3,2), 'warm us', round(s['ms_l2_warm']*1e3,2), 'verify', l.get('verify',{}).get('bit_identical', l.get('verify')))"
done
done
