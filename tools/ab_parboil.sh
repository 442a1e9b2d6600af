# A/B on the Parboil JDS config: cold-L2 and warm kernel times, verification.
# usage: tools/ab_parboil.sh [variant ...]   (variants/NAME/liblilac_b200.so; "rowthread" = the
# thread-per-row kernel via LILAC_B200_JDS=rowthread)
for round in 1 2; do
for v in base "$@"; do
  L=; E=
  if [ $v = rowthread ]; then E=rowthread; elif [ $v != base ]; then L=variants/$v/liblilac_b200.so; fi
  LILAC_B200_JDS=$E LILAC_B200_LIB=$L python bench.py --config parboil --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -n 1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); s=l['spmv']; print('$v', 'cold us', round(s['ms_cold']*1e3,2), 'warm us', round(s['ms_l2_warm']*1e3,2), 'verify', json.dumps(l.get('verify'))[:200])"
done
done
