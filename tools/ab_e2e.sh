#!/bin/bash
# A/B of the NPB C e2e host loop (examples/npb_host_cg.c links the in-tree
# library, so each variant is swapped into place rather than preloaded):
#   tools/ab_e2e.sh VARIANT...   (variants/NAME/liblilac_b200.so; "base" = the in-tree build)
LIB=paper_2001_07938_b200/liblilac_b200.so
cp $LIB /tmp/base_lib.so
for round in 1 2; do
for v in base "$@"; do
  if [ $v = base ]; then cp /tmp/base_lib.so $LIB; else cp variants/$v/liblilac_b200.so $LIB; fi
  python tools/e2e_breakdown.py --steps 20 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('e2e $v', round(d['ms_per_step'],3), round(d['value'],1))"
done
done
cp /tmp/base_lib.so $LIB
