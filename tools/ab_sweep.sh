#!/bin/bash
# A/B of library variants on tiled SpMV kernel times (NPB C and row blocks):
#   tools/ab_sweep.sh VARIANT... (variants/NAME/liblilac_b200.so; "base" = the in-tree build)
for round in 1 2; do
for v in base "$@"; do
  for sh in 1:0 4:0 8:0; do
    if [ $v = base ]; then L=; else L=variants/$v/liblilac_b200.so; fi
    LILAC_B200_LIB=$L python tools/kernel_sweep.py --matrix npb_c --shard $sh --kernels auto --reps 50 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['shard'], d['kernel'], round(d['us'],2), d['ok'])"
  done
done
done
