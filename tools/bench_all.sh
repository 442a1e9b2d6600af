#!/bin/bash
# Every BASELINE config through bench.py on one GPU, both arms; one JSON line
# each into gpurun_out/bench_lines.jsonl (logs beside it).
# usage: tools/bench_all.sh [steps] [warmup] [configs...]
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
K=${1:-20}; W=${2:-5}; shift 2 || true
CONFIGS=${*:-"npb_c npb_a parboil kron stencil"}
for c in $CONFIGS; do
  for impl in ours reference; do
    log=gpurun_out/bench_${c}_${impl}.log
    timeout 1500 python bench.py --config "$c" --impl "$impl" --steps "$K" --warmup "$W" > "$log" 2>&1
    rc=$?
    echo "== $c $impl rc=$rc" >> gpurun_out/bench_all.txt
    tail -n 1 "$log" >> gpurun_out/bench_lines.jsonl
  done
done
