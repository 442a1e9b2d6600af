# Tiled SpMV correctness + timing probes on NPB class C (run under gpurun from the repo root).
python tools/tiled_check.py 2>&1 | tail -1
for p in ${PROBES:-0 1 2 3 5 6}; do LILAC_B200_TILED_PROBE=$p python tools/spmv_probe.py --only npb 2>&1 | grep tiled/again | sed "s/^/probe$p /"; done
