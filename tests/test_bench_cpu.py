"""bench.py on CPU: the multi-rank launcher and the reference arm.

* `bench.py --gpus N --dry-run` (no torchrun) spawns N ranks itself; over gloo
  they drive the sharded CG with the product's host-side sharding logic
  (b200_partition_rows, b200_shard_footprint, b200_dist_send_ranges) and the
  device driver's exchange order, and must verify (NPB class S zeta; the
  stencil's halo plan against a one-process CG).
* `--impl reference` prints the contract line with the same config.workload
  string as our arm (WORKLOADS), on the reference's own CPU harness.
"""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_gpus2_spawns_two_ranks_npb():
    line = run("--gpus", "2", "--dry-run")
    assert line["n_gpus"] == 2 and line["dry_run"] == "gloo" and line["verified"] is True
    b = line["config"]["bounds"]
    assert b[0] == 0 and b[-1] == 1400 and len(b) == 3
    # NPB's random columns: every rank reads every slice whole
    for s in range(2):
        for r in range(2):
            assert line["send_ranges"][s][r] == [0, b[s + 1] - b[s]]


def test_gpus3_stencil_halo_plan():
    line = run("--gpus", "3", "--dry-run", "--config", "stencil")
    assert line["n_gpus"] == 3 and line["verified"] is True
    b = line["config"]["bounds"]
    halo = 20 * 20 + 20 + 1
    plan = line["send_ranges"]
    assert plan[0][2] == [0, 0] and plan[2][0] == [0, 0]  # non-neighbours exchange nothing
    assert plan[0][1] == [b[1] - b[0] - halo, b[1] - b[0]]  # the last nx^2+nx+1 rows go up
    assert plan[1][0] == [0, halo]


def test_partition_and_plan_match_oracle():
    import oracle_lib as O
    from paper_2001_07938_b200 import device as D
    from paper_2001_07938_b200 import workloads as W
    rp, ci, val = W.gen_stencil27(9)
    for k in (1, 2, 3, 5, 8):
        b = D.partition_rows(rp, k)
        assert np.array_equal(b, O.partition_rows(rp, k))
        fps = [D.shard_footprint(rp[b[g]:b[g + 1] + 1], ci) for g in range(k)]
        for g in range(k):
            seg = ci[rp[b[g]]:rp[b[g + 1]]]
            assert fps[g] == ((int(seg.min()), int(seg.max()) + 1) if len(seg) else (0, 0))
        plan = D.send_ranges(b, [f[0] for f in fps], [f[1] for f in fps])
        for s in range(k):
            for r in range(k):
                lo, hi = max(b[s], fps[r][0]), min(b[s + 1], fps[r][1])
                want = [lo - b[s], hi - b[s]] if hi > lo else [0, 0]
                assert plan[s, r].tolist() == want


def test_reference_arm_parboil_line():
    line = run("--impl", "reference", "--config", "parboil", "--steps", "2", "--warmup", "1")
    import bench
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "GFLOP/s"
    assert line["config"]["workload"] == bench.WORKLOADS["parboil"][0]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["cores"] >= 1
    for k in ("metric", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "dtype"):
        assert k in line
