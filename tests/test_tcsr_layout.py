"""Runs tests/cpp/test_tcsr: the tiled CSR layout builder (csrc/tcsr_build.cpp)
replayed on the CPU by a restatement of the kernel's walk — every stored
nonzero exactly once, y = A x within 1e-12 sum|a x| — on random long rows,
0-3 nonzero rows with empties over more tiles than SMs, banded and
single-column matrices. Host only (the builder runs at upload on the host)."""
import os
import subprocess

import pytest

from paper_2001_07938_b200 import build as B

BIN = os.path.join(B.ROOT, "tests", "cpp", "test_tcsr")


def test_tiled_layout_builder_replay():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/test_tcsr not built (python -c 'import __graft_entry__ as g; g.build()')")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("ok ") == 4, r.stdout


def test_lane_range_layout_builder_replay():
    """tests/cpp/test_lrc: the lane-range layout (csrc/lrcsr_build.cpp) replayed
    by a CPU restatement of lrcsr.cu — lane walks, warp combine, unit carries
    and the fix-up — on power-law, short, unit-aligned and single-nonzero
    matrices: every row written once, y within 1e-12 sum|a x|."""
    binp = os.path.join(B.ROOT, "tests", "cpp", "test_lrc")
    if not os.path.exists(binp):
        pytest.skip("tests/cpp/test_lrc not built")
    r = subprocess.run([binp], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("ok ") == 4, r.stdout


@pytest.mark.gpu
def test_lane_range_device_builder_matches_host_builder():
    """tests/cpp/test_lrc_dev: lrc_build_device (hot set by device histogram +
    radix sort, encoded columns, descriptors, compact-row map) bit-identical to
    the host builder that test_lrc replays."""
    binp = os.path.join(B.ROOT, "tests", "cpp", "test_lrc_dev")
    assert os.path.exists(binp), "tests/cpp/test_lrc_dev not built"
    r = subprocess.run([binp], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("ok ") == 4, r.stdout
