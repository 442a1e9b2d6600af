"""Runs tests/cpp/test_marshal (the reference's marshal suite restated against
the B200 runtime, plus SPEC acceptance #5/#6 and the B200 extensions). Host
only: page-protection traps are real SIGSEGVs, so it runs in a subprocess."""
import os
import subprocess

import pytest

from paper_2001_07938_b200 import build as B

BIN = os.path.join(B.ROOT, "tests", "cpp", "test_marshal")




def test_marshal_runtime_suite():
    B.build_cpp_tests()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=120)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed checks" in r.stdout
    assert r.stdout.count("\nok ") + r.stdout.startswith("ok ") >= 24
