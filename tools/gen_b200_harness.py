"""Generate the B200 harness TU from paper_2001_07938_b200/specs/b200.lilac
with the REFERENCE's own harness generator (harnessgen::gen_all, run from
oracle/_ref), and store it as the golden tests/golden/b200gen_spmv_csr.gen.cpp.
The TU is then compiled unchanged against include/lilac/marshal.hpp by
paper_2001_07938_b200/build.py.

    python tools/gen_b200_harness.py [--check]
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_lib as O  # noqa: E402

SPEC = os.path.join(ROOT, "paper_2001_07938_b200", "specs", "b200.lilac")
GOLDEN = os.path.join(ROOT, "tests", "golden", "b200gen_spmv_csr.gen.cpp")


def generate() -> str:
    R = O.ref()
    spec = open(SPEC).read().encode()
    buf = C.create_string_buffer(1 << 20)
    n = R.ref_gen_harness(spec, b"b200gen_spmv_csr", buf, len(buf))
    if n < 0:
        raise RuntimeError(R.ref_last_error().decode())
    return buf.value.decode()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--check", action="store_true", help="fail if the golden differs")
    a = ap.parse_args()
    src = generate()
    if a.check:
        if open(GOLDEN).read() != src:
            sys.exit("generated harness differs from the golden")
        print("golden up to date")
        return
    with open(GOLDEN, "w") as f:
        f.write(src)
    print("wrote", GOLDEN)


if __name__ == "__main__":
    main()
