"""Build a variant of liblilac_b200.so with extra compile-time flags, for
kernel experiments (not the product build):

    python tools/build_variant.py NAME -DLILAC_TILE_THREADS=512 -DLILAC_TILE_PIPE=4
    LILAC_B200_LIB=variants/NAME/liblilac_b200.so python tools/kernel_sweep.py ...
"""
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2001_07938_b200 import build as B  # noqa: E402


def main():
    name, extra = sys.argv[1], sys.argv[2:]
    out = os.path.join(ROOT, "variants", name)
    os.makedirs(out, exist_ok=True)
    jobs, objs = [], []
    for src in sorted(glob.glob(os.path.join(B.CSRC, "*.cu")) + glob.glob(os.path.join(B.CSRC, "*.cpp"))):
        obj = os.path.join(out, os.path.basename(src) + ".o")
        objs.append(obj)
        if src.endswith(".cu"):
            jobs.append([B.NVCC, *B.NVCCFLAGS, *extra, "-c", src, "-o", obj])
        else:
            jobs.append(["g++", *B.CXXFLAGS, *extra, "-c", src, "-o", obj])
    with cf.ThreadPoolExecutor(max_workers=8) as ex:
        for f in [ex.submit(subprocess.run, j, check=True) for j in jobs]:
            f.result()
    lib = os.path.join(out, "liblilac_b200.so")
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o", lib, *objs, "-Xlinker", "-Bsymbolic",
                    "-lpthread", "-ldl", "-lrt"], check=True)
    for o in objs:
        os.remove(o)
    print(lib)


if __name__ == "__main__":
    main()
