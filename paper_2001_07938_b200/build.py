"""Build the native library in-tree: paper_2001_07938_b200/liblilac_b200.so.

nvcc for the sm_100a kernels (-gencode arch=compute_100a,code=sm_100a,
-lineinfo so ncu's source page maps to our code), g++ for the host runtime,
static cudart. Incremental (mtime-based), parallel. Also builds the C++
marshal-runtime test binary tests/cpp/test_marshal (no GPU needed to run it).

    python -m paper_2001_07938_b200.build [--force] [-v]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "liblilac_b200.so")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CXXFLAGS = ["-std=c++17", "-O2", "-fPIC", "-Wall", "-Wextra", "-Wno-unused-parameter",
            f"-I{INCLUDE}", f"-I{CSRC}", f"-I{CUDA_HOME}/include"]
NVCCFLAGS = ["-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC",
             f"-I{INCLUDE}", f"-I{CSRC}", "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def _headers():
    return glob.glob(os.path.join(CSRC, "*.hpp")) + glob.glob(os.path.join(INCLUDE, "**", "*.h*"), recursive=True)


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _run(cmd: list[str], verbose: bool):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ... ({cmd[-1]})")
    if verbose and (r.stdout or r.stderr):
        sys.stderr.write(r.stdout + r.stderr)
    return r


def build(force: bool = False, verbose: bool = False) -> str:
    if not os.path.exists(NVCC):
        raise RuntimeError(f"nvcc not found at {NVCC}")
    os.makedirs(OBJ, exist_ok=True)
    hdrs = _headers()
    jobs = []
    objs = []
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp"))):
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, [src, *hdrs, __file__]):
            if src.endswith(".cu"):
                cmd = [NVCC, *NVCCFLAGS, "-c", src, "-o", obj]
            else:
                cmd = ["g++", *CXXFLAGS, "-c", src, "-o", obj]
            jobs.append(cmd)
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            for f in [ex.submit(_run, j, verbose) for j in jobs]:
                f.result()
    if force or jobs or _stale(LIB, objs):
        tmp = LIB + ".tmp"
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs,
              "-Xlinker", "-Bsymbolic", "-lpthread", "-ldl", "-lrt"], verbose)
        os.replace(tmp, LIB)
    build_cpp_tests(force, verbose)
    build_generated_harness(force, verbose)
    build_python_ext(force, verbose)
    build_examples(force, verbose)
    return LIB


EX_LIB = os.path.join(PKG, "libnpb_host_cg.so")


def build_examples(force: bool = False, verbose: bool = False):
    """examples/npb_host_cg.c — a C host program on the harness ABI (the e2e
    leg of bench.py), linked to liblilac_b200.so."""
    src = os.path.join(PKG, "examples", "npb_host_cg.c")
    if force or _stale(EX_LIB, [src, LIB, os.path.join(INCLUDE, "lilac_b200.h")]):
        _run(["gcc", "-std=c11", "-O2", "-fPIC", "-shared", "-Wall", f"-I{INCLUDE}", "-o", EX_LIB, src, f"-L{PKG}",
              "-llilac_b200", "-Wl,-rpath,$ORIGIN", "-lm"], verbose)


def build_python_ext(force: bool = False, verbose: bool = False):
    """paper_2001_07938_b200/_harness*.so: the CPython binding of the harness
    entry points (csrc/pyext/harness_module.c), linked to liblilac_b200.so."""
    import sysconfig
    src = os.path.join(CSRC, "pyext", "harness_module.c")
    out = os.path.join(PKG, "_harness" + sysconfig.get_config_var("EXT_SUFFIX"))
    if force or _stale(out, [src, LIB, os.path.join(INCLUDE, "lilac_b200.h")]):
        _run(["gcc", "-O2", "-fPIC", "-shared", "-Wall", f"-I{sysconfig.get_paths()['include']}", f"-I{INCLUDE}",
              "-o", out, src, f"-L{PKG}", "-llilac_b200", "-Wl,-rpath,$ORIGIN"], verbose)
    return out


GEN_LIB = os.path.join(PKG, "liblilac_b200_gen.so")


def build_generated_harness(force: bool = False, verbose: bool = False):
    """tests/golden/b200gen_spmv_csr.gen.cpp — emitted by the reference's own
    harness generator from specs/b200.lilac (tools/gen_b200_harness.py) — is
    compiled unchanged against include/lilac/marshal.hpp and linked to the
    B200 library: the drop-in behind the reference's plugin API."""
    src = os.path.join(ROOT, "tests", "golden", "b200gen_spmv_csr.gen.cpp")
    if not os.path.exists(src):
        return
    deps = [src, LIB, os.path.join(INCLUDE, "lilac", "marshal.hpp"), os.path.join(INCLUDE, "lilac_b200.h")]
    if force or _stale(GEN_LIB, deps):
        _run(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-Wno-unused-parameter", f"-I{INCLUDE}",
              "-o", GEN_LIB, src, f"-L{PKG}", "-llilac_b200",
              "-Wl,-rpath,$ORIGIN", "-lpthread"], verbose)


def build_cpp_tests(force: bool = False, verbose: bool = False):
    """tests/cpp/test_marshal: the reference's marshal suite restated against
    our runtime (host only, links csrc/marshal.cpp directly)."""
    src = os.path.join(ROOT, "tests", "cpp", "test_marshal.cpp")
    if not os.path.exists(src):
        return
    out = os.path.join(ROOT, "tests", "cpp", "test_marshal")
    deps = [src, os.path.join(CSRC, "marshal.cpp"), os.path.join(INCLUDE, "lilac", "marshal.hpp"),
            os.path.join(ROOT, "tests", "cpp", "check.hpp")]
    if force or _stale(out, deps):
        _run(["g++", "-std=c++17", "-O1", "-g", f"-I{INCLUDE}", "-o", out, src,
              os.path.join(CSRC, "marshal.cpp"), "-lpthread"], verbose)
    # tests/cpp/test_tcsr, test_lrc: the tiled / lane-range layout builders replayed on the CPU
    for name in ("test_tcsr", "test_lrc", "test_lrc_dev"):
        src = os.path.join(ROOT, "tests", "cpp", name + ".cpp")
        out = os.path.join(ROOT, "tests", "cpp", name)
        if os.path.exists(src) and (force or _stale(out, [src, LIB] + _headers())):
            extra = [f"-L{CUDA_HOME}/lib64", "-lcudart"] if name == "test_lrc_dev" else []
            _run(["g++", "-std=c++17", "-O2", f"-I{INCLUDE}", f"-I{CSRC}", f"-I{CUDA_HOME}/include", "-o", out, src,
                  f"-L{PKG}", "-llilac_b200", "-Wl,-rpath,$ORIGIN/../../paper_2001_07938_b200", "-lpthread"] + extra,
                 verbose)


def clean():
    shutil.rmtree(OBJ, ignore_errors=True)
    if os.path.exists(LIB):
        os.remove(LIB)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("--clean", action="store_true")
    a = ap.parse_args()
    if a.clean:
        clean()
    else:
        print(build(a.force, a.verbose))
