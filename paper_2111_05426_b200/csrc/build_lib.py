"""build_lib.py -- compile libdistir.so for sm_100a in-tree.

distir.cu (C ABI, host planner, enumerate / plan / scatter / top-k / raw
kernels) and one translation unit per k_simulate<KIND, MODE> instantiation
(sim_inst.cu) are compiled in parallel and linked into one shared library.
Loaded by path (no package import: the binding refuses to import without the
library), by ``__graft_entry__.build()`` and the tools; also a script:

    python paper_2111_05426_b200/csrc/build_lib.py [-DNAME[=VALUE] ...] [-o OUT.so]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

CSRC = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.dirname(CSRC)
ROOT = os.path.dirname(PKG)
SO_PATH = os.path.join(PKG, "libdistir.so")
BUILD = os.path.join(ROOT, "build", "distir")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-lineinfo", "-O3", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC"]
SIM_INSTANCES = [(0, m) for m in range(9)] + [(1, m) for m in range(5)]


def sources():
    """Every file the library depends on (for staleness checks)."""
    fs = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))
          if f.endswith((".cu", ".cuh"))]
    return fs + [os.path.join(ROOT, "include", "distir.h")]


def stale(so=SO_PATH):
    if not os.path.exists(so):
        return True
    t = os.path.getmtime(so)
    return any(os.path.getmtime(s) > t for s in sources())


def build(defines=(), out=SO_PATH, jobs=None, verbose=False, force=True):
    """Compile and link; returns the library path.  `defines` are extra
    -D flags (experiments, instrumentation)."""
    if not force and not stale(out):
        return out
    tag = "".join(c if c.isalnum() else "_" for c in "_".join(defines))[:80] or "default"
    bdir = os.path.join(BUILD, tag)
    os.makedirs(bdir, exist_ok=True)
    extra = list(defines) + (["-Xptxas", "-v"] if verbose else [])
    jobs_ = [(os.path.join(bdir, "distir.o"), os.path.join(CSRC, "distir.cu"), [])]
    for kd, md in SIM_INSTANCES:
        jobs_.append((os.path.join(bdir, "sim_%d_%d.o" % (kd, md)),
                      os.path.join(CSRC, "sim_inst.cu"),
                      ["-DSIM_KIND=%d" % kd, "-DSIM_MODE=%d" % md]))

    def compile_one(job):
        obj, src, d = job
        cmd = ["nvcc"] + FLAGS + extra + d + ["-c", "-o", obj, src]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return obj, r.returncode, r.stdout + r.stderr

    n = jobs or min(len(jobs_), os.cpu_count() or 1)
    # the largest instantiations first
    with cf.ThreadPoolExecutor(n) as ex:
        results = list(ex.map(compile_one, jobs_[1:] + jobs_[:1]))
    errs = [(o, log) for o, rc, log in results if rc != 0]
    for o, rc, log in results:
        if log.strip() and (verbose or rc != 0):
            sys.stderr.write("== %s\n%s\n" % (os.path.basename(o), log))
    if errs:
        raise RuntimeError("nvcc failed for %s" % ", ".join(os.path.basename(o) for o, _ in errs))
    objs = [j[0] for j in jobs_]
    tmp = out + ".tmp"
    subprocess.check_call(["nvcc"] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl"])
    os.replace(tmp, out)
    return out


def main(argv):
    defines, out, verbose = [], SO_PATH, False
    i = 0
    while i < len(argv):
        a = argv[i]
        if a == "-o":
            out = os.path.abspath(argv[i + 1])
            i += 1
        elif a == "-v":
            verbose = True
        elif a.startswith("-D"):
            defines.append(a)
        else:
            raise SystemExit("usage: build_lib.py [-DNAME[=VALUE] ...] [-v] [-o OUT.so]")
        i += 1
    print(build(defines, out=out, verbose=verbose))


if __name__ == "__main__":
    main(sys.argv[1:])
