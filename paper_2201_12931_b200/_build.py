"""Build libvoxb200.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

Used by __graft_entry__.build() and `python -m paper_2201_12931_b200._build`.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libvoxb200.so")
OBJ = os.path.join(HERE, "build")
SOURCES = ["hex8_apply.cu", "vectors.cu", "multigrid.cu", "design.cu", "runtime.cu", "dist.cu", "dist_design.cu", "galerkin.cu",
           "peer.cu", "dist_galerkin.cu", "tail.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    raise RuntimeError("nvcc not found")


def _stale(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines=(), tag: str = "") -> str:
    """Compile libvoxb200.so; `defines`/`tag` build a dev variant libvoxb200_<tag>.so
    (selected at import time with VT_LIB_PATH) for A/B kernel experiments."""
    obj_dir = OBJ + (f"_{tag}" if tag else "")
    out = OUT.replace(".so", f"_{tag}.so") if tag else OUT
    os.makedirs(obj_dir, exist_ok=True)
    nvcc = _nvcc()
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(HERE, "..", "include", "voxb200.h"))
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(obj_dir, src.replace(".cu", ".o"))
        if force or _stale(o, [s] + headers):
            jobs.append([nvcc, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", s, "-o", o])

    def run(cmd):
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
        if verbose:
            sys.stderr.write(p.stderr)
        return p.stderr

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        logs = list(ex.map(run, jobs))
    objs = [os.path.join(obj_dir, s.replace(".cu", ".o")) for s in SOURCES]
    if jobs or not os.path.exists(out):
        run([nvcc, *ARCH, "-shared", "-o", out, *objs, "-Xcompiler", "-fPIC", "-ldl"])
    with open(os.path.join(obj_dir, "ptxas.log"), "a") as fh:
        fh.writelines(logs)
    return out


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    tag = next((a[6:] for a in sys.argv[1:] if a.startswith("--tag=")), "")
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, defines=defs, tag=tag))
