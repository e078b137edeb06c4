"""Build the native library (sm_100a) in-tree: csrc/*.cu -> _native/libnautilus_b200.so.

    python -m paper_2604_14825_b200.build [--force] [--jobs N]

Every translation unit is compiled with
``nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` in parallel and
linked into one shared library exporting the C ABI of include/nautilus_b200.h.
The .so is git-ignored but travels to GPU boxes with the repo snapshot.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_native")
OBJ_DIR = os.path.join(OUT_DIR, "obj")
LIB = os.path.join(OUT_DIR, "libnautilus_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I" + os.path.join(REPO, "include")]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[str]:
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def headers() -> list[str]:
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return hs + [os.path.join(REPO, "include", "nautilus_b200.h")]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def _compile(src: str, force: bool, defines=(), obj_dir=OBJ_DIR) -> tuple[str, str]:
    obj = os.path.join(obj_dir, os.path.basename(src).replace(".cu", ".o"))
    newest_dep = max([_mtime(src)] + [_mtime(h) for h in headers()])
    if not force and _mtime(obj) > newest_dep:
        return obj, ""
    cmd = [nvcc()] + ARCH + FLAGS + ["-D" + d for d in defines] + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, jobs: int | None = None, verbose: bool = False, defines=(),
          out: str | None = None) -> str:
    """Build the library; `defines`/`out` build an experiment variant (e.g. NT_POLY_EVERY=0)."""
    lib = out or LIB
    obj_dir = OBJ_DIR if not defines else os.path.join(OUT_DIR, "obj_" + "_".join(
        d.replace("=", "") for d in defines))
    os.makedirs(obj_dir, exist_ok=True)
    srcs = sources()
    jobs = jobs or min(len(srcs), os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(lambda s: _compile(s, force, defines, obj_dir), srcs))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                print(log, file=sys.stderr)
    if force or not os.path.exists(lib) or _mtime(lib) < max(_mtime(o) for o in objs):
        # static cudart; the driver API (cuTensorMapEncodeTiled) is resolved at run
        # time through cudaGetDriverEntryPoint, so libcuda is not a link dependency
        cmd = [nvcc()] + ARCH + ["-shared", "-o", lib] + objs
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--jobs", type=int, default=None)
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("-D", "--define", action="append", default=[])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    out = os.path.join(OUT_DIR, a.out) if a.out else None
    print(build(a.force, a.jobs, a.verbose, tuple(a.define), out))


if __name__ == "__main__":
    main()
