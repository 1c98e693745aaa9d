"""Build libsgrpo_b200.so in-tree (nvcc, sm_100a only).

    python -m paper_2509_21792_b200.build          # incremental
    python -m paper_2509_21792_b200.build --force  # rebuild everything
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libsgrpo_b200.so")
DEVSRC = os.path.join(PKG, "devsrc")
DEVLIB = os.path.join(PKG, "libsgrpo_b200_dev.so")  # test-only self-tests / microbenchmarks
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills", "-I", os.path.join(os.path.dirname(PKG), "include")]


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _headers_mtime():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hs.append(os.path.join(os.path.dirname(PKG), "include", "sgrpo_b200.h"))
    hs.append(os.path.join(os.path.dirname(PKG), "include", "sgrpo_b200_dev.h"))
    return max(os.path.getmtime(h) for h in hs)


def _compile(src: str, force: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), _headers_mtime()):
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)
    return obj


def _link(out: str, objs, force: bool):
    if force or not os.path.exists(out) or os.path.getmtime(out) < max(os.path.getmtime(o) for o in objs):
        # NCCL (system libnccl.so.2) for the data-parallel gradient / statistics all-reduce
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", out, *objs, "-lnccl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")


def build(force: bool = False) -> str:
    """libsgrpo_b200.so (the product: kernels, engine, C-ABI) and libsgrpo_b200_dev.so (the
    same kernels + the test-only self-test / microbenchmark entry points of devsrc/)."""
    os.makedirs(OBJ, exist_ok=True)
    srcs = _sources()
    dev = sorted(os.path.join(DEVSRC, f) for f in os.listdir(DEVSRC) if f.endswith(".cpp"))
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs) + len(dev))) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), srcs + dev))
    prod, dev_objs = objs[:len(srcs)], objs[len(srcs):]
    _link(LIB, prod, force)
    _link(DEVLIB, [o for o in prod if not o.endswith("capi.cpp.o")] + dev_objs, force)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
