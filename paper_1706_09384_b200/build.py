"""Build libhmx.so in-tree for sm_100a (nvcc; no JIT cache, so the .so travels
with the repo snapshot to the GPU box).

    python -m paper_1706_09384_b200.build [--force]
"""

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(HERE, "libhmx.so")
SOURCES = ["capi.cu", "aca.cu", "recompress.cu", "dense.cu", "matvec.cu", "gmres.cu", "estimate.cu", "rsvd.cu", "hlu.cu", "geometry.cpp"]
HEADERS = ["hmx_common.cuh", "green.cuh", "hmatrix.h", "hmx_host.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
         "-diag-suppress", "128,550"] + os.environ.get("HMX_NVCC_EXTRA", "").split()


def _newest_dep():
    deps = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "hmx.h")]
    return max(os.path.getmtime(p) for p in deps)


def _compile(src, force):
    out = os.path.join(OBJ, src + ".o")
    path = os.path.join(CSRC, src)
    if not force and os.path.exists(out):
        if os.path.getmtime(out) >= max(os.path.getmtime(path), _newest_dep()):
            return out
    cmd = [NVCC, *FLAGS, *ARCH, "-c", path, "-o", out]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
    return out


def build(force=False, verbose=True):
    os.makedirs(OBJ, exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), SOURCES))
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, "-shared", *ARCH, "-o", LIB, *objs, "-lcublas", "-lcusolver"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
