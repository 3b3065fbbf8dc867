"""Build libb200hydro.so in-tree for sm_100a (nvcc, no JIT cache).

    python -m paper_2112_07075_b200.build [--force]
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "hx_api.cu")
DEPS = [os.path.join(HERE, "csrc", f) for f in ("hx_api.cu", "hx_core.cuh", "hx_kernels.cuh", "hx_brick.cuh", "hx_rates.cuh", "hx_remap.cuh", "hx_peer.cuh", "hx_tma.cuh", "hx_node.cuh", "hx_async.cuh")] + [
    os.path.join(ROOT, "include", "b200hydro.h")]
OUT = os.path.join(HERE, "libb200hydro.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force: bool = False, verbose: bool = True) -> str:
    if not force and up_to_date():
        return OUT
    extra = os.environ.get("HX_NVCC_EXTRA", "").split()
    cmd = [NVCC, *FLAGS, *extra, "-o", OUT + ".tmp", SRC]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv)
