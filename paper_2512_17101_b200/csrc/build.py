"""Build libdgb200.so in-tree with nvcc for sm_100a (cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "libdgb200.so")
SOURCES = ["dgb200.cu", "dgb_nsflux.cu", "dgb_msflux.cu", "dgb_msflux2.cu", "dgb_msflux3.cu", "dgb_msflux4.cu", "dgb_arrayops.cu"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-shared", "-Xcompiler", "-fPIC"]


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = SOURCES + [f for f in os.listdir(HERE) if f.endswith((".cuh", ".h"))] + [os.path.join("..", "..", "include", "dgb200.h")]
    return any(os.path.getmtime(os.path.join(HERE, d)) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines: list[str] | None = None, out: str | None = None,
          sources: list[str] | None = None) -> str:
    """``defines``/``out`` build a tuning variant beside the default library (select it with
    the environment variable DGB_LIB, see _cabi.py); used by scripts/ab_variants.py."""
    if out is None and not force and not needs_build():
        return OUT
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, "--threads", "0"] + FLAGS + (["-Xptxas", "-v"] if verbose else []) + \
          [f"-D{d}" for d in (defines or [])] + ["-o", out or OUT] + (sources or SOURCES)
    res = subprocess.run(cmd, cwd=HERE, capture_output=True, text=True)
    if verbose:
        sys.stderr.write(res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{res.stderr}")
    return out or OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
