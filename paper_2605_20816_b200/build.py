"""In-tree build of libpgx.so for sm_100a (nvcc, no JIT cache).

Each kernel family is its own translation unit (csrc/k_*.cu, plus the C ABI in
csrc/pgx_api.cu); they compile in parallel and link into one shared library.
"""

from __future__ import annotations

import os
import subprocess
import time
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "lib")
OBJ_DIR = os.path.join(LIB_DIR, "obj")
LIB_PATH = os.path.join(LIB_DIR, "libpgx.so")
ROOT = os.path.dirname(HERE)

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "-I", os.path.join(ROOT, "include")]


# units compiled once per instantiation subset (see PGX_INST_SET in the source)
SPLIT = {
    "k_grid1.cu": ["PGX_INST_2D_LO", "PGX_INST_2D_6", "PGX_INST_2D_7", "PGX_INST_2D_8",
                   "PGX_INST_3D_LO", "PGX_INST_3D_3", "PGX_INST_3D_4"],
    "k_grid2.cu": ["PGX_INST_2D_LO", "PGX_INST_2D_6", "PGX_INST_2D_7", "PGX_INST_2D_8",
                   "PGX_INST_3D_LO", "PGX_INST_3D_3", "PGX_INST_3D_4"],
}


def sources() -> list[tuple[str, str | None]]:
    out = []
    for f in sorted(f for f in os.listdir(CSRC) if f.endswith(".cu")):
        out += [(f, s) for s in SPLIT[f]] if f in SPLIT else [(f, None)]
    return out


def _newest_dep() -> float:
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(ROOT, "include", "pgx.h"))
    deps.append(os.path.abspath(__file__))
    return max(os.path.getmtime(d) for d in deps)


def _compile(unit: tuple[str, str | None]) -> tuple[str, int, str]:
    src, subset = unit
    obj = os.path.join(OBJ_DIR, src[:-3] + (f".{subset}" if subset else "") + ".o")
    extra = [f"-DPGX_INST_SET={subset}"] if subset else []
    extra += os.environ.get("PGX_XFLAGS", "").split()  # experiment defines (tools/mkvar.sh)
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
    t0 = time.time()
    proc = subprocess.run(cmd, capture_output=True, text=True)
    return obj, proc.returncode, f"[{time.time() - t0:.0f} s]\n" + proc.stdout + proc.stderr


def build_library(force: bool = False, verbose: bool = False) -> str:
    """Compile csrc/*.cu into lib/libpgx.so (skipped when up to date)."""
    os.makedirs(OBJ_DIR, exist_ok=True)
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= _newest_dep():
        return LIB_PATH
    srcs = sources()
    with ThreadPoolExecutor(max_workers=min(len(srcs), max(1, os.cpu_count() or 1))) as ex:
        results = list(ex.map(_compile, srcs))
    with open(os.path.join(LIB_DIR, "ptxas.log"), "w") as f:
        for (obj, rc, log), src in zip(results, srcs):
            f.write(f"==== {src[0]} {src[1] or ''} (rc={rc})\n{log}")
    bad = [(src, log) for (obj, rc, log), src in zip(results, srcs) if rc != 0]
    if bad:
        src, log = bad[0]
        raise RuntimeError(f"nvcc failed on {src[0]} {src[1] or ''}:\n{log[-4000:]}")
    tmp = LIB_PATH + ".tmp"
    link = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", *[r[0] for r in results], "-o", tmp]
    proc = subprocess.run(link, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{proc.stderr[-4000:]}")
    if verbose:
        print(proc.stderr[-2000:])
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    print(build_library(force=True))
