"""Build libubqp.so in-tree with nvcc for sm_100a (B200) only.

    python -m paper_1706_00037_b200.build          # or __graft_entry__.build()

Each translation unit is compiled on its own (in parallel, no cross-file device code) and
the objects are linked into one shared library.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libubqp.so"
OBJ = PKG / "_obj"
SOURCES = ["abi.cu", "gen.cu", "eval_tc.cu", "screen.cu", "ascend.cu", "ascend_real.cu", "ascend_sparse.cu", "ascend_warp.cu", "ascend_mw.cu"]
HEADERS = ["ubqp_internal.cuh", "warp_keys.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off",
    "--expt-relaxed-constexpr",
    # no --split-compile: its parallel partitioning made ptxas output vary between builds
]


def _sources():
    return [s for s in SOURCES if (CSRC / s).exists()]


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in _sources() + HEADERS] + [PKG.parent / "include" / "ubqp.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build_lib(force: bool = False, verbose: bool = False, out: Path | None = None) -> Path:
    """Compile every source and link libubqp.so (or `out`, for A/B variants)."""
    target = Path(out) if out else LIB
    if out is None and not force and not _stale():
        return LIB
    OBJ.mkdir(exist_ok=True)
    extra = os.environ.get("UBQP_NVCC_EXTRA", "").split()

    def compile_one(src: str) -> Path:
        obj = OBJ / (src + f".{os.getpid()}.o")
        cmd = [NVCC, *NVCC_FLAGS, *extra, "-c", "-o", str(obj), str(CSRC / src)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        return obj

    with ThreadPoolExecutor(max_workers=len(_sources())) as ex:
        objs = list(ex.map(compile_one, _sources()))
    target.parent.mkdir(parents=True, exist_ok=True)
    tmp = target.with_name(target.name + f".tmp{os.getpid()}")
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
                           "-o", str(tmp), *map(str, objs)])
    for o in objs:
        o.unlink()
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    build_lib(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
