"""Build the sm_100a shared library `libblade_ms.so` in-tree with nvcc (no JIT cache).

    python -m paper_1802_06130_b200.build [--force]

Flags: -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo, static cudart.
No --use_fast_math: the selector's div/atan2 must stay IEEE (H1; the FAST selector's
strength / coherence tests use sqrt.approx.f32 explicitly, R22).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIB = PKG / "libblade_ms.so"
SOURCES = [CSRC / "blade_ms.cu", CSRC / "tab_down.cu", CSRC / "tab_stage.cu", CSRC / "tab_stage_pairs.cu",
           CSRC / "tab_stage_pairs2.cu", CSRC / "tab_stage_gbank.cu", CSRC / "tab_stage_ch3wide.cu", CSRC / "tab_tma.cu", CSRC / "tab_tma_ch3wide.cu",
           CSRC / "tab_ph.cu", CSRC / "tab_train.cu", CSRC / "tab_train_pairs.cu"]
DEPS = SOURCES + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [INCLUDE / "blade_ms.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, extra: list[str] | None = None,
          out: Path | None = None) -> Path:
    """Compile every translation unit in parallel (nvcc -c), then link the shared library."""
    from concurrent.futures import ThreadPoolExecutor
    lib = out or LIB
    if out is None and not force and not needs_build():
        return lib
    objdir = PKG.parent / "build" / ("obj" if out is None else f"obj_{lib.stem}")
    objdir.mkdir(parents=True, exist_ok=True)
    flags = ["-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-I", str(INCLUDE),
             *(extra or [])]
    if verbose:
        flags.append("-Xptxas=-v")

    def compile_one(src: Path) -> Path:
        obj = objdir / (src.stem + ".o")
        subprocess.check_call([nvcc(), *flags, "-c", "-o", str(obj), str(src)])
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = lib.with_suffix(f".so.tmp{os.getpid()}")
    subprocess.check_call([nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs)])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
