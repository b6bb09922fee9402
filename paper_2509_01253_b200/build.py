"""Build libsfhr_b200.so in-tree with nvcc for sm_100a (no torch JIT cache).

    python -m paper_2509_01253_b200.build          # incremental
    python -m paper_2509_01253_b200.build --force
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
ROOT = PKG.parent
INCLUDE = ROOT / "include"
OBJ = PKG / "_build"
LIB = PKG / "libsfhr_b200.so"

SOURCES = ["keyswitch.cu", "keyswitch_tc.cu", "ring_ops.cu", "linear_mma.cu", "ntt64.cu", "wire.cu", "capi.cu", "plan.cpp", "perm.cpp"]
# (object name, source, extra -D flags): the stage-kernel template fan-out is
# split into one translation unit per (t, l) so it compiles in parallel
UNITS = [(s, s, []) for s in SOURCES] + [
    (f"keyswitch_t{t}_l{l}.cu", "keyswitch.cu", [f"-DSFHR_KS_T={t}", f"-DSFHR_KS_L={l}"])
    for t in (3, 5, 7) for l in (1, 2, 3, 4, 5)]
HEADERS = ["sfhr_common.cuh", "sfhr_kernels.h", "plan.h", "tc_ptx.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
              "--expt-relaxed-constexpr", f"-I{INCLUDE}", f"-I{CSRC}"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _deps_mtime(src: str | None = None) -> float:
    """Newest input of one unit (its source + shared headers), or of everything."""
    if src is None:
        files = list(CSRC.glob("*")) + list(INCLUDE.glob("*.h"))
    else:
        files = [CSRC / src] + [CSRC / h for h in HEADERS] + list(INCLUDE.glob("*.h"))
    return max(f.stat().st_mtime for f in files)


def _compile(unit, verbose: bool) -> Path:
    name, src, defs = unit
    out = OBJ / (name + ".o")
    if out.exists() and out.stat().st_mtime >= _deps_mtime(src):
        return out
    cmd = [_nvcc(), *ARCH, *NVCC_FLAGS, *defs, "-c", str(CSRC / src), "-o", str(out)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose:
        sys.stderr.write(r.stderr)
    return out


def build_variant(name: str, defines: dict) -> Path:
    """Experimental build with -D macros into lib<name>.so (A/B kernel studies)."""
    out_dir = OBJ / name
    out_dir.mkdir(parents=True, exist_ok=True)
    flags = [f"-D{k}={v}" for k, v in defines.items()]

    def comp(unit):
        name, src, defs = unit
        o = out_dir / (name + ".o")
        cmd = [_nvcc(), *ARCH, *NVCC_FLAGS, *flags, *defs, "-c", str(CSRC / src), "-o", str(o)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(r.stderr)
        return o

    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 8) as ex:
        objs = list(ex.map(comp, UNITS))
    lib = PKG / f"lib{name}.so"
    r = subprocess.run([_nvcc(), *ARCH, "-shared", "-o", str(lib), *map(str, objs), "-lcudart"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(r.stderr)
    return lib


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    if force:
        for f in OBJ.glob("*.o"):
            f.unlink()
    if LIB.exists() and not force and LIB.stat().st_mtime >= _deps_mtime():
        return LIB
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 8) as ex:
        objs = list(ex.map(lambda u: _compile(u, verbose), UNITS))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [_nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
