"""Build libskc.so (sm_100a) in-tree with nvcc.

The shared library is the product: every hot-path call of the package goes
through its C ABI (include/skc.h).  It is built in-tree so it travels with the
repository snapshot to the GPU box; nothing is JIT-compiled at import time.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "build"
LIB = PKG / "libskc.so"
SOURCES = ["skc_api.cu", "skc_filter.cu", "skc_layer.cu", "skc_sparse.cu", "skc_fused.cu", "skc_fit.cu",
           "skc_kawase.cu", "skc_pst.cu", "skc_gather.cu"]
GEN = OBJ / "skc_kawase_gen.inc"      # straight-line pass bodies (csrc/gen_kawase.py)

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
                "-I", str(ROOT / "include"), "-I", str(OBJ)]


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def _headers():
    return [CSRC / "skc_common.cuh", CSRC / "skc_tile.cuh", ROOT / "include" / "skc.h"]


def _generate(force: bool) -> None:
    gen = CSRC / "gen_kawase.py"
    if force or _stale(GEN, [gen]):
        r = subprocess.run([sys.executable, str(gen), str(GEN)], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"gen_kawase.py failed\n{r.stdout}\n{r.stderr}")


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    _generate(force)
    jobs = []
    for src in SOURCES:
        s = CSRC / src
        o = OBJ / (s.stem + ".o")
        deps = [s, *_headers()] + ([GEN] if src == "skc_kawase.cu" else [])
        if force or _stale(o, deps):
            jobs.append([NVCC, *FLAGS, "-c", str(s), "-o", str(o)])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose:
            sys.stdout.write(r.stdout + r.stderr)

    with ThreadPoolExecutor(max_workers=max(1, len(jobs))) as ex:
        list(ex.map(run, jobs))
    objs = [OBJ / (Path(s).stem + ".o") for s in SOURCES]
    if force or jobs or _stale(LIB, objs):
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs), "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
