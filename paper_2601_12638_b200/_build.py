"""Build libpmx.so in-tree with nvcc for sm_100a (no --use_fast_math: the binning
divide, the quantize estimate and the fp16 cast must stay IEEE)."""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
BUILD = ROOT / "build" / "pmx"
LIB = PKG / "libpmx.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-O3",
              f"-I{INCLUDE}", f"-I{CSRC}"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _deps():
    return _sources() + sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h")) + [Path(__file__)]


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in _deps())


def build(force: bool = False, verbose: bool = False, ptxas_verbose: bool = False) -> Path:
    out = Path(os.environ["PMX_BUILD_OUT"]).resolve() if os.environ.get("PMX_BUILD_OUT") else LIB
    if out == LIB and not force and up_to_date():
        return LIB
    # PMX_BUILD_OUT: a variant library (trace / ablation builds) with its own object dir
    bdir = BUILD if out == LIB else BUILD.parent / ("pmx_" + out.parent.name + "_" + out.stem)
    out.parent.mkdir(parents=True, exist_ok=True)
    bdir.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()
    extra = ["-Xptxas", "-v"] if ptxas_verbose else []
    if os.environ.get("PMX_TRACE_BUILD") == "1":  # per-role conv timeline (tools/op_profile.py --trace)
        extra += ["-DPMX_CONV_TRACE"]
    if os.environ.get("PMX_DECODE_TRACE") == "1":  # per-phase decode timeline (experiments only)
        extra += ["-DPMX_DECODE_TRACE"]
    if os.environ.get("PMX_PFN_TRACE") == "1":  # per-phase PFN timeline (experiments only)
        extra += ["-DPMX_PFN_TRACE"]
    if os.environ.get("PMX_ABLATE"):  # epilogue ablation builds (experiments only)
        extra += [f"-DPMX_ABLATE={int(os.environ['PMX_ABLATE'])}"]

    def compile_one(src: Path) -> Path:
        obj = bdir / (src.stem + ".o")
        cmd = [nvcc, *ARCH, *NVCC_FLAGS, *extra, "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{r.stdout}\n{r.stderr}")
        if (verbose or ptxas_verbose) and r.stderr:
            print(r.stderr, file=sys.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, _sources()))
    tmp = out.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ptxas_verbose="--ptxas" in sys.argv)
    print(os.environ.get("PMX_BUILD_OUT", LIB))
