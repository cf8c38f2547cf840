"""In-tree build of the sm_100a kernel library and the CPU oracle.

`build_all()` is what `__graft_entry__.build()` runs: nvcc compiles every
CUDA unit for sm_100a (`-gencode arch=compute_100a,code=sm_100a -lineinfo`)
into `paper_1909_13772_b200/_lbm_b200.so`, and gcc builds the test-only
oracle `oracle/build/liblbm_oracle.so`.  Both land in the source tree so the
snapshot that `gpurun` ships carries them (they are git-ignored).
"""
from __future__ import annotations

import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "_lbm_b200.so"
OBJ = PKG / "build"
ORACLE_DIR = ROOT / "oracle"
ORACLE_LIB = ORACLE_DIR / "build" / "liblbm_oracle.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "--expt-relaxed-constexpr", "-Xptxas", "-v"]
# (source, extra flags): the fp64 unit and the C-ABI unit keep every
# floating-point operation separately rounded (-fmad=false) for bitwise parity
# with the reference; the fp32-storage unit may contract to FMA.
UNITS = [
    ("lbm_inst_f64.cu", ["-fmad=false"]),
    ("lbm_inst_f32.cu", ["-fmad=true"]),
    ("lbm_capi.cu", ["-fmad=false"]),
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the B200 kernel library cannot be built")


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def _run(cmd, log=None):
    res = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        log.write(" ".join(cmd) + "\n" + res.stdout + res.stderr + "\n")
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:4])} ...")
    return res


def build_kernels(force: bool = False, verbose: bool = False, defines=(), out: Path | None = None) -> Path:
    """Build the library.  `defines` / `out` produce tuning variants (e.g.
    defines=("LBM_FUSED_MINB=5",), out=.../_lbm_b200_minb5.so) that
    _lib.load() picks up through LBM_B200_LIB."""
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [ROOT / "include" / "lbm_b200.h"]
    tag = "".join("_" + d.replace("=", "").lower() for d in defines)
    objdir = OBJ / ("default" if not tag else tag.strip("_"))
    objdir.mkdir(parents=True, exist_ok=True)
    lib = out or LIB
    nvcc = _nvcc()
    objs, cmds = [], []
    for src, extra in UNITS:
        s = CSRC / src
        o = objdir / (Path(src).stem + ".o")
        objs.append(o)
        if force or _stale(o, [s, *headers]):
            cmds.append([nvcc, *ARCH, *NVCC_COMMON, *extra, *(f"-D{d}" for d in defines),
                         "-I", str(ROOT / "include"), "-c", str(s), "-o", str(o)])
    with open(objdir / "ptxas.log", "w") as log:
        # the units are independent: compile them concurrently
        with ThreadPoolExecutor(max_workers=len(UNITS)) as pool:
            for cmd in cmds:
                if verbose:
                    print(" ".join(cmd), flush=True)
            for res in pool.map(_run, cmds):
                log.write(res.args[-3] + "\n" + res.stdout + res.stderr + "\n")
        if force or _stale(lib, objs):
            _run([nvcc, *ARCH, "-shared", "-o", str(lib), *map(str, objs), "-lcudart"], log)
    if not tag:
        (OBJ / "ptxas.log").write_text((objdir / "ptxas.log").read_text())
    return lib


def build_oracle(force: bool = False) -> Path:
    src = ORACLE_DIR / "lbm_oracle.c"
    ORACLE_LIB.parent.mkdir(exist_ok=True)
    if force or _stale(ORACLE_LIB, [src]):
        # -ffp-contract=off: no FMA, same per-op rounding as numpy's ufuncs
        _run(["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
              "-fno-fast-math", "-std=c11", "-o", str(ORACLE_LIB), str(src), "-lm"])
    return ORACLE_LIB


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_kernels(force=force, verbose=verbose)
    if (ORACLE_DIR / "lbm_oracle.c").exists():
        build_oracle(force=force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose=True)
