"""Build the in-tree C-ABI library paper_2511_03655_b200/lib/libirk.so.

nvcc compiles the CUDA sources for sm_100a only (-gencode
arch=compute_100a,code=sm_100a), with -lineinfo (ncu source view) and
--fmad=false (no contraction: the canonical IEEE operation sequence is what
is written).  The host tableau (__float128) is compiled by g++.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "lib")
LIB = os.path.join(OUT, "libirk.so")

CU_SOURCES = ["irk_api.cu", "probe.cu"]
CPP_SOURCES = ["tableau.cpp"]
HEADERS = ["fp64.cuh", "problems.cuh", "ens_common.cuh", "ensemble_g1.cuh", "ensemble_g8.cuh", "ensemble_fo.cuh", "ensemble_nbody.cuh", "ensemble_nbody8.cuh", "ensemble_nbody8m.cuh", "ensemble_g8m.cuh", "ensemble_chain.cuh", "nbody_direct.cuh",
           "balance.cuh",
           "tableau.h"]

GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-fno-fast-math", "-Xptxas", "-v", *GENCODE]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _nccl_include() -> str:
    """nccl.h of the torch wheel's NCCL 2.28 (types only; NCCL is dlopen'ed at run time)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in list(spec.submodule_search_locations or []) if spec else []:
        p = os.path.join(base, "nccl", "include")
        if os.path.exists(os.path.join(p, "nccl.h")):
            return p
    return "/usr/include"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in CU_SOURCES + CPP_SOURCES + HEADERS]
    deps += [os.path.join(ROOT, "include", h) for h in ("irk.h", "irk_probe.h")]
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = (), extra_flags: tuple = ()) -> str:
    """Compile libirk.so (or, for A/B experiments, a variant with extra -D flags to `out`)."""
    lib_path = out or LIB
    if not force and out is None and not _stale():
        return LIB
    os.makedirs(OUT, exist_ok=True)
    bdir = os.path.join(OUT, "obj") if out is None else lib_path + ".obj"  # variants build in parallel
    os.makedirs(bdir, exist_ok=True)
    nvcc = _nvcc()
    objs = []
    for src in CPP_SOURCES:
        o = os.path.join(bdir, src + ".o")
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-fno-fast-math", "-c",
                               os.path.join(CSRC, src), "-o", o])
        objs.append(o)
    log = []
    for src in CU_SOURCES:
        o = os.path.join(bdir, src + ".o")
        r = subprocess.run([nvcc, *NVCC_FLAGS, *extra_flags, *[f"-D{x}" for x in defines], "-I", os.path.join(ROOT, "include"),
                            "-I", _nccl_include(), "-c",
                            os.path.join(CSRC, src), "-o", o], capture_output=True, text=True)
        log.append(r.stdout + r.stderr)
        if r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        objs.append(o)
    tmp = lib_path + f".tmp{os.getpid()}"
    os.makedirs(os.path.dirname(lib_path), exist_ok=True)
    subprocess.check_call([nvcc, "-shared", *GENCODE, "-Xcompiler", "-fPIC", "-o", tmp, *objs,
                           "-cudart", "static", "-ldl"])
    os.replace(tmp, lib_path)
    with open(lib_path + ".ptxas.log" if out else os.path.join(OUT, "ptxas.log"), "w") as f:
        f.write("\n".join(log))
    if verbose:
        print("\n".join(log))
    return lib_path


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
