"""Build the sm_100a C-ABI library in-tree.

    python -m paper_2502_03000_b200.build

nvcc cross-compiles for B200 without a GPU.  Output:
paper_2502_03000_b200/_lib/liblm_b200.so (git-ignored, travels to the GPU
box with the repo snapshot).  Links the CUDA runtime dynamically so the
process shares torch's runtime instance (same primary context, same
current device), plus NVRTC for the element-wise program JIT.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import pathlib
import shutil
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
OBJ = ROOT / "build" / "obj"
LIB_DIR = PKG / "_lib"
LIB = LIB_DIR / "liblm_b200.so"
CUDA_HOME = pathlib.Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include():
    """nccl.h of the NCCL torch ships (the library is dlopen'ed at run time)."""
    for site in sys.path:
        inc = pathlib.Path(site) / "nvidia" / "nccl" / "include"
        if (inc / "nccl.h").exists():
            return [f"-I{inc}"]
    return []


NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
                     "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills", f"-I{INCLUDE}", f"-I{CSRC}",
                     "-cudart", "shared"] + _nccl_include()


def sources():
    return sorted(CSRC.glob("*.cu"))


def _needs(target: pathlib.Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _compile(src: pathlib.Path, verbose: bool) -> pathlib.Path:
    obj = OBJ / (src.stem + ".o")
    headers = list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    if _needs(obj, [src, *headers]):
        cmd = [NVCC, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> pathlib.Path:
    if shutil.which(NVCC) is None and not pathlib.Path(NVCC).exists():
        raise RuntimeError("nvcc not found; set CUDA_HOME")
    if force and OBJ.exists():
        shutil.rmtree(OBJ)
    OBJ.mkdir(parents=True, exist_ok=True)
    LIB_DIR.mkdir(parents=True, exist_ok=True)
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if force or _needs(LIB, objs):
        tmp = LIB.with_suffix(f".so.{os.getpid()}.tmp")
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "shared", "-o", str(tmp), *map(str, objs),
               f"-L{CUDA_HOME / 'lib64'}", "-lnvrtc", "-ldl", "-Xlinker", f"-rpath,{CUDA_HOME / 'lib64'}"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
