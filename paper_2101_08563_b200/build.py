"""In-tree build of libffca.so (sm_100a) and the oracle test library.

nvcc cross-compiles for sm_100a without a GPU.  Each fit_m<M>.cu holds one
channel count's kernel instantiations so the translation units compile in
parallel; objects are cached under build/ and relinked only when stale.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build"
LIB = PKG / "libffca.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
           "--expt-relaxed-constexpr", "-I", str(ROOT / "include")]
CXXFLAGS = ["-O3", "-std=c++17", "-fPIC", "-Wall", "-I", str(ROOT / "include"),
            "-I", "/usr/local/cuda/include"]


def _headers() -> list[Path]:
    return sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.hpp")) + \
        sorted((ROOT / "include").rglob("*.h*"))


def _stale(obj: Path, src: Path, deps: list[Path]) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(d.stat().st_mtime > t for d in [src, *deps])


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")


def build_lib(verbose: bool = False, jobs: int | None = None) -> Path:
    BUILD.mkdir(exist_ok=True)
    deps = _headers()
    cu = sorted(CSRC.glob("*.cu"))
    cpp = sorted(CSRC.glob("*.cpp"))
    jobs_list = []
    objs = []
    for src in cu:
        obj = BUILD / (src.stem + ".o")
        objs.append(obj)
        if _stale(obj, src, deps):
            jobs_list.append([NVCC, *ARCH, *NVFLAGS, "-c", str(src), "-o", str(obj)])
    for src in cpp:
        obj = BUILD / (src.stem + ".cpp.o")
        objs.append(obj)
        if _stale(obj, src, deps):
            jobs_list.append(["g++", *CXXFLAGS, "-c", str(src), "-o", str(obj)])
    if jobs_list:
        n = jobs or min(len(jobs_list), os.cpu_count() or 4)
        with cf.ThreadPoolExecutor(n) as ex:
            for cmd, fut in [(c, ex.submit(_run, c)) for c in jobs_list]:
                if verbose:
                    print("[build]", Path(cmd[-3]).name, file=sys.stderr)
                fut.result()
    if jobs_list or not LIB.exists() or any(o.stat().st_mtime > LIB.stat().st_mtime for o in objs):
        _run([NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart"])
    return LIB


def build_oracle() -> None:
    """Test infrastructure only (checker + CPU baseline), never the product."""
    _run(["make", "-s", "-C", str(ROOT / "oracle")])


def build_all(verbose: bool = False) -> None:
    build_oracle()
    build_lib(verbose=verbose)


if __name__ == "__main__":
    build_all(verbose=True)
    print(LIB)
