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
CXXFLAGS = ["-O3", "-std=c++17", "-fPIC", "-Wall", "-Wno-class-memaccess", "-I", str(ROOT / "include"),
            "-I", "/usr/local/cuda/include"]


def _headers() -> list[Path]:
    return sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.hpp")) + \
        sorted((ROOT / "include").rglob("*.h*"))


def _includes(src: Path, seen: set | None = None) -> set:
    """Local headers src includes, transitively (quoted includes only)."""
    import re
    seen = set() if seen is None else seen
    for m in re.finditer(r'#include\s+"([^"]+)"', src.read_text()):
        h = (src.parent / m.group(1)).resolve()
        if not h.exists():
            h = (ROOT / "include" / m.group(1)).resolve()
        if h.exists() and h not in seen:
            seen.add(h)
            _includes(h, seen)
    return seen


def _stale(obj: Path, src: Path, deps: list[Path]) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(d.stat().st_mtime > t for d in [src, *deps])


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")


def build_lib(verbose: bool = False, jobs: int | None = None, variant: str = "",
              only: list[str] | None = None) -> Path:
    """Build libffca.so; variant "timing" builds the phase-timing diagnostics
    library libffca_timing.so (-DFFCA_PHASE_TIMING) in build_timing/.
    `only` restricts the CUDA sources (diagnostics builds of one shape)."""
    global LIB
    lib = LIB if not variant else PKG / f"libffca_{variant}.so"
    bdir = BUILD if not variant else ROOT / f"build_{variant}"
    extra = [] if not variant else [f"-DFFCA_PHASE_{variant.upper()}"]
    if variant.startswith("x_"):  # tuning experiments: FFCA_NVCC_EXTRA="-DFOO=1 ..."
        extra = os.environ.get("FFCA_NVCC_EXTRA", "").split()
    bdir.mkdir(exist_ok=True)
    cu = sorted(CSRC.glob("*.cu"))
    cpp = sorted(CSRC.glob("*.cpp"))
    jobs_list = []
    objs = []
    for src in cu:
        obj = bdir / (src.stem + ".o")
        if only and src.stem not in only and src.stem != "ffca_api":
            if variant:  # diagnostics / experiment builds link the production objects
                objs.append(BUILD / (src.stem + ".o"))
            continue
        objs.append(obj)
        if _stale(obj, src, sorted(_includes(src))):
            jobs_list.append([NVCC, *ARCH, *NVFLAGS, *extra, "-c", str(src), "-o", str(obj)])
    for src in cpp:
        obj = bdir / (src.stem + ".cpp.o")
        objs.append(obj)
        if _stale(obj, src, sorted(_includes(src))):
            jobs_list.append(["g++", *CXXFLAGS, "-c", str(src), "-o", str(obj)])
    saved, LIB = LIB, lib
    if jobs_list:
        n = jobs or min(len(jobs_list), os.cpu_count() or 4)
        with cf.ThreadPoolExecutor(n) as ex:
            for cmd, fut in [(c, ex.submit(_run, c)) for c in jobs_list]:
                if verbose:
                    print("[build]", Path(cmd[-3]).name, file=sys.stderr)
                fut.result()
    try:
        if jobs_list or not LIB.exists() or any(o.stat().st_mtime > LIB.stat().st_mtime for o in objs):
            _run([NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart"])
        return LIB
    finally:
        LIB = saved


def build_oracle() -> None:
    """Test infrastructure only (checker + CPU baseline), never the product."""
    _run(["make", "-s", "-C", str(ROOT / "oracle")])


def build_cpp_e2e() -> Path:
    """bench.py's C++-API end-to-end leg (tools/cpp_e2e.cpp) against libffca.so."""
    src = ROOT / "tools" / "cpp_e2e.cpp"
    out = ROOT / "tools" / "cpp_e2e.so"
    if _stale(out, src, [LIB, *sorted((ROOT / "include").rglob("*.h*"))]):
        _run(["g++", "-O2", "-std=c++20", "-fPIC", "-shared", "-Wno-class-memaccess",
              "-I", str(ROOT / "include"), str(src), "-L", str(PKG), "-lffca",
              "-Wl,-rpath," + str(PKG), "-pthread", "-o", str(out)])
    return out


def build_all(verbose: bool = False) -> None:
    build_oracle()
    build_lib(verbose=verbose)
    build_cpp_e2e()


if __name__ == "__main__":
    build_all(verbose=True)
    print(LIB)
