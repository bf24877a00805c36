"""In-tree build of libsmoe.so (sm_100a) with nvcc; no JIT cache, no torch types."""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libsmoe.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
         "--expt-relaxed-constexpr", "-I", str(ROOT / "include")]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or Path(cand).exists()):
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src, *CSRC.glob("*.cuh"), *CSRC.glob("*.h"), ROOT / "include" / "smoe.h"]
    return any(d.stat().st_mtime > obj.stat().st_mtime for d in deps)


def build(verbose: bool = False, ptxas_info: bool = False, variant: str = "",
          defines: tuple[str, ...] = ()) -> Path:
    """variant: an A/B or instrumented build (`-D` defines) into
    _build/<variant>/ and libsmoe_<variant>.so, loaded with SMOE_LIB=<path>."""
    bdir = BUILD / variant if variant else BUILD
    lib = PKG / f"libsmoe_{variant}.so" if variant else LIB
    bdir.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()
    extra = (["-Xptxas", "-v"] if ptxas_info else []) + [f"-D{d}" for d in defines]

    def compile_one(src: Path) -> Path:
        obj = bdir / (src.stem + ".o")
        if _stale(obj, src) or ptxas_info:
            cmd = [nvcc, *ARCH, *FLAGS, *extra, "-c", str(src), "-o", str(obj)]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
            if ptxas_info or verbose:
                print(r.stderr, file=sys.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(compile_one, sources()))
    if not lib.exists() or any(o.stat().st_mtime > lib.stat().st_mtime for o in objs):
        cmd = [nvcc, *ARCH, "-shared", "-o", str(lib), *map(str, objs)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return lib


if __name__ == "__main__":
    # python -m paper_2503_04398_b200.build [-v] [--ptxas] [--variant NAME -DFOO ...]
    av = sys.argv[1:]
    var = av[av.index("--variant") + 1] if "--variant" in av else ""
    defs = tuple(a[2:] for a in av if a.startswith("-D"))
    print(build(verbose="-v" in av, ptxas_info="--ptxas" in av, variant=var, defines=defs))
