"""Build the native library in-tree: nvcc for sm_100a, no JIT cache.

    python -m paper_1302_2073_b200.build
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
# translation units, compiled in parallel and linked into one library
SRCS = [PKG / "csrc" / n for n in ("prost_b200.cu", "tmem_k.cu", "tmem_blk_k.cu", "tmem_cl_k.cu", "resident_k.cu")]
DEPS = sorted((PKG / "csrc").glob("*.cu*")) + sorted((ROOT / "include").glob("*.h")) + [
    Path(__file__).resolve()]
OUT = PKG / "_lib" / "libprost_b200.so"

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC", f"-I{ROOT / 'include'}",
    # fp32 denormals flushed: every penalty input is >= mu > 0, and rsqrtf then
    # maps to a single MUFU.RSQ (the fp64 parity instantiation is unaffected)
    "-ftz=true",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or Path(cand).exists()):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not OUT.exists():
        return False
    t = OUT.stat().st_mtime
    return all(d.stat().st_mtime <= t for d in DEPS)


def build(force: bool = False, verbose: bool = False, out: Path = OUT, extra=()) -> Path:
    """Compile every translation unit (in parallel) and link the shared
    library; `extra` adds nvcc flags (experiment variants, e.g. -DPROST_WC=3)."""
    if not force and out == OUT and not extra and up_to_date():
        return OUT
    out.parent.mkdir(parents=True, exist_ok=True)
    objdir = PKG / "_lib" / "obj" / out.stem
    objdir.mkdir(parents=True, exist_ok=True)
    procs = []
    for src in SRCS:
        obj = objdir / (src.stem + ".o")
        cmd = [nvcc(), *NVCC_FLAGS, *extra, "-c", "-o", str(obj), str(src)]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((subprocess.Popen(cmd), obj))
    failed = [obj for p, obj in procs if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, f"nvcc ({', '.join(o.name for o in failed)})")
    tmp = out.with_suffix(".so.tmp")
    link = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(tmp),
            *[str(obj) for _, obj in procs]]
    if verbose:
        print(" ".join(link), flush=True)
    subprocess.run(link, check=True)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if a != "--force"]
    out = Path(args[0]) if args and not args[0].startswith("-") else OUT
    extra = [a for a in args if a.startswith("-D")]
    print(build(force="--force" in sys.argv, verbose=True, out=out, extra=extra))
