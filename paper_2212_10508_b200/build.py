"""In-tree build of libparalangevin_b200.so (sm_100a) with nvcc.

    python -m paper_2212_10508_b200.build        # or __graft_entry__.build()

Every .cu under csrc/ is compiled for ``-gencode arch=compute_100a,code=sm_100a``
with ``-lineinfo`` and linked into one shared library next to this file, so the
.so travels to the GPU box with the repository snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libparalangevin_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _deps_mtime():
    return max(os.path.getmtime(os.path.join(CSRC, f)) for f in os.listdir(CSRC)) if os.listdir(CSRC) else 0


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    newest = max(_deps_mtime(), os.path.getmtime(os.path.join(ROOT, "include", "paralangevin_b200.h")),
                 os.path.getmtime(__file__))
    return os.path.getmtime(LIB) >= newest


def build(force: bool = False, verbose: bool = False, variant: str | None = None, defines=()) -> str:
    """Build the library; ``variant`` + ``defines`` (-DNAME...) make an A/B copy
    libparalangevin_b200_<variant>.so (loaded when PL_LIB_VARIANT=<variant>)."""
    lib_out = LIB if not variant else os.path.join(HERE, f"libparalangevin_b200_{variant}.so")
    obj_dir = OBJ if not variant else os.path.join(OBJ, variant)
    if not variant and not force and up_to_date():
        return LIB
    os.makedirs(obj_dir, exist_ok=True)
    cc = nvcc()

    def one(src):
        obj = os.path.join(obj_dir, src.replace(".cu", ".o"))
        cmd = [cc, *ARCH, *FLAGS, *defines, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        return obj, r.stderr

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as pool:
        results = list(pool.map(one, _sources()))
    if verbose:
        for obj, log in results:
            sys.stderr.write(log)
    with open(os.path.join(obj_dir, "ptxas.log"), "w") as fh:
        for obj, log in results:
            fh.write(f"== {os.path.basename(obj)}\n{log}\n")
    tmp = lib_out + ".tmp"
    cmd = [cc, *ARCH, "-shared", "-o", tmp, *[o for o, _ in results], "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib_out)
    return lib_out


if __name__ == "__main__":
    args = sys.argv[1:]
    var = args[args.index("--variant") + 1] if "--variant" in args else None
    print(build(force="--force" in args, verbose="-v" in args, variant=var,
                defines=[a for a in args if a.startswith("-D")]))
