"""Build libqcpgrad.so (sm_100a) in-tree with nvcc.

    python -m paper_2508_17522_b200.build

The shared library lands in ``paper_2508_17522_b200/_lib/`` so it travels
with the repository snapshot to the GPU box.
"""

import hashlib
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lib")
SOURCES = ["api.cu", "operator.cu", "assembly.cu", "cones.cu", "transpose.cu", "sell.cu", "comm.cu", "engine.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "-I", os.path.join(ROOT, "include"),
]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose=False, force=False, out=None, defines=()):
    """Compile every source and link libqcpgrad.so into ``out`` (default ``_lib/``).

    ``defines`` (e.g. ``["QG_PSD_DMMA=0"]``) builds an A/B variant of the
    compile-time switches; load it with ``QG_LIB_PATH``.
    """
    default_out = out is None or os.path.abspath(out) == os.path.abspath(globals()["OUT"])
    if defines and default_out:
        raise ValueError("variant builds (defines) must go to their own --out directory, not the production _lib/")
    OUT = out or globals()["OUT"]
    os.makedirs(OUT, exist_ok=True)
    # objects compiled with other flags / defines are never reused: the stamp
    # holds a hash of the compile line; a mismatch forces a full rebuild
    stamp = os.path.join(OUT, ".build_stamp")
    want = hashlib.sha256("\0".join(NVCC_FLAGS + sorted(defines)).encode()).hexdigest()
    try:
        with open(stamp) as f:
            force = force or f.read().strip() != want
    except OSError:
        force = True
    headers = [os.path.join(SRC, f) for f in os.listdir(SRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(ROOT, "include", "qcpgrad.h"))
    objs = []

    def compile_one(src):
        s = os.path.join(SRC, src)
        o = os.path.join(OUT, src.replace(".cu", ".o"))
        if force or _newer(o, [s] + headers):
            cmd = [nvcc()] + NVCC_FLAGS + [f"-D{d}" for d in defines] + ["-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd))
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        return o

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    lib = os.path.join(OUT, "libqcpgrad.so")
    if force or _newer(lib, objs):
        cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
               "-o", lib] + objs + ["-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    with open(stamp, "w") as f:
        f.write(want)
    return lib


if __name__ == "__main__":
    # python -m paper_2508_17522_b200.build [-v] [-f] [--out DIR] [-D NAME=VAL ...]
    a = sys.argv[1:]
    out = a[a.index("--out") + 1] if "--out" in a else None
    defs = [a[i + 1] for i, x in enumerate(a) if x == "-D"]
    print(build(verbose="-v" in a, force="-f" in a, out=out, defines=defs))
