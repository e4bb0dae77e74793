"""Build the sm_100a C-ABI library in-tree: paper_1908_04081_b200/_lib/libsscg.so.

    python -m paper_1908_04081_b200.build [--force]

Plain nvcc (no torch extension machinery): every .cu under csrc/ is compiled
for `-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`; small.cu (the
scalar control kernel) additionally with `-fmad=false` so its arithmetic rounds
op by op like the reference's Python floats.  The CUDA runtime is linked
statically, so the .so only needs the driver on the GPU box.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libsscg.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["mpk.cu", "tmarch.cu", "gram.cu", "rec.cu", "small.cu", "hscg.cu", "setup.cu", "dist.cu", "plan.cu"]
NO_FMAD = {"small.cu", "hscg.cu"}


def nvcc():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA library cannot be built")


def nccl_include():
    """nccl.h for the (dlopen'ed) NCCL types: the torch-bundled one, else the system one."""
    try:
        import nvidia.nccl  # noqa: F401
        for base in nvidia.nccl.__path__:
            inc = os.path.join(base, "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return inc
    except Exception:
        pass
    return "/usr/include"


def nccl_library():
    """libnccl.so.2 to dlopen at run time (same copy torch.distributed uses)."""
    try:
        import nvidia.nccl  # noqa: F401
        for base in nvidia.nccl.__path__:
            lib = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(lib):
                return lib
    except Exception:
        pass
    return "libnccl.so.2"


def _digest():
    h = hashlib.sha256()
    for name in sorted(os.listdir(CSRC)) + ["../../include/sscg.h", "../build.py"]:
        path = os.path.normpath(os.path.join(CSRC, name))
        if os.path.isfile(path):
            h.update(name.encode())
            with open(path, "rb") as f:
                h.update(f.read())
    return h.hexdigest()


def build(force=False, verbose=False, out=None, defines=()):
    """Compile (if sources changed) and return the path of libsscg.so
    (`out` / `defines`: side builds of experimental variants)."""
    os.makedirs(OUT_DIR, exist_ok=True)
    lib_path = out or LIB
    stamp = lib_path + ".sha256" if out else os.path.join(OUT_DIR, "libsscg.sha256")
    dig = _digest() + "".join(defines)
    if not force and os.path.exists(lib_path) and os.path.exists(stamp):
        with open(stamp) as f:
            if f.read().strip() == dig:
                return lib_path
    cc = nvcc()
    objs = []
    base = [cc, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", INCLUDE,
            "-I", nccl_include(), "--expt-relaxed-constexpr"] + ARCH + ["-D" + d for d in defines]
    cmds = []
    for src in SOURCES:
        obj = os.path.join(OUT_DIR, (os.path.basename(lib_path) + "." if out else "") +
                           src.replace(".cu", ".o"))
        cmds.append(base + (["-fmad=false"] if src in NO_FMAD else []) + [
            "-c", os.path.join(CSRC, src), "-o", obj])
        objs.append(obj)
    # translation units compile independently: one nvcc per source, in parallel
    from concurrent.futures import ThreadPoolExecutor
    jobs = max(1, min(len(cmds), int(os.environ.get("SSCG_BUILD_JOBS", os.cpu_count() or 1))))
    with ThreadPoolExecutor(jobs) as ex:
        for cmd, proc in zip(cmds, ex.map(lambda c: subprocess.run(c, capture_output=True,
                                                                     text=True), cmds)):
            if verbose:
                print(" ".join(cmd))
                sys.stdout.write(proc.stdout + proc.stderr)
            if proc.returncode != 0:
                sys.stderr.write(proc.stdout + proc.stderr)
                raise subprocess.CalledProcessError(proc.returncode, cmd)
    tmp = lib_path + ".tmp"
    cmd = [cc, "-shared", "-o", tmp] + objs + ARCH + ["-cudart", "static", "-ldl",
                                                       "-Xlinker", "--no-undefined"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib_path)
    for o in objs:
        os.remove(o)
    with open(stamp, "w") as f:
        f.write(dig)
    return lib_path


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
