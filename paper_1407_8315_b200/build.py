"""Build libsfdt_b200.so in-tree (nvcc for sm_100a, gcc for host tables).

    python -m paper_1407_8315_b200.build        (or __graft_entry__.build())
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsfdt_b200.so")
CU_SOURCES = ["exact.cu", "kernels.cu", "general.cu", "runtime.cu", "dropin.cu"]
C_SOURCES = ["twiddle.c"]
# per-source defines: the exact-path decode chains call the long scalar
# routines (cx.cuh SFDT_HEAVY) instead of inlining them -- 2-2.6x less code per
# kernel, measured faster where the chains are long (tools/decode_kernels.cu)
EXTRA_FLAGS = {"exact.cu": ["-DSFDT_NOINLINE_HEAVY"]}
HEADERS = ["cx.cuh", "common.cuh", "decode.cuh", "decode_coop.cuh", "fft.cuh", "general.cuh"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off", "--fmad=false",
    "-Xptxas", "-O3", "-cudart", "static",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = CU_SOURCES + C_SOURCES + HEADERS
    return any(os.path.getmtime(os.path.join(CSRC, f)) > t for f in deps) or \
        os.path.getmtime(os.path.join(HERE, "..", "include", "sfdt.h")) > t


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return OUT
    nvcc = _nvcc()
    objdir = os.path.join(HERE, "_obj")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for src in C_SOURCES:
        obj = os.path.join(objdir, src + ".o")
        subprocess.run(["gcc", "-O2", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-std=gnu11",
                        "-c", os.path.join(CSRC, src), "-o", obj], check=True)
        objs.append(obj)
    def compile_cu(src):
        obj = os.path.join(objdir, src + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *EXTRA_FLAGS.get(src, []), "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(CU_SOURCES)) as pool:
        objs.extend(pool.map(compile_cu, CU_SOURCES))
    tmp = OUT + ".tmp"
    subprocess.run([nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
                    "-o", tmp, *objs, "-lm"], check=True)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
