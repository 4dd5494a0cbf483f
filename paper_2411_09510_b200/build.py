"""Build libmxb200.so (sm_100a) in-tree with nvcc.

    python -m paper_2411_09510_b200.build

Translation units are compiled in parallel and linked into one shared
library with the CUDA runtime linked statically, so the .so has no
dependency beyond the driver and travels with the repo snapshot.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libmxb200.so")
# objects live outside the repo so the gpurun snapshot carries only the .so
BUILD = os.environ.get("MXB200_BUILD_DIR", "/tmp/mxb200_build")
# -lineinfo (ncu source view) only where the profiled kernels live: it
# roughly doubles object size
LINEINFO = {"k_quant_bf16.cu", "k_dqsum_bf16.cu", "k_fused_inst.cu", "k_requant.cu", "k_gemm.cu"}
# sources compiled several times with -D slices (template instantiation split
# so the slices build in parallel)
VARIANTS = {
    "k_quant_bf16.cu": [{"MXB_B": b} for b in (8, 16, 32, 64)],
    "k_fused_inst.cu": [{"MXB_OUT": o, "MXB_B": b} for o in (0, 1) for b in (8, 16, 32, 64)],
}

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "-I", os.path.join(ROOT, "include")]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found")
    return cand


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _digest(deps) -> str:
    """Content hash of every source and the flags: an edit made while a build
    runs is never mistaken for built (mtimes would be)."""
    import hashlib

    h = hashlib.sha256(repr((ARCH, FLAGS, sorted(LINEINFO), VARIANTS)).encode())
    for d in sorted(deps):
        h.update(os.path.relpath(d, ROOT).encode())  # checkout-independent
        with open(d, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = sources()
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")] + [
        os.path.join(ROOT, "include", "mxb200.h")]
    digest = _digest(deps)
    stamp = OUT + ".digest"
    if not force and os.path.exists(OUT) and os.path.exists(stamp) and \
            open(stamp).read().strip() == digest:
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    nv = nvcc()

    jobs = []
    for src in srcs:
        for var in VARIANTS.get(os.path.basename(src), [{}]):
            jobs.append((src, var))

    headers = [d for d in deps if not d.endswith(".cu")]

    def compile_one(job):
        src, var = job
        tag = "".join(f".{k}{v}" for k, v in var.items())
        obj = os.path.join(BUILD, os.path.basename(src) + tag + ".o")
        extra = ["-lineinfo"] if os.path.basename(src) in LINEINFO else []
        extra += [f"-D{k}={v}" for k, v in var.items()]
        cmd = [nv, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj]
        # object cache: this source + every header + the command line
        key = _digest([src] + headers) + repr(cmd)
        if not force and os.path.exists(obj) and os.path.exists(obj + ".key") and \
                open(obj + ".key").read() == key:
            return obj
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{p.stderr}")
        with open(obj + ".key", "w") as f:
            f.write(key)
        with open(obj + ".ptxas.txt", "w") as f:
            f.write(p.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        # longest jobs first
        jobs.sort(key=lambda j: ("k_fused_inst" not in j[0], "k_quant_bf16" not in j[0]))
        objs = list(ex.map(compile_one, jobs))
    tmp = OUT + ".tmp"
    cmd = [nv, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"link failed:\n{p.stderr}")
    os.replace(tmp, OUT)
    with open(stamp, "w") as f:
        f.write(digest + "\n")
    if verbose:
        print(f"built {OUT}")
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
