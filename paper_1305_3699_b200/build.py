"""Build libmr_rns.so in-tree: one nvcc translation unit per channel count k (sm_100a), the host
runtime (g++), linked into a single shared library exporting the C ABI of include/mr_rns.h.

    python -m paper_1305_3699_b200.build [--force] [-j N]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# MR_BUILD_OBJ / MR_BUILD_LIB: build a variant (e.g. with MR_NVCC_DEFS) elsewhere, for A/B runs (tools/ab.sh)
OBJ = os.environ.get("MR_BUILD_OBJ") or os.path.join(CSRC, "obj")
LIB = os.environ.get("MR_BUILD_LIB") or os.path.join(HERE, "libmr_rns.so")
ROOT = os.path.dirname(HERE)
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
KS = [1, 2, 3, 5, 9, 17, 33, 49, 65, 97, 129]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                  "-I", os.path.join(ROOT, "include")] + os.environ.get("MR_NVCC_DEFS", "").split()


def _deps() -> list[str]:
    return [os.path.join(CSRC, f) for f in ("mr_kernels.cuh", "mr_tcw.cuh", "mr_internal.h")] + [
        os.path.join(ROOT, "include", "mr_rns.h")]


def _stale(out: str, srcs: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def _run(cmd: list[str], log: str) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ... (see {log})")


def build(force: bool = False, jobs: int | None = None) -> str:
    os.makedirs(OBJ, exist_ok=True)
    deps = _deps()
    steps = []
    objs = []
    for k in KS:
        src = os.path.join(CSRC, f"mr_k{k}.cu")
        obj = os.path.join(OBJ, f"mr_k{k}.o")
        objs.append(obj)
        if force or _stale(obj, [src] + deps):
            steps.append(([NVCC] + NVFLAGS + ["-c", src, "-o", obj], obj + ".log"))
    for cu in ("mr_keygen", "mr_wide", "mr_lanes", "mr_drbg", "mr_tcw257", "mr_tcw505"):
        src = os.path.join(CSRC, cu + ".cu")
        obj = os.path.join(OBJ, cu + ".o")
        objs.append(obj)
        extra = []
        if force or _stale(obj, [src] + deps + extra):
            steps.append(([NVCC] + NVFLAGS + ["-c", src, "-o", obj], obj + ".log"))
    for cpp in ("mr_host", "mr_keygen_host"):
        host_src = os.path.join(CSRC, cpp + ".cpp")
        host_obj = os.path.join(OBJ, cpp + ".o")
        objs.append(host_obj)
        if force or _stale(host_obj, [host_src] + deps):
            steps.append((["g++", "-O2", "-std=c++17", "-fPIC", "-Wall", "-fvisibility=hidden",
                           "-I", os.path.join(CUDA, "include"), "-c", host_src, "-o", host_obj]
                          + [d for d in os.environ.get("MR_NVCC_DEFS", "").split() if d.startswith("-D")],
                          host_obj + ".log"))
    if steps:
        jobs = jobs or min(len(steps), os.cpu_count() or 4)
        with cf.ThreadPoolExecutor(jobs) as ex:
            for f in [ex.submit(_run, c, log) for c, log in steps]:
                f.result()
    if force or steps or _stale(LIB, objs):
        tmp = LIB + ".tmp"
        _run([NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart_static", "-lrt", "-lpthread", "-ldl",
                                                         "-Xlinker", "--no-undefined"],
             os.path.join(OBJ, "link.log"))
        shutil.move(tmp, LIB)
    return LIB


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    a = ap.parse_args()
    print(build(a.force, a.j))


if __name__ == "__main__":
    main()
