"""Build the native library in-tree: paper_2009_02823_b200/libsvgb200.so (sm_100a).

    python -m paper_2009_02823_b200._build

The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsvgb200.so")
SOURCES = ["engine.cu", "kernels.cu", "kernels_reg.cu", "jit.cu", "plan.cpp"]
# device headers embedded into the library for the run-time compiled pass kernels (jit.cu)
JIT_HEADERS = [("kHdrDevice", "device.cuh"), ("kHdrTileOps", "tile_ops.cuh"), ("kHdrRegOps", "reg_ops.cuh")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "svgrad_b200.h")]
    if not force and not _stale(LIB, deps):
        return LIB
    objs = []
    tmp = os.path.join(PKG, "_obj")
    os.makedirs(tmp, exist_ok=True)
    with open(os.path.join(tmp, "jit_headers.inc"), "w") as f:
        for name, fname in JIT_HEADERS:
            with open(os.path.join(CSRC, fname)) as h:
                text = h.read()
            assert ")SVGB\"" not in text
            f.write(f'static const char {name}[] = R"SVGB({text})SVGB";\n')
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-lineinfo", "-I", os.path.join(ROOT, "include"), "-I", tmp]
    headers = [d for d in deps if not d.endswith((".cu", ".cpp"))]
    cmds = []
    for src in SOURCES:
        obj = os.path.join(tmp, src + ".o")
        objs.append(obj)
        if not force and not _stale(obj, [os.path.join(CSRC, src), *headers]):
            continue  # incremental: object newer than its source and every header
        cmd = [nvcc(), *ARCH, *common, "-Xptxas", "-v" if verbose else "-O3", "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cpp"):
            cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-g", "-I", os.path.join(ROOT, "include"),
                   "-c", os.path.join(CSRC, src), "-o", obj]
        cmds.append(cmd)
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        for fut in [ex.submit(subprocess.run, c, check=True) for c in cmds]:
            fut.result()
    tmp_lib = LIB + ".tmp"
    subprocess.run([nvcc(), *ARCH, "-shared", "-o", tmp_lib, *objs, "-lcudart", "-ldl"], check=True)
    os.replace(tmp_lib, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
