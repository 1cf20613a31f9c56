"""Build libs2o_cuda.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2602_22575_b200.build  [--force]

The .so lands in paper_2602_22575_b200/lib/ (git-ignored, travels to the GPU box).
"""
from __future__ import annotations

import argparse
import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
# S2O_VARIANT_DIR (dev A/B aid): build csrc/ found there into <dir>/lib instead of the package's
_VARIANT = os.environ.get("S2O_VARIANT_DIR")
CSRC = os.path.join(_VARIANT, "csrc") if _VARIANT else os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(_VARIANT, "lib") if _VARIANT else os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libs2o_cuda.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SRCS = ["capi.cu", "plan.cu", "attn_generic.cu", "attn_sm100.cu", "baseline.cu"]
CPP_SRCS = ["synthetic.cpp"]


EXTRA = os.environ.get("S2O_NVCC_FLAGS", "").split()  # e.g. -DS2O_TIMELINE (profiling aid)


def _stamp() -> str:
    h = hashlib.sha1()
    h.update(" ".join(EXTRA).encode())
    for name in sorted(os.listdir(CSRC)) + ["../../include/s2o_cuda.h", "../build.py"]:
        path = os.path.join(CSRC, name)
        if os.path.isfile(path):
            with open(path, "rb") as f:
                h.update(name.encode() + f.read())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(LIB_DIR, exist_ok=True)
    stamp_file = LIB + ".stamp"
    stamp = _stamp()
    if not force and os.path.exists(LIB) and os.path.exists(stamp_file):
        with open(stamp_file) as f:
            if f.read().strip() == stamp:
                return LIB
    obj_dir = os.path.join(LIB_DIR, "obj")
    os.makedirs(obj_dir, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    objs = []
    procs = []
    for src in CU_SRCS:
        obj = os.path.join(obj_dir, src + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-Xptxas", "-v" if verbose else "-O3", "--expt-relaxed-constexpr",
               *EXTRA, *inc, "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    for src in CPP_SRCS:
        obj = os.path.join(obj_dir, src + ".o")
        cmd = ["g++", "-std=c++20", "-O3", "-fPIC", "-ffp-contract=off", "-pthread", *inc,
               "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        text = out.decode(errors="replace")
        if p.returncode != 0:
            failed = True
            sys.stderr.write(f"[build] {src} FAILED\n{text}\n")
        elif verbose and text.strip():
            sys.stderr.write(f"[build] {src}\n{text}\n")
    if failed:
        raise RuntimeError("libs2o_cuda build failed")
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lpthread"]
    subprocess.run(cmd, check=True)
    with open(stamp_file, "w") as f:
        f.write(stamp)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    args = ap.parse_args()
    print(build(force=args.force, verbose=args.verbose))
