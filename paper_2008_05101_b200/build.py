"""Build libternkit_b200.so in-tree with nvcc for sm_100a (no JIT cache).

Translation units compile in parallel (one nvcc per .cu), then link into the
shared library.  `profile=True` builds tools/libternkit_b200_profile.so with
-DTK_PROFILE: the experiment knobs and in-kernel timestamps of
csrc/tk_internal.cuh compiled in, for the A/B scripts under tools/ only; the
product library never reads the environment.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libternkit_b200.so")
PROFILE_OUT = os.path.join(os.path.dirname(HERE), "tools", "libternkit_b200_profile.so")
SOURCES = ["tk_api.cu", "tk_codec.cu", "tk_popc.cu", "tk_tc.cu", "tk_net.cu", "tk_mlp.cu", "tk_binary.cu", "tk_stem.cu"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    *ARCH,
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xcompiler", "-ffp-contract=off",  # host fuse_bn uses explicit fmaf only
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    return "nvcc"


def sources() -> list[str]:
    return [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]


def needs_build(out: str = OUT) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = sources() + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    deps.append(os.path.join(HERE, "..", "include", "ternkit_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, profile: bool = False) -> str:
    out = PROFILE_OUT if profile else OUT
    if not force and not needs_build(out):
        return out
    flags = NVCC_FLAGS + (["-DTK_PROFILE"] if profile else []) + (["-Xptxas=-v"] if verbose else [])
    objdir = os.path.join(os.path.dirname(out), ".obj_profile" if profile else ".obj")
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src: str) -> str:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [nvcc(), *flags, "-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(f"nvcc failed on {os.path.basename(src)}:\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        return obj

    srcs = sources()
    with ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(compile_one, srcs))
    subprocess.run([nvcc(), *ARCH, "-shared", "-o", out + ".tmp", *objs], check=True, cwd=CSRC)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, profile="--profile" in sys.argv))
