"""Build libspecedge.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension)."""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libspecedge.so")
STAMP = LIB + ".sha256"   # source hash of the library build (git-ignored with the .so)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-O3",
    "--expt-relaxed-constexpr", "-Xptxas", "-v",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))) + \
        [os.path.join(HERE, "..", "include", "specedge.h")]


def source_hash() -> str:
    """sha256 over every source / header the library is built from, the flags and the nvcc path:
    the library is reused only if it was built from exactly these bytes (file mtimes are not
    trusted: a snapshot copy or a checkout can leave an old .so newer than changed sources)."""
    h = hashlib.sha256()
    for p in deps():
        h.update(os.path.relpath(p, HERE).encode())
        with open(p, "rb") as f:
            h.update(hashlib.sha256(f.read()).digest())
    h.update(" ".join(FLAGS + [NVCC]).encode())
    return h.hexdigest()


def up_to_date() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return False
    with open(STAMP) as f:
        return f.read().strip() == source_hash()


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """defines / out: experiment builds (e.g. -DSPECEDGE_EMU8=3 into a separate .so, selected at
    load time with SPECEDGE_LIB=path); the default build writes libspecedge.so."""
    lib = out or LIB
    if not force and not defines and out is None and up_to_date():
        return LIB
    objs = []
    procs = []
    tag = "" if not defines else "_" + "_".join(d.replace("=", "") for d in defines)
    for src in sources():
        obj = os.path.join(CSRC, os.path.basename(src)[:-3] + tag + ".o")
        objs.append(obj)
        cmd = [NVCC] + [f for f in FLAGS if f != "-shared"] + [f"-D{d}" for d in defines] + \
            ["-c", src, "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        if verbose or p.returncode != 0:
            sys.stderr.write(out)
        if p.returncode != 0:
            failed = True
    if failed:
        raise RuntimeError("nvcc failed")
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib + ".tmp"] + objs + ["-ldl"]
    subprocess.run(cmd, check=True)
    os.replace(lib + ".tmp", lib)
    for o in objs:
        os.remove(o)
    if lib == LIB and not defines:
        with open(STAMP, "w") as f:
            f.write(source_hash() + "\n")
    elif lib == LIB and os.path.exists(STAMP):
        os.remove(STAMP)
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    defs = [a[len("--define="):] for a in args if a.startswith("--define=")]
    outp = next((a[len("--out="):] for a in args if a.startswith("--out=")), None)
    print(build(force="--force" in args, verbose=not defs, defines=defs, out=outp))
