"""Build libfdirw.so in-tree with nvcc for sm_100a (B200).  `python -m paper_2408_11376_b200.build`."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libfdirw.so")
SOURCES = ["fdirw_api.cu", "kgen.cu", "kgen_bal.cu", "superpose.cu", "dedup.cu", "coarse.cu", "absorb.cu", "p2p.cu", "comm.cpp"]
HEADERS = ["fdirw_internal.h", "layout.cuh", "bulk.cuh", "mx8.cuh", "kgen_common.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr"]


SHA_FILE = LIB + ".sha256"
LAST_MODE = None  # "compiled" or "reused": what the last build() call did


def source_sha() -> str:
    """sha256 over every source, header, this builder and the nvcc version: the library's
    build id (compiled into it as fdirw_build_id(), and stored beside it)."""
    import hashlib

    h = hashlib.sha256()
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [
        os.path.join(HERE, "..", "include", "fdirw.h"), os.path.abspath(__file__)]
    for d in deps:
        h.update(os.path.basename(d).encode())
        h.update(open(d, "rb").read())
    h.update(" ".join(ARCH + FLAGS).encode())
    try:
        h.update(subprocess.check_output([NVCC, "--version"]))
    except Exception:
        pass
    return h.hexdigest()


def _stale(sha: str) -> bool:
    """Rebuild unless the library on disk was built from exactly these sources (content hash,
    not mtimes: a snapshot copied to another machine keeps its .so only if it still matches)."""
    if not os.path.exists(LIB) or not os.path.exists(SHA_FILE):
        return True
    return open(SHA_FILE).read().strip() != sha


def build(force: bool = False, verbose: bool = False) -> str:
    global LAST_MODE
    sha = source_sha()
    if not force and not _stale(sha):
        LAST_MODE = "reused"
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    cmds, objs = [], []
    for src in SOURCES:
        obj = os.path.join(objdir, src + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, "-DFDIRW_BUILD_ID=\"%s\"" % sha, "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu") and verbose:
            cmd += ["-Xptxas", "-v"]
        if src.endswith(".cpp"):
            cmd = [NVCC, *ARCH, *FLAGS, "-DFDIRW_BUILD_ID=\"%s\"" % sha, "-x", "c++", "-c", os.path.join(CSRC, src),
                   "-o", obj]
        cmds.append(cmd)
        objs.append(obj)
    # the translation units compile independently: one nvcc per source, in parallel
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as ex:
        for rc, cmd in zip(ex.map(subprocess.call, cmds), cmds):
            if rc != 0:
                raise subprocess.CalledProcessError(rc, cmd)
    tmp = LIB + ".tmp%d" % os.getpid()
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-ldl", "-lcudart_static", "-lrt", "-lpthread"])
    os.replace(tmp, LIB)
    with open(SHA_FILE, "w") as f:
        f.write(sha + "\n")
    LAST_MODE = "compiled"
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
