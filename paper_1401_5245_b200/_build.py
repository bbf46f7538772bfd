"""Build the sm_100a shared library in-tree (no JIT cache: the .so must travel
with the repo snapshot to the GPU box)."""

from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "lib")
LIB_PATH = os.path.join(LIB_DIR, "libbitedge_cuda.so")
# one translation unit per concern, compiled in parallel then linked
SOURCES = ["capi_edges.cu", "capi_words.cu", "capi_p4.cu", "capi_host.cu"]
HEADERS = ["capi_internal.cuh", "edge_tile.cuh", "edge_stream.cuh", "edge_reg.cuh", "edge_flat.cuh",
           os.path.join("..", "..", "include", "bitedge.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


EXT_SRC = "dropin_ext.c"


def ext_path() -> str:
    import sysconfig

    return os.path.join(HERE, "_dropin" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_ext() -> str:
    """The CPython binding of the drop-in's per-image call (csrc/dropin_ext.c),
    linked against the library (rpath $ORIGIN/lib)."""
    import sysconfig

    import numpy

    out = ext_path()
    tmp = out + ".tmp"
    cmd = [os.environ.get("CC", "gcc"), "-O2", "-shared", "-fPIC", "-std=c11",
           "-I", sysconfig.get_paths()["include"], "-I", numpy.get_include(),
           os.path.join(CSRC, EXT_SRC), "-L", LIB_DIR, "-lbitedge_cuda",
           "-Wl,-rpath,$ORIGIN/lib", "-o", tmp]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"extension build failed:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, out)
    return out


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB_PATH) or not os.path.exists(ext_path()):
        return True
    t = min(os.path.getmtime(LIB_PATH), os.path.getmtime(ext_path()))
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS + [EXT_SRC]]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB_PATH
    import concurrent.futures as cf
    import tempfile

    os.makedirs(LIB_DIR, exist_ok=True)
    tmpdir = tempfile.mkdtemp(prefix="bitedge_build_")
    inc = ["-I", os.path.join(ROOT, "include")]

    def compile_one(src):
        obj = os.path.join(tmpdir, os.path.splitext(src)[0] + ".o")
        cmd = [nvcc(), *NVCC_FLAGS, *inc, "-c", "-o", obj, os.path.join(CSRC, src)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
        return obj, res.stderr

    try:
        with cf.ThreadPoolExecutor(len(SOURCES)) as ex:
            results = list(ex.map(compile_one, SOURCES))
        tmp = LIB_PATH + ".tmp"
        cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *[o for o, _ in results]]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc link failed:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
        os.replace(tmp, LIB_PATH)
    finally:
        shutil.rmtree(tmpdir, ignore_errors=True)
    build_ext()
    log = "".join(err for _, err in results)
    if verbose:
        print(log)
    with open(os.path.join(LIB_DIR, "ptxas.log"), "w") as f:
        f.write(log)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force=True, verbose=True))
