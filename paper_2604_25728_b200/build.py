"""Build libsqngd.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels
with the repo snapshot to the GPU box)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsqngd.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_path() -> str:
    try:
        import nvidia.nccl  # noqa: F401

        for p in nvidia.nccl.__path__:
            cand = os.path.join(p, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                return cand
    except Exception:
        pass
    return "libnccl.so.2"


def flags(verbose: bool = False) -> list[str]:
    f = [
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-O3", "-lineinfo", "--std=c++17",
        "-Xcompiler", "-fPIC",
        "-I", os.path.join(ROOT, "include"),
        f'-DSQNGD_NCCL_PATH="{_nccl_path()}"',
    ]
    if verbose:
        f += ["-Xptxas", "-v"]
    return f


def sources() -> list[str]:
    # translation units compiled in parallel: the AF/loss/gradient path, the generator, the Alg. 1 driver
    return [os.path.join(CSRC, "sqngd.cu"), os.path.join(CSRC, "net.cu"), os.path.join(CSRC, "run.cu")]


def deps(src: str | None = None) -> list[str]:
    """Files a translation unit depends on (all of csrc/ and the header when src is None)."""
    hdr = os.path.join(ROOT, "include", "sqngd.h")
    allf = [p for p in glob.glob(os.path.join(CSRC, "*")) if not p.endswith(".o")]
    if src is None:
        return sorted(allf + [hdr])
    if os.path.basename(src) == "net.cu":
        return [src] + [os.path.join(CSRC, f) for f in ("net.cuh", "adam.cuh")]
    if os.path.basename(src) == "run.cu":
        return [src, os.path.join(CSRC, "run.cuh"), hdr]
    return sorted([p for p in allf if os.path.basename(p) not in ("net.cu", "run.cu")] + [hdr])


def build(force: bool = False, verbose: bool = False) -> str:
    newest = max(os.path.getmtime(p) for p in deps())
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= newest:
        return LIB
    objs, procs = [], []
    for src in sources():  # objects are kept (git-ignored) so an unchanged unit is not recompiled
        obj = os.path.join(CSRC, os.path.basename(src) + ".o")
        objs.append(obj)
        stale = force or not os.path.exists(obj) or os.path.getmtime(obj) < max(
            os.path.getmtime(p) for p in deps(src))
        if stale:
            procs.append(subprocess.Popen([NVCC, *flags(verbose), "-c", "-o", obj + ".tmp", src]))
            procs[-1].obj = obj
    rcs = [p.wait() for p in procs]
    if any(rcs):
        raise subprocess.CalledProcessError(max(rcs), "nvcc")
    for p in procs:
        os.replace(p.obj + ".tmp", p.obj)
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB + ".tmp",
                           *objs, "-ldl"])
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
