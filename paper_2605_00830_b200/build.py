"""Build libfastged.so in-tree: nvcc for sm_100a, -lineinfo, shared C ABI (include/fastged.h)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libfastged.so")
SRCS = [os.path.join(HERE, "csrc", "fastged.cu")]
DEPS = SRCS + [os.path.join(HERE, "csrc", f) for f in ("batch_kernel.cuh", "large_kernel.cuh",
                                                       "shard_host.inc", "editpath.inc")] + \
    [os.path.join(ROOT, "include", "fastged.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O2,-Wall,-fopenmp", "-Xptxas", "-v", "-shared",
]


def nccl_dir() -> str:
    """NCCL headers/library shipped with the torch wheels (nvidia-nccl-cu12)."""
    try:
        import nvidia.nccl
        return os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
    except Exception:
        return "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl"


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _stamp(flags) -> str:
    """What the in-tree library was built from: the nvcc flags (an A/B or debug build must never be
    mistaken for the product build)."""
    return " ".join(flags)


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    if any(os.path.getmtime(d) > t for d in DEPS):
        return True
    try:
        with open(LIB + ".flags") as f:
            return f.read() != _stamp(NVCC_FLAGS)
    except OSError:
        return True


def build(force: bool = False, verbose: bool = False, out: str = None, extra_flags=()) -> str:
    """Build the product library in-tree (LIB), or -- with `out` -- a variant with `extra_flags`
    (A/B or debug builds) at `out`, leaving the in-tree library untouched."""
    flags = list(NVCC_FLAGS) + list(extra_flags)
    if out is None:
        if extra_flags:
            raise ValueError("variant builds need an output path outside the package")
        if not force and not stale():
            return LIB
    target = out or LIB
    tmp = target + f".tmp{os.getpid()}"
    nd = nccl_dir()
    cmd = [nvcc(), *flags, "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include"), "-o", tmp, *SRCS,
           "-lcudart", "-lgomp", "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath," + os.path.join(nd, "lib")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "csrc", "ptxas.log") if out is None else target + ".ptxas.log"
    with open(log, "w") as f:
        f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libfastged.so (see %s)" % log)
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, target)
    if out is None:
        with open(LIB + ".flags", "w") as f:
            f.write(_stamp(flags))
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
