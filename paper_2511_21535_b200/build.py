"""Build libp2p.so in-tree: nvcc for sm_100a only (-gencode arch=compute_100a,code=sm_100a), -lineinfo so ncu's
source page maps to the kernels.  Called by __graft_entry__.build(); also runnable as
`python -m paper_2511_21535_b200.build`."""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libp2p.so")
BUILD = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    if spec and spec.submodule_search_locations:
        for base in spec.submodule_search_locations:
            d = os.path.join(base, "nccl")
            if os.path.exists(os.path.join(d, "include", "nccl.h")):
                return d
    raise RuntimeError("NCCL wheel (nvidia/nccl) not found next to torch")


FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _compile(src: str, incs) -> tuple:
    obj = os.path.join(BUILD, os.path.basename(src).replace(".cu", ".o"))
    extra = os.environ.get("P2P_NVCC_FLAGS", "").split()  # experiments only (e.g. -DP2P_RS_MATCH)
    cmd = [NVCC, *FLAGS, *extra, *incs, "-c", src, "-o", obj]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{p.stderr}")
    return obj, p.stderr


STAMP = OUT + ".flags"  # the flag set libp2p.so was built with: a different P2P_NVCC_FLAGS forces a rebuild


def _flag_stamp() -> str:
    return " ".join([NVCC, *FLAGS, *os.environ.get("P2P_NVCC_FLAGS", "").split()])


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = srcs + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.hpp")) + \
        [os.path.join(ROOT, "include", "p2p.h"), __file__]
    stamp_ok = os.path.exists(STAMP) and open(STAMP).read() == _flag_stamp()
    if not force and stamp_ok and os.path.exists(OUT) and \
            os.path.getmtime(OUT) >= max(os.path.getmtime(d) for d in deps):
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    nccl = _nccl_dir()
    incs = ["-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", os.path.join(nccl, "include")]
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        res = list(ex.map(lambda s: _compile(s, incs), srcs))
    if verbose:
        for obj, log in res:
            print(log, file=sys.stderr)
    with open(os.path.join(BUILD, "ptxas.log"), "w") as f:
        for obj, log in res:
            f.write(f"== {os.path.basename(obj)}\n{log}\n")
    tmp = OUT + ".tmp%d" % os.getpid()
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *[o for o, _ in res],
           "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nccl, "lib")]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"link failed:\n{p.stderr}")
    os.replace(tmp, OUT)
    with open(STAMP, "w") as f:
        f.write(_flag_stamp())
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
