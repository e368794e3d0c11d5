"""Build libsamu.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
import sysconfig
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libsamu.so")
SOURCES = ["k_sample.cu", "k_simulate.cu", "k_reduce.cu", "k_fit.cu", "samu_host.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir():
    site = sysconfig.get_paths()["purelib"]
    d = os.path.join(site, "nvidia", "nccl")
    if os.path.exists(os.path.join(d, "include", "nccl.h")):
        return d
    return None


def build(force: bool = False, verbose: bool = False) -> str:
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, "samu_internal.cuh"),
                                                       os.path.join(ROOT, "include", "samu.h")]
    # the flags and defines of a build are part of its identity: a variant / debug build (e.g.
    # SAMU_DEFINES=SAMU_K2_STATS) is never mistaken for the default one
    defines = os.environ.get("SAMU_DEFINES", "").split()
    extra = os.environ.get("SAMU_NVCC_EXTRA", "").split()
    stamp_txt = " ".join(["defines:"] + defines + ["extra:"] + extra)
    stamp = SO + ".flags"
    same_flags = os.path.exists(stamp) and open(stamp).read() == stamp_txt
    if (not force and same_flags and os.path.exists(SO)
            and os.path.getmtime(SO) >= max(os.path.getmtime(d) for d in deps)):
        return SO
    nccl = _nccl_dir()
    inc = ["-I", os.path.join(nccl, "include")] if nccl else []
    flags = ARCH + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3"] + inc
    flags += [f"-D{d}" for d in defines]
    flags += extra   # experiments (scripts/variants.sh)
    build_dir = os.path.join(HERE, "build")
    os.makedirs(build_dir, exist_ok=True)

    def one(src):
        obj = os.path.join(build_dir, src.replace(".cu", ".o"))
        cmd = [NVCC] + flags + ["-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose:
            print(r.stderr)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(one, SOURCES))
    link = [NVCC] + ARCH + ["-shared", "-o", SO + ".tmp"] + objs
    if nccl:
        link += ["-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nccl, "lib")]
    else:
        link += ["-lnccl"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(SO + ".tmp", SO)
    with open(stamp, "w") as f:
        f.write(stamp_txt)
    return SO


if __name__ == "__main__":
    import sys
    print(build(force="-f" in sys.argv, verbose="-v" in sys.argv))
