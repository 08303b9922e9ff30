"""Build libsacd.so in-tree for sm_100a with nvcc (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["capi.cu", "kernels.cu", "layout.cu"]
OUT = os.path.join(HERE, "libsacd.so")
# library flavours: the product build, the MTTKRP tuning-variant build (tools/mttkrp_tune.py,
# test_mttkrp_variants_bitwise) and the device-assert build (tests/test_debug_build.py)
FLAVOURS = {"default": ("libsacd.so", []), "tuning": ("libsacd_tuning.so", ["-DSACD_TUNING"]),
            "debug": ("libsacd_debug.so", ["-DSACD_DEBUG"])}
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

def _nccl_dir():
    """NCCL shipped with the PyTorch wheel (nvidia-nccl): headers + libnccl.so.2."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("nccl.h not found (nvidia-nccl wheel)")


NCCL = _nccl_dir()
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", f"-I{ROOT}/include", f"-I{NCCL}/include"]
LIBS = [f"-L{NCCL}/lib", "-l:libnccl.so.2", f"-Xlinker", f"-rpath={NCCL}/lib"]


def _paths(flavour):
    out = os.path.join(HERE, FLAVOURS[flavour][0])
    return out, out + ".stamp"


def _fingerprint(flavour="default") -> str:
    """sha256 over every csrc file, sacd.h, this file, the flags and the nvcc version: the .so
    is rebuilt whenever any of them differs from the stamp written next to it (a prebuilt
    .so that travels to the GPU box is reused only if it is exactly HEAD's build)."""
    import hashlib
    h = hashlib.sha256()
    deps = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)) + [os.path.join(ROOT, "include", "sacd.h"),
                                                                        os.path.abspath(__file__)]
    # names relative to the repo root and flags with the root / NCCL prefixes removed: the
    # checkout's location (a scratch path on the GPU box) must not make a matching .so stale
    rel = lambda x: x.replace(ROOT, "<root>").replace(NCCL, "<nccl>")
    for d in deps:
        h.update(rel(d).encode())
        with open(d, "rb") as fh:
            h.update(fh.read())
    h.update(repr(([rel(f) for f in FLAGS], [rel(f) for f in LIBS], SOURCES, FLAVOURS[flavour])).encode())
    try:
        h.update(subprocess.run([NVCC, "--version"], capture_output=True, text=True).stdout.encode())
    except OSError:
        h.update(b"no-nvcc")
    return h.hexdigest()


def _stale(flavour="default") -> bool:
    out, stamp = _paths(flavour)
    if not os.path.exists(out) or not os.path.exists(stamp):
        return True
    with open(stamp) as fh:
        return fh.read().strip() != _fingerprint(flavour)


def build(force: bool = False, verbose: bool = False, flavour: str = "default") -> str:
    OUT, STAMP = _paths(flavour)
    if not force and not _stale(flavour):
        return OUT
    # fingerprint of the sources as they are BEFORE nvcc reads them: an edit made while the
    # compile runs must leave the stamp stale
    fp = _fingerprint(flavour)
    cmd = [NVCC, *FLAGS, *FLAVOURS[flavour][1], "-o", OUT + ".tmp", *[os.path.join(CSRC, s) for s in SOURCES], *LIBS]
    log = os.path.join(HERE, f"build_{flavour}.log")
    with open(log, "w") as fh:
        r = subprocess.run(cmd, stdout=fh, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        sys.stderr.write(open(log).read()[-6000:])
        raise RuntimeError(f"nvcc failed ({r.returncode}); see {log}")
    os.replace(OUT + ".tmp", OUT)
    with open(STAMP, "w") as fh:
        fh.write(fp + "\n")
    if verbose:
        print(f"built {OUT}")
    return OUT


def build_gather_bench(verbose: bool = False) -> str:
    """tools/gather_bench (the measured gather peak of the MTTKRP's composite roofline)."""
    src = os.path.join(ROOT, "tools", "gather_bench.cu")
    out = os.path.join(ROOT, "tools", "gather_bench")
    if os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(src):
        return out
    subprocess.run([NVCC, "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-o", out,
                    src], check=True)
    if verbose:
        print(f"built {out}")
    return out


if __name__ == "__main__":
    fl = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--flavour=")), "default")
    build(force="--force" in sys.argv, verbose=True, flavour=fl)
