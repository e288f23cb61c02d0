"""Build the in-tree CUDA library libnmpcmc_gpu.so for sm_100a with nvcc.

Flags that matter for results: --fmad=false (no implicit FMA contraction,
SURVEY.md Appendix A.1) and no fast-math; the host code gets
-ffp-contract=off for the same reason. -lineinfo keeps ncu source mapping.
"""
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libnmpcmc_gpu.so")
SOURCES = ["nmpcmc_gpu.cu", "nmpcmc_multi.cu", "host_api.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "--fmad=false", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-Xptxas", "-v",
    "-shared",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "nmpcmc_gpu.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile the library. Experiments only: NMPCMC_NVCC_EXTRA adds flags
    (e.g. -DNMPCMC_IPM_SMEM=1) and NMPCMC_BUILD_OUT redirects the output."""
    out = os.environ.get("NMPCMC_BUILD_OUT") or LIB
    extra = os.environ.get("NMPCMC_NVCC_EXTRA", "").split()
    if not force and not extra and out == LIB and not _stale():
        return LIB
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    cmd = [NVCC, *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           *[os.path.join(CSRC, s) for s in SOURCES], "-ldl", "-o", out]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(LIBDIR, "build.log") if out == LIB else out + ".build.log"
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stdout.write(res.stderr)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
