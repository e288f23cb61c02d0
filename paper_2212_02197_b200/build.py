"""Build the in-tree CUDA library libnmpcmc_gpu.so for sm_100a with nvcc.

Flags that matter for results: --fmad=false (no implicit FMA contraction,
SURVEY.md Appendix A.1) and no fast-math; the host code gets
-ffp-contract=off for the same reason. -lineinfo keeps ncu source mapping.
Each translation unit (one per kernel family, launchers.h) compiles to its
own object in parallel; one nvcc -shared links them.
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libnmpcmc_gpu.so")
# largest first: the NMPC kernel units dominate the build
SOURCES = ["k_gen.cu", "k_nmpc.cu", "k_misc.cu", "nmpcmc_multi.cu", "nmpcmc_gpu.cu", "controllers_api.cu", "host_api.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "--fmad=false", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-Xptxas", "-v",
]


def _stale(out) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "nmpcmc_gpu.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile the library. Experiments only: NMPCMC_NVCC_EXTRA adds flags
    (e.g. -DNMPCMC_IPM_SMEM=1) and NMPCMC_BUILD_OUT redirects the output."""
    out = os.environ.get("NMPCMC_BUILD_OUT") or LIB
    extra = os.environ.get("NMPCMC_NVCC_EXTRA", "").split()
    if not force and not extra and out == LIB and not _stale(out):
        return LIB
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    # experiment builds get their own object directory, so several can run at once
    objdir = os.path.join(os.path.dirname(os.path.abspath(out)),
                          "obj" + ("_" + os.path.splitext(os.path.basename(out))[0] if (extra or out != LIB) else ""))
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        cmd = [NVCC, *NVCC_FLAGS, *extra, *inc, "-c", os.path.join(CSRC, src), "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        return obj, " ".join(cmd) + "\n" + res.stdout + res.stderr, res.returncode

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as pool:
        results = list(pool.map(compile_one, SOURCES))
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *[r[0] for r in results], "-ldl",
            "-o", out]
    log_text = "".join(r[1] for r in results)
    ok = all(r[2] == 0 for r in results)
    if ok:
        res = subprocess.run(link, capture_output=True, text=True)
        log_text += " ".join(link) + "\n" + res.stdout + res.stderr
        ok = res.returncode == 0
    log = os.path.join(LIBDIR, "build.log") if out == LIB else out + ".build.log"
    os.makedirs(os.path.dirname(log), exist_ok=True)
    with open(log, "w") as fh:
        fh.write(log_text)
    if not ok:
        sys.stderr.write("\n".join(line for line in log_text.splitlines() if "error" in line.lower()) + "\n")
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stdout.write(log_text if "-v" in sys.argv else "")
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
