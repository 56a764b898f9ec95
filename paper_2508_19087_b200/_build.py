"""Compile the CUDA sources into the in-tree shared library libapt.so (sm_100a only)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libapt.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
SOURCES = ["apt.cu", "pack.cu", "gemm_tc.cu", "gemv.cu", "gemm_skinny.cu", "gemm_dec.cu", "gemm_pf.cu", "gemm_grp.cu", "epilogue_zp.cu"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-shared", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I" + os.path.join(HERE, "..", "include")]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "apt.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """One object per source, compiled in parallel under build/ (recompiled when the source, any header
    or the flags changed), then linked into the shared library."""
    if not force and out == LIB and not _stale():
        return LIB
    import hashlib
    from concurrent.futures import ThreadPoolExecutor
    flags = FLAGS + (["-Xptxas", "-v"] if verbose else []) + ["-D" + d for d in defines]
    tag = hashlib.sha1(" ".join(flags).encode()).hexdigest()[:10]
    odir = os.path.join(HERE, "..", "build", "obj-" + tag)
    os.makedirs(odir, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if not f.endswith(".cu")] + \
        [os.path.join(HERE, "..", "include", "apt.h")]
    hdr_t = max(os.path.getmtime(h) for h in headers)

    def compile_one(src):
        cu = os.path.join(CSRC, src)
        obj = os.path.join(odir, src[:-3] + ".o")
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(cu), hdr_t):
            cmd = [NVCC] + [f for f in flags if f != "-shared"] + ["-c", cu, "-o", obj + ".tmp"]
            subprocess.check_call(cmd)
            os.replace(obj + ".tmp", obj)
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared"] + objs + ["-o", out + ".tmp"])
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    import sys
    print(build(force=True, verbose="-v" in sys.argv))
