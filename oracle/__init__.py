"""CPU oracle for the APT bit-plane GEMM — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import anything under oracle/.  The product
package never does.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build_c_oracle(force: bool = False) -> str:
    """Compile oracle_gemm.c -> liboracle.so (gcc -O3 -fopenmp)."""
    import subprocess
    src = os.path.join(_HERE, "oracle_gemm.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-o", LIB_PATH, src])
    return LIB_PATH


def c_lib():
    global _lib
    if _lib is None:
        build_c_oracle()
        lib = ctypes.CDLL(LIB_PATH)
        lib.apt_oracle_threads.restype = ctypes.c_int
        lib.apt_oracle_gemm_i64.restype = None
        lib.apt_oracle_gemm_i64.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                            ctypes.c_int32]
        _lib = lib
    return _lib


def c_gemm_i64(a: np.ndarray, w: np.ndarray) -> np.ndarray:
    """C oracle: Y = A . W^T over int8 signed codes, int64 result."""
    a = np.ascontiguousarray(a, dtype=np.int8)
    w = np.ascontiguousarray(w, dtype=np.int8)
    m, k = a.shape
    n, k2 = w.shape
    assert k == k2
    y = np.zeros((m, n), dtype=np.int64)
    c_lib().apt_oracle_gemm_i64(a.ctypes.data, k, w.ctypes.data, k, y.ctypes.data, n, m, n, k)
    return y


def c_threads() -> int:
    return int(c_lib().apt_oracle_threads())
