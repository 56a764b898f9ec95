"""ctypes binding of libapt.so (include/apt.h).  Argument marshalling only.

The library is built in-tree by ``__graft_entry__.build()``; importing this module without it raises
immediately — there is no fallback implementation of any kind.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# APT_LIB_VARIANT selects an in-tree experiment build (tools/ only); default is libapt.so
LIB_PATH = os.path.join(_HERE, os.environ.get("APT_LIB_VARIANT", "libapt.so"))

APT_OK, APT_ERR_INVALID_ARGUMENT, APT_ERR_UNSUPPORTED, APT_ERR_WORKSPACE, APT_ERR_CUDA = range(5)
APT_ENC_SIGNED, APT_ENC_BIPOLAR = 0, 1
APT_OUT_I32_SIGNED, APT_OUT_I32_BIPOLAR, APT_OUT_F16_SCALED = 0, 1, 2
APT_LAYOUT_ROW, APT_LAYOUT_COL = 0, 1
APT_KERNEL_AUTO, APT_KERNEL_TC, APT_KERNEL_GEMV, APT_KERNEL_SKINNY, APT_KERNEL_DEC, APT_KERNEL_PF = 0, 2, 3, 4, 5, 6
APT_MMA_I8, APT_MMA_MXF4 = 0, 1
ABI_VERSION = 8  # include/apt.h APT_ABI_VERSION this binding marshals for
APT_PACK_ROWS, APT_PACK_TILED = 0, 1

EXPORTED = ["apt_packed_plane_bytes", "apt_pack_bipolar", "apt_quantize_pack", "apt_select_config", "apt_gemm_workspace_bytes", "apt_gemm_zp_workspace_bytes",
            "apt_gemm", "apt_status_string", "apt_abi_version", "apt_table_load", "apt_table_clear", "apt_table_size",
            "apt_table_lookup", "apt_enumerate_configs", "apt_recombine_plane_products",
            "apt_gemm_grouped_workspace_bytes", "apt_gemm_grouped", "apt_pack_grouped"]


class AptPacked(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int32), ("k", ctypes.c_int32), ("k_words", ctypes.c_int32),
                ("bits", ctypes.c_int32), ("planes", ctypes.c_void_p), ("row_sum", ctypes.c_void_p),
                ("digits", ctypes.c_void_p), ("layout", ctypes.c_int32)]


class AptScales(ctypes.Structure):
    _fields_ = [("w_scale", ctypes.c_void_p), ("a_scale", ctypes.c_void_p), ("w_zero", ctypes.c_void_p),
                ("a_zero", ctypes.c_void_p), ("w_gscale", ctypes.c_void_p), ("a_gscale", ctypes.c_void_p),
                ("group_size", ctypes.c_int32)]


class AptGemmProblem(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int32), ("N", ctypes.c_int32), ("K", ctypes.c_int32), ("wbits", ctypes.c_int32),
                ("abits", ctypes.c_int32), ("W", AptPacked), ("A", AptPacked), ("scales", AptScales),
                ("kind", ctypes.c_int32), ("layout", ctypes.c_int32), ("out", ctypes.c_void_p), ("ldo", ctypes.c_int64),
                ("out_peers", ctypes.c_void_p * 7), ("n_peers", ctypes.c_int32)]


APT_GROUP_MAX = 64
APT_MAX_PEERS = 7
APT_PACK_GROUP_MAX_ROWS = 64


class AptPackProblem(ctypes.Structure):
    _fields_ = [("src", ctypes.c_void_p), ("quantize", ctypes.c_int32), ("rows", ctypes.c_int32), ("k", ctypes.c_int32),
                ("bits", ctypes.c_int32), ("ld", ctypes.c_int64), ("out", ctypes.POINTER(AptPacked)),
                ("scale", ctypes.c_void_p), ("range_error", ctypes.c_void_p)]


class AptConfig(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("kernel", "w_digit", "a_digit", "bm", "bn", "bk", "stages", "split_k", "cta_pair",
                 "cluster_n", "mma_kind")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


class AptError(RuntimeError):
    def __init__(self, fn, status):
        self.status = status
        super().__init__(f"{fn} failed: {status_string(status)} ({status})")


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no fallback path exists)")
        L = ctypes.CDLL(LIB_PATH)
        L.apt_packed_plane_bytes.restype = ctypes.c_size_t
        L.apt_packed_plane_bytes.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]
        L.apt_pack_bipolar.restype = ctypes.c_int
        L.apt_pack_bipolar.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                       ctypes.c_int32, ctypes.c_int, ctypes.POINTER(AptPacked), ctypes.c_void_p,
                                       ctypes.c_void_p]
        L.apt_quantize_pack.restype = ctypes.c_int
        L.apt_quantize_pack.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                        ctypes.c_int32, ctypes.POINTER(AptPacked), ctypes.c_void_p, ctypes.c_void_p]
        L.apt_select_config.restype = ctypes.c_int
        L.apt_select_config.argtypes = [ctypes.c_int32] * 5 + [ctypes.POINTER(AptConfig)]
        L.apt_gemm_workspace_bytes.restype = ctypes.c_size_t
        L.apt_gemm_workspace_bytes.argtypes = [ctypes.POINTER(AptConfig), ctypes.c_int32, ctypes.c_int32,
                                               ctypes.c_int32]
        L.apt_gemm_zp_workspace_bytes.restype = ctypes.c_size_t
        L.apt_gemm_zp_workspace_bytes.argtypes = [ctypes.POINTER(AptConfig), ctypes.c_int32, ctypes.c_int32,
                                                  ctypes.c_int32]
        L.apt_gemm.restype = ctypes.c_int
        L.apt_gemm.argtypes = [ctypes.c_int32] * 5 + [ctypes.POINTER(AptPacked), ctypes.POINTER(AptPacked),
                                                      ctypes.POINTER(AptScales), ctypes.c_int, ctypes.c_int,
                                                      ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(AptConfig),
                                                      ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
        L.apt_status_string.restype = ctypes.c_char_p
        L.apt_status_string.argtypes = [ctypes.c_int]
        L.apt_abi_version.restype = ctypes.c_int32
        L.apt_abi_version.argtypes = []
        L.apt_table_load.restype = ctypes.c_int
        L.apt_table_load.argtypes = [ctypes.c_char_p]
        L.apt_table_clear.restype = None
        L.apt_table_clear.argtypes = []
        L.apt_table_size.restype = ctypes.c_int32
        L.apt_table_size.argtypes = []
        L.apt_table_lookup.restype = ctypes.c_int
        L.apt_table_lookup.argtypes = [ctypes.c_int32] * 5 + [ctypes.POINTER(AptConfig), ctypes.POINTER(ctypes.c_double)]
        L.apt_recombine_plane_products.restype = ctypes.c_int
        L.apt_recombine_plane_products.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                                   ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        L.apt_enumerate_configs.restype = ctypes.c_int32
        L.apt_enumerate_configs.argtypes = [ctypes.c_int32] * 5 + [ctypes.POINTER(AptConfig), ctypes.c_int32]
        L.apt_gemm_grouped_workspace_bytes.restype = ctypes.c_size_t
        L.apt_gemm_grouped_workspace_bytes.argtypes = [ctypes.c_int32]
        L.apt_gemm_grouped.restype = ctypes.c_int
        L.apt_gemm_grouped.argtypes = [ctypes.c_int32, ctypes.POINTER(AptGemmProblem), ctypes.c_void_p, ctypes.c_size_t,
                                       ctypes.c_void_p]
        L.apt_pack_grouped.restype = ctypes.c_int
        L.apt_pack_grouped.argtypes = [ctypes.c_int32, ctypes.POINTER(AptPackProblem), ctypes.c_void_p]
        v = int(L.apt_abi_version())
        if v != ABI_VERSION:
            raise ImportError(f"{LIB_PATH} has ABI version {v}, this binding needs {ABI_VERSION}: rebuild it")
        _lib = L
        # the shipped autotuned configuration table (NEXT-3), loaded with the library: APT_TABLE = a path
        # or "none"; default tables/b200.apt next to this file
        path = os.environ.get("APT_TABLE", os.path.join(_HERE, "tables", "b200.apt"))
        if path.lower() != "none" and os.path.exists(path):
            check("apt_table_load", L.apt_table_load(path.encode()))
    return _lib


def status_string(status: int) -> str:
    return lib().apt_status_string(status).decode()


def check(fn: str, status: int):
    if status != APT_OK:
        raise AptError(fn, status)
