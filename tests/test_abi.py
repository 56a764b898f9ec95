"""C-ABI checks that need no GPU: the library loads, exports every symbol include/apt.h
declares, the host-only selector is legal/deterministic, and argument errors are returned
synchronously before any launch."""
import ctypes
import os
import re

import pytest
import torch

from paper_2508_19087_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "apt.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"APT_API\s+[\w\s\*]+?\b(apt_\w+)\s*\(", src)))


def test_header_symbols_exported():
    syms = _declared_symbols()
    assert set(syms) == set(L.EXPORTED)
    lib = L.lib()
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.apt_abi_version() == L.ABI_VERSION == 8


def test_status_strings():
    assert L.status_string(0) == "APT_OK"
    assert L.status_string(2) == "APT_ERR_UNSUPPORTED"


def test_plane_bytes():
    lib = L.lib()
    R, T = L.APT_PACK_ROWS, L.APT_PACK_TILED
    assert lib.apt_packed_plane_bytes(4096, 4096, 2, R) == 2 * 4096 * 128 * 4
    assert lib.apt_packed_plane_bytes(3, 1, 8, R) == 8 * 3 * 8 * 4
    assert lib.apt_packed_plane_bytes(3, 257, 3, R) == 3 * 3 * 16 * 4
    assert lib.apt_packed_plane_bytes(3, 257, 3, T) == 3 * 128 * 16 * 4
    assert lib.apt_packed_plane_bytes(11008, 4096, 4, T) == 4 * 11008 * 128 * 4
    assert lib.apt_packed_plane_bytes(0, 5, 2, R) == 0
    assert lib.apt_packed_plane_bytes(5, 5, 9, R) == 0
    assert lib.apt_packed_plane_bytes(5, 5, 2, 7) == 0


def _select(M, N, K, wb, ab):
    c = L.AptConfig()
    rc = L.lib().apt_select_config(M, N, K, wb, ab, ctypes.byref(c))
    return rc, c


@pytest.fixture(params=["analytic", "table"])
def table_mode(request):
    """Selector checks with the table cleared (the analytic rules) and with the shipped autotuned table."""
    import paper_2508_19087_b200 as P
    P.clear_table()
    if request.param == "table":
        P.load_default_table()
    yield request.param
    P.clear_table()
    P.load_default_table()


@pytest.mark.parametrize("M", [1, 2, 3, 8, 16, 64, 2048])
@pytest.mark.parametrize("N,K", [(4096, 4096), (11008, 4096), (4096, 11008), (256, 256), (7, 1)])
@pytest.mark.parametrize("wb,ab", [(1, 2), (2, 2), (3, 4), (4, 4), (8, 8)])
def test_selector_legal_and_deterministic(M, N, K, wb, ab, table_mode):
    rc, c = _select(M, N, K, wb, ab)
    assert rc == L.APT_OK
    rc2, c2 = _select(M, N, K, wb, ab)
    assert c.as_dict() == c2.as_dict()
    kw = -(-K // 256) * 8
    assert c.w_digit == wb and c.a_digit == ab
    assert c.mma_kind == L.APT_MMA_I8 or (c.mma_kind == L.APT_MMA_MXF4 and wb <= 3 and ab <= 3
                                          and c.kernel in (L.APT_KERNEL_TC, L.APT_KERNEL_PF) and table_mode == "table")
    if c.kernel == L.APT_KERNEL_GEMV:
        assert M <= 2 and c.bm == 32 and c.bn == M and c.split_k in (8, 16) and c.stages == 1
        assert c.cluster_n == 1 and c.cta_pair == 0
    elif c.kernel == L.APT_KERNEL_SKINNY:
        assert M <= 16 and c.bm == 16 and c.bn in (8, 16) and c.bk == 256
        assert c.split_k in (4, 8, 16) and c.stages == 1 and c.cluster_n == 1 and c.cta_pair == 0
        if table_mode == "analytic":
            assert 2 < M <= 8 and K <= 4096 and c.bn == 8 and c.split_k in (4, 8)
    elif c.kernel == L.APT_KERNEL_PF:
        assert c.bm == 128 and c.bn in (128, 192, 256) and c.split_k == 1 and c.cluster_n == 1 and M > 2
        if table_mode == "analytic":  # token-rich shapes: the persistent 256-token tile
            assert M > 64 and c.bn == 256 and c.stages == 3 and c.mma_kind == L.APT_MMA_I8
    elif c.kernel == L.APT_KERNEL_DEC:
        assert table_mode == "table" and M <= 16 and c.bm == 32 and c.bn == (8 if M <= 8 else 16) and c.bk == 256
        assert c.stages in (4, 8) and 1 <= c.split_k <= 32 and c.cluster_n == 1 and c.cta_pair == 0
    else:
        assert c.kernel == L.APT_KERNEL_TC and M > 2
        assert c.bm == 128 and c.bn in (16, 64, 128, 256) and c.cluster_n in (1, 2, 4)
        assert 1 <= c.split_k <= 8 and c.cluster_n * c.split_k <= 8
        assert c.split_k == 1 or (c.bn <= 64 and c.cluster_n == 1)
        if table_mode == "analytic":
            assert c.bn >= min(M, 128 if M > 64 else 64)


def test_selector_errors():
    assert _select(0, 1, 1, 2, 2)[0] == L.APT_ERR_INVALID_ARGUMENT
    assert _select(1, 1, 1, 0, 2)[0] == L.APT_ERR_INVALID_ARGUMENT
    assert _select(1, 1, 1, 2, 9)[0] == L.APT_ERR_INVALID_ARGUMENT
    assert _select(1, 1, 33025, 8, 8)[0] == L.APT_ERR_UNSUPPORTED
    assert _select(1, 1, 33024, 8, 8)[0] == L.APT_OK


def _fake_packed(rows, k, bits, addr=0x10000):
    return L.AptPacked(rows, k, -(-k // 256) * 8, bits, addr, addr + 0x1000000, None, L.APT_PACK_ROWS)


def _gemm(M, N, K, wb, ab, W, A, kind=0, layout=0, out=0x30000, ldo=None, scales=None, cfg=None):
    lib = L.lib()
    ldo = ldo if ldo is not None else (N if layout == 0 else M)
    return lib.apt_gemm(M, N, K, wb, ab, ctypes.byref(W) if W else None, ctypes.byref(A) if A else None,
                        ctypes.byref(scales) if scales else None, kind, layout, out, ldo,
                        ctypes.byref(cfg) if cfg else None, None, 0, None)


def test_gemm_argument_errors_before_launch():
    W, A = _fake_packed(64, 256, 2), _fake_packed(16, 256, 2)
    E = L.APT_ERR_INVALID_ARGUMENT
    assert _gemm(16, 64, 256, 2, 2, None, A) == E
    assert _gemm(16, 64, 256, 2, 2, W, None) == E
    assert _gemm(16, 64, 256, 3, 2, W, A) == E                      # bits mismatch
    assert _gemm(16, 65, 256, 2, 2, W, A) == E                      # N mismatch
    assert _gemm(15, 64, 256, 2, 2, W, A) == E                      # M mismatch
    assert _gemm(16, 64, 257, 2, 2, W, A) == E                      # K mismatch
    assert _gemm(16, 64, 256, 2, 2, W, A, out=0) == E               # null out
    assert _gemm(16, 64, 256, 2, 2, W, A, ldo=63) == E              # ldo < N
    assert _gemm(16, 64, 256, 2, 2, W, A, layout=1, ldo=15) == E    # ldo < M
    assert _gemm(16, 64, 256, 2, 2, W, A, kind=2) == E              # fp16 needs w_scale
    assert _gemm(16, 64, 256, 2, 2, W, A, kind=7) == E
    Wm = _fake_packed(64, 256, 2, addr=0x10004)                     # misaligned planes
    assert _gemm(16, 64, 256, 2, 2, Wm, A) == E
    bad = L.AptConfig(1, 2, 2, 32, 16, 256, 2, 4, 0, 1, 0)  # kernel 1 (removed in ABI 3)
    assert _gemm(16, 64, 256, 2, 2, W, A, cfg=bad) == L.APT_ERR_UNSUPPORTED
    bad = L.AptConfig(L.APT_KERNEL_SKINNY, 2, 2, 16, 24, 256, 1, 8, 0, 1, 0)  # bn 24 illegal
    assert _gemm(16, 64, 256, 2, 2, W, A, cfg=bad) == L.APT_ERR_UNSUPPORTED
    bad = L.AptConfig(L.APT_KERNEL_SKINNY, 2, 2, 16, 16, 256, 1, 8, 0, 1, 5)  # unknown mma_kind
    assert _gemm(16, 64, 256, 2, 2, W, A, cfg=bad) == L.APT_ERR_UNSUPPORTED
    Wb, Ab = _fake_packed(64, 40000, 8), _fake_packed(16, 40000, 8)
    assert _gemm(16, 64, 40000, 8, 8, Wb, Ab) == L.APT_ERR_UNSUPPORTED


def test_pack_argument_errors():
    lib = L.lib()
    out = L.AptPacked(0, 0, 0, 0, 0x10000, 0x20000, None, L.APT_PACK_ROWS)
    E = L.APT_ERR_INVALID_ARGUMENT
    assert lib.apt_pack_bipolar(None, 4, 4, 4, 2, 0, ctypes.byref(out), None, None) == E
    assert lib.apt_pack_bipolar(0x1000, 4, 4, 3, 2, 0, ctypes.byref(out), None, None) == E   # ld < k
    assert lib.apt_pack_bipolar(0x1000, 4, 4, 4, 9, 0, ctypes.byref(out), None, None) == E
    assert lib.apt_pack_bipolar(0x1000, 4, 4, 4, 8, 1, ctypes.byref(out), None, None) == E   # bipolar n=8
    assert lib.apt_pack_bipolar(0x1000, 0, 4, 4, 2, 0, ctypes.byref(out), None, None) == E
    out.layout = 5
    assert lib.apt_pack_bipolar(0x1000, 4, 4, 4, 2, 0, ctypes.byref(out), None, None) == E


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device path")
def test_no_device_means_cuda_error_not_fallback():
    W, A = _fake_packed(64, 256, 2), _fake_packed(16, 256, 2)
    assert _gemm(16, 64, 256, 2, 2, W, A) == L.APT_ERR_WORKSPACE   # tcgen05 path needs a digit view
    A.digits = 0x50000
    assert _gemm(16, 64, 256, 2, 2, W, A) == L.APT_ERR_CUDA
    out = L.AptPacked(0, 0, 0, 0, 0x10000, 0x20000, None, L.APT_PACK_ROWS)
    assert L.lib().apt_pack_bipolar(0x1000, 4, 4, 4, 2, 0, ctypes.byref(out), None, None) == L.APT_ERR_CUDA


def test_python_pack_validates_out():
    """A caller-supplied `out` must match the codes' shape/bits exactly (no OOB writes)."""
    import paper_2508_19087_b200 as P
    from paper_2508_19087_b200 import api
    out = api.Packed(torch.zeros((2, 4, 8), dtype=torch.int32), torch.zeros(4, dtype=torch.int32), 4, 256, 2)
    api._check_out(out, 4, 256, 2, False, False)
    for args in ((4, 256, 3), (5, 256, 2), (4, 300, 2)):
        with pytest.raises(ValueError):
            api._check_out(out, *args, False, False)
    with pytest.raises(ValueError):
        api._check_out(out, 4, 256, 2, True, False)      # tiled buffers need 128-row padding
    with pytest.raises(ValueError):
        api._check_out(out, 4, 256, 2, False, True)      # digit view requested but absent


def test_python_api_refuses_cpu_tensors():
    import paper_2508_19087_b200 as P
    with pytest.raises(ValueError):
        P.pack(torch.zeros((2, 2), dtype=torch.int8), 2)


def test_grouped_argument_errors_without_gpu():
    """apt_gemm_grouped rejects a bad group size / null array before touching the device."""
    lib = L.lib()
    assert lib.apt_gemm_grouped(0, None, None, 0, None) == L.APT_ERR_INVALID_ARGUMENT
    assert lib.apt_gemm_grouped(L.APT_GROUP_MAX + 1, None, None, 0, None) == L.APT_ERR_INVALID_ARGUMENT
    arr = (L.AptGemmProblem * 1)()
    arr[0].M = 17  # more tokens than the decode kernel's 16
    assert lib.apt_gemm_grouped(1, arr, None, 0, None) == L.APT_ERR_INVALID_ARGUMENT
    assert lib.apt_gemm_grouped_workspace_bytes(0) == 0
    assert lib.apt_gemm_grouped_workspace_bytes(1) >= 16384 + 148 * 4 * 2 * 4 * 512 * 4
