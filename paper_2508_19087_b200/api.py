"""Thin torch-facing binding over the C ABI (argument marshalling only).

Every step of the hot path runs in libapt.so's CUDA kernels; torch provides device memory,
streams and process groups.  Names follow include/apt.h and the paper's notation:
``W`` = weights [N, K] (``wbits`` = p_w), ``A`` = activations [M, K] (``abits`` = p_a).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib as L

KPAD_QUANTUM = 256

_OUT_KINDS = {"i32": L.APT_OUT_I32_SIGNED, "bipolar": L.APT_OUT_I32_BIPOLAR, "f16": L.APT_OUT_F16_SCALED}
_LAYOUTS = {"row": L.APT_LAYOUT_ROW, "col": L.APT_LAYOUT_COL}
_ENCODINGS = {"signed": L.APT_ENC_SIGNED, "bipolar": L.APT_ENC_BIPOLAR}


def kpad(k: int) -> int:
    return -(-k // KPAD_QUANTUM) * KPAD_QUANTUM


def _stream_handle(stream) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)


def _require_cuda(t: torch.Tensor, name: str):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (the APT path has no CPU implementation)")


@dataclass
class Packed:
    """The packed "unified matrix": planes [bits][rows][k_words] uint32 (stored as int32
    tensor), row_sum [rows] int32, and optionally the kernel-order u8 digit view [rows][Kpad]
    (written by the pack kernel in the same pass; used for activations)."""
    planes: torch.Tensor
    row_sum: torch.Tensor
    rows: int
    k: int
    bits: int
    digits: torch.Tensor | None = None
    tiled: bool = False  # planes in the tile-major layout (APT_PACK_TILED) the GEMM streams fastest

    @property
    def k_words(self) -> int:
        return kpad(self.k) // 32

    def struct(self) -> L.AptPacked:
        return L.AptPacked(self.rows, self.k, self.k_words, self.bits, self.planes.data_ptr(),
                           self.row_sum.data_ptr(), self.digits.data_ptr() if self.digits is not None else None,
                           L.APT_PACK_TILED if self.tiled else L.APT_PACK_ROWS)

    def narrow_rows(self, start: int, length: int) -> "Packed":
        """Rows [start, start+length) as a new packed matrix (copies the plane slices)."""
        if self.tiled:
            raise ValueError("narrow_rows needs the row-major plane layout")
        planes = self.planes[:, start:start + length].contiguous()
        digits = self.digits[start:start + length].contiguous() if self.digits is not None else None
        return Packed(planes, self.row_sum[start:start + length].contiguous(), length, self.k, self.bits, digits)


def alloc_packed(rows: int, k: int, bits: int, device, digits: bool = False, tiled: bool = False) -> Packed:
    """Buffers for a packed operand; ``digits=True`` also allocates the u8 digit view (activations),
    ``tiled=True`` stores the planes tile-major (weights)."""
    kw = kpad(k) // 32
    prow = -(-rows // 128) * 128 if tiled else rows
    planes = torch.empty((bits, prow, kw), dtype=torch.int32, device=device)
    row_sum = torch.empty((rows,), dtype=torch.int32, device=device)
    dig = torch.empty((rows, kw * 32), dtype=torch.uint8, device=device) if digits else None
    return Packed(planes, row_sum, rows, k, bits, dig, tiled)


def _check_out(out: "Packed", rows: int, k: int, bits: int, tiled: bool, digits: bool):
    """A caller-supplied output must describe exactly the buffers apt_pack_bipolar will write."""
    want = alloc_shapes(rows, k, bits, digits, tiled)
    if (out.rows, out.k, out.bits, bool(out.tiled)) != (rows, k, bits, bool(tiled)):
        raise ValueError(f"out describes (rows={out.rows}, k={out.k}, bits={out.bits}, tiled={out.tiled}), "
                         f"the codes need (rows={rows}, k={k}, bits={bits}, tiled={tiled})")
    for name, t, shape, dt in (("planes", out.planes, want[0], torch.int32), ("row_sum", out.row_sum, want[1], torch.int32),
                               ("digits", out.digits, want[2], torch.uint8)):
        if shape is None:
            continue
        if t is None or tuple(t.shape) != shape or t.dtype != dt or not t.is_contiguous():
            raise ValueError(f"out.{name} must be a contiguous {dt} tensor of shape {shape}")
    if out.planes.device != out.row_sum.device:
        raise ValueError("out buffers live on different devices")


def alloc_shapes(rows: int, k: int, bits: int, digits: bool, tiled: bool):
    kw = kpad(k) // 32
    prow = -(-rows // 128) * 128 if tiled else rows
    return (bits, prow, kw), (rows,), ((rows, kw * 32) if digits else None)


def pack(codes: torch.Tensor, bits: int, encoding: str = "signed", out: Packed | None = None,
         range_error: torch.Tensor | None = None, stream=None, digits: bool = False, tiled: bool = False) -> Packed:
    """apt_pack_bipolar: int8 codes [rows, k] (row stride ``codes.stride(0)``) -> Packed.
    ``digits=True`` (activations) also emits the kernel-order u8 digit view in the same pass;
    ``tiled=True`` (weights) writes the planes tile-major."""
    _require_cuda(codes, "codes")
    if codes.dtype != torch.int8 or codes.dim() != 2 or codes.stride(1) != 1:
        raise ValueError("codes must be a 2-D int8 tensor with unit stride along K")
    rows, k = codes.shape
    if out is None:
        out = alloc_packed(rows, k, bits, codes.device, digits=digits, tiled=tiled)
    else:
        _check_out(out, rows, k, bits, out.tiled, out.digits is not None)
        if out.planes.device != codes.device:
            raise ValueError("out lives on another device than codes")
    st = out.struct()
    rc = L.lib().apt_pack_bipolar(codes.data_ptr(), rows, k, codes.stride(0), bits, _ENCODINGS[encoding],
                                  ctypes.byref(st), range_error.data_ptr() if range_error is not None else None,
                                  _stream_handle(stream))
    L.check("apt_pack_bipolar", rc)
    return out


def quantize_pack(x: torch.Tensor, bits: int, out: Packed | None = None, scale: torch.Tensor | None = None,
                  stream=None, digits: bool = True, tiled: bool = False) -> tuple[Packed, torch.Tensor]:
    """apt_quantize_pack: fp16 activations [rows, k] -> (Packed signed codes, fp32 per-row scale).
    Symmetric per-token quantization (z = 0) fused with the bit-plane pack; pass the scale
    as ``a_scale`` of :func:`gemm`."""
    _require_cuda(x, "x")
    if x.dtype != torch.float16 or x.dim() != 2 or x.stride(1) != 1:
        raise ValueError("x must be a 2-D float16 tensor with unit stride along K")
    rows, k = x.shape
    if out is None:
        out = alloc_packed(rows, k, bits, x.device, digits=digits, tiled=tiled)
    else:
        _check_out(out, rows, k, bits, out.tiled, out.digits is not None)
        if out.planes.device != x.device:
            raise ValueError("out lives on another device than x")
    if scale is None:
        scale = torch.empty(rows, dtype=torch.float32, device=x.device)
    elif scale.dtype != torch.float32 or not scale.is_contiguous() or scale.numel() < rows or scale.device != x.device:
        raise ValueError("scale must be a contiguous fp32 tensor of >= rows elements on x's device")
    st = out.struct()
    rc = L.lib().apt_quantize_pack(x.data_ptr(), rows, k, x.stride(0), bits, ctypes.byref(st), scale.data_ptr(),
                                   _stream_handle(stream))
    L.check("apt_quantize_pack", rc)
    return out, scale


_WS = {}


def default_workspace(device, nbytes: int) -> torch.Tensor:
    """The per-device default apt_gemm workspace: zero-filled when (re)allocated, because the split-K
    tickets inside it must start at zero (apt_gemm leaves them zero).  Calls on one device share it,
    so concurrent streams must pass their own ``workspace``."""
    dev = torch.device(device)
    key = (dev.type, dev.index if dev.index is not None else torch.cuda.current_device())
    ws = _WS.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.zeros((max(nbytes, 1 << 20),), dtype=torch.uint8, device=dev)
        _WS[key] = ws
    return ws


# ----------------------------------------------------------------------------- autotuned table (NEXT-3)

TABLE_DIR = __import__("os").path.join(__import__("os").path.dirname(__import__("os").path.abspath(__file__)), "tables")
DEFAULT_TABLE = __import__("os").path.join(TABLE_DIR, "b200.apt")


def load_table(path: str) -> int:
    """apt_table_load: merge an autotuned configuration table (§5.2) into the library's table;
    apt_select_config consults it before its analytic rules.  Returns the table size."""
    L.check("apt_table_load", L.lib().apt_table_load(str(path).encode()))
    return int(L.lib().apt_table_size())


def clear_table() -> None:
    L.lib().apt_table_clear()


def table_size() -> int:
    return int(L.lib().apt_table_size())


def table_lookup(M: int, N: int, K: int, wbits: int, abits: int):
    """(config dict, distance) of the nearest table row (distance 0 = exact key), or None if empty."""
    c = L.AptConfig()
    d = ctypes.c_double()
    rc = L.lib().apt_table_lookup(M, N, K, wbits, abits, ctypes.byref(c), ctypes.byref(d))
    if rc == L.APT_ERR_UNSUPPORTED:
        return None
    L.check("apt_table_lookup", rc)
    return c.as_dict(), float(d.value)


def enumerate_configs(M: int, N: int, K: int, wbits: int, abits: int) -> list:
    """apt_enumerate_configs: every legal configuration for the problem (the Best Kernel Search space)."""
    n = int(L.lib().apt_enumerate_configs(M, N, K, wbits, abits, None, 0))
    arr = (L.AptConfig * max(n, 1))()
    L.lib().apt_enumerate_configs(M, N, K, wbits, abits, arr, n)
    return [arr[i].as_dict() for i in range(n)]


def load_default_table() -> int:
    """Load the shipped B200 table (tables/b200.apt, written by tools/tune.py) unless APT_TABLE says
    otherwise: a path, or "none"."""
    import os
    path = os.environ.get("APT_TABLE", DEFAULT_TABLE)
    if path.lower() == "none" or not os.path.exists(path):
        return table_size()
    return load_table(path)


def select_config(M: int, N: int, K: int, wbits: int, abits: int) -> dict:
    """apt_select_config (p = wbits, q = abits)."""
    c = L.AptConfig()
    L.check("apt_select_config", L.lib().apt_select_config(M, N, K, wbits, abits, ctypes.byref(c)))
    return c.as_dict()


def _config_struct(cfg: dict | None):
    if cfg is None:
        return None
    c = L.AptConfig()
    for n, _ in c._fields_:
        setattr(c, n, int(cfg[n]))
    return c


def workspace_bytes(cfg: dict, M: int, N: int, K: int) -> int:
    c = _config_struct(cfg)
    return int(L.lib().apt_gemm_workspace_bytes(ctypes.byref(c), M, N, K))


def gemm(W: Packed, A: Packed, out_kind: str = "i32", layout: str = "row", w_scale: torch.Tensor | None = None,
         a_scale: torch.Tensor | None = None, out: torch.Tensor | None = None, config: dict | None = None,
         workspace: torch.Tensor | None = None, stream=None, w_zero: torch.Tensor | None = None,
         a_zero: torch.Tensor | None = None, w_gscale: torch.Tensor | None = None,
         a_gscale: torch.Tensor | None = None) -> torch.Tensor:
    """apt_gemm: Y = A . W^T (exact int32), Y' (bipolar), or fp16-scaled, in row ([M,N]) or col
    ([N,M]) layout.  ``w_gscale`` ([Kpad/128, N] fp32) / ``a_gscale`` ([Kpad/128, M]) select group-wise
    (128) scales for the fp16 output (include/apt.h apt_scales)."""
    M, N, K = A.rows, W.rows, W.k
    if A.k != K:
        raise ValueError("A and W have different K")
    _require_cuda(W.planes, "W.planes")
    _require_cuda(A.planes, "A.planes")
    kind = _OUT_KINDS[out_kind]
    lay = _LAYOUTS[layout]
    shape = (M, N) if lay == L.APT_LAYOUT_ROW else (N, M)
    dtype = torch.float16 if kind == L.APT_OUT_F16_SCALED else torch.int32
    if out is None:
        out = torch.empty(shape, dtype=dtype, device=W.planes.device)
    if out.dtype != dtype or out.dim() != 2 or out.stride(1) != 1 or tuple(out.shape) != shape:
        raise ValueError(f"out must be a {dtype} tensor of shape {shape} with unit inner stride")
    sc = _scales_struct(w_scale, a_scale, w_zero, a_zero, w_gscale, a_gscale, K, N, M)
    c = _config_struct(config)
    zp = kind == L.APT_OUT_F16_SCALED and (w_zero is not None or a_zero is not None)
    gs = w_gscale is not None
    cc = c
    if cc is None:
        cc = L.AptConfig()
        L.check("apt_select_config", L.lib().apt_select_config(M, N, K, W.bits, A.bits, ctypes.byref(cc)))
    fn = L.lib().apt_gemm_zp_workspace_bytes if zp else L.lib().apt_gemm_workspace_bytes
    ws_need = int(fn(ctypes.byref(cc), M, N, K))
    if A.digits is not None and not zp and cc.kernel != L.APT_KERNEL_DEC and cc.mma_kind != L.APT_MMA_MXF4:
        ws_need = 0  # the digit view replaces the token expansion area (kind::mxf4 expands e2m1 tokens)
    if gs or (zp and M <= 16 and W.tiled and A.digits is not None and config is None):
        # the grouped kernel's route (group scales; zero points fused at decode token counts)
        ws_need = max(ws_need, int(L.lib().apt_gemm_grouped_workspace_bytes(1)))
    if ws_need > 0 and (workspace is None or workspace.numel() * workspace.element_size() < ws_need):
        if workspace is not None:
            raise ValueError(f"workspace holds {workspace.numel() * workspace.element_size()} bytes, "
                             f"apt_gemm needs {ws_need}")
        workspace = default_workspace(W.planes.device, ws_need)
    ws_ptr = workspace.data_ptr() if workspace is not None else None
    ws_len = workspace.numel() * workspace.element_size() if workspace is not None else 0
    ws, as_ = W.struct(), A.struct()
    rc = L.lib().apt_gemm(M, N, K, W.bits, A.bits, ctypes.byref(ws), ctypes.byref(as_),
                          ctypes.byref(sc) if sc is not None else None, kind, lay, out.data_ptr(), out.stride(0),
                          ctypes.byref(c) if c is not None else None, ws_ptr, ws_len, _stream_handle(stream))
    L.check("apt_gemm", rc)
    return out


def _scales_struct(w_scale, a_scale, w_zero, a_zero, w_gscale, a_gscale, K, N, M):
    """apt_scales from fp32 device tensors (None = NULL); group scales [Kpad/128, N] / [Kpad/128, M]."""
    ts = (("w_scale", w_scale, N), ("a_scale", a_scale, M), ("w_zero", w_zero, N), ("a_zero", a_zero, M),
          ("w_gscale", w_gscale, kpad(K) // 128 * N), ("a_gscale", a_gscale, kpad(K) // 128 * M))
    if all(t is None for _, t, _ in ts):
        return None
    for nm, t, size in ts:
        if t is not None:
            _require_cuda(t, nm)
            if t.dtype != torch.float32 or not t.is_contiguous() or t.numel() < size:
                raise ValueError(f"{nm} must be a contiguous fp32 tensor of >= {size} elements")
    if a_gscale is not None and w_gscale is None:
        raise ValueError("a_gscale needs w_gscale (group-wise scales)")
    return L.AptScales(*(t.data_ptr() if t is not None else None for _, t, _ in ts),
                       128 if w_gscale is not None else 0)


def grouped_workspace(device) -> torch.Tensor:
    """A zero-initialised workspace large enough for apt_gemm_grouped (and, since its ticket area is
    shared, usable by apt_gemm calls on the same stream as well)."""
    nbytes = int(L.lib().apt_gemm_grouped_workspace_bytes(1))
    return default_workspace(device, nbytes)


def gemm_grouped(problems, workspace: torch.Tensor | None = None, stream=None) -> list:
    """apt_gemm_grouped: several INDEPENDENT decode GEMMs (M <= 16 each) in one persistent launch.

    ``problems`` is a sequence of dicts with the keys of :func:`gemm`: ``W`` (tile-major Packed),
    ``A`` (Packed with its digit view), and optionally ``out_kind``, ``layout``, ``w_scale``,
    ``a_scale``, ``w_zero``, ``a_zero``, ``w_gscale``, ``a_gscale``, ``out``, ``out_peers`` (up to 7
    further outputs written with the same values at the same offsets: tensors shaped like ``out`` or device
    pointers, e.g. symmetric-memory peer buffers, NEXT-4 ii).  Returns the list of outputs; each equals
    ``gemm`` on the same arguments."""
    problems = list(problems)
    n = len(problems)
    if not 1 <= n <= L.APT_GROUP_MAX:
        raise ValueError(f"apt_gemm_grouped takes 1..{L.APT_GROUP_MAX} problems, got {n}")
    arr = (L.AptGemmProblem * n)()
    outs = []
    dev = None
    for i, pr in enumerate(problems):
        W, A = pr["W"], pr["A"]
        _require_cuda(W.planes, "W.planes")
        _require_cuda(A.planes, "A.planes")
        dev = W.planes.device
        if A.k != W.k:
            raise ValueError(f"problem {i}: A and W have different K")
        M, N, K = A.rows, W.rows, W.k
        kind = _OUT_KINDS[pr.get("out_kind", "i32")]
        lay = _LAYOUTS[pr.get("layout", "row")]
        shape = (M, N) if lay == L.APT_LAYOUT_ROW else (N, M)
        dtype = torch.float16 if kind == L.APT_OUT_F16_SCALED else torch.int32
        out = pr.get("out")
        if out is None:
            out = torch.empty(shape, dtype=dtype, device=dev)
        if out.dtype != dtype or out.dim() != 2 or out.stride(1) != 1 or tuple(out.shape) != shape:
            raise ValueError(f"problem {i}: out must be a {dtype} tensor of shape {shape} with unit inner stride")
        sc = _scales_struct(pr.get("w_scale"), pr.get("a_scale"), pr.get("w_zero"), pr.get("a_zero"),
                            pr.get("w_gscale"), pr.get("a_gscale"), K, N, M)
        p = arr[i]
        p.M, p.N, p.K, p.wbits, p.abits = M, N, K, W.bits, A.bits
        p.W, p.A = W.struct(), A.struct()
        if sc is not None:
            p.scales = sc
        p.kind, p.layout, p.out, p.ldo = kind, lay, out.data_ptr(), out.stride(0)
        peers = list(pr.get("out_peers") or [])
        if len(peers) > L.APT_MAX_PEERS:
            raise ValueError(f"problem {i}: at most {L.APT_MAX_PEERS} peer outputs")
        for j, t in enumerate(peers):  # tensors shaped like out, or raw device pointers (symmetric memory)
            if isinstance(t, torch.Tensor) and (t.dtype != dtype or tuple(t.shape) != shape or t.stride() != out.stride()):
                raise ValueError(f"problem {i}: peer output {j} must match out's dtype, shape and strides")
            p.out_peers[j] = t.data_ptr() if isinstance(t, torch.Tensor) else int(t)
        p.n_peers = len(peers)
        outs.append(out)
    if workspace is None:
        workspace = grouped_workspace(dev)
    rc = L.lib().apt_gemm_grouped(n, arr, workspace.data_ptr(), workspace.numel() * workspace.element_size(),
                                  _stream_handle(stream))
    L.check("apt_gemm_grouped", rc)
    return outs


def pack_grouped(problems, stream=None) -> list:
    """apt_pack_grouped: several independent ACTIVATION packs (digit views, <= 64 rows each) in one launch.

    Each problem is a dict with ``out`` (a Packed with a digit view, e.g. ``alloc_packed(..., digits=True)``)
    and ``bits``, plus either ``codes`` (int8 [rows, k], apt_pack_bipolar semantics) or ``x`` (fp16
    [rows, k], apt_quantize_pack semantics, per-row scales written to ``scale``).  Returns the outs."""
    problems = list(problems)
    n = len(problems)
    if not 1 <= n <= L.APT_GROUP_MAX:
        raise ValueError(f"apt_pack_grouped takes 1..{L.APT_GROUP_MAX} problems, got {n}")
    arr = (L.AptPackProblem * n)()
    structs = []
    for i, pr in enumerate(problems):
        out, bits = pr["out"], int(pr["bits"])
        quant = "x" in pr
        src = pr["x"] if quant else pr["codes"]
        _require_cuda(src, "x" if quant else "codes")
        want = torch.float16 if quant else torch.int8
        if src.dtype != want or src.dim() != 2 or src.stride(1) != 1:
            raise ValueError(f"problem {i}: {'x' if quant else 'codes'} must be a 2-D {want} tensor with unit stride along K")
        rows, k = src.shape
        if out.digits is None or out.tiled:
            raise ValueError(f"problem {i}: out must be a row-layout Packed with a digit view")
        _check_out(out, rows, k, bits, False, True)
        scale = pr.get("scale")
        if quant and (scale is None or scale.dtype != torch.float32 or not scale.is_contiguous() or scale.numel() < rows):
            raise ValueError(f"problem {i}: quantize needs a contiguous fp32 scale of >= rows elements")
        st = out.struct()
        structs.append(st)
        p = arr[i]
        p.src, p.quantize, p.rows, p.k, p.bits, p.ld = src.data_ptr(), int(quant), rows, k, bits, src.stride(0)
        p.out = ctypes.pointer(st)
        p.scale = scale.data_ptr() if quant else None
        re_ = pr.get("range_error")
        p.range_error = re_.data_ptr() if re_ is not None else None
    L.check("apt_pack_grouped", L.lib().apt_pack_grouped(n, arr, _stream_handle(stream)))
    return [pr["out"] for pr in problems]
