"""B200-native APT-LLM arbitrary-precision W_p x A_q integer MatMul (arXiv 2508.19087).

Public API (torch tensors in, CUDA kernels of libapt.so underneath):
    pack(codes, bits)                    -> Packed bit-planes          (apt_pack_bipolar)
    quantize_pack(x_fp16, bits)          -> (Packed, per-token scale)  (apt_quantize_pack)
    pack_grouped([dict(codes=|x=, bits=, out=), ...]) -> several activation packs, one launch (apt_pack_grouped)
    gemm(W, A, out_kind=..., ...)         -> int32 / fp16 result        (apt_gemm)
    gemm_grouped([dict(W=, A=, ...), ...]) -> outputs of independent decode GEMMs, one launch (apt_gemm_grouped)
    select_config(M, N, K, wbits, abits) -> kernel configuration       (apt_select_config)
    load_table / table_lookup / enumerate_configs -> autotuned table (apt_table_*, NEXT-3)
    tp.TPLinear / tp.tp_gemm             -> N-split tensor parallel GEMM + all-gather
"""
from .api import Packed, alloc_packed, gemm, kpad, pack, quantize_pack, select_config, workspace_bytes, default_workspace  # noqa: F401
from .api import gemm_grouped, grouped_workspace, pack_grouped  # noqa: F401
from .api import clear_table, enumerate_configs, load_default_table, load_table, table_lookup, table_size  # noqa: F401
from . import _lib  # noqa: F401

__all__ = ["Packed", "alloc_packed", "gemm", "gemm_grouped", "grouped_workspace", "pack_grouped", "kpad", "pack", "quantize_pack", "select_config", "workspace_bytes", "default_workspace",
           "load_table", "clear_table", "table_size", "table_lookup", "enumerate_configs", "load_default_table"]
