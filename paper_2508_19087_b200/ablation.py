"""The paper's ablation on B200 (§6.5): the "Basic" design — one 1-bit x
1-bit GEMM per plane pair (digit width 1: the paper's bit-plane products) with the recovery
(shift-add) done in global memory — against the product path (digits of full width, the
shift-add folded into the operand rebuild and the tensor core's accumulate).

Every arithmetic step runs in libapt.so kernels: the plane pairs through apt_gemm (W1 x A1 codes,
bipolar int32 output = sum_k (2a_i - 1)(2w_j - 1)), the recovery through apt_recombine_plane_products.
"""
from __future__ import annotations

import torch

from . import _lib as L
from . import api


def split_planes(codes: torch.Tensor, bits: int) -> list[torch.Tensor]:
    """Signed n-bit codes -> n one-bit signed code matrices (bit i of u = x + 2^(n-1), minus 1: {-1, 0}),
    whose bipolar values 2x'+1 = 2 u_i - 1 are the paper's +-1 planes.  Input preparation
    (like weight packing, offline), int8 in and out."""
    u = codes.to(torch.int16) + (1 << (bits - 1))
    return [(((u >> i) & 1) - 1).to(torch.int8).contiguous() for i in range(bits)]


class PlanePairs:
    """Both operands as 1-bit packed planes, ready for the Basic ablation."""

    def __init__(self, a_codes: torch.Tensor, abits: int, w_codes: torch.Tensor, wbits: int):
        self.abits, self.wbits = abits, wbits
        self.M, self.N = a_codes.shape[0], w_codes.shape[0]
        self.A = [api.pack(p, 1, digits=True) for p in split_planes(a_codes, abits)]
        self.W = [api.pack(p, 1, tiled=True) for p in split_planes(w_codes, wbits)]
        self.parts = torch.empty((abits * wbits, self.M, self.N), dtype=torch.int32, device=a_codes.device)
        self.cfg = api.select_config(self.M, self.N, w_codes.shape[1], 1, 1)

    def basic(self, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """Y' (bipolar product, int32 [M, N]) the Basic way: p_a * p_w plane-pair GEMMs to HBM, then the
        shift-add recovery in global memory."""
        for i, Ai in enumerate(self.A):
            for j, Wj in enumerate(self.W):
                api.gemm(Wj, Ai, out_kind="bipolar", out=self.parts[i * self.wbits + j], config=self.cfg, stream=stream)
        if out is None:
            out = torch.empty((self.M, self.N), dtype=torch.int32, device=self.parts.device)
        n = self.M * self.N
        L.check("apt_recombine_plane_products",
                L.lib().apt_recombine_plane_products(self.parts.data_ptr(), self.abits, self.wbits, n, n,
                                                     out.data_ptr(), api._stream_handle(stream)))
        return out
