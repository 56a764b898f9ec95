"""N-split tensor parallelism for the APT GEMM (north_star: "partitioned across the 8xB200 box by
splitting N (the weight output rows) tensor-parallel, with an NCCL all-gather of output columns").

Each rank owns a contiguous slice of weight rows [r*N/P, (r+1)*N/P), packs it once, computes its
slice of the output in COLUMN layout (Y_r^T, [N/P, M], contiguous), and one all-gather assembles
Y^T = [N, M] with no permute pass.  For large M the GEMM is chunked along M so that
the gather of chunk c overlaps the GEMM of chunk c+1 on a second stream.

torch.distributed is the plumbing (process groups, NCCL); every arithmetic step runs in libapt.so.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import api


def shard_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row slice of rank `rank`: (start, length).  N must divide evenly (the Llama shapes
    4096, 8192, 11008, 28672 all divide by 1, 2, 4 and 8)."""
    if n % world != 0:
        raise ValueError(f"N={n} is not divisible by the tensor-parallel world size {world}")
    per = n // world
    return rank * per, per


def _all_gather_rows(out_full: torch.Tensor, local: torch.Tensor, group=None):
    """Gather equal row blocks of every rank into out_full ([P*rows, cols]) in rank order."""
    try:
        dist.all_gather_into_tensor(out_full, local, group=group)
    except (RuntimeError, NotImplementedError, ValueError):
        world = dist.get_world_size(group)
        parts = list(out_full.chunk(world, dim=0))
        dist.all_gather(parts, local, group=group)


def tp_gemm(W_local: api.Packed, A: api.Packed, n_total: int, out_kind: str = "i32",
            w_scale_local: torch.Tensor | None = None, a_scale: torch.Tensor | None = None,
            group=None, m_chunks: int = 1, local_gemm=None) -> torch.Tensor:
    """Y^T [n_total, M] = gather over ranks of (A . W_r^T)^T.

    ``local_gemm(W_local, A_chunk_rows, out_kind, w_scale_local, a_scale_chunk) -> [N/P, m]`` is the
    per-rank compute; it defaults to the CUDA kernel (api.gemm, column layout).  Tests on CPU
    inject the oracle here to exercise the sharding and collective logic with gloo.
    """
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    n_local = W_local.rows
    if n_local * world != n_total:
        raise ValueError("W_local rows x world size != n_total")
    M = A.rows
    dtype = torch.float16 if out_kind == "f16" else torch.int32
    device = W_local.planes.device
    yt = torch.empty((n_total, M), dtype=dtype, device=device)
    if local_gemm is None:
        def local_gemm(Wl, Ac, kind, ws, as_):
            return api.gemm(Wl, Ac, out_kind=kind, layout="col", w_scale=ws, a_scale=as_)
    if m_chunks <= 1 or world == 1:
        y_local = local_gemm(W_local, A, out_kind, w_scale_local, a_scale)
        if world == 1:
            return y_local
        _all_gather_rows(yt, y_local.contiguous(), group)
        return yt
    # chunk M: gather chunk c on a side stream while chunk c+1 computes
    bounds = [(M * c) // m_chunks for c in range(m_chunks + 1)]
    comm = torch.cuda.Stream(device=device) if device.type == "cuda" else None
    pending = []
    for c in range(m_chunks):
        m0, m1 = bounds[c], bounds[c + 1]
        if m1 <= m0:
            continue
        A_c = A.narrow_rows(m0, m1 - m0)
        y_c = local_gemm(W_local, A_c, out_kind, w_scale_local, a_scale[m0:m1] if a_scale is not None else None)
        buf = torch.empty((n_total, m1 - m0), dtype=dtype, device=device)
        if comm is not None:
            ev = torch.cuda.Event()
            ev.record()
            with torch.cuda.stream(comm):
                comm.wait_event(ev)
                _all_gather_rows(buf, y_c.contiguous(), group)
        else:
            _all_gather_rows(buf, y_c.contiguous(), group)
        pending.append((m0, m1, buf, y_c))
    if comm is not None:
        torch.cuda.current_stream(device).wait_stream(comm)
    for m0, m1, buf, _ in pending:
        yt[:, m0:m1].copy_(buf)
    return yt
