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


def tp_gemm(W_local: api.Packed, A, n_total: int, out_kind: str = "i32",
            w_scale_local: torch.Tensor | None = None, a_scale: torch.Tensor | None = None,
            group=None, m_chunks: int = 1, local_gemm=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """Gathered Y^T over the ranks' weight-row slices: (A . W_r^T)^T stacked in rank order.

    ``A`` is one Packed activation [M, K] or a list of ``m_chunks`` Packed row chunks of equal size (pack
    the chunks directly to avoid the plane copies ``Packed.narrow_rows`` makes).  Returns Y^T [n_total, M]
    for one chunk, else the chunk-major [m_chunks, n_total, M / m_chunks]: chunk c's gather lands in its own
    contiguous block, so there is no permute or copy pass, and the gather of chunk c runs on a
    side stream while the GEMM of chunk c + 1 computes.

    ``local_gemm(W_local, A_chunk, out_kind, w_scale_local, a_scale_chunk) -> [N/P, m]`` is the per-rank
    compute; it defaults to the CUDA kernel (api.gemm, column layout).  Tests on CPU inject the oracle here
    to exercise the sharding and collective logic with gloo.
    """
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    n_local = W_local.rows
    if n_local * world != n_total:
        raise ValueError("W_local rows x world size != n_total")
    chunks = list(A) if isinstance(A, (list, tuple)) else None
    if chunks is not None:
        m_chunks = len(chunks)
    M = sum(c.rows for c in chunks) if chunks is not None else A.rows
    m_chunks = max(1, m_chunks)
    if M % m_chunks != 0:
        raise ValueError(f"M={M} is not divisible into {m_chunks} equal chunks")
    mc = M // m_chunks
    if chunks is None:
        chunks = [A] if m_chunks == 1 else [A.narrow_rows(c * mc, mc) for c in range(m_chunks)]
    if any(c.rows != mc for c in chunks):
        raise ValueError("activation chunks must have equal row counts")
    dtype = torch.float16 if out_kind == "f16" else torch.int32
    device = W_local.planes.device
    direct = local_gemm is None  # the CUDA kernel can write a single rank's blocks in place
    if local_gemm is None:
        def local_gemm(Wl, Ac, kind, ws, as_):
            return api.gemm(Wl, Ac, out_kind=kind, layout="col", w_scale=ws, a_scale=as_)
    shape = (n_total, M) if m_chunks == 1 else (m_chunks, n_total, mc)
    if out is None:
        out = torch.empty(shape, dtype=dtype, device=device)
    elif tuple(out.shape) != shape or out.dtype != dtype or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous {dtype} tensor of shape {shape}")
    blocks = [out] if m_chunks == 1 else [out[c] for c in range(m_chunks)]
    comm = torch.cuda.Stream(device=device) if (device.type == "cuda" and world > 1 and m_chunks > 1) else None
    for c, A_c in enumerate(chunks):
        as_c = a_scale[c * mc:(c + 1) * mc] if a_scale is not None else None
        if world == 1:
            # single rank: the local GEMM writes the block directly
            if direct:
                api.gemm(W_local, A_c, out_kind=out_kind, layout="col", w_scale=w_scale_local, a_scale=as_c,
                         out=blocks[c])
            else:
                blocks[c].copy_(local_gemm(W_local, A_c, out_kind, w_scale_local, as_c))
            continue
        y_c = local_gemm(W_local, A_c, out_kind, w_scale_local, as_c)
        if comm is not None:
            ev = torch.cuda.Event()
            ev.record()
            with torch.cuda.stream(comm):
                comm.wait_event(ev)
                _all_gather_rows(blocks[c], y_c.contiguous(), group)
                y_c.record_stream(comm)
        else:
            _all_gather_rows(blocks[c], y_c.contiguous(), group)
    if comm is not None:
        torch.cuda.current_stream(device).wait_stream(comm)
    return out


# ----------------------------------------------------------------------------- epilogue-direct peer stores

def peer_slice_offset(rank: int, n_local: int, m: int, elem_bytes: int) -> int:
    """Byte offset of rank `rank`'s slice (weight rows [rank n_local, (rank + 1) n_local)) in a gathered
    column-layout output Y^T [world n_local, m]."""
    return rank * n_local * m * elem_bytes


def symmetric_outputs(shapes, dtype, group=None):
    """Gathered outputs [N_total, M] in symmetric memory (torch.distributed._symmetric_memory) and their
    rendezvous handles: every rank can store into every other rank's buffer over NVLink."""
    import torch.distributed._symmetric_memory as symm_mem
    dev = torch.device("cuda", torch.cuda.current_device())
    grp = group if group is not None else dist.group.WORLD
    bufs = [symm_mem.empty(tuple(sh), dtype=dtype, device=dev) for sh in shapes]
    handles = [symm_mem.rendezvous(b, grp) for b in bufs]
    return bufs, handles


def tp_grouped_decode_peer(problems_local, gathered, handles, group=None, stream=None):
    """N-split decode GEMMs whose epilogue is the all-gather (SURVEY §8f NEXT-4 ii).

    ``problems_local`` are apt_gemm_grouped problems of this rank (``W`` = its row slice, tile-major; ``A``
    replicated with its digit view; scales etc. as api.gemm_grouped); ``gathered[i]`` is the symmetric
    [N_total, M] column-layout output of problem i and ``handles[i]`` its rendezvous handle.  Rank r writes
    its slice Y_r^T into rows [r N/P, (r+1) N/P) of its own buffer AND of every peer's buffer straight from
    the GEMM's epilogue (peer pointers of the symmetric allocation, same offsets), then one symmetric-memory
    barrier makes every slice visible on every rank: no staging buffer, no collective copy."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    probs = []
    for pr, buf, h in zip(problems_local, gathered, handles):
        n_local, m = pr["W"].rows, pr["A"].rows
        if buf.shape[0] != n_local * world or buf.shape[1] != m:
            raise ValueError("gathered output must be [N_local * world, M]")
        base = buf.data_ptr() - int(h.buffer_ptrs[rank])  # the tensor's offset inside the symmetric allocation
        off = peer_slice_offset(rank, n_local, m, buf.element_size())
        peers = [int(h.buffer_ptrs[j]) + base + off for j in range(world) if j != rank]
        probs.append(dict(pr, layout="col", out=buf[rank * n_local:(rank + 1) * n_local], out_peers=peers))
    api.gemm_grouped(probs, stream=stream)
    if world > 1 and handles:
        handles[0].barrier()  # stream-ordered: every rank's epilogue stores are visible after it
    return gathered
