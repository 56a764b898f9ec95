"""World-size-2 gloo tests of the tensor-parallel N-split + all-gather logic (CPU).

The per-rank compute is injected as the CPU oracle (tests only), so these tests exercise the
sharding, the column-layout gather and the M-chunked path of paper_2508_19087_b200.tp without a
GPU; the CUDA local GEMM itself is covered by the gpu parity tests.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import apt_oracle as O
from synth import signed_codes


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, n, k, wbits, abits, chunks, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2508_19087_b200 import api, tp
        a = signed_codes(m, k, abits, seed=1)
        w = signed_codes(n, k, wbits, seed=2)
        start, length = tp.shard_rows(n, world, rank)
        w_loc = w[start:start + length]
        planes, rs = O.pack_planes(w_loc, wbits)
        W_local = api.Packed(torch.from_numpy(planes.view(np.int32)), torch.from_numpy(rs.astype(np.int32)),
                             length, k, wbits)
        ap, ars = O.pack_planes(a, abits)
        A = api.Packed(torch.from_numpy(ap.view(np.int32)), torch.from_numpy(ars.astype(np.int32)), m, k, abits)

        def oracle_local(Wl, Ac, kind, ws, as_):
            codes_a = O.unpack_planes(Ac.planes.numpy().view(np.uint32), Ac.k, Ac.bits)
            codes_w = O.unpack_planes(Wl.planes.numpy().view(np.uint32), Wl.k, Wl.bits)
            return torch.from_numpy(O.gemm_signed(codes_a, codes_w).T.astype(np.int32).copy())

        yt = tp.tp_gemm(W_local, A, n, out_kind="i32", m_chunks=chunks, local_gemm=oracle_local)
        ref = O.gemm_signed(a, w).T  # [n, m]
        if chunks > 1:  # chunk-major [chunks, n, m / chunks]: chunk c = columns c*mc .. of Y^T
            mc = m // chunks
            ref = np.stack([ref[:, c * mc:(c + 1) * mc] for c in range(chunks)])
        ok = np.array_equal(yt.numpy().astype(np.int64), ref)
        q.put((rank, bool(ok), tuple(yt.shape)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("chunks", [1, 3])
def test_tp_gather_matches_single_device(chunks):
    world, m, n, k = 2, 9, 64, 300
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, k, 3, 2, chunks, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert all(shape == ((n, m) if chunks == 1 else (chunks, n, m // chunks)) for _, _, shape in res)


def test_shard_rows():
    from paper_2508_19087_b200 import tp
    assert tp.shard_rows(28672, 8, 3) == (3 * 3584, 3584)
    assert tp.shard_rows(8192, 4, 0) == (0, 2048)
    with pytest.raises(ValueError):
        tp.shard_rows(100, 8, 0)


def test_peer_slice_offsets_tile_the_gathered_output():
    """The byte offsets of the ranks' slices (epilogue-direct peer stores) tile the gathered column-layout
    output exactly: rank r's rows [r n/P, (r+1) n/P) of Y^T [n, m], no overlap, no gap."""
    from paper_2508_19087_b200 import tp
    for world in (1, 2, 4, 8):
        n, m, es = 4096, 16, 2
        n_local = n // world
        spans = [(tp.peer_slice_offset(r, n_local, m, es), tp.peer_slice_offset(r, n_local, m, es) + n_local * m * es)
                 for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == n * m * es
        assert all(spans[r][1] == spans[r + 1][0] for r in range(world - 1))
