"""GPU parity of the grouped decode GEMM (apt_gemm_grouped, gemm_grp.cu) against the CPU oracle.

Each problem of a group must equal the oracle exactly like a single apt_gemm call (int32 bit-exact,
fp16 within 1e-3 of the fp64-scaled oracle), whatever the group around it: the
stream-K schedule splits row tiles between warps at arbitrary K blocks and across problem boundaries.
"""
import numpy as np
import pytest
import torch

from oracle import apt_oracle as O
from oracle import c_gemm_i64
from synth import config_seed, log_uniform_scales, signed_codes

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2508_19087_b200")

DEV = "cuda:0"
TOL = 1e-3


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _problem(m, n, k, pw, pa, seed, kind="i32", layout="row"):
    a = signed_codes(m, k, pa, seed=seed)
    w = signed_codes(n, k, pw, seed=seed + 1)
    ws = log_uniform_scales(n, -10, -6, seed=seed + 2)
    as_ = log_uniform_scales(m, -6, -2, seed=seed + 3)
    pr = dict(W=P.pack(_dev(w), pw, tiled=True), A=P.pack(_dev(a), pa, digits=True), out_kind=kind, layout=layout)
    if kind == "f16":
        pr.update(w_scale=_dev(ws), a_scale=_dev(as_))
    return pr, (a, w, ws, as_, pw, pa)


def _check(out, kind, layout, a, w, ws, as_, pw, pa, exact_ref=None):
    got = out.cpu().numpy()
    if layout == "col":
        got = got.T
    ref = exact_ref if exact_ref is not None else O.gemm_signed(a, w)
    if kind == "i32":
        assert np.array_equal(got.astype(np.int64), ref)
    elif kind == "bipolar":
        assert np.array_equal(got.astype(np.int64), O.gemm_bipolar(a, pa, w, pw))
    else:
        r = O.scale_fp64(ref, ws, as_)
        assert (np.abs(got.astype(np.float64) - r) <= TOL * np.abs(r) + 2.0 ** -24).all()


def _tickets_zero():
    torch.cuda.synchronize()
    ws = P.grouped_workspace(DEV)
    assert int(ws[:16384].count_nonzero().item()) == 0


RAGGED = [  # (m, n, k, pw, pa): N not a multiple of 32 / 128, K not a multiple of 256, tiny and long K
    (1, 333, 700, 1, 2), (3, 100, 64, 2, 2), (8, 41, 1300, 3, 4), (9, 256, 4096, 4, 4), (16, 300, 4096, 2, 8),
    (16, 1, 1, 1, 1), (5, 77, 2600, 4, 3), (2, 129, 513, 1, 8), (12, 64, 9000, 3, 2), (16, 40, 256, 4, 4),
]


@pytest.mark.parametrize("kind,layout", [("i32", "row"), ("bipolar", "col"), ("f16", "row"), ("f16", "col")])
def test_grouped_ragged_mixed(kind, layout):
    """Ten ragged problems of mixed width / token count in one launch."""
    prs, refs = zip(*[_problem(m, n, k, pw, pa, 500 + 7 * i, kind, layout) for i, (m, n, k, pw, pa) in enumerate(RAGGED)])
    outs = P.gemm_grouped(prs)
    for out, ref in zip(outs, refs):
        _check(out, kind, layout, *ref)
    _tickets_zero()


@pytest.mark.parametrize("wmax", [2, 4, 8])
@pytest.mark.parametrize("count", [1, 2, 7, 64])
def test_grouped_counts_and_width_classes(wmax, count):
    """1..64 problems (APT_GROUP_MAX), every kernel width class (WBMAX 2 / 4 / 8 rings)."""
    rng = np.random.default_rng(wmax * 100 + count)
    cases = []
    for i in range(count):
        m = int(rng.integers(1, 17))
        n = int(rng.integers(1, 400))
        k = int(rng.integers(1, 3000))
        pw = int(rng.integers(1, wmax + 1)) if i else wmax
        pa = int(rng.integers(1, 9))
        cases.append((m, n, k, pw, pa))
    prs, refs = zip(*[_problem(*c, seed=900 + 11 * i) for i, c in enumerate(cases)])
    outs = P.gemm_grouped(prs)
    for out, ref in zip(outs, refs):
        _check(out, "i32", "row", *ref)
    _tickets_zero()


def test_grouped_equals_apt_gemm_bitwise():
    """Same bits as the per-call apt_gemm (int32 and fp16) on decode-shaped problems."""
    cases = [(1, 4096, 4096, 1, 2), (8, 4096, 11008, 2, 2), (16, 11008, 4096, 4, 4), (16, 4096, 4096, 3, 4)]
    for kind in ("i32", "f16"):
        prs = [_problem(*c, seed=40 + i, kind=kind)[0] for i, c in enumerate(cases)]
        outs = P.gemm_grouped(prs)
        for pr, out in zip(prs, outs):
            one = P.gemm(pr["W"], pr["A"], out_kind=kind, w_scale=pr.get("w_scale"), a_scale=pr.get("a_scale"))
            assert torch.equal(one.view(torch.int16) if kind == "f16" else one,
                               out.view(torch.int16) if kind == "f16" else out)


LLAMA7B = [(4096, 4096), (11008, 4096), (4096, 11008)]
PRECISIONS = [(1, 2), (2, 2), (3, 4), (4, 4)]


@pytest.mark.parametrize("by_precision", [False, True])
def test_grouped_llama7b_decode_full(by_precision):
    """BASELINE configs[1] exactly as bench.py times the grouped leg: the 36 decode linears (fp16,
    per-channel w_scale, per-token a_scale) in one launch, or one launch per precision; every output
    element within 1e-3 of the fp64-scaled C int64 oracle."""
    groups = [[pq] for pq in PRECISIONS] if by_precision else [PRECISIONS]
    for precs in groups:
        prs, refs = [], []
        for (pw, pa) in precs:
            for (n, k) in LLAMA7B:
                for m in (1, 8, 16):
                    seed = config_seed(1, pw, pa, salt=13) + n + m
                    pr, ref = _problem(m, n, k, pw, pa, seed, kind="f16")
                    prs.append(pr)
                    refs.append(ref)
        outs = P.gemm_grouped(prs)
        for out, (a, w, ws, as_, pw, pa) in zip(outs, refs):
            _check(out, "f16", "row", a, w, ws, as_, pw, pa, exact_ref=c_gemm_i64(a, w))
    _tickets_zero()


def test_grouped_repeat_and_repack_stream_order():
    """50 back-to-back grouped calls on one stream, with the activations re-packed (different codes into
    the same buffers) right before every call: each call sees its own codes."""
    cases = [(16, 4096, 4096, 2, 2), (8, 11008, 4096, 4, 4), (1, 4096, 11008, 1, 2)]
    prs = [_problem(*c, seed=70 + i)[0] for i, c in enumerate(cases)]
    for it in range(50):
        refs = []
        for (m, n, k, pw, pa), pr, i in zip(cases, prs, range(3)):
            a = signed_codes(m, k, pa, seed=10000 + 3 * it + i)
            P.pack(_dev(a), pa, out=pr["A"])
            refs.append(a)
        outs = P.gemm_grouped(prs)
        if it % 10 == 9:
            for out, a, pr, (m, n, k, pw, pa) in zip(outs, refs, prs, cases):
                w = signed_codes(n, k, pw, seed=70 + cases.index((m, n, k, pw, pa)) + 1)
                assert np.array_equal(out.cpu().numpy().astype(np.int64), c_gemm_i64(a, w))
    _tickets_zero()


def test_grouped_extremes():
    """All-extreme codes at the largest K the unsigned digit sum allows (Kpad * 255 * 255 < 2^32)."""
    k = 66048
    prs, exp = [], []
    for av, wv, pw in ((-128, -2, 2), (127, 1, 2), (-128, 7, 4), (-1, -1, 1)):
        a = np.full((16, k), av, dtype=np.int8)
        w = np.full((40, k), wv, dtype=np.int8)
        prs.append(dict(W=P.pack(_dev(w), pw, tiled=True), A=P.pack(_dev(a), 8, digits=True)))
        exp.append(np.full((16, 40), k * av * wv, dtype=np.int64))
    for out, e in zip(P.gemm_grouped(prs), exp):
        assert np.array_equal(out.cpu().numpy().astype(np.int64), e)


def test_grouped_rejects():
    """Argument errors come back before any launch."""
    pr, _ = _problem(4, 64, 256, 2, 2, seed=3)
    bad_rows = dict(pr, W=P.pack(_dev(signed_codes(64, 256, 2, seed=4)), 2))  # canonical (row) layout
    bad_dig = dict(pr, A=P.pack(_dev(signed_codes(4, 256, 2, seed=5)), 2))     # no digit view
    bad_m = dict(pr, A=P.pack(_dev(signed_codes(17, 256, 2, seed=6)), 2, digits=True))
    for bad in (bad_rows, bad_dig, bad_m):
        with pytest.raises(P._lib.AptError):
            P.gemm_grouped([pr, bad])
    with pytest.raises(ValueError):
        P.gemm_grouped([pr] * 65)


# ----------------------------------------------------------------------------- grouped activation packs

PACK_CASES = [(1, 4096, 2), (8, 4096, 4), (16, 11008, 2), (3, 33, 1), (5, 257, 8), (64, 4096, 3), (16, 11008, 4),
              (2, 700, 5), (1, 1, 6), (9, 1300, 7)]


def test_pack_grouped_codes_matches_oracle_and_single():
    """apt_pack_grouped (int8 codes) == oracle.pack_planes (planes, row sums) and == the single-call
    apt_pack_bipolar digit view, bit for bit, for every problem of a mixed-width, ragged group."""
    prs, ref = [], []
    for i, (rows, k, bits) in enumerate(PACK_CASES):
        c = signed_codes(rows, k, bits, seed=300 + i)
        prs.append(dict(codes=_dev(c), bits=bits, out=P.alloc_packed(rows, k, bits, DEV, digits=True)))
        ref.append(c)
    P.pack_grouped(prs)
    torch.cuda.synchronize()
    for pr, c, (rows, k, bits) in zip(prs, ref, PACK_CASES):
        planes, rs = O.pack_planes(c, bits)
        out = pr["out"]
        assert np.array_equal(out.planes.cpu().numpy().view(np.uint32), planes)
        assert np.array_equal(out.row_sum.cpu().numpy().astype(np.int64), rs)
        one = P.pack(pr["codes"], bits, digits=True)
        assert torch.equal(one.digits, out.digits)


def test_pack_grouped_quantize_matches_oracle():
    """apt_pack_grouped (fp16, quantize) == oracle.quantize_symmetric + pack_planes: scales, planes, row
    sums bit-exact, digit view == the single-call apt_quantize_pack's."""
    from synth import fp16_activations
    prs, xs = [], []
    for i, (rows, k, bits) in enumerate(PACK_CASES):
        bits = max(bits, 2)
        x = fp16_activations(rows, k, seed=700 + i)
        prs.append(dict(x=_dev(x), bits=bits, out=P.alloc_packed(rows, k, bits, DEV, digits=True),
                        scale=torch.empty(rows, dtype=torch.float32, device=DEV)))
        xs.append(x)
    P.pack_grouped(prs)
    torch.cuda.synchronize()
    for pr, x in zip(prs, xs):
        bits = pr["bits"]
        codes, so = O.quantize_symmetric(x, bits)
        planes, rs = O.pack_planes(codes, bits)
        assert np.array_equal(pr["scale"].cpu().numpy(), so)
        assert np.array_equal(pr["out"].planes.cpu().numpy().view(np.uint32), planes)
        assert np.array_equal(pr["out"].row_sum.cpu().numpy().astype(np.int64), rs)
        one, _ = P.quantize_pack(pr["x"], bits)
        assert torch.equal(one.digits, pr["out"].digits)


def test_pack_grouped_then_gemm_grouped_stream_order():
    """The bench's step on one stream, 30 times with fresh codes each time: grouped packs straight into the
    grouped GEMM's activation buffers, every output equal to the C oracle."""
    cases = [(16, 4096, 4096, 2, 2), (8, 11008, 4096, 4, 4), (1, 4096, 11008, 1, 2)]
    W = [signed_codes(n, k, pw, seed=900 + i) for i, (m, n, k, pw, pa) in enumerate(cases)]
    prs = [dict(W=P.pack(_dev(w), pw, tiled=True), A=P.alloc_packed(m, k, pa, DEV, digits=True))
           for w, (m, n, k, pw, pa) in zip(W, cases)]
    for it in range(30):
        a = [signed_codes(m, k, pa, seed=5000 + 3 * it + i) for i, (m, n, k, pw, pa) in enumerate(cases)]
        P.pack_grouped([dict(codes=_dev(ai), bits=c[4], out=pr["A"]) for ai, c, pr in zip(a, cases, prs)])
        outs = P.gemm_grouped(prs)
        if it % 10 == 9:
            for out, ai, w in zip(outs, a, W):
                assert np.array_equal(out.cpu().numpy().astype(np.int64), c_gemm_i64(ai, w))


def test_pack_grouped_rejects():
    c = _dev(signed_codes(4, 256, 2, seed=1))
    with pytest.raises(ValueError):  # no digit view
        P.pack_grouped([dict(codes=c, bits=2, out=P.alloc_packed(4, 256, 2, DEV))])
    big = _dev(signed_codes(65, 256, 2, seed=2))  # more rows than the one-word-per-thread pack takes
    with pytest.raises(P._lib.AptError):
        P.pack_grouped([dict(codes=big, bits=2, out=P.alloc_packed(65, 256, 2, DEV, digits=True))])


# ----------------------------------------------------------------------------- NEXT-2: group scales, fused zero points

def _gs_problem(m, n, k, pw, pa, seed, a_groups=True, layout="row"):
    a = signed_codes(m, k, pa, seed=seed)
    w = signed_codes(n, k, pw, seed=seed + 1)
    G = O.kpad(k) // 128
    rng = np.random.default_rng(seed)
    wg = np.exp2(rng.uniform(-10, -6, (G, n))).astype(np.float32)
    ag = np.exp2(rng.uniform(-6, -2, (G, m))).astype(np.float32) if a_groups else None
    sa = np.exp2(rng.uniform(-6, -2, m)).astype(np.float32)
    pr = dict(W=P.pack(_dev(w), pw, tiled=True), A=P.pack(_dev(a), pa, digits=True), out_kind="f16", layout=layout,
              w_gscale=_dev(wg))
    if a_groups:
        pr["a_gscale"] = _dev(ag)
    else:
        pr["a_scale"] = _dev(sa)
    return pr, (a, w, wg, ag, sa)


def _gs_check(got, a, w, wg, ag, sa, layout="row"):
    """Reading R-G: fp32 sums of the groups' exactly computed products, one fp16 rounding; bound
    2^-11 |ref| (the rounding) + 2^-16 sum_g |Y_g s_w s_a| (fp32 accumulation over <= 256 groups) + 2^-24."""
    got = got.cpu().numpy().astype(np.float64)
    if layout == "col":
        got = got.T
    ref = O.group_dequant_gemm_fp64(a, w, wg, ag, None if ag is not None else sa)
    k = a.shape[1]
    mag = np.zeros_like(ref)
    for g in range(-(-k // 128)):
        yg = np.abs(O.gemm_signed(a[:, 128 * g:128 * g + 128], w[:, 128 * g:128 * g + 128]).astype(np.float64))
        s_a = ag[g].astype(np.float64) if ag is not None else sa.astype(np.float64)
        mag += yg * wg[g].astype(np.float64)[None, :] * s_a[:, None]
    assert (np.abs(got - ref) <= 2.0 ** -11 * np.abs(ref) + 2.0 ** -16 * mag + 2.0 ** -24).all()


@pytest.mark.parametrize("wmax", [2, 4, 8])
def test_group_scales_grouped(wmax):
    """apt_gemm_grouped with group-wise (128) scales on ragged problems of every width up to wmax, with and
    without activation group scales, both layouts, vs oracle.group_dequant_gemm_fp64."""
    rng = np.random.default_rng(40 + wmax)
    cases = [(int(rng.integers(1, 17)), int(rng.integers(1, 300)), int(rng.integers(1, 2000)),
              int(rng.integers(1, wmax + 1)) if i else wmax, int(rng.integers(1, 9))) for i in range(9)]
    prs, refs = [], []
    for i, c in enumerate(cases):
        pr, ref = _gs_problem(*c, seed=1200 + 17 * i, a_groups=bool(i % 2), layout="col" if i % 3 == 0 else "row")
        prs.append(pr)
        refs.append((ref, pr["layout"]))
    outs = P.gemm_grouped(prs)
    for out, (ref, lay) in zip(outs, refs):
        _gs_check(out, *ref, layout=lay)
    _tickets_zero()


@pytest.mark.parametrize("m", [1, 8, 16, 17, 100, 1030])
def test_group_scales_apt_gemm_any_m(m):
    """apt_gemm with group scales at any token count (chunks of 16 tokens, several grouped launches for
    m > 1024), Llama-like K = 4096 with K = 11008's ragged group count exercised at small m."""
    k = 11008 if m <= 16 else 4096
    n = 4096 if m <= 16 else 384
    pr, ref = _gs_problem(m, n, k, 4, 4, seed=77 + m, a_groups=m % 2 == 0)
    got = P.gemm(pr["W"], pr["A"], out_kind="f16", w_gscale=pr["w_gscale"], a_gscale=pr.get("a_gscale"),
                 a_scale=pr.get("a_scale"))
    _gs_check(got, *ref)
    _tickets_zero()


def test_group_scales_llama7b_decode_bench_shapes():
    """Group scales (W4A4, 128-groups on both operands, the Atom-128G configuration) at the 9 decode shapes
    of BASELINE configs[1] in one grouped launch, every output element vs the fp64 oracle."""
    prs, refs = [], []
    for (n, k) in LLAMA7B:
        for m in (1, 8, 16):
            pr, ref = _gs_problem(m, n, k, 4, 4, seed=n + k + m)
            prs.append(pr)
            refs.append(ref)
    for out, ref in zip(P.gemm_grouped(prs), refs):
        _gs_check(out, *ref)


@pytest.mark.parametrize("m", [1, 5, 16])
def test_zero_points_fused_decode(m):
    """Zero points at decode token counts go through the grouped kernel's epilogue (one launch); the
    result is bit-identical to the two-pass int32-Y route (forced by passing a config) and within the
    zero-point bound of the fp64 dequantize-then-multiply oracle."""
    n, k, pa, pw = 4096, 4096, 4, 3
    a = signed_codes(m, k, pa, seed=60 + m)
    w = signed_codes(n, k, pw, seed=61)
    rng = np.random.default_rng(m)
    ws = log_uniform_scales(n, -10, -6, seed=7)
    as_ = log_uniform_scales(m, -6, -2, seed=8)
    wz = (rng.uniform(-1, 1, n) * 2.0 ** -8).astype(np.float32)
    az = (rng.uniform(-1, 1, m) * 2.0 ** -3).astype(np.float32)
    A = P.pack(_dev(a), pa, digits=True)
    W = P.pack(_dev(w), pw, tiled=True)
    kw = dict(out_kind="f16", w_scale=_dev(ws), a_scale=_dev(as_), w_zero=_dev(wz), a_zero=_dev(az))
    fused = P.gemm(W, A, **kw)
    two_pass = P.gemm(W, A, config=P.select_config(m, n, k, pw, pa), **kw)
    assert torch.equal(fused.view(torch.int16), two_pass.view(torch.int16))
    ref = O.dequant_gemm_fp64(a, w, ws, as_, wz, az)
    y = O.gemm_signed(a, w).astype(np.float64)
    ra, rw = a.astype(np.float64).sum(1), w.astype(np.float64).sum(1)
    mag = (np.abs(y * ws[None, :] * as_[:, None]) + np.abs(rw[None, :] * ws[None, :] * az[:, None]) +
           np.abs(ra[:, None] * as_[:, None] * wz[None, :]) + np.abs(k * az[:, None] * wz[None, :]))
    assert (np.abs(fused.cpu().numpy().astype(np.float64) - ref) <= 1e-3 * mag + 2.0 ** -24).all()
    # the same problem inside a group with others
    outs = P.gemm_grouped([dict(W=W, A=A, **kw), _problem(16, 300, 700, 2, 2, seed=5, kind="f16")[0]])
    assert torch.equal(outs[0].view(torch.int16), fused.view(torch.int16))


# ----------------------------------------------------------------------------- NEXT-4 ii: epilogue-direct peer stores

@pytest.mark.parametrize("kind", ["i32", "f16", "gs"])
def test_peer_outputs_bitwise(kind):
    """The epilogue writes every element to out and to each peer output (up to 7) at the same offset:
    every copy bit-identical to the plain output, in row and column layout."""
    for layout in ("row", "col"):
        prs = []
        for i, (m, n, k, pw, pa) in enumerate([(16, 300, 1000, 4, 4), (1, 129, 513, 2, 2), (8, 256, 4096, 1, 8)]):
            if kind == "gs":
                pr, _ = _gs_problem(m, n, k, pw, pa, seed=80 + i, layout=layout)
            else:
                pr, _ = _problem(m, n, k, pw, pa, seed=80 + i, kind=kind, layout=layout)
            prs.append(pr)
        plain = [o.clone() for o in P.gemm_grouped(prs)]
        peered = []
        for pr, o in zip(prs, plain):
            peers = [torch.full_like(o, 7) for _ in range(3 if kind == "i32" else 7)]
            peered.append(peers)
            pr["out_peers"] = peers
            pr["out"] = torch.zeros_like(o)
        outs = P.gemm_grouped(prs)
        for o, p0, peers in zip(outs, plain, peered):
            assert torch.equal(o.view(torch.int16) if o.dtype == torch.float16 else o,
                               p0.view(torch.int16) if p0.dtype == torch.float16 else p0)
            for t in peers:
                assert torch.equal(t.view(torch.int16) if t.dtype == torch.float16 else t,
                                   o.view(torch.int16) if o.dtype == torch.float16 else o)


def test_tp_peer_decode_symmetric_memory_one_rank():
    """tp.tp_grouped_decode_peer on a one-rank NCCL group with symmetric-memory outputs (the code path
    of the multi-GPU decode; with one rank there are no peers, so this checks the plumbing and the slice
    placement against the oracle).  Skipped when symmetric memory is unavailable."""
    import os
    import torch.distributed as dist
    from paper_2508_19087_b200 import tp
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device(DEV))
    try:
        bufs, hs = tp.symmetric_outputs([(4096, 16), (11008, 8)], torch.float16)
    except Exception as exc:  # pragma: no cover - depends on the driver / torch build
        pytest.skip(f"symmetric memory unavailable: {exc!r}")
    prs, refs = [], []
    for i, (m, n, k, pw, pa) in enumerate([(16, 4096, 4096, 2, 2), (8, 11008, 4096, 4, 4)]):
        pr, ref = _problem(m, n, k, pw, pa, seed=300 + i, kind="f16")
        prs.append(pr)
        refs.append(ref)
    tp.tp_grouped_decode_peer(prs, bufs, hs)
    torch.cuda.synchronize()
    for b, (a, w, ws, as_, pw, pa) in zip(bufs, refs):
        _check(b, "f16", "col", a, w, ws, as_, pw, pa, exact_ref=c_gemm_i64(a, w))


def test_group_scales_deterministic():
    """The fp32 group-scale sums of a row tile split between CTAs are added in a fixed order: repeated
    launches give identical bits (the 9 decode shapes of W4A4, many split tiles)."""
    prs = []
    for (n, k) in LLAMA7B:
        for m in (1, 8, 16):
            prs.append(_gs_problem(m, n, k, 4, 4, seed=n + 3 * k + m)[0])
    first = [o.clone() for o in P.gemm_grouped(prs)]
    for _ in range(5):
        for a, b in zip(first, P.gemm_grouped(prs)):
            assert torch.equal(a.view(torch.int16), b.view(torch.int16))
