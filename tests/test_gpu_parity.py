"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Bars: packed planes and row sums bit-exact; int32 outputs (signed and
bipolar) bit-exact; fp16-scaled output within 1e-3 relative of the fp64 oracle.
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


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _pack_both(a_codes, abits, w_codes, wbits, tiled=True):
    A = P.pack(_dev(a_codes), abits)
    W = P.pack(_dev(w_codes), wbits, tiled=tiled)
    return A, W


def _tiled_from_rows(planes):
    """Tile-major view of canonical planes [bits][rows][kw] (APT_PACK_TILED, pad rows ignored)."""
    bits, rows, kw = planes.shape
    rb = -(-rows // 128)
    full = np.zeros((bits, rb * 128, kw), dtype=planes.dtype)
    full[:, :rows] = planes
    # [bits][rb][kw/8][2][128][4]
    return full.reshape(bits, rb, 128, kw // 8, 2, 4).transpose(0, 1, 3, 4, 2, 5)


# ----------------------------------------------------------------------------- pack (T6)

@pytest.mark.parametrize("bits", range(1, 9))
@pytest.mark.parametrize("rows,k", [(1, 1), (3, 31), (5, 33), (7, 255), (2, 257), (17, 4096), (3, 11008)])
def test_pack_matches_oracle(bits, rows, k):
    codes = signed_codes(rows, k, bits, seed=31 * bits + k + rows)
    got = P.pack(_dev(codes), bits)
    planes, rs = O.pack_planes(codes, bits)
    torch.cuda.synchronize()
    assert np.array_equal(got.planes.cpu().numpy().view(np.uint32), planes)
    assert np.array_equal(got.row_sum.cpu().numpy().astype(np.int64), rs)


@pytest.mark.parametrize("bits", [1, 3, 4, 8])
@pytest.mark.parametrize("rows,k", [(1, 1), (130, 700), (256, 4096)])
def test_pack_tiled_layout(bits, rows, k):
    """APT_PACK_TILED holds exactly the canonical words, tile-major (pad rows excluded)."""
    codes = signed_codes(rows, k, bits, seed=7 * bits + rows)
    got = P.pack(_dev(codes), bits, tiled=True)
    planes, rs = O.pack_planes(codes, bits)
    g = got.planes.cpu().numpy().view(np.uint32)
    rb = -(-rows // 128)
    g = g.reshape(bits, rb, planes.shape[2] // 8, 2, 128, 4)
    want = _tiled_from_rows(planes)
    for r in range(rows):
        assert np.array_equal(g[:, r // 128, :, :, r % 128, :], want[:, r // 128, :, :, r % 128, :])
    assert np.array_equal(got.row_sum.cpu().numpy().astype(np.int64), rs)


@pytest.mark.parametrize("bits", range(1, 8))
def test_pack_bipolar_encoding(bits):
    codes = signed_codes(9, 300, bits, seed=bits)
    bip = (2 * codes.astype(np.int64) + 1).astype(np.int8)
    got = P.pack(_dev(bip), bits, encoding="bipolar")
    planes, rs = O.pack_planes(codes, bits)
    assert np.array_equal(got.planes.cpu().numpy().view(np.uint32), planes)
    assert np.array_equal(got.row_sum.cpu().numpy().astype(np.int64), rs)


def test_pack_strided_rows():
    codes = signed_codes(6, 500, 3, seed=5)
    big = np.zeros((6, 777), dtype=np.int8)
    big[:, :500] = codes
    t = _dev(big)[:, :500]
    got = P.pack(t, 3)
    planes, _ = O.pack_planes(codes, 3)
    assert np.array_equal(got.planes.cpu().numpy().view(np.uint32), planes)


def test_pack_range_error_flag():
    codes = signed_codes(4, 100, 3, seed=9)
    codes[2, 17] = 5  # outside [-4, 3]
    flag = torch.zeros(1, dtype=torch.int32, device=DEV)
    P.pack(_dev(codes), 3, range_error=flag)
    assert int(flag.item()) == 2 * 100 + 17 + 1
    flag.zero_()
    P.pack(_dev(signed_codes(4, 100, 3, seed=9)), 3, range_error=flag)
    assert int(flag.item()) == 0


# ----------------------------------------------------------------------------- GEMM (T7)

def _check_gemm(a, abits, w, wbits, config=None, layouts=("row",), tiled=True):
    A, W = _pack_both(a, abits, w, wbits, tiled=tiled)
    y = O.gemm_signed(a, w)
    yb = O.gemm_bipolar(a, abits, w, wbits) if a.shape[1] * a.shape[0] * w.shape[0] < 3e6 else \
        4 * y + 2 * a.astype(np.int64).sum(1)[:, None] + 2 * w.astype(np.int64).sum(1)[None, :] + a.shape[1]
    for lay in layouts:
        got = P.gemm(W, A, out_kind="i32", layout=lay, config=config).cpu().numpy()
        got = got if lay == "row" else got.T
        assert np.array_equal(got.astype(np.int64), y), f"signed mismatch ({lay})"
        gotb = P.gemm(W, A, out_kind="bipolar", layout=lay, config=config).cpu().numpy()
        gotb = gotb if lay == "row" else gotb.T
        assert np.array_equal(gotb.astype(np.int64), yb), f"bipolar mismatch ({lay})"


@pytest.mark.parametrize("seed", range(20))
def test_config1_w2a2(seed):
    """BASELINE configs[0]: W2A2, M=16, N=K=256 (tiled and row-major weight planes)."""
    a = signed_codes(16, 256, 2, seed=config_seed(0, 2, 2, seed))
    w = signed_codes(256, 256, 2, seed=config_seed(0, 2, 2, seed) + 7)
    _check_gemm(a, 2, w, 2, layouts=("row", "col"), tiled=bool(seed % 2))


def test_random_set():
    """SPEC acceptance 1: random M, N, K in [1,300], p, q in [1,8] (200 instances)."""
    rng = np.random.default_rng(2024)
    for t in range(200):
        m, n, k = (int(v) for v in rng.integers(1, 301, size=3))
        pa, pw = (int(v) for v in rng.integers(1, 9, size=2))
        a = signed_codes(m, k, pa, seed=10 * t)
        w = signed_codes(n, k, pw, seed=10 * t + 1)
        _check_gemm(a, pa, w, pw)


@pytest.mark.parametrize("pa,pw", [(p, q) for p in range(1, 9) for q in range(1, 9)])
def test_all_precisions_ragged(pa, pw):
    """Every W_p x A_q combination on a shape with ragged M, N and K tails."""
    a = signed_codes(37, 700, pa, seed=100 * pa + pw)
    w = signed_codes(131, 700, pw, seed=100 * pw + pa + 5)
    _check_gemm(a, pa, w, pw)


def test_extreme_codes_overflow_edge():
    """All-minimum codes at the largest K the int32 bound allows for W8A8 (|Y| = K * 2^14)."""
    k = 33024
    a = np.full((3, k), -128, dtype=np.int8)
    w = np.full((70, k), -128, dtype=np.int8)
    _check_gemm(a, 8, w, 8)
    a[:, ::2] = 127
    _check_gemm(a, 8, w, 8)


def test_bound_rejected():
    a = signed_codes(2, 33025, 8, seed=1)
    A, W = _pack_both(a, 8, a, 8)
    with pytest.raises(RuntimeError, match="UNSUPPORTED"):
        P.gemm(W, A)


def _family_cfgs(m, n, k, wb, ab):
    """One legal configuration of every kernel family for an M <= 4 problem."""
    base = P.select_config(m, n, k, wb, ab)
    return {
        "gemv": dict(base, kernel=3, bm=32, bn=m, bk=128, split_k=8, stages=1, cta_pair=0, cluster_n=1),
        "skinny": dict(base, kernel=4, bm=16, bn=8, bk=256, split_k=8, stages=1, cta_pair=0, cluster_n=1),
        "tc": dict(base, kernel=2, bm=128, bn=16, bk=128, split_k=2, stages=_tc_stages(wb, 16), cta_pair=0,
                   cluster_n=1),
        "dec": dict(base, kernel=5, bm=32, bn=8 if m <= 8 else 16, bk=256, stages=4, split_k=3, cta_pair=0,
                    cluster_n=1),
    }


@pytest.mark.parametrize("wb,ab", [(3, 4), (1, 2), (8, 8)])
def test_config_invariance_families(wb, ab):
    """the GEMV, skinny mma.sync and tcgen05 kernels agree bit for bit on one problem (and
    with the oracle)."""
    m, n, k = 3, 333, 3000
    a = signed_codes(m, k, ab, seed=8 + wb)
    w = signed_codes(n, k, wb, seed=9 + ab)
    A = P.pack(_dev(a), ab, digits=True)
    W = P.pack(_dev(w), wb, tiled=True)
    ref = O.gemm_signed(a, w)
    for name, cfg in _family_cfgs(m, n, k, wb, ab).items():
        got = P.gemm(W, A, config=cfg).cpu().numpy().astype(np.int64)
        assert np.array_equal(got, ref), name


# ----------------------------------------------------------------------------- stream order (PDL)

@pytest.mark.parametrize("family", ["gemv", "skinny", "tc", "dec", "auto16"])
def test_repack_same_buffer_stream_order(family):
    """Stream order under programmatic dependent launch (include/apt.h "General contract"): pack W1
    into a buffer, GEMM, re-pack DIFFERENT codes W2 into the SAME buffer and GEMM immediately on one
    stream, 50 times, no host synchronisation in between.  Every GEMM must see the weights packed
    just before it (the GEMMs read weight planes / row sums / scales before griddepcontrol.wait)."""
    n, k = 28672, 4096  # the pack spans many waves
    m = 16 if family == "auto16" else 3
    wb, ab = 3, 4
    a = signed_codes(m, k, ab, seed=1)
    w1 = signed_codes(n, k, wb, seed=2)
    w2 = signed_codes(n, k, wb, seed=3)
    y1, y2 = c_gemm_i64(a, w1), c_gemm_i64(a, w2)
    A = P.pack(_dev(a), ab, digits=True)
    cfg = None if family == "auto16" else _family_cfgs(m, n, k, wb, ab)[family]
    d1, d2 = _dev(w1), _dev(w2)
    W = P.alloc_packed(n, k, wb, DEV, tiled=True)
    outs = []
    for it in range(50):
        P.pack(d1 if it % 2 == 0 else d2, wb, out=W)
        outs.append(P.gemm(W, A, config=cfg))
    torch.cuda.synchronize()
    for it, o in enumerate(outs):
        assert np.array_equal(o.cpu().numpy().astype(np.int64), y1 if it % 2 == 0 else y2), it


def _tc_stages(wb, bn):
    cw = 8
    slots = (6 if wb <= 4 else 3) if bn <= 64 else 2
    v = ((108 if bn <= 128 else 216) * 1024 - slots * wb * 128 * cw * 4 - (128 * (bn + 8) * 4 if bn <= 64 else 0)
         - 4096) // (bn * 128)
    return max(2, min(8, v))


@pytest.mark.parametrize("bn,cn,split", [(128, 1, 1), (128, 2, 1), (128, 4, 1), (256, 1, 1), (256, 2, 1),
                                         (16, 1, 2), (16, 1, 3), (16, 1, 8), (64, 1, 1), (64, 1, 5)])
@pytest.mark.parametrize("wb,ab", [(5, 3), (2, 8)])
def test_config_invariance_tc(bn, cn, split, wb, ab):
    """S:336 for the tcgen05 kernel: token tile width, cluster multicast and cluster split-K do not
    change the bits."""
    a = signed_codes(300, 3000, ab, seed=5)
    w = signed_codes(600, 3000, wb, seed=6)
    cfg = P.select_config(300, 600, 3000, wb, ab)
    cfg.update(kernel=2, bn=bn, cluster_n=cn, split_k=split, stages=_tc_stages(wb, bn))
    _check_gemm(a, ab, w, wb, config=cfg)


@pytest.mark.parametrize("m,pa,pw", [(1, 2, 1), (16, 4, 3), (300, 8, 2)])
def test_activation_digit_view(m, pa, pw):
    """The pack kernel's optional digit view: each 32-element word is a permutation of the word's
    offset digits u = x + 2^(n-1), and GEMMs reading it equal GEMMs expanding the planes."""
    k, n = 1000, 96
    a = signed_codes(m, k, pa, seed=40 + m)
    w = signed_codes(n, k, pw, seed=41 + m)
    A = P.pack(_dev(a), pa, digits=True)
    A0 = P.pack(_dev(a), pa)
    W = P.pack(_dev(w), pw)
    dig = A.digits.cpu().numpy().astype(np.int64)
    kp = O.kpad(k)
    u = np.zeros((m, kp), dtype=np.int64) + (1 << (pa - 1))
    u[:, :k] = O.offset_bits_matrix(a, pa)
    assert dig.shape == (m, kp)
    assert np.array_equal(np.sort(dig.reshape(m, -1, 32), axis=2), np.sort(u.reshape(m, -1, 32), axis=2))
    ref = O.gemm_signed(a, w)
    for kind in ("i32", "bipolar"):
        g1 = P.gemm(W, A, out_kind=kind).cpu().numpy()
        g0 = P.gemm(W, A0, out_kind=kind).cpu().numpy()
        assert np.array_equal(g1, g0)
    assert np.array_equal(P.gemm(W, A).cpu().numpy().astype(np.int64), ref)


# ----------------------------------------------------------------------------- fp16 epilogue (T9)

@pytest.mark.parametrize("pa,pw,m", [(2, 2, 16), (4, 4, 8), (8, 8, 5), (4, 3, 1)])
def test_f16_scaled(pa, pw, m):
    n, k = 300, 1000
    a = signed_codes(m, k, pa, seed=7 + pa)
    w = signed_codes(n, k, pw, seed=8 + pw)
    ws = log_uniform_scales(n, -10, -6, seed=1)
    as_ = log_uniform_scales(m, -6, -2, seed=2)
    A, W = _pack_both(a, pa, w, pw)
    ref = O.scale_fp64(O.gemm_signed(a, w), ws, as_)
    for lay in ("row", "col"):
        got = P.gemm(W, A, out_kind="f16", layout=lay, w_scale=_dev(ws), a_scale=_dev(as_)).cpu().numpy()
        got = (got if lay == "row" else got.T).astype(np.float64)
        err = np.abs(got - ref)
        assert (err <= 1e-3 * np.abs(ref) + 2.0 ** -24).all()
    got = P.gemm(W, A, out_kind="f16", w_scale=_dev(ws)).cpu().numpy().astype(np.float64)
    ref1 = O.scale_fp64(O.gemm_signed(a, w), ws, None)
    assert (np.abs(got - ref1) <= 1e-3 * np.abs(ref1) + 2.0 ** -24).all()


# ----------------------------------------------------------------------------- full-size configs (T8)

LLAMA7B = [(4096, 4096), (11008, 4096), (4096, 11008)]


@pytest.mark.parametrize("n,k", LLAMA7B)
@pytest.mark.parametrize("m", [1, 8, 16])
@pytest.mark.parametrize("pw,pa", [(1, 2), (2, 2), (3, 4), (4, 4)])
def test_llama7b_decode_full(n, k, m, pw, pa):
    """BASELINE configs[1] at full size in the bench's launch configuration (selector default),
    every output element vs the C int64 oracle."""
    a = signed_codes(m, k, pa, seed=config_seed(1, pw, pa))
    w = signed_codes(n, k, pw, seed=config_seed(1, pw, pa) + 1)
    A, W = _pack_both(a, pa, w, pw)
    got = P.gemm(W, A).cpu().numpy().astype(np.int64)
    assert np.array_equal(got, c_gemm_i64(a, w))


@pytest.mark.parametrize("n,k", LLAMA7B)
@pytest.mark.parametrize("m", [1, 8, 16])
@pytest.mark.parametrize("pw,pa", [(1, 2), (2, 2), (3, 4), (4, 4)])
def test_llama7b_decode_full_f16(n, k, m, pw, pa):
    """The bench's exact call at every BASELINE configs[1] shape: fp16 output with per-channel
    w_scale and per-token a_scale (selector default config), every element within 1e-3 of the
    fp64-scaled oracle (reading Q10/Q14)."""
    a = signed_codes(m, k, pa, seed=config_seed(1, pw, pa, salt=7))
    w = signed_codes(n, k, pw, seed=config_seed(1, pw, pa, salt=7) + 1)
    ws = log_uniform_scales(n, -10, -6, seed=n + pw)
    as_ = log_uniform_scales(m, -6, -2, seed=m + pa)
    A = P.pack(_dev(a), pa, digits=True)
    W = P.pack(_dev(w), pw, tiled=True)
    got = P.gemm(W, A, out_kind="f16", w_scale=_dev(ws), a_scale=_dev(as_)).cpu().numpy().astype(np.float64)
    ref = O.scale_fp64(c_gemm_i64(a, w), ws, as_)
    assert (np.abs(got - ref) <= 1e-3 * np.abs(ref) + 2.0 ** -24).all()


@pytest.mark.parametrize("n,k", LLAMA7B)
@pytest.mark.parametrize("pw,pa", [(2, 8), (4, 4)])
def test_llama7b_prefill_full(n, k, pw, pa):
    """BASELINE configs[2] (M=2048) at full size in the selector's launch configuration: EVERY
    output element vs the oracle (gemm_signed_blas, exact), plus the row-sum identity."""
    m = 2048
    a = signed_codes(m, k, pa, seed=config_seed(2, pw, pa))
    w = signed_codes(n, k, pw, seed=config_seed(2, pw, pa) + 1)
    A, W = _pack_both(a, pa, w, pw)
    got = P.gemm(W, A).cpu().numpy().astype(np.int64)
    assert np.array_equal(got, O.gemm_signed_blas(a, w))
    wsum = w.astype(np.int64).sum(0)
    assert np.array_equal(got.sum(1), a.astype(np.int64) @ wsum)


# ----------------------------------------------------------------------------- fused quantize + pack (NEXT-1)

@pytest.mark.parametrize("bits", range(2, 9))
@pytest.mark.parametrize("rows,k", [(1, 1), (3, 33), (16, 4096), (5, 11008), (2, 1000)])
def test_quantize_pack_matches_oracle(bits, rows, k):
    """apt_quantize_pack vs oracle.quantize_symmetric + oracle.pack_planes: scales, planes, row sums
    bit-exact; the digit view holds the same offset digits."""
    from synth import fp16_activations
    x = fp16_activations(rows, k, seed=bits * 1000 + rows + k)
    if rows > 2:
        x[2] = 0  # an all-zero row: s = 0, codes 0
    Pk, s = P.quantize_pack(_dev(x), bits)
    codes, so = O.quantize_symmetric(x, bits)
    planes, rs = O.pack_planes(codes, bits)
    torch.cuda.synchronize()
    assert np.array_equal(s.cpu().numpy(), so)
    assert np.array_equal(Pk.planes.cpu().numpy().view(np.uint32), planes)
    assert np.array_equal(Pk.row_sum.cpu().numpy().astype(np.int64), rs)
    dig = Pk.digits.cpu().numpy().astype(np.int64)
    u = np.zeros((rows, O.kpad(k)), dtype=np.int64) + (1 << (bits - 1))
    u[:, :k] = O.offset_bits_matrix(codes, bits)
    assert np.array_equal(np.sort(dig.reshape(rows, -1, 32), axis=2), np.sort(u.reshape(rows, -1, 32), axis=2))


def test_quantize_pack_ties_and_strides():
    """Exact half-integer quotients (rint half-to-even) and a row stride > k."""
    x = np.zeros((4, 300), dtype=np.float16)
    x[:, 0] = 7.0                           # n = 4: s = 1.0 exactly
    x[:, 1:15] = np.arange(-3.5, 3.5, 0.5)  # ties at +-0.5, +-1.5, ... and exact integers
    big = np.zeros((4, 320), dtype=np.float16)
    big[:, :300] = x
    t = _dev(big)[:, :300]
    Pk, s = P.quantize_pack(t, 4)
    codes, so = O.quantize_symmetric(x, 4)
    planes, _ = O.pack_planes(codes, 4)
    assert np.array_equal(s.cpu().numpy(), so) and so[0] == 1.0
    assert np.array_equal(Pk.planes.cpu().numpy().view(np.uint32), planes)


@pytest.mark.parametrize("m,pa,pw", [(1, 4, 2), (16, 4, 4), (300, 8, 2)])
def test_quantize_pack_then_gemm_f16(m, pa, pw):
    """fp16 activations -> apt_quantize_pack -> apt_gemm(fp16, a_scale = the quantize scale) vs the
    fp64-scaled oracle on the oracle's own codes and scales."""
    from synth import fp16_activations
    n, k = 384, 4096
    x = fp16_activations(m, k, seed=m + 10 * pa)
    w = signed_codes(n, k, pw, seed=5)
    ws = log_uniform_scales(n, -10, -6, seed=6)
    A, s = P.quantize_pack(_dev(x), pa)
    W = P.pack(_dev(w), pw, tiled=True)
    got = P.gemm(W, A, out_kind="f16", w_scale=_dev(ws), a_scale=s).cpu().numpy().astype(np.float64)
    codes, so = O.quantize_symmetric(x, pa)
    ref = O.scale_fp64(O.gemm_signed(codes, w), ws, so)
    assert (np.abs(got - ref) <= 1e-3 * np.abs(ref) + 2.0 ** -24).all()


# ----------------------------------------------------------------------------- SIMT GEMV (M <= 4)

def _gemv_cfg(m, n, k, wb, ab, warps=8):
    return dict(P.select_config(m, n, k, wb, ab), kernel=3, bm=32, bn=m, bk=128, split_k=warps, stages=1,
                cta_pair=0, cluster_n=1)


@pytest.mark.parametrize("m", [1, 2, 3, 4])
@pytest.mark.parametrize("pw,pa", [(1, 1), (1, 2), (2, 2), (3, 4), (4, 4), (5, 3), (8, 8), (7, 1)])
@pytest.mark.parametrize("tiled", [True, False])
@pytest.mark.parametrize("warps", [8, 16])
def test_gemv_matches_oracle(m, pw, pa, tiled, warps):
    """APT_KERNEL_GEMV: int32 signed and bipolar bit-exact, fp16 within 1e-3, on a ragged shape
    (N not a multiple of 32 or 128, K not a multiple of 256, fewer K steps than warps)."""
    for n, k in ((333, 700), (100, 64)):
        a = signed_codes(m, k, pa, seed=50 + m + pa)
        w = signed_codes(n, k, pw, seed=60 + pw + n)
        A = P.pack(_dev(a), pa, digits=True)
        W = P.pack(_dev(w), pw, tiled=tiled)
        cfg = _gemv_cfg(m, n, k, pw, pa, warps)
        ref = O.gemm_signed(a, w)
        assert np.array_equal(P.gemm(W, A, config=cfg).cpu().numpy().astype(np.int64), ref)
        got = P.gemm(W, A, out_kind="bipolar", layout="col", config=cfg).cpu().numpy().astype(np.int64)
        assert np.array_equal(got.T, O.gemm_bipolar(a, pa, w, pw))
        ws = log_uniform_scales(n, -10, -6, seed=3)
        as_ = log_uniform_scales(m, -6, -2, seed=4)
        got = P.gemm(W, A, out_kind="f16", w_scale=_dev(ws), a_scale=_dev(as_), config=cfg).cpu().numpy()
        r = O.scale_fp64(ref, ws, as_)
        assert (np.abs(got.astype(np.float64) - r) <= 1e-3 * np.abs(r) + 2.0 ** -24).all()


def test_gemv_without_digit_view():
    """Activations packed without the digit view: the GEMV reads the workspace expansion."""
    m, n, k = 1, 256, 4096
    a = signed_codes(m, k, 4, seed=1)
    w = signed_codes(n, k, 3, seed=2)
    A = P.pack(_dev(a), 4)
    W = P.pack(_dev(w), 3, tiled=True)
    got = P.gemm(W, A, config=_gemv_cfg(m, n, k, 3, 4)).cpu().numpy().astype(np.int64)
    assert np.array_equal(got, O.gemm_signed(a, w))


@pytest.mark.parametrize("n,k", LLAMA7B)
@pytest.mark.parametrize("pw,pa", [(1, 2), (2, 2), (3, 4), (4, 4)])
def test_gemv_llama7b_full(n, k, pw, pa):
    """BASELINE configs[1] at M = 1 through the GEMV, every element vs the C oracle."""
    a = signed_codes(1, k, pa, seed=config_seed(1, pw, pa, salt=3))
    w = signed_codes(n, k, pw, seed=config_seed(1, pw, pa, salt=3) + 1)
    A, W = _pack_both(a, pa, w, pw)
    cfg = P.select_config(1, n, k, pw, pa)
    assert cfg["kernel"] == 3  # the selector's M = 1 choice, in its launch configuration
    got = P.gemm(W, A, config=cfg).cpu().numpy().astype(np.int64)
    assert np.array_equal(got, c_gemm_i64(a, w))


# ----------------------------------------------------------------------------- configs[3], configs[4] at full size

@pytest.mark.parametrize("n,k", [(8192, 8192), (28672, 8192)])
def test_llama70b_full_and_tp_slices(n, k):
    """BASELINE configs[3] (Llama-3-70B linears, M = 4096, W2A4) at full size in the selector's launch
    configuration: EVERY output element vs the oracle (gemm_signed_blas, exact), and the N-split
    tensor-parallel slices (P = 8, column layout, as each rank computes them) concatenate to the
    single-GPU result bit for bit."""
    m, pw, pa = 4096, 2, 4
    a = signed_codes(m, k, pa, seed=config_seed(3, pw, pa))
    w = signed_codes(n, k, pw, seed=config_seed(3, pw, pa) + 1)
    A, W = _pack_both(a, pa, w, pw)
    full = P.gemm(W, A)
    assert np.array_equal(full.cpu().numpy().astype(np.int64), O.gemm_signed_blas(a, w))
    p = 8
    rows = n // p
    for r in range(p):
        Wr = P.pack(_dev(w[r * rows:(r + 1) * rows]), pw, tiled=True)
        yt = P.gemm(Wr, A, layout="col")  # [rows, M] = the rank's block of Y^T
        assert torch.equal(yt.t(), full[:, r * rows:(r + 1) * rows])


@pytest.mark.parametrize("pw", range(1, 9))
def test_sweep_4096_cube_full(pw):
    """BASELINE configs[4]: 4096^3 for every (p_w, p_a) in 1..8 x 1..8 with the selector's config,
    EVERY output element vs the oracle (gemm_signed_blas, exact)."""
    n = m = k = 4096
    w = signed_codes(n, k, pw, seed=config_seed(4, pw, 0))
    W = P.pack(_dev(w), pw, tiled=True)
    for pa in range(1, 9):
        a = signed_codes(m, k, pa, seed=config_seed(4, pw, pa))
        A = P.pack(_dev(a), pa, digits=True)
        got = P.gemm(W, A).cpu().numpy()
        assert np.array_equal(got.astype(np.int64), O.gemm_signed_blas(a, w)), pa


# ----------------------------------------------------------------------------- mma.sync skinny GEMM (M <= 16)

def _skinny_cfg(m, n, k, wb, ab, bn=16, warps=8):
    return dict(P.select_config(m, n, k, wb, ab), kernel=4, bm=16, bn=bn, bk=256, split_k=warps, stages=1,
                cta_pair=0, cluster_n=1)


@pytest.mark.parametrize("m,bn", [(1, 8), (5, 8), (8, 8), (9, 16), (16, 16), (16, 8), (21, 16)])
@pytest.mark.parametrize("pw,pa", [(1, 1), (1, 2), (2, 2), (3, 4), (4, 4), (6, 5), (8, 8)])
@pytest.mark.parametrize("warps", [4, 8, 16])
def test_skinny_matches_oracle(m, bn, pw, pa, warps):
    """APT_KERNEL_SKINNY: int32 signed / bipolar bit-exact and fp16 within 1e-3 on ragged shapes
    (N not a multiple of 16, K not a multiple of 256, fewer iterations than warps, M > bn -> 2 tiles),
    tile-major and canonical weights."""
    for n, k, tiled in ((333, 700, True), (100, 64, False), (40, 1300, True)):
        a = signed_codes(m, k, pa, seed=70 + m + pa)
        w = signed_codes(n, k, pw, seed=80 + pw + n)
        A = P.pack(_dev(a), pa, digits=True)
        W = P.pack(_dev(w), pw, tiled=tiled)
        cfg = _skinny_cfg(m, n, k, pw, pa, bn, warps)
        ref = O.gemm_signed(a, w)
        assert np.array_equal(P.gemm(W, A, config=cfg).cpu().numpy().astype(np.int64), ref)
        got = P.gemm(W, A, out_kind="bipolar", layout="col", config=cfg).cpu().numpy().astype(np.int64)
        assert np.array_equal(got.T, O.gemm_bipolar(a, pa, w, pw))
        ws = log_uniform_scales(n, -10, -6, seed=5)
        as_ = log_uniform_scales(m, -6, -2, seed=6)
        got = P.gemm(W, A, out_kind="f16", w_scale=_dev(ws), a_scale=_dev(as_), config=cfg).cpu().numpy()
        r = O.scale_fp64(ref, ws, as_)
        assert (np.abs(got.astype(np.float64) - r) <= 1e-3 * np.abs(r) + 2.0 ** -24).all()


@pytest.mark.parametrize("n,k", LLAMA7B)
@pytest.mark.parametrize("m", [8, 16])
@pytest.mark.parametrize("pw,pa", [(1, 2), (4, 4)])
def test_skinny_llama7b_full(n, k, m, pw, pa):
    a = signed_codes(m, k, pa, seed=config_seed(1, pw, pa, salt=5))
    w = signed_codes(n, k, pw, seed=config_seed(1, pw, pa, salt=5) + 1)
    A, W = _pack_both(a, pa, w, pw)
    got = P.gemm(W, A, config=_skinny_cfg(m, n, k, pw, pa, bn=8 if m <= 8 else 16)).cpu().numpy().astype(np.int64)
    assert np.array_equal(got, c_gemm_i64(a, w))


# ----------------------------------------------------------------------------- zero-point epilogue (NEXT-2)

@pytest.mark.parametrize("m,n,k", [(1, 300, 1000), (5, 300, 1000), (16, 200, 4096), (300, 256, 1000)])
@pytest.mark.parametrize("zeros", ["a", "w", "both"])
def test_zero_point_epilogue(m, n, k, zeros):
    """fp16 output with zero points (apt_scales.w_zero / a_zero: int32 Y of every kernel family the
    selector reaches — GEMV, skinny, tcgen05 decode and prefill tiles — then the zero-point pass) vs
    the fp64 dequantize-then-multiply
    oracle.  Bound: fp32 evaluation of four terms + one fp16 rounding, relative to the sum of the
    terms' magnitudes (cancellation-safe): 1e-3 * (|t1| + |t2| + |t3| + |t4|) + 2^-24."""
    pa, pw = 4, 3
    a = signed_codes(m, k, pa, seed=90 + m)
    w = signed_codes(n, k, pw, seed=91 + n)
    rng = np.random.default_rng(m + n)
    ws = log_uniform_scales(n, -10, -6, seed=7)
    as_ = log_uniform_scales(m, -6, -2, seed=8)
    wz = (rng.uniform(-1, 1, n) * 2.0 ** -8).astype(np.float32) if zeros in ("w", "both") else None
    az = rng.uniform(-1, 1, m).astype(np.float32) * 2.0 ** -3 if zeros in ("a", "both") else None
    az = az.astype(np.float32) if az is not None else None
    A, W = _pack_both(a, pa, w, pw)
    got = P.gemm(W, A, out_kind="f16", w_scale=_dev(ws), a_scale=_dev(as_),
                 w_zero=_dev(wz) if wz is not None else None, a_zero=_dev(az) if az is not None else None)
    got = got.cpu().numpy().astype(np.float64)
    ref = O.dequant_gemm_fp64(a, w, ws, as_, wz, az)
    y = O.gemm_signed(a, w).astype(np.float64)
    ra, rw = a.astype(np.float64).sum(1), w.astype(np.float64).sum(1)
    az0 = np.zeros(m) if az is None else az.astype(np.float64)
    wz0 = np.zeros(n) if wz is None else wz.astype(np.float64)
    mag = (np.abs(y * ws[None, :] * as_[:, None]) + np.abs(rw[None, :] * ws[None, :] * az0[:, None]) +
           np.abs(ra[:, None] * as_[:, None] * wz0[None, :]) + np.abs(k * az0[:, None] * wz0[None, :]))
    assert (np.abs(got - ref) <= 1e-3 * mag + 2.0 ** -24).all()


# ----------------------------------------------------------------------------- register-fed decode GEMM (M <= 16)

def _dec_cfg(m, n, k, wb, ab, split=1, warps=4):
    return dict(P.select_config(m, n, k, wb, ab), kernel=5, bm=32, bn=8 if m <= 8 else 16, bk=256,
                stages=warps, split_k=split, cta_pair=0, cluster_n=1)


@pytest.mark.parametrize("m", [1, 3, 8, 9, 16])
@pytest.mark.parametrize("pw,pa", [(1, 1), (1, 2), (2, 2), (2, 8), (3, 4), (4, 4), (5, 3), (8, 8)])
@pytest.mark.parametrize("split,warps", [(1, 4), (1, 8), (2, 4), (3, 8), (16, 4)])
def test_dec_matches_oracle(m, pw, pa, split, warps):
    """APT_KERNEL_DEC: int32 signed / bipolar bit-exact and fp16 within 1e-3 on ragged shapes (N not a
    multiple of 8, 32 or 128; K not a multiple of 256; more K splits and warps than 256-element blocks),
    tile-major and canonical weights, row and column layouts; the split-K tickets are left zero."""
    for n, k, tiled in ((333, 700, True), (100, 64, False), (41, 1300, True), (256, 4096, False), (300, 4096, True)):
        a = signed_codes(m, k, pa, seed=170 + m + pa)
        w = signed_codes(n, k, pw, seed=180 + pw + n)
        A = P.pack(_dev(a), pa, digits=True)
        W = P.pack(_dev(w), pw, tiled=tiled)
        cfg = _dec_cfg(m, n, k, pw, pa, split, warps)
        ref = O.gemm_signed(a, w)
        assert np.array_equal(P.gemm(W, A, config=cfg).cpu().numpy().astype(np.int64), ref)
        got = P.gemm(W, A, out_kind="bipolar", layout="col", config=cfg).cpu().numpy().astype(np.int64)
        assert np.array_equal(got.T, O.gemm_bipolar(a, pa, w, pw))
        ws = log_uniform_scales(n, -10, -6, seed=15)
        as_ = log_uniform_scales(m, -6, -2, seed=16)
        got = P.gemm(W, A, out_kind="f16", w_scale=_dev(ws), a_scale=_dev(as_), config=cfg).cpu().numpy()
        r = O.scale_fp64(ref, ws, as_)
        assert (np.abs(got.astype(np.float64) - r) <= 1e-3 * np.abs(r) + 2.0 ** -24).all()
    if split > 1:
        ws_t = P.default_workspace(DEV, 0)
        torch.cuda.synchronize()
        # the split-K tickets (include/apt.h: the first APT_WS_TICKET_BYTES of the workspace) are left zero
        assert int(ws_t[:16384].count_nonzero().item()) == 0


def test_dec_without_digit_view_and_extremes():
    """The DEC kernel reading the workspace token expansion (no digit view), and all-extreme codes at
    the largest K its 2^32 unsigned-sum bound allows for 2-bit weights x 8-bit activations."""
    m, n, k = 5, 200, 4096
    a = signed_codes(m, k, 4, seed=1)
    w = signed_codes(n, k, 2, seed=2)
    A = P.pack(_dev(a), 4)
    W = P.pack(_dev(w), 2, tiled=True)
    got = P.gemm(W, A, config=_dec_cfg(m, n, k, 2, 4, 4)).cpu().numpy().astype(np.int64)
    assert np.array_equal(got, O.gemm_signed(a, w))
    k = 66048  # Kpad * 255 * 255 < 2^32
    for av, wv in ((-128, -2), (127, 1), (-128, 1)):
        a = np.full((16, k), av, dtype=np.int8)
        w = np.full((40, k), wv, dtype=np.int8)
        A = P.pack(_dev(a), 8, digits=True)
        W = P.pack(_dev(w), 2, tiled=True)
        got = P.gemm(W, A, config=_dec_cfg(16, 40, k, 2, 8, 17)).cpu().numpy().astype(np.int64)
        assert np.array_equal(got, np.full((16, 40), k * av * wv, dtype=np.int64))


@pytest.mark.parametrize("n,k", LLAMA7B)
@pytest.mark.parametrize("m", [1, 8, 16])
@pytest.mark.parametrize("pw,pa", [(1, 2), (2, 2), (3, 4), (4, 4)])
@pytest.mark.parametrize("split,warps", [(1, 8), (2, 4)])
def test_dec_llama7b_full(n, k, m, pw, pa, split, warps):
    """BASELINE configs[1] at full size through APT_KERNEL_DEC, fp16 + a_scale (the bench's call):
    every element within 1e-3 of the fp64-scaled C oracle."""
    a = signed_codes(m, k, pa, seed=config_seed(1, pw, pa, salt=11))
    w = signed_codes(n, k, pw, seed=config_seed(1, pw, pa, salt=11) + 1)
    ws = log_uniform_scales(n, -10, -6, seed=n + pw + 1)
    as_ = log_uniform_scales(m, -6, -2, seed=m + pa + 1)
    A = P.pack(_dev(a), pa, digits=True)
    W = P.pack(_dev(w), pw, tiled=True)
    cfg = _dec_cfg(m, n, k, pw, pa, split, warps)
    got = P.gemm(W, A, out_kind="f16", w_scale=_dev(ws), a_scale=_dev(as_), config=cfg).cpu().numpy()
    ref = O.scale_fp64(c_gemm_i64(a, w), ws, as_)
    assert (np.abs(got.astype(np.float64) - ref) <= 1e-3 * np.abs(ref) + 2.0 ** -24).all()


# ----------------------------------------------------------------------------- kind::mxf4 path (p_w, p_a <= 3)

def _mx_cfg(m, n, k, wb, ab, bn=256):
    return dict(P.select_config(m, n, k, wb, ab), kernel=2, bm=128, bn=bn, bk=128, stages=_tc_stages(wb, bn), split_k=1,
                cta_pair=0, cluster_n=1, mma_kind=1)


@pytest.mark.parametrize("k", [4096, 28672])
def test_mxf4_exactness_torture(k):
    """the f32 accumulation of the e2m1 products must be exact.  All-extreme
    products (|x y| = 16 and 9) over K = 28,672 (|sum| = 458,752 < 2^24), a large running sum followed by
    +-1 terms that an accumulator truncating low bits would drop, and alternating signs within every
    64-element MMA K block — bit-exact against the int64 oracle."""
    m, n = 256, 256
    rng = np.random.default_rng(k)
    a = np.empty((m, k), dtype=np.int8)
    w = np.empty((n, k), dtype=np.int8)
    a[:64], w[:64] = -4, -4                                   # +16 everywhere
    a[64:128], w[64:128] = 3, 3                               # +9 / cross terms -12
    half = k // 2
    a[128:192, :half], a[128:192, half:] = -4, rng.choice([-1, 1], size=(64, k - half))
    w[128:192, :half], w[128:192, half:] = -4, 1             # big sum, then +-1 tail
    a[192:] = np.where(np.arange(k) % 2 == 0, -4, 1)[None, :]  # alternating 16 / small within each block
    w[192:] = rng.integers(-4, 4, size=(n - 192, k))
    A = P.pack(_dev(a), 3)
    W = P.pack(_dev(w), 3, tiled=True)
    ref = c_gemm_i64(a, w)
    for bn in (128, 256):
        got = P.gemm(W, A, config=_mx_cfg(m, n, k, 3, 3, bn)).cpu().numpy().astype(np.int64)
        assert np.array_equal(got, ref), bn


@pytest.mark.parametrize("pw,pa", [(p, q) for p in (1, 2, 3) for q in (1, 2, 3)])
@pytest.mark.parametrize("bn,tiled", [(128, True), (256, True), (256, False)])
def test_mxf4_matches_oracle(pw, pa, bn, tiled):
    """kind::mxf4 on ragged shapes (M, N not multiples of the tile, K not a multiple of 256): int32 signed
    and bipolar bit-exact, fp16 within 1e-3, row and column layouts, tile-major and canonical weights."""
    for m, n, k in ((300, 333, 700), (17, 129, 256), (513, 200, 1500)):
        a = signed_codes(m, k, pa, seed=210 + pa + m)
        w = signed_codes(n, k, pw, seed=220 + pw + n)
        A = P.pack(_dev(a), pa, digits=True)
        W = P.pack(_dev(w), pw, tiled=tiled)
        cfg = _mx_cfg(m, n, k, pw, pa, bn)
        ref = O.gemm_signed(a, w)
        assert np.array_equal(P.gemm(W, A, config=cfg).cpu().numpy().astype(np.int64), ref)
        got = P.gemm(W, A, out_kind="bipolar", layout="col", config=cfg).cpu().numpy().astype(np.int64)
        assert np.array_equal(got.T, O.gemm_bipolar(a, pa, w, pw))
        ws = log_uniform_scales(n, -10, -6, seed=25)
        as_ = log_uniform_scales(m, -6, -2, seed=26)
        got = P.gemm(W, A, out_kind="f16", w_scale=_dev(ws), a_scale=_dev(as_), config=cfg).cpu().numpy()
        r = O.scale_fp64(ref, ws, as_)
        assert (np.abs(got.astype(np.float64) - r) <= 1e-3 * np.abs(r) + 2.0 ** -24).all()


@pytest.mark.parametrize("pw", [1, 2, 3])
def test_mxf4_sweep_4096_cube_full(pw):
    """BASELINE configs[4] at full size through kind::mxf4 for every (p_w, p_a) <= 3: EVERY output
    element vs the oracle (gemm_signed_blas, exact)."""
    n = m = k = 4096
    w = signed_codes(n, k, pw, seed=config_seed(4, pw, 0, salt=9))
    W = P.pack(_dev(w), pw, tiled=True)
    for pa in (1, 2, 3):
        a = signed_codes(m, k, pa, seed=config_seed(4, pw, pa, salt=9))
        A = P.pack(_dev(a), pa)
        got = P.gemm(W, A, config=_mx_cfg(m, n, k, pw, pa)).cpu().numpy()
        assert np.array_equal(got.astype(np.int64), O.gemm_signed_blas(a, w)), pa


@pytest.mark.parametrize("chunks", [1, 4])
def test_tp_gemm_single_rank_chunked(chunks):
    """tp.tp_gemm on one rank: Y^T [N, M] (one chunk) or chunk-major [C, N, M/C] written in place by the
    column-layout GEMM, fp16 within 1e-3 of the oracle, from pre-packed activation chunks."""
    from paper_2508_19087_b200 import tp
    m, n, k, pw, pa = 512, 1024, 2048, 2, 4
    a = signed_codes(m, k, pa, seed=301)
    w = signed_codes(n, k, pw, seed=302)
    ws = log_uniform_scales(n, -10, -6, seed=303)
    as_ = log_uniform_scales(m, -6, -2, seed=304)
    W = P.pack(_dev(w), pw, tiled=True)
    mc = m // chunks
    A = [P.pack(_dev(a[c * mc:(c + 1) * mc]), pa, digits=True) for c in range(chunks)]
    yt = tp.tp_gemm(W, A if chunks > 1 else A[0], n, out_kind="f16", w_scale_local=_dev(ws), a_scale=_dev(as_),
                    m_chunks=chunks).cpu().numpy().astype(np.float64)
    ref = O.scale_fp64(O.gemm_signed(a, w), ws, as_).T
    if chunks > 1:
        ref = np.stack([ref[:, c * mc:(c + 1) * mc] for c in range(chunks)])
    assert yt.shape == ref.shape
    assert (np.abs(yt - ref) <= 1e-3 * np.abs(ref) + 2.0 ** -24).all()


# ----------------------------------------------------------------------------- ablation: the paper's Basic design (NEXT-4)

@pytest.mark.parametrize("m,n,k,pw,pa", [(16, 256, 700, 2, 2), (5, 130, 300, 3, 4), (300, 200, 1000, 4, 4),
                                         (16, 64, 256, 8, 8)])
def test_ablation_basic_plane_pairs(m, n, k, pw, pa):
    """The Basic design (one 1-bit x 1-bit GEMM per plane pair, recovered in global memory by
    apt_recombine_plane_products) gives the bipolar product bit for bit — the same result as the
    fused product path and the oracle's recombination (I1)."""
    from paper_2508_19087_b200 import ablation
    a = signed_codes(m, k, pa, seed=401 + m)
    w = signed_codes(n, k, pw, seed=402 + n)
    pp = ablation.PlanePairs(_dev(a), pa, _dev(w), pw)
    got = pp.basic().cpu().numpy().astype(np.int64)
    ref = O.recombine(O.plane_products(a, pa, w, pw))
    assert np.array_equal(got, O.gemm_bipolar(a, pa, w, pw))
    assert np.array_equal(got, ref)
    A, W = _pack_both(a, pa, w, pw)
    assert np.array_equal(P.gemm(W, A, out_kind="bipolar").cpu().numpy().astype(np.int64), got)


# ----------------------------------------------------------------------------- persistent tcgen05 tile (APT_KERNEL_PF)

def _pf_cfg(m, n, k, wb, ab, mx=0, bn=128):
    return dict(P.select_config(m, n, k, wb, ab), kernel=6, bm=128, bn=bn, bk=128, stages={128: 6, 192: 4, 256: 3}[bn],
                split_k=1, cta_pair=0, cluster_n=1, mma_kind=mx)


@pytest.mark.parametrize("pw,pa,mx,bn", [(1, 1, 0, 128), (2, 8, 0, 128), (4, 4, 0, 128), (5, 3, 0, 128), (8, 8, 0, 128),
                                         (3, 3, 1, 128), (1, 2, 1, 128), (2, 3, 1, 128),
                                         (1, 1, 0, 192), (2, 8, 0, 192), (4, 4, 0, 192), (5, 3, 0, 192), (8, 8, 0, 192),
                                         (1, 1, 0, 256), (2, 8, 0, 256), (4, 4, 0, 256), (5, 3, 0, 256), (8, 8, 0, 256)])
@pytest.mark.parametrize("tiled", [True, False])
def test_pf_matches_oracle(pw, pa, mx, bn, tiled):
    """APT_KERNEL_PF (i8 and mxf4): int32 signed / bipolar bit-exact and fp16 within 1e-3 on ragged shapes
    (M, N not multiples of 128, K not a multiple of 256, more tiles than SMs and fewer), row and column
    layouts, tile-major and canonical weights, with and without the activation digit view."""
    for m, n, k in ((300, 333, 700), (129, 130, 1300), (2048, 1100, 512), (70, 40, 256)):
        a = signed_codes(m, k, pa, seed=510 + pa + m)
        w = signed_codes(n, k, pw, seed=520 + pw + n)
        A = P.pack(_dev(a), pa, digits=(m % 2 == 0))
        W = P.pack(_dev(w), pw, tiled=tiled)
        cfg = _pf_cfg(m, n, k, pw, pa, mx, bn)
        ref = O.gemm_signed(a, w)
        assert np.array_equal(P.gemm(W, A, config=cfg).cpu().numpy().astype(np.int64), ref)
        got = P.gemm(W, A, out_kind="bipolar", layout="col", config=cfg).cpu().numpy().astype(np.int64)
        assert np.array_equal(got.T, ref * 4 + 2 * a.astype(np.int64).sum(1)[:, None] + 2 * w.astype(np.int64).sum(1)[None, :] + k)
        ws = log_uniform_scales(n, -10, -6, seed=35)
        as_ = log_uniform_scales(m, -6, -2, seed=36)
        r = O.scale_fp64(ref, ws, as_)
        for lay in ("row", "col"):
            got = P.gemm(W, A, out_kind="f16", layout=lay, w_scale=_dev(ws), a_scale=_dev(as_), config=cfg).cpu().numpy()
            got = (got if lay == "row" else got.T).astype(np.float64)
            assert (np.abs(got - r) <= 1e-3 * np.abs(r) + 2.0 ** -24).all()


@pytest.mark.parametrize("n,k", LLAMA7B)
@pytest.mark.parametrize("pw,pa", [(2, 8), (4, 4)])
@pytest.mark.parametrize("bn", [128, 192, 256])
def test_pf_llama7b_prefill_full(n, k, pw, pa, bn):
    """BASELINE configs[2] at full size through APT_KERNEL_PF: EVERY output element vs the oracle."""
    m = 2048
    a = signed_codes(m, k, pa, seed=config_seed(2, pw, pa, salt=13))
    w = signed_codes(n, k, pw, seed=config_seed(2, pw, pa, salt=13) + 1)
    A, W = _pack_both(a, pa, w, pw)
    got = P.gemm(W, A, config=_pf_cfg(m, n, k, pw, pa, bn=bn)).cpu().numpy().astype(np.int64)
    assert np.array_equal(got, O.gemm_signed_blas(a, w))
