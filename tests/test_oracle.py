"""Pins for the CPU oracle (oracle/), run without a GPU.

Each test pins an oracle function to something other than itself: the
paper's closed forms, SPEC worked examples
(tests/golden/), exhaustive enumeration, brute force with Python ints, and
library special cases (numpy int64 matmul).  See DESIGN.md "Oracle pins".
"""
import json
import os
from fractions import Fraction
from itertools import product

import numpy as np
import pytest

from oracle import apt_oracle as O
from oracle import c_gemm_i64
from synth import signed_codes


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


def _bits_lsb(s_msb_first):
    return [int(c) for c in reversed(s_msb_first)]


# ---------------------------------------------------------------- §3.1 format

def test_bipolar_value_spec_examples(golden_dir):
    g = _load(golden_dir, "spec_examples.json")
    for ex in g["bipolar_value"]:
        assert O.bipolar_value(_bits_lsb(ex["bits_msb_first"])) == ex["value"], ex["cite"]


def test_signed_bipolar_spec_examples(golden_dir):
    g = _load(golden_dir, "spec_examples.json")
    for ex in g["signed_to_bipolar"]:
        assert O.signed_to_bipolar_bits(ex["signed"], ex["n"]) == _bits_lsb(ex["bits_msb_first"]), ex["cite"]
        assert O.signed_to_bipolar(ex["signed"], ex["n"]) == ex["value"], ex["cite"]
    for ex in g["bipolar_to_signed"]:
        assert O.bipolar_to_signed(ex["value"], ex["n"]) == ex["signed"], ex["cite"]


@pytest.mark.parametrize("n", range(1, 9))
def test_exhaustive_affine_law_and_bijection(n):
    """P:203 x' = 2x+1 over every n-bit pattern (510 patterns over n=1..8);
    the bipolar pattern read as unsigned equals x + 2^(n-1) (offset binary);
    the map is a bijection onto the odd integers in +-(2^n-1)."""
    images = set()
    for pattern in range(1 << n):
        x = pattern - (1 << n) if pattern >= (1 << (n - 1)) else pattern  # two's complement value
        bits = O.signed_to_bipolar_bits(x, n)
        u = sum(b << i for i, b in enumerate(bits))
        assert u == x + (1 << (n - 1))
        v = O.signed_to_bipolar(x, n)
        assert v == 2 * x + 1
        assert O.bipolar_to_signed(v, n) == x
        images.add(v)
    assert images == set(range(-(1 << n) + 1, 1 << n, 2))


def test_one_bit_convention():
    """Reading Q4 / S:156-160: n=1 signed {-1,0} -> bipolar {-1,+1}."""
    assert O.signed_to_bipolar(-1, 1) == -1
    assert O.signed_to_bipolar(0, 1) == 1
    assert O.signed_range(1) == (-1, 0)


def test_offset_bits_rejects_out_of_range():
    with pytest.raises(ValueError):
        O.offset_bits_matrix(np.array([[2]]), 2)
    with pytest.raises(ValueError):
        O.offset_bits_matrix(np.array([[-3]]), 2)


# ---------------------------------------------------------------- §4.1 packing

def test_pack_layout_examples(golden_dir):
    g = _load(golden_dir, "spec_examples.json")["pack_1x1"]
    x = O.bipolar_to_signed(g["bipolar_value"], g["n"])
    planes, rs = O.pack_planes(np.array([[x]]), g["n"])
    assert planes.shape == (2, 1, 256 // 32)
    assert (planes[0, 0, 0] & 1) == g["plane0_word0_bit0"]
    assert (planes[1, 0, 0] & 1) == g["plane1_word0_bit0"]
    assert rs.tolist() == [x]
    # 1x33 row: element 32 lands in word 1 bit 0 (S:187 translated to 32-bit words)
    row = np.zeros((1, 33), dtype=np.int64)
    row[0, 32] = 1  # n=2: code 1 -> u=3 sets plane 0; code 0 -> u=2 leaves plane 0 clear
    planes, _ = O.pack_planes(row, 2)
    assert (planes[0, 0, 1] & 1) == 1 and (planes[0, 0, 0]) == 0
    # code 0 everywhere else (u = 2): plane 1 carries every element incl. the pad
    assert planes[1, 0, 0] == 0xFFFFFFFF and planes[1, 0, 7] == 0xFFFFFFFF


def test_unpack_all_zero_bits(golden_dir):
    g = _load(golden_dir, "spec_examples.json")["unpack_all_zero_bits"]
    planes = np.zeros((g["n"], g["rows"], 8), dtype=np.uint32)
    codes = O.unpack_planes(planes, g["cols"], g["n"])
    bip = 2 * codes + 1
    assert (bip == g["bipolar_value"]).all()


def test_pack_roundtrip_footprint_and_padding():
    rng = np.random.default_rng(7)
    for t in range(60):
        rows = int(rng.integers(1, 40))
        k = int(rng.integers(1, 600))
        n = int(rng.integers(1, 9))
        codes = signed_codes(rows, k, n, seed=1000 + t)
        planes, rs = O.pack_planes(codes, n)
        kp = O.kpad(k)
        assert kp % 256 == 0 and kp >= k and kp - k < 256
        assert planes.shape == (n, rows, kp // 32)        # footprint n*rows*Kpad/32 words
        assert planes.dtype == np.uint32
        full = O.unpack_planes(planes, kp, n)
        assert (full[:, :k] == codes).all()               # unpack . pack = id
        assert (full[:, k:] == 0).all()                   # pads hold signed code 0 (reading Q6)
        assert (rs == codes.astype(np.int64).sum(axis=1)).all()


# ---------------------------------------------------------------- §3.2 reconstitution

def test_xor_dot_examples(golden_dir):
    g = _load(golden_dir, "spec_examples.json")["xor_dot"]
    for ex in g:
        k = ex["k"]
        words = (k + 31) // 32
        def bits(v):
            if v == "ones":
                return [1] * k
            if v == "zeros":
                return [0] * k
            return [(v >> c) & 1 for c in range(k)]
        def pack(bl):
            w = np.zeros((1, 1, max(words, 1)), dtype=np.uint32)
            for c, b in enumerate(bl):
                w[0, 0, c // 32] |= np.uint32(b << (c % 32))
            return w
        got = O.plane_products_xor(pack(bits(ex["a"])), pack(bits(ex["b"])), k)
        assert int(got[0, 0, 0, 0]) == ex["dot"], ex["cite"]


def test_recover_tile_example(golden_dir):
    g = _load(golden_dir, "spec_examples.json")["recover_tile"]
    yij = np.zeros((g["p"], g["q"], 1, 1), dtype=np.int64)
    for i, j, v in g["cells_ij"]:
        yij[i, j, 0, 0] = v
    assert int(O.recombine(yij)[0, 0]) == g["value"], g["cite"]


def test_gemm_all_ones_bits(golden_dir):
    g = _load(golden_dir, "spec_examples.json")["gemm_all_ones_bits"]
    # all-ones bit in a 1-bit bipolar operand = bipolar +1 = signed code 0
    a = np.zeros((1, g["k"]), dtype=np.int64)
    w = np.zeros((1, g["k"]), dtype=np.int64)
    assert int(O.gemm_bipolar(a, 1, w, 1)[0, 0]) == g["value"], g["cite"]
    o = _load(golden_dir, "spec_examples.json")["oracle_1x1"]
    assert o["x_bipolar"] * o["w_bipolar"] == o["value"]
    a1 = np.array([[O.bipolar_to_signed(o["x_bipolar"], 2)]])
    w1 = np.array([[O.bipolar_to_signed(o["w_bipolar"], 2)]])
    assert int(O.gemm_bipolar(a1, 2, w1, 2)[0, 0]) == o["value"], o["cite"]


def test_worked_example_s300(golden_dir):
    g = _load(golden_dir, "worked_example_s300.json")
    n = g["bits"]
    w_sig = np.array([[O.bipolar_to_signed(v, n) for v in r] for r in g["W_bipolar"]])
    x_km = np.array([[O.bipolar_to_signed(v, n) for v in r] for r in g["X_bipolar_KxM"]])
    assert w_sig.tolist() == g["W_signed"] and x_km.tolist() == g["X_signed_KxM"]
    a = x_km.T  # our A is [M, K] (reading Q2)
    wp = O.plane_matrices(w_sig, n)
    xp = O.plane_matrices(a, n)
    for i in range(n):
        assert wp[i].tolist() == g["W_planes_pm1"][str(i)]
        assert xp[i].T.tolist() == g["X_planes_pm1"][str(i)]
    yij = O.plane_products(a, n, w_sig, n)  # [act plane][weight plane][m][n]
    for i in range(n):
        for j in range(n):
            assert yij[j, i].T.tolist() == g["Y_planes_Wi_Xj"][f"{i},{j}"]
    assert O.recombine(yij).T.tolist() == g["Y_bipolar"]
    assert O.gemm_signed(a, w_sig).T.tolist() == g["Y_signed"]


def _random_instance(rng, seed, maxdim=40):
    m = int(rng.integers(1, maxdim))
    n = int(rng.integers(1, maxdim))
    k = int(rng.integers(1, 300))
    pa = int(rng.integers(1, 9))
    pw = int(rng.integers(1, 9))
    a = signed_codes(m, k, pa, seed=seed)
    w = signed_codes(n, k, pw, seed=seed + 1)
    return a, pa, w, pw, k


def test_identities_random():
    """I1 recomposition, I2 bipolar/signed rank-1 link, I3 offset
    (AND) form, and the XOR route == the +-1 route, on random instances."""
    rng = np.random.default_rng(11)
    for t in range(60):
        a, pa, w, pw, k = _random_instance(rng, 5000 + 2 * t)
        y = O.gemm_signed(a, w)
        yb = O.gemm_bipolar(a, pa, w, pw)
        # I1: direct bipolar product over element values 2x+1
        ab = 2 * a.astype(np.int64) + 1
        wb = 2 * w.astype(np.int64) + 1
        assert (yb == ab @ wb.T).all()
        # I2: Y' = 4Y + 2 RA[m] + 2 RW[n] + K
        ra = a.astype(np.int64).sum(1)
        rw = w.astype(np.int64).sum(1)
        assert (yb == 4 * y + 2 * ra[:, None] + 2 * rw[None, :] + k).all()
        # I3: Y = U - 2^(pw-1) UA - 2^(pa-1) UW + K 2^(pa+pw-2), U = sum u_a u_w
        ua = O.offset_bits_matrix(a, pa)
        uw = O.offset_bits_matrix(w, pw)
        u = ua @ uw.T
        assert (y == u - (1 << (pw - 1)) * ua.sum(1)[:, None] - (1 << (pa - 1)) * uw.sum(1)[None, :]
                + k * (1 << (pa + pw - 2))).all()
        # XOR route on the packed words == +-1 plane products
        if t < 15:
            pa_planes, _ = O.pack_planes(a, pa)
            pw_planes, _ = O.pack_planes(w, pw)
            assert (O.plane_products_xor(pa_planes, pw_planes, k) == O.plane_products(a, pa, w, pw)).all()


@pytest.mark.parametrize("pa,pw", [(p, q) for p in range(1, 9) for q in range(1, 9)])
def test_bruteforce_k1_all_precisions(pa, pw):
    """K = 1, every activation code x every weight code: Y = a*w and Y' = (2a+1)(2w+1)."""
    lo_a, hi_a = O.signed_range(pa)
    lo_w, hi_w = O.signed_range(pw)
    a = np.arange(lo_a, hi_a + 1).reshape(-1, 1)
    w = np.arange(lo_w, hi_w + 1).reshape(-1, 1)
    y = O.gemm_signed(a, w)
    yb = O.gemm_bipolar(a, pa, w, pw)
    for i, av in enumerate(range(lo_a, hi_a + 1)):
        for j, wv in enumerate(range(lo_w, hi_w + 1)):
            assert y[i, j] == av * wv
            assert yb[i, j] == (2 * av + 1) * (2 * wv + 1)


@pytest.mark.parametrize("pa,pw,k", [(3, 3, 2), (2, 2, 3), (4, 1, 2), (1, 4, 3)])
def test_bruteforce_all_rows(pa, pw, k):
    """Every possible activation row x every possible weight row."""
    ra = list(product(range(*[O.signed_range(pa)[0], O.signed_range(pa)[1] + 1]), repeat=k))
    rw = list(product(range(*[O.signed_range(pw)[0], O.signed_range(pw)[1] + 1]), repeat=k))
    a = np.array(ra, dtype=np.int64)
    w = np.array(rw, dtype=np.int64)
    ref = np.array(O.gemm_python(ra, rw), dtype=np.int64)
    assert (O.gemm_signed(a, w) == ref).all()
    refb = np.array(O.gemm_python([[2 * x + 1 for x in r] for r in ra], [[2 * x + 1 for x in r] for r in rw]))
    assert (O.gemm_bipolar(a, pa, w, pw) == refb).all()


def test_closed_forms():
    for pa, pw in [(1, 1), (2, 3), (8, 8), (4, 2)]:
        k = 300
        lo_a, hi_a = O.signed_range(pa)
        lo_w, hi_w = O.signed_range(pw)
        for av, wv in [(lo_a, lo_w), (hi_a, lo_w), (hi_a, hi_w), (0, lo_w)]:
            a = np.full((3, k), av)
            w = np.full((5, k), wv)
            assert (O.gemm_signed(a, w) == k * av * wv).all()
            assert (O.gemm_bipolar(a, pa, w, pw) == k * (2 * av + 1) * (2 * wv + 1)).all()


def test_c_oracle_matches_library_and_bigint():
    rng = np.random.default_rng(3)
    for t in range(10):
        m, n, k = (int(v) for v in rng.integers(1, 70, size=3))
        a = signed_codes(m, k, 8, seed=77 + t)
        w = signed_codes(n, k, 8, seed=99 + t)
        got = c_gemm_i64(a, w)
        assert (got == a.astype(np.int64) @ w.astype(np.int64).T).all()
        if t < 3:
            assert got.tolist() == O.gemm_python(a.tolist(), w.tolist())


def test_blas_oracle_exact():
    """gemm_signed_blas (fp64 BLAS as the one step) equals the C int64 loop and the Python big-int
    loop bit for bit: random shapes and precisions, chunk boundaries, the all-minimum W8A8 edge at
    K = 33024 (|Y| = K 2^14, every partial sum an exact fp64 integer), and alternating signs."""
    rng = np.random.default_rng(11)
    for t in range(12):
        m, n, k = (int(v) for v in rng.integers(1, 90, size=3))
        pa, pw = (int(v) for v in rng.integers(1, 9, size=2))
        a = signed_codes(m, k, pa, seed=500 + t)
        w = signed_codes(n, k, pw, seed=600 + t)
        got = O.gemm_signed_blas(a, w, chunk=7)
        assert got.dtype == np.int64 and (got == c_gemm_i64(a, w)).all()
        if t < 2:
            assert got.tolist() == O.gemm_python(a.tolist(), w.tolist())
    k = 33024
    a = np.full((2, k), -128, dtype=np.int8)
    w = np.full((3, k), -128, dtype=np.int8)
    assert (O.gemm_signed_blas(a, w) == k * 2 ** 14).all()
    a[:, ::2] = 127
    assert (O.gemm_signed_blas(a, w) == c_gemm_i64(a, w)).all()


def test_scale_fp64_within_two_roundings():
    rng = np.random.default_rng(5)
    y = rng.integers(-(1 << 30), 1 << 30, size=(4, 6))
    ws = np.exp2(rng.uniform(-10, -6, 6)).astype(np.float32)
    a_s = np.exp2(rng.uniform(-6, -2, 4)).astype(np.float32)
    out = O.scale_fp64(y, ws, a_s)
    for m in range(4):
        for n in range(6):
            exact = O.scale_exact(y[m, n], ws[n], a_s[m])
            assert abs(Fraction(float(out[m, n])) - exact) <= abs(exact) * Fraction(2, 1 << 53)


def test_int32_bound():
    assert O.int32_bound_ok(33024, 8, 8)           # 33024 * 255^2 = 2147385600 < 2^31
    assert not O.int32_bound_ok(33025, 8, 8)       # Kpad = 33280 -> 2163832000 >= 2^31
    assert O.int32_bound_ok(28672, 8, 8)           # largest BASELINE K
    assert O.kpad(28672) == 28672 and O.kpad(1) == 256 and O.kpad(257) == 512


# ---------------------------------------------------------------- quantize (reading R-Q)
def test_quantize_worked_example():
    # n = 2: qmax = 1, s = max|x| = 1.0; 0.5 is a tie -> rint half-to-even -> 0; 0.75 -> 1
    codes, s = O.quantize_symmetric(np.array([[0.5, -1.0, 0.25, 0.75]], dtype=np.float16), 2)
    assert s.tolist() == [1.0]
    assert codes.tolist() == [[0, -1, 0, 1]]
    # n = 4: qmax = 7, s = fl32(3.5 / 7) = 0.5 exactly; x / s exact: 3.5 -> 7, -1.25 -> -2.5 -> -2, 0.75 -> 1.5 -> 2
    codes, s = O.quantize_symmetric(np.array([[3.5, -1.25, 0.75, 0.0]], dtype=np.float16), 4)
    assert s.tolist() == [0.5]
    assert codes.tolist() == [[7, -2, 2, 0]]


def test_quantize_zero_row_and_range():
    codes, s = O.quantize_symmetric(np.zeros((2, 5), dtype=np.float16), 3)
    assert s.tolist() == [0.0, 0.0] and not codes.any()
    with pytest.raises(ValueError):
        O.quantize_symmetric(np.ones((1, 4), dtype=np.float16), 1)


@pytest.mark.parametrize("n", [2, 3, 4, 5, 8])
def test_quantize_exact_rational_properties(n):
    """Pins against exact arithmetic (fractions), not the formula: s is the fp32 nearest to
    max|x| / qmax; every code is the integer nearest to the exact x / s (away from near-ties, where
    the fp32 quotient may legitimately decide), the row maximum maps to +-qmax, and the dequantised
    value is within s/2 of x (P:199-201 linear quantization with z = 0)."""
    rng = np.random.default_rng(100 + n)
    x = (rng.standard_normal((6, 97)) * rng.choice([1e-3, 1.0, 30.0], size=(6, 1))).astype(np.float16)
    x[2, :] = np.float16(0)
    x[2, 5] = np.float16(-2.0)
    codes, s = O.quantize_symmetric(x, n)
    qmax = (1 << (n - 1)) - 1
    for r in range(x.shape[0]):
        xr = [Fraction(float(v)) for v in x[r]]
        amax = max(abs(v) for v in xr)
        exact = amax / qmax
        sr = Fraction(float(s[r]))
        # fp32 round-to-nearest: relative error <= 2^-24
        assert abs(sr - exact) <= exact * Fraction(1, 1 << 24)
        if amax == 0:
            assert not codes[r].any()
            continue
        imax = max(range(len(xr)), key=lambda c: abs(xr[c]))
        assert abs(int(codes[r, imax])) == qmax
        for c, v in enumerate(xr):
            t = v / sr
            q = int(codes[r, c])
            assert -(qmax + 1) <= q <= qmax
            assert abs(v - sr * q) <= sr / 2 * (1 + Fraction(1, 1 << 20))
            frac = t - (t.numerator // t.denominator)
            if abs(frac - Fraction(1, 2)) > Fraction(1, 1 << 18):
                assert q == round(t)


def test_quantize_power_of_two_invariance():
    rng = np.random.default_rng(7)
    x = rng.standard_normal((3, 64)).astype(np.float16)
    c1, s1 = O.quantize_symmetric(x, 4)
    c2, s2 = O.quantize_symmetric((x.astype(np.float32) * 8).astype(np.float16), 4)
    assert np.array_equal(c1, c2) and np.array_equal(s2, s1 * 8)


def test_dequant_gemm_exact_brute_force():
    """dequant_gemm_fp64 vs exact rational brute force sum_k (s_a x + z_a)(s_w w + z_w) on tiny inputs
    (pins the zero-point definition of), and the zero-free case equals scale_fp64."""
    rng = np.random.default_rng(11)
    for _ in range(20):
        m, n, k = rng.integers(1, 5, size=3)
        a = signed_codes(m, k, 4, seed=int(rng.integers(1 << 30)))
        w = signed_codes(n, k, 3, seed=int(rng.integers(1 << 30)))
        ws, as_ = rng.uniform(0.01, 1, n).astype(np.float32), rng.uniform(0.01, 1, m).astype(np.float32)
        wz, az = rng.uniform(-1, 1, n).astype(np.float32), rng.uniform(-1, 1, m).astype(np.float32)
        got = O.dequant_gemm_fp64(a, w, ws, as_, wz, az)
        for i in range(m):
            for j in range(n):
                ex = sum((Fraction(float(as_[i])) * int(a[i, q]) + Fraction(float(az[i]))) *
                         (Fraction(float(ws[j])) * int(w[j, q]) + Fraction(float(wz[j]))) for q in range(k))
                assert abs(Fraction(got[i, j]) - ex) <= Fraction(1, 1 << 40) * (1 + abs(ex))
        assert np.allclose(O.dequant_gemm_fp64(a, w, ws, as_), O.scale_fp64(O.gemm_signed(a, w), ws, as_),
                           rtol=1e-14, atol=0)


def test_group_dequant_gemm_exact_brute_force():
    """group_dequant_gemm_fp64 vs exact rational brute force sum_k (s_a[g(k)] x)(s_w[g(k)] w) with
    g(k) = k // group on tiny inputs spanning several groups (group sizes 4 and 128), with and without
    activation group scales."""
    rng = np.random.default_rng(12)
    for it in range(16):
        group = 4 if it % 2 else 128
        m, n = (int(v) for v in rng.integers(1, 4, size=2))
        k = int(rng.integers(1, 3 * group + 2))
        G = -(-k // group)
        a = signed_codes(m, k, 4, seed=int(rng.integers(1 << 30)))
        w = signed_codes(n, k, 3, seed=int(rng.integers(1 << 30)))
        wg = rng.uniform(0.01, 1, (G, n)).astype(np.float32)
        ag = rng.uniform(0.01, 1, (G, m)).astype(np.float32) if it % 4 < 2 else None
        sa = rng.uniform(0.01, 1, m).astype(np.float32)
        got = O.group_dequant_gemm_fp64(a, w, wg, ag, None if ag is not None else sa, group=group)
        for i in range(m):
            for j in range(n):
                ex = Fraction(0)
                for q in range(k):
                    g = q // group
                    s_a = Fraction(float(ag[g, i])) if ag is not None else Fraction(float(sa[i]))
                    ex += s_a * int(a[i, q]) * Fraction(float(wg[g, j])) * int(w[j, q])
                assert abs(Fraction(got[i, j]) - ex) <= Fraction(1, 1 << 40) * (1 + abs(ex))


def test_group_dequant_gemm_reduces_to_per_channel():
    """Equal scales on every group reduce to the per-channel / per-token epilogue (scale_fp64 of the
    exact int64 product), and a single group (K <= 128) to dequant_gemm_fp64 with that group's scales."""
    rng = np.random.default_rng(13)
    a = signed_codes(5, 700, 4, seed=1)
    w = signed_codes(9, 700, 2, seed=2)
    ws, as_ = rng.uniform(0.01, 1, 9).astype(np.float32), rng.uniform(0.01, 1, 5).astype(np.float32)
    G = -(-700 // 128)
    got = O.group_dequant_gemm_fp64(a, w, np.tile(ws, (G, 1)), np.tile(as_, (G, 1)))
    assert np.allclose(got, O.scale_fp64(O.gemm_signed(a, w), ws, as_), rtol=1e-13, atol=0)
    a1, w1 = a[:, :100], w[:, :100]
    wg, ag = rng.uniform(0.01, 1, (1, 9)).astype(np.float32), rng.uniform(0.01, 1, (1, 5)).astype(np.float32)
    assert np.allclose(O.group_dequant_gemm_fp64(a1, w1, wg, ag), O.dequant_gemm_fp64(a1, w1, wg[0], ag[0]),
                       rtol=1e-13, atol=0)
