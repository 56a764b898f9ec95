"""CPU oracle for the APT-LLM arbitrary-precision W_p x A_q integer MatMul.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  The product path (``paper_2508_19087_b200``) never imports it and
shares no code with it: no kernels, no helpers, no tables, no constants.

Everything here is plain numpy (int64 / float64) or Python ints, written in
the paper's order and notation.  Citations: ``P:<line>`` is a line of
``PAPER.md`` (arXiv 2508.19087), ``S:<line>`` a line of ``SPEC.md``.

Notation:
  * A  = activation codes, shape [M, K], ``abits`` = p_a bits  (paper's X, p)
  * W  = weight codes,     shape [N, K], ``wbits`` = p_w bits  (paper's W, q)
  * signed code x in [-2^(n-1), 2^(n-1)-1]  (n = 1 -> {-1, 0}, reading Q4)
  * bipolar value x' = 2x + 1, odd, in [-(2^n-1), 2^n-1]
  * offset bits  u = x + 2^(n-1)  = the bipolar bit pattern
  * Y [m, n]  = sum_k A[m,k] * W[n,k]  over signed codes  (north_star oracle)
  * Y'[m, n]  = sum_k A'[m,k] * W'[n,k] over bipolar values (Fig. 4)

Pinned by ``tests/test_oracle.py`` (closed forms, SPEC worked examples,
exhaustive enumeration, brute force, library special cases).  Every function
below is pinned; none is "parity unpinned".
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np

KPAD_QUANTUM = 256  # reading Q6/Q5: packed rows are padded to a multiple of 256 elements
WORD_BITS = 32      # P:252 "32-bit unsigned integers"


# --------------------------------------------------------------------------
# §3.1 bipolar-INT format
# --------------------------------------------------------------------------

def signed_range(n: int) -> tuple[int, int]:
    """Signed n-bit two's-complement range (n=1 -> {-1,0}, reading Q4)."""
    assert 1 <= n <= 8
    return -(1 << (n - 1)), (1 << (n - 1)) - 1


def bipolar_value(bits: list[int]) -> int:
    """P:188 (§3.1 eq.): (x)_D = sum_{i=0}^{n-1} (2 x^(i) - 1) * 2^i.

    ``bits[i]`` is x^(i), bit i (LSB first)."""
    return sum((2 * b - 1) * (1 << i) for i, b in enumerate(bits))


def twos_complement_bits(x: int, n: int) -> list[int]:
    """The n-bit two's-complement pattern of a signed code, LSB first."""
    lo, hi = signed_range(n)
    assert lo <= x <= hi, (x, n)
    pattern = x & ((1 << n) - 1)
    return [(pattern >> i) & 1 for i in range(n)]


def signed_to_bipolar_bits(x: int, n: int) -> list[int]:
    """P:202 (§3.1): "simply flipping the sign bit of a signed INT yields the
    corresponding bipolar-INT data".  Returns the bipolar bit pattern."""
    bits = twos_complement_bits(x, n)
    bits[n - 1] ^= 1
    return bits


def signed_to_bipolar(x: int, n: int) -> int:
    """value-level correspondence x' = 2x + 1 (computed through the bit
    flip of P:202 and the valuation of P:188, so the test of x' == 2x+1 is a
    real check)."""
    return bipolar_value(signed_to_bipolar_bits(x, n))


def bipolar_to_signed(v: int, n: int) -> int:
    """Inverse of P:203: x = (x' - 1) / 2 for odd x' in +-(2^n-1)."""
    assert v % 2 != 0 and -(1 << n) < v < (1 << n), (v, n)
    return (v - 1) // 2


def offset_bits_matrix(codes: np.ndarray, n: int) -> np.ndarray:
    """Bit-plane decomposition (Fig. 4; §4.1 Step 1): for a
    signed-code matrix return u = bipolar bit pattern per element as int64,
    u = (two's-complement pattern) XOR 2^(n-1)  (the sign-bit flip)."""
    c = np.asarray(codes, dtype=np.int64)
    lo, hi = signed_range(n)
    if c.size and (c.min() < lo or c.max() > hi):
        raise ValueError(f"codes out of the signed {n}-bit range")
    return (c & ((1 << n) - 1)) ^ (1 << (n - 1))


def plane_matrices(codes: np.ndarray, n: int) -> list[np.ndarray]:
    """W^(i): the n bit-level matrices as +-1 int64 matrices, i = 0..n-1,
    each bit read as 2*bit-1 ("reinterprets the 0 value as -1")."""
    u = offset_bits_matrix(codes, n)
    return [2 * ((u >> i) & 1) - 1 for i in range(n)]


# --------------------------------------------------------------------------
# §4.1 decomposition & reassembly into the "unified matrix"
# --------------------------------------------------------------------------

def kpad(k: int) -> int:
    return ((k + KPAD_QUANTUM - 1) // KPAD_QUANTUM) * KPAD_QUANTUM if k > 0 else 0


def pack_planes(codes: np.ndarray, n: int) -> tuple[np.ndarray, np.ndarray]:
    """§4.1 Steps 1-3, in the layout of reading Q5/Q6:

    Step 1: split into n 1-bit matrices (bit i of the bipolar pattern u).
    Step 2: pack each row into 32-bit unsigned words, element c -> bit c%32 of
            word c//32 (LSB first); K padded to Kpad = round_up(K,256) with the
            signed code 0 (so pads contribute exactly 0 to signed products).
    Step 3: concatenate the n planes into one array [n][rows][Kpad/32].

    Also returns row_sum[r] = sum_{k<K} signed code (int64).
    """
    c = np.asarray(codes, dtype=np.int64)
    rows, k = c.shape
    kp = kpad(k)
    padded = np.zeros((rows, kp), dtype=np.int64)  # signed code 0 in the pad
    padded[:, :k] = c
    u = offset_bits_matrix(padded, n)
    words = np.zeros((n, rows, kp // WORD_BITS), dtype=np.uint64)
    for i in range(n):
        plane_bits = (u >> i) & 1                                  # Step 1
        grouped = plane_bits.reshape(rows, kp // WORD_BITS, WORD_BITS)
        for b in range(WORD_BITS):                                 # Step 2
            words[i] |= grouped[:, :, b].astype(np.uint64) << np.uint64(b)
    row_sum = c.sum(axis=1) if k else np.zeros(rows, dtype=np.int64)
    return words.astype(np.uint32), row_sum.astype(np.int64)      # Step 3


def unpack_planes(planes: np.ndarray, k: int, n: int) -> np.ndarray:
    """Inverse of ``pack_planes``: planes [n][rows][words] -> signed
    codes [rows, k] (x = u - 2^(n-1))."""
    planes = np.asarray(planes, dtype=np.uint64)
    nn, rows, words = planes.shape
    assert nn == n
    u = np.zeros((rows, words * WORD_BITS), dtype=np.int64)
    for i in range(n):
        for b in range(WORD_BITS):
            bit = ((planes[i] >> np.uint64(b)) & np.uint64(1)).astype(np.int64)
            u[:, b::WORD_BITS] |= bit << i
    return (u - (1 << (n - 1)))[:, :k]


# --------------------------------------------------------------------------
# §3.2 bit-wise MatMul reconstitution
# --------------------------------------------------------------------------

def plane_products(a_codes: np.ndarray, abits: int, w_codes: np.ndarray, wbits: int) -> np.ndarray:
    """pairwise 1-bit MatMuls Y^(i,j) = X^(i) . W^(j)^T over +-1 planes,
    i < abits (activation planes), j < wbits (weight planes).  Returns an
    int64 array [abits][wbits][M][N].  (A library matmul on +-1 int64
    matrices is the step; no blocking.)"""
    xp = plane_matrices(a_codes, abits)
    wp = plane_matrices(w_codes, wbits)
    m, n = xp[0].shape[0], wp[0].shape[0]
    out = np.zeros((abits, wbits, m, n), dtype=np.int64)
    for i in range(abits):
        for j in range(wbits):
            out[i, j] = xp[i] @ wp[j].T
    return out


def plane_products_xor(a_planes: np.ndarray, w_planes: np.ndarray, k: int) -> np.ndarray:
    """P:227 "AND or XOR logic gates", XOR form: over the packed
    words, Y^(i,j)[m][n] = K - 2*popcount(a_i XOR w_j) restricted to the K
    logical bits (pad bits masked off).  A second, independent route to
    ``plane_products``."""
    a_planes = np.asarray(a_planes, dtype=np.uint32)
    w_planes = np.asarray(w_planes, dtype=np.uint32)
    pa, m, words = a_planes.shape
    pw, n, words2 = w_planes.shape
    assert words == words2
    mask = np.zeros(words, dtype=np.uint64)
    for c in range(k):
        mask[c // WORD_BITS] |= np.uint64(1) << np.uint64(c % WORD_BITS)
    out = np.zeros((pa, pw, m, n), dtype=np.int64)
    for i in range(pa):
        for j in range(pw):
            x = (a_planes[i][:, None, :].astype(np.uint64) ^ w_planes[j][None, :, :].astype(np.uint64)) & mask
            pop = np.zeros((m, n), dtype=np.int64)
            for b in range(WORD_BITS):
                pop += ((x >> np.uint64(b)) & np.uint64(1)).astype(np.int64).sum(axis=2)
            out[i, j] = k - 2 * pop
    return out


def recombine(yij: np.ndarray) -> np.ndarray:
    """P:228 data recovery: Y' = sum_{i,j} 2^(i+j) * Y^(i,j)  ("each Y^(i,j) is
    shifted according to its respective bit positions (i,j) ... aggregated
    through summation")."""
    pa, pw = yij.shape[:2]
    out = np.zeros(yij.shape[2:], dtype=np.int64)
    for i in range(pa):
        for j in range(pw):
            out += yij[i, j] << (i + j)
    return out


def gemm_bipolar(a_codes, abits, w_codes, wbits) -> np.ndarray:
    """The paper's algorithm end to end: decompose, +-1 plane
    products, shift-add recovery -> Y' (bipolar product), int64."""
    return recombine(plane_products(a_codes, abits, w_codes, wbits))


def gemm_signed(a_codes: np.ndarray, w_codes: np.ndarray) -> np.ndarray:
    """The plain definition (north_star: "a plain CPU int64 GEMM on the unpacked
    signed integers"): Y[m][n] = sum_k A[m][k] * W[n][k], int64."""
    a = np.asarray(a_codes, dtype=np.int64)
    w = np.asarray(w_codes, dtype=np.int64)
    return a @ w.T


def gemm_signed_blas(a_codes: np.ndarray, w_codes: np.ndarray, chunk: int = 4096) -> np.ndarray:
    """The same plain definition Y = A . W^T evaluated with a library fp64 matmul (BLAS dgemm) as
    the one step, for full-size outputs (BASELINE configs[2]-[4], up to 4096 x 28672 x 8192) that
    the int64 loops cannot finish in seconds.  Exact: every product |a w| <= 2^14 and every partial
    sum, in whatever order BLAS adds, is an integer of magnitude <= K * 2^14 < 2^53, so each fp64
    operation is exact and the result equals the int64 GEMM bit for bit (asserted for K < 2^39).
    W is processed in row chunks to bound host memory."""
    a = np.asarray(a_codes)
    w = np.asarray(w_codes)
    assert a.shape[1] == w.shape[1] and a.shape[1] < (1 << 39)
    af = a.astype(np.float64)
    out = np.empty((a.shape[0], w.shape[0]), dtype=np.int64)
    for n0 in range(0, w.shape[0], chunk):
        out[:, n0:n0 + chunk] = (af @ w[n0:n0 + chunk].astype(np.float64).T).astype(np.int64)
    return out


def gemm_python(a_rows, w_rows) -> list[list[int]]:
    """Arbitrary-precision Python-int triple loop ("second independent
    implementation"); tiny inputs only."""
    return [[sum(int(x) * int(y) for x, y in zip(ar, wr)) for wr in w_rows] for ar in a_rows]


# --------------------------------------------------------------------------
# Overflow guard (reading Q8) and the fp16 scale epilogue (reading Q10)
# --------------------------------------------------------------------------

def int32_bound_ok(k: int, abits: int, wbits: int) -> bool:
    """Reading Q8 ("32-bit"): the library accepts a problem iff the
    bipolar-product bound K_pad * (2^p_a - 1) * (2^p_w - 1) < 2^31 (this also
    bounds |Y| and every unsigned partial sum)."""
    return kpad(k) * ((1 << abits) - 1) * ((1 << wbits) - 1) < (1 << 31)


def scale_fp64(y: np.ndarray, w_scale: np.ndarray, a_scale: np.ndarray | None) -> np.ndarray:
    """Reading Q10 (P:201-207 linear quantization W = s*W_hat): the reference
    for the fp16 epilogue, ref[m][n] = Y[m][n] * w_scale[n] * a_scale[m] in fp64
    (scales are fp32 values promoted exactly)."""
    y = np.asarray(y, dtype=np.float64)
    ws = np.asarray(w_scale, dtype=np.float32).astype(np.float64)
    out = y * ws[None, :]
    if a_scale is not None:
        out = out * np.asarray(a_scale, dtype=np.float32).astype(np.float64)[:, None]
    return out


def scale_exact(y: int, ws: float, a_s: float) -> Fraction:
    """Exact rational value of Y*ws*as (pins ``scale_fp64``)."""
    return Fraction(int(y)) * Fraction(float(ws)) * Fraction(float(a_s))


# --------------------------------------------------------------------------
# §3.1 linear quantization, per-token symmetric: the step before
# the pack (reading R-Q)
# --------------------------------------------------------------------------

def quantize_symmetric(x: np.ndarray, n: int) -> tuple[np.ndarray, np.ndarray]:
    """P:199-201 "W = s W_hat + z" with z = 0 and one scale s per row (token),
    for n-bit signed codes (n >= 2).  The integer decision is taken in IEEE
    fp32, the precision of the CUDA kernel (tier rule: both sides decide in the
    same precision):
        s[r]      = fl32( max_c |x[r,c]| / (2^(n-1) - 1) )
        x_hat[r,c] = clamp(rint(fl32(x[r,c] / s[r])), -2^(n-1), 2^(n-1)-1)   (0 if s = 0)
    ``x`` holds fp16 values (any float array; converted to fp32 exactly).
    Returns (int8 codes [rows, k], float32 scales [rows])."""
    if n < 2 or n > 8:
        raise ValueError("symmetric quantization needs n in [2, 8]")
    x32 = np.asarray(x, dtype=np.float16).astype(np.float32)
    qmax = np.float32((1 << (n - 1)) - 1)
    codes = np.zeros(x32.shape, dtype=np.int8)
    scales = np.zeros(x32.shape[0], dtype=np.float32)
    lo, hi = signed_range(n)
    for r in range(x32.shape[0]):
        amax = np.float32(np.max(np.abs(x32[r]))) if x32.shape[1] else np.float32(0)
        s = np.float32(amax / qmax)          # fp32 / fp32 -> IEEE round to nearest
        scales[r] = s
        if s == 0:
            continue
        q = np.rint(x32[r] / s)              # fp32 division, then half-to-even
        codes[r] = np.clip(q, lo, hi).astype(np.int8)
    return codes, scales


def group_dequant_gemm_fp64(a_codes: np.ndarray, w_codes: np.ndarray, w_gscale, a_gscale=None, a_scale=None,
                            group: int = 128) -> np.ndarray:
    """Group-wise scales (the 128-group configurations Atom-128G / QuaRot-128G of the
    PPL table, with the linear quantization x = s x_hat of P:199-201 applied per K-group):
    element k of a row belongs to group g = k // group; the weights dequantize as
    W[n][k] = w_gscale[g][n] * w_hat[n][k] and the activations as A[m][k] = a_gscale[g][m] * a_hat[m][k]
    (or a_scale[m] * a_hat[m][k] on every group when a_gscale is None; scale 1 when both are None).  The
    plain definition, in fp64: dequantize both operands, then out = A . W^T.  w_gscale: [ceil(K/group)][N]
    fp32 (group-major, the GPTQ layout), a_gscale: [ceil(K/group)][M]."""
    m, k = a_codes.shape
    n = w_codes.shape[0]
    gi = np.arange(k) // group                                   # group of every K element
    wg = np.asarray(w_gscale, dtype=np.float64)                  # [G][N]
    Wd = wg[gi, :].T * w_codes.astype(np.float64)                # [N][K]
    if a_gscale is not None:
        Ad = np.asarray(a_gscale, dtype=np.float64)[gi, :].T * a_codes.astype(np.float64)
    else:
        sa = np.ones(m) if a_scale is None else np.asarray(a_scale, dtype=np.float64)
        Ad = sa[:, None] * a_codes.astype(np.float64)
    return Ad @ Wd.T


def dequant_gemm_fp64(a_codes: np.ndarray, w_codes: np.ndarray, w_scale, a_scale, w_zero=None,
                      a_zero=None) -> np.ndarray:
    """P:199-201 linear quantization with zero points on both operands, the plain
    definition: dequantize X = a_scale x_hat + a_zero and W = w_scale w_hat + w_zero in fp64, then
    out = X . W^T (fp64 matmul).  Scales / zeros are fp32 arrays (or None: scale 1, zero 0)."""
    m, k = a_codes.shape
    n = w_codes.shape[0]
    def vec(v, size, default):
        return np.full(size, default, dtype=np.float64) if v is None else np.asarray(v, dtype=np.float64)
    X = vec(a_scale, m, 1.0)[:, None] * a_codes.astype(np.float64) + vec(a_zero, m, 0.0)[:, None]
    W = vec(w_scale, n, 1.0)[:, None] * w_codes.astype(np.float64) + vec(w_zero, n, 0.0)[:, None]
    return X @ W.T
