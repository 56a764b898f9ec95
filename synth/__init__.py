"""Seeded synthetic input generators shared by tests, bench and smoke.

Holds none of the method's arithmetic: only random integer codes of a given
signed bit width and random positive fp32 scales.
"""
import numpy as np


def signed_codes(rows: int, k: int, bits: int, seed: int) -> np.ndarray:
    """i.i.d. uniform signed codes over [-2^(bits-1), 2^(bits-1)-1] as int8 [rows, k]."""
    rng = np.random.Generator(np.random.PCG64(seed))
    lo, hi = -(1 << (bits - 1)), (1 << (bits - 1)) - 1
    return rng.integers(lo, hi + 1, size=(rows, k), dtype=np.int64).astype(np.int8)


def log_uniform_scales(n: int, lo_exp: float, hi_exp: float, seed: int) -> np.ndarray:
    """Positive fp32 scales 2^U(lo_exp, hi_exp) (w_scale: -10..-6, a_scale: -6..-2)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.exp2(rng.uniform(lo_exp, hi_exp, size=n)).astype(np.float32)


def config_seed(config_id: int, wbits: int, abits: int, salt: int = 0) -> int:
    """seed = 1000*config_id + 10*wbits + abits (+ salt), SURVEY §8(d)."""
    return 1000 * config_id + 10 * wbits + abits + 100000 * salt


def fp16_activations(rows: int, k: int, seed: int, outlier_channels: int = 8) -> np.ndarray:
    """fp16 activations [rows, k]: N(0, 1) with a few outlier channels scaled by 20 (the
    channel-wise outliers of LLM activations), per-row magnitudes 2^U(-3, 3)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    x = rng.standard_normal((rows, k))
    if k > 0 and outlier_channels > 0:
        x[:, rng.choice(k, size=min(k, outlier_channels), replace=False)] *= 20.0
    x *= np.exp2(rng.uniform(-3, 3, size=(rows, 1)))
    return x.astype(np.float16)
