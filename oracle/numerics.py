"""Number formats used by FireQ, written out from their definitions.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

E4M3 "fn" flavour ("FP8 (E4M3)"; P:504-510 min subnormal 2^-9;
P:554 overflow threshold 1.75*2^8 = 448): 1 sign, 4 exponent (bias 7),
3 mantissa bits, no infinities, one NaN per sign (S.1111.111).

Rounding readings (R2, R5-R8, R17):
  * e4m3_rn  -- round to nearest, ties to even mantissa, |x| above 448
                saturates to +-448 (P:554 treats 448 as the ceiling;
                PTX cvt.rn.satfinite semantics).  The sign of the exact value
                is kept, so a negative value that rounds to zero is -0
                (code 0x80), as in IEEE arithmetic.
  * e4m3_rz_nonneg -- largest grid value <= x (toward zero), capped at 448;
                forced for the group scale by Lemma 1.
  * bf16_rn  -- IEEE binary16-brain round to nearest even ("BF16
                scaling factor"; P:130 BF16 output).

All values are carried as numpy float64 arrays holding exact dyadic values.
"""
import numpy as np

E4M3_MAX = 448.0                 # 1.75 * 2^8
E4M3_MIN_SUBNORMAL = 2.0 ** -9
E4M3_MIN_NORMAL = 2.0 ** -6
UNDERFLOW_T = 7.0 * 2.0 ** -9    # Lemma 1 threshold, P:504 / eq:pts_first_condition


def e4m3_decode_bitfield(code):
    """Value of one E4M3 code from its bit fields (scalar, exact)."""
    code = int(code) & 0xFF
    s = -1.0 if code & 0x80 else 1.0
    e = (code >> 3) & 0xF
    f = code & 0x7
    if e == 0xF and f == 0x7:
        return float("nan")
    if e == 0:
        return s * f * 2.0 ** -9          # subnormal: 0.f * 2^(1-7)
    return s * (1.0 + f / 8.0) * 2.0 ** (e - 7)


# 256-entry decode table and the sorted non-negative finite grid (codes 0..126).
E4M3_DECODE = np.array([e4m3_decode_bitfield(c) for c in range(256)], dtype=np.float64)
E4M3_POS_GRID = E4M3_DECODE[:127].copy()          # strictly increasing, 0 .. 448
assert np.all(np.diff(E4M3_POS_GRID) > 0) and E4M3_POS_GRID[-1] == E4M3_MAX


def e4m3_decode(codes):
    """uint8 codes -> float64 values (NaN for the two NaN codes)."""
    return E4M3_DECODE[np.asarray(codes, dtype=np.uint8)]


def e4m3_encode(values):
    """Exact grid values (float64, finite, |v| <= 448) -> uint8 codes.

    The sign bit is the sign bit of the float64 (so -0.0 -> 0x80).
    Raises if a value is not on the grid.
    """
    v = np.asarray(values, dtype=np.float64)
    a = np.abs(v)
    idx = np.searchsorted(E4M3_POS_GRID, a)
    idx = np.minimum(idx, 126)
    if not np.all(E4M3_POS_GRID[idx] == a):
        raise ValueError("e4m3_encode: value not on the E4M3 grid")
    return (idx.astype(np.uint8) | (np.signbit(v).astype(np.uint8) << 7)).astype(np.uint8)


def e4m3_rn(x):
    """Round float64 values to E4M3: nearest, ties-to-even, saturate at 448.

    Written as the textbook quantum rule: for |x| in binade [2^E, 2^(E+1)),
    E >= -6, the grid spacing is 2^(E-3); below 2^-6 the (subnormal) spacing
    is 2^-9.  |x| / spacing is exact in float64 (power-of-two scaling) and
    np.rint rounds half to even, which is ties-to-even on the mantissa.
    """
    x = np.asarray(x, dtype=np.float64)
    a = np.abs(x)
    with np.errstate(divide="ignore"):
        _, e = np.frexp(a)                 # a = m * 2^e, m in [0.5, 1)
    E = np.maximum(e - 1, -6)              # a in [2^E, 2^(E+1)) for normals
    q = np.ldexp(1.0, E - 3)
    r = np.rint(a / q) * q
    r = np.minimum(r, E4M3_MAX)            # satfinite
    return np.copysign(r, x)


def e4m3_rz_nonneg(x):
    """Largest E4M3 grid value <= x (x >= 0), capped at 448."""
    x = np.asarray(x, dtype=np.float64)
    if np.any(x < 0):
        raise ValueError("e4m3_rz_nonneg expects x >= 0")
    idx = np.searchsorted(E4M3_POS_GRID, x, side="right") - 1
    return E4M3_POS_GRID[np.clip(idx, 0, 126)]


def bf16_rn(x):
    """Round float64 values to bfloat16 (8-bit significand), nearest-even.

    Same quantum rule as e4m3_rn with 7 fraction bits, min normal 2^-126,
    subnormal spacing 2^-133; overflow (never reached here) goes to inf.
    """
    x = np.asarray(x, dtype=np.float64)
    a = np.abs(x)
    with np.errstate(divide="ignore"):
        _, e = np.frexp(a)
    E = np.maximum(e - 1, -126)
    q = np.ldexp(1.0, E - 7)
    r = np.rint(a / q) * q
    r = np.where(r >= 2.0 ** 128, np.inf, r)
    return np.copysign(r, x)


def bf16_to_bits(values):
    """Exact bf16 values (float64) -> uint16 bit patterns."""
    f = np.asarray(values, dtype=np.float64).astype(np.float32)
    if not np.all(f.astype(np.float64) == np.asarray(values, dtype=np.float64)):
        raise ValueError("bf16_to_bits: not representable")
    u = f.view(np.uint32)
    if np.any(u & 0xFFFF):
        raise ValueError("bf16_to_bits: value not on the bf16 grid")
    return (u >> 16).astype(np.uint16)


def bf16_from_bits(bits):
    """uint16 bf16 bit patterns -> float64 values."""
    u = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    return u.view(np.float32).astype(np.float64)


def f32(x):
    """float64 -> nearest float32 (IEEE RN), returned as float64."""
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)
