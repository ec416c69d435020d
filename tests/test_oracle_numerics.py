"""Pins for oracle/numerics.py against things other than itself.

* torch's float8_e4m3fn / bfloat16 casts (library routines),
* exact-rational brute force over the E4M3 grid (Fractions),
* the paper's constants: 448 = 1.75*2^8, min subnormal 2^-9,
* SPEC's worked examples.
"""
import bisect
from fractions import Fraction

import numpy as np
import pytest
import torch

from oracle import numerics as nm

GRID = [Fraction(v) for v in nm.E4M3_POS_GRID]


def rn_exact(x: Fraction) -> Fraction:
    """Nearest E4M3 value by exact distance; ties -> even code; saturating."""
    a = abs(x)
    if a >= 448:
        r = Fraction(448)
    else:
        i = bisect.bisect_right(GRID, a) - 1          # GRID[i] <= a < GRID[i+1]
        cand = [j for j in (i, i + 1) if 0 <= j < 127]
        r = GRID[min(cand, key=lambda j: (abs(GRID[j] - a), j % 2))]
    return -r if x < 0 else r


def rz_exact(x: Fraction) -> Fraction:
    return GRID[bisect.bisect_right(GRID, x) - 1] if x < 448 else Fraction(448)


def test_decode_matches_torch_all_codes():
    t = torch.arange(256, dtype=torch.int32).to(torch.uint8).view(torch.float8_e4m3fn).float().numpy()
    a = np.nan_to_num(t.astype(np.float64), nan=-1234.0)
    b = np.nan_to_num(nm.E4M3_DECODE, nan=-1234.0)
    assert np.array_equal(a, b)


def test_paper_constants():
    assert nm.E4M3_POS_GRID[-1] == 1.75 * 2 ** 8 == 448.0
    assert nm.E4M3_POS_GRID[1] == 2.0 ** -9
    assert nm.E4M3_POS_GRID.size == 127
    assert np.isnan(nm.E4M3_DECODE[0x7F]) and np.isnan(nm.E4M3_DECODE[0xFF])


def test_roundtrip_all_codes():
    codes = np.array([c for c in range(256) if c not in (0x7F, 0xFF)], dtype=np.uint8)
    v = nm.e4m3_decode(codes)
    assert np.array_equal(nm.e4m3_encode(nm.e4m3_rn(v)), codes)


def test_spec_examples():
    x = 1.5 * 2.0 ** -10
    assert nm.e4m3_rz_nonneg(x) == 0.0                   # S:62 toward zero -> +0
    assert nm.e4m3_rn(x) == 2.0 ** -9                    # S:62 nearest -> 2^-9
    assert nm.e4m3_rn(448.0) == 448.0 and nm.e4m3_rn(0.0) == 0.0
    assert nm.e4m3_rn(2.0 ** -9) == 2.0 ** -9


def _probe_values(rng):
    g = nm.E4M3_POS_GRID
    mids = (g[:-1] + g[1:]) / 2
    vals = [g, mids, np.nextafter(mids, 0), np.nextafter(mids, 1e9),
            rng.uniform(0, 500, 2000), np.exp2(rng.uniform(-14, 9, 2000)),
            np.array([448.0, 460.0, 464.0, 463.99, 464.01, 479.0, 500.0, 1e6, 2.0 ** -10, 2.0 ** -11])]
    v = np.concatenate(vals)
    return np.concatenate([v, -v])


def test_rn_vs_exact_rational():
    rng = np.random.default_rng(0)
    v = _probe_values(rng)
    got = nm.e4m3_rn(v)
    for x, y in zip(v, got):
        e = rn_exact(Fraction(float(x)))
        assert Fraction(float(y)) == e, (x, y, e)
        if e == 0:
            assert np.signbit(y) == np.signbit(x)     # IEEE sign of a rounded zero


def test_rn_vs_torch_in_range():
    rng = np.random.default_rng(1)
    v = _probe_values(rng)
    v = v[np.abs(v) <= 464.0].astype(np.float32)   # torch does not saturate above 464
    t = torch.from_numpy(v).to(torch.float8_e4m3fn).float().numpy().astype(np.float64)
    assert np.array_equal(t, nm.e4m3_rn(v.astype(np.float64)))


def test_rz_vs_exact_rational():
    rng = np.random.default_rng(2)
    v = np.abs(_probe_values(rng))
    got = nm.e4m3_rz_nonneg(v)
    for x, y in zip(v, got):
        assert Fraction(float(y)) == rz_exact(Fraction(float(x)))
    # RZ never increases magnitude, and everything below 2^-9 goes to zero (Lemma 1 mechanism)
    assert np.all(got <= v)
    assert np.all(nm.e4m3_rz_nonneg(np.exp2(rng.uniform(-40, -9.0001, 100))) == 0)


def test_bf16_vs_torch():
    rng = np.random.default_rng(3)
    f = np.concatenate([rng.standard_normal(5000) * 10.0 ** rng.integers(-30, 30, 5000),
                        np.exp2(rng.uniform(-140, -120, 200))]).astype(np.float32)
    t = torch.from_numpy(f).to(torch.bfloat16).float().numpy().astype(np.float64)
    assert np.array_equal(t, nm.bf16_rn(f.astype(np.float64)))


def test_bf16_ties_to_even_exact():
    # 1 + 2^-8 is the midpoint of 1 and 1+2^-7 -> rounds to 1 (even); 1 + 3*2^-8 -> 1 + 2^-6
    assert nm.bf16_rn(1 + 2.0 ** -8) == 1.0
    assert nm.bf16_rn(1 + 3 * 2.0 ** -8) == 1 + 2.0 ** -6
    assert nm.bf16_rn(1 + 2.0 ** -8 + 2.0 ** -40) == 1 + 2.0 ** -7


def test_bf16_bits_roundtrip():
    bits = np.arange(0, 65536, 7, dtype=np.uint32).astype(np.uint16)
    vals = nm.bf16_from_bits(bits)
    ok = np.isfinite(vals)
    assert np.array_equal(nm.bf16_to_bits(vals[ok]), bits[ok])
