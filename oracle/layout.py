"""Packed INT4 weight / scale layout, version 1 -- TEST INFRASTRUCTURE ONLY.

The paper fixes the codes (INT4 in [-8, 7]) and the grouping (128
consecutive N_in elements of one output row share one FP8 scale, P:112,
reading A1 in DESIGN.md) but not the byte layout.  Layout v1 (DESIGN.md
"Data layout in HBM") is chosen so that one (128-row tile, 128-K group)
block is a contiguous 8 KiB bulk copy and so that, inside the block, the
16 bytes holding K-slice j (32 codes) of row r are at ((j*128 + r)*16):
a warp reading slice j of 32 consecutive rows touches 512 contiguous bytes.

Element (n, k) of W [N][K]:
  nt = n // 128, r = n % 128, g = k // 128, j = (k % 128) // 32,
  b = (k % 32) // 2, nibble = k % 2 (0 = low nibble)
  byte = (((nt * G + g) * 4 + j) * 128 + r) * 16 + b,   G = K // 128
  nibble value = code & 0xF (4-bit two's complement)
Scale sigma(n, g): byte (nt * G + g) * 128 + r.

Written independently of the CUDA path's index arithmetic; the tests also
check that the map is a bijection and un-tile it back to canonical order.
"""
import numpy as np

TILE_N = 128
GROUP = 128
LAYOUT_VERSION = 1


def packed_byte_index(n, k, K):
    """Byte offset and nibble (0 low, 1 high) of element (n, k)."""
    n = np.asarray(n, dtype=np.int64)
    k = np.asarray(k, dtype=np.int64)
    G = K // GROUP
    nt, r = n // TILE_N, n % TILE_N
    g, kk = k // GROUP, k % GROUP
    j, b = kk // 32, (kk % 32) // 2
    byte = (((nt * G + g) * 4 + j) * TILE_N + r) * 16 + b
    return byte, k % 2


def scale_index(n, g, K):
    n = np.asarray(n, dtype=np.int64)
    g = np.asarray(g, dtype=np.int64)
    G = K // GROUP
    return (n // TILE_N * G + g) * TILE_N + n % TILE_N


def pack_codes(codes):
    """codes int [N][K] in [-8, 7] -> packed uint8 [N*K/2] (layout v1)."""
    codes = np.asarray(codes)
    N, K = codes.shape
    assert N % TILE_N == 0 and K % GROUP == 0
    assert codes.min() >= -8 and codes.max() <= 7
    nib = (codes.astype(np.int64) & 0xF).astype(np.uint8)
    n, k = np.meshgrid(np.arange(N), np.arange(K), indexing="ij")
    byte, half = packed_byte_index(n, k, K)
    out = np.zeros(N * K // 2, dtype=np.uint8)
    lo = half == 0
    out[byte[lo]] |= nib[lo]
    out[byte[~lo]] |= (nib[~lo] << 4).astype(np.uint8)
    return out


def unpack_codes(packed, N, K):
    """Inverse of pack_codes: packed uint8 -> codes int8 [N][K]."""
    packed = np.asarray(packed, dtype=np.uint8)
    n, k = np.meshgrid(np.arange(N), np.arange(K), indexing="ij")
    byte, half = packed_byte_index(n, k, K)
    nib = np.where(half == 0, packed[byte] & 0xF, packed[byte] >> 4).astype(np.int16)
    return np.where(nib >= 8, nib - 16, nib).astype(np.int8)


def pack_scales(scale_codes):
    """sigma codes uint8 [N][K/128] -> blocked uint8 [N*K/128]."""
    sc = np.asarray(scale_codes, dtype=np.uint8)
    N, G = sc.shape
    n, g = np.meshgrid(np.arange(N), np.arange(G), indexing="ij")
    out = np.zeros(N * G, dtype=np.uint8)
    out[scale_index(n, g, G * GROUP)] = sc
    return out


def pack_scales16(scale_bits):
    """sigma_BF16 bit patterns uint16 [N][K/128] -> blocked uint16 [N*K/128] (same block order)."""
    sc = np.asarray(scale_bits, dtype=np.uint16)
    N, G = sc.shape
    n, g = np.meshgrid(np.arange(N), np.arange(G), indexing="ij")
    out = np.zeros(N * G, dtype=np.uint16)
    out[scale_index(n, g, G * GROUP)] = sc
    return out


def unpack_scales(blocked, N, K):
    G = K // GROUP
    n, g = np.meshgrid(np.arange(N), np.arange(G), indexing="ij")
    return np.asarray(blocked, dtype=np.uint8)[scale_index(n, g, K)]
