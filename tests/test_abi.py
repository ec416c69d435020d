"""The C-ABI library loads on CPU and exports every function include/fireq.h declares.

No compute calls (no GPU here): only pure host entry points (sizes, status strings)
and argument validation paths that return before touching CUDA.
"""
import ctypes
import os
import re

import pytest

from paper_2505_20839_b200 import fireq as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "fireq.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fireq_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(F.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return F.load()


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(F.EXPORTS) <= set(names)


def test_host_only_entry_points(lib):
    assert lib.fireq_weight_layout_version() == 1
    assert lib.fireq_packed_weight_bytes(4096, 4096) == 4096 * 4096 // 2
    assert lib.fireq_weight_scale_bytes(4096, 4096) == 4096 * 4096 // 128
    assert lib.fireq_quantize_weight_workspace_bytes(128, 4096) >= 4096 * 8
    assert lib.fireq_status_string(0) == b"FIREQ_SUCCESS"
    assert lib.fireq_status_string(3) == b"FIREQ_ERROR_MISALIGNED"


def test_argument_validation_without_gpu(lib):
    P = ctypes.c_void_p
    # NULL pointers -> INVALID_VALUE before any CUDA call
    st = lib.fireq_w4a8_gemm(None, None, 16, 4096, None, None, 4096, 0, None, None, 4096, 0, None, 0, None)
    assert st == 1 and b"NULL" in lib.fireq_last_error()
    # bad shape -> UNSUPPORTED_SHAPE; misaligned -> MISALIGNED
    buf = ctypes.create_string_buffer(1 << 12)
    base = ctypes.addressof(buf)
    a16 = P((base + 15) & ~15)
    st = lib.fireq_w4a8_gemm(a16, a16, 16, 4000, a16, a16, 4096, 0, None, a16, 4096, 0, a16, 1, None)
    assert st == 2
    st = lib.fireq_w4a8_gemm(P(a16.value + 1), a16, 16, 4096, a16, a16, 4096, 0, None, a16, 4096, 0, a16, 1, None)
    assert st == 3
    st = lib.fireq_quantize_weight(a16, 128, 128, 7, a16, a16, None, None, a16, a16, 1 << 20, None)
    assert st == 1                                    # cas_mode 7
    st = lib.fireq_quantize_act(a16, 0, 128, 128, None, a16, a16, None)
    assert st == 1                                    # M = 0


def test_fused_ffn_host_checks(lib):
    P = ctypes.c_void_p
    assert lib.fireq_ffn_workspace_bytes(16, 4096, 11008) > 0
    assert lib.fireq_ffn_workspace_bytes(16, 4000, 11008) == 0          # not a multiple of 128
    buf = ctypes.create_string_buffer(1 << 12)
    a16 = P((ctypes.addressof(buf) + 15) & ~15)
    args = lambda M, x: (x, 4096, None, M, 4096, 11008, a16, a16, 0, None, a16, a16, 0, None, 0, a16, a16, 4096,
                         a16, 1 << 20, None, 0, None, 0, None)
    assert lib.fireq_ffn_w4a8_decode(*args(16, None)) == 1               # NULL x
    assert lib.fireq_ffn_w4a8_decode(*args(0, a16)) == 2                 # M >= 1
    assert lib.fireq_ffn_w4a8_decode(*args(16, P(a16.value + 2))) == 3  # misaligned x
    bad_r = list(args(16, a16)); bad_r[13] = a16; bad_r[14] = 100         # residual with ldr < d_model
    assert lib.fireq_ffn_w4a8_decode(*bad_r) == 3
    # fireq_w4a8_gemm_residual: NULL residual / ldr < N
    g = lambda r, ldr: lib.fireq_w4a8_gemm_residual(a16, a16, 16, 4096, a16, a16, 4096, 0, None, r, ldr, a16, 4096,
                                                    a16, 1 << 20, None)
    assert g(None, 4096) == 1 and g(a16, 100) == 3
    assert lib.fireq_interleave_gate_up(a16, a16, 100, 4096, a16, None) == 2


def test_kv4q8_host_checks(lib):
    """fireq_quantize_kv / fireq_kv4q8_attention argument validation (no GPU work)."""
    P = ctypes.c_void_p
    buf = ctypes.create_string_buffer(1 << 12)
    a16 = P((ctypes.addressof(buf) + 15) & ~15)
    ws = 1 << 20
    assert lib.fireq_quantize_kv(None, 256, 128, None, a16, a16, a16, a16, ws, None) == 1     # NULL X
    assert lib.fireq_quantize_kv(a16, 200, 128, None, a16, a16, a16, a16, ws, None) == 2      # N % 128
    assert lib.fireq_quantize_kv(a16, 256, 128, None, a16, a16, a16, a16, 16, None) == 7      # workspace

    def att(B=1, N=256, Hq=2, Hkv=1, d=128, causal=1, tau=0.088, q=a16, ldo=256):
        return lib.fireq_kv4q8_attention(q, a16, B, N, Hq, Hkv, d, a16, a16, a16, a16, a16, a16, causal,
                                         ctypes.c_float(tau), a16, ldo, None)
    assert att(q=None) == 1                     # NULL q
    assert att(causal=2) == 1                   # causal must be 0 / 1
    assert att(tau=0.0) == 1                    # tau > 0
    assert att(d=64) == 2                       # d = 128 only
    assert att(N=200) == 2                      # N % 128
    assert att(Hq=3, Hkv=2) == 2                # Hq % Hkv
    assert att(ldo=128) == 3                    # ldo >= Hq d
    assert att(q=P(a16.value + 4)) == 3         # misaligned
