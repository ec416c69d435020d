"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO FireQ arithmetic: it only draws random numbers with the
shapes and value structure of the paper's workloads (Llama linear layers,
P:303-316) and rounds them to bf16 storage.  Recipe:

  weights     W[n,k] = bf16(0.02 * r_n * s_k * z),  z ~ N(0,1),
              log r_n ~ N(0, 0.3^2)  (row scale), log s_k ~ N(0, 0.5^2)
              (input-channel skew, the structure CAS targets),
              8 input channels x8 (outlier channels), 1% of rows x0.05
              (creates pre-PTS underflow-risk groups, App. E.3),
              0.1% exact zeros.
  activations X[m,k] = bf16(z * a_k), a_k = 1 except 4 "massive" channels x20.

Seeds: numpy PCG64(seed).  bf16 rounding uses torch's float32 -> bfloat16
cast (round to nearest even), a storage conversion, not part of the method.
"""
import numpy as np
import torch

SEED_BASE = 20250527

# Linear-layer shapes (N_out, N_in) of the configs in BASELINE.json.
SHAPES = {
    "llama2-7b.q": (4096, 4096),
    "llama2-7b.gate": (11008, 4096),
    "llama2-7b.up": (11008, 4096),
    "llama2-7b.down": (4096, 11008),
    "llama3-8b.q": (4096, 4096),
    "llama3-8b.k": (1024, 4096),
    "llama3-8b.v": (1024, 4096),
    "llama3-8b.o": (4096, 4096),
    "llama3-8b.gate": (14336, 4096),
    "llama3-8b.up": (14336, 4096),
    "llama3-8b.down": (4096, 14336),
    "llama2-70b.gate": (28672, 8192),
    "llama2-70b.up": (28672, 8192),
    "llama2-70b.down": (8192, 28672),
}


def to_bf16_bits(a):
    """float array -> uint16 bf16 bit patterns (RNE via torch)."""
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16).copy()


def bits_to_f64(bits):
    u = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    return u.view(np.float32).astype(np.float64)


def bits_to_torch(bits):
    """uint16 bf16 bits (numpy) -> torch.bfloat16 tensor (CPU)."""
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16)


def weights(N, K, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    z = rng.standard_normal((N, K), dtype=np.float32)
    r = np.exp(rng.normal(0.0, 0.3, size=N)).astype(np.float32)
    s = np.exp(rng.normal(0.0, 0.5, size=K)).astype(np.float32)
    s[rng.choice(K, size=min(8, K), replace=False)] *= 8.0
    small = rng.choice(N, size=max(1, N // 100), replace=False)
    r[small] *= 0.05
    w = 0.02 * z * r[:, None] * s[None, :]
    nz = rng.choice(N * K, size=(N * K) // 1000, replace=False)
    w.reshape(-1)[nz] = 0.0
    return to_bf16_bits(w)


def activations(M, K, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    z = rng.standard_normal((M, K), dtype=np.float32)
    a = np.ones(K, dtype=np.float32)
    a[rng.choice(K, size=min(4, K), replace=False)] = 20.0
    return to_bf16_bits(z * a[None, :])


def layer_seed(config_idx, layer_idx):
    return SEED_BASE + 100 * config_idx + layer_idx


def attention(B, N, Hq, Hkv, seed, d=128):
    """Post-RoPE query / key / value heads of a Llama-style attention layer (bf16 bits):
    Q [B][Hq][N][d] ~ N(0, 1); K [B][Hkv][N][d] ~ N(0, 1) with 2 outlier channels per kv head
    (x16, the key outliers CRS targets) and their RoPE pair channels (x4); V ~ N(0, 1)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    q = rng.standard_normal((B, Hq, N, d), dtype=np.float32)
    k = rng.standard_normal((B, Hkv, N, d), dtype=np.float32)
    v = rng.standard_normal((B, Hkv, N, d), dtype=np.float32)
    for hk in range(Hkv):
        for c in rng.choice(d // 2, size=2, replace=False):
            k[:, hk, :, c] *= 16.0
            k[:, hk, :, c + d // 2] *= 4.0
    return to_bf16_bits(q), to_bf16_bits(k), to_bf16_bits(v)
