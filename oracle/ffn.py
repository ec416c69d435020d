"""Llama FFN built from the FireQ linear layer -- TEST INFRASTRUCTURE ONLY.

The paper's FFN benchmark (Fig. fig:int4-fp8-kernel) runs the gate,
up and down projections as INT4 x FP8 GEMMs; Step 3 of the kernel lists SiLU and
element-wise multiplication among the epilogue operations.  CAS needs one
Lambda for projections that share an input (the preceding layer can absorb only
one Lambda^-1), so gate and up are quantized as ONE matrix
[gate; up] (reading R20), and the down projection's Lambda^-1 is merged
into the up projection's output channels (gamma, "merged offline").

  x_hat, beta = A1..A3(x, c_gu)
  [g | u]     = bf16( fireq_linear(x_hat, W_gu) * gamma ),  gamma = [1 .. 1 | c_down]
  h           = bf16( silu(g) * u ),  silu(g) = g / (1 + exp(-g))      (fp64 here)
  y           = bf16( fireq_linear(A2..A3(h), W_down) [+ residual] )   (Step 3 "addition")
"""
import numpy as np

from .numerics import bf16_rn
from . import gemm, quant


def silu_mul(g, u):
    g = np.asarray(g, dtype=np.float64)
    return bf16_rn(g / (1.0 + np.exp(-g)) * np.asarray(u, dtype=np.float64))


def ffn_reference(X, q_gu, q_down, n_ff, residual=None):
    """X bf16 values [M][d]; q_gu / q_down: oracle QuantizedWeight (packed); residual: values [M][d]
    added in the down projection's epilogue (or None).  Returns y (bf16 values) and its fp64 value."""
    N_gu, d = 2 * n_ff, X.shape[1]
    xq, beta = quant.quantize_act(X, q_gu.c)
    gamma = np.concatenate([np.ones(n_ff), q_down.c])
    r = gemm.gemm_reference(xq, beta, q_gu.packed, q_gu.scales, N_gu, d, q_gu.n, gamma=gamma)
    gu = bf16_rn(r)
    h = silu_mul(gu[:, :n_ff], gu[:, n_ff:])
    hq, hbeta = quant.quantize_act(h)
    y = gemm.gemm_reference(hq, hbeta, q_down.packed, q_down.scales, d, n_ff, q_down.n, residual=residual)
    return bf16_rn(y), y
