// quant_weight.cu -- fireq_quantize_weight: offline W1..W6 (CAS, PTS, INT4 group
// quantization with FP8 scales, layout-v1 packing).  P:141-175.
// Exact semantics are the readings in include/fireq.h / DESIGN.md; every
// floating-point step is an IEEE-rounded operation the oracle reproduces
// (no FMA contraction: explicit __fmul_rn / __fdiv_rn / __dadd_rn).
#include <climits>
#include "common.cuh"

namespace fireq {
namespace {

constexpr float kUnderflowT = 7.0f * 0x1p-9f;   // Lemma 1 threshold 7*2^-9

struct WStats {
    unsigned max_bits;     // max |W_bar| as float bits (non-negative floats order as uints)
    unsigned mnz_bits;     // min nonzero |W_bar|
    int n2;                // min over elements of the overflow-band exponent n_w in [0, 60]
    int bad;               // non-finite input seen
    int n;                 // resolved PTS exponent
    int status;
};

__global__ void k_stats_init(WStats* st) {
    st->max_bits = 0u;
    st->mnz_bits = 0x7F800000u;
    st->n2 = INT_MAX;
    st->bad = 0;
    st->n = 0;
    st->status = 0;
}

// W1 part 1: absmean_k = fp32( (sum_{n ascending} |W[n,k]| in fp64) / N ), one thread per k.
__global__ void k_col_absmean(const __nv_bfloat16* __restrict__ W, int64_t N, int64_t K,
                              float* __restrict__ absmean) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    double acc = 0.0;
    int64_t n = 0;
    for (; n + 8 <= N; n += 8) {
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __bfloat162float(W[(n + i) * K + k]);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc = __dadd_rn(acc, (double)fabsf(v[i]));   // sequential order
    }
    for (; n < N; ++n) acc = __dadd_rn(acc, (double)fabsf(__bfloat162float(W[n * K + k])));
    absmean[k] = __double2float_rn(__ddiv_rn(acc, (double)N));
}

// W1 part 2: omega_bar (sequential fp64 sum over k), lambda_k, c_k.
__global__ void k_cas_finalize(const float* __restrict__ absmean, int64_t K, int cas_mode,
                               float* __restrict__ lam_ws, float* __restrict__ lam_out,
                               __nv_bfloat16* __restrict__ c_out) {
    __shared__ float omega_s;
    if (threadIdx.x == 0 && cas_mode == 1) {
        double s = 0.0;
        for (int64_t k = 0; k < K; ++k) s = __dadd_rn(s, (double)absmean[k]);
        omega_s = __double2float_rn(__ddiv_rn(s, (double)K));
    }
    __syncthreads();
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
        float lam = 1.0f;
        if (cas_mode == 1) {
            const float a = absmean[k];
            lam = a > 0.0f ? __double2float_rn(__ddiv_rn((double)omega_s, (double)a)) : 1.0f;
        } else if (cas_mode == 2) {
            lam = lam_out ? lam_out[k] : 1.0f;     // caller-given multiplier (KV cache: 1 / t, CRS)
        }
        lam_ws[k] = lam;
        if (lam_out && cas_mode != 2) lam_out[k] = lam;
        if (c_out) c_out[k] = __float2bfloat16_rn(__fdiv_rn(1.0f, lam));
    }
}

// Overflow-band exponent of one element (eq:pts_second_condition): the unique
// integer n with 7*2^(5-n) <= a < 7*2^(6-n), i.e. a*2^n in [224, 448).
// a = f * 2^ex with f in [0.5, 1): a*2^n in [1.75*2^7, 1.75*2^8) gives
// n = 8 - ex if f >= 0.875 else 9 - ex.
__device__ __forceinline__ int band_exponent(float a) {
    int ex;
    const float f = frexpf(a, &ex);
    return f >= 0.875f ? 8 - ex : 9 - ex;
}

// W2 + W3 statistics over all elements: max, min nonzero, min band exponent >= 0.
__global__ void k_wstats(const __nv_bfloat16* __restrict__ W, int64_t total, int64_t K,
                         const float* __restrict__ lam, WStats* st) {
    unsigned mx = 0u, mnz = 0x7F800000u;
    int n2 = INT_MAX, bad = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 8;
    for (int64_t base = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8; base < total; base += stride) {
        const uint4 raw = *reinterpret_cast<const uint4*>(W + base);
        const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&raw);
        const int64_t k0 = base % K;          // K % 8 == 0: the 8 elements share a row
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float wb = __fmul_rn(__bfloat162float(h[i]), lam[k0 + i]);
            const float a = fabsf(wb);
            if (!(a <= 3.4028235e38f)) { bad = 1; continue; }   // NaN or inf
            const unsigned ab = __float_as_uint(a);
            mx = max(mx, ab);
            if (ab != 0u) {
                mnz = min(mnz, ab);
                const int nw = band_exponent(a);
                if (nw >= 0 && nw <= 60) n2 = min(n2, nw);
            }
        }
    }
    // warp reduce, then one atomic per warp
    for (int o = 16; o; o >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mnz = min(mnz, __shfl_xor_sync(0xffffffffu, mnz, o));
        n2 = min(n2, __shfl_xor_sync(0xffffffffu, n2, o));
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&st->max_bits, mx);
        atomicMin(&st->mnz_bits, mnz);
        atomicMin(&st->n2, n2);
        if (bad) atomicOr(&st->bad, 1);
    }
}

// W3: n = min(n1, n2) (Def. 2); writes {n, status}.
__global__ void k_pts(WStats* st, int32_t* pts_and_status) {
    int status = FIREQ_SUCCESS;
    int n = 0;
    if (st->bad) {
        status = FIREQ_ERROR_INVALID_VALUE;
    } else {
        int n1 = 0;
        if (st->max_bits != 0u) {
            // smallest n >= 0 with mnz * 2^n >= 7*2^-9 (exact in fp64)
            const double mnz = (double)__uint_as_float(st->mnz_bits);
            while (n1 <= 200 && mnz * ldexp(1.0, n1) < (double)kUnderflowT) ++n1;
        }
        n = min(n1, st->n2);
        if (n > 60) status = FIREQ_ERROR_INVALID_VALUE;   // degenerate tensor
    }
    st->n = n;
    st->status = status;
    pts_and_status[0] = n;
    pts_and_status[1] = status;
}

// W4..W6: one warp per (row n, group g).  Lane l owns k = g*128 + 4l .. 4l+3.
// BF16S: the sigma_BF16 variant (App. B.1; DESIGN reading R25): sigma =
// bf16_RN(m / 7) (the fp32 quotient of an fp32 m by 7 is never moved onto a bf16 midpoint, so
// this is the exact-rational RNE), stored as bf16 [N/128][K/128][128].
template <bool BF16S>
__global__ void k_group_quant_pack(const __nv_bfloat16* __restrict__ W, int64_t N, int64_t K,
                                   const float* __restrict__ lam, const WStats* __restrict__ st,
                                   uint8_t* __restrict__ packed, uint8_t* __restrict__ scales) {
    const int lane = threadIdx.x & 31;
    const int64_t G = K / 128;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wid >= N * G) return;
    const int64_t n = wid / G, g = wid % G;
    const int64_t k = g * 128 + 4 * lane;
    const float p2n = __int_as_float((127 + st->n) << 23);          // 2^n, n in [0, 60]
    const uint2 raw = *reinterpret_cast<const uint2*>(W + n * K + k);
    const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&raw);
    float wt[4];
    float m = 0.0f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        wt[i] = __fmul_rn(__fmul_rn(__bfloat162float(h[i]), lam[k + i]), p2n);  // W_tilde = W_bar*2^n
        m = fmaxf(m, fabsf(wt[i]));
    }
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    // W4: sigma = largest E4M3 s with 7*s <= m.  RN(m/7) is at most one grid step
    // above it; 7*s is exact in fp32 (<= 7 significant bits), so compare exactly.
    uint32_t sc;
    float sigma;
    if (BF16S) {
        const __nv_bfloat16 sb = __float2bfloat16_rn(__fdiv_rn(m, 7.0f));
        sc = (uint32_t)__bfloat16_as_ushort(sb);
        sigma = __bfloat162float(sb);
    } else {
        sc = e4m3_rn(__fdiv_rn(m, 7.0f));
        if (__fmul_rn(7.0f, e4m3_decode(sc)) > m) sc -= 1u;
        sigma = e4m3_decode(sc);
    }
    // W5: codes
    uint32_t nib[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int c = 0;
        if (sigma > 0.0f) {
            c = (int)rintf(__fdiv_rn(wt[i], sigma));
            c = max(-8, min(7, c));
        }
        nib[i] = (uint32_t)c & 0xFu;
    }
    // W6: layout v1 -- byte (((nt*G + g)*4 + j)*128 + r)*16 + b, low nibble = even k.
    const int64_t nt = n / 128, r = n % 128;
    const int j = lane / 8, b = (lane % 8) * 2;
    const int64_t off = (((nt * G + g) * 4 + j) * 128 + r) * 16 + b;
    const uint16_t two = (uint16_t)(nib[0] | (nib[1] << 4) | (nib[2] << 8) | (nib[3] << 12));
    *reinterpret_cast<uint16_t*>(packed + off) = two;
    if (lane == 0) {
        if (BF16S) reinterpret_cast<uint16_t*>(scales)[(nt * G + g) * 128 + r] = (uint16_t)sc;
        else scales[(nt * G + g) * 128 + r] = (uint8_t)sc;
    }
}

}  // namespace

size_t wq_workspace_bytes(int64_t K) {
    return (size_t)K * 8 + 256;
}

fireq_status_t quantize_weight_impl(const __nv_bfloat16* W, int64_t N, int64_t K, int cas_mode,
                                    uint8_t* w_packed, uint8_t* w_scales, float* cas_lambda,
                                    __nv_bfloat16* cas_inv, int32_t* pts_and_status, void* ws,
                                    cudaStream_t stream, bool bf16_scales) {
    uint8_t* base = static_cast<uint8_t*>(ws);
    WStats* st = reinterpret_cast<WStats*>(base);
    float* absmean = reinterpret_cast<float*>(base + 256);
    float* lam = absmean + K;
    k_stats_init<<<1, 1, 0, stream>>>(st);
    if (cas_mode == 1) {
        k_col_absmean<<<(unsigned)((K + 127) / 128), 128, 0, stream>>>(W, N, K, absmean);
    }
    k_cas_finalize<<<1, 1024, 0, stream>>>(absmean, K, cas_mode, lam, cas_lambda, cas_inv);
    const int64_t total = N * K;
    const int64_t threads_needed = (total / 8 + 255) / 256;
    const unsigned blocks = (unsigned)std::min<int64_t>(threads_needed, (int64_t)sm_count() * 8);
    k_wstats<<<blocks, 256, 0, stream>>>(W, total, K, lam, st);
    k_pts<<<1, 1, 0, stream>>>(st, pts_and_status);
    const int64_t warps = N * (K / 128);
    if (bf16_scales)
        k_group_quant_pack<true><<<(unsigned)((warps + 7) / 8), 256, 0, stream>>>(W, N, K, lam, st, w_packed, w_scales);
    else
        k_group_quant_pack<false><<<(unsigned)((warps + 7) / 8), 256, 0, stream>>>(W, N, K, lam, st, w_packed, w_scales);
    return check_launch(bf16_scales ? "fireq_quantize_weight_bf16s" : "fireq_quantize_weight");
}

// Row order of the fused FFN's gate_up weight: 128-row tile t
// holds gate rows [64 t, 64 t + 64) followed by the up rows of the same channels, so one
// CTA's epilogue sees both operands of SwiGLU.  A row permutation: CAS lambda (per input
// channel), PTS n and every row's codes are those of the plain [gate; up] stacking.
__global__ void k_interleave_gate_up(const uint4* __restrict__ wg, const uint4* __restrict__ wu, int64_t d_ff,
                                     int64_t vec_per_row, uint4* __restrict__ out) {
    const int64_t total = 2 * d_ff * vec_per_row;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t n = i / vec_per_row, v = i - n * vec_per_row;
        const int64_t t = n >> 7, r = n & 127;
        const int64_t j = t * 64 + (r & 63);
        out[i] = (r < 64 ? wg : wu)[j * vec_per_row + v];
    }
}

fireq_status_t interleave_gate_up_impl(const __nv_bfloat16* wg, const __nv_bfloat16* wu, int64_t d_ff,
                                       int64_t d_model, __nv_bfloat16* out, cudaStream_t stream) {
    const int64_t vpr = d_model / 8;
    const int64_t total = 2 * d_ff * vpr;
    const int blocks = (int)std::min<int64_t>(4096, (total + 255) / 256);
    k_interleave_gate_up<<<blocks, 256, 0, stream>>>(reinterpret_cast<const uint4*>(wg),
                                                      reinterpret_cast<const uint4*>(wu), d_ff, vpr,
                                                      reinterpret_cast<uint4*>(out));
    return check_launch("fireq_interleave_gate_up");
}

}  // namespace fireq
