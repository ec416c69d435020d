// quant_act.cu -- fireq_quantize_act (A1..A3, Eq. 2, per token P:482) and the
// FFN helper fireq_silu_mul_quantize_act (SiLU * up, then A2..A3).
//
// One CTA per token row: each thread keeps its 8-element vectors of x' in registers between
// the amax pass and the encode pass (the kernel can also split a row over a cluster of CTAs
// with a DSMEM amax reduction, but the launcher uses CL = 1: at decode sizes the cluster
// launch and its two cluster barriers cost more latency than they save, measured).
// Memory-bound: 2 B read + 1 B written per element.  Launched with PDL.
#include <algorithm>

#include "common.cuh"
#include "ptx.cuh"

namespace fireq {
namespace {

constexpr int kThreads = 256;

// x / beta for the E4M3 encode: q0 = x * rcp(beta), one exact-residual correction (as the
// SwiGLU tail of gemm.cu); see DESIGN reading R22 for why the E4M3 rounding is unchanged.
__device__ __forceinline__ float q_div(float x, float beta, float rcp) {
    // beta below the fp32 normal range: 1/beta may overflow (and its residual lose bits), so
    // use the IEEE quotient (warp-uniform: one beta per row)
    if (beta < 0x1p-126f) return __fdiv_rn(x, beta);
    const float q0 = __fmul_rn(x, rcp);
    const float e = __fmaf_rn(-q0, beta, x);
    // x = -0: the correction's +0 would lose the sign; OR-ing x's sign bit is a no-op otherwise
    // (beta > 0, so a nonzero or underflowed quotient already carries x's sign)
    return __int_as_float(__float_as_int(__fmaf_rn(e, rcp, q0)) | (__float_as_int(x) & 0x80000000));
}

__device__ __forceinline__ float block_max(float v, float* red) {
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        v = l < (int)(blockDim.x >> 5) ? red[l] : 0.0f;
        for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (l == 0) red[0] = v;
    }
    __syncthreads();
    return red[0];
}

// x' for 8 consecutive elements (A1): bf16(x * c) when c is given (product exact in fp32).
struct Src {
    const __nv_bfloat16* X;
    const __nv_bfloat16* U;   // silu-mul mode: X = gate, U = up
    const __nv_bfloat16* c;
    int mode;                 // 0 = plain, 1 = channel multiplier, 2 = silu(g) * u
    int transposed;           // element (m, k) at X[k * ld + m] (Y^T of the column-parallel GEMM)
    int64_t ld;
};

// 8 consecutive k of row m; row-major rows are loaded as one 16-B vector, transposed
// inputs element by element (decode-sized M only).
__device__ __forceinline__ uint4 load8_raw(const __nv_bfloat16* base, const Src& s, int64_t m, int64_t k) {
    if (!s.transposed) return *reinterpret_cast<const uint4*>(base + m * s.ld + k);
    uint4 r;
    __nv_bfloat16* h = reinterpret_cast<__nv_bfloat16*>(&r);
#pragma unroll
    for (int i = 0; i < 8; ++i) h[i] = base[(k + i) * s.ld + m];
    return r;
}

// x' (bf16 values, A1 / SiLU*mul) of 8 consecutive elements, packed as 8 bf16.
__device__ __forceinline__ uint4 xprime8(const Src& s, int64_t m, int64_t k) {
    const uint4 rx = load8_raw(s.X, s, m, k);
    if (s.mode == 0) return rx;
    const __nv_bfloat16* hx = reinterpret_cast<const __nv_bfloat16*>(&rx);
    uint4 out;
    __nv_bfloat16* ho = reinterpret_cast<__nv_bfloat16*>(&out);
    if (s.mode == 1) {
        const uint4 rc = *reinterpret_cast<const uint4*>(s.c + k);
        const __nv_bfloat16* hc = reinterpret_cast<const __nv_bfloat16*>(&rc);
#pragma unroll
        for (int i = 0; i < 8; ++i)
            ho[i] = __float2bfloat16_rn(__fmul_rn(__bfloat162float(hx[i]), __bfloat162float(hc[i])));
    } else {
        const uint4 ru = load8_raw(s.U, s, m, k);
        const __nv_bfloat16* hu = reinterpret_cast<const __nv_bfloat16*>(&ru);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float g = __bfloat162float(hx[i]);
            const float silu = __fdividef(g, 1.0f + __expf(-g));     // SiLU: tolerance-checked (DESIGN R17)
            ho[i] = __float2bfloat16_rn(__fmul_rn(silu, __bfloat162float(hu[i])));
        }
    }
    return out;
}

// Grid (CL, rows), cluster (CL, 1, 1): CTA `rank` of a cluster quantizes columns
// [rank*K/CL, (rank+1)*K/CL) of token row m; with CL > 1 the row amax is combined across
// the cluster through distributed shared memory (DSMEM).  The launcher uses CL = 1.  Each
// thread keeps its (at most R) 8-element vectors of x' in registers between the passes.
// MINB > 1 (large M): at most 512 threads and >= MINB resident CTAs per SM, so the compiler
// keeps <= 32 registers and enough rows are in flight (with 1024 possible threads it chose 59
// registers: 2 CTAs per SM, 29% of HBM bandwidth on 16384 x 11008, measured)
template <int R, int MINB>
__global__ void __launch_bounds__(MINB > 1 ? 512 : 1024, MINB) k_act_quant(Src s, int64_t M, int64_t K, int cl,
                                                   uint8_t* __restrict__ xq,
                                                   __nv_bfloat16* __restrict__ beta_out,
                                                   unsigned long long* span) {
    __shared__ float red[32];
    span_begin(span);
    ptx::pdl_trigger();
    ptx::pdl_wait();                       // X / G / U come from the previous kernel
    const int rank = cl > 1 ? (int)ptx::cluster_ctarank() : 0;
    const int64_t chunk = K / cl;
    const int64_t k0 = rank * chunk, k1 = k0 + chunk;
    const int nt = blockDim.x;
    for (int64_t m = blockIdx.y; m < M; m += gridDim.y) {
        uint4 xv[R];
        float amax = 0.0f;
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int64_t k = k0 + ((int64_t)j * nt + threadIdx.x) * 8;
            if (k < k1) {
                xv[j] = xprime8(s, m, k);
                const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&xv[j]);
#pragma unroll
                for (int i = 0; i < 8; ++i) amax = fmaxf(amax, fabsf(__bfloat162float(h[i])));
            }
        }
        amax = block_max(amax, red);           // red[0] = this CTA's max
        if (cl > 1) {
            ptx::cluster_sync();               // every CTA's red[0] is written
            if (threadIdx.x < 32) {
                float v = 0.0f;
                if (threadIdx.x < (unsigned)cl)
                    v = ptx::ld_shared_cluster_f32(ptx::mapa_shared(ptx::smem_u32(&red[0]), threadIdx.x));
                for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
                if (threadIdx.x == 0) red[1] = v;
            }
            ptx::cluster_sync();               // remote reads done before any CTA moves on / exits
            amax = red[1];
        }
        // A2: beta = bf16_RN(amax / 448) (fp32 division then RNE; equals exact RNE for bf16 operands)
        const __nv_bfloat16 beta_h = amax > 0.0f ? __float2bfloat16_rn(__fdiv_rn(amax, 448.0f))
                                                 : __float2bfloat16_rn(1.0f);
        const float beta = __bfloat162float(beta_h);
        const float rcp = __frcp_rn(beta);
        if (threadIdx.x == 0 && rank == 0) beta_out[m] = beta_h;
        // A3: x_hat = E4M3_RN_satfinite(x' / beta).  The quotient from the reciprocal plus one
        // exact-residual FMA (q_div) rounds to the same E4M3 value as the IEEE quotient for
        // bf16 x' and beta (DESIGN reading R22) at a third of __fdiv_rn's instructions.
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int64_t k = k0 + ((int64_t)j * nt + threadIdx.x) * 8;
            if (k < k1) {
                const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&xv[j]);
                float v[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] = __bfloat162float(h[i]);
                uint2 o;
                o.x = e4m3x2_rn(q_div(v[0], beta, rcp), q_div(v[1], beta, rcp)) |
                      (e4m3x2_rn(q_div(v[2], beta, rcp), q_div(v[3], beta, rcp)) << 16);
                o.y = e4m3x2_rn(q_div(v[4], beta, rcp), q_div(v[5], beta, rcp)) |
                      (e4m3x2_rn(q_div(v[6], beta, rcp), q_div(v[7], beta, rcp)) << 16);
                *reinterpret_cast<uint2*>(xq + m * K + k) = o;
            }
        }
        __syncthreads();                       // red[] reuse by the next row
    }
    span_end(span);
}

template <int R, int MINB>
cudaError_t launch_act(const Src& s, int64_t M, int64_t K, int cl, int threads, uint8_t* xq, __nv_bfloat16* beta,
                       cudaStream_t stream) {
    const unsigned rows = (unsigned)std::min<int64_t>(M, 65535);
    return launch_ex(k_act_quant<R, MINB>, dim3((unsigned)cl, rows), dim3(threads), 0, stream, (unsigned)cl, false, s, M, K, cl,
                     xq, beta, next_span_slot());
}

// ---------------------------------------------------------------------------------------
// Transposed inputs at large M (the column-parallel path's Y^T, element (m, k) at X[k * ld + m]):
// one CTA per block of 32 tokens (256 threads: warp w reads rows k = w, w + 8, ..., 64 contiguous
// bytes each; 128-token CTAs measured 3x slower -- too few CTAs in flight).  Pass 1:
// per-token max |x'| (A2); pass 2 re-reads, encodes (A3) into a shared [128 tokens][64 k] tile
// and writes each token's 64 codes as 16-byte stores.  x' (A1 / SiLU*mul) is formed exactly as
// in k_act_quant.
constexpr int kTT = 32;        // tokens per CTA
constexpr int kTK = 64;        // rows per pass-2 chunk
constexpr int kTRow = 8;       // row interleave (256 threads = 32 tokens x 8 rows)
__device__ __forceinline__ float xprime_t(const Src& s, int64_t m, int64_t k) {
    const float x = __bfloat162float(s.X[k * s.ld + m]);
    if (s.mode == 0) return x;
    if (s.mode == 1) return __bfloat162float(__float2bfloat16_rn(__fmul_rn(x, __bfloat162float(s.c[k]))));
    const float u = __bfloat162float(s.U[k * s.ld + m]);
    const float silu = __fdividef(x, 1.0f + __expf(-x));
    return __bfloat162float(__float2bfloat16_rn(__fmul_rn(silu, u)));
}

__global__ void __launch_bounds__(256) k_act_quant_t(Src s, int64_t M, int64_t K, uint8_t* __restrict__ xq,
                                                     __nv_bfloat16* __restrict__ beta_out) {
    __shared__ float red[kTRow][kTT];
    __shared__ float sb[2][kTT];
    __shared__ __align__(16) uint8_t tile[kTT][kTK];
    ptx::pdl_trigger();
    ptx::pdl_wait();
    const int tl = threadIdx.x & (kTT - 1), kr = threadIdx.x / kTT;     // token in block, row phase
    const int64_t m = (int64_t)blockIdx.x * kTT + tl;
    const bool valid = m < M;
    float amax = 0.0f;
    if (valid)
        for (int64_t k = kr; k < K; k += kTRow) amax = fmaxf(amax, fabsf(xprime_t(s, m, k)));
    red[kr][tl] = amax;
    __syncthreads();
    if (kr == 0) {
        float v = red[0][tl];
#pragma unroll
        for (int q = 1; q < kTRow; ++q) v = fmaxf(v, red[q][tl]);
        const __nv_bfloat16 bh = v > 0.0f ? __float2bfloat16_rn(__fdiv_rn(v, 448.0f)) : __float2bfloat16_rn(1.0f);
        sb[0][tl] = __bfloat162float(bh);
        sb[1][tl] = __frcp_rn(__bfloat162float(bh));
        if (valid) beta_out[m] = bh;
    }
    __syncthreads();
    const float beta = sb[0][tl], rcp = sb[1][tl];
    for (int64_t k0 = 0; k0 < K; k0 += kTK) {
#pragma unroll 4
        for (int kk = kr; kk < kTK; kk += kTRow) {
            const float v = valid ? q_div(xprime_t(s, m, k0 + kk), beta, rcp) : 0.0f;
            tile[tl][kk] = (uint8_t)(e4m3x2_rn(v, 0.0f) & 0xFFu);
        }
        __syncthreads();
        // 32 tokens x 64 codes = 128 16-byte pieces
        if (threadIdx.x < kTT * kTK / 16) {
            const int t = threadIdx.x >> 2, piece = threadIdx.x & 3;
            const int64_t mt = (int64_t)blockIdx.x * kTT + t;
            if (mt < M)
                *reinterpret_cast<uint4*>(xq + mt * K + k0 + piece * 16) =
                    *reinterpret_cast<const uint4*>(&tile[t][piece * 16]);
        }
        __syncthreads();
    }
}

}  // namespace

fireq_status_t quantize_act_impl(const __nv_bfloat16* X, const __nv_bfloat16* U, int64_t M, int64_t K,
                                 int64_t ld, const __nv_bfloat16* c, int mode, bool transposed, uint8_t* xq,
                                 __nv_bfloat16* beta, cudaStream_t stream) {
    Src s{X, U, c, mode, transposed ? 1 : 0, ld};
    if (transposed && M >= 64) {
        const cudaError_t e = launch_ex(k_act_quant_t, dim3((unsigned)((M + kTT - 1) / kTT)), dim3(256), 0, stream, 1u,
                                        false, s, M, K, xq, beta);
        if (e != cudaSuccess) return fail(FIREQ_ERROR_CUDA, std::string("act quant launch: ") + cudaGetErrorString(e));
        return check_launch(mode == 2 ? "fireq_silu_mul_quantize_act_t" : "fireq_quantize_act_t");
    }
    // One CTA per token row (a cluster/DSMEM split of the row measured slower at decode:
    // cluster launch + two cluster barriers cost more latency than they save).
    // (transposed decode inputs read 2-byte elements at a stride of M: split each row over a
    // cluster of 8 CTAs so that 8x more loads are in flight)
    const int cl = (transposed && (K / 8) % 8 == 0) ? 8 : 1;
    const int64_t vecs = (K / cl + 7) / 8;
    // decode-sized M: as many threads as vectors (<= 2 per thread); large M: <= 4 per thread
    const int64_t want = M <= 64 ? (vecs + 1) / 2 : (vecs + 3) / 4;
    const bool big = M > 64;
    const int threads = (int)std::min<int64_t>(big ? 512 : 1024, std::max<int64_t>(128, (want + 31) / 32 * 32));
    const int64_t per = (vecs + threads - 1) / threads;
    cudaError_t e;
    if (big) {
        if (per <= 2) e = launch_act<2, 4>(s, M, K, cl, threads, xq, beta, stream);
        else if (per <= 4) e = launch_act<4, 3>(s, M, K, cl, threads, xq, beta, stream);
        else if (per <= 8) e = launch_act<8, 2>(s, M, K, cl, threads, xq, beta, stream);
        else if (per <= 16) e = launch_act<16, 1>(s, M, K, cl, threads, xq, beta, stream);
        else e = launch_act<32, 1>(s, M, K, cl, threads, xq, beta, stream);
    } else if (per <= 1) e = launch_act<1, 1>(s, M, K, cl, threads, xq, beta, stream);
    else if (per <= 2) e = launch_act<2, 1>(s, M, K, cl, threads, xq, beta, stream);
    else if (per <= 4) e = launch_act<4, 1>(s, M, K, cl, threads, xq, beta, stream);
    else if (per <= 8) e = launch_act<8, 1>(s, M, K, cl, threads, xq, beta, stream);
    else if (per <= 16) e = launch_act<16, 1>(s, M, K, cl, threads, xq, beta, stream);
    else e = launch_act<32, 1>(s, M, K, cl, threads, xq, beta, stream);
    if (e != cudaSuccess) return fail(FIREQ_ERROR_CUDA, std::string("act quant launch: ") + cudaGetErrorString(e));
    return check_launch(mode == 2 ? "fireq_silu_mul_quantize_act" : "fireq_quantize_act");
}

}  // namespace fireq
