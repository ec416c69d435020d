// quant_act.cu -- fireq_quantize_act (A1..A3, Eq. 2, per token P:482) and the
// FFN helper fireq_silu_mul_quantize_act (SiLU * up, then A2..A3).
//
// Decode-sized M (<= 64) and transposed inputs: one CTA per token row (k_act_quant): each
// thread keeps its 8-element vectors of x' in registers between the amax pass and the
// encode pass (the kernel can also split a row over a cluster of CTAs with a DSMEM amax
// reduction, used for transposed decode inputs only: at decode sizes the cluster launch and
// its two cluster barriers cost more latency than they save, measured).
// Large M, row-major: persistent CTAs with a TMA row ring and warp-pipelined passes
// (k_act_quant_rows, below).  Memory-bound: 2 B read + 1 B written per element (4 + 1 for
// SiLU*mul).  Launched with PDL.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

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

// q_div for a row whose beta is a normal fp32 number (the caller branches once per row).
__device__ __forceinline__ float q_div_normal(float x, float beta, float rcp) {
    const float q0 = __fmul_rn(x, rcp);
    const float e = __fmaf_rn(-q0, beta, x);
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

// x' (bf16 values, A1 / SiLU*mul) of 8 consecutive elements k..k+7, packed as 8 bf16, from
// the loaded raw vectors rx (X or gate) and ru (up, mode 2).
__device__ __forceinline__ uint4 xprime8_from(int mode, const __nv_bfloat16* c, uint4 rx, uint4 ru, int64_t k) {
    if (mode == 0) return rx;
    const __nv_bfloat16* hx = reinterpret_cast<const __nv_bfloat16*>(&rx);
    uint4 out;
    __nv_bfloat162* ho2 = reinterpret_cast<__nv_bfloat162*>(&out);
    if (mode == 1) {
        const uint4 rc = *reinterpret_cast<const uint4*>(c + k);
        const __nv_bfloat16* hc = reinterpret_cast<const __nv_bfloat16*>(&rc);
#pragma unroll
        for (int i = 0; i < 8; i += 2)
            ho2[i / 2] = __floats2bfloat162_rn(__fmul_rn(__bfloat162float(hx[i]), __bfloat162float(hc[i])),
                                               __fmul_rn(__bfloat162float(hx[i + 1]), __bfloat162float(hc[i + 1])));
    } else {
        const __nv_bfloat16* hu = reinterpret_cast<const __nv_bfloat16*>(&ru);
#pragma unroll
        for (int i = 0; i < 8; i += 2)      // SiLU: tolerance-checked (DESIGN R17)
            ho2[i / 2] = __floats2bfloat162_rn(__fmul_rn(silu_f(__bfloat162float(hx[i])), __bfloat162float(hu[i])),
                                               __fmul_rn(silu_f(__bfloat162float(hx[i + 1])), __bfloat162float(hu[i + 1])));
    }
    return out;
}

__device__ __forceinline__ uint4 xprime8(const Src& s, int64_t m, int64_t k) {
    const uint4 rx = load8_raw(s.X, s, m, k);
    const uint4 ru = s.mode == 2 ? load8_raw(s.U, s, m, k) : rx;
    return xprime8_from(s.mode, s.c, rx, ru, k);
}

// A3 for 8 consecutive elements: 8 E4M3 codes.  TINY: beta below the fp32 normal range
// (row-uniform; the caller picks the instantiation once per row).
template <bool TINY>
__device__ __forceinline__ uint2 encode8(uint4 xv, float beta, float rcp) {
    const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&xv);
    float q[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float v = __bfloat162float(h[i]);
        q[i] = TINY ? q_div(v, beta, rcp) : q_div_normal(v, beta, rcp);
    }
    uint2 o;
    o.x = e4m3x2_rn(q[0], q[1]) | (e4m3x2_rn(q[2], q[3]) << 16);
    o.y = e4m3x2_rn(q[4], q[5]) | (e4m3x2_rn(q[6], q[7]) << 16);
    return o;
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
        const bool tiny = beta < 0x1p-126f;
        if (threadIdx.x == 0 && rank == 0) beta_out[m] = beta_h;
        // A3: x_hat = E4M3_RN_satfinite(x' / beta).  The quotient from the reciprocal plus one
        // exact-residual FMA (q_div) rounds to the same E4M3 value as the IEEE quotient for
        // bf16 x' and beta (DESIGN reading R22) at a third of __fdiv_rn's instructions.
        auto encode_row = [&](auto tiny_c) {
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const int64_t k = k0 + ((int64_t)j * nt + threadIdx.x) * 8;
                if (k < k1)
                    *reinterpret_cast<uint2*>(xq + m * K + k) = encode8<decltype(tiny_c)::value>(xv[j], beta, rcp);
            }
        };
        if (tiny) encode_row(std::true_type{});
        else encode_row(std::false_type{});
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
// Large M, row-major rows: persistent CTAs (grid = SMs x resident CTAs), CTA b takes rows
// b, b + grid, ...  A producer warp streams each row into shared memory by one bulk copy per
// operand (TMA, evict-first: read once) through a ring of S stages; T / 32 consumer warps
// each own vectors v = j * T + tid of every row.  Per consumer warp, software-pipelined over
// rows with no CTA-wide barrier:
//   pass 1 of row i+1 (x' into registers, warp max -> red[], arrive on the row's max barrier;
//   arrive on the stage's empty barrier so the producer refills it), then
//   pass 2 of row i (wait for row i's max barrier, combine the warp maxima, beta, encode, store).
// The one-CTA-per-row kernel (k_act_quant) reached 50-59% of HBM here; a barrier-per-row
// version of this ring stalled on its two __syncthreads per row (ncu: "barrier" first).
// Arithmetic: xprime_pair / encode_pair, bitwise the values of xprime8_from / encode8.
constexpr int kRowMaxStages = 8;
constexpr uint32_t kRowSmemMax = 200 * 1024 / 2;     // the largest ring: T = 512, two CTAs per SM

// Lean per-pair arithmetic (bf16 pairs unpacked with one integer op each, fp32 pairs on the
// packed FMUL2 / FFMA2 / FADD2 path); the row max is taken on the fp32 products before their
// bf16 rounding (RN is monotonic and odd, so max |bf16(p)| = bf16(max |p|): rounded per row).
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t pack_bf2(float2 p) {
    const __nv_bfloat162 b = __floats2bfloat162_rn(p.x, p.y);
    return *reinterpret_cast<const uint32_t*>(&b);
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(addr));
    return r;
}
// x' of one pair and its contribution to the (unrounded) row max.
template <int MODE>
__device__ __forceinline__ uint32_t xprime_pair(uint32_t x, uint32_t c_or_u, float& pmax) {
    if (MODE == 0) {
        pmax = fmaxf(pmax, fmaxf(fabsf(bf_lo(x)), fabsf(bf_hi(x))));
        return x;
    }
    float2 p;
    if (MODE == 1) {
        p = __fmul2_rn(make_float2(bf_lo(x), bf_hi(x)), make_float2(bf_lo(c_or_u), bf_hi(c_or_u)));
    } else {
        const float2 g = make_float2(bf_lo(x), bf_hi(x));
        const float2 t = __fmul2_rn(g, make_float2(-1.4426950408889634f, -1.4426950408889634f));
        const float2 d = __fadd2_rn(make_float2(1.0f, 1.0f), make_float2(ex2_ftz(t.x), ex2_ftz(t.y)));
        const float2 sl = __fmul2_rn(g, make_float2(rcp_ftz(d.x), rcp_ftz(d.y)));
        p = __fmul2_rn(sl, make_float2(bf_lo(c_or_u), bf_hi(c_or_u)));
    }
    pmax = fmaxf(pmax, fmaxf(fabsf(p.x), fabsf(p.y)));
    return pack_bf2(p);
}
// A3 of one pair (beta a normal fp32 number): two E4M3 codes, (hi << 8) | lo.
__device__ __forceinline__ uint32_t encode_pair(uint32_t w, float2 beta_neg2, float2 rcp2) {
    const float2 v = make_float2(bf_lo(w), bf_hi(w));
    const float2 q0 = __fmul2_rn(v, rcp2);
    const float2 e = __ffma2_rn(q0, beta_neg2, v);          // x - q0 * beta, exact residual
    const float2 q = __ffma2_rn(e, rcp2, q0);
    // x = -0: keep its sign (see q_div)
    return e4m3x2_rn(__uint_as_float(__float_as_uint(q.x) | ((w << 16) & 0x80000000u)),
                     __uint_as_float(__float_as_uint(q.y) | (w & 0x80000000u)));
}

template <int MODE, int R, int T>
__global__ void __launch_bounds__(T + 32, T == 128 ? 6 : 1024 / T) k_act_quant_rows(Src s, int64_t M, int64_t K, int S,
                                                                        uint8_t* __restrict__ xq,
                                                                        __nv_bfloat16* __restrict__ beta_out,
                                                                        unsigned long long* span) {
    constexpr int NW = T / 32;                 // consumer warps; warp NW is the producer
    extern __shared__ __align__(128) uint8_t ring[];
    __shared__ uint64_t full[kRowMaxStages], empty[kRowMaxStages], maxbar[2];
    __shared__ float red[4][NW];
    span_begin(span);
    const uint32_t rowb = (uint32_t)(K * 2);
    const uint32_t stage_bytes = (MODE == 2 ? 2 : 1) * rowb;
    const int vecs = (int)(K / 8);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            ptx::mbar_init(&full[i], 1);
            ptx::mbar_init(&empty[i], NW);
        }
        ptx::mbar_init(&maxbar[0], NW);
        ptx::mbar_init(&maxbar[1], NW);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    ptx::pdl_trigger();
    ptx::pdl_wait();                           // X / G / U come from the previous kernel
    const int64_t G = gridDim.x;
    if (warp == NW) {                          // producer
        if (lane == 0) {
            const uint64_t pol = ptx::policy_evict_first();
            int n = 0;
            for (int64_t row = blockIdx.x; row < M; row += G, ++n) {
                const int slot = n % S;
                if (n >= S) ptx::mbar_wait(&empty[slot], (uint32_t)(((n / S) - 1) & 1));
                uint8_t* dst = ring + (size_t)slot * stage_bytes;
                ptx::mbar_arrive_expect_tx(&full[slot], stage_bytes);
                ptx::bulk_g2s(dst, s.X + row * s.ld, rowb, &full[slot], pol);
                if (MODE == 2) ptx::bulk_g2s(dst + rowb, s.U + row * s.ld, rowb, &full[slot], pol);
            }
        }
        span_end(span);
        return;
    }
    const uint32_t ring_u32 = ptx::smem_u32(ring);
    // pass 1 of the n-th row of this CTA into xv; publishes the warp max
    auto pass1 = [&](int n, uint4 (&xv)[R]) {
        const int slot = n % S;
        ptx::mbar_wait(&full[slot], (uint32_t)((n / S) & 1));
        const uint32_t st = ring_u32 + (uint32_t)slot * stage_bytes;
        float pmax = 0.0f;
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int v = j * T + (int)threadIdx.x;
            if (v < vecs) {
                const uint4 rx = lds128(st + (uint32_t)v * 16);
                const uint4 ru = MODE == 2 ? lds128(st + rowb + (uint32_t)v * 16)
                               : MODE == 1 ? __ldg(reinterpret_cast<const uint4*>(s.c) + v) : rx;   // c: L1-resident
                xv[j].x = xprime_pair<MODE>(rx.x, ru.x, pmax);
                xv[j].y = xprime_pair<MODE>(rx.y, ru.y, pmax);
                xv[j].z = xprime_pair<MODE>(rx.z, ru.z, pmax);
                xv[j].w = xprime_pair<MODE>(rx.w, ru.w, pmax);
            }
        }
        for (int o = 16; o; o >>= 1) pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
        __syncwarp();                          // every lane is done reading the stage
        if (lane == 0) {
            red[n & 3][warp] = pmax;
            ptx::mbar_arrive(&empty[slot]);
            ptx::mbar_arrive(&maxbar[n & 1]);  // release: red[] is visible to the waiters
        }
    };
    // pass 2 of the n-th row (m) from xv
    auto pass2 = [&](int n, int64_t m, const uint4 (&xv)[R]) {
        ptx::mbar_wait(&maxbar[n & 1], (uint32_t)((n >> 1) & 1));
        float pm = lane < NW ? red[n & 3][lane] : 0.0f;
        for (int o = 16; o; o >>= 1) pm = fmaxf(pm, __shfl_xor_sync(0xffffffffu, pm, o));
        // the row max of |x'| = bf16_RN(max |p|) (mode 0: already a bf16 value)
        const float amax = MODE == 0 ? pm : __bfloat162float(__float2bfloat16_rn(pm));
        // A2 / A3 exactly as k_act_quant
        const __nv_bfloat16 beta_h = amax > 0.0f ? __float2bfloat16_rn(__fdiv_rn(amax, 448.0f))
                                                 : __float2bfloat16_rn(1.0f);
        const float beta = __bfloat162float(beta_h);
        const float rcp = __frcp_rn(beta);
        if (threadIdx.x == 0) beta_out[m] = beta_h;
        uint8_t* xrow = xq + m * K;
        if (beta < 0x1p-126f) {               // row-uniform: the IEEE-quotient path of q_div
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const int v = j * T + (int)threadIdx.x;
                if (v < vecs) *reinterpret_cast<uint2*>(xrow + v * 8) = encode8<true>(xv[j], beta, rcp);
            }
        } else {
            const float2 bn2 = make_float2(-beta, -beta), r2 = make_float2(rcp, rcp);
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const int v = j * T + (int)threadIdx.x;
                if (v < vecs) {
                    uint2 o;
                    o.x = encode_pair(xv[j].x, bn2, r2) | (encode_pair(xv[j].y, bn2, r2) << 16);
                    o.y = encode_pair(xv[j].z, bn2, r2) | (encode_pair(xv[j].w, bn2, r2) << 16);
                    *reinterpret_cast<uint2*>(xrow + v * 8) = o;
                }
            }
        }
    };
    // red[n & 3] is rewritten by row n + 4 only after every warp arrived for row n + 3, i.e.
    // after every warp finished pass 2 of row n + 2 > n; maxbar[n & 1]'s next phase (row n + 2)
    // cannot complete before this warp arrives for it, after its pass 2 of row n.
    uint4 xa[R], xb[R];
    int64_t m = blockIdx.x;
    int n = 0;
    if (m < M) pass1(0, xa);
    while (m < M) {
        const int64_t m1 = m + G;
        if (m1 < M) pass1(n + 1, xb);
        pass2(n, m, xa);
        m = m1;
        ++n;
        if (m >= M) break;
        const int64_t m2 = m + G;
        if (m2 < M) pass1(n + 1, xa);
        pass2(n, m, xb);
        m = m2;
        ++n;
    }
    span_end(span);
}

template <int MODE, int R, int T>
cudaError_t launch_rows(const Src& s, int64_t M, int64_t K, int S, uint32_t smem, uint8_t* xq,
                        __nv_bfloat16* beta, cudaStream_t stream) {
    auto kern = k_act_quant_rows<MODE, R, T>;
    cudaError_t e;
    int dev = 0, sms = 0, per_sm = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    // the ring never exceeds kRowSmemMax: raise the dynamic shared memory limit once per device
    static uint32_t smem_set[64] = {};
    if (dev < 0 || dev >= 64 || smem_set[dev] < smem) {
        if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRowSmemMax)) != cudaSuccess)
            return e;
        if (dev >= 0 && dev < 64) smem_set[dev] = kRowSmemMax;
    }
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T + 32, smem)) != cudaSuccess) return e;
    const int64_t grid = std::min<int64_t>(M, (int64_t)sms * std::max(per_sm, 1));
    return launch_ex(kern, dim3((unsigned)grid), dim3(T + 32), smem, stream, 1u, false, s, M, K, S, xq, beta,
                     next_span_slot());
}

template <int MODE, int T>
cudaError_t launch_rows_r(const Src& s, int64_t M, int64_t K, int S, uint32_t smem, uint8_t* xq,
                          __nv_bfloat16* beta, cudaStream_t stream) {
    const int64_t per = (K / 8 + T - 1) / T;
    if (per <= 1) return launch_rows<MODE, 1, T>(s, M, K, S, smem, xq, beta, stream);
    if (per <= 2) return launch_rows<MODE, 2, T>(s, M, K, S, smem, xq, beta, stream);
    if (per <= 3) return launch_rows<MODE, 3, T>(s, M, K, S, smem, xq, beta, stream);
    return launch_rows<MODE, 4, T>(s, M, K, S, smem, xq, beta, stream);
}

template <int MODE>
cudaError_t launch_rows_t(int T, const Src& s, int64_t M, int64_t K, int S, uint32_t smem, uint8_t* xq,
                          __nv_bfloat16* beta, cudaStream_t stream) {
    if (T == 128) return launch_rows_r<MODE, 128>(s, M, K, S, smem, xq, beta, stream);
    return launch_rows_r<MODE, 512>(s, M, K, S, smem, xq, beta, stream);
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
    // large M, row-major: the persistent TMA-ring kernel.  T consumer threads (+ a producer
    // warp) per CTA, 1024 / T CTAs per SM, at most 4 vectors per thread (K <= 16384); S
    // stages of a row in 200 KB / (1024 / T) of shared memory.
    static const bool rows_off = getenv("FIREQ_ACT_ROWS_OFF") != nullptr;     // A/B switch
    static const int rows_t = getenv("FIREQ_ACT_ROWS_T") ? atoi(getenv("FIREQ_ACT_ROWS_T")) : 0;
    if (!transposed && M > 64 && !rows_off) {
        const int64_t stage_bytes = (mode == 2 ? 4 : 2) * K;
        const int64_t vecs = K / 8;
        int T = rows_t == 128 || rows_t == 512 ? rows_t : (mode == 2 ? 512 : 128);
        if ((vecs + T - 1) / T > 4) T = 512;
        const int64_t budget = (200 * 1024) / (T == 128 ? 6 : 1024 / T);
        const int S = (int)std::min<int64_t>(kRowMaxStages, budget / stage_bytes);
        if ((vecs + T - 1) / T <= 4 && S >= 2) {
            const uint32_t smem = (uint32_t)(S * stage_bytes);
            cudaError_t e = mode == 0 ? launch_rows_t<0>(T, s, M, K, S, smem, xq, beta, stream)
                          : mode == 1 ? launch_rows_t<1>(T, s, M, K, S, smem, xq, beta, stream)
                                      : launch_rows_t<2>(T, s, M, K, S, smem, xq, beta, stream);
            if (e != cudaSuccess) return fail(FIREQ_ERROR_CUDA, std::string("act quant launch: ") + cudaGetErrorString(e));
            return check_launch(mode == 2 ? "fireq_silu_mul_quantize_act" : "fireq_quantize_act");
        }
    }
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
