// gemm_dev.cuh -- device building blocks shared by the W4A8 GEMM (gemm.cu) and the
// persistent decode FFN (ffn_decode.cu): tile constants, the UMMA descriptors, the
// INT4 -> FP8 LUT converters (Step 1) and the E4M3 activation encoder (A3).
#pragma once
#include <cstdint>
#include <cuda.h>

#include "common.cuh"
#include "ptx.cuh"

namespace fireq {
namespace dev {

constexpr int kGroup = 128;            // K per group (one FP8 scale)
constexpr int kTileN = 128;            // weight rows per tile = MMA M
constexpr int kWBytes = kTileN * kGroup / 2;   // 8192 packed bytes per (tile, group)
constexpr int kLutEntries = 127 * 16;
constexpr int kMaxDevices = 64;

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row core groups 1024 B apart.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;                  // LBO (unused for swizzled K-major) = 16 B
    d |= (uint64_t)(1024 >> 4) << 32;        // SBO = 1024 B
    d |= (uint64_t)1 << 46;                  // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;                  // SWIZZLE_128B
    return d;
}

// Instruction descriptor, kind::f8f6f4: E4M3 x E4M3 -> F32, K-major A and B, M = 128.
__host__ __device__ constexpr uint32_t make_idesc(int ntok, bool negate_a) {
    return (1u << 4)                          // D format F32
         | (0u << 7) | (0u << 10)             // A, B = E4M3
         | ((negate_a ? 1u : 0u) << 13)
         | ((uint32_t)(ntok >> 3) << 17)      // N >> 3
         | ((uint32_t)(128 >> 4) << 24);      // M >> 4
}

// 16 output bytes pair (lo/hi word) per input word, sign-split.
__device__ __forceinline__ void conv_sign_split(uint32_t w, uint32_t L0, uint32_t L1, uint32_t N0, uint32_t N1,
                                                uint32_t& p0, uint32_t& p1, uint32_t& n0, uint32_t& n1) {
    const uint32_t x = w ^ 0x88888888u;
    const uint32_t wh = ptx::hi16_prmt(w);      // byte permute: full ALU rate (IMAD.HI: half rate)
    const uint32_t xh = ptx::hi16_prmt(x);
    p0 = ptx::prmt(L0, L1, w);
    p1 = ptx::prmt(L0, L1, wh);
    n0 = ptx::prmt(N0, N1, x);
    n1 = ptx::prmt(N0, N1, xh);
}

__device__ __forceinline__ void conv_mask_select(uint32_t w, uint32_t L0, uint32_t L1, uint32_t L2, uint32_t L3,
                                                 uint32_t& r0, uint32_t& r1) {
    const uint32_t x = w ^ 0x88888888u;
    const uint32_t t = ptx::shl4_fma(w);
    const uint32_t wh = ptx::hi16_prmt(w);
    const uint32_t xh = ptx::hi16_prmt(x);
    const uint32_t m0 = ptx::prmt(w, t, 0x9D8Cu);     // 0xFF where nibble 0..3 is negative
    const uint32_t m1 = ptx::prmt(w, t, 0xBFAEu);     // nibbles 4..7
    r0 = ptx::lop3_mux(ptx::prmt(L0, L1, w), ptx::prmt(L2, L3, x), m0);
    r1 = ptx::lop3_mux(ptx::prmt(L0, L1, wh), ptx::prmt(L2, L3, xh), m1);
}

// x / beta -> E4M3 (A3) with the quotient x' / beta correctly rounded to fp32 (as
// __fdiv_rn) from the reciprocal: q0 = x' * rcp, one exact-residual correction.  The
// corrected quotient is exact whenever x' / beta is representable, otherwise within
// 1 ulp; a quotient of two 8-bit-significand numbers that is not exactly an E4M3
// midpoint lies > 2^-13 relative away from every midpoint, so the E4M3 rounding equals
// that of the correctly rounded quotient (reading R23).
// Out of line: the IEEE division is a long instruction sequence, and an inlined copy per
// element bloats the kernels' cold paths (instruction-cache misses on every launch).
static __device__ __noinline__ float fdiv_rn_slow(float x, float beta) { return __fdiv_rn(x, beta); }
__device__ __forceinline__ float div_for_e4m3(float x, float beta, float rcp) {
    if (beta < 0x1p-126f) return fdiv_rn_slow(x, beta);   // subnormal beta: 1/beta may overflow
    const float q0 = __fmul_rn(x, rcp);
    const float e = __fmaf_rn(-q0, beta, x);
    // x = -0: the correction's +0 would lose the sign; OR-ing x's sign bit is a no-op otherwise
    // (beta > 0, so a nonzero or underflowed quotient already carries x's sign)
    return __int_as_float(__float_as_int(__fmaf_rn(e, rcp, q0)) | (__float_as_int(x) & 0x80000000));
}

// LUT-of-LUTs in shared memory: entry [s][u] = E4M3_RN(v(u) * sigma_s), v(u) = u < 8 ? u : u - 16,
// for all 127 finite non-negative sigma codes s (Step 1's 16-entry table).  v * sigma is
// exact in fp32.  Threads t0, t0 + stride, ... of the calling group fill it.
__device__ __forceinline__ void build_lut(uint8_t* lut, int t0, int stride) {
    for (int e = t0; e < kLutEntries; e += stride) {
        const int s = e >> 4, u = e & 15;
        const float v = (float)(u < 8 ? u : u - 16);
        lut[e] = (uint8_t)e4m3_rn(__fmul_rn(v, e4m3_decode((uint32_t)s)));
    }
}

}  // namespace dev

// host: 2-D TMA descriptor of an E4M3 activation matrix [M][K] with (K-box 128, row-box ntok)
// boxes and the 128-B swizzle of the UMMA K-major operand; cached (fireq_clear_cache).
bool make_x_map(CUtensorMap* out, const uint8_t* x, int64_t M, int64_t K, int ntok);

}  // namespace fireq
