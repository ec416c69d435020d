// gemm_bf16s.cu -- fireq_w4a8_gemm_bf16s: the sigma_BF16 comparison variant of the linear
// layer ("we include a comparison using BF16 scaling factors (sigma_BF16)", App. B.1
// P:525-527; DESIGN reading R25).
//
// With a BF16 group scale the dequantized weight code * sigma is not an FP8 value, so the
// scale cannot be folded into the converter's lookup table: the tensor core multiplies the
// raw INT4 codes (exact in E4M3) with x_hat, ONE 128-K group at a time, and CUDA cores scale
// each group's FP32 partial by its row's sigma and accumulate (per-group scaled accumulation):
//   acc[m][n] = sum_g sigma_{n,g} * (sum_{k in g} dec(x_hat[m][k]) * code[n][k])     (FP32)
//   y[m][n]   = bf16_RN(acc[m][n] * beta_m * 2^-pts)
// That per-group round trip through TMEM and the CUDA cores is the variant's cost (the paper
// measured ~0.6x the sigma_FP8 kernel's FFN throughput on H100).
//
// Grid (n_tiles * S, m_tiles): CTA (t, s, mt) runs tile t over the groups [s G / S, (s+1) G / S)
// for tokens [mt NTOK, +NTOK); partials [S][M][N] fp32 are summed in s order by a second kernel.
// Roles: converter warpgroup (codes -> E4M3 integers, sign-split, into 3 TMEM A slots), scaler
// warpgroup (TMEM partial x sigma -> FP32 running sum in registers), weight / activation TMA
// producers, MMA issuer.
#include <algorithm>

#include "common.cuh"
#include "gemm_dev.cuh"
#include "ptx.cuh"

namespace fireq {
using namespace dev;
namespace {

constexpr int STAGES = 8;                 // one group per stage
constexpr int ASL = 3;                    // TMEM A slots (sign-split, 64 columns each; 256 allocated)
constexpr int kThreads = 128 + 128 + 96;  // converters, scaler, W / X producers + MMA issuer

template <int NTOK>
struct CfgB {
    static constexpr int kX = NTOK * kGroup;                         // activation tile per group
    static constexpr int kOffX = 0;
    static constexpr int kOffW = kOffX + STAGES * kX;
    static constexpr int kOffS = kOffW + STAGES * kWBytes;
    static constexpr int kOffSig = kOffS + STAGES * kTileN * 2;      // [8][128] fp32 sigma ring
    static constexpr int kOffBar = kOffSig + 8 * kTileN * 4;
    static constexpr int kNumBars = 3 * STAGES + ASL + 4;
    static constexpr int kOffMisc = kOffBar + kNumBars * 8;
    static constexpr int kSmem = kOffMisc + 16 + 1024;
    static constexpr int kAcc0 = 0;                                   // 2 accumulators of NTOK columns
    static constexpr int kA0 = 64;
    static_assert(kA0 >= 2 * NTOK && kA0 + ASL * 64 <= 256, "TMEM budget");
};

struct ArgsB {
    const uint8_t* w_packed;
    const uint16_t* w_scales;     // bf16 [N/128][K/128][128]
    float* partial;               // [S][M][N]
    int M, N, K, G, S, n_tiles;
};

// sign-split pools of the fixed table E4M3(v), v = -8..7 (the LUT of sigma = 1): POS = {0..7},
// NEGMAG = {8, 7, ..., 1}
constexpr uint32_t kPos0 = 0x44403800u, kPos1 = 0x4E4C4A48u;   // 0, 1, 2, 3 | 4, 5, 6, 7
constexpr uint32_t kNeg0 = 0x4A4C4E50u, kNeg1 = 0x38404448u;   // 8, 7, 6, 5 | 4, 3, 2, 1

template <int NTOK>
__global__ void __launch_bounds__(kThreads, 2)
k_w4a8_gemm_bf16s(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ ArgsB a) {
    using C = CfgB<NTOK>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sX = smem + C::kOffX;
    uint8_t* sW = smem + C::kOffW;
    uint16_t* sS = reinterpret_cast<uint16_t*>(smem + C::kOffS);
    float* sSig = reinterpret_cast<float*>(smem + C::kOffSig);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
    uint64_t* fullW = bars;
    uint64_t* fullX = fullW + STAGES;
    uint64_t* empty = fullX + STAGES;
    uint64_t* afull = empty + STAGES;
    uint64_t* accfull = afull + ASL;
    uint64_t* accempty = accfull + 2;
    uint32_t* misc = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x / a.S, sp = blockIdx.x % a.S, mt = blockIdx.y;
    const int g0 = sp * a.G / a.S, g1 = (sp + 1) * a.G / a.S, ng = g1 - g0;

    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            ptx::mbar_init(&fullW[i], 1);
            ptx::mbar_init(&fullX[i], 1);
            ptx::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < ASL; ++i) ptx::mbar_init(&afull[i], 4);
        for (int i = 0; i < 2; ++i) { ptx::mbar_init(&accfull[i], 1); ptx::mbar_init(&accempty[i], 4); }
        ptx::fence_mbar_init();
        ptx::prefetch_tmap(&tmap_x);
    }
    if (warp == 4) {
        ptx::tmem_alloc(&misc[0], 256);          // 2 accumulators + 3 A slots: two CTAs per SM fit
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = misc[0];

    if (warp == 8) {
        // ---------------------------------------------------- weight producer
        const uint64_t pol = gridDim.y == 1 ? ptx::policy_evict_first()      // read by one m-tile
                                            : ptx::policy_evict_last();
        for (int i = 0; i < ng; ++i) {
            const int s = i % STAGES;
            ptx::mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
            if (ptx::elect_one()) {
                const size_t blk = (size_t)t * a.G + g0 + i;
                ptx::mbar_arrive_expect_tx(&fullW[s], kWBytes + kTileN * 2);
                ptx::bulk_g2s(sW + s * kWBytes, a.w_packed + blk * kWBytes, kWBytes, &fullW[s], pol);
                ptx::bulk_g2s(sS + s * kTileN, a.w_scales + blk * kTileN, kTileN * 2, &fullW[s], pol);
            }
            __syncwarp();
        }
    } else if (warp == 9) {
        // ---------------------------------------------------- activation producer
        ptx::pdl_wait();
        for (int i = 0; i < ng; ++i) {
            const int s = i % STAGES;
            ptx::mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
            if (ptx::elect_one()) {
                ptx::mbar_arrive_expect_tx(&fullX[s], C::kX);
                ptx::tma_2d_g2s(sX + s * C::kX, &tmap_x, (g0 + i) * kGroup, mt * NTOK, &fullX[s],
                                ptx::policy_evict_last());
            }
            __syncwarp();
        }
    } else if (warp == 10) {
        // ---------------------------------------------------- MMA issuer: one group per accumulator
        constexpr uint32_t idp = make_idesc(NTOK, false), idn = make_idesc(NTOK, true);
        const uint32_t sx0 = ptx::smem_u32(sX);
        for (int i = 0; i < ng; ++i) {
            const int s = i % STAGES, as = i % ASL, b = i & 1;
            ptx::mbar_wait(&afull[as], (i / ASL) & 1);
            ptx::mbar_wait(&fullX[s], (i / STAGES) & 1);
            ptx::mbar_wait(&accempty[b], ((i >> 1) & 1) ^ 1);
            ptx::tc_fence_after();
            const uint32_t d = tmem + C::kAcc0 + b * NTOK, ta = tmem + C::kA0 + as * 64;
            const uint64_t bd0 = smem_desc_sw128(sx0 + s * C::kX);
            if (ptx::elect_one()) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint64_t bd = bd0 + (uint64_t)(j * 32 >> 4);
                    ptx::mma_f8f6f4_ts(d, ta + j * 8, bd, idp, j == 0 ? 0u : 1u);
                    ptx::mma_f8f6f4_ts(d, ta + 32 + j * 8, bd, idn, 1u);
                }
                ptx::mma_commit(&empty[s]);       // SMEM stage + A slot
                ptx::mma_commit(&accfull[b]);
            }
            __syncwarp();
        }
    } else if (warp < 4) {
        // ---------------------------------------------------- converter warpgroup
        const int r = threadIdx.x & 127;
        const uint32_t lane_base = (uint32_t)(r & ~31) << 16;
        for (int i = 0; i < ng; ++i) {
            const int s = i % STAGES, as = i % ASL;
            ptx::mbar_wait(&fullW[s], (i / STAGES) & 1);
            // A slot as was read by the MMAs of group i - ASL (stage (i - ASL) % 8; ASL < STAGES,
            // so that barrier phase is unambiguous)
            if (i >= ASL) ptx::mbar_wait(&empty[(i - ASL) % STAGES], ((i - ASL) / STAGES) & 1);
            ptx::tc_fence_after();
            // this row's sigma for the scaler (ring of 8: the write for group i waits, above, for
            // the MMAs of group i - ASL, which needed accumulator (i - ASL) % 2, i.e. the scaler
            // had finished group i - ASL - 2 >= i - 8)
            sSig[(i & 7) * kTileN + r] = __bfloat162float(__ushort_as_bfloat16(sS[s * kTileN + r]));
            const uint32_t ta = tmem + lane_base + C::kA0 + as * 64;
            const uint8_t* wrow = sW + s * kWBytes + r * 16;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint4 wv = *reinterpret_cast<const uint4*>(wrow + j * 128 * 16);
                uint32_t P[8], Q[8];
                conv_sign_split(wv.x, kPos0, kPos1, kNeg0, kNeg1, P[0], P[1], Q[0], Q[1]);
                conv_sign_split(wv.y, kPos0, kPos1, kNeg0, kNeg1, P[2], P[3], Q[2], Q[3]);
                conv_sign_split(wv.z, kPos0, kPos1, kNeg0, kNeg1, P[4], P[5], Q[4], Q[5]);
                conv_sign_split(wv.w, kPos0, kPos1, kNeg0, kNeg1, P[6], P[7], Q[6], Q[7]);
                ptx::tmem_st_x8(ta + j * 8, P);
                ptx::tmem_st_x8(ta + 32 + j * 8, Q);
            }
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&afull[as]);
        }
    } else if (warp < 8) {
        // ---------------------------------------------------- scaler warpgroup
        const int r = threadIdx.x & 127;
        const uint32_t lane_base = (uint32_t)(r & ~31) << 16;
        float run[NTOK];
#pragma unroll
        for (int c = 0; c < NTOK; ++c) run[c] = 0.0f;
        for (int i = 0; i < ng; ++i) {
            const int b = i & 1;
            ptx::mbar_wait(&accfull[b], (i >> 1) & 1);
            ptx::tc_fence_after();
            const float sig = sSig[(i & 7) * kTileN + r];
#pragma unroll
            for (int c0 = 0; c0 < NTOK; c0 += 16) {
                uint32_t v[16];
                ptx::tmem_ld_x16(tmem + lane_base + C::kAcc0 + b * NTOK + c0, v);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < 16; ++c) run[c0 + c] = __fmaf_rn(sig, __uint_as_float(v[c]), run[c0 + c]);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&accempty[b]);
        }
        const int n = t * kTileN + r;
        float* part = a.partial + (size_t)sp * a.M * a.N;
#pragma unroll
        for (int c = 0; c < NTOK; ++c) {
            const int m = mt * NTOK + c;
            if (m < a.M) part[(size_t)m * a.N + n] = run[c];
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 4) ptx::tmem_dealloc(tmem, 256);
}

// y = bf16(sum_s partial[s] * beta_m * 2^-n), summed in s order
__global__ void k_bf16s_reduce(const float* __restrict__ partial, const __nv_bfloat16* __restrict__ x_scale,
                               int M, int N, int S, int pts_n, __nv_bfloat16* __restrict__ Y, int64_t ldy) {
    ptx::pdl_wait();
    const int64_t total = (int64_t)M * N;
    const float p2 = exp2_neg(pts_n);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = i / N, n = i - m * N;
        float acc = 0.0f;
        for (int s = 0; s < S; ++s) acc = __fadd_rn(acc, partial[(size_t)s * total + i]);
        Y[m * ldy + n] = __float2bfloat16_rn(__fmul_rn(acc, __fmul_rn(__bfloat162float(x_scale[m]), p2)));
    }
}

int splits_for(int64_t M, int64_t N, int64_t K, int ntok) {
    const int64_t ctas = (N / kTileN) * ((M + ntok - 1) / ntok);
    const int64_t G = K / kGroup;
    const int64_t want = (2 * sm_count() + ctas - 1) / ctas;
    return (int)std::max<int64_t>(1, std::min<int64_t>(G, want));
}

template <int NTOK>
fireq_status_t launch_bf16s(const CUtensorMap& map, const ArgsB& a, int m_tiles, cudaStream_t stream) {
    using C = CfgB<NTOK>;
    static bool attr[kMaxDevices] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return fail(FIREQ_ERROR_CUDA, "cudaGetDevice");
    if (!attr[dev]) {
        if (cudaFuncSetAttribute(k_w4a8_gemm_bf16s<NTOK>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem) !=
            cudaSuccess)
            return fail(FIREQ_ERROR_CUDA, "cudaFuncSetAttribute(smem) failed");
        attr[dev] = true;
    }
    const cudaError_t e = launch_ex(k_w4a8_gemm_bf16s<NTOK>, dim3((unsigned)(a.n_tiles * a.S), (unsigned)m_tiles),
                                    dim3(kThreads), C::kSmem, stream, 1u, false, map, a);
    if (e != cudaSuccess) return fail(FIREQ_ERROR_CUDA, std::string("fireq_w4a8_gemm_bf16s launch: ") + cudaGetErrorString(e));
    return FIREQ_SUCCESS;
}

}  // namespace

size_t gemm_bf16s_workspace_bytes(int64_t M, int64_t N, int64_t K) {
    const int ntok = M <= 16 ? 16 : 32;
    return (size_t)splits_for(M, N, K, ntok) * M * N * sizeof(float);
}

fireq_status_t gemm_bf16s_impl(const uint8_t* x_fp8, const __nv_bfloat16* x_scale, int64_t M, int64_t K,
                               const uint8_t* w_packed, const uint16_t* w_scales, int64_t N, int32_t pts_n,
                               __nv_bfloat16* Y, int64_t ldy, void* ws, size_t ws_bytes, cudaStream_t stream) {
    const int ntok = M <= 16 ? 16 : 32;
    if (ws_bytes < gemm_bf16s_workspace_bytes(M, N, K))
        return fail(FIREQ_ERROR_WORKSPACE, "fireq_w4a8_gemm_bf16s: workspace too small");
    CUtensorMap map;
    if (!make_x_map(&map, x_fp8, M, K, ntok)) return fail(FIREQ_ERROR_CUDA, "cuTensorMapEncodeTiled failed");
    ArgsB a{};
    a.w_packed = w_packed;
    a.w_scales = w_scales;
    a.partial = static_cast<float*>(ws);
    a.M = (int)M;
    a.N = (int)N;
    a.K = (int)K;
    a.G = (int)(K / kGroup);
    a.S = splits_for(M, N, K, ntok);
    a.n_tiles = (int)(N / kTileN);
    const int m_tiles = (int)((M + ntok - 1) / ntok);
    fireq_status_t st = ntok == 16 ? launch_bf16s<16>(map, a, m_tiles, stream) : launch_bf16s<32>(map, a, m_tiles, stream);
    if (st != FIREQ_SUCCESS) return st;
    const int64_t total = M * N;
    const unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 8);
    const cudaError_t e = launch_ex(k_bf16s_reduce, dim3(blocks), dim3(256), 0, stream, 1u, false,
                                    static_cast<const float*>(ws), x_scale, (int)M, (int)N, a.S, pts_n, Y, ldy);
    if (e != cudaSuccess) return fail(FIREQ_ERROR_CUDA, std::string("bf16s reduce launch: ") + cudaGetErrorString(e));
    return check_launch("fireq_w4a8_gemm_bf16s");
}

}  // namespace fireq
