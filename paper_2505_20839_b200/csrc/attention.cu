// attention.cu -- fireq_kv4q8_attention: the paper's second kernel (section 3.2
// P:178-291) on sm_100a: prefill self-attention with FP8 queries and an INT4 key / value cache
// (KV4Q8-FP), the scores S = Q K^T and the output O = P V computed by the same INT4 x FP8
// tensor-core path as the linear layers (LUT conversion of INT4 codes to FP8 by CUDA
// cores; FP32 accumulation), the softmax quantized to FP8.
//
// One CTA per (sequence b, query head h, 128-query tile i); the causal tile i visits kv tiles
// 0..i.  Warp roles:
//   warps 0-3   key converters, warps 11-14 value converters: INT4 K / V^T blocks (layout v1, 8 KB + 128 FP8 scales per
//               128 x 128 block) -> FP8 in shared memory, 128-byte swizzled K-major rows (the
//               UMMA B operand), thread r <-> row r, 16-entry LUT per row
//   warps 4-7, 15-18   softmax + epilogue, two halves of the kv / d columns: thread r <-> query
//               row r <-> TMEM lane r
//   warp 8      TMA producer (Q tile once; packed K / V^T blocks into a 2-slot ring)
//   warp 9      MMA issuer: S = Q K^T (A = Q in SMEM, B = K in SMEM, D = S in TMEM), then
//               O += P V (A = P_hat in TMEM written by the softmax warps, B = V^T in SMEM)
//   warp 10     TMEM allocator
// Blackwell mapping of the paper's three-stage pipeline (Alg. 1): the scores of kv tile j are
// computed while the softmax of tile j - 1 runs (two S buffers in TMEM) and O += P_{j-1} V_{j-1}
// is issued after S_j -- wgmma_ss / softmax / wgmma_rs become tcgen05.mma (SMEM x SMEM) /
// tcgen05.ld -> CUDA cores -> tcgen05.st / tcgen05.mma (TMEM x SMEM).  The softmax is Alg. 1's
// online softmax with B_c = 128: running row max m, P_j = exp(x_j - m) quantized to FP8 per
// tile, O rescaled by exp(m_old - m_new) in TMEM before O += P_j V_j (line 14).  The value cache is stored transposed (V^T, groups of 128
// tokens per channel), so the PV product needs no transposed load (P:236 transposes V in TMA).
#include "common.cuh"
#include "gemm_dev.cuh"
#include "ptx.cuh"

namespace fireq {
using namespace dev;
bool make_x_map(CUtensorMap* out, const uint8_t* x, int64_t M, int64_t K, int ntok);
extern unsigned long long* g_trace;
namespace {

constexpr int kD = 128;                 // head dimension (one 128-group per K row)
constexpr int kTile = 128;              // queries per CTA = kv per tile
constexpr int kThreads = 19 * 32;    // + warps 11-14 value converters, 15-18 second softmax half

struct AttnArgs {
    const uint8_t* k_packed;            // [B][Hkv] x layout v1 [N][d]
    const uint8_t* k_scales;
    const uint8_t* vt_packed;           // [B][Hkv] x layout v1 [d][N]
    const uint8_t* vt_scales;
    const int32_t* k_pts;               // [B][Hkv][2] (fireq_quantize_kv pts_and_status of each head)
    const int32_t* v_pts;
    const __nv_bfloat16* q_scale;       // beta_q [B][Hq][N]
    __nv_bfloat16* O;                   // [B * N][ldo], head h at columns [h d, h d + d)
    int64_t ldo;
    int N, Hq, Hkv, B, T;               // T = N / 128
    int causal;
    float tau_log2e;                    // softmax scale tau * log2(e)
    unsigned long long* trace;          // profile builds: per-tile event clocks of CTA 0
};
#ifndef FIREQ_PROFILE
#define FIREQ_PROFILE 0
#endif
// profile builds: trace[tile * 8 + ev] = clock64() in CTA 0 (the heaviest query tile)
#define ATT_EVT(j, ev) do { if (FIREQ_PROFILE && a.trace && blockIdx.x == 0 && (j) < 64) \
    a.trace[(j) * 8 + (ev)] = clock64(); } while (0)

// shared memory carve-up (offsets from a 1024-aligned base)
constexpr int kOffQ = 0;                                 // Q tile, 16 KB, SW128
constexpr int kRing = 3;                                 // depth of the packed / converted K / V rings
constexpr int kOffKc = 16384;                            // kRing x K tile 16 KB, SW128
constexpr int kOffVc = kOffKc + kRing * 16384;           // kRing x V^T tile 16 KB, SW128
constexpr int kOffPk = kOffVc + kRing * 16384;           // kRing x {K 8 KB | V 8 KB | sK 128 | sV 128}
constexpr int kPkSlot = 16640;
constexpr int kOffLut = kOffPk + kRing * kPkSlot;
constexpr int kOffBar = kOffLut + 2048;
constexpr int kNumBars = 28;
constexpr int kOffX = kOffBar + kNumBars * 8;              // softmax halves' row maxima [2][2][128] + l [2][128]
constexpr int kOffMisc = kOffX + 6 * 128 * 4;
constexpr int kSmemBytes = kOffMisc + 64 + 1024;

// TMEM columns
constexpr uint32_t kTS = 0;             // S[2]: 128 columns each
constexpr uint32_t kTO = 256;           // O: 128 columns
constexpr uint32_t kTP = 384;           // P_hat[2]: 32 columns each (128 FP8 per lane)

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// One 128 x 128 block of layout v1 (row r's K-slice j at (j * 128 + r) * 16) -> FP8 row r of a
// 128-byte-swizzled K-major tile (16-byte unit u of row r at (r >> 3) * 1024 + (r & 7) * 128 +
// ((u ^ (r & 7)) * 16)): the mask-select converter, one LUT per row (the row's 128-group).
__device__ __forceinline__ void convert_row(const uint8_t* packed, const uint8_t* sig, const uint4* lut,
                                            uint8_t* dst, int r) {
    const uint4 L = lut[sig[r] & 0x7F];
    uint8_t* row = dst + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint4 wv = *reinterpret_cast<const uint4*>(packed + (j * 128 + r) * 16);
        uint4 o0, o1;
        conv_mask_select(wv.x, L.x, L.y, L.z, L.w, o0.x, o0.y);
        conv_mask_select(wv.y, L.x, L.y, L.z, L.w, o0.z, o0.w);
        conv_mask_select(wv.z, L.x, L.y, L.z, L.w, o1.x, o1.y);
        conv_mask_select(wv.w, L.x, L.y, L.z, L.w, o1.z, o1.w);
        *reinterpret_cast<uint4*>(row + (((2 * j) ^ (r & 7)) * 16)) = o0;
        *reinterpret_cast<uint4*>(row + (((2 * j + 1) ^ (r & 7)) * 16)) = o1;
    }
}

__global__ void __launch_bounds__(kThreads, 1)
k_kv4q8_attn(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ AttnArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sQ = smem + kOffQ;
    uint4* sLut = reinterpret_cast<uint4*>(smem + kOffLut);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
    uint64_t* qfull = bars;
    uint64_t* pk_full = bars + 1;       // [kRing] packed K + V of tile j landed
    uint64_t* pk_empty = bars + 4;      // [kRing] both converter warpgroups have read them
    uint64_t* kc_full = bars + 7;       // [kRing] K_j converted (FP8, SMEM)
    uint64_t* kc_empty = bars + 10;     // [kRing] S_j MMAs done reading it
    uint64_t* vc_full = bars + 13;      // [kRing] V^T_j converted
    uint64_t* vc_empty = bars + 16;     // [kRing] O_j MMAs done reading it
    uint64_t* s_full = bars + 19;       // [2]
    uint64_t* s_empty = bars + 21;      // [2]
    uint64_t* p_full = bars + 23;       // [2]
    uint64_t* pempty = bars + 25;       // [2] P_hat slot free (O MMAs that read it done)
    uint64_t* ofull = bars + 27;        // O complete
    uint32_t* misc = reinterpret_cast<uint32_t*>(smem + kOffMisc);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // heavy (late) query tiles first: tile i of a causal head visits i + 1 kv tiles
    const int per_tile = a.B * a.Hq;
    const int i = a.T - 1 - (int)blockIdx.x / per_tile;
    const int bh = (int)blockIdx.x % per_tile;
    const int b = bh / a.Hq, h = bh % a.Hq;
    const int hk = h / (a.Hq / a.Hkv);
    const int nkv = a.causal ? i + 1 : a.T;
    const size_t kvh = (size_t)b * a.Hkv + hk;
    const size_t blk = (size_t)a.N * kD / 2, sblk = (size_t)a.N * kD / 128;
    const uint8_t* kp = a.k_packed + kvh * blk;
    const uint8_t* ks = a.k_scales + kvh * sblk;
    const uint8_t* vp = a.vt_packed + kvh * blk;
    const uint8_t* vs = a.vt_scales + kvh * sblk;

    // ------------------------------------------------------------ setup
    if (warp == 8 && lane == 0) {
        ptx::mbar_init(qfull, 1);
        for (int s = 0; s < kRing; ++s) {
            ptx::mbar_init(&pk_full[s], 1);
            ptx::mbar_init(&pk_empty[s], 8);
            ptx::mbar_init(&kc_full[s], 4);
            ptx::mbar_init(&kc_empty[s], 1);
            ptx::mbar_init(&vc_full[s], 4);
            ptx::mbar_init(&vc_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(&s_full[s], 1);
            ptx::mbar_init(&s_empty[s], 8);
            ptx::mbar_init(&p_full[s], 8);
            ptx::mbar_init(&pempty[s], 1);
        }
        ptx::mbar_init(ofull, 1);
        ptx::fence_mbar_init();
        ptx::prefetch_tmap(&tmap_q);
    }
    if (warp == 10) {
        ptx::tmem_alloc(&misc[0], 512);
        ptx::tmem_relinquish();
    }
    build_lut(reinterpret_cast<uint8_t*>(sLut), threadIdx.x, kThreads);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = misc[0];

    if (warp == 8) {
        // ------------------------------------------------------- producer
        ptx::pdl_wait();                     // Q, beta_q and the caches come from earlier kernels
        const uint64_t pol = ptx::policy_evict_last();    // K / V blocks are re-read by the Hq / Hkv heads
        if (ptx::elect_one()) {
            ptx::mbar_arrive_expect_tx(qfull, kTile * kD);
            ptx::tma_2d_g2s(sQ, &tmap_q, 0, ((b * a.Hq + h) * a.N) + i * kTile, qfull, ptx::policy_evict_first());
        }
        __syncwarp();
        for (int j = 0; j < nkv; ++j) {
            const int s = j % kRing, ph = (j / kRing) & 1;
            ptx::mbar_wait(&pk_empty[s], ph ^ 1);
            if (ptx::elect_one()) {
                uint8_t* dst = smem + kOffPk + s * kPkSlot;
                ptx::mbar_arrive_expect_tx(&pk_full[s], 2 * (8192 + 128));
                ptx::bulk_g2s(dst, kp + (size_t)j * 8192, 8192, &pk_full[s], pol);
                ptx::bulk_g2s(dst + 16384, ks + (size_t)j * 128, 128, &pk_full[s], pol);
                ptx::bulk_g2s(dst + 8192, vp + (size_t)j * 8192, 8192, &pk_full[s], pol);
                ptx::bulk_g2s(dst + 16384 + 128, vs + (size_t)j * 128, 128, &pk_full[s], pol);
            }
            __syncwarp();
        }
    } else if (warp < 4 || (warp >= 11 && warp < 15)) {
        // ------------------------------------------------------- converters (warps 0-3: K, 11-14: V^T)
        const bool vconv = warp >= 11;
        const int r = vconv ? (int)threadIdx.x - 11 * 32 : (int)threadIdx.x;
        uint64_t* c_full = vconv ? vc_full : kc_full;
        uint64_t* c_empty = vconv ? vc_empty : kc_empty;
        for (int j = 0; j < nkv; ++j) {
            const int s = j % kRing, ph = (j / kRing) & 1;
            ptx::mbar_wait(&pk_full[s], ph);
            ptx::mbar_wait(&c_empty[s], ph ^ 1);
            const uint8_t* src = smem + kOffPk + s * kPkSlot;
            if (!vconv) convert_row(src, src + 16384, sLut, smem + kOffKc + s * 16384, r);
            else convert_row(src + 8192, src + 16384 + 128, sLut, smem + kOffVc + s * 16384, r);
            ptx::fence_proxy_async_smem();   // generic-proxy stores -> the MMA's async-proxy reads
            __syncwarp();
            if (lane == 0) {
                ptx::mbar_arrive(&c_full[s]);
                ptx::mbar_arrive(&pk_empty[s]);
            }
        }
    } else if (warp == 9) {
        // ------------------------------------------------------- MMA issuer
        constexpr uint32_t idesc = make_idesc(kTile, false);   // M = 128, N = 128, E4M3 x E4M3 -> F32
        ptx::mbar_wait(qfull, 0);
        ptx::tc_fence_after();
        const uint64_t qdesc = smem_desc_sw128(ptx::smem_u32(sQ));
        // O += P_hat(j) V^T(j) once the softmax has written P_hat(j) and rescaled O (Alg. 1 line 14)
        auto issue_o = [&](int j) {
            const int s = j & 1, sv = j % kRing;
            ptx::mbar_wait(&vc_full[sv], (j / kRing) & 1);
            ptx::mbar_wait(&p_full[s], (j >> 1) & 1);
            ptx::tc_fence_after();
            if (ptx::elect_one()) {
                const uint64_t vdesc = smem_desc_sw128(ptx::smem_u32(smem + kOffVc + sv * 16384));
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    ptx::mma_f8f6f4_ts(tmem + kTO, tmem + kTP + s * 32 + k * 8, vdesc + (uint64_t)(k * 2), idesc,
                                       (j > 0 || k > 0) ? 1u : 0u);
                ptx::mma_commit(&pempty[s]);
                ptx::mma_commit(&vc_empty[sv]);
            }
            if (lane == 0) ATT_EVT(j, 7);
            __syncwarp();
        };
        for (int j = 0; j < nkv; ++j) {
            const int s = j & 1, ph = (j >> 1) & 1, sk = j % kRing;
            ptx::mbar_wait(&kc_full[sk], (j / kRing) & 1);
            ptx::mbar_wait(&s_empty[s], ph ^ 1);
            ptx::tc_fence_after();
            if (ptx::elect_one()) {          // S_j = Q K_j^T (Alg. 1 line 12), before O += P_{j-1} V_{j-1}
                const uint64_t kdesc = smem_desc_sw128(ptx::smem_u32(smem + kOffKc + sk * 16384));
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    ptx::mma_f8f6f4_ss(tmem + kTS + s * 128, qdesc + (uint64_t)(k * 2), kdesc + (uint64_t)(k * 2), idesc,
                                       k > 0 ? 1u : 0u);
                ptx::mma_commit(&s_full[s]);
                ptx::mma_commit(&kc_empty[sk]);
            }
            if (lane == 0) ATT_EVT(j, 6);
            __syncwarp();
            if (j > 0) issue_o(j - 1);
        }
        issue_o(nkv - 1);
        if (ptx::elect_one()) ptx::mma_commit(ofull);
        __syncwarp();
    } else if ((warp >= 4 && warp < 8) || warp >= 15) {
        // ------------------------------------------------------- online softmax + epilogue (Alg. 1)
        // Two warpgroups share the rows: half hf takes kv columns [64 hf, 64 hf + 64) of S, TMEM
        // columns [16 hf, 16 hf + 16) of P_hat and d columns [64 hf, 64 hf + 64) of O; the row max
        // of each tile is exchanged through shared memory (one named barrier per tile).
        const int hf = warp >= 15 ? 1 : 0;
        // query row == TMEM lane; a warp reaches only TMEM lanes [32 (warp % 4), + 32)
        const int r = (warp & 3) * 32 + lane;
        const uint32_t lane_base = (uint32_t)(r & ~31) << 16;
        float* xmax = reinterpret_cast<float*>(smem + kOffX);      // [tile parity][half][row]
        float* xl = xmax + 4 * 128;                                // [half][row]
        const int q = i * kTile + r;
        const float bq = __bfloat162float(a.q_scale[((size_t)b * a.Hq + h) * a.N + q]);
        const int nk = a.k_pts[2 * kvh], nv = a.v_pts[2 * kvh];
        const float sc = bq * exp2_neg(nk) * a.tau_log2e;  // acc -> log2-domain logit (sc > 0)
        constexpr float kLog2_448 = 8.807354922057604f;    // 448 P = exp2(x - m + log2 448)
        float m2 = -INFINITY, l = 0.0f;                    // l accumulates 448 P (this half's columns)
        for (int j = 0; j < nkv; ++j) {
            const int s = j & 1, ph = (j >> 1) & 1;
            const bool diag = a.causal && j == i;
            if (hf == 0 && r == 0) ATT_EVT(j, 0);
            ptx::mbar_wait(&s_full[s], ph);
            if (hf == 0 && r == 0) ATT_EVT(j, 1);
            ptx::tc_fence_after();
            const uint32_t ts = tmem + lane_base + kTS + s * 128 + hf * 64;
            // m_new = max(m_old, rowmax(x_j)) (lines 10-11), max over the raw accumulators (sc > 0)
            // (the causal mask matters on the diagonal tile only: a separate loop keeps the
            // per-element selects out of the others)
            float mx = -INFINITY;
            if (!diag) {
                uint32_t v[64];
                ptx::tmem_ld_x64(ts, v);                       // one load for the half's 64 scores
                ptx::tmem_wait_ld();
                // four independent max chains (a single chain is 32 dependent FMNMX)
                float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                for (int c = 0; c < 64; c += 8)
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        m4[q] = fmaxf(m4[q], fmaxf(__uint_as_float(v[c + q]), __uint_as_float(v[c + 4 + q])));
                mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
            } else {
#pragma unroll 1
                for (int c0 = 0; c0 < 64; c0 += 16) {
                    uint32_t v[16];
                    ptx::tmem_ld_x16(ts + c0, v);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int c = 0; c < 16; ++c)
                        if (hf * 64 + c0 + c <= r) mx = fmaxf(mx, __uint_as_float(v[c]));
                }
            }
            xmax[(s * 2 + hf) * 128 + r] = mx;
            ptx::named_bar_sync(3, 256);
            mx = fmaxf(mx, xmax[(s * 2 + (hf ^ 1)) * 128 + r]);
            if (hf == 0 && r == 0) ATT_EVT(j, 2);
            const float mnew = fmaxf(m2, mx * sc);
            const float resc = ex2_approx(m2 - mnew);        // s_i = exp(m_old - m_new); 0 on tile 0
            m2 = mnew;
            l *= resc;
            const float off = mnew - kLog2_448;
            // 448 P_j = exp2(x_j - m_new + log2 448), l += rowsum, P_hat_j = E4M3_RN(448 P_j) (line 13).
            // The P slot was last read by the O MMA of tile j - 2, complete once O(j - 1) is.
            if (hf == 0 && r == 0) ATT_EVT(j, 3);
            if (j >= 1) ptx::mbar_wait(&pempty[(j - 1) & 1], ((j - 1) >> 1) & 1);
            if (hf == 0 && r == 0) ATT_EVT(j, 4);
            ptx::tc_fence_after();
            const uint32_t tp = tmem + lane_base + kTP + s * 32 + hf * 16;
            {
                uint32_t v[64], w16[16];
                ptx::tmem_ld_x64(ts, v);                      // the half's 64 scores, one load
                ptx::tmem_wait_ld();
                // exponent arguments on the packed FFMA2 path (per element the same RN fma);
                // the row sum in four independent partial sums (one chain was 64 dependent FADDs)
                const float2 sc2 = make_float2(sc, sc), noff2 = make_float2(-off, -off);
                float2 la = make_float2(0.0f, 0.0f), lb = make_float2(0.0f, 0.0f);
#pragma unroll
                for (int c4 = 0; c4 < 16; ++c4) {
                    float p[4];
#pragma unroll
                    for (int e = 0; e < 4; e += 2) {
                        const int c = 4 * c4 + e;
                        const float2 t = __ffma2_rn(make_float2(__uint_as_float(v[c]), __uint_as_float(v[c + 1])), sc2, noff2);
                        p[e] = ex2_approx(t.x);
                        p[e + 1] = ex2_approx(t.y);
                        if (diag && hf * 64 + c > r) p[e] = 0.0f;
                        if (diag && hf * 64 + c + 1 > r) p[e + 1] = 0.0f;
                    }
                    la = __fadd2_rn(la, make_float2(p[0], p[1]));
                    lb = __fadd2_rn(lb, make_float2(p[2], p[3]));
                    w16[c4] = e4m3x2_rn(p[0], p[1]) | (e4m3x2_rn(p[2], p[3]) << 16);
                }
                l += (la.x + la.y) + (lb.x + lb.y);
                ptx::tmem_st_x16(tp, w16);
            }
            if (j >= 1 && __any_sync(0xffffffffu, resc != 1.0f)) {
                // one 64-column TMEM load and one store (not four dependent round trips)
                const uint32_t to = tmem + lane_base + kTO + hf * 64;
                uint32_t o[64];
                ptx::tmem_ld_x64(to, o);
                ptx::tmem_wait_ld();
                const float2 rs2 = make_float2(resc, resc);
#pragma unroll
                for (int c = 0; c < 64; c += 2) {
                    const float2 oo = __fmul2_rn(make_float2(__uint_as_float(o[c]), __uint_as_float(o[c + 1])), rs2);
                    o[c] = __float_as_uint(oo.x);
                    o[c + 1] = __float_as_uint(oo.y);
                }
                ptx::tmem_st_x64(to, o);
            }
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                ptx::mbar_arrive(&s_empty[s]);
                ptx::mbar_arrive(&p_full[s]);
            }
            if (hf == 0 && r == 0) ATT_EVT(j, 5);
        }
        // epilogue: O = acc * 2^-n_v / (448 l) -> BF16, token-major [B N][ldo] at head h's columns
        xl[hf * 128 + r] = l;
        ptx::named_bar_sync(3, 256);
        const float ltot = xl[r] + xl[128 + r];
        ptx::mbar_wait(ofull, 0);
        ptx::tc_fence_after();
        const float f = exp2_neg(nv) / ltot;
        __nv_bfloat16* orow = a.O + ((size_t)b * a.N + q) * a.ldo + (size_t)h * kD + hf * 64;
#pragma unroll 1
        for (int c0 = 0; c0 < 64; c0 += 16) {
            uint32_t v[16];
            ptx::tmem_ld_x16(tmem + lane_base + kTO + hf * 64 + c0, v);
            ptx::tmem_wait_ld();
            __align__(16) __nv_bfloat16 y[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) y[c] = __float2bfloat16_rn(__uint_as_float(v[c]) * f);
            reinterpret_cast<uint4*>(orow + c0)[0] = reinterpret_cast<const uint4*>(y)[0];
            reinterpret_cast<uint4*>(orow + c0)[1] = reinterpret_cast<const uint4*>(y)[1];
        }
    }
    // ------------------------------------------------------------ teardown
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 10) ptx::tmem_dealloc(tmem, 512);
}

}  // namespace

fireq_status_t kv4q8_attention_impl(const uint8_t* q_fp8, const __nv_bfloat16* q_scale, const uint8_t* k_packed,
                                    const uint8_t* k_scales, const int32_t* k_pts, const uint8_t* vt_packed,
                                    const uint8_t* vt_scales, const int32_t* v_pts, int64_t B, int64_t N,
                                    int64_t Hq, int64_t Hkv, int causal, float tau, __nv_bfloat16* O, int64_t ldo,
                                    cudaStream_t stream) {
    CUtensorMap map;
    if (!make_x_map(&map, q_fp8, B * Hq * N, kD, kTile)) return fail(FIREQ_ERROR_CUDA, "cuTensorMapEncodeTiled failed");
    AttnArgs args{};
    args.k_packed = k_packed;
    args.k_scales = k_scales;
    args.vt_packed = vt_packed;
    args.vt_scales = vt_scales;
    args.k_pts = k_pts;
    args.v_pts = v_pts;
    args.q_scale = q_scale;
    args.O = O;
    args.ldo = ldo;
    args.N = (int)N;
    args.Hq = (int)Hq;
    args.Hkv = (int)Hkv;
    args.B = (int)B;
    args.T = (int)(N / kTile);
    args.causal = causal;
    args.tau_log2e = tau * 1.4426950408889634f;
    args.trace = FIREQ_PROFILE ? g_trace : nullptr;
    static bool attr_done[kMaxDevices] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices)
        return fail(FIREQ_ERROR_CUDA, "cudaGetDevice failed");
    if (!attr_done[dev]) {
        if (cudaFuncSetAttribute(k_kv4q8_attn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes) != cudaSuccess)
            return fail(FIREQ_ERROR_CUDA, "cudaFuncSetAttribute(smem) failed");
        attr_done[dev] = true;
    }
    const cudaError_t e = launch_ex(k_kv4q8_attn, dim3((unsigned)(B * Hq * args.T)), dim3(kThreads), kSmemBytes,
                                    stream, 1u, false, map, args);
    if (e != cudaSuccess) return fail(FIREQ_ERROR_CUDA, std::string("fireq_kv4q8_attention launch: ") + cudaGetErrorString(e));
    return check_launch("fireq_kv4q8_attention");
}

}  // namespace fireq
