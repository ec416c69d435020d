// mainloop_bench.cu -- the decode GEMM mainloop in isolation (not product code).
// One CTA per SM streams its share of a packed INT4 weight matrix (TMA bulk copies into an
// NS-stage ring, GPS groups of 128x128 per stage), NCONV converter warpgroups turn stages into
// TMEM A operands (sign-split) in ASTAGES slots, one warp issues the MMAs (N = 16 tokens,
// activation tile static in shared memory) with one commit per stage.  No epilogue.
// Prints cycles per 128x128 group and the achieved HBM bandwidth.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2505_20839_b200/csrc/ptx.cuh"
using namespace fireq;

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
__device__ __forceinline__ void conv_ss(uint32_t w, uint32_t L0, uint32_t L1, uint32_t N0, uint32_t N1,
                                        uint32_t& p0, uint32_t& p1, uint32_t& n0, uint32_t& n1) {
    const uint32_t x = w ^ 0x88888888u;
    const uint32_t wh = ptx::hi16_prmt(w), xh = ptx::hi16_prmt(x);
    p0 = ptx::prmt(L0, L1, w); p1 = ptx::prmt(L0, L1, wh);
    n0 = ptx::prmt(N0, N1, x); n1 = ptx::prmt(N0, N1, xh);
}

// MODE 0 full (static activation tile), 1 no conversion, 2 no MMA, 3 activation tiles per stage
// by TMA bulk copy (behind the weights in the TMA queue), 4 activation tiles per stage by cp.async;
// in 3 / 4 the converters wait for the stage's activation tile before arriving (as the GEMM does)
template <int NCONV, int NS, int ASTAGES, int GPS, int MODE>
__global__ void __launch_bounds__(128 * NCONV + 96, 1)
k_main(const uint8_t* __restrict__ w, const uint8_t* __restrict__ xg, int groups_per_cta, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    constexpr int kWStage = GPS * 8192;
    uint8_t* sW = smem;                               // NS stages
    uint8_t* sX = smem + NS * kWStage;                // 2 KB static activation tile, or the X ring
    uint4* sLut = reinterpret_cast<uint4*>(sX + NS * GPS * 2048);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sX + NS * GPS * 2048 + 2048);
    uint64_t* fullW = bars;
    uint64_t* empty = fullW + NS;
    uint64_t* afull = empty + NS;
    uint64_t* done = afull + ASTAGES;
    uint64_t* fullX = done + 1;
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) { sX[i] = 0x38; reinterpret_cast<uint8_t*>(sLut)[i] = (uint8_t)(i & 0x7F); }
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) { ptx::mbar_init(&fullW[i], 1); ptx::mbar_init(&empty[i], 1); }
        for (int i = 0; i < ASTAGES; ++i) ptx::mbar_init(&afull[i], 4);
        for (int i = 0; i < NS; ++i) ptx::mbar_init(&fullX[i], MODE == 4 ? 32 : 1);
        ptx::mbar_init(done, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) { ptx::tmem_alloc(&tbase, 512); ptx::tmem_relinquish(); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tbase;
    const int nst = groups_per_cta / GPS;
    const uint8_t* wbase = w + (size_t)blockIdx.x * groups_per_cta * 8192;
    unsigned long long t0 = clock64();
    if (warp == 4 * NCONV) {                          // weight producer
        const uint64_t pol = ptx::policy_evict_first();
        for (int i = 0; i < nst; ++i) {
            const int s = i % NS;
            ptx::mbar_wait(&empty[s], ((i / NS) & 1) ^ 1);
            if (ptx::elect_one()) {
                ptx::mbar_arrive_expect_tx(&fullW[s], kWStage);
                ptx::bulk_g2s(sW + s * kWStage, wbase + (size_t)i * kWStage, kWStage, &fullW[s], pol);
            }
            __syncwarp();
        }
    } else if (warp == 4 * NCONV + 2) {               // activation producer (modes 3 / 4)
        if (MODE == 3 || MODE == 4) {
            for (int i = 0; i < nst; ++i) {
                const int s = i % NS;
                ptx::mbar_wait(&empty[s], ((i / NS) & 1) ^ 1);
                const uint8_t* src = xg + (size_t)((i * GPS) % 32) * 2048;
                if (MODE == 3) {
                    if (ptx::elect_one()) {
                        ptx::mbar_arrive_expect_tx(&fullX[s], GPS * 2048);
                        ptx::bulk_g2s(sX + s * GPS * 2048, src, GPS * 2048, &fullX[s], ptx::policy_evict_last());
                    }
                    __syncwarp();
                } else {
#pragma unroll
                    for (int c = 0; c < GPS * 4; ++c)
                        ptx::cp_async_16(sX + s * GPS * 2048 + (c * 32 + lane) * 16, src + (c * 32 + lane) * 16, 16u);
                    ptx::cp_async_mbar_arrive(&fullX[s]);
                }
            }
        }
    } else if (warp == 4 * NCONV + 1) {               // MMA issuer
        const uint32_t idp = (1u << 4) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint32_t idn = idp | (1u << 13);
        const uint64_t bd0 = desc_sw128(ptx::smem_u32(sX));
        for (int i = 0; i < nst; ++i) {
            const int s = i % NS, as = i % ASTAGES;
            ptx::mbar_wait(&afull[as], (i / ASTAGES) & 1);
            ptx::tc_fence_after();
            if (MODE == 4) ptx::fence_proxy_async_smem();
            const uint32_t ta = tmem + 32 + as * GPS * 64;
            const uint64_t bdx = (MODE == 3 || MODE == 4) ? desc_sw128(ptx::smem_u32(sX + s * GPS * 2048)) : bd0;
            if (ptx::elect_one()) {
                if (MODE != 2) {
#pragma unroll
                    for (int q = 0; q < GPS; ++q)
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const uint64_t bd = bdx + (uint64_t)(q * 128 + j * 2);
                            ptx::mma_f8f6f4_ts(tmem, ta + q * 64 + j * 8, bd, idp, 1u);
                            ptx::mma_f8f6f4_ts(tmem, ta + q * 64 + 32 + j * 8, bd, idn, 1u);
                        }
                }
                ptx::mma_commit(&empty[s]);
            }
            __syncwarp();
        }
        if (ptx::elect_one()) ptx::mma_commit(done);
        __syncwarp();
        ptx::mbar_wait(done, 0);
        unsigned long long t1 = clock64();
        if (lane == 0) out[blockIdx.x] = t1 - t0;
    } else if (warp < 4 * NCONV) {                    // converters: stage i by warpgroup i % NCONV
        const int wg = warp >> 2, r = threadIdx.x & 127;
        const uint32_t lane_base = (uint32_t)(r & ~31) << 16;
        for (int i = wg; i < nst; i += NCONV) {
            const int s = i % NS, as = i % ASTAGES;
            ptx::mbar_wait(&fullW[s], (i / NS) & 1);
            if (i >= ASTAGES) ptx::mbar_wait(&empty[(i - ASTAGES) % NS], ((i - ASTAGES) / NS) & 1);
            ptx::tc_fence_after();
            if (MODE != 1) {
#pragma unroll
                for (int q = 0; q < GPS; ++q) {
                    const uint32_t ta = tmem + lane_base + 32 + (as * GPS + q) * 64;
                    const uint4 L = sLut[(sW[s * kWStage + q * 8192 + r]) & 0x7F];
                    const uint32_t N0 = L.z & 0x7F7F7F7Fu, N1 = L.w & 0x7F7F7F7Fu;
                    const uint8_t* wrow = sW + s * kWStage + q * 8192 + r * 16;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint4 wv = *reinterpret_cast<const uint4*>(wrow + j * 128 * 16);
                        uint32_t P[8], Q[8];
                        conv_ss(wv.x, L.x, L.y, N0, N1, P[0], P[1], Q[0], Q[1]);
                        conv_ss(wv.y, L.x, L.y, N0, N1, P[2], P[3], Q[2], Q[3]);
                        conv_ss(wv.z, L.x, L.y, N0, N1, P[4], P[5], Q[4], Q[5]);
                        conv_ss(wv.w, L.x, L.y, N0, N1, P[6], P[7], Q[6], Q[7]);
                        ptx::tmem_st_x8(ta + j * 8, P);
                        ptx::tmem_st_x8(ta + 32 + j * 8, Q);
                    }
                }
                ptx::tmem_wait_st();
            }
            if (MODE == 3 || MODE == 4) ptx::mbar_wait(&fullX[s], (i / NS) & 1);
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&afull[as]);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

template <int NCONV, int NS, int ASTAGES, int GPS, int MODE>
void run(const char* name, const uint8_t* w, int gpc, unsigned long long* d, const uint8_t* xg) {
    auto k = k_main<NCONV, NS, ASTAGES, GPS, MODE>;
    const int smem = NS * GPS * 8192 + NS * GPS * 2048 + 2048 + 1024 + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<<<148, 128 * NCONV + 96, smem>>>(w, xg, gpc, d);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int i = 0; i < reps; ++i) k<<<148, 128 * NCONV + 96, smem>>>(w, xg, gpc, d);
    cudaEventRecord(e1);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("%s: error\n", name); return; }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> h(148);
    cudaMemcpy(h.data(), d, 148 * 8, cudaMemcpyDeviceToHost);
    double s = 0; for (auto v : h) s += v;
    const double bytes = 148.0 * gpc * 8192;
    printf("%-44s %6.1f cyc/group  %6.0f GB/s (%.2f us/launch)\n", name, s / 148 / gpc, bytes / (ms / reps * 1e-3) / 1e9,
           ms / reps * 1e3);
}

int main() {
    const int gpc = 128;                                // groups per CTA (1 MB of packed weights each)
    uint8_t* w;
    cudaMalloc(&w, (size_t)148 * gpc * 8192);
    cudaMemset(w, 0x5A, (size_t)148 * gpc * 8192);
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    uint8_t* xg;
    cudaMalloc(&xg, 32 * 2048);
    cudaMemset(xg, 0x38, 32 * 2048);
    run<3, 8, 3, 2, 0>("NCONV3 NS8 A3 GPS2 static X", w, gpc, d, xg);
    run<3, 8, 3, 2, 3>("NCONV3 NS8 A3 GPS2 X by TMA (queued behind W)", w, gpc, d, xg);
    run<3, 8, 3, 2, 4>("NCONV3 NS8 A3 GPS2 X by cp.async", w, gpc, d, xg);
    run<3, 8, 3, 2, 1>("NCONV3 NS8 A3 GPS2 no-conversion", w, gpc, d, xg);
    run<2, 8, 3, 2, 4>("NCONV2 NS8 A3 GPS2 X by cp.async", w, gpc, d, xg);
    return 0;
}
