// mainloop_joint.cu -- decode mainloop in isolation (not product code): does converting each
// pipeline stage JOINTLY by all converter warpgroups (each takes 1/NCONV of the stage's 32-K
// chunks) beat one warpgroup per stage?  With one warpgroup per stage a stage's conversion
// latency is NCONV x the converter throughput time, and the TMEM A ring (ASTAGES slots) must
// cover that latency plus the MMAs; jointly the latency is 1 x.
// One CTA per SM streams 2 MB of packed INT4 (148 x 2 MB > L2, so HBM) through an NS-stage
// ring; X tiles by bulk copy; sign-split conversion into TMEM; one MMA warp (N = 16).
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

template <int NCONV, int NS, int ASTAGES, int GPS, bool JOINT>
__global__ void __launch_bounds__(128 * NCONV + 96, 1)
k_main(const uint8_t* __restrict__ w, const uint8_t* __restrict__ xg, int groups_per_cta, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    constexpr int kWStage = GPS * 8192;
    constexpr int kASz = GPS * 64;
    constexpr int CH = JOINT ? GPS * 4 / NCONV : GPS * 4;     // 32-K chunks per warpgroup per stage
    static_assert(!JOINT || (GPS * 4) % NCONV == 0, "chunks must split evenly");
    static_assert(32 + ASTAGES * kASz <= 512, "TMEM");
    uint8_t* sW = smem;
    uint8_t* sX = smem + NS * kWStage;
    uint4* sLut = reinterpret_cast<uint4*>(sX + NS * GPS * 2048);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sX + NS * GPS * 2048 + 2048);
    uint64_t* fullW = bars;
    uint64_t* empty = fullW + NS;
    uint64_t* afull = empty + NS;
    uint64_t* done = afull + ASTAGES;
    uint64_t* fullX = done + 1;
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) reinterpret_cast<uint8_t*>(sLut)[i] = (uint8_t)(i & 0x7F);
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) { ptx::mbar_init(&fullW[i], 1); ptx::mbar_init(&empty[i], 1); ptx::mbar_init(&fullX[i], 1); }
        for (int i = 0; i < ASTAGES; ++i) ptx::mbar_init(&afull[i], JOINT ? 4 * NCONV : 4);
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
    } else if (warp == 4 * NCONV + 2) {               // activation producer
        for (int i = 0; i < nst; ++i) {
            const int s = i % NS;
            ptx::mbar_wait(&empty[s], ((i / NS) & 1) ^ 1);
            const uint8_t* src = xg + (size_t)((i * GPS) % 32) * 2048;
            if (ptx::elect_one()) {
                ptx::mbar_arrive_expect_tx(&fullX[s], GPS * 2048);
                ptx::bulk_g2s(sX + s * GPS * 2048, src, GPS * 2048, &fullX[s], ptx::policy_evict_last());
            }
            __syncwarp();
        }
    } else if (warp == 4 * NCONV + 1) {               // MMA issuer
        const uint32_t idp = (1u << 4) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint32_t idn = idp | (1u << 13);
        for (int i = 0; i < nst; ++i) {
            const int s = i % NS, as = i % ASTAGES;
            ptx::mbar_wait(&afull[as], (i / ASTAGES) & 1);
            ptx::tc_fence_after();
            const uint32_t ta = tmem + 32 + as * kASz;
            const uint64_t bdx = desc_sw128(ptx::smem_u32(sX + s * GPS * 2048));
            if (ptx::elect_one()) {
#pragma unroll
                for (int q = 0; q < GPS; ++q)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint64_t bd = bdx + (uint64_t)(q * 128 + j * 2);
                        ptx::mma_f8f6f4_ts(tmem, ta + q * 64 + j * 8, bd, idp, 1u);
                        ptx::mma_f8f6f4_ts(tmem, ta + q * 64 + 32 + j * 8, bd, idn, 1u);
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
    } else if (warp < 4 * NCONV) {                    // converters
        const int wg = warp >> 2, r = threadIdx.x & 127;
        const uint32_t lane_base = (uint32_t)(r & ~31) << 16;
        const int i0 = JOINT ? 0 : wg, di = JOINT ? 1 : NCONV;
        const int c0 = JOINT ? wg * CH : 0;
        for (int i = i0; i < nst; i += di) {
            const int s = i % NS, as = i % ASTAGES;
            ptx::mbar_wait(&fullW[s], (i / NS) & 1);
            if (i >= ASTAGES) ptx::mbar_wait(&empty[(i - ASTAGES) % NS], ((i - ASTAGES) / NS) & 1);
            ptx::tc_fence_after();
            uint4 L = make_uint4(0, 0, 0, 0);
            uint32_t N0 = 0, N1 = 0;
            int qprev = -1;
#pragma unroll
            for (int cc = 0; cc < CH; ++cc) {
                const int c = c0 + cc, q = c >> 2, j = c & 3;
                if (q != qprev) {    // (compile-time except for wg-dependent c0: loaded per group)
                    L = sLut[(sW[s * kWStage + q * 8192 + r]) & 0x7F];
                    N0 = L.z & 0x7F7F7F7Fu; N1 = L.w & 0x7F7F7F7Fu;
                    qprev = q;
                }
                const uint32_t ta = tmem + lane_base + 32 + as * kASz + q * 64;
                const uint4 wv = *reinterpret_cast<const uint4*>(sW + s * kWStage + q * 8192 + r * 16 + j * 128 * 16);
                uint32_t P[8], Q[8];
                conv_ss(wv.x, L.x, L.y, N0, N1, P[0], P[1], Q[0], Q[1]);
                conv_ss(wv.y, L.x, L.y, N0, N1, P[2], P[3], Q[2], Q[3]);
                conv_ss(wv.z, L.x, L.y, N0, N1, P[4], P[5], Q[4], Q[5]);
                conv_ss(wv.w, L.x, L.y, N0, N1, P[6], P[7], Q[6], Q[7]);
                ptx::tmem_st_x8(ta + j * 8, P);
                ptx::tmem_st_x8(ta + 32 + j * 8, Q);
            }
            ptx::tmem_wait_st();
            ptx::mbar_wait(&fullX[s], (i / NS) & 1);
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

template <int NCONV, int NS, int ASTAGES, int GPS, bool JOINT>
void run(const char* name, const uint8_t* w, int gpc, unsigned long long* d, const uint8_t* xg) {
    auto k = k_main<NCONV, NS, ASTAGES, GPS, JOINT>;
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
    double s = 0, mx = 0; for (auto v : h) { s += v; mx = v > mx ? v : mx; }
    const double bytes = 148.0 * gpc * 8192;
    printf("%-40s %6.1f cyc/group (max CTA %6.1f)  %6.0f GB/s over the launch (%.2f us)\n", name, s / 148 / gpc,
           mx / gpc, bytes / (ms / reps * 1e-3) / 1e9, ms / reps * 1e3);
}

int main() {
    const int gpc = 256;                                // groups per CTA (2 MB each; 310 MB total > L2)
    uint8_t* w;
    cudaMalloc(&w, (size_t)148 * gpc * 8192);
    cudaMemset(w, 0x5A, (size_t)148 * gpc * 8192);
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    uint8_t* xg;
    cudaMalloc(&xg, 32 * 2048);
    cudaMemset(xg, 0x38, 32 * 2048);
    for (int rep = 0; rep < 2; ++rep) {
        run<3, 8, 3, 2, false>("per-stage NCONV3 NS8 A3 GPS2 (product)", w, gpc, d, xg);
        run<2, 8, 3, 2, false>("per-stage NCONV2 NS8 A3 GPS2", w, gpc, d, xg);
        run<2, 8, 3, 2, true>("joint NCONV2 NS8 A3 GPS2", w, gpc, d, xg);
        run<4, 8, 3, 2, true>("joint NCONV4 NS8 A3 GPS2", w, gpc, d, xg);
        run<2, 10, 6, 1, true>("joint NCONV2 NS10 A6 GPS1", w, gpc, d, xg);
        run<4, 10, 6, 1, true>("joint NCONV4 NS10 A6 GPS1", w, gpc, d, xg);
        run<2, 10, 7, 1, true>("joint NCONV2 NS10 A7 GPS1", w, gpc, d, xg);
        run<1, 8, 3, 2, false>("per-stage NCONV1 NS8 A3 GPS2", w, gpc, d, xg);
    }
    return 0;
}
