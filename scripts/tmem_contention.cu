// tmem_contention.cu -- do converter TMEM stores slow the tensor core down? (not product code)
// One CTA per SM: NCONV converter warpgroups convert packed INT4 (shared memory) into TMEM in a
// loop (sign-split or mask-select), while one warp issues tcgen05.mma (M=128, N=16, K=32, A from
// TMEM) in blocks of 16 per elected thread with one commit per block.  Each side is timed alone
// and together: cycles per group (converter) and per MMA.
#include <cstdio>
#include <cstdint>
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

template <int NCONV>
__global__ void k(int conv_groups, int mma_blocks, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    uint8_t* sW = smem;                    // 16 KB packed
    uint4* sLut = reinterpret_cast<uint4*>(smem + 16384);
    uint8_t* sX = smem + 16384 + 2048 + 1024;   // B operand, 1024-aligned: 2 KB
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) sW[i] = (uint8_t)(i * 37 + 11);
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) reinterpret_cast<uint8_t*>(sLut)[i] = (uint8_t)(i & 0x7F);
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sX[i] = 0x38;
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    if (threadIdx.x < 32) { ptx::tmem_alloc(&tbase, 512); ptx::tmem_relinquish(); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tbase;
    const int warp = threadIdx.x >> 5;
    if (warp < 4 * NCONV) {
        const int wg = warp >> 2, r = threadIdx.x & 127;
        const uint32_t ta = tmem + ((uint32_t)(r & ~31) << 16) + 64 + wg * 64;   // cols 64.. (MMA A uses 0..63)
        unsigned long long t0 = clock64();
        for (int it = 0; it < conv_groups; ++it) {
            const int qq = it & 1;
            const uint4 L = sLut[(sW[qq * 8192 + r] + it) & 0x7F];
            const uint32_t N0 = L.z & 0x7F7F7F7Fu, N1 = L.w & 0x7F7F7F7Fu;
            const uint8_t* wrow = sW + qq * 8192 + r * 16;
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
            ptx::tmem_wait_st();
        }
        unsigned long long t1 = clock64();
        if (r == 0) out[blockIdx.x * 8 + wg] = t1 - t0;
        if (r == 96) out[blockIdx.x * 8 + 3 + wg] = t1 - t0;
    } else if (warp == 4 * NCONV) {
        const uint32_t idesc = (1u << 4) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t bd = desc_sw128(ptx::smem_u32(sX));
        unsigned long long t0 = clock64();
        for (int b = 0; b < mma_blocks; ++b) {
            if (ptx::elect_one()) {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    ptx::mma_f8f6f4_ts(tmem + 480, tmem + (j & 7) * 8, bd + (uint64_t)((j & 3) * 2), idesc, 1u);
                if ((b & 3) == 3) ptx::mma_commit(&bar);
            }
            __syncwarp();
            if ((b & 3) == 3) ptx::mbar_wait(&bar, (b >> 2) & 1);
        }
        unsigned long long t1 = clock64();
        if ((threadIdx.x & 31) == 0) out[blockIdx.x * 8 + 7] = t1 - t0;
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x < 32) ptx::tmem_dealloc(tmem, 512);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8 * 8);
    const int smem = 16384 + 2048 + 1024 + 4096 + 1024;
    cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int G = 2000, B = 1000;
    for (int mode = 0; mode < 3; ++mode) {
        cudaMemset(d, 0, 148 * 64);
        k<3><<<148, 128 * 3 + 32, smem>>>(mode == 1 ? 0 : G, mode == 0 ? 0 : B, d);
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); return 1; }
        unsigned long long h[8];
        cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
        const char* nm[3] = {"converters alone", "MMA alone", "both"};
        printf("%-18s conv warp0 (MMA's SMSP) %.1f / warp3 %.1f cyc/group (SM, 3 WGs)   mma %.1f cyc/MMA\n", nm[mode],
               mode == 1 ? 0.0 : (double)h[0] / G / 3, mode == 1 ? 0.0 : (double)h[3] / G / 3,
               mode == 0 ? 0.0 : (double)h[7] / (B * 16));
    }
    return 0;
}
