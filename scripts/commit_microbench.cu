// commit_microbench.cu -- cost of tcgen05.commit between tcgen05.mma (not product code):
// one warp issues R MMAs (kind::f8f6f4, M=128, N=16, K=32, A from TMEM) with a commit to an
// mbarrier after every k MMAs (k = 1 .. 32); cycles per MMA.
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

template <int MODE>   // 0: elect per MMA; 1: lane 0 alone (other lanes idle at a barrier), no elect;
                     // 2: elect per 8 unrolled MMAs
__global__ void k(int reps, int every, int nbars, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bars[8];
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) smem[i] = 0x38;
    if (threadIdx.x == 0) { for (int i = 0; i < 8; ++i) ptx::mbar_init(&bars[i], 1); ptx::fence_mbar_init(); }
    if (threadIdx.x < 32) { ptx::tmem_alloc(&tbase, 512); ptx::tmem_relinquish(); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tm = tbase;
    if (threadIdx.x < 32) {
        const uint32_t idesc = (1u << 4) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t bd = desc_sw128(ptx::smem_u32(smem));
        unsigned long long t0 = clock64();
        int nc = 0;
        if (MODE == 0) {
            for (int i = 0; i < reps; ++i) {
                if (ptx::elect_one()) {
                    ptx::mma_f8f6f4_ts(tm, tm + 64 + (i & 7) * 8, bd + (uint64_t)((i & 3) * 2), idesc, 1);
                    if ((i + 1) % every == 0) {
                        for (int b = 0; b < nbars; ++b) ptx::mma_commit(&bars[b]);
                    }
                }
                __syncwarp();
                if ((i + 1) % every == 0) ++nc;
            }
            if (ptx::elect_one()) ptx::mma_commit(&bars[7]);
            __syncwarp();
        } else if (MODE == 1) {
            if (threadIdx.x == 0) {
                for (int i = 0; i < reps; ++i) {
                    ptx::mma_f8f6f4_ts(tm, tm + 64 + (i & 7) * 8, bd + (uint64_t)((i & 3) * 2), idesc, 1);
                    if ((i + 1) % every == 0) {
                        for (int b = 0; b < nbars; ++b) ptx::mma_commit(&bars[b]);
                    }
                }
                ptx::mma_commit(&bars[7]);
            }
            __syncwarp();
        } else {
            for (int i = 0; i < reps; i += 8) {
                if (ptx::elect_one()) {
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        ptx::mma_f8f6f4_ts(tm, tm + 64 + j * 8, bd + (uint64_t)((j & 3) * 2), idesc, 1);
                    if ((i + 8) % every == 0) {
                        for (int b = 0; b < nbars; ++b) ptx::mma_commit(&bars[b]);
                    }
                }
                __syncwarp();
            }
            if (ptx::elect_one()) ptx::mma_commit(&bars[7]);
            __syncwarp();
        }
        ptx::mbar_wait(&bars[7], 0);
        unsigned long long t1 = clock64();
        if (threadIdx.x == 0) out[0] = t1 - t0;
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x < 32) ptx::tmem_dealloc(tm, 512);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 64);
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
    cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
    const int reps = 4096;
    for (int mode = 0; mode < 3; ++mode)
    for (int nb : {1, 3})
        for (int every : {1, 8, 16, 100000}) {
            if (mode == 2 && every < 8) continue;
            if (mode == 0) k<0><<<1, 128, 20000>>>(reps, every, nb, d);
            if (mode == 1) k<1><<<1, 128, 20000>>>(reps, every, nb, d);
            if (mode == 2) k<2><<<1, 128, 20000>>>(reps, every, nb, d);
            if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); return 1; }
            unsigned long long h;
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("mode %d commit x%d every %6d MMAs: %.2f cyc/MMA\n", mode, nb, every, (double)h / reps);
        }
    return 0;
}
