// conv_microbench.cu -- B200 microbenchmarks (not product code) for the decode GEMM:
//  (1) INT4 -> FP8 converter throughput (sign-split / mask-select), SMEM -> registers -> TMEM,
//      128 threads per warpgroup, 1..4 warpgroups, with and without the tcgen05.st / wait::st;
//  (2) tcgen05.mma f8f6f4 N=16 rate when alternating the negate bit and moving B.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o conv_microbench conv_microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_2505_20839_b200/csrc/ptx.cuh"

using namespace fireq;

__device__ __forceinline__ void conv_ss(uint32_t w, uint32_t L0, uint32_t L1, uint32_t N0, uint32_t N1,
                                        uint32_t& p0, uint32_t& p1, uint32_t& n0, uint32_t& n1) {
    const uint32_t x = w ^ 0x88888888u;
    const uint32_t wh = ptx::hi16_fma(w);
    const uint32_t xh = ptx::hi16_fma(x);
    p0 = ptx::prmt(L0, L1, w);
    p1 = ptx::prmt(L0, L1, wh);
    n0 = ptx::prmt(N0, N1, x);
    n1 = ptx::prmt(N0, N1, xh);
}

__device__ __forceinline__ void conv_ms(uint32_t w, uint32_t L0, uint32_t L1, uint32_t L2, uint32_t L3,
                                        uint32_t& r0, uint32_t& r1) {
    const uint32_t x = w ^ 0x88888888u;
    const uint32_t t = ptx::shl4_fma(w);
    const uint32_t wh = ptx::hi16_fma(w);
    const uint32_t xh = ptx::hi16_fma(x);
    const uint32_t m0 = ptx::prmt(w, t, 0x9D8Cu);
    const uint32_t m1 = ptx::prmt(w, t, 0xBFAEu);
    r0 = ptx::lop3_mux(ptx::prmt(L0, L1, w), ptx::prmt(L2, L3, x), m0);
    r1 = ptx::lop3_mux(ptx::prmt(L0, L1, wh), ptx::prmt(L2, L3, xh), m1);
}

// mask-select converter: one operand, 8 words per 32-element chunk
__global__ void k_conv_ms(int groups, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint32_t tbase;
    uint8_t* sW = smem_raw;
    uint8_t* sS = smem_raw + 32768;
    uint4* sLut = reinterpret_cast<uint4*>(smem_raw + 32768 + 1024);
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 32768; i += blockDim.x) sW[i] = (uint8_t)(i * 37 + 11);
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sS[i] = (uint8_t)(i % 120);
    for (int i = threadIdx.x; i < 127 * 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sLut)[i] = i * 0x01010101u;
    if (warp == 0) { ptx::tmem_alloc(&tbase, 512); ptx::tmem_relinquish(); }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tm = tbase;
    const int r = threadIdx.x & 127;
    const int wg = threadIdx.x >> 7;
    const uint32_t lane_base = (uint32_t)(r & ~31) << 16;
    unsigned long long t0 = clock64();
    for (int gi = wg; gi < groups; gi += blockDim.x / 128) {
        const int s = gi & 3;
        const uint4 L = sLut[sS[s * 128 + r]];
        const uint8_t* wrow = sW + s * 8192 + r * 16;
        const uint32_t ta = tm + lane_base + (wg & 3) * 32;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint4 wv = *reinterpret_cast<const uint4*>(wrow + j * 128 * 16);
            uint32_t R[8];
            conv_ms(wv.x, L.x, L.y, L.z, L.w, R[0], R[1]);
            conv_ms(wv.y, L.x, L.y, L.z, L.w, R[2], R[3]);
            conv_ms(wv.z, L.x, L.y, L.z, L.w, R[4], R[5]);
            conv_ms(wv.w, L.x, L.y, L.z, L.w, R[6], R[7]);
            ptx::tmem_st_x8(ta + j * 8, R);
        }
        ptx::tmem_wait_st();
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc(tm, 512);
}

// mode bit0: skip tcgen05.st (sum into a register instead); bit1: skip wait::st
template <int MODE>
__global__ void k_conv(int groups, uint32_t* sink, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint32_t tbase;
    uint8_t* sW = smem_raw;                        // 4 stages x 8 KB packed
    uint8_t* sS = smem_raw + 32768;                // sigma codes
    uint4* sLut = reinterpret_cast<uint4*>(smem_raw + 32768 + 1024);
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 32768; i += blockDim.x) sW[i] = (uint8_t)(i * 37 + 11);
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sS[i] = (uint8_t)(i % 120);
    for (int i = threadIdx.x; i < 127 * 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sLut)[i] = i * 0x01010101u;
    if (warp == 0) { ptx::tmem_alloc(&tbase, 512); ptx::tmem_relinquish(); }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tm = tbase;
    const int r = threadIdx.x & 127;
    const int wg = threadIdx.x >> 7;
    const uint32_t lane_base = (uint32_t)(r & ~31) << 16;
    uint32_t acc = 0;
    unsigned long long t0 = clock64();
    for (int gi = wg; gi < groups; gi += blockDim.x / 128) {
        const int s = gi & 3;
        const uint4 L = sLut[sS[s * 128 + r]];
        const uint32_t N0 = L.z & 0x7F7F7F7Fu, N1 = L.w & 0x7F7F7F7Fu;
        const uint8_t* wrow = sW + s * 8192 + r * 16;
        const uint32_t ta = tm + lane_base + (wg & 3) * 64;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint4 wv = *reinterpret_cast<const uint4*>(wrow + j * 128 * 16);
            uint32_t P[8], Q[8];
            conv_ss(wv.x, L.x, L.y, N0, N1, P[0], P[1], Q[0], Q[1]);
            conv_ss(wv.y, L.x, L.y, N0, N1, P[2], P[3], Q[2], Q[3]);
            conv_ss(wv.z, L.x, L.y, N0, N1, P[4], P[5], Q[4], Q[5]);
            conv_ss(wv.w, L.x, L.y, N0, N1, P[6], P[7], Q[6], Q[7]);
            if (MODE & 1) {
#pragma unroll
                for (int k = 0; k < 8; ++k) acc += P[k] ^ Q[k];
            } else {
                ptx::tmem_st_x8(ta + j * 8, P);
                ptx::tmem_st_x8(ta + 32 + j * 8, Q);
            }
        }
        if (!(MODE & 3)) ptx::tmem_wait_st();
    }
    unsigned long long t1 = clock64();
    if (!(MODE & 1)) ptx::tmem_wait_st();
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc(tm, 512);
}

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// MMA rate: variant 0 = same idesc, same B; 1 = alternate negate; 2 = B moves every 2 MMAs;
// 3 = like the kernel's stage: 2 groups x 4 k-steps x {pos, neg}, then 2 commits.
__global__ void k_mma(int variant, int reps, int abase, int dbase, unsigned long long* out, int sttm) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) smem_raw[i] = 0x38;
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    if (warp == 0) { ptx::tmem_alloc(&tbase, 512); ptx::tmem_relinquish(); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tm = tbase;
    if (warp == 0) {
        const uint32_t ip = (1u << 4) | (2u << 17) | (8u << 24);
        const uint32_t in = ip | (1u << 13);
        const uint32_t sb = ptx::smem_u32(smem_raw);
        unsigned long long t0 = clock64();
        for (int it = 0; it < reps; ++it) {
            if (ptx::elect_one()) {
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const uint64_t bdesc = desc_sw128(sb + (variant >= 2 ? q * 2048 + (it & 1) * 4096 : 0));
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint64_t bd = bdesc + (uint64_t)(j * 2);
                        ptx::mma_f8f6f4_ts(tm + dbase, tm + abase + (q * 4 + j) * 8, bd, ip, 1u);
                        ptx::mma_f8f6f4_ts(tm + dbase, tm + abase + 64 + (q * 4 + j) * 8, bd, variant == 0 ? ip : in, 1u);
                    }
                }
                if (variant == 3) { ptx::mma_commit(&bar); ptx::mma_commit(&bar); }
            }
            __syncwarp();
        }
        if (ptx::elect_one()) ptx::mma_commit(&bar);
        __syncwarp();
        ptx::mbar_wait(&bar, 0);
        unsigned long long t1 = clock64();
        if (threadIdx.x == 0) out[0] = t1 - t0;
        if (threadIdx.x == 0) *((volatile int*)&smem_raw[20000]) = 1;
    } else if (sttm && warp >= 4) {
        // background TMEM stores (like converter warps), columns 384..447
        const uint32_t lb = (uint32_t)((warp & 3) * 32) << 16;
        uint32_t v[8] = {1, 2, 3, 4, 5, 6, 7, 8};
        for (int it = 0; it < reps * 4; ++it) {
            ptx::tmem_st_x8(tm + lb + 384 + (it & 7) * 8, v);
            if ((it & 7) == 7) ptx::tmem_wait_st();
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc(tm, 512);
}

// Converter warpgroups (warps 0..11) and one MMA warp (warp 12) running concurrently.
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__global__ void k_mix(int groups, int reps, int conv_on, unsigned long long* out, int fence_mode) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint32_t tbase;
    __shared__ uint64_t bar;
    uint8_t* sW = smem_raw;
    uint8_t* sS = smem_raw + 32768;
    uint4* sLut = reinterpret_cast<uint4*>(smem_raw + 32768 + 1024);
    uint8_t* sB = smem_raw + 40960;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 32768; i += blockDim.x) sW[i] = (uint8_t)(i * 37 + 11);
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sS[i] = (uint8_t)(i % 120);
    for (int i = threadIdx.x; i < 127 * 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sLut)[i] = i * 0x01010101u;
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) sB[i] = 0x38;
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    if (warp == 0) { ptx::tmem_alloc(&tbase, 512); ptx::tmem_relinquish(); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tm = tbase;
    if (warp < 12 && conv_on) {
        const int r = threadIdx.x & 127;
        const int wg = threadIdx.x >> 7;
        const uint32_t lane_base = (uint32_t)(r & ~31) << 16;
        for (int gi = wg; gi < groups; gi += 3) {
            const int s = gi & 3;
            const uint4 L = sLut[sS[s * 128 + r]];
            const uint32_t N0 = L.z & 0x7F7F7F7Fu, N1 = L.w & 0x7F7F7F7Fu;
            const uint8_t* wrow = sW + s * 8192 + r * 16;
            const uint32_t ta = tm + lane_base + 256 + wg * 64;
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
    }
    if (warp == 12) {
        const uint32_t ip = (1u << 4) | (2u << 17) | (8u << 24);
        const uint32_t in = ip | (1u << 13);
        const uint32_t sb = ptx::smem_u32(sB);
        __shared__ uint64_t bar2;
        if (lane_id() == 0) { ptx::mbar_init(&bar2, 1); ptx::fence_mbar_init(); ptx::mbar_arrive(&bar2); }
        __syncwarp();
        unsigned long long t0 = clock64();
        for (int it = 0; it < reps; ++it) {
            if (fence_mode & 1) ptx::mbar_wait(&bar2, 0);       // completed phase: returns immediately
            if (fence_mode & 2) ptx::tc_fence_after();
            if (ptx::elect_one()) {
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const uint64_t bdesc = desc_sw128(sb + q * 2048 + (it & 1) * 4096);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint64_t bd = bdesc + (uint64_t)(j * 2);
                        ptx::mma_f8f6f4_ts(tm, tm + 32 + (q * 4 + j) * 8, bd, ip, 1u);
                        ptx::mma_f8f6f4_ts(tm, tm + 32 + 64 + (q * 4 + j) * 8, bd, in, 1u);
                    }
                }
                ptx::mma_commit(&bar);
            }
            __syncwarp();
        }
        if (ptx::elect_one()) ptx::mma_commit(&bar);
        __syncwarp();
        unsigned long long t1 = clock64();
        if (threadIdx.x == 384) out[blockIdx.x] = t1 - t0;
        ptx::mbar_wait(&bar, (reps + 1 - 1) & 1);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc(tm, 512);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 1024 * 8);
    uint32_t* sink;
    cudaMalloc(&sink, 148 * 1024 * 4);
    unsigned long long h[4];
    const int smem = 64 * 1024;
    cudaFuncSetAttribute(k_conv<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_conv<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_conv<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int groups = 2048;
    for (int mode = 0; mode < 3; ++mode) {
        for (int wgs : {1, 2, 3, 4}) {
            if (mode == 0) k_conv<0><<<148, 128 * wgs, smem>>>(groups, sink, d);
            if (mode == 1) k_conv<1><<<148, 128 * wgs, smem>>>(groups, sink, d);
            if (mode == 2) k_conv<2><<<148, 128 * wgs, smem>>>(groups, sink, d);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
            printf("conv mode=%d (%s) WGs=%d: %.1f cycles/group/SM  (%.1f el/cycle)\n", mode,
                   mode == 0 ? "sttm+wait" : mode == 1 ? "no sttm" : "sttm, no wait", wgs, (double)h[0] / groups,
                   16384.0 * groups / h[0]);
        }
    }
    cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    cudaFuncSetAttribute(k_conv_ms, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int wgs : {2, 3, 4}) {
        k_conv_ms<<<148, 128 * wgs, smem>>>(groups, d);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        printf("conv mask-select WGs=%d: %.1f cycles/group/SM (%.1f el/cycle)\n", wgs, (double)h[0] / groups, 16384.0 * groups / h[0]);
    }
    for (int st = 0; st < 2; ++st) {
        k_mma<<<148, st ? 256 + 128 * 3 : 128, 32768>>>(3, 512, 256, 0, d, st);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        printf("mma N=16 16-MMA stages with%s concurrent STTM: %.1f cycles per MMA\n", st ? "" : "out", (double)h[0] / (512 * 16));
    }
    cudaFuncSetAttribute(k_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int cv = 0; cv < 8; ++cv) {
        k_mix<<<148, 13 * 32, 64 * 1024>>>(4096, 512, cv & 1, d, cv >> 1);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        printf("mix: MMA issue with%s converters, wait=%d fence=%d: %.1f cycles per MMA (issue-side)\n", (cv & 1) ? "" : "out", (cv >> 1) & 1, (cv >> 2) & 1, (double)h[0] / (512 * 16));
    }
    for (int v = 0; v < 6; ++v) {
        const int reps = 512;
        const int abase = v == 4 ? 32 : v == 5 ? 160 : 256;
        const int dbase = v == 5 ? 16 : 0;
        k_mma<<<v >= 4 ? 148 : 1, 128, 32768>>>(v >= 4 ? 3 : v, reps, abase, dbase, d, 0);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        printf("mma variant %d (abase %d, dbase %d, grid %d): %.1f cycles per MMA (N=16), %.0f cycles per 16-MMA stage\n", v, abase, dbase, v >= 4 ? 148 : 1, (double)h[0] / (reps * 16),
               (double)h[0] / reps);
    }
    return 0;
}
