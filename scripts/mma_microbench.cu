// mma_microbench.cu -- day-1 B200 microbenchmarks (not product code):
//  (1) tcgen05.mma.kind::f8f6f4 issue/completion rate, A from TMEM (TS) vs SMEM (SS),
//      M = 128, N in {16..256}, K = 32 per instruction;
//  (2) commit -> mbarrier round-trip latency;
//  (3) ALU-pipe throughput of PRMT / LOP3 and FMA-pipe IMAD.HI per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_microbench mma_microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda.h>
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
__device__ __forceinline__ uint32_t elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}" : "=r"(pred));
    return pred;
}
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc) : "memory");
}

__global__ void k_mma_rate(int ntok, int ss, int reps, int nacc, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 64 * 1024; i += blockDim.x) smem[i] = 0x38;   // 1.0 in e4m3
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    if (warp == 0) { ptx::tmem_alloc(&tbase, 512); ptx::tmem_relinquish(); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tm = tbase;
    if (warp == 0) {
        const uint32_t idesc = (1u << 4) | ((uint32_t)(ntok >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t bd = desc_sw128(ptx::smem_u32(smem));
        const uint64_t ad = desc_sw128(ptx::smem_u32(smem + 32768));
        // warm
        for (int i = 0; i < 8; ++i) {
            if (elect_one()) { if (ss) mma_ss(tm, ad, bd, idesc, i); else ptx::mma_f8f6f4_ts(tm, tm + 256, bd, idesc, i); }
            __syncwarp();
        }
        if (elect_one()) ptx::mma_commit(&bar);
        __syncwarp();
        ptx::mbar_wait(&bar, 0);
        // commit round trip latency (1 MMA)
        unsigned long long t0 = clock64();
        if (elect_one()) { if (ss) mma_ss(tm, ad, bd, idesc, 1); else ptx::mma_f8f6f4_ts(tm, tm + 256, bd, idesc, 1);
        ptx::mma_commit(&bar); }
        __syncwarp();
        ptx::mbar_wait(&bar, 1);
        unsigned long long t1 = clock64();
        // throughput
        for (int i = 0; i < reps; ++i) {
            const uint64_t b2 = bd + (uint64_t)((i & 3) * 2);
            const uint32_t dcol = tm + (uint32_t)((i % nacc) * ntok);
            if (elect_one()) {
            if (ss) mma_ss(dcol, ad + (uint64_t)((i & 3) * 2), b2, idesc, 1);
            else ptx::mma_f8f6f4_ts(dcol, tm + 256 + (i & 7) * 8, b2, idesc, 1);
            }
            __syncwarp();
        }
        if (elect_one()) ptx::mma_commit(&bar);
        __syncwarp();
        ptx::mbar_wait(&bar, 0);
        unsigned long long t2 = clock64();
        // unrolled: 32 MMAs per elected block, operands hoisted
        const uint32_t ta0 = tm + 256;
        for (int i = 0; i < reps / 32; ++i) {
            if (elect_one()) {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    if (ss) mma_ss(tm, ad + (uint64_t)((j & 3) * 2), bd + (uint64_t)((j & 3) * 2), idesc, 1);
                    else ptx::mma_f8f6f4_ts(tm, ta0 + (j & 7) * 8, bd + (uint64_t)((j & 3) * 2), idesc, 1);
                }
            }
            __syncwarp();
        }
        if (elect_one()) ptx::mma_commit(&bar);
        __syncwarp();
        ptx::mbar_wait(&bar, 1);
        unsigned long long t3 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x * 2 + 2] = t3 - t2;
        if (threadIdx.x == 0) { out[blockIdx.x * 2 + 0] = t1 - t0;
        out[blockIdx.x * 2 + 1] = t2 - t1; }
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc(tm, 512);
}

// ALU pipe throughput: each thread runs independent chains of prmt (or lop3 / imad.hi).
template <int OP>
__global__ void k_alu(int iters, uint32_t seed, uint32_t* sink, unsigned long long* cyc) {
    uint32_t a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = seed * (i + 1) + threadIdx.x;
    const uint32_t L0 = seed ^ 0x12345678u, L1 = seed ^ 0x9abcdef0u;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) a[i] = ptx::prmt(L0, L1, a[i]);
            else if (OP == 1) a[i] = ptx::lop3_mux(a[i], L0, L1);
            else if (OP == 2) a[i] = ptx::hi16_fma(a[i]) + 0;
            else { a[i] = ptx::prmt(L0, L1, a[i]); a[i] = ptx::hi16_fma(a[i]); }
        }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s ^= a[i];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 1024 * 8);
    unsigned long long h[4];
    cudaFuncSetAttribute(k_mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    const int reps = 4096;
    for (int ss = 0; ss < 2; ++ss) {
        for (int ntok : {16, 32, 64, 128, 256}) for (int nacc : {1, 2, 4, 8}) {
            if (ntok * nacc > 256) continue;
            k_mma_rate<<<1, 128, 80 * 1024>>>(ntok, ss, reps, nacc, d);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
            printf("mma %s M=128 N=%3d K=32 nacc=%d: commit-roundtrip %llu cyc, %.2f cyc/MMA  (%.0f MAC/cyc)\n",
                   ss ? "SS" : "TS", ntok, nacc, h[0], (double)h[1] / reps, 128.0 * ntok * 32 * reps / h[1]);
            printf("      unrolled x32: %.2f cyc/MMA (%.0f MAC/cyc)\n", (double)h[2] / reps, 128.0 * ntok * 32 * reps / h[2]);
        }
    }
    uint32_t* sink;
    cudaMalloc(&sink, 148 * 1024 * 4);
    const char* names[4] = {"PRMT", "LOP3", "IMAD.HI", "PRMT+IMAD.HI"};
    for (int op = 0; op < 4; ++op) {
        const int iters = 4096, threads = 1024;
        if (op == 0) k_alu<0><<<148, threads>>>(iters, 7, sink, d);
        if (op == 1) k_alu<1><<<148, threads>>>(iters, 7, sink, d);
        if (op == 2) k_alu<2><<<148, threads>>>(iters, 7, sink, d);
        if (op == 3) k_alu<3><<<148, threads>>>(iters, 7, sink, d);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        const double ops = (double)iters * 8 * threads * (op == 3 ? 2 : 1);
        printf("%-14s %.1f thread-ops/cycle/SM\n", names[op], ops / h[0]);
    }
    return 0;
}
