// conv_tput.cu -- converter throughput microbenchmark (not product code).
// NCONV converter warpgroups per CTA (one CTA per SM) convert packed INT4 rows from
// shared memory into TMEM (the GEMM's A operand) in a loop, with no MMA and no
// barriers: cycles per 128x128 group is the converter's steady-state cost.
// Variants: sign-split (SS) / mask-select (MS); tcgen05.wait::st per stage or not;
// STTM asm with or without a "memory" clobber.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2505_20839_b200/csrc/ptx.cuh"
using namespace fireq;

__device__ __forceinline__ void sttm8_nomem(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                 ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
}
__device__ __forceinline__ void sttm4_nomem(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};"
                 ::"r"(taddr), "r"(a), "r"(b), "r"(c), "r"(d));
}
__device__ __forceinline__ void conv_ss(uint32_t w, uint32_t L0, uint32_t L1, uint32_t N0, uint32_t N1,
                                        uint32_t& p0, uint32_t& p1, uint32_t& n0, uint32_t& n1) {
    const uint32_t x = w ^ 0x88888888u;
    const uint32_t wh = ptx::hi16_prmt(w), xh = ptx::hi16_prmt(x);
    p0 = ptx::prmt(L0, L1, w); p1 = ptx::prmt(L0, L1, wh);
    n0 = ptx::prmt(N0, N1, x); n1 = ptx::prmt(N0, N1, xh);
}
__device__ __forceinline__ void conv_ms(uint32_t w, uint32_t L0, uint32_t L1, uint32_t L2, uint32_t L3,
                                        uint32_t& r0, uint32_t& r1) {
    const uint32_t x = w ^ 0x88888888u;
    const uint32_t t = ptx::shl4_fma(w);
    const uint32_t wh = ptx::hi16_prmt(w), xh = ptx::hi16_prmt(x);
    const uint32_t m0 = ptx::prmt(w, t, 0x9D8Cu), m1 = ptx::prmt(w, t, 0xBFAEu);
    r0 = ptx::lop3_mux(ptx::prmt(L0, L1, w), ptx::prmt(L2, L3, x), m0);
    r1 = ptx::lop3_mux(ptx::prmt(L0, L1, wh), ptx::prmt(L2, L3, xh), m1);
}

template <int NCONV, bool SS, bool WAITST, bool MEMCLOB, int GPS>
__global__ void __launch_bounds__(128 * NCONV) k_conv(int stages, unsigned long long* out, uint32_t* sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tbase;
    uint8_t* sW = smem;                                // [2][8 KB] packed
    uint4* sLut = reinterpret_cast<uint4*>(smem + 2 * 8192);
    uint8_t* sS = smem + 2 * 8192 + 2048;
    for (int i = threadIdx.x; i < 2 * 8192; i += blockDim.x) sW[i] = (uint8_t)(i * 37 + 11);
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) reinterpret_cast<uint8_t*>(sLut)[i] = (uint8_t)(i & 0x7F);
    for (int i = threadIdx.x; i < 2 * 128; i += blockDim.x) sS[i] = (uint8_t)(40 + (i & 15));
    if (threadIdx.x < 32) { ptx::tmem_alloc(&tbase, 512); ptx::tmem_relinquish(); }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tbase;
    const int wg = threadIdx.x >> 7, r = threadIdx.x & 127;
    const uint32_t lane_base = (uint32_t)(r & ~31) << 16;
    constexpr int kASz = GPS * (SS ? 64 : 32);
    const uint32_t ta = tmem + lane_base + (uint32_t)(wg * kASz);
    unsigned long long t0 = clock64();
    for (int it = 0; it < stages; ++it) {
#pragma unroll
        for (int q = 0; q < GPS; ++q) {
            // every input changes with the iteration (loop-invariant conversions would be hoisted)
            const int qq = (q + it) & 1;
            const uint4 L = sLut[sS[qq * 128 + r] & 0x7F];
            const uint8_t* wrow = sW + qq * 8192 + r * 16;
            if (SS) {
                const uint32_t N0 = L.z & 0x7F7F7F7Fu, N1 = L.w & 0x7F7F7F7Fu;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint4 wv = *reinterpret_cast<const uint4*>(wrow + j * 128 * 16);
                    uint32_t P[8], Q[8];
                    conv_ss(wv.x, L.x, L.y, N0, N1, P[0], P[1], Q[0], Q[1]);
                    conv_ss(wv.y, L.x, L.y, N0, N1, P[2], P[3], Q[2], Q[3]);
                    conv_ss(wv.z, L.x, L.y, N0, N1, P[4], P[5], Q[4], Q[5]);
                    conv_ss(wv.w, L.x, L.y, N0, N1, P[6], P[7], Q[6], Q[7]);
                    if (MEMCLOB) {
                        ptx::tmem_st_x8(ta + (q * 4 + j) * 8, P);
                        ptx::tmem_st_x8(ta + GPS * 32 + (q * 4 + j) * 8, Q);
                    } else {
                        sttm8_nomem(ta + (q * 4 + j) * 8, P);
                        sttm8_nomem(ta + GPS * 32 + (q * 4 + j) * 8, Q);
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint4 wv = *reinterpret_cast<const uint4*>(wrow + j * 128 * 16);
                    uint32_t R[8];
                    conv_ms(wv.x, L.x, L.y, L.z, L.w, R[0], R[1]);
                    conv_ms(wv.y, L.x, L.y, L.z, L.w, R[2], R[3]);
                    conv_ms(wv.z, L.x, L.y, L.z, L.w, R[4], R[5]);
                    conv_ms(wv.w, L.x, L.y, L.z, L.w, R[6], R[7]);
                    if (MEMCLOB) ptx::tmem_st_x8(ta + (q * 4 + j) * 8, R);
                    else sttm8_nomem(ta + (q * 4 + j) * 8, R);
                }
            }
        }
        if (WAITST) ptx::tmem_wait_st();
    }
    ptx::tmem_wait_st();
    __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x < 32) ptx::tmem_dealloc(tmem, 512);
}

template <int NCONV, bool SS, bool WAITST, bool MEMCLOB, int GPS>
void run(const char* name, unsigned long long* d, uint32_t* sink) {
    auto k = k_conv<NCONV, SS, WAITST, MEMCLOB, GPS>;
    const int smem = 2 * 8192 + 2048 + 2 * 128 + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int stages = 2000;
    k<<<148, 128 * NCONV, smem>>>(stages, d, sink);
    k<<<148, 128 * NCONV, smem>>>(stages, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0; for (int i = 0; i < 148; ++i) s += h[i];
    const double cyc = s / 148 / stages;
    printf("%-40s %7.1f cyc/stage  %7.1f cyc/group (per SM, %d WGs converting concurrently)\n", name, cyc,
           cyc / (GPS * NCONV), NCONV);
}

int main() {
    unsigned long long* d; uint32_t* sink;
    cudaMalloc(&d, 148 * 8); cudaMalloc(&sink, 4096);
    run<3, true, true, true, 2>("SS NCONV3 GPS2 waitst memclob (current)", d, sink);
    run<3, true, false, true, 2>("SS NCONV3 GPS2 no-waitst memclob", d, sink);
    run<3, true, true, false, 2>("SS NCONV3 GPS2 waitst no-memclob", d, sink);
    run<3, true, false, false, 2>("SS NCONV3 GPS2 no-waitst no-memclob", d, sink);
    run<2, true, true, false, 2>("SS NCONV2 GPS2 waitst no-memclob", d, sink);
    run<4, true, true, false, 1>("SS NCONV4 GPS1 waitst no-memclob", d, sink);
    run<1, true, true, false, 2>("SS NCONV1 GPS2 waitst no-memclob", d, sink);
    run<3, false, true, true, 2>("MS NCONV3 GPS2 waitst memclob", d, sink);
    run<3, false, true, false, 2>("MS NCONV3 GPS2 waitst no-memclob", d, sink);
    run<2, false, true, false, 2>("MS NCONV2 GPS2 waitst no-memclob", d, sink);
    run<4, false, true, false, 2>("MS NCONV4 GPS2 waitst no-memclob", d, sink);
    return 0;
}
