// How fast can 148 persistent CTAs stream a decode layer's weights (46 MB) through a
// bulk-copy ring?  Pure load pipeline: TMA bulk copy -> mbarrier -> consumer releases
// the slot at once.  Sweeps chunk size and bytes in flight per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/stream_microbench scripts/stream_microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su32(b)),
                 "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)), "l"(pol) : "memory");
}

__global__ void k_stream(const uint8_t* src, size_t total, int chunk, int stages, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + stages * chunk);
    const long long nch = total / chunk;
    const long long c0 = nch * blockIdx.x / gridDim.x, c1 = nch * (blockIdx.x + 1) / gridDim.x;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    if (threadIdx.x == 0) {
        for (int i = 0; i < stages; ++i) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        unsigned long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        long long issued = c0;
        for (int i = 0; i < stages && issued < c1; ++i, ++issued) {
            expect_tx(&bars[i], chunk);
            bulk(sm + i * chunk, src + issued * chunk, chunk, &bars[i], pol);
        }
        for (long long c = c0; c < c1; ++c) {
            const int i = (c - c0) % stages;
            wait(&bars[i], ((c - c0) / stages) & 1);
            if (issued < c1) {
                expect_tx(&bars[i], chunk);
                bulk(sm + i * chunk, src + issued * chunk, chunk, &bars[i], pol);
                ++issued;
            }
        }
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        out[blockIdx.x * 2] = t0;
        out[blockIdx.x * 2 + 1] = t1;
    }
}

int main() {
    const size_t total = 46ull << 20;
    const size_t flush_n = 512ull << 20;
    uint8_t *src, *flush;
    cudaMalloc(&src, total);
    cudaMalloc(&flush, flush_n);
    cudaMemset(src, 1, total);
    unsigned long long* out;
    cudaMalloc(&out, 4096 * 16);
    unsigned long long h[4096 * 2];
    int chunks[] = {8192, 16384, 32768};
    int inflight[] = {65536, 98304, 131072, 163840, 196608};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int grid_mul = 1; grid_mul <= 2; ++grid_mul)
    for (int ch : chunks)
        for (int inf : inflight) {
            const int stages = inf / ch;
            const int smem = stages * ch + 64 * 8;
            if (grid_mul == 2 && smem > 110 * 1024) continue;
            cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            const int grid = 148 * grid_mul;
            float best = 1e9, span_best = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                cudaMemset(flush, rep, flush_n);
                cudaEventRecord(e0);
                k_stream<<<grid, 32, smem>>>(src, total, ch, stages, out);
                cudaEventRecord(e1);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                cudaMemcpy(h, out, grid * 16, cudaMemcpyDeviceToHost);
                unsigned long long lo = ~0ull, hi = 0;
                for (int b = 0; b < grid; ++b) { lo = h[2 * b] < lo ? h[2 * b] : lo; hi = h[2 * b + 1] > hi ? h[2 * b + 1] : hi; }
                if (rep > 0) {
                    best = ms * 1e3f < best ? ms * 1e3f : best;
                    span_best = (hi - lo) / 1e3f < span_best ? (hi - lo) / 1e3f : span_best;
                }
            }
            printf("grid %3d chunk %6d inflight/CTA %7d: event %.2f us, device span %.2f us -> %.0f GB/s\n", grid, ch,
                   inf, best, span_best, total / (span_best * 1e3));
        }
    return 0;
}
