// stream_ldgsts.cu -- the stream_microbench.cu ring, filled by the warp's 32 lanes with 16-byte
// cp.async (LDGSTS) copies instead of one TMA bulk copy per stage: is the TMA engine's per-SM
// issue rate what caps a one-CTA-per-SM weight stream?  (not product code)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sl scripts/stream_ldgsts.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su32(b)),
                 "r"(ph) : "memory");
}
__device__ __forceinline__ void cp16_plain(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void arrive_noinc(uint64_t* b) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(b)) : "memory");
}

// WARPS warps per CTA each own a ring of `stages` chunks (chunk bytes each) of the CTA's range.
__global__ void k_stream(const uint8_t* src, size_t total, int chunk, int stages, int warps, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* ring = sm + (size_t)w * stages * chunk;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)warps * stages * chunk) + w * stages;
    const long long nch = total / chunk;
    const long long per_cta0 = nch * blockIdx.x / gridDim.x, per_cta1 = nch * (blockIdx.x + 1) / gridDim.x;
    const long long c0 = per_cta0 + (per_cta1 - per_cta0) * w / warps, c1 = per_cta0 + (per_cta1 - per_cta0) * (w + 1) / warps;
    if (lane == 0) {
        for (int i = 0; i < stages; ++i) mbar_init(&bars[i], 32);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    long long issued = c0;
    auto issue = [&](int i, long long c) {
        const uint8_t* g = src + c * chunk;
        uint8_t* d = ring + (size_t)i * chunk;
        for (int off = lane * 16; off < chunk; off += 512) cp16_plain(d + off, g + off);
        arrive_noinc(&bars[i]);
    };
    for (int i = 0; i < stages && issued < c1; ++i, ++issued) issue(i, issued);
    for (long long c = c0; c < c1; ++c) {
        const int i = (c - c0) % stages;
        wait(&bars[i], ((c - c0) / stages) & 1);
        __syncwarp();
        if (issued < c1) { issue(i, issued); ++issued; }
    }
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (lane == 0) {
        out[(blockIdx.x * warps + w) * 2] = t0;
        out[(blockIdx.x * warps + w) * 2 + 1] = t1;
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
    cudaMalloc(&out, 148 * 16 * 16);
    static unsigned long long h[148 * 16 * 2];
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Cfg { int chunk, stages, warps; } cfgs[] = {{16384, 8, 1}, {16384, 6, 2}, {8192, 6, 4}, {8192, 3, 8}, {4096, 6, 8}};
    for (auto cf : cfgs) {
        const int smem = cf.warps * cf.stages * cf.chunk + cf.warps * cf.stages * 8;
        cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        float best = 1e9, span_best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            cudaMemset(flush, rep, flush_n);
            cudaEventRecord(e0);
            k_stream<<<148, 32 * cf.warps, smem>>>(src, total, cf.chunk, cf.stages, cf.warps, out);
            cudaEventRecord(e1);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const int n = 148 * cf.warps;
            cudaMemcpy(h, out, n * 16, cudaMemcpyDeviceToHost);
            unsigned long long lo = ~0ull, hi = 0;
            for (int b = 0; b < n; ++b) { lo = h[2 * b] < lo ? h[2 * b] : lo; hi = h[2 * b + 1] > hi ? h[2 * b + 1] : hi; }
            if (rep > 0) {
                best = ms * 1e3f < best ? ms * 1e3f : best;
                span_best = (hi - lo) / 1e3f < span_best ? (hi - lo) / 1e3f : span_best;
            }
        }
        printf("LDGSTS warps %d chunk %6d stages %d (in flight/CTA %7d): event %.2f us, device span %.2f us -> %.0f GB/s\n",
               cf.warps, cf.chunk, cf.stages, cf.warps * cf.stages * cf.chunk, best, span_best, total / (span_best * 1e3));
    }
    return 0;
}
