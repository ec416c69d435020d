// common.cuh -- shared device helpers and host-side status plumbing for libfireq.
#pragma once
#include <cstdint>
#include <cstdio>
#include <string>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "../../include/fireq.h"

namespace fireq {

// --------------------------------------------------------------- host status
void set_error(const std::string& msg);
fireq_status_t fail(fireq_status_t st, const std::string& msg);
fireq_status_t check_launch(const char* what);
int sm_count();
int max_smem_optin();

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Launch with programmatic stream serialization (PDL), an optional cluster shape and,
// for grids whose CTAs wait on each other, the cooperative attribute (all CTAs resident).
template <typename Kern, typename... Args>
cudaError_t launch_ex(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t stream, unsigned cluster_x,
                      bool cooperative, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attrs[3];
    unsigned n = 0;
    attrs[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
    if (cluster_x > 1) {
        attrs[n].id = cudaLaunchAttributeClusterDimension;
        attrs[n].val.clusterDim.x = cluster_x;
        attrs[n].val.clusterDim.y = 1;
        attrs[n].val.clusterDim.z = 1;
        ++n;
    }
    if (cooperative) {
        attrs[n].id = cudaLaunchAttributeCooperative;
        attrs[n].val.cooperative = 1;
        ++n;
    }
    cfg.attrs = attrs;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// --------------------------------------------------------------- span tracing
// Profile builds (FIREQ_PROFILE=1): when enabled with fireq_debug_set_spans, every
// launch records {min CTA start, max CTA end} (%globaltimer ns) into the next slot.
unsigned long long* next_span_slot();
#ifndef FIREQ_PROFILE
#define FIREQ_PROFILE 0
#endif
__device__ __forceinline__ unsigned long long span_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void span_begin(unsigned long long* sp) {
#if FIREQ_PROFILE
    if (sp && threadIdx.x == 0) atomicMin(sp, span_now());
#endif
}
__device__ __forceinline__ void span_end(unsigned long long* sp) {
#if FIREQ_PROFILE
    if (sp && threadIdx.x == 0) atomicMax(sp + 1, span_now());
#endif
}

// --------------------------------------------------------------- device math
// E4M3 code -> float, from the bit fields (exact).
__device__ __forceinline__ float e4m3_decode(uint32_t c) {
    const uint32_t e = (c >> 3) & 0xF, f = c & 7;
    const float mag = e ? __int_as_float(((e + 120u) << 23) | (f << 20))  // (1+f/8)*2^(e-7)
                        : (float)f * 0x1p-9f;                              // subnormal f*2^-9
    return (c & 0x80) ? -mag : mag;
}
// float -> E4M3 code, round to nearest even, saturate to +-448 (hardware cvt).
__device__ __forceinline__ uint32_t e4m3_rn(float x) {
    uint16_t r;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(0.0f), "f"(x));
    return r & 0xFFu;
}
// two floats -> two E4M3 codes packed as (hi << 8) | lo
__device__ __forceinline__ uint32_t e4m3x2_rn(float lo, float hi) {
    uint16_t r;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
    return r;
}
// SiLU(g) = g / (1 + exp(-g)) as __fdividef(g, 1.0f + __expf(-g)) computes it, written with
// the flush-to-zero MUFU forms: the non-ftz forms only add denormal range fix-ups, which never
// change this result (1 + a denormal rounds to 1; 1/(1 + e) is denormal only where
// __fdividef returns 0 too).  Bitwise equal for every bf16 g against 4096 bf16 u
// (scripts/silu_ftz_identity.cu, 0 mismatches on the B200).
__device__ __forceinline__ float ex2_ftz(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_ftz(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float silu_f(float g) {
    return __fmul_rn(g, rcp_ftz(__fadd_rn(1.0f, ex2_ftz(__fmul_rn(-g, 1.4426950408889634f)))));
}

// 2^-n for 0 <= n <= 126, exact.
__device__ __forceinline__ float exp2_neg(int n) { return __int_as_float((127 - n) << 23); }

}  // namespace fireq
