// p2p.cu -- completion signalling of the comm-fused column-parallel layer
// (fireq_w4a8_gemm_colpar_p2p).  The GEMM has stored this rank's Y^T slice into every rank's
// symmetric buffer over NVLink (CUDA-IPC mappings, gemm.cu); this one-CTA kernel, launched
// after it in stream order, advances the local call counter (flag word 63; every rank advances
// its own once per call, so all agree on the epoch -- also across CUDA-graph replays, where a
// host-side epoch would be frozen), publishes the epoch in every peer's flag area (release,
// system scope: the GEMM's stores happen before it, so a peer that acquires the flag sees them)
// and waits until every peer has published it here (acquire): then the full Y^T is local.
// It replaces the NCCL all-gather (north_star (d)).
#include "common.cuh"

namespace fireq {
namespace {

__global__ void k_symm_signal_wait(unsigned* const* __restrict__ flags, int nranks, int rank) {
    __shared__ unsigned s_epoch;
    const int q = threadIdx.x;
    if (q == 0) {
        unsigned* counter = flags[rank] + 63;
        s_epoch = *counter + 1u;
        *counter = s_epoch;
    }
    __syncthreads();
    const unsigned epoch = s_epoch;
    if (q >= nranks) return;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flags[q] + rank), "r"(epoch) : "memory");
    const unsigned* mine = flags[rank] + q;
    unsigned v;
    do {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
        if (v < epoch) __nanosleep(64);
    } while (v < epoch);
}

}  // namespace

fireq_status_t symm_signal_wait(unsigned* const* flag_ptrs, int nranks, int rank, cudaStream_t stream) {
    // a plain launch (no programmatic serialization): the GEMM before it has completed
    k_symm_signal_wait<<<1, 32, 0, stream>>>(flag_ptrs, nranks, rank);
    return check_launch("fireq_w4a8_gemm_colpar_p2p (signal/wait)");
}

}  // namespace fireq
