/*
 * fireq.h -- C ABI of the B200 (sm_100a) FireQ W4A8-FP linear layer.
 *
 * FireQ (arXiv 2505.20839).  Citations: P:NNN = line of the paper text
 * (/root/reference/PAPER.md at build time; not needed at run time).
 *
 * The operation is the linear layer Y = X W^T (Eq. 3) with
 *   - W in bf16 [N][K] (N = N_out, K = N_in) quantized OFFLINE to INT4
 *     codes in [-8, 7] with one FP8-E4M3 scale sigma per 128 consecutive K
 *     elements of a row (Eq. 1), after channel-wise absmean
 *     scaling (CAS, Def. 1) and per-tensor power-of-two scaling
 *     (PTS, Def. 2);
 *   - X in bf16 [M][K] quantized ONLINE to FP8-E4M3 with one BF16 scale beta per
 *     token (Eq. 2);
 *   - the GEMM dequantizing INT4 through a 16-entry FP8 lookup table
 *     {-8 sigma .. 7 sigma} (Step 1), multiplying on FP8 tensor cores
 *     with FP32 accumulation (Step 2) and producing BF16 (Step 3,
 *     P:130), with beta and the PTS inverse 2^-n applied to the output.
 * Exact semantics (every rounding) are the readings listed in DESIGN.md.
 *
 * Conventions for every entry point
 *   - All array pointers are DEVICE pointers unless marked "host".  The caller
 *     allocates and frees every buffer; the library never allocates device
 *     memory inside a call and never synchronizes the host.
 *   - Work is enqueued on `stream` (a cudaStream_t passed as void*; NULL = the
 *     legacy default stream) and is asynchronous; device faults surface at the
 *     caller's next synchronization.
 *   - A non-SUCCESS status means nothing was enqueued (argument errors) or a
 *     launch failed (FIREQ_ERROR_CUDA); fireq_last_error() then returns a
 *     thread-local human-readable detail.
 *   - Row-major everywhere; "ld*" are leading dimensions in elements.
 *   - Some GEMM schedules (stream-K remainders, the fused FFN) have CTAs wait on
 *     other CTAs of the same grid; those grids are at most one CTA per SM and rely
 *     on all their CTAs being resident together (as CUTLASS's stream-K does).  Do
 *     not run them concurrently with a kernel that holds SMs for its whole
 *     duration, or set FIREQ_COOPERATIVE=1 in the environment: such grids are then
 *     launched cooperatively (guaranteed co-residency; the launch fails rather than
 *     hangs; ~1.4 us slower per launch).
 */
#ifndef FIREQ_H_
#define FIREQ_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    FIREQ_SUCCESS = 0,
    FIREQ_ERROR_INVALID_VALUE = 1,      /* NULL pointer, bad enum, M < 1, ...        */
    FIREQ_ERROR_UNSUPPORTED_SHAPE = 2,  /* N or K not a multiple of 128, too large  */
    FIREQ_ERROR_MISALIGNED = 3,         /* pointer not 16-byte aligned / bad ld     */
    FIREQ_ERROR_CUDA = 4,               /* a CUDA runtime/driver call failed        */
    FIREQ_ERROR_NCCL = 5,               /* an NCCL call failed                      */
    FIREQ_ERROR_NOT_INITIALIZED = 6,    /* comm handle missing / destroyed          */
    FIREQ_ERROR_WORKSPACE = 7           /* workspace NULL or smaller than required  */
} fireq_status_t;

/* Status name, e.g. "FIREQ_ERROR_MISALIGNED".  Static storage. */
const char* fireq_status_string(fireq_status_t status);
/* Detail of the last failing call on this host thread ("" if none). */
const char* fireq_last_error(void);

/* Drops the library's cached TMA descriptors (keyed by activation pointer, shape
 * and tile; they embed device addresses).  Call after freeing activation buffers
 * that may be reallocated at the same address with different contents layout, or
 * before cudaDeviceReset.  Host-only, thread-safe. */
void fireq_clear_cache(void);

/* Version of the packed weight layout produced by fireq_quantize_weight
 * (currently 1). */
int fireq_weight_layout_version(void);

/* ------------------------------------------------------------------ sizes */
/* Bytes of packed INT4 codes for an N x K weight: N*K/2. */
size_t fireq_packed_weight_bytes(int64_t N, int64_t K);
/* Bytes of FP8-E4M3 group scales: N*K/128. */
size_t fireq_weight_scale_bytes(int64_t N, int64_t K);
/* Device workspace needed by fireq_quantize_weight. */
size_t fireq_quantize_weight_workspace_bytes(int64_t N, int64_t K);
/* Device workspace needed by fireq_w4a8_gemm for this problem (split-K partial
 * sums + per-tile arrival counters).  The counters must be ZERO before the first
 * call that uses a workspace; every call leaves them zero again, so one
 * cudaMemset at allocation time suffices.  A workspace must not be shared by
 * two GEMMs that may run concurrently. */
size_t fireq_w4a8_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K);

/* ------------------------------------------------------- offline quantizer */
/*
 * fireq_quantize_weight -- steps W1..W6 (P:141-175, P:45-48,
 * P:498-511):
 *   W1 CAS: absmean_k = fp32(sum_n |W[n,k]| (fp64, ascending n) / N),
 *      omega_bar = fp32(sum_k absmean_k (fp64, ascending k) / K),
 *      lambda_k = fp32(fp64(omega_bar) / fp64(absmean_k)) (1 if absmean_k = 0);
 *      cas_mode 0 = off (lambda = 1, the Lambda_1 case of P:152), 1 = absmean.
 *   W2 W_bar = fp32(W) * lambda_k (one fp32 rounding).
 *   W3 PTS: n = smallest n >= 0 with (every nonzero |W_bar| * 2^n >= 7*2^-9) or
 *      (some 7*2^(5-n) <= |W_bar| < 7*2^(6-n)); W_tilde = W_bar * 2^n.
 *   W4 sigma = largest E4M3 value s with 7 s <= max_group |W_tilde| (capped 448).
 *   W5 code = clamp(round_half_even(W_tilde / sigma), -8, 7), 0 if sigma = 0.
 *   W6 pack into layout v1.
 * Arguments
 *   W            bf16 [N][K], row-major, 16-B aligned.  Must be finite.
 *   N, K         multiples of 128, N*K < 2^40.
 *   cas_mode     0 or 1.
 *   w_packed     out, uint8 [fireq_packed_weight_bytes(N, K)], layout v1.
 *   w_scales     out, uint8 [fireq_weight_scale_bytes(N, K)] E4M3 codes, layout v1.
 *   cas_lambda   out, float [K] (lambda_k), may be NULL.
 *   cas_inv      out, bf16 [K]: c_k = bf16(1.0f / lambda_k), the Lambda^-1 that
 *                the activation quantizer (or the previous layer) applies
 *                (P:148-152); may be NULL.
 *   pts_and_status  out, int32 [2]: {n, status}; status is FIREQ_SUCCESS or
 *                FIREQ_ERROR_INVALID_VALUE (non-finite input, or no n <= 60).
 *                The caller reads it back once (offline) and passes n to the GEMM.
 *   workspace    >= fireq_quantize_weight_workspace_bytes(N, K) bytes.
 */
fireq_status_t fireq_quantize_weight(const void* W, int64_t N, int64_t K, int cas_mode,
                                     uint8_t* w_packed, uint8_t* w_scales,
                                     float* cas_lambda, void* cas_inv,
                                     int32_t* pts_and_status,
                                     void* workspace, size_t workspace_bytes,
                                     void* stream);

/* ------------------------------------------------------- online quantizer */
/*
 * fireq_quantize_act -- steps A1..A3 (Eq. 2; per token):
 *   A1 x' = chan_mul ? bf16(x * c_k) : x
 *   A2 beta_m = bf16_RN(max_k |x'| / 448), 1 if the row is all zero
 *   A3 x_hat = E4M3_RN_satfinite(x' / beta_m)  (IEEE sign; fp32 division)
 * Arguments
 *   X        bf16 [M][ldx] (first K columns used), 16-B aligned, ldx % 8 == 0.
 *   chan_mul bf16 [K] or NULL.
 *   x_fp8    out, uint8 E4M3 [M][K] (dense, leading dimension K), 16-B aligned.
 *   x_scale  out, bf16 [M].
 * K % 128 == 0 (matches the GEMM), M >= 1.  Non-finite input gives
 * unspecified output (not checked on the hot path).
 */
fireq_status_t fireq_quantize_act(const void* X, int64_t M, int64_t K, int64_t ldx,
                                  const void* chan_mul, uint8_t* x_fp8, void* x_scale,
                                  void* stream);

/*
 * fireq_silu_mul_quantize_act -- FFN helper (P:130 lists SiLU and elementwise
 * multiplication among the epilogue operations): h = bf16(silu(g) * u) with
 * silu(g) = g / (1 + exp(-g)) in fp32, then A2..A3 on h.  G and U are bf16
 * [M][ld] (the gate and up projections).  Used by the FFN benchmark.
 */
fireq_status_t fireq_silu_mul_quantize_act(const void* G, const void* U, int64_t M, int64_t K,
                                           int64_t ld, uint8_t* x_fp8, void* x_scale,
                                           void* stream);

/*
 * Transposed-input variants (the Y^T layout produced by the column-parallel GEMM and
 * its in-place all-gather): element (m, k) of the activation is read from
 * Xt[k * ldt + m] (Xt is [K][ldt], ldt >= M).  Same arithmetic and outputs
 * (x_fp8 [M][K] row-major, x_scale [M]) as the row-major functions above.
 */
fireq_status_t fireq_quantize_act_t(const void* Xt, int64_t M, int64_t K, int64_t ldt,
                                    const void* chan_mul, uint8_t* x_fp8, void* x_scale,
                                    void* stream);
fireq_status_t fireq_silu_mul_quantize_act_t(const void* Gt, const void* Ut, int64_t M, int64_t K,
                                             int64_t ldt, uint8_t* x_fp8, void* x_scale,
                                             void* stream);

/* ------------------------------------------------------------------ GEMM */
/*
 * fireq_w4a8_gemm -- Steps 1..3 of the INT4 x FP8 kernel:
 *   y[m][n] = bf16_RN( acc[m][n] * (beta_m * 2^-pts_exponent) [* gamma_n] )
 *   acc[m][n] = sum_k dec(x_fp8[m][k]) * dec(LUT_{n, k/128}[code[n][k]]) in FP32
 *   LUT_{n,g}[v] = E4M3_RN(v * sigma_{n,g}), v in [-8, 7].
 * The FP32 accumulation order is the tensor core's (tolerance-checked, G4).
 * Arguments
 *   x_fp8        uint8 E4M3 [M][K] dense (from fireq_quantize_act), 16-B aligned.
 *   x_scale      bf16 [M] (beta).
 *   M            >= 1 tokens.   K: multiple of 128, <= 65536.
 *   w_packed, w_scales  from fireq_quantize_weight (layout v1), N multiple of 128.
 *   pts_exponent host int n in [0, 60] (pts_and_status[0]).
 *   out_chan_scale  float [N] gamma or NULL.
 *   Y            out bf16: out_layout 0 -> Y[M][ldy] (ldy >= N), 1 -> Y^T [N][ldy]
 *                (ldy >= M).  16-B aligned; ldy % 8 == 0 for layout 0 (any ldy >= M
                for Y^T; 16-B vector stores when ldy % 8 == 0).  Rows/cols outside
 *                [0,M) x [0,N) are never written.
 *   workspace    >= fireq_w4a8_gemm_workspace_bytes(M, N, K) (see there).
 */
fireq_status_t fireq_w4a8_gemm(const uint8_t* x_fp8, const void* x_scale, int64_t M, int64_t K,
                               const uint8_t* w_packed, const uint8_t* w_scales, int64_t N,
                               int32_t pts_exponent, const float* out_chan_scale,
                               void* Y, int64_t ldy, int out_layout,
                               void* workspace, size_t workspace_bytes, void* stream);

/*
 * fireq_w4a8_gemm_prefetch -- fireq_w4a8_gemm plus an L2 prefetch hint: once each CTA
 * has issued its own weight loads it streams its share of [next_packed, +bytes) and
 * [next_scales, +bytes) (the NEXT layer's packed weights / scales, 16-byte aligned,
 * either may be NULL) into L2 (cp.async.bulk.prefetch.L2), so that HBM stays busy
 * through this GEMM's tail and the small kernels that follow and the next GEMM's
 * weights come from L2.  A performance hint only: results are identical.
 */
fireq_status_t fireq_w4a8_gemm_prefetch(const uint8_t* x_fp8, const void* x_scale, int64_t M, int64_t K,
                                        const uint8_t* w_packed, const uint8_t* w_scales, int64_t N,
                                        int32_t pts_exponent, const float* out_chan_scale,
                                        void* Y, int64_t ldy, int out_layout,
                                        void* workspace, size_t workspace_bytes,
                                        const void* next_packed, size_t next_packed_bytes,
                                        const void* next_scales, size_t next_scales_bytes,
                                        void* stream);

/*
 * fireq_w4a8_gemm_residual -- fireq_w4a8_gemm (row-major Y) with Step 3's element-wise
 * addition fused into the epilogue (Fig. 2 Step 3 "activation addition"; the
 * residual connection around a Llama block):
 *   Y[m][n] = BF16_RN( fp32(fp32(acc * (beta_m 2^-n)) * gamma_n) + R[m][n] )
 * (gamma_n only when out_chan_scale is non-NULL; one BF16 rounding at the end).
 *   residual  bf16 [M][ldr], ldr >= N, device, 16-byte aligned; may equal Y (in place).
 * Everything else as fireq_w4a8_gemm with out_layout 0.  NULL residual ->
 * FIREQ_ERROR_INVALID_VALUE.
 */
fireq_status_t fireq_w4a8_gemm_residual(const uint8_t* x_fp8, const void* x_scale, int64_t M, int64_t K,
                                        const uint8_t* w_packed, const uint8_t* w_scales, int64_t N,
                                        int32_t pts_exponent, const float* out_chan_scale,
                                        const void* residual, int64_t ldr, void* Y, int64_t ldy,
                                        void* workspace, size_t workspace_bytes, void* stream);

/* --------------------------------------------------------- multi-GPU layer */
/* Opaque NCCL communicator wrapper (caller-owned, not thread-safe). */
typedef struct fireq_comm* fireq_comm_t;

/* host: writes a 128-byte NCCL unique id into id[128] (rank 0 calls it and
 * broadcasts the bytes by any host means). */
fireq_status_t fireq_comm_get_unique_id(uint8_t id[128]);
/* host: collective over nranks processes, one GPU each (the current device). */
fireq_status_t fireq_comm_init(fireq_comm_t* out, int nranks, int rank, const uint8_t id[128]);
fireq_status_t fireq_comm_destroy(fireq_comm_t comm);

/*
 * fireq_w4a8_gemm_colpar -- column-parallel (N-sharded) linear layer
 * (BASELINE north_star (d)): this rank holds rows [rank*N_local, (rank+1)*N_local)
 * of the quantized weight (byte slices of the full packing, layout v1, because
 * CAS lambda and PTS n are computed on the full tensor before sharding; a shard
 * may end in zero-padded rows so that all shards have equal N_local, a multiple
 * of 128).  X is replicated.  The rank computes its slice with fireq_w4a8_gemm in
 * the Y^T layout directly into its slot of Yt_full [N_local*nranks][M] and an
 * in-place ncclAllGather (bf16) over NVLink completes Y^T on every rank, on `stream`
 * (also at nranks == 1, where it is a no-op copy).
 *   out_chan_scale_local  float [N_local] gamma for this shard's rows, or NULL.
 *   Yt_full   out bf16 [nranks*N_local][M] (Y^T, ld = M; any M >= 1).
 */
fireq_status_t fireq_w4a8_gemm_colpar(const uint8_t* x_fp8, const void* x_scale, int64_t M,
                                      int64_t K, const uint8_t* w_packed_local,
                                      const uint8_t* w_scales_local, int64_t N_local,
                                      int32_t pts_exponent, const float* out_chan_scale_local,
                                      void* Yt_full, void* workspace, size_t workspace_bytes,
                                      fireq_comm_t comm, void* stream);

/* ------------------------------------------------- sigma_BF16 comparison variant */
/*
 * The paper's comparison point with BF16 group scales (App. B.1; DESIGN
 * reading R25): W1-W3 as fireq_quantize_weight (CAS lambda, PTS n), then per 128-group
 * sigma = bf16_RN(max|W_tilde| / 7) and codes = clamp(RNE(W_tilde / sigma), -8, 7) (sigma = 0
 * -> 0).  Codes in layout v1; scales bf16 [N/128][K/128][128] (N*K/64 bytes).
 */
size_t fireq_weight_scale_bytes_bf16s(int64_t N, int64_t K);
fireq_status_t fireq_quantize_weight_bf16s(const void* W, int64_t N, int64_t K, int cas_mode,
                                           uint8_t* w_packed, void* w_scales_bf16, float* cas_lambda,
                                           void* cas_inv, int32_t* pts_and_status, void* workspace,
                                           size_t workspace_bytes, void* stream);
/* Device workspace of fireq_w4a8_gemm_bf16s (FP32 split-K partials). */
size_t fireq_w4a8_gemm_bf16s_workspace_bytes(int64_t M, int64_t N, int64_t K);
/*
 * fireq_w4a8_gemm_bf16s -- y[m][n] = bf16_RN(beta_m 2^-n sum_g sigma_{n,g} * P_g[m][n]) with
 * P_g = sum_{k in g} dec(x_fp8[m][k]) * code[n][k] on the FP8 tensor cores (codes are exact
 * E4M3 integers) and the per-group scaling + accumulation in FP32 on CUDA cores.  Row-major Y
 * [M][ldy], ldy >= N.  Tolerance-checked against the oracle (G4).
 */
fireq_status_t fireq_w4a8_gemm_bf16s(const uint8_t* x_fp8, const void* x_scale, int64_t M, int64_t K,
                                     const uint8_t* w_packed, const void* w_scales_bf16, int64_t N,
                                     int32_t pts_exponent, void* Y, int64_t ldy, void* workspace,
                                     size_t workspace_bytes, void* stream);

/* ------------------------------ comm-fused column parallelism (NVLink, CUDA IPC) */
/*
 * A symmetric buffer is one device allocation per rank, same size on every rank:
 *   [256 B: epoch flags, one u32 per source rank][Y^T data, nranks * N_local * M bf16]
 * Each rank exports the IPC handle of its buffer (fireq_symm_handle: handle of the containing
 * allocation + the buffer's offset in it), exchanges handles and offsets by any host means,
 * and opens the group (fireq_symm_open maps every peer's buffer; nranks <= 8, one GPU
 * per process; peers on the same node).  The flags must be zero before the first use.
 */
typedef struct fireq_symm* fireq_symm_t;
/* bytes of a symmetric buffer holding data_bytes of Y^T (256 + data_bytes). */
size_t fireq_symm_bytes(int64_t data_bytes);
/* host: the IPC handle (64 bytes) of the allocation containing `buffer` and the buffer's byte
 * offset inside it (allocators hand out interior pointers). */
fireq_status_t fireq_symm_handle(void* buffer, uint8_t handle[64], int64_t* offset);
/* host: handles [nranks][64] (entry `rank` ignored), offsets [nranks] of each rank's buffer
 * inside the allocation its handle names (NULL = 0); local_buffer 16-B aligned. */
fireq_status_t fireq_symm_open(fireq_symm_t* out, int nranks, int rank, void* local_buffer, size_t bytes,
                               const uint8_t* handles, const int64_t* offsets);
/* host: synchronizes the device, unmaps the peers' buffers, frees the handle. */
fireq_status_t fireq_symm_close(fireq_symm_t symm);
/*
 * fireq_w4a8_gemm_colpar_p2p -- the column-parallel layer with the all-gather fused into the
 * GEMM epilogue: this rank's Y^T slice [rank*N_local, (rank+1)*N_local) x M is
 * stored by the epilogue straight into the same slot of EVERY rank's symmetric buffer (NVLink
 * stores), then a one-CTA kernel advances the buffer's call counter, publishes it in every
 * peer's flag area (release, system scope) and waits for all peers' flags to reach it
 * (acquire): on return (stream order) the local buffer's Y^T [nranks*N_local][M] (data at
 * offset 256, ld = M) is complete.  No NCCL.  Every rank must make the same sequence of calls
 * on a buffer (the epochs then agree; CUDA-graph replays advance them on the device).
 * Other arguments as fireq_w4a8_gemm_colpar.  Same values as the NCCL path, bit for bit.
 */
fireq_status_t fireq_w4a8_gemm_colpar_p2p(const uint8_t* x_fp8, const void* x_scale, int64_t M, int64_t K,
                                          const uint8_t* w_packed_local, const uint8_t* w_scales_local,
                                          int64_t N_local, int32_t pts_exponent,
                                          const float* out_chan_scale_local, fireq_symm_t symm,
                                          void* workspace, size_t workspace_bytes, void* stream);

/* --------------------------------------------------------- introspection */
/* Debug/test: writes the 127 x 16 LUT-of-LUTs the GEMM builds on chip
 * (entry [s][u] = E4M3_RN(v(u) * dec(s)), v(u) = u < 8 ? u : u - 16) into the
 * device buffer out[2032], on `stream`. */
fireq_status_t fireq_debug_lut_table(uint8_t* out, void* stream);
/* Debug/profiling (profile builds only; no-op otherwise): when buf != NULL, every
 * later fireq_w4a8_gemm launch records a
 * per-CTA %globaltimer timeline into the device buffer buf ([ctas][8] uint64:
 * start, setup done, first stage landed, MMA issue done, epilogue done, end).
 * Pass NULL to disable.  Not thread-safe; for benchmarks only. */
fireq_status_t fireq_debug_set_trace(void* buf);
/* Debug/profiling (profile builds only; no-op otherwise): subsequent launches of the
 * library record {first CTA start, last CTA end} (%globaltimer ns) into consecutive
 * slots of the device buffer buf ([cap][2] uint64, caller pre-fills {UINT64_MAX, 0}).
 * NULL disables.  Not thread-safe; for benchmarks only. */
fireq_status_t fireq_debug_set_spans(void* buf, int cap);
/* ------------------------------------------------------ fused decode FFN */
/*
 * fireq_interleave_gate_up -- row order of the fused FFN's gate_up weight:
 * 128-row tile t = gate rows [64t, 64t+64) followed by up rows [64t, 64t+64).
 * W_gate, W_up bf16 [d_ff][d_model]; W_gu out, bf16 [2 d_ff][d_model] (caller
 * owned, device, 16-B aligned).  A row permutation only: quantizing W_gu with
 * fireq_quantize_weight gives every row the codes/scales of the plain
 * [gate; up] stacking (CAS lambda is per input channel, PTS n per tensor).
 */
fireq_status_t fireq_interleave_gate_up(const void* W_gate, const void* W_up, int64_t d_ff,
                                        int64_t d_model, void* W_gu, void* stream);

/* Workspace for fireq_ffn_w4a8_decode (0 for invalid shapes).  Zero-fill it once
 * before first use; every call leaves its counters zeroed again. */
size_t fireq_ffn_workspace_bytes(int64_t M, int64_t d_model, int64_t d_ff);

/*
 * fireq_ffn_w4a8_decode -- a Llama FFN block y = W_down (silu(W_gate x) * (W_up x)) [+ r]
 * with Step 3's element-wise operations fused into the GEMM epilogues, as four
 * kernels (the name is historical: any M):
 *   1. fireq_quantize_act(x, c_gu)                      (A1..A3, Eq. 2)
 *   2. gate_up GEMM over the interleaved W_gu (steps 1-3) whose epilogue forms
 *      h = bf16(silu(g) * u * c_down) from the bf16-rounded g and u (exactly
 *      fireq_silu_mul_quantize_act's x') and writes h;
 *   3. fireq_quantize_act(h)                            (A1..A3)
 *   4. down GEMM on (h_hat, beta_h), residual added in its epilogue
 *      (fireq_w4a8_gemm_residual) when residual != NULL.
 * Arguments
 *   x        bf16 [M][ldx], ldx >= d_model, ldx % 8 == 0.
 *   c_gu     bf16 [d_model]: CAS multiplier of W_gu (QuantizedWeight.c) or NULL.
 *   gu_*     fireq_quantize_weight output for the INTERLEAVED W_gu
 *            (fireq_interleave_gate_up), N = 2 d_ff, K = d_model.
 *   c_down   bf16 [d_ff]: CAS multiplier of W_down (applied to u) or NULL.
 *   d_*      fireq_quantize_weight output for W_down, N = d_model, K = d_ff.
 *   residual bf16 [M][ldr] (ldr >= d_model) added to y, or NULL; may equal x or y.
 *   h        out, bf16 [M][d_ff]: the SwiGLU output (before quantization).
 *   y        out, bf16 [M][ldy], ldy >= d_model.
 *   next_*   optional L2 prefetch of the next layer's weights (may be NULL).
 * Shapes: M >= 1 (decode batches and prefill; each GEMM takes its own plan for M), d_model,
 * d_ff multiples of 128; otherwise FIREQ_ERROR_UNSUPPORTED_SHAPE (the two variants below:
 * M <= 16).  Same arithmetic as the unfused chain
 * (quantize_act -> gemm -> silu_mul_quantize_act -> gemm[_residual]) up to the fp32
 * summation order of split gate_up tiles; y equals
 * fireq_w4a8_gemm[_residual](quantize_act(h), W_down) exactly.
 * Environment (read once per process): FIREQ_FFN_MODE=3 -- three kernels, the gate_up
 * kernel quantizing h in its tail behind a grid-wide barrier (per-token max|h| by
 * atomics); FIREQ_FFN_PERSISTENT=1 -- ONE persistent launch (x quantized in-kernel,
 * three grid-wide barriers, the down phase scheduled stream-K: y then equals the
 * standalone down GEMM under FIREQ_NO_CSPLIT=1 exactly).  Both measured slower on B200
 * and kept for the record.
 */
fireq_status_t fireq_ffn_w4a8_decode(const void* x, int64_t ldx, const void* c_gu, int64_t M,
                                     int64_t d_model, int64_t d_ff, const uint8_t* gu_packed,
                                     const uint8_t* gu_scales, int32_t gu_pts, const void* c_down,
                                     const uint8_t* d_packed, const uint8_t* d_scales, int32_t d_pts,
                                     const void* residual, int64_t ldr, void* h, void* y, int64_t ldy,
                                     void* workspace, size_t workspace_bytes, const void* next_packed,
                                     size_t next_packed_bytes, const void* next_scales,
                                     size_t next_scales_bytes, void* stream);

/* ------------------------------------------------------ KV4Q8 attention (NEXT f4) */
/*
 * fireq_quantize_kv -- one head's INT4 KV-cache block (DESIGN R30-R35):
 * X bf16 [N][d] (contiguous; N, d multiples of 128) quantized exactly as fireq_quantize_weight
 * with a CALLER-GIVEN per-column multiplier in place of CAS: X_bar = fp32(X) * lambda_k
 * (lambda = 1/t for the post-RoPE key channels CRS rescales; NULL = 1), PTS exponent
 * n (W3), 128-groups along each row with RZ FP8 scales (W4-W6), layout v1.
 *   keys:   X = K_post of one (sequence, kv head) [N tokens][d]  -> one group per token row
 *   values: X = V^T of one (sequence, kv head) [d][N tokens]      -> groups of 128 tokens
 * pts_and_status: device int32[2] {n, status} as fireq_quantize_weight.
 * workspace >= fireq_quantize_weight_workspace_bytes(N, d).
 */
fireq_status_t fireq_quantize_kv(const void* X, int64_t N, int64_t d, const float* chan_lambda,
                                 uint8_t* packed, uint8_t* scales, int32_t* pts_and_status,
                                 void* workspace, size_t workspace_bytes, void* stream);

/*
 * fireq_kv4q8_attention -- prefill self-attention with FP8 queries and the INT4 KV cache
 * (KV4Q8-FP; S = Q K^T and O = P V through the INT4 x FP8 path; softmax
 * quantized to FP8; the three-stage overlap of Alg. 1 P:227-291 on tcgen05):
 *   S[q][k]  = beta_q[q] 2^-n_k sum_c dec(q_hat[q][c]) LUT_k(K[k][c])      (FP32 accumulation)
 *   x        = tau S,  causal: k > q excluded;  m = max_k x;  P = exp(x - m);  l = sum_k P
 *   P_hat    = E4M3_RN(448 P)
 *   O[q][c]  = BF16( 2^-n_v / 448 / l * sum_k dec(P_hat[q][k]) LUT_v(V^T[c][k]) )
 * Arguments (device pointers)
 *   q_fp8    E4M3 [B][Hq][N][d] (fireq_quantize_act per (token, head) row, post-RoPE, CRS
 *            multiplier c = t applied as A1's channel multiplier), q_scale bf16 [B][Hq][N].
 *   k_*      [B][Hkv] consecutive fireq_quantize_kv outputs of K_post [N][d]
 *            (packed N d / 2 bytes, scales N d / 128 bytes per head), k_pts int32 [B][Hkv][2].
 *   vt_*     [B][Hkv] consecutive fireq_quantize_kv outputs of V^T [d][N], v_pts likewise.
 *   d = 128, N % 128 == 0, Hq % Hkv == 0 (grouped-query: q head h reads kv head h / (Hq/Hkv)).
 *   causal   1 = causal mask; tau > 0 (usually 1/sqrt(d)).
 *   O        out, bf16 [B N][ldo] (token-major, head h at columns [h d, h d + d): the o_proj
 *            input), ldo >= Hq d, ldo % 8 == 0.
 */
fireq_status_t fireq_kv4q8_attention(const uint8_t* q_fp8, const void* q_scale, int64_t B, int64_t N,
                                     int64_t Hq, int64_t Hkv, int64_t d, const uint8_t* k_packed,
                                     const uint8_t* k_scales, const int32_t* k_pts,
                                     const uint8_t* vt_packed, const uint8_t* vt_scales,
                                     const int32_t* v_pts, int causal, float tau, void* O, int64_t ldo,
                                     void* stream);

/* The schedule fireq_w4a8_gemm chooses for (M, N, K), for benchmarks and tests:
 * writes {ntok, mode, ctas, sign_split} into cfg_out[4] (host).  mode 0 = whole
 * tiles, 1 = whole tiles + stream-K remainder (global-memory fixup), 2 = cluster
 * split-K (ctas / tiles CTAs per tile, DSMEM reduction). */
fireq_status_t fireq_gemm_plan(int64_t M, int64_t N, int64_t K, int32_t cfg_out[4]);

#ifdef __cplusplus
}
#endif
#endif /* FIREQ_H_ */
