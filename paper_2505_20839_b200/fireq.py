"""Thin ctypes binding of libfireq.so (include/fireq.h) -- argument marshalling only.

Every step of the FireQ path runs in the library's CUDA kernels; this module only
turns torch CUDA tensors into device pointers + the current CUDA stream and maps
status codes to exceptions.  There is no CPU or PyTorch fallback: if the library
is missing, or a tensor is not on a CUDA device, the call raises.
"""
import ctypes
import math
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfireq.so")

_lib = None

EXPORTS = [
    "fireq_status_string", "fireq_last_error", "fireq_weight_layout_version",
    "fireq_packed_weight_bytes", "fireq_weight_scale_bytes",
    "fireq_quantize_weight_workspace_bytes", "fireq_w4a8_gemm_workspace_bytes",
    "fireq_quantize_weight", "fireq_quantize_act", "fireq_silu_mul_quantize_act",
    "fireq_w4a8_gemm", "fireq_comm_get_unique_id", "fireq_comm_init", "fireq_comm_destroy",
    "fireq_w4a8_gemm_colpar", "fireq_debug_lut_table", "fireq_gemm_plan", "fireq_debug_set_trace",
    "fireq_quantize_act_t", "fireq_silu_mul_quantize_act_t", "fireq_debug_set_spans",
    "fireq_w4a8_gemm_prefetch", "fireq_interleave_gate_up", "fireq_ffn_workspace_bytes",
    "fireq_ffn_w4a8_decode", "fireq_clear_cache", "fireq_symm_bytes", "fireq_symm_handle", "fireq_symm_open",
    "fireq_symm_close", "fireq_w4a8_gemm_colpar_p2p", "fireq_weight_scale_bytes_bf16s",
    "fireq_quantize_weight_bf16s", "fireq_w4a8_gemm_bf16s_workspace_bytes", "fireq_w4a8_gemm_bf16s",
]


class FireqError(RuntimeError):
    pass


def load(path=LIB_PATH):
    """Load libfireq.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise FireqError(f"libfireq.so not found at {path}: run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    P, I64, I32, SZ, C = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t, ctypes.c_int
    sig = {
        "fireq_status_string": ([C], ctypes.c_char_p),
        "fireq_last_error": ([], ctypes.c_char_p),
        "fireq_clear_cache": ([], None),
        "fireq_symm_bytes": ([I64], SZ),
        "fireq_weight_scale_bytes_bf16s": ([I64, I64], SZ),
        "fireq_quantize_weight_bf16s": ([P, I64, I64, C, P, P, P, P, P, P, SZ, P], C),
        "fireq_w4a8_gemm_bf16s_workspace_bytes": ([I64, I64, I64], SZ),
        "fireq_w4a8_gemm_bf16s": ([P, P, I64, I64, P, P, I64, I32, P, I64, P, SZ, P], C),
        "fireq_symm_handle": ([P, P, P], C),
        "fireq_symm_open": ([P, C, C, P, SZ, P, P], C),
        "fireq_symm_close": ([P], C),
        "fireq_w4a8_gemm_colpar_p2p": ([P, P, I64, I64, P, P, I64, I32, P, P, P, SZ, P], C),
        "fireq_weight_layout_version": ([], C),
        "fireq_packed_weight_bytes": ([I64, I64], SZ),
        "fireq_weight_scale_bytes": ([I64, I64], SZ),
        "fireq_quantize_weight_workspace_bytes": ([I64, I64], SZ),
        "fireq_w4a8_gemm_workspace_bytes": ([I64, I64, I64], SZ),
        "fireq_quantize_weight": ([P, I64, I64, C, P, P, P, P, P, P, SZ, P], C),
        "fireq_quantize_act": ([P, I64, I64, I64, P, P, P, P], C),
        "fireq_silu_mul_quantize_act": ([P, P, I64, I64, I64, P, P, P], C),
        "fireq_w4a8_gemm": ([P, P, I64, I64, P, P, I64, I32, P, P, I64, C, P, SZ, P], C),
        "fireq_w4a8_gemm_prefetch": ([P, P, I64, I64, P, P, I64, I32, P, P, I64, C, P, SZ, P, SZ, P, SZ, P], C),
        "fireq_comm_get_unique_id": ([P], C),
        "fireq_comm_init": ([P, C, C, P], C),
        "fireq_comm_destroy": ([P], C),
        "fireq_w4a8_gemm_colpar": ([P, P, I64, I64, P, P, I64, I32, P, P, P, SZ, P, P], C),
        "fireq_quantize_act_t": ([P, I64, I64, I64, P, P, P, P], C),
        "fireq_silu_mul_quantize_act_t": ([P, P, I64, I64, I64, P, P, P], C),
        "fireq_debug_lut_table": ([P, P], C),
        "fireq_gemm_plan": ([I64, I64, I64, P], C),
        "fireq_debug_set_trace": ([P], C),
        "fireq_debug_set_spans": ([P, C], C),
        "fireq_interleave_gate_up": ([P, P, I64, I64, P, P], C),
        "fireq_ffn_workspace_bytes": ([I64, I64, I64], SZ),
        "fireq_ffn_w4a8_decode": ([P, I64, P, I64, I64, I64, P, P, I32, P, P, P, I32, P, I64, P, P, I64, P, SZ, P, SZ,
                                   P, SZ, P], C),
        "fireq_w4a8_gemm_residual": ([P, P, I64, I64, P, P, I64, I32, P, P, I64, P, I64, P, SZ, P], C),
        "fireq_quantize_kv": ([P, I64, I64, P, P, P, P, P, SZ, P], C),
        "fireq_kv4q8_attention": ([P, P, I64, I64, I64, I64, I64, P, P, P, P, P, P, C, ctypes.c_float, P, I64, P], C),
    }
    for name, (args, res) in sig.items():
        if os.environ.get("FIREQ_LOAD_PARTIAL") and not hasattr(lib, name):   # bisecting older builds
            continue
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def lib():
    return load()


def _check(status, what):
    if status != 0:
        L = lib()
        raise FireqError(f"{what}: {L.fireq_status_string(status).decode()}: {L.fireq_last_error().decode()}")


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise FireqError("fireq: tensors must live on a CUDA device (no CPU path)")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _zeros_on(nbytes, device, stream=None):
    """Zeroed uint8 scratch allocated AND zeroed on `stream` (the stream the kernel is
    enqueued on): the memset is ordered before the kernel, and the caching allocator
    frees it in that stream's order."""
    if stream is None:
        return torch.zeros(int(nbytes), dtype=torch.uint8, device=device)
    with torch.cuda.stream(stream):
        return torch.zeros(int(nbytes), dtype=torch.uint8, device=device)


def clear_cache():
    """fireq_clear_cache: drop the library's cached TMA descriptors."""
    lib().fireq_clear_cache()


# ------------------------------------------------------------------- sizes
def packed_weight_bytes(N, K):
    return lib().fireq_packed_weight_bytes(N, K)


def weight_scale_bytes(N, K):
    return lib().fireq_weight_scale_bytes(N, K)


def gemm_workspace_bytes(M, N, K):
    return lib().fireq_w4a8_gemm_workspace_bytes(M, N, K)


def layout_version():
    return lib().fireq_weight_layout_version()


def gemm_plan(M, N, K):
    cfg = (ctypes.c_int32 * 4)()
    _check(lib().fireq_gemm_plan(M, N, K, ctypes.cast(cfg, ctypes.c_void_p)), "fireq_gemm_plan")
    return {"ntok": cfg[0], "mode": ("tiles", "stream-k", "cluster-split-k", "split-k-dsmem")[cfg[1]], "ctas": cfg[2], "sign_split": bool(cfg[3])}


# ------------------------------------------------------------------- calls
class QuantizedWeight:
    """Device tensors produced by fireq_quantize_weight."""

    def __init__(self, packed, scales, lam, c, pts_and_status, N, K):
        self.packed, self.scales, self.lam, self.c = packed, scales, lam, c
        self.pts_and_status = pts_and_status
        self.N, self.K = N, K
        self._n = None

    @property
    def n(self):
        """PTS exponent (reads the device scalar back once, as the C ABI prescribes)."""
        if self._n is None:
            # the quantizer ran asynchronously on the caller's stream, which need not be the
            # current one: synchronize the device before the (offline, once) read-back
            torch.cuda.synchronize(self.pts_and_status.device)
            host = self.pts_and_status.cpu()
            if int(host[1]) != 0:
                raise FireqError(f"fireq_quantize_weight device status {int(host[1])}")
            self._n = int(host[0])
        return self._n


def quantize_weight(W, cas_mode=1, stream=None, out=None):
    """W: bf16 [N][K] CUDA tensor -> QuantizedWeight (all device tensors)."""
    assert W.dtype == torch.bfloat16 and W.dim() == 2 and W.is_contiguous()
    N, K = W.shape
    dev = W.device
    L = lib()
    if out is None:
        packed = torch.empty(L.fireq_packed_weight_bytes(N, K), dtype=torch.uint8, device=dev)
        scales = torch.empty(L.fireq_weight_scale_bytes(N, K), dtype=torch.uint8, device=dev)
    else:
        packed, scales = out
    lam = torch.empty(K, dtype=torch.float32, device=dev)
    c = torch.empty(K, dtype=torch.bfloat16, device=dev)
    ps = torch.empty(2, dtype=torch.int32, device=dev)
    ws = torch.empty(L.fireq_quantize_weight_workspace_bytes(N, K), dtype=torch.uint8, device=dev)
    _check(L.fireq_quantize_weight(_ptr(W), N, K, cas_mode, _ptr(packed), _ptr(scales), _ptr(lam), _ptr(c),
                                   _ptr(ps), _ptr(ws), ws.numel(), _stream(stream)), "fireq_quantize_weight")
    if stream is not None:
        ws.record_stream(stream)          # the scratch is freed while the kernels may still run
    return QuantizedWeight(packed, scales, lam, c, ps, N, K)


def quantize_act(X, chan_mul=None, stream=None, out=None):
    """X: bf16 [M][ld] -> (x_fp8 uint8 [M][K], beta bf16 [M]).  K = X.shape[1]."""
    assert X.dtype == torch.bfloat16 and X.dim() == 2 and X.stride(1) == 1
    M, K = X.shape
    if out is None:
        xq = torch.empty((M, K), dtype=torch.uint8, device=X.device)
        beta = torch.empty(M, dtype=torch.bfloat16, device=X.device)
    else:
        xq, beta = out
    _check(lib().fireq_quantize_act(_ptr(X), M, K, X.stride(0), _ptr(chan_mul), _ptr(xq), _ptr(beta),
                                    _stream(stream)), "fireq_quantize_act")
    return xq, beta


def silu_mul_quantize_act(G, U, stream=None, out=None):
    assert G.shape == U.shape and G.stride() == U.stride()
    M, K = G.shape
    if out is None:
        xq = torch.empty((M, K), dtype=torch.uint8, device=G.device)
        beta = torch.empty(M, dtype=torch.bfloat16, device=G.device)
    else:
        xq, beta = out
    _check(lib().fireq_silu_mul_quantize_act(_ptr(G), _ptr(U), M, K, G.stride(0), _ptr(xq), _ptr(beta),
                                             _stream(stream)), "fireq_silu_mul_quantize_act")
    return xq, beta


def quantize_act_t(Xt, M, K, chan_mul=None, stream=None, out=None):
    """Transposed input Xt [K][ldt] (element (m, k) at Xt[k, m]) -> (x_fp8 [M][K], beta [M])."""
    assert Xt.dtype == torch.bfloat16 and Xt.stride(1) == 1
    if out is None:
        xq = torch.empty((M, K), dtype=torch.uint8, device=Xt.device)
        beta = torch.empty(M, dtype=torch.bfloat16, device=Xt.device)
    else:
        xq, beta = out
    _check(lib().fireq_quantize_act_t(_ptr(Xt), M, K, Xt.stride(0), _ptr(chan_mul), _ptr(xq), _ptr(beta),
                                      _stream(stream)), "fireq_quantize_act_t")
    return xq, beta


def silu_mul_quantize_act_t(Gt, Ut, M, K, stream=None, out=None):
    """Gt, Ut [K][ldt] (Y^T layout) -> quantized silu(g) * u as (x_fp8 [M][K], beta [M])."""
    assert Gt.stride() == Ut.stride() and Gt.stride(1) == 1
    if out is None:
        xq = torch.empty((M, K), dtype=torch.uint8, device=Gt.device)
        beta = torch.empty(M, dtype=torch.bfloat16, device=Gt.device)
    else:
        xq, beta = out
    _check(lib().fireq_silu_mul_quantize_act_t(_ptr(Gt), _ptr(Ut), M, K, Gt.stride(0), _ptr(xq), _ptr(beta),
                                               _stream(stream)), "fireq_silu_mul_quantize_act_t")
    return xq, beta


class Workspace:
    """Zero-initialised GEMM workspace (the counters must start at zero, fireq.h)."""

    def __init__(self, nbytes, device="cuda", stream=None):
        self.t = _zeros_on(max(int(nbytes), 256), device, stream)

    def ensure(self, nbytes, stream=None):
        """Grow (re-zeroed on `stream`, the stream of the kernel that will use it)."""
        if self.t.numel() < nbytes:
            self.t = _zeros_on(nbytes, self.t.device, stream)
        return self.t


def w4a8_gemm(xq, beta, packed, scales, N, pts_n, gamma=None, out=None, out_layout=0, workspace=None,
              stream=None, prefetch=None, residual=None):
    """Y = fireq_w4a8_gemm(...): bf16 [M][N] (out_layout 0) or [N][M] (out_layout 1).

    prefetch: optional (next_packed, next_scales) uint8 tensors of the next layer, streamed
    into L2 once this GEMM's own weight loads are issued (fireq_w4a8_gemm_prefetch).
    residual: optional bf16 [M][>= N] added before the BF16 rounding (fireq_w4a8_gemm_residual,
    row-major Y only; may be `out` itself).
    """
    M, K = xq.shape
    L = lib()
    need = L.fireq_w4a8_gemm_workspace_bytes(M, N, K)
    ws = workspace.ensure(need, stream) if workspace is not None else _zeros_on(need, xq.device, stream)
    if out is None:
        out = torch.empty((M, N) if out_layout == 0 else (N, M), dtype=torch.bfloat16, device=xq.device)
    ldy = out.stride(0)
    if residual is not None:
        if out_layout != 0 or prefetch is not None:
            raise FireqError("w4a8_gemm: residual needs out_layout 0 and no prefetch")
        _check(L.fireq_w4a8_gemm_residual(_ptr(xq), _ptr(beta), M, K, _ptr(packed), _ptr(scales), N, pts_n,
                                          _ptr(gamma), _ptr(residual), residual.stride(0), _ptr(out), ldy, _ptr(ws),
                                          ws.numel(), _stream(stream)), "fireq_w4a8_gemm_residual")
    elif prefetch is None:
        _check(L.fireq_w4a8_gemm(_ptr(xq), _ptr(beta), M, K, _ptr(packed), _ptr(scales), N, pts_n, _ptr(gamma),
                                 _ptr(out), ldy, out_layout, _ptr(ws), ws.numel(), _stream(stream)), "fireq_w4a8_gemm")
    else:
        pp, ps = prefetch
        _check(L.fireq_w4a8_gemm_prefetch(_ptr(xq), _ptr(beta), M, K, _ptr(packed), _ptr(scales), N, pts_n,
                                          _ptr(gamma), _ptr(out), ldy, out_layout, _ptr(ws), ws.numel(),
                                          _ptr(pp), pp.numel() if pp is not None else 0,
                                          _ptr(ps), ps.numel() if ps is not None else 0, _stream(stream)),
               "fireq_w4a8_gemm_prefetch")
    return out


def interleave_gate_up(W_gate, W_up, stream=None, out=None):
    """W_gu (bf16 [2 d_ff][d_model]) in the fused FFN's row order (fireq_interleave_gate_up)."""
    d_ff, d_model = W_gate.shape
    if out is None:
        out = torch.empty((2 * d_ff, d_model), dtype=torch.bfloat16, device=W_gate.device)
    _check(lib().fireq_interleave_gate_up(_ptr(W_gate), _ptr(W_up), d_ff, d_model, _ptr(out), _stream(stream)),
           "fireq_interleave_gate_up")
    return out


def ffn_workspace_bytes(M, d_model, d_ff):
    return lib().fireq_ffn_workspace_bytes(M, d_model, d_ff)


def ffn_w4a8_decode(x, q_gu, q_d, h=None, out=None, workspace=None, stream=None, prefetch=None, residual=None):
    """y = fireq_ffn_w4a8_decode(x, ...) [+ residual]: the fused decode FFN block.

    q_gu: QuantizedWeight of the interleaved W_gu (interleave_gate_up); q_d: of W_down.
    workspace: Workspace of ffn_workspace_bytes (zeroed once, left zeroed by each call).
    """
    M, d_model = x.shape
    d_ff = q_d.K
    L = lib()
    need = L.fireq_ffn_workspace_bytes(M, d_model, d_ff)
    ws = workspace.ensure(need, stream) if workspace is not None else _zeros_on(need, x.device, stream)
    if h is None:
        h = torch.empty((M, d_ff), dtype=torch.bfloat16, device=x.device)
    if out is None:
        out = torch.empty((M, d_model), dtype=torch.bfloat16, device=x.device)
    pp, ps = prefetch if prefetch is not None else (None, None)
    _check(L.fireq_ffn_w4a8_decode(_ptr(x), x.stride(0), _ptr(q_gu.c), M, d_model, d_ff, _ptr(q_gu.packed),
                                   _ptr(q_gu.scales), q_gu.n, _ptr(q_d.c), _ptr(q_d.packed), _ptr(q_d.scales), q_d.n,
                                   _ptr(residual), residual.stride(0) if residual is not None else 0,
                                   _ptr(h), _ptr(out), out.stride(0), _ptr(ws), ws.numel(),
                                   _ptr(pp), pp.numel() if pp is not None else 0,
                                   _ptr(ps), ps.numel() if ps is not None else 0, _stream(stream)),
           "fireq_ffn_w4a8_decode")
    return out


def debug_set_trace(buf):
    """buf: uint64 CUDA tensor [ctas*8] or None."""
    _check(lib().fireq_debug_set_trace(_ptr(buf) if buf is not None else None), "fireq_debug_set_trace")


def debug_set_spans(buf):
    """buf: int64 CUDA tensor [cap, 2] pre-filled with {-1 (= UINT64_MAX), 0}, or None."""
    _check(lib().fireq_debug_set_spans(_ptr(buf) if buf is not None else None,
                                       0 if buf is None else buf.shape[0]), "fireq_debug_set_spans")


def debug_lut_table(device="cuda"):
    out = torch.empty(127 * 16, dtype=torch.uint8, device=device)
    _check(lib().fireq_debug_lut_table(_ptr(out), _stream()), "fireq_debug_lut_table")
    return out


# --------------------------------------------------------------- multi-GPU
class Comm:
    """NCCL communicator wrapper (fireq_comm_t)."""

    def __init__(self, nranks, rank, uid_bytes):
        self.h = ctypes.c_void_p()
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(bytes(uid_bytes))
        _check(lib().fireq_comm_init(ctypes.byref(self.h), nranks, rank, ctypes.cast(buf, ctypes.c_void_p)),
               "fireq_comm_init")
        self.nranks, self.rank = nranks, rank

    @staticmethod
    def unique_id():
        buf = (ctypes.c_uint8 * 128)()
        _check(lib().fireq_comm_get_unique_id(ctypes.cast(buf, ctypes.c_void_p)), "fireq_comm_get_unique_id")
        return bytes(buf)

    def destroy(self):
        if self.h:
            _check(lib().fireq_comm_destroy(self.h), "fireq_comm_destroy")
            self.h = ctypes.c_void_p()


def w4a8_gemm_colpar(xq, beta, packed_local, scales_local, N_local, pts_n, comm, Yt_full, workspace,
                     gamma_local=None, stream=None):
    """Column-parallel GEMM: this rank's Y^T slice + in-place NCCL all-gather into Yt_full [P*N_local][M]."""
    M, K = xq.shape
    ws = workspace.ensure(lib().fireq_w4a8_gemm_workspace_bytes(M, N_local, K), stream)
    _check(lib().fireq_w4a8_gemm_colpar(_ptr(xq), _ptr(beta), M, K, _ptr(packed_local), _ptr(scales_local), N_local,
                                        pts_n, _ptr(gamma_local), _ptr(Yt_full), _ptr(ws), ws.numel(), comm.h,
                                        _stream(stream)),
           "fireq_w4a8_gemm_colpar")
    return Yt_full


# ------------------------------------------------ comm-fused column parallelism (IPC)
class Symmetric:
    """A symmetric buffer (fireq_symm_*): [256 B flags][Y^T nranks*N_local x M bf16] on every rank,
    peers mapped through CUDA IPC.  exchange(obj) -> list of every rank's obj (e.g. a
    torch.distributed all_gather_object), used once for the handles."""

    def __init__(self, nranks, rank, N_local, M, exchange, device="cuda"):
        L = lib()
        self.nranks, self.rank, self.N_local, self.M = nranks, rank, N_local, M
        nbytes = L.fireq_symm_bytes(nranks * N_local * M * 2)
        self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        torch.cuda.synchronize(self.buf.device)
        h = (ctypes.c_uint8 * 64)()
        off = ctypes.c_int64()
        _check(L.fireq_symm_handle(_ptr(self.buf), ctypes.cast(h, ctypes.c_void_p), ctypes.byref(off)),
               "fireq_symm_handle")
        allh = exchange((bytes(h), off.value))
        hs = (ctypes.c_uint8 * (64 * nranks))()
        offs = (ctypes.c_int64 * nranks)()
        for q, (hq, oq) in enumerate(allh):
            ctypes.memmove(ctypes.addressof(hs) + 64 * q, hq, 64)
            offs[q] = oq
        self.h = ctypes.c_void_p()
        _check(L.fireq_symm_open(ctypes.byref(self.h), nranks, rank, _ptr(self.buf), nbytes,
                                 ctypes.cast(hs, ctypes.c_void_p), ctypes.cast(offs, ctypes.c_void_p)),
               "fireq_symm_open")
        self.yt = self.buf[256:256 + nranks * N_local * M * 2].view(torch.bfloat16).view(nranks * N_local, M)

    def close(self):
        if self.h:
            _check(lib().fireq_symm_close(self.h), "fireq_symm_close")
            self.h = ctypes.c_void_p()


def w4a8_gemm_colpar_p2p(xq, beta, packed_local, scales_local, N_local, pts_n, symm, workspace, gamma_local=None,
                         stream=None):
    """Column-parallel GEMM with the all-gather fused into the epilogue (NVLink stores into every
    rank's symmetric buffer + device-side epoch flags; graph-capturable).  Returns symm.yt (the full Y^T) -- complete in stream order."""
    M, K = xq.shape
    ws = workspace.ensure(lib().fireq_w4a8_gemm_workspace_bytes(M, N_local, K), stream)
    _check(lib().fireq_w4a8_gemm_colpar_p2p(_ptr(xq), _ptr(beta), M, K, _ptr(packed_local), _ptr(scales_local),
                                            N_local, pts_n, _ptr(gamma_local), symm.h, _ptr(ws),
                                            ws.numel(), _stream(stream)),
           "fireq_w4a8_gemm_colpar_p2p")
    return symm.yt


# ------------------------------------------------------------ sigma_BF16 variant
def quantize_weight_bf16s(W, cas_mode=1, stream=None):
    """fireq_quantize_weight_bf16s: QuantizedWeight whose .scales are bf16 [N/128][K/128][128]."""
    assert W.dtype == torch.bfloat16 and W.dim() == 2 and W.is_contiguous()
    N, K = W.shape
    dev = W.device
    L = lib()
    packed = torch.empty(L.fireq_packed_weight_bytes(N, K), dtype=torch.uint8, device=dev)
    scales = torch.empty(N * K // 128, dtype=torch.bfloat16, device=dev)
    lam = torch.empty(K, dtype=torch.float32, device=dev)
    c = torch.empty(K, dtype=torch.bfloat16, device=dev)
    ps = torch.empty(2, dtype=torch.int32, device=dev)
    ws = _zeros_on(L.fireq_quantize_weight_workspace_bytes(N, K), dev, stream)
    _check(L.fireq_quantize_weight_bf16s(_ptr(W), N, K, cas_mode, _ptr(packed), _ptr(scales), _ptr(lam), _ptr(c),
                                         _ptr(ps), _ptr(ws), ws.numel(), _stream(stream)),
           "fireq_quantize_weight_bf16s")
    return QuantizedWeight(packed, scales, lam, c, ps, N, K)


def w4a8_gemm_bf16s(xq, beta, packed, scales_bf16, N, pts_n, out=None, workspace=None, stream=None):
    """Y = fireq_w4a8_gemm_bf16s(...): bf16 [M][N] (per-group scaled FP32 accumulation)."""
    M, K = xq.shape
    L = lib()
    need = L.fireq_w4a8_gemm_bf16s_workspace_bytes(M, N, K)
    ws = workspace.ensure(need, stream) if workspace is not None else _zeros_on(need, xq.device, stream)
    if out is None:
        out = torch.empty((M, N), dtype=torch.bfloat16, device=xq.device)
    _check(L.fireq_w4a8_gemm_bf16s(_ptr(xq), _ptr(beta), M, K, _ptr(packed), _ptr(scales_bf16), N, pts_n, _ptr(out),
                                   out.stride(0), _ptr(ws), ws.numel(), _stream(stream)), "fireq_w4a8_gemm_bf16s")
    return out


# ------------------------------------------------------------------ KV4Q8 attention (f4)
class KVCache:
    """INT4 keys and values of B sequences x Hkv heads (fireq_quantize_kv per head).

    k_packed / k_scales: uint8 [B*Hkv][N*d/2] / [B*Hkv][N*d/128] (layout v1 of K_post [N][d]);
    vt_packed / vt_scales: the same for V^T [d][N]; k_pts / v_pts: int32 [B*Hkv][2] {n, status}.
    """

    def __init__(self, K, V, chan_lambda=None, stream=None):
        """K, V: bf16 [B][Hkv][N][d] (K post-RoPE); chan_lambda: fp32 [B*Hkv][d] or [Hkv][d] or None."""
        B, Hkv, N, d = K.shape
        dev = K.device
        self.B, self.Hkv, self.N, self.d = B, Hkv, N, d
        H = B * Hkv
        self.k_packed = torch.empty((H, N * d // 2), dtype=torch.uint8, device=dev)
        self.k_scales = torch.empty((H, N * d // 128), dtype=torch.uint8, device=dev)
        self.vt_packed = torch.empty_like(self.k_packed)
        self.vt_scales = torch.empty_like(self.k_scales)
        self.k_pts = torch.zeros((H, 2), dtype=torch.int32, device=dev)
        self.v_pts = torch.zeros((H, 2), dtype=torch.int32, device=dev)
        L = lib()
        need = max(L.fireq_quantize_weight_workspace_bytes(N, d), L.fireq_quantize_weight_workspace_bytes(d, N))
        ws = _zeros_on(need, dev, stream)
        Kc = K.reshape(H, N, d).contiguous()
        Vt = V.reshape(H, N, d).transpose(1, 2).contiguous()          # [H][d][N]
        for x in range(H):
            lam = None
            if chan_lambda is not None:
                lam = chan_lambda[x] if chan_lambda.shape[0] == H else chan_lambda[x % Hkv]
                lam = lam.contiguous()
            _check(L.fireq_quantize_kv(_ptr(Kc[x]), N, d, _ptr(lam), _ptr(self.k_packed[x]), _ptr(self.k_scales[x]),
                                       _ptr(self.k_pts[x]), _ptr(ws), ws.numel(), _stream(stream)), "fireq_quantize_kv")
            _check(L.fireq_quantize_kv(_ptr(Vt[x]), d, N, None, _ptr(self.vt_packed[x]), _ptr(self.vt_scales[x]),
                                       _ptr(self.v_pts[x]), _ptr(ws), ws.numel(), _stream(stream)), "fireq_quantize_kv")
        if stream is not None:          # the temporaries are freed while the kernels may still run
            for t in (ws, Kc, Vt):
                t.record_stream(stream)


def kv4q8_attention(q_fp8, q_scale, cache, Hq, causal=True, tau=None, out=None, stream=None):
    """O = fireq_kv4q8_attention(...): q_fp8 uint8 [B][Hq][N][d], q_scale bf16 [B][Hq][N] ->
    bf16 [B*N][Hq*d] (token-major)."""
    B, N, d = cache.B, cache.N, cache.d
    if out is None:
        out = torch.empty((B * N, Hq * d), dtype=torch.bfloat16, device=q_fp8.device)
    tau = 1.0 / math.sqrt(d) if tau is None else tau
    _check(lib().fireq_kv4q8_attention(_ptr(q_fp8), _ptr(q_scale), B, N, Hq, cache.Hkv, d, _ptr(cache.k_packed),
                                       _ptr(cache.k_scales), _ptr(cache.k_pts), _ptr(cache.vt_packed),
                                       _ptr(cache.vt_scales), _ptr(cache.v_pts), 1 if causal else 0, tau, _ptr(out),
                                       out.stride(0), _stream(stream)), "fireq_kv4q8_attention")
    return out
