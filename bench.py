"""bench.py -- FireQ W4A8-FP linear layer on B200: the driver's benchmark contract.

Headline (BASELINE.json metric "... Llama FFN latency at batch 16", configs[1]):
one step = one Llama2-7B FFN at decode batch M = 16 through the library's online
hot path (all on-device, inputs resident in HBM):

  fireq_quantize_act(x, c_gu)            A1-A3  (FP8 activations, BF16 beta)
  fireq_w4a8_gemm(W_gu = [gate; up])     Steps 1-3 (INT4 x FP8 on tcgen05), gamma = [1 | c_down]
  fireq_silu_mul_quantize_act(g, u)      SiLU * up then A2-A3
  fireq_w4a8_gemm(W_down)

The weights are quantized offline by fireq_quantize_weight (W1-W6; timed once and
reported under "offline": the paper quantizes offline).  Four rotating copies
of the quantized FFN weights (4 x 68.7 MB > 2 x L2) are cycled so every step streams
its weights from HBM.  Each step is one CUDA graph replay (4 kernel launches).

Also reported (same run): the dominant kernel's roofline (the gate_up GEMM, HBM
bound at decode), single-GEMM decode figures, the prefill FFN (M = 16 x 1024,
FP8-tensor bound), an end-to-end figure through host buffers, GPU clocks, and the
CPU oracle timed on a bounded sample (cpu_baseline).

Run:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fireq|reference]
N > 1 (torchrun): column-parallel FFN (N-sharded gate_up and down, NCCL all-gather
of the BF16 outputs in the Y^T layout, in place).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

D_MODEL, D_FF = 4096, 11008          # Llama2-7B FFN (BASELINE configs[1])
M_DECODE = 16
M_PREFILL = 16 * 1024
ROTATIONS = 4
METRIC = "Llama2-7B FFN latency at batch 16 (W4A8-FP: INT4 weights + FP8 g128 scales, FP8 activations)"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ helpers
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms while running."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.idx = device_index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for i, nm in enumerate(names):
                if len(s) > 4 + i and s[4 + i].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def gemm_bytes(M, N, K):
    """Algorithmic bytes of one fireq_w4a8_gemm: packed W + sigma + X_hat + beta + Y."""
    return N * K // 2 + N * K // 128 + M * K + 2 * M + 2 * M * N


def act_bytes(M, K, chan=False):
    return 3 * M * K + 2 * M + (2 * K if chan else 0)


# ------------------------------------------------------------------ workload
class FFN:
    """Quantized Llama FFN weights + activation buffers on one GPU (optionally an N-shard)."""

    def __init__(self, F, M, rotations, dev, shard=None):
        self.F, self.M, self.dev = F, M, dev
        wg = synth.weights(D_FF, D_MODEL, synth.layer_seed(1, 0))
        wu = synth.weights(D_FF, D_MODEL, synth.layer_seed(1, 1))
        wd = synth.weights(D_MODEL, D_FF, synth.layer_seed(1, 2))
        W_gu = synth.bits_to_torch(np.concatenate([wg, wu], axis=0)).to(dev)
        W_d = synth.bits_to_torch(wd).to(dev)
        # offline quantization (W1-W6), timed once
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        q_gu = F.quantize_weight(W_gu, cas_mode=1)
        q_d = F.quantize_weight(W_d, cas_mode=1)
        torch.cuda.synchronize()
        self.offline_s = time.perf_counter() - t0
        self.n_gu, self.n_d = q_gu.n, q_d.n
        self.c_gu = q_gu.c
        self.gamma = torch.cat([torch.ones(D_FF, device=dev), q_d.c.float()])
        self.rot = []
        for r in range(rotations):
            self.rot.append((q_gu.packed.clone(), q_gu.scales.clone(), q_d.packed.clone(), q_d.scales.clone()))
        del W_gu, W_d
        x = synth.activations(M, D_MODEL, synth.layer_seed(1, 3))
        self.x = synth.bits_to_torch(x).to(dev)
        self.xq = torch.empty((M, D_MODEL), dtype=torch.uint8, device=dev)
        self.beta = torch.empty(M, dtype=torch.bfloat16, device=dev)
        self.gu = torch.empty((M, 2 * D_FF), dtype=torch.bfloat16, device=dev)
        self.hq = torch.empty((M, D_FF), dtype=torch.uint8, device=dev)
        self.hbeta = torch.empty(M, dtype=torch.bfloat16, device=dev)
        self.y = torch.empty((M, D_MODEL), dtype=torch.bfloat16, device=dev)
        self.ws1 = F.Workspace(F.gemm_workspace_bytes(M, 2 * D_FF, D_MODEL), dev)
        self.ws2 = F.Workspace(F.gemm_workspace_bytes(M, D_MODEL, D_FF), dev)

    def step(self, r, stream=None, prefetch=os.environ.get("BENCH_PREFETCH", "1") == "1", x=None, y=None):
        """One FFN: each GEMM also streams the next GEMM's weights into L2 once its own loads
        are issued (gate_up -> this step's down; down -> the next step's gate_up).
        x / y: other input / output buffers than self.x / self.y (the pipelined e2e)."""
        F = self.F
        p_gu, s_gu, p_d, s_d = self.rot[r]
        nxt = self.rot[(r + 1) % len(self.rot)]
        F.quantize_act(self.x if x is None else x, chan_mul=self.c_gu, out=(self.xq, self.beta), stream=stream)
        F.w4a8_gemm(self.xq, self.beta, p_gu, s_gu, 2 * D_FF, self.n_gu, gamma=self.gamma, out=self.gu,
                    workspace=self.ws1, stream=stream, prefetch=(p_d, s_d) if prefetch else None)
        F.silu_mul_quantize_act(self.gu[:, :D_FF], self.gu[:, D_FF:], out=(self.hq, self.hbeta), stream=stream)
        F.w4a8_gemm(self.hq, self.hbeta, p_d, s_d, D_MODEL, self.n_d, out=self.y if y is None else y, workspace=self.ws2, stream=stream,
                    prefetch=(nxt[0], nxt[1]) if prefetch else None)

    KERNELS_PER_STEP = 4

    def bytes_per_step(self):
        M = self.M
        return (act_bytes(M, D_MODEL, True) + gemm_bytes(M, 2 * D_FF, D_MODEL) + 2 * M * 2 * D_FF  # gu re-read
                + act_bytes(M, D_FF) + gemm_bytes(M, D_MODEL, D_FF))

    def flops_per_step(self):
        return 2 * self.M * (2 * D_FF * D_MODEL + D_MODEL * D_FF)


class FusedFFN:
    """The same FFN through fireq_ffn_w4a8_decode: 4 kernels per step (quantize_act(x);
    gate_up with the SwiGLU epilogue; quantize_act(h); down [+ residual in its epilogue]).
    W_gu in the interleaved row order."""

    KERNELS_PER_STEP = 4

    def __init__(self, F, M, rotations, dev):
        from types import SimpleNamespace as NS
        self.F, self.M, self.dev = F, M, dev
        Wg = synth.bits_to_torch(synth.weights(D_FF, D_MODEL, synth.layer_seed(1, 0))).to(dev)
        Wu = synth.bits_to_torch(synth.weights(D_FF, D_MODEL, synth.layer_seed(1, 1))).to(dev)
        W_d = synth.bits_to_torch(synth.weights(D_MODEL, D_FF, synth.layer_seed(1, 2))).to(dev)
        W_il = F.interleave_gate_up(Wg, Wu)
        q_gu = F.quantize_weight(W_il, cas_mode=1)
        q_d = F.quantize_weight(W_d, cas_mode=1)
        del Wg, Wu, W_d, W_il
        self.rot = []
        for _ in range(rotations):
            self.rot.append((NS(packed=q_gu.packed.clone(), scales=q_gu.scales.clone(), c=q_gu.c, n=q_gu.n, K=D_MODEL),
                             NS(packed=q_d.packed.clone(), scales=q_d.scales.clone(), c=q_d.c, n=q_d.n, K=D_FF)))
        self.x = synth.bits_to_torch(synth.activations(M, D_MODEL, synth.layer_seed(1, 3))).to(dev)
        self.h = torch.empty((M, D_FF), dtype=torch.bfloat16, device=dev)
        self.y = torch.empty((M, D_MODEL), dtype=torch.bfloat16, device=dev)
        self.ws = F.Workspace(F.ffn_workspace_bytes(M, D_MODEL, D_FF), dev)

    def step(self, r, stream=None, residual=False, x=None, y=None):
        q_gu, q_d = self.rot[r]
        nxt = self.rot[(r + 1) % len(self.rot)][0]
        pf = (nxt.packed, nxt.scales) if os.environ.get("BENCH_PREFETCH", "1") == "1" else None
        x = self.x if x is None else x
        self.F.ffn_w4a8_decode(x, q_gu, q_d, h=self.h, out=self.y if y is None else y, workspace=self.ws,
                               stream=stream, prefetch=pf, residual=x if residual else None)

    def bytes_per_step(self):
        M = self.M
        # quantize_act(x) + gate_up (W, x_hat, h written, h re-read + h_hat written) + down
        return (act_bytes(M, D_MODEL, True) + gemm_bytes(M, 2 * D_FF, D_MODEL) - 2 * M * 2 * D_FF + 2 * M * D_FF
                + 2 * D_FF + act_bytes(M, D_FF) + gemm_bytes(M, D_MODEL, D_FF))


def capture(fn, stream):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        fn()
    return g


def time_steps(g_multi, g_single, steps, warmup, stream, barrier=None):
    """Exactly `steps` steps: steps // R replays of the R-step graph + the remainder singly."""
    R = len(g_single)
    for i in range(max(1, warmup // R)):
        g_multi.replay()
    torch.cuda.synchronize()
    if barrier:
        barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(steps // R):
            g_multi.replay()
        for r in range(steps % R):
            g_single[r].replay()
        e1.record(stream)
    torch.cuda.synchronize()
    if barrier:
        barrier()
    return e0.elapsed_time(e1)


def time_graphs(graphs, steps, warmup, stream, barrier=None):
    """Replay graphs round-robin; returns total ms for exactly `steps` replays (CUDA events)."""
    for i in range(warmup):
        graphs[i % len(graphs)].replay()
    torch.cuda.synchronize()
    if barrier:
        barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for i in range(steps):
            graphs[i % len(graphs)].replay()
        e1.record(stream)
    torch.cuda.synchronize()
    if barrier:
        barrier()
    return e0.elapsed_time(e1)


# ------------------------------------------------------------------ CPU oracle
def host_info():
    """nproc, sockets and CPU model of the host the oracle runs on (lscpu)."""
    info = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core"):
                info[k.strip()] = v.strip()
    except Exception:
        pass
    return info


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([p.get("num_threads", 1) for p in threadpool_info()] + [1])
    except Exception:
        return 1


class OracleFFN:
    """The oracle's Llama2-7B FFN step (decode batch 16), as it stands: A1-A3 on x, the
    fp64 LUT-dequant reference GEMM over the full [gate; up] (22016 x 4096), SiLU * up,
    A2-A3 on h, the fp64 reference down GEMM (4096 x 11008).  Weights are packed codes
    and scale codes (layout v1) drawn at random: the oracle's time does not depend on
    their values; the GPU arm's weights are quantized offline the same way."""

    def __init__(self, M=M_DECODE):
        from oracle import numerics as nm
        rng = np.random.default_rng(0)
        self.M = M
        self.X = synth.bits_to_f64(synth.activations(M, D_MODEL, 1))
        self.c = nm.bf16_rn(np.exp(rng.normal(0.0, 0.3, D_MODEL)))
        self.p_gu = rng.integers(0, 256, 2 * D_FF * D_MODEL // 2, dtype=np.uint8)
        self.s_gu = rng.integers(40, 60, 2 * D_FF * D_MODEL // 128).astype(np.uint8)
        self.p_d = rng.integers(0, 256, D_MODEL * D_FF // 2, dtype=np.uint8)
        self.s_d = rng.integers(40, 60, D_MODEL * D_FF // 128).astype(np.uint8)

    def step(self):
        """One full FFN step; returns {phase: seconds} (no sampling, no extrapolation)."""
        from oracle import gemm as og, quant as oq, ffn as of, numerics as nm
        t0 = time.perf_counter()
        xq, beta = oq.quantize_act(self.X, self.c)
        t1 = time.perf_counter()
        r = og.gemm_reference(xq, beta, self.p_gu, self.s_gu, 2 * D_FF, D_MODEL, 10)
        t2 = time.perf_counter()
        h = of.silu_mul(nm.bf16_rn(r[:, :D_FF]), nm.bf16_rn(r[:, D_FF:]))
        hq, hb = oq.quantize_act(h)
        t3 = time.perf_counter()
        og.gemm_reference(hq, hb, self.p_d, self.s_d, D_MODEL, D_FF, 10)
        t4 = time.perf_counter()
        return {"quantize_act_x": t1 - t0, "gemm_gate_up": t2 - t1, "silu_mul_quantize_act_h": t3 - t2,
                "gemm_down": t4 - t3, "total": t4 - t0}


def oracle_c1_phases(reps=3):
    """BASELINE configs[0] (C1: q_proj 4096 x 4096, M = 16) per phase: quantize-weight,
    quantize-act, fp64 reference GEMM -- median of `reps` with all BLAS threads, and one run
    with a single thread."""
    from oracle import gemm as og, quant as oq
    W = synth.bits_to_f64(synth.weights(4096, 4096, synth.layer_seed(0, 0)))
    X = synth.bits_to_f64(synth.activations(16, 4096, synth.layer_seed(0, 1)))

    def once():
        t0 = time.perf_counter()
        q = oq.quantize_weight(W, 1)
        t1 = time.perf_counter()
        xq, beta = oq.quantize_act(X, q.c)
        t2 = time.perf_counter()
        og.gemm_reference(xq, beta, q.packed, q.scales, 4096, 4096, q.n)
        t3 = time.perf_counter()
        return t1 - t0, t2 - t1, t3 - t2

    runs = [once() for _ in range(reps)]
    med = [statistics.median(r[i] for r in runs) for i in range(3)]
    one = None
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1):
            one = once()
    except Exception:
        pass
    ms = lambda v: round(v * 1e3, 2)
    out = {"workload": "C1 q_proj M=16 K=4096 N=4096", "threads": blas_threads(),
           "quantize_weight_ms": ms(med[0]), "quantize_act_ms": ms(med[1]), "gemm_ms": ms(med[2])}
    if one:
        out["one_thread"] = {"quantize_weight_ms": ms(one[0]), "quantize_act_ms": ms(one[1]), "gemm_ms": ms(one[2])}
    return out


def cpu_oracle_baseline():
    """cpu_baseline of the GPU arm: one FULL oracle FFN step (the metric's unit, no scaling)
    with its phases, plus C1's per-phase times, on this host's cores."""
    ffn = OracleFFN()
    ph = ffn.step()
    return {"value": round(ph["total"] * 1e6, 1), "unit": "us", "cores": blas_threads(), "kind": "oracle",
            "sample": "one full Llama2-7B FFN step at batch 16 (act-quant x, fp64 LUT-dequant gate_up 22016x4096, "
                      "SiLU*up + act-quant h, fp64 down 4096x11008); no sampling or extrapolation",
            "phases_ms": {k: round(v * 1e3, 1) for k, v in ph.items() if k != "total"},
            "c1": oracle_c1_phases(), "host": host_info()}


# ------------------------------------------------------------------ arms
def run_reference(args, rank, world):
    """--impl reference: there is no installable reference implementation (the reference is a
    paper), so this arm times the CPU oracle as it stands: every step is one FULL oracle FFN
    step (about 8 s on a 16-core host), so value x steps is the wall time of the timed loop."""
    if rank != 0:
        return
    ffn = OracleFFN()
    for _ in range(args.warmup):
        ffn.step()
    t0 = time.perf_counter()
    steps = [ffn.step() for _ in range(args.steps)]
    wall = time.perf_counter() - t0
    v = statistics.median(s["total"] for s in steps) * 1e6
    cb = {"value": round(v, 1), "unit": "us", "cores": blas_threads(), "kind": "oracle",
          "sample": f"{args.steps} full Llama2-7B FFN steps at batch 16 (median), no extrapolation; timed loop "
                    f"{wall:.1f} s", "host": host_info(),
          "phases_ms": {k: round(statistics.median(s[k] for s in steps) * 1e3, 1) for k in steps[0] if k != "total"}}
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 1), "unit": "us", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(v / 1e3, 3), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "llama2-7b-ffn-decode-b16", "tokens": M_DECODE, "d_model": D_MODEL,
                       "d_ff": D_FF},
            "cpu_baseline": cb, "e2e": {"value": round(v, 1), "unit": "us", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_fireq(args, rank, world, dev):
    from paper_2505_20839_b200 import fireq as F
    F.load()
    peaks, peak_src = load_peaks()
    stream = torch.cuda.Stream(device=dev)
    if world > 1 or args.colpar:
        from paper_2505_20839_b200 import multigpu
        return multigpu.run_colpar_bench(args, rank, world, dev, F, stream, peaks, peak_src, clock_cls=ClockSampler)

    # ---------------- decode FFN (headline): the FFN block fireq_ffn_w4a8_decode (quantize_act(x);
    # gate_up with the SwiGLU epilogue; quantize_act(h); down).  The same FFN as the 4-call chain
    # (quantize_act, gemm, silu_mul_quantize_act, gemm) is timed below as `chain_api_us`.
    ffn = FFN(F, M_DECODE, ROTATIONS, dev)
    fused = FusedFFN(F, M_DECODE, ROTATIONS, dev)
    step_bytes = fused.bytes_per_step()
    h2d_bytes, d2h_bytes = fused.x.numel() * 2, fused.y.numel() * 2
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for r in range(ROTATIONS):          # first launches outside capture (TMA maps, func attrs)
            fused.step(r, stream)
            ffn.step(r, stream)
    torch.cuda.synchronize()
    # one graph = ROTATIONS consecutive steps (distinct weight copies), PDL edges inside;
    # a remainder uses single-step graphs so that exactly args.steps steps are timed.
    g_multi = capture(lambda: [fused.step(r, stream) for r in range(ROTATIONS)], stream)
    g_single = [capture(lambda r=r: fused.step(r, stream), stream) for r in range(ROTATIONS)]
    clocks = ClockSampler(dev.index or 0)
    clocks.start()
    time.sleep(0.25)
    # long enough for the clock sampler: repeat the timed region, keep the K-step one
    time_steps(g_multi, g_single, max(2000, args.steps), args.warmup, stream)
    total_ms = time_steps(g_multi, g_single, args.steps, args.warmup, stream)
    clocks.stop()
    us_per_step = total_ms * 1e3 / args.steps

    # end to end through host buffers: every step copies its own input x_r (pinned host) to the
    # device, runs the public calls and reads its result y_r back to pinned host memory.
    # Serial: H2D -> step -> D2H on one stream.  Pipelined (reported as e2e.value): the copies run
    # on their own streams into double-buffered device x / y, so step r+1's H2D and step r-1's
    # D2H overlap step r's kernels; the dependencies are H2D_r -> step_r -> D2H_r, and the buffer
    # reuse edges step_{r-2} -> H2D_r (x) and D2H_{r-2} -> step_r (y).
    x_hosts = [(fused.x * (1 + 0.25 * r)).cpu().pin_memory() for r in range(ROTATIONS)]
    y_hosts = [torch.empty_like(fused.y, device="cpu").pin_memory() for _ in range(ROTATIONS)]

    def e2e_serial_step(r):
        fused.x.copy_(x_hosts[r], non_blocking=True)
        fused.step(r, stream)
        y_hosts[r].copy_(fused.y, non_blocking=True)

    s_h2d = torch.cuda.Stream(device=dev)
    s_d2h = torch.cuda.Stream(device=dev)
    E2E_GROUP = int(os.environ.get("BENCH_E2E_GROUP", "4"))
    NBUF = 4 * ROTATIONS                          # one device x / y per step of a 16-step graph
    xd = [torch.empty_like(fused.x) for _ in range(NBUF)]
    yd = [torch.empty_like(fused.y) for _ in range(NBUF)]

    def e2e_pipelined(rs):
        """Steps rs (a graph body, len(rs) <= NBUF): fork the copy streams from `stream`, join them
        at the end.  Step i's input is uploaded into its own device buffer on the H2D stream; the
        compute stream waits for the uploads of a group of E2E_GROUP steps before the group's first
        step (so the steps inside a group keep their kernel-to-kernel PDL edges), and each step's
        result is downloaded on the D2H stream as soon as its last kernel is done."""
        ev = lambda: torch.cuda.Event()  # noqa: E731
        fork = ev()
        fork.record(stream)
        s_h2d.wait_event(fork)
        s_d2h.wait_event(fork)
        h2d_done = []
        with torch.cuda.stream(s_h2d):
            for i, r in enumerate(rs):
                xd[i].copy_(x_hosts[r], non_blocking=True)
                h2d_done.append(ev())
                h2d_done[i].record(s_h2d)
        for i, r in enumerate(rs):
            if i % E2E_GROUP == 0:
                stream.wait_event(h2d_done[min(i + E2E_GROUP, len(rs)) - 1])
            fused.step(r, stream, x=xd[i], y=yd[i])
            done = ev()
            done.record(stream)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(done)
                y_hosts[r].copy_(yd[i], non_blocking=True)
        stream.wait_stream(s_h2d)
        stream.wait_stream(s_d2h)

    with torch.cuda.stream(stream):
        for r in range(ROTATIONS):
            e2e_serial_step(r)
        e2e_pipelined(list(range(ROTATIONS)))
    torch.cuda.synchronize()
    g_e2e_multi = capture(lambda: [e2e_serial_step(r) for r in range(ROTATIONS)], stream)
    g_e2e = [capture(lambda r=r: e2e_serial_step(r), stream) for r in range(ROTATIONS)]
    e2e_serial_ms = time_steps(g_e2e_multi, g_e2e, args.steps, args.warmup, stream) / args.steps
    del g_e2e_multi, g_e2e
    # 16 steps per graph: the pipeline fills and drains once per graph replay
    seq = [r % ROTATIONS for r in range(4 * ROTATIONS)]
    g_e2e_multi = capture(lambda: e2e_pipelined(seq), stream)
    g_e2e = [capture(lambda r=r: e2e_pipelined([r]), stream) for r in seq]
    e2e_ms = time_steps(g_e2e_multi, g_e2e, args.steps, args.warmup, stream) / args.steps
    del g_e2e_multi, g_e2e
    # the pipelined result equals the serial one (same inputs, same kernels)
    y_pipe = [y.clone() for y in y_hosts]
    with torch.cuda.stream(stream):
        for r in range(ROTATIONS):
            e2e_serial_step(r)
    torch.cuda.synchronize()
    e2e_same = all(torch.equal(a, b) for a, b in zip(y_pipe, y_hosts))

    # ---------------- dominant kernel: the gate_up GEMM alone (HBM bound), rotating weights
    def gu_only(r):
        p_gu, s_gu, _, _ = ffn.rot[r]
        F.w4a8_gemm(ffn.xq, ffn.beta, p_gu, s_gu, 2 * D_FF, ffn.n_gu, gamma=ffn.gamma, out=ffn.gu,
                    workspace=ffn.ws1, stream=stream)

    def d_only(r):
        _, _, p_d, s_d = ffn.rot[r]
        F.w4a8_gemm(ffn.hq, ffn.hbeta, p_d, s_d, D_MODEL, ffn.n_d, out=ffn.y, workspace=ffn.ws2, stream=stream)

    # one launch per weight copy, copies in rotation (4 x 46.6 MB > L2): every launch streams
    # its weights from HBM; 32 PDL-chained launches per graph, so graph-replay gaps do not
    # count as kernel time
    reps, per_graph = 25, 8
    g_gu = capture(lambda: [gu_only(r) for _ in range(per_graph) for r in range(ROTATIONS)], stream)
    ms_gu = time_graphs([g_gu], reps, 2, stream) / (reps * ROTATIONS * per_graph)
    g_d = capture(lambda: [d_only(r) for _ in range(per_graph) for r in range(ROTATIONS)], stream)
    ms_d = time_graphs([g_d], reps, 2, stream) / (reps * ROTATIONS * per_graph)
    b_gu = gemm_bytes(M_DECODE, 2 * D_FF, D_MODEL)
    gbs_gu = b_gu / (ms_gu * 1e-3) / 1e9
    b_d = gemm_bytes(M_DECODE, D_MODEL, D_FF)
    gbs_d = b_d / (ms_d * 1e-3) / 1e9
    # ---------------- the same FFN as the 4-call chain (quantize_act, gemm, silu_mul_quantize_act, gemm)
    gc_multi = capture(lambda: [ffn.step(r, stream) for r in range(ROTATIONS)], stream)
    gc_single = [capture(lambda r=r: ffn.step(r, stream), stream) for r in range(ROTATIONS)]
    chain_us = time_steps(gc_multi, gc_single, args.steps, args.warmup, stream) * 1e3 / args.steps
    del gc_multi, gc_single
    # the unfused FFN block: the 4-kernel chain + the residual add as its own kernel
    def chain_res(r):
        ffn.step(r, stream)
        ffn.y.add_(ffn.x)
    g_cr = capture(lambda: [chain_res(r) for r in range(ROTATIONS)], stream)
    g_cr1 = [capture(lambda r=r: chain_res(r), stream) for r in range(ROTATIONS)]
    chain_res_us = time_steps(g_cr, g_cr1, args.steps, args.warmup, stream) * 1e3 / args.steps
    del g_cr, g_cr1
    # the FFN block with its residual connection fused into the down GEMM's epilogue
    gf_multi = capture(lambda: [fused.step(r, stream, residual=True) for r in range(ROTATIONS)], stream)
    gf_single = [capture(lambda r=r: fused.step(r, stream, residual=True), stream) for r in range(ROTATIONS)]
    fused_res_us = time_steps(gf_multi, gf_single, args.steps, args.warmup, stream) * 1e3 / args.steps
    del gf_multi, gf_single, fused
    torch.cuda.empty_cache()

    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("gemm_gate_up_m16_bytes_per_launch")

    # ---------------- prefill FFN (FP8 tensor bound) and single-GEMM figures
    del g_multi, g_single, g_gu, g_d
    chain_info = decode_chain_figures(F, dev, stream, peaks)
    chain_info["fused_qkv_gate_up"] = decode_chain_figures(F, dev, stream, peaks, fused=True)
    pre_info = prefill_figures(F, dev, stream, peaks) if not args.no_prefill else None
    # BASELINE configs[3] at P = 1 (the column-parallel runs report P = 2/4/8)
    from paper_2505_20839_b200.c4 import c4_figures
    c4_info = c4_figures(F, dev, stream, 0, 1, comm=None) if not args.no_c4 else None
    attn_info = attention_figures(F, dev, stream, peaks) if not args.no_attention else None

    # ---------------- cpu baseline (oracle on a bounded sample)
    cpu = cpu_oracle_baseline() if not args.no_cpu else None

    hbm = peaks["hbm_gbs"]
    line = {
        "metric": METRIC, "value": round(us_per_step, 3), "unit": "us", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(us_per_step / 1e3, 6), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "fp8e4m3 x int4 -> f32 acc -> bf16", "data": "synthetic",
        "config": {"workload": "llama2-7b-ffn-decode-b16", "tokens": M_DECODE, "d_model": D_MODEL, "d_ff": D_FF,
                   "gemms": "gate_up 22016x4096 (fused, gamma=[1|c_down]) + down 4096x11008",
                   "api": "fireq_ffn_w4a8_decode (quantize_act(x); gate_up + SwiGLU epilogue; quantize_act(h); "
                          "down)",
                   "parallelism": "single GPU",
                   "l2": f"{ROTATIONS} rotating weight copies ({ROTATIONS * (b_gu + b_d) / 1e6:.0f} MB > 2x L2)",
                   "graph": f"CUDA graphs of {ROTATIONS} steps (4 PDL-chained kernels per step)"},
        "gpu_launches": FusedFFN.KERNELS_PER_STEP * args.steps,
        "step_gbs": round(step_bytes / (us_per_step * 1e-6) / 1e9, 1),
        "step_hbm_frac": round(step_bytes / (us_per_step * 1e-6) / 1e9 / peaks["hbm_gbs"], 4),
        "chain_api_us": round(chain_us, 3),
        "chain_api": "fireq_quantize_act, fireq_w4a8_gemm, fireq_silu_mul_quantize_act, fireq_w4a8_gemm",
        "ffn_block_residual": {"fused_us": round(fused_res_us, 3), "unfused_chain_plus_add_us": round(chain_res_us, 3),
                               "fused": "fireq_ffn_w4a8_decode: SwiGLU in gate_up's epilogue, residual in down's",
                               "unfused": "the 4-kernel chain + y += x as its own kernel"},
        "roofline": {"bound": "hbm", "kernel": "fireq_w4a8_gemm gate_up M=16 N=22016 K=4096",
                     "kernel_note": "the step's dominant kernel is this GEMM with the SwiGLU pair epilogue inside "
                                    "fireq_ffn_w4a8_decode (not callable alone); timed here through fireq_w4a8_gemm "
                                    "with the plain epilogue, same weights, same mainloop",
                     "achieved": round(gbs_gu, 1), "peak": hbm, "unit": "GB/s", "frac": round(gbs_gu / hbm, 4),
                     "traffic": traffic, "traffic_source": "stored: profiles/traffic.json, ncu --set full "
                     "dram__bytes_read.sum + dram__bytes_write.sum of this kernel (not measured in this run)",
                     "algorithmic_bytes": b_gu, "launch_us": round(ms_gu * 1e3, 3),
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})"},
        "gemm_down": {"us": round(ms_d * 1e3, 3), "gbs": round(gbs_d, 1), "frac": round(gbs_d / hbm, 4)},
        "e2e": {"value": round(e2e_ms * 1e3, 3), "unit": "us", "h2d_bytes_per_step": h2d_bytes,
                "d2h_bytes_per_step": d2h_bytes,
                "mode": f"pipelined: per-step H2D / D2H on copy streams into per-step device buffers, the compute stream waits for the uploads of {E2E_GROUP} steps at a time; graphs of 16 steps",
                "serial_us": round(e2e_serial_ms * 1e3, 3), "pipelined_equals_serial": e2e_same},
        "offline": {"quantize_weight_ms_gate_up_and_down": round(ffn.offline_s * 1e3, 2)},
        "clocks": clocks.summary(),
    }
    line["decode_chain"] = chain_info
    if pre_info:
        line["prefill"] = pre_info
    if c4_info:
        line["c4_llama2_70b_ffn"] = c4_info
    if attn_info:
        line["kv4q8_attention"] = attn_info
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


def decode_chain_figures(F, dev, stream, peaks, layers=4, fused=False):
    """SURVEY §8(d) d4 primary decode number (steady state): one CUDA graph of PDL-chained
    decode GEMMs (M = 16) over DISTINCT weight matrices -- the 7 Llama3-8B linear shapes
    x 4 layers, 436 MB of packed weights (> 2 x L2) -- GB/s = sum of algorithmic bytes /
    time.  One layer is quantized from the synthetic generator; the other layers are
    copies at distinct addresses (values do not change the speed)."""
    M = M_DECODE
    shapes = [("q", 4096, 4096), ("k", 1024, 4096), ("v", 1024, 4096), ("o", 4096, 4096),
              ("gate", 14336, 4096), ("up", 14336, 4096), ("down", 4096, 14336)]
    if fused:      # serving-style merged projections: [q; k; v] and [gate; up] as one weight each
        shapes = [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]
    xs = {}
    gemms = []
    for name, N, K in shapes:
        W = synth.bits_to_torch(synth.weights(N, K, synth.layer_seed(3, len(gemms)))).to(dev)
        qw = F.quantize_weight(W, cas_mode=1)
        n = qw.n
        del W
        if K not in xs:
            X = synth.bits_to_torch(synth.activations(M, K, synth.layer_seed(3, 100 + K % 97))).to(dev)
            xs[K] = F.quantize_act(X)
        copies = [(qw.packed, qw.scales)] + [(qw.packed.clone(), qw.scales.clone()) for _ in range(layers - 1)]
        out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
        ws = F.Workspace(F.gemm_workspace_bytes(M, N, K), dev)
        gemms.append((N, K, n, copies, out, ws))
    torch.cuda.synchronize()

    seq = [(layer, i) for layer in range(layers) for i in range(len(gemms))]

    def chain(prefetch):
        for j, (layer, i) in enumerate(seq):
            N, K, n, copies, out, ws = gemms[i]
            xq, beta = xs[K]
            p, sc = copies[layer]
            nl, ni = seq[(j + 1) % len(seq)]
            nxt = gemms[ni][3][nl] if prefetch else None     # stream the next GEMM's weights into L2
            F.w4a8_gemm(xq, beta, p, sc, N, n, out=out, workspace=ws, stream=stream, prefetch=nxt)

    nbytes = layers * sum(gemm_bytes(M, N, K) for _, N, K in shapes)
    res = {"workload": "llama3-8b-decode-linear-chain" + ("-fused-qkv-gate-up" if fused else ""),
           "tokens": M, "layers": layers,
           "gemms": layers * len(shapes), "weight_mb": round(nbytes / 1e6, 1),
           "graph": "PDL-chained fireq_w4a8_gemm launches"}
    for key, pf in (("plain", False), ("l2_prefetch_next", True)):
        with torch.cuda.stream(stream):
            chain(pf)
        torch.cuda.synchronize()
        g = capture(lambda: chain(pf), stream)
        reps = 30
        ms = time_graphs([g], reps, 3, stream) / reps
        gbs = nbytes / (ms * 1e-3) / 1e9
        res[key] = {"us_per_layer": round(ms * 1e3 / layers, 2), "gbs": round(gbs, 1),
                    "frac": round(gbs / peaks["hbm_gbs"], 4)}
        del g
    del gemms, xs
    torch.cuda.empty_cache()
    return res


def prefill_figures(F, dev, stream, peaks):
    """Prefill FFN at M = 16 x 1024: tensor-bound; TFLOP/s of each GEMM vs the FP8 peak."""
    M = M_PREFILL
    fp8_peak = 2.0 * peaks["bf16_tflops"]           # dense FP8 = 2 x measured bf16 (guide's nominal ratio)
    ffn = FFN(F, M, 1, dev)
    with torch.cuda.stream(stream):
        ffn.step(0, stream)
    torch.cuda.synchronize()
    p_gu, s_gu, p_d, s_d = ffn.rot[0]

    def t(fn, reps=5):
        with torch.cuda.stream(stream):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(reps):
                fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    ms_gu = t(lambda: F.w4a8_gemm(ffn.xq, ffn.beta, p_gu, s_gu, 2 * D_FF, ffn.n_gu, gamma=ffn.gamma, out=ffn.gu,
                                  workspace=ffn.ws1, stream=stream))
    ms_d = t(lambda: F.w4a8_gemm(ffn.hq, ffn.hbeta, p_d, s_d, D_MODEL, ffn.n_d, out=ffn.y, workspace=ffn.ws2,
                                 stream=stream))
    ms_ffn = t(lambda: ffn.step(0, stream), reps=3)
    flops = ffn.flops_per_step()
    del ffn
    torch.cuda.empty_cache()
    fused = FusedFFN(F, M, 1, dev)       # fireq_ffn_w4a8_decode at prefill M (SwiGLU in gate_up's epilogue)
    ms_fused = t(lambda: fused.step(0, stream), reps=3)
    del fused
    torch.cuda.empty_cache()
    tf_gu = 2 * M * 2 * D_FF * D_MODEL / (ms_gu * 1e-3) / 1e12
    tf_d = 2 * M * D_MODEL * D_FF / (ms_d * 1e-3) / 1e12
    tf_ffn = flops / (ms_ffn * 1e-3) / 1e12
    tf_fused = flops / (ms_fused * 1e-3) / 1e12
    return {"workload": "llama2-7b-ffn-prefill-16x1024", "ffn_ms": round(ms_ffn, 3), "ffn_tflops": round(tf_ffn, 1),
            "fused_ffn_api_ms": round(ms_fused, 3), "frac_fused_ffn": round(tf_fused / fp8_peak, 4),
            "gate_up_ms": round(ms_gu, 3), "gate_up_tflops": round(tf_gu, 1), "down_ms": round(ms_d, 3),
            "down_tflops": round(tf_d, 1), "fp8_peak_tflops": fp8_peak,
            "frac_gate_up": round(tf_gu / fp8_peak, 4), "frac_ffn": round(tf_ffn / fp8_peak, 4),
            "peak_source": "2 x MEASURED_PEAKS bf16_tflops (burst)"}


def attention_figures(F, dev, stream, peaks, B=16, N=1024, Hq=32, Hkv=8):
    """KV4Q8 prefill attention (NEXT f4) on Llama3-8B's attention shape (32 query heads, 8 kv
    heads, d = 128), B sequences of N tokens, causal: fireq_kv4q8_attention timed over a graph of
    launches; algorithmic flops = 4 d sum_q (q + 1) per (sequence, head) (S and O, causal)."""
    fp8_peak = 2.0 * peaks["bf16_tflops"]
    qb, kb, vb = synth.attention(B, N, Hq, Hkv, synth.layer_seed(6, 0))
    Q, K, V = (synth.bits_to_torch(x).to(dev) for x in (qb, kb, vb))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cache = F.KVCache(K, V)
    torch.cuda.synchronize()
    cache_ms = (time.perf_counter() - t0) * 1e3
    xq, beta = F.quantize_act(Q.reshape(B * Hq * N, 128))
    q_fp8, q_scale = xq.reshape(B, Hq, N, 128), beta.reshape(B, Hq, N)
    out = torch.empty((B * N, Hq * 128), dtype=torch.bfloat16, device=dev)
    with torch.cuda.stream(stream):
        F.kv4q8_attention(q_fp8, q_scale, cache, Hq, out=out, stream=stream)
    torch.cuda.synchronize()
    per = 10
    g = capture(lambda: [F.kv4q8_attention(q_fp8, q_scale, cache, Hq, out=out, stream=stream) for _ in range(per)],
                stream)
    ms = time_graphs([g], 10, 2, stream) / (10 * per)
    flops = 4.0 * 128 * B * Hq * N * (N + 1) / 2
    tf = flops / (ms * 1e-3) / 1e12
    del cache, g
    torch.cuda.empty_cache()
    return {"workload": f"llama3-8b-attention-prefill-{B}x{N}", "heads": f"{Hq} q / {Hkv} kv, d=128, causal",
            "kernel": "fireq_kv4q8_attention (INT4 K/V cache, FP8 Q and softmax, Alg. 1 online softmax)",
            "us": round(ms * 1e3, 2), "tflops_algorithmic": round(tf, 1), "fp8_peak_tflops": fp8_peak,
            "frac_fp8": round(tf / fp8_peak, 4), "kv_cache_quantize_ms_host_loop": round(cache_ms, 2),
            "peak_source": "2 x MEASURED_PEAKS bf16_tflops (burst)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", choices=["fireq", "reference"], default="fireq")
    ap.add_argument("--no-prefill", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the Llama2-70B column-parallel figures")
    ap.add_argument("--no-attention", action="store_true", help="skip the KV4Q8 attention figures")
    ap.add_argument("--colpar", action="store_true", help="column-parallel path even at N=1 (testing)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if not torch.cuda.is_available():
        raise SystemExit("bench.py --impl fireq needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist_on = world > 1 or args.colpar
    if dist_on:
        # NCCL may print its version on stdout; the bench's stdout is ONE JSON line
        if not os.environ.get("FIREQ_KEEP_NCCL_DEBUG"):
            os.environ["NCCL_DEBUG"] = "NONE"
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        torch.distributed.init_process_group("nccl", device_id=dev)
    try:
        run_fireq(args, rank, world, dev)
    finally:
        if dist_on:
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
