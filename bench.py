"""FlashButterfly-B200 benchmark (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

A step = one pass of the hot path over one batch of synthetic input:
K1 kernel prep (regularize + kernel spectrum, once per call like the
reference, regularize.cpp:157) + forward + backward (du, dK, dD).
Metric (BASELINE.json): long-conv fwd+bwd elements/sec, E = B*H*N per step.

Multi-GPU (torchrun, one process per GPU): heads are sharded with no
communication (weak scaling: every rank owns a full per-GPU workload of H
heads); the barrier + max-over-ranks device time give the job time.

--impl reference runs the reference's own CPU implementation (the
unmodified /root/reference sources compiled in oracle/_ref) on the host
cores of this box, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # BASELINE.json configs[i] -> (B, H, N, dtype, engine, workload)
    1: dict(B=1, H=1, N=1024, dtype="f32", engine="auto",
            workload="config1: single-channel causal B=1 H=1 N=1024 fp32 fwd+bwd"),
    2: dict(B=32, H=256, N=4096, dtype="bf16", engine="single",
            workload="config2: LRA-scale B=32 H=256 N=4096 single-pass fwd+bwd, Squash/Smooth"),
    3: dict(B=16, H=128, N=65536, dtype="bf16", engine="three",
            workload="config3: Path256-scale B=16 H=128 N=65536 three-pass fwd+bwd"),
    4: dict(B=8, H=768, N=1024, dtype="bf16", engine="learned", r=16,
            workload="config4: learned-butterfly B=8 H=768 n=1024 fwd+bwd incl. block gradients"),
    # config 5 (sweep N=256..1M at B*H=2048): --config 5 --n N
    5: dict(B=8, H=256, N=4096, dtype="bf16", engine="auto",
            workload="config5: sequence-length sweep at B*H=2048"),
    # config 5-4M: N = 4M sequence-sharded over the ranks (report only);
    # --bh lowers B*H when few GPUs hold the whole sequence
    6: dict(B=8, H=256, N=4194304, dtype="f32", engine="seqshard",
            workload="config5-4M: N=4M sequence-sharded four-step fwd+bwd"),
}
LAM, P = 0.003, 1


def load_peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.mark_at = 0
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.05)

    def mark(self):
        """Start of the timed region (samples before it come from warm-up)."""
        self.mark_at = len(self.samples)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        # timed-region samples, plus the last warm-up sample when the timed
        # region is shorter than one polling interval
        timed = self.samples[max(0, self.mark_at - 1):]
        if not timed:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        self.samples = timed
        sm = sorted(float(s[0]) for s in self.samples)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(self.samples[0][1]),
                "reasons": reasons, "samples": len(sm)}


def _traffic(config, direction):
    """Measured DRAM bytes per launch of the dominant kernel (profiles/traffic.json)."""
    prof = ROOT / "profiles" / "traffic.json"
    if not prof.exists():
        return None
    return json.loads(prof.read_text()).get(f"config{config}", {}).get(direction)


def alg_bytes(cfg, s):
    """Algorithmic HBM bytes per step."""
    E = cfg["B"] * cfg["H"] * cfg["N"]
    HN = cfg["H"] * cfg["N"]
    if cfg["engine"] == "three":
        return 25 * s * E + 48 * HN
    return 5 * s * E + 32 * HN


def run_ours(args, cfg, rank, world, local_rank):
    import torch

    import paper_2302_06646_b200 as fb
    from paper_2302_06646_b200 import _lib

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    dt = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}[cfg["dtype"]]
    s = torch.tensor([], dtype=dt).element_size()
    B, H, N = cfg["B"], cfg["H"], cfg["N"]
    eng = {"auto": fb.Engine.AUTO, "single": fb.Engine.BUTTERFLY,
           "three": fb.Engine.THREE_PASS}[cfg["engine"]]
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    # synthetic data (random-init kernels, geometric decay like init_kernels)
    u = torch.randn(B, H, N, device=dev, generator=g).to(dt)
    dy = torch.randn(B, H, N, device=dev, generator=g).to(dt)
    pos = torch.arange(N, device=dev, dtype=torch.float32) / N
    decay = (H / 2.0) ** (torch.arange(H, device=dev, dtype=torch.float32) / H)
    K = torch.randn(H, N, device=dev, generator=g) * torch.exp(-pos[None, :] * decay[:, None])
    D = torch.randn(H, device=dev, generator=g)
    rc = fb.RegularizationConfig(lambda_=LAM, smooth_width=P)
    plan = fb.LongConvPlan(N, H, fb.ConvMode.CAUSAL, dt, eng, dev)
    ws = plan.workspace(B)
    y = torch.empty_like(u)
    du = torch.empty_like(u)
    dK = torch.empty(H, N, device=dev)
    dD = torch.empty(H, device=dev)
    L = _lib.lib()
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    import ctypes as C

    c = rc.to_c()
    P_ = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    h = plan._h
    n_events = []

    # training step: the forward keeps its transform of u for the backward
    # (tensor-core plans; fb_saved_size is 0 otherwise and the calls recompute)
    nsaved = plan.saved_size(B)
    saved = torch.empty(max(nsaved, 1), dtype=torch.uint8, device=dev)
    Ps = P_(saved) if nsaved else C.c_void_p(0)

    def step(rec=None):
        _lib.check(L.fb_kernel_prep(h, P_(K), P_(D), C.byref(c), 0, C.c_void_p(sp)))
        if rec is not None:
            rec[0].record(stream)
        _lib.check(L.fb_fwd_save(h, P_(u), P_(y), Ps, B, P_(ws), C.c_void_p(sp)))
        if rec is not None:
            rec[1].record(stream)
        _lib.check(L.fb_bwd_saved(h, P_(dy), P_(u), Ps, P_(du), P_(dK), C.c_void_p(0), P_(dD), B,
                                  P_(ws), C.c_void_p(sp)))
        if rec is not None:
            rec[2].record(stream)

    recs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # the sampler runs from warm-up through the timed region (nvidia-smi polls
    # every ~50 ms; a short timed region alone would see one sample)
    with ClockSampler(local_rank) as clk:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        clk.mark()
        t0.record(stream)
        for i in range(args.steps):
            step(recs[i])
        t1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = t0.elapsed_time(t1)
    fwd_ms = sum(r[0].elapsed_time(r[1]) for r in recs) / args.steps
    bwd_ms = sum(r[1].elapsed_time(r[2]) for r in recs) / args.steps
    tmax = torch.tensor([ms], device=dev)
    if dist:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms = float(tmax.item())
    ms_step = ms / args.steps
    E = B * H * N
    value = E * world / (ms_step / 1e3)

    # ---------------- e2e: public API with host buffers, copies timed -------
    # fb_host_runner: heads in chunks, H2D / kernels / D2H overlapped on three
    # streams (the call a user with host arrays makes)
    hu = u.cpu().pin_memory()
    hdy = dy.cpu().pin_memory()
    hK = K.cpu().pin_memory()
    hD = D.cpu().pin_memory()
    hy = torch.empty_like(hu).pin_memory()
    hdu = torch.empty_like(hu).pin_memory()
    hdK = torch.empty_like(hK).pin_memory()
    hdD = torch.empty_like(hD).pin_memory()
    runner = fb.HostRunner(N, H, B, dt, engine=eng, heads_per_chunk=max(1, H // 8), device=dev)

    def e2e_step():
        runner.run(hu, hdy, hK, hD, rc, out=(hy, hdu, hdK, hdD))

    for _ in range(max(1, args.warmup)):
        e2e_step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_steps = max(1, min(args.steps, 10))
    if dist:
        dist.barrier()
    e0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    ems = torch.tensor([e0.elapsed_time(e1) / e2e_steps], device=dev)
    if dist:
        dist.all_reduce(ems, op=dist.ReduceOp.MAX)
    e2e_val = E * world / (float(ems.item()) / 1e3)
    h2d = (hu.numel() + hdy.numel()) * s + (hK.numel() + hD.numel()) * 4
    d2h = (hy.numel() + hdu.numel()) * s + (hdK.numel() + hdD.numel()) * 4

    if dist:
        dist.barrier()
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return None

    hbm_peak, tc_peak, peak_kind = load_peaks()
    # dominant kernel: the backward (K4a sp_bwd / K4b passes)
    HN = H * N
    # algorithmic bytes per launch: single-pass reads/writes each
    # signal once plus k_f (8 B per bin, n = 2N bins per head); three-pass adds
    # the complex intermediates (2s bytes per real element each, 2N-padded)
    if plan.engine == fb.Engine.THREE_PASS:
        bwd_bytes = 16 * s * E + 52 * HN
        fwd_bytes = 11 * s * E + 16 * HN
    else:
        bwd_bytes = 3 * s * E + 16 * HN
        fwd_bytes = 2 * s * E + 16 * HN
    dom = "bwd" if bwd_ms >= fwd_ms else "fwd"
    dom_bytes, dom_ms = (bwd_bytes, bwd_ms) if dom == "bwd" else (fwd_bytes, fwd_ms)
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    step_bytes = alg_bytes(cfg, s)
    prof = ROOT / "profiles" / "traffic.json"
    traffic = None
    if prof.exists():
        traffic = json.loads(prof.read_text()).get(f"config{args.config}", {}).get(dom)
    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, args.cpu_sample_heads)
    # our kernel launches per timed step (prep + fwd + bwd, training-step path):
    # single-pass: K1 spectrum, forward, backward, backward tail;
    # three-pass: regularize, kernel columns, kernel rows | pass 1, rows, pass 3 |
    # pass 1 (dy), rows, pass 3 (du), dK rows, dD, regularizer chain rule
    launches_per_step = 12 if plan.engine == fb.Engine.THREE_PASS else 4
    out = {
        "metric": "long-conv fwd+bwd elements/sec (E=B*H*N per step: K1 prep + fwd + bwd)",
        "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": cfg["dtype"],
        "data": "synthetic (torch.randn signals, random geometric-decay kernels)",
        "config": {"workload": cfg["workload"], "B": B, "H": H, "N": N,
                   "engine": plan.engine.name.lower(), "transform_len": plan.n,
                   "lambda": LAM, "smooth_width": P, "mode": "causal",
                   "sharding": f"heads, {H} per GPU, no communication",
                   "saved_activation": ("bwd reuses the fwd transform of u "
                                        f"({nsaved / 2**20:.0f} MiB, bf16)" if nsaved else None),
                   "l2": "inputs larger than L2 (u, dy, y, du = "
                         f"{4 * E * s / 2**20:.0f} MiB per GPU)"},
        "fwd_ms": fwd_ms, "bwd_ms": bwd_ms,
        "roofline": {"bound": "hbm",
                     "kernel": (f"{dom}: tc_{dom}_kernel (tcgen05)" if plan.tensor_cores else
                                f"{dom}: sp_{dom}_kernel" if plan.engine.name != "THREE_PASS" else
                                f"{dom}: three-pass launches (pass 1 cols, pass 2 rows on "
                                "tcgen05, pass 3 cols)"),
                     "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic,
                     "alg_bytes_per_launch": dom_bytes, "peak_kind": peak_kind},
        "step_roofline": {"alg_bytes": step_bytes,
                          "achieved_GBs": step_bytes / (ms_step / 1e3) / 1e9,
                          "frac": step_bytes / (ms_step / 1e3) / 1e9 / hbm_peak},
        "e2e": {"value": e2e_val, "unit": "elements/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": float(ems.item())},
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "gpu_launches": launches_per_step * args.steps,
    }
    print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()
    return out


def run_learned(args, cfg, rank, world, local_rank):
    """Config 4: learned butterfly fwd + bwd (block + input gradients) over
    B*H rows of n complex, bf16 rows, per-head fp32 complex blocks."""
    import torch

    import paper_2302_06646_b200 as fb

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    B, H, n, r = cfg["B"], cfg["H"], cfg["N"], cfg["r"]
    dt = torch.bfloat16
    plan = fb.LearnedButterflyPlan(n, r, H, dt, dev)
    g = torch.Generator(device=dev)
    g.manual_seed(99 + rank)
    blocks = plan.dft_blocks() + 0.1 * torch.randn(H, plan.param_count, dtype=torch.complex64,
                                                   device=dev, generator=g)
    x = torch.randn(B, H, n, 2, device=dev, generator=g).to(dt)
    up = torch.randn(B, H, n, 2, device=dev, generator=g).to(dt)
    stream = torch.cuda.current_stream()
    recs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def step(rec=None):
        if rec:
            rec[0].record(stream)
        plan.forward(blocks, x)
        if rec:
            rec[1].record(stream)
        plan.gradients(blocks, x, up)
        if rec:
            rec[2].record(stream)

    with ClockSampler(local_rank) as clk:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        clk.mark()
        t0.record(stream)
        for i in range(args.steps):
            step(recs[i])
        t1.record(stream)
        torch.cuda.synchronize()
    tmax = torch.tensor([t0.elapsed_time(t1)], device=dev)
    if dist:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms_step = float(tmax.item()) / args.steps
    fwd_ms = sum(q[0].elapsed_time(q[1]) for q in recs) / args.steps
    bwd_ms = sum(q[1].elapsed_time(q[2]) for q in recs) / args.steps
    E = B * H * n
    value = E * world / (ms_step / 1e3)
    # e2e: host rows in, host results out
    hx, hu = x.cpu().pin_memory(), up.cpu().pin_memory()
    hy = torch.empty_like(hx).pin_memory()
    hdx = torch.empty_like(hx).pin_memory()
    hdb = torch.empty(H, plan.param_count, dtype=torch.complex64).pin_memory()
    xx, uu = torch.empty_like(x), torch.empty_like(up)

    def e2e():
        xx.copy_(hx, non_blocking=True)
        uu.copy_(hu, non_blocking=True)
        yy = plan.forward(blocks, xx)
        db, dx = plan.gradients(blocks, xx, uu)
        hy.copy_(yy, non_blocking=True)
        hdx.copy_(dx, non_blocking=True)
        hdb.copy_(db, non_blocking=True)

    e2e()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = max(1, min(args.steps, 10))
    e0.record(stream)
    for _ in range(k):
        e2e()
    e1.record(stream)
    torch.cuda.synchronize()
    ems = e0.elapsed_time(e1) / k
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return None
    hbm_peak, _, peak_kind = load_peaks()
    bytes_step = 20 * E  # bf16 complex rows: fwd x,y; bwd x,g,dx
    out = {
        "metric": "learned-butterfly fwd+bwd rows*n elements/sec (incl. block gradients)",
        "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (randn rows, DFT-initialised blocks + 0.1 randn)",
        "config": {"workload": cfg["workload"], "B": B, "H": H, "n": n, "r": r,
                   "factors": plan.factors, "params_per_head": plan.param_count,
                   "l2": "rows 100 MiB per tensor"},
        "fwd_ms": fwd_ms, "bwd_ms": bwd_ms,
        "roofline": {"bound": "hbm", "kernel": "bwd: lx_bwd_kernel + lb_reduce_kernel",
                     "achieved": 12 * E / (bwd_ms / 1e3) / 1e9,
                     "peak": hbm_peak, "unit": "GB/s",
                     "frac": 12 * E / (bwd_ms / 1e3) / 1e9 / hbm_peak,
                     "traffic": _traffic(4, "bwd"),
                     "alg_bytes_per_launch": 12 * E, "peak_kind": peak_kind},
        "step_roofline": {"alg_bytes": bytes_step,
                          "achieved_GBs": bytes_step / (ms_step / 1e3) / 1e9,
                          "frac": bytes_step / (ms_step / 1e3) / 1e9 / hbm_peak},
        "e2e": {"value": E * world / (ems / 1e3), "unit": "elements/s",
                "h2d_bytes_per_step": 2 * E * 4, "d2h_bytes_per_step": 2 * E * 4 + H * plan.param_count * 8,
                "ms_per_step": ems},
        "cpu_baseline": None if args.no_cpu_baseline else cpu_baseline(cfg, args.cpu_sample_heads),
        "clocks": clk.summary(),
        "gpu_launches": 3 * args.steps,  # forward, backward, block-gradient reduction
    }
    print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()
    return out


def reference_cpu_run(cfg, heads, steps=1, threads=None):
    """Reference CPU path (oracle/_ref = unmodified reference sources):
    regularized_long_conv(kButterfly, kCausal, threads=nproc) + the backward
    composed from conv_butterfly.  Returns (elements, seconds)."""
    import numpy as np

    from oracle.oracle import RefOracle, ref_available

    if not ref_available():
        raise RuntimeError("oracle/_ref/liblongconv_ref.so missing")
    ref = RefOracle(threads)
    B, N = cfg["B"], cfg["N"]
    rng = np.random.default_rng(0)
    if cfg["engine"] == "learned":
        # learned_forward + learned_gradients (butterfly.cpp:235-307) per row
        r = cfg["r"]
        base = ref.learned_init(N, r)
        blocks = base + 0.1 * (rng.standard_normal(base.size) + 1j * rng.standard_normal(base.size))
        x = rng.standard_normal((B, heads, N)) + 1j * rng.standard_normal((B, heads, N))
        g = rng.standard_normal((B, heads, N)) + 1j * rng.standard_normal((B, heads, N))
        t0 = time.perf_counter()
        for _ in range(steps):
            for b in range(B):
                for h in range(heads):
                    ref.learned_forward(blocks, x[b, h], r)
                    ref.learned_gradients(blocks, x[b, h], g[b, h], r)
        return B * heads * N * steps, time.perf_counter() - t0
    u = rng.standard_normal((B, heads, N))
    dy = rng.standard_normal((B, heads, N))
    K, D = ref.init_kernels(1, heads, N, 3)
    engine = 2 if cfg["engine"] == "three" else 1
    t0 = time.perf_counter()
    for _ in range(steps):
        Kbar = ref.regularize_bank(K, LAM, P)
        ref.regularized_long_conv(u, K, D, LAM, P, engine=engine)
        _, dKbar, _ = ref.long_conv_backward(u, dy, Kbar, D)
        ref.regularizer_backward(K, LAM, P, dKbar)
    return B * heads * N * steps, time.perf_counter() - t0


def cpu_baseline(cfg, heads):
    heads = min(cfg["H"], heads)
    threads = os.cpu_count() or 1
    try:
        el, sec = reference_cpu_run(cfg, heads, 1, threads)
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "elements/s", "error": str(e)}
    if cfg["engine"] == "learned":
        threads = 1  # learned_forward / learned_gradients are single-threaded per row
    return {"value": el / sec, "unit": "elements/s", "cores": threads, "kind": "reference",
            "sample": f"B={cfg['B']} H={heads} (of {cfg['H']}) N={cfg['N']}, fp64, "
                      f"{sec:.1f}s: regularize_bank + regularized_long_conv(kButterfly) + "
                      "composed conv_butterfly backward; channels independent so the rate "
                      "extrapolates linearly",
            "host": platform.processor() or platform.machine()}


def run_reference(args, cfg, rank):
    if rank != 0:
        return
    heads = min(cfg["H"], args.cpu_sample_heads)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup if args.warmup < 1 else 1):
        reference_cpu_run(cfg, max(1, heads // 8), 1, threads)
    el, sec = reference_cpu_run(cfg, heads, args.steps, threads)
    val = el / sec
    out = {
        "impl": "reference",
        "metric": "long-conv fwd+bwd elements/sec (E=B*H*N per step: K1 prep + fwd + bwd)",
        "value": val, "unit": "elements/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sec / args.steps * 1e3 * cfg["H"] / heads,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": cfg["workload"], "B": cfg["B"], "H": cfg["H"],
                                        "N": cfg["N"]},
        "cpu_baseline": {"value": val, "unit": "elements/s", "cores": threads,
                         "kind": "reference",
                         "sample": f"each step B={cfg['B']} H={heads} of {cfg['H']} heads"},
        "e2e": {"value": val, "unit": "elements/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def run_seqshard(args, cfg, rank, world, local_rank):
    """Config 5-4M: the layer forward + backward with the sequence sharded over
    the ranks (seqshard.sharded_long_conv / _backward: our column and row
    kernels, NCCL all_to_all_single transposes).  Weak in nothing: the whole
    job is one sequence batch; value = B*H*N / max-over-ranks step time."""
    import torch

    from paper_2302_06646_b200 import seqshard as ss

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    B, H, N = cfg["B"], cfg["H"], cfg["N"]
    if args.bh:
        H = max(1, args.bh // B)
    n, l = 2 * N, 8192
    m = n // l
    sh = ss.SeqShard(l=l, m=m, world=world, rank=rank)
    g = torch.Generator(device=dev)
    g.manual_seed(77 + rank)
    half = m // 2
    u = torch.randn(B, H, half, sh.lp, device=dev, generator=g)
    dy = torch.randn(B, H, half, sh.lp, device=dev, generator=g)
    t = (torch.arange(half, device=dev)[:, None] * l + sh.tau0 +
         torch.arange(sh.lp, device=dev)[None, :]).float()
    kbar = torch.randn(H, half, sh.lp, device=dev, generator=g) * torch.exp(-t / 2e5)[None]
    D = torch.randn(H, device=dev, generator=g)
    passes = ss.GpuPasses(n, device=dev)

    def step():
        y = ss.sharded_long_conv(u, kbar, D, sh, passes)
        du, dk, dD = ss.sharded_long_conv_backward(dy, u, kbar, D, sh, passes)
        return y, du, dk, dD

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    tmax = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
    if dist:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms = float(tmax.item())
    E = B * H * N
    if rank == 0:
        print(json.dumps({
            "metric": "long-conv fwd+bwd elements/sec (E=B*H*N per step)", "value": E / (ms / 1e3),
            "unit": "elements/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (randn signals, decaying random Kbar)",
            "config": {"workload": cfg["workload"], "B": B, "H": H, "N": N, "transform_len": n,
                       "l": l, "m": m, "sharding": f"sequence over {world} rank(s), tau-slices of "
                       f"{sh.lp} columns; 4 all-to-alls fwd, 6 bwd",
                       "bh_reduced": bool(args.bh), "report_only": True},
            "roofline": None, "cpu_baseline": None, "clocks": clk.summary(),
            "gpu_launches": None, "e2e": None}))
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-heads", type=int, default=32)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--n", type=int, default=None, help="sequence length (config 5 sweep)")
    ap.add_argument("--bh", type=int, default=None, help="B*H override (config 6, few GPUs)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    cfg = dict(CONFIGS[args.config])
    if args.n is not None:
        cfg["N"] = args.n
        cfg["workload"] = cfg["workload"] + f", N={args.n}"
    if args.config == 4 and args.impl == "ours":
        run_learned(args, cfg, rank, world, local_rank)
        return
    if args.config == 6 and args.impl == "ours":
        run_seqshard(args, cfg, rank, world, local_rank)
        return
    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return
    if world != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    run_ours(args, cfg, rank, world, local_rank)


if __name__ == "__main__":
    main()
