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
    2: dict(B=32, H=256, N=4096, dtype="bf16", engine="single", e2e_chunks=4,
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


def alg_bytes(B, H, N, s, three_pass):
    """Algorithmic HBM bytes per step, for the engine the plan
    resolved to: single-pass 5sE + 32HN, three-pass 25sE + 48HN."""
    E, HN = B * H * N, H * N
    return 25 * s * E + 48 * HN if three_pass else 5 * s * E + 32 * HN


def kernel_alg_bytes(B, H, N, s, three_pass):
    """Algorithmic bytes of one launch of the forward's / backward's main
    kernel: single-pass fwd reads u, writes y, reads k_f
    (2sE + 16HN), bwd reads dy and u, writes du, reads k_f (3sE + 16HN);
    three-pass rows kernels move the complex intermediate (2s bytes per real
    element per sweep): fwd reads X1, writes W, reads the Kf2 rows
    (4sE + 16HN); bwd reads dy's rows and U, writes du's rows, reads Kf2,
    writes the dK rows (6sE + 32HN)."""
    E, HN = B * H * N, H * N
    if three_pass:
        return 4 * s * E + 16 * HN, 6 * s * E + 32 * HN
    return 2 * s * E + 16 * HN, 3 * s * E + 16 * HN


def _timed_layer(args, fb, _lib, cfg, dev, Hloc, head0, clk=None):
    """Build one plan for Hloc heads (global heads head0 ..) and time
    args.steps training steps (K1 prep + fwd + bwd) after args.warmup
    warm-up steps.  Returns a dict of timings and the plan / tensors."""
    import ctypes as C

    import torch

    dt = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}[cfg["dtype"]]
    B, N, H = cfg["B"], cfg["N"], Hloc
    eng = {"auto": fb.Engine.AUTO, "single": fb.Engine.BUTTERFLY,
           "three": fb.Engine.THREE_PASS}[cfg["engine"]]
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + head0)
    # synthetic data (random-init kernels, geometric decay like init_kernels)
    u = torch.randn(B, H, N, device=dev, generator=g).to(dt)
    dy = torch.randn(B, H, N, device=dev, generator=g).to(dt)
    pos = torch.arange(N, device=dev, dtype=torch.float32) / N
    hh = torch.arange(head0, head0 + H, device=dev, dtype=torch.float32)
    decay = (cfg["H"] / 2.0) ** (hh / cfg["H"])
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
    c = rc.to_c()
    P_ = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    h = plan._h
    # training step: the forward keeps its transform of u for the backward
    nsaved = plan.saved_size(B)
    saved = torch.empty(max(nsaved, 1), dtype=torch.uint8, device=dev)
    Ps = P_(saved) if nsaved else C.c_void_p(0)

    def step(rec=None, kev=None):
        _lib.check(L.fb_kernel_prep(h, P_(K), P_(D), C.byref(c), 0, C.c_void_p(sp)))
        if rec is not None:
            rec[0].record(stream)
            # the main kernels alone, bracketed on their launching stream
            _lib.check(L.fb_plan_profile_events(h, 0, kev[0], kev[1]))
            _lib.check(L.fb_plan_profile_events(h, 1, kev[2], kev[3]))
        _lib.check(L.fb_fwd_save(h, P_(u), P_(y), Ps, B, P_(ws), C.c_void_p(sp)))
        if rec is not None:
            rec[1].record(stream)
        _lib.check(L.fb_bwd_saved(h, P_(dy), P_(u), Ps, P_(du), P_(dK), C.c_void_p(0), P_(dD), B,
                                  P_(ws), C.c_void_p(sp)))
        if rec is not None:
            rec[2].record(stream)

    Ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    recs = [[Ev() for _ in range(3)] for _ in range(args.steps)]
    kevs = [[Ev() for _ in range(4)] for _ in range(args.steps)]
    for kv in kevs:  # materialise the cudaEvent_t handles
        for e in kv:
            e.record(stream)
    torch.cuda.synchronize()
    kptr = [[C.c_void_p(e.cuda_event) for e in kv] for kv in kevs]
    t0, t1 = Ev(), Ev()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if torch.distributed.is_initialized():
        torch.distributed.barrier()
    torch.cuda.synchronize()
    if clk is not None:
        clk.mark()
    t0.record(stream)
    for i in range(args.steps):
        step(recs[i], kptr[i])
    t1.record(stream)
    torch.cuda.synchronize()
    K_ = args.steps
    return dict(
        ms=t0.elapsed_time(t1), plan=plan, dt=dt, eng=eng, nsaved=nsaved, tensors=(u, dy, K, D),
        fwd_ms=sum(r[0].elapsed_time(r[1]) for r in recs) / K_,
        bwd_ms=sum(r[1].elapsed_time(r[2]) for r in recs) / K_,
        kfwd_ms=sum(k[0].elapsed_time(k[1]) for k in kevs) / K_,
        kbwd_ms=sum(k[2].elapsed_time(k[3]) for k in kevs) / K_)


def run_ours(args, cfg, rank, world, local_rank):
    import torch

    import paper_2302_06646_b200 as fb
    from paper_2302_06646_b200 import _lib
    from paper_2302_06646_b200.seqshard import head_shard

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    B, H, N = cfg["B"], cfg["H"], cfg["N"]
    # strong scaling (default): each rank owns head_shard(H, world, rank) of
    # the configured job, no communication; weak scaling: every rank runs the
    # full per-GPU job (second field when world > 1)
    strong = args.scaling == "strong"
    hs = head_shard(H, world, rank) if strong else slice(0, H)
    Hloc = hs.stop - hs.start

    def tmax(x):
        t = torch.tensor([x], device=dev)
        if dist:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    with ClockSampler(local_rank) as clk:
        r = _timed_layer(args, fb, _lib, cfg, dev, Hloc, hs.start, clk)
    if dist:
        dist.barrier()
    ms_step = tmax(r["ms"]) / args.steps
    E_job = B * H * N if strong else B * H * N * world
    value = E_job / (ms_step / 1e3)
    other = None
    if world > 1:  # the other scaling mode, same timing rules
        r2 = _timed_layer(args, fb, _lib, cfg, dev, H if strong else H // world,
                          0 if strong else head_shard(H, world, rank).start)
        ms2 = tmax(r2["ms"]) / args.steps
        E2 = B * H * N * world if strong else B * H * N
        other = {"scaling": "weak" if strong else "strong", "value": E2 / (ms2 / 1e3),
                 "ms_per_step": ms2, "heads_per_gpu": H if strong else H // world}
        del r2
    plan, dt = r["plan"], r["dt"]
    s = torch.tensor([], dtype=dt).element_size()
    u, dy, K, D = r["tensors"]
    three = plan.engine == fb.Engine.THREE_PASS

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
    rc = fb.RegularizationConfig(lambda_=LAM, smooth_width=P)
    # head chunks of the host runner (copies of one chunk overlap the kernels
    # of the previous one; measured: 4 for config 2, 8 for config 3)
    runner = fb.HostRunner(N, Hloc, B, dt, engine=r["eng"], heads_per_chunk=max(1, Hloc // cfg.get("e2e_chunks", 8)),
                           device=dev)
    stream = torch.cuda.current_stream()

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
    ems = tmax(e0.elapsed_time(e1) / e2e_steps)
    e2e_val = E_job / (ems / 1e3)
    h2d = (hu.numel() + hdy.numel()) * s + (hK.numel() + hD.numel()) * 4
    d2h = (hy.numel() + hdu.numel()) * s + (hdK.numel() + hdD.numel()) * 4

    if dist:
        dist.barrier()
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return None

    hbm_peak, tc_peak, peak_kind = load_peaks()
    # dominant kernel: the larger of the forward's / backward's main kernel,
    # each timed alone by events the plan records around its launch
    kb_fwd, kb_bwd = kernel_alg_bytes(B, Hloc, N, s, three)
    if r["kbwd_ms"] >= r["kfwd_ms"]:
        dom, dom_bytes, dom_ms = "bwd", kb_bwd, r["kbwd_ms"]
    else:
        dom, dom_bytes, dom_ms = "fwd", kb_fwd, r["kfwd_ms"]
    kname = {(False, True): f"tc_{dom}_kernel (tcgen05)", (False, False): f"sp_{dom}_kernel",
             (True, True): f"tc_rows_{dom}_kernel (tcgen05)",
             (True, False): "tp_pass2" + ("_bwd" if dom == "bwd" else "") + "_kernel"}
    rows_tc = three and dt in (torch.bfloat16, torch.float16)
    kern = kname[(three, plan.tensor_cores or rows_tc)]
    if not three and plan.tensor_cores and N <= 1024:  # the radix-16 short single pass
        kern = f"sc_{dom}_kernel (tcgen05, radix-16 stages)"
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    step_bytes = alg_bytes(B, Hloc, N, s, three)
    traffic = _traffic(args.config if cfg["dtype"] == CONFIGS[args.config]["dtype"] else -1, dom)
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline(cfg, args.cpu_sample_heads)
    # our kernel launches per timed step (prep + fwd + bwd, training-step path):
    # single-pass: K1 spectrum, forward, backward, backward tail;
    # three-pass: regularize, kernel columns, kernel rows | pass 1, rows, pass 3 |
    # pass 1 (dy), rows, pass 3 (du), dK rows, dD, regularizer chain rule
    launches_per_step = 12 if three else 4
    out = {
        "metric": "long-conv fwd+bwd elements/sec (E=B*H*N per step: K1 prep + fwd + bwd)",
        "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": cfg["dtype"],
        "data": "synthetic (torch.randn signals, random geometric-decay kernels)",
        "config": {"workload": cfg["workload"], "B": B, "H": H, "N": N,
                   "engine": plan.engine.name.lower(), "transform_len": plan.n,
                   "lambda": LAM, "smooth_width": P, "mode": "causal",
                   "sharding": (f"heads: head_shard(H={H}, {world}, rank) = {Hloc} per GPU, "
                                "no communication"),
                   "saved_activation": (f"bwd reuses the fwd transform of u "
                                        f"({r['nsaved'] / 2**20:.0f} MiB)" if r["nsaved"] else None),
                   "l2": "inputs larger than L2 (u, dy, y, du = "
                         f"{4 * B * Hloc * N * s / 2**20:.0f} MiB per GPU)"},
        "fwd_ms": r["fwd_ms"], "bwd_ms": r["bwd_ms"],
        "main_kernel_ms": {"fwd": r["kfwd_ms"], "bwd": r["kbwd_ms"]},
        "roofline": {"bound": "hbm", "kernel": f"{dom}: {kern}",
                     "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic,
                     "traffic_over_alg": (traffic / dom_bytes) if traffic else None,
                     "alg_bytes_per_launch": dom_bytes, "launch_ms": dom_ms,
                     "peak_kind": peak_kind},
        "step_roofline": {"alg_bytes": step_bytes,
                          "formula": "25sE+48HN (three-pass)" if three else "5sE+32HN (single-pass)",
                          "achieved_GBs": step_bytes / (ms_step / 1e3) / 1e9,
                          "frac": step_bytes / (ms_step / 1e3) / 1e9 / hbm_peak},
        "e2e": {"value": e2e_val, "unit": "elements/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": ems},
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "gpu_launches": launches_per_step * args.steps,
    }
    if other:
        out["other_scaling"] = other
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
                   "factors": plan.factors, "params_per_head": plan.param_count, "engine": plan.engine,
                   "l2": "rows 100 MiB per tensor"},
        "fwd_ms": fwd_ms, "bwd_ms": bwd_ms,
        "roofline": {"bound": "hbm", "kernel": ("bwd: lt_bwd_kernel (tcgen05) + lb_reduce_kernel"
                                                if plan.engine == "tcgen05" else
                                                "bwd: lx_bwd_kernel + lb_reduce_kernel"),
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
    """Reference CPU path (oracle/_ref = unmodified reference sources), one
    step per call: regularize_bank once (regularize.cpp:93-107), the forward
    regularized_long_conv(kButterfly, kCausal, threads) on that regularized
    bank with the identity regularizer (lambda = 0, p = 0: no second
    smooth/squash pass), the backward composed from conv_butterfly
     and the regularizer chain rule.  Returns (elements,
    seconds) over `steps` steps of B x heads x N."""
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
        ref.regularized_long_conv(u, Kbar, D, 0.0, 0, engine=engine)
        _, dKbar, _ = ref.long_conv_backward(u, dy, Kbar, D)
        ref.regularizer_backward(K, LAM, P, dKbar)
    return B * heads * N * steps, time.perf_counter() - t0


def cpu_baseline(cfg, heads):
    """One reference step on the host cores: the whole configured workload
    when it is a few seconds of CPU work (configs 1, 2, 4), else `heads`
    heads of it (configs with N >= 64K; channels are independent)."""
    full = cfg["B"] * cfg["H"] * cfg["N"] <= 64 * 2**20
    heads = cfg["H"] if full else min(cfg["H"], heads)
    threads = os.cpu_count() or 1
    try:
        el, sec = reference_cpu_run(cfg, heads, 1, threads)
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "elements/s", "error": str(e)}
    if cfg["engine"] == "learned":
        threads = 1  # learned_forward / learned_gradients are single-threaded per row
    return {"value": el / sec, "unit": "elements/s", "cores": threads, "kind": "reference",
            "sample": f"B={cfg['B']} H={heads} (of {cfg['H']}) N={cfg['N']}, fp64, one step "
                      f"in {sec:.1f}s: "
                      + ("learned_forward + learned_gradients per row" if cfg["engine"] == "learned"
                         else "regularize_bank + regularized_long_conv(kButterfly) + "
                              "composed conv_butterfly backward + regularizer chain rule")
                      + ("" if heads == cfg["H"] else "; a head sample (channels independent)"),
            "host": platform.processor() or platform.machine()}


def run_reference(args, cfg, rank):
    """--impl reference: the reference's CPU implementation, rank 0 only, all
    host threads; every step is the WHOLE configured workload (no head
    sampling or extrapolation) for configs of up to 64M elements (config 2:
    ~2.5 s per step on 16 cores), a head sample above that."""
    if rank != 0:
        return
    full = cfg["B"] * cfg["H"] * cfg["N"] <= 64 * 2**20
    heads = cfg["H"] if full else min(cfg["H"], args.cpu_sample_heads)
    threads = os.cpu_count() or 1
    if args.warmup > 0:  # one warm-up step (page-in, thread spawn); the rest are timed
        reference_cpu_run(cfg, heads, 1, threads)
    el, sec = reference_cpu_run(cfg, heads, args.steps, threads)
    val = el / sec
    out = {
        "impl": "reference",
        "metric": ("learned-butterfly fwd+bwd rows*n elements/sec (incl. block gradients)"
                   if cfg["engine"] == "learned" else
                   "long-conv fwd+bwd elements/sec (E=B*H*N per step: K1 prep + fwd + bwd)"),
        "value": val, "unit": "elements/s", "n_gpus": 1, "steps": args.steps,
        "warmup": min(args.warmup, 1), "ms_per_step": sec / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": cfg["workload"], "B": cfg["B"], "H": cfg["H"],
                                        "N": cfg["N"], "heads_timed": heads},
        "cpu_baseline": {"value": val, "unit": "elements/s", "cores": threads,
                         "kind": "reference",
                         "sample": (f"each step the full B={cfg['B']} H={cfg['H']} N={cfg['N']} "
                                    "workload" if heads == cfg["H"] else
                                    f"each step B={cfg['B']} H={heads} of {cfg['H']} heads")},
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

    wire, chunks = args.wire, args.chunks

    def step():
        y = ss.sharded_long_conv(u, kbar, D, sh, passes, wire=wire, chunks=chunks)
        du, dk, dD = ss.sharded_long_conv_backward(dy, u, kbar, D, sh, passes, wire=wire)
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
                       "all_to_all_wire": wire, "fwd_channel_chunks": chunks,
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
    ap.add_argument("--wire", default="f32", choices=["f32", "bf16"],
                    help="config 6: all-to-all payload type")
    ap.add_argument("--chunks", type=int, default=1,
                    help="config 6: channel-pair chunks of the pipelined forward exchange")
    ap.add_argument("--bh", type=int, default=None, help="B*H override (config 6, few GPUs)")
    ap.add_argument("--dtype", default=None, choices=["f32", "bf16", "f16"],
                    help="I/O dtype override (e.g. the fp32 validation line of config 2)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N>1: strong = head_shard(H) per rank (default), weak = full job per rank")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    cfg = dict(CONFIGS[args.config])
    if args.n is not None:
        cfg["N"] = args.n
        cfg["workload"] = cfg["workload"] + f", N={args.n}"
    if args.dtype is not None and args.dtype != cfg["dtype"]:
        cfg["dtype"] = args.dtype
        cfg["workload"] = cfg["workload"] + f", {args.dtype} I/O"
        if cfg["engine"] == "single" and args.dtype == "f32":
            cfg["engine"] = "auto"  # fp32 validation mode: the CUDA-core single pass
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
