#!/usr/bin/env python
"""Benchmark of the hot path: GMRES iterations/s of the MgNet-preconditioned restarted GMRES
solve (rte_apply + MgNet V-cycle + CGS2 Arnoldi + Givens per iteration) on one config of
BASELINE.json (default: config 5, 512^2 cells x M=256 ordinates, MgNet L=6 C0=32, GMRES(30)).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config k] [--impl ours|reference]

A "step" is one whole GMRES(30) restart cycle: 30 inner iterations (V-cycle + apply + Arnoldi +
Givens each) and the cycle end (back-solve, x += P(V y), the fp64 restart residual), DESIGN.md §7.
Whole cycles, because an Arnoldi step's cost grows with j: a partial cycle would time only the
cheap early steps.  The timed region is ONE gmres_solve call of exactly K cycles (30 K inner
iterations) from x0 = 0, bracketed by a barrier and torch.cuda.synchronize() on both sides and
timed with CUDA events on the launching stream; the reported time is the max over ranks, and
value = inner iterations / s.  Config-5 vectors are 256 MiB (> 126 MB L2), so every step
streams its inputs from HBM ("inputs larger than L2").  Multi-GPU: config 5 is ONE medium and does
not shard without a halo exchange, so N ranks run N independent replicas (DESIGN.md §8,
"replicas only"); value = total iterations of all ranks / max-over-ranks time ("scaling": "weak").
Batched configs (config 4) shard their independent samples across ranks, no data-path collective:
value = K iterations of the whole batch / max-over-ranks time ("scaling": "strong").

Rank 0 prints ONE JSON line.  --impl reference times the fp64 CPU oracle (oracle/, the
reference arm of this tier) on the host cores for the same metric and config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import benchlib  # noqa: E402

METRIC = "GMRES iter/s (rte_apply + MgNet V-cycle) at N²×M; % of roofline"
UNIT = "GMRES iter/s"
TF32_PER_BF16 = 1.1 / 2.25      # guide's nominal dense ratio (B200_PROFILING.md table)
N_SM = 148


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


def _workload_name(cfg):
    return (f"cfg{cfg.k}: {cfg.B}x{cfg.N}^2 cells x M={cfg.M} ordinates "
            f"({cfg.B * cfg.N * cfg.N * cfg.M / 1e6:.1f}M unknowns), MgNet L={cfg.L} C0={cfg.C0} nu={cfg.nu}, "
            f"GMRES({cfg.restart}) fixed budget")


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws <= 1:
        return None, 0, 1, 0
    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    backend = "nccl" if torch.cuda.is_available() else "gloo"
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    dist.init_process_group(backend=backend)
    return dist, rank, ws, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (B200_PROFILING.md)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev_index):
        self.proc = None
        self.dev = dev_index

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


def _device_index(torch, local):
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = [v.strip() for v in vis.split(",") if v.strip()]
        if local < len(ids):
            return ids[local]
    return local


def _tensor_peaks(peaks):
    """3xTF32 algorithmic-fp32 peaks (TFLOP/s): measured bf16 x the guide's nominal tf32/bf16 ratio /
    3 MMAs per product; burst (a kernel timed alone / at full clocks) and sustained (power-capped)."""
    burst = peaks.get("bf16_tflops", 1590.0) * TF32_PER_BF16 / 3.0
    sus = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1400.0)) * TF32_PER_BF16 / 3.0
    return burst, sus


def _class_roofline_ms(c, peaks, tensor_peak):
    """Roofline time of one class's launches: max(algorithmic bytes / HBM, flops / its compute peak)."""
    smax = peaks.get("sm_max_mhz", 1965.0)
    t_hbm = c["bytes"] / (peaks["hbm_gbs"] * 1e9) * 1e3
    kind = c["kind"]
    if kind == "tensor_3xtf32":
        t_c = c["flops"] / (tensor_peak * 1e12) * 1e3
    elif kind == "fp32_simt":
        t_c = c["flops"] / (N_SM * 128 * 2 * smax * 1e6) * 1e3
    elif kind == "fp64_simt":
        t_c = c["flops"] / (N_SM * 64 * 2 * smax * 1e6) * 1e3
    else:
        t_c = 0.0
    return max(t_hbm, t_c)


# timing classes that are not the V-cycle (the Arnoldi/Givens/restart bookkeeping and the operator)
_NOT_VCYCLE = ("apply_", "cgs_", "dcgs_", "norm", "combine", "axpy64", "givens", "cycle_init", "backsolve", "rhs",
               "scale_f64")


def _composite_roofline(classes, select, peaks, label):
    """Roofline of a multi-launch operator (the V-cycle): its roofline time is the sum over its
    kernels of max(bytes/HBM, flops/peak); frac = roofline time / measured device time.  Both the
    burst and the sustained 3xTF32 denominators are reported."""
    sel = [c for c in classes if select(c["name"])]
    if not sel:
        return None
    burst, sus = _tensor_peaks(peaks)
    meas = sum(c["ms"] for c in sel)
    r_b = sum(_class_roofline_ms(c, peaks, burst) for c in sel)
    r_s = sum(_class_roofline_ms(c, peaks, sus) for c in sel)
    return {"what": label, "measured_ms": meas, "roofline_ms_burst": r_b, "roofline_ms_sustained": r_s,
            "frac": r_b / meas if meas else None, "frac_sustained": r_s / meas if meas else None,
            "flops": sum(c["flops"] for c in sel), "bytes": sum(c["bytes"] for c in sel),
            "classes": sorted(c["name"] for c in sel),
            "peaks": {"tensor_3xtf32_burst_tflops": burst, "tensor_3xtf32_sustained_tflops": sus,
                      "hbm_gbs": peaks["hbm_gbs"]},
            "note": "per-class device times of the profiled solve (every launch bracketed by CUDA events)"}


def _vcycle_direct(roof_v, classes, ops, timed_ms=None):
    """The V-cycle fraction from whole mgnet_vcycle calls timed back to back by one pair of CUDA events
    (the production launch sequence: programmatic dependent launch overlaps each kernel's prologue with
    its predecessor's tail, which the per-launch events of the profiled solve prevent).  The roofline
    time per V-cycle is the profiled solve's composite divided by its number of V-cycles (= launches of
    the once-per-V-cycle 1x1 lift / head classes).  `frac` becomes this directly timed figure; the
    per-class sums stay as frac_profiled / frac_sustained_profiled."""
    per_s = ops.get("mgnet_vcycle_per_s")
    once = [c["launches"] for c in classes if c["name"].startswith("conv1x1")]
    if roof_v is None or not per_s or not once:
        return roof_v
    n_v = min(once)
    ms = 1e3 / per_s
    roof_v["vcycles_profiled"] = n_v
    roof_v["frac_profiled"] = roof_v["frac"]
    roof_v["frac_sustained_profiled"] = roof_v["frac_sustained"]
    roof_v["measured_ms_per_vcycle"] = ms
    roof_v["roofline_ms_per_vcycle_burst"] = roof_v["roofline_ms_burst"] / n_v
    roof_v["roofline_ms_per_vcycle_sustained"] = roof_v["roofline_ms_sustained"] / n_v
    roof_v["frac"] = roof_v["roofline_ms_burst"] / n_v / ms
    roof_v["frac_sustained"] = roof_v["roofline_ms_sustained"] / n_v / ms
    roof_v["note"] = ("frac / frac_sustained: whole mgnet_vcycle calls on the seeded random vector (ops.input) "
                      "timed back to back by one pair of CUDA "
                      "events (production launch sequence, PDL overlap intact) against the per-V-cycle roofline "
                      "time; frac_profiled: per-class device times of the profiled solve (every launch "
                      "bracketed by CUDA events, which serialises the PDL overlap)")
    if timed_ms:
        # inside the timed solve: an upper bound on the V-cycle's time there = the timed region minus the
        # profiled device time of every non-V-cycle class (long HBM-bound kernels, whose per-launch event
        # overhead is negligible), so every inter-kernel gap of the step is charged to the V-cycle
        nonv = sum(c["ms"] for c in classes if c["name"].startswith(_NOT_VCYCLE))
        ms_in = (timed_ms - nonv) / n_v
        roof_v["in_solve"] = {"ms_per_vcycle_upper_bound": ms_in,
                              "frac": roof_v["roofline_ms_per_vcycle_burst"] / ms_in,
                              "frac_sustained": roof_v["roofline_ms_per_vcycle_sustained"] / ms_in,
                              "how": "(timed region - profiled device time of the non-V-cycle classes) / V-cycles"}
    return roof_v


def _roofline(classes, peaks, src, top=None):
    """Roofline of one kernel class (default: the dominant one, max total device time)."""
    if not classes:
        return None, None
    if top is None:
        top = max(classes, key=lambda c: c["ms"])
    avg_ms = top["ms"] / max(top["launches"], 1)
    per_launch_flops = top["flops"] / max(top["launches"], 1)
    per_launch_bytes = top["bytes"] / max(top["launches"], 1)
    smax = peaks.get("sm_max_mhz", 1965.0)
    kind = top["kind"]
    if kind == "tensor_3xtf32" and per_launch_bytes / (peaks["hbm_gbs"] * 1e9) > \
            per_launch_flops / (_tensor_peaks(peaks)[0] * 1e12):
        kind = "hbm"  # below the ridge (e.g. the apply at M <= 128): the binding bound is HBM
    if kind == "hbm":
        ach = per_launch_bytes / (avg_ms * 1e-3) / 1e9
        peak, unit, bound = peaks["hbm_gbs"], "GB/s", "hbm"
        note = f"HBM copy bandwidth ({src} MEASURED_PEAKS.json hbm_gbs)"
    elif kind == "tensor_3xtf32":
        ach = per_launch_flops / (avg_ms * 1e-3) / 1e12
        peak, peak_sus = _tensor_peaks(peaks)
        unit, bound = "TFLOP/s", "tensor"
        note = (f"3xTF32 fp32-emulation peak = {src} burst bf16 {peaks.get('bf16_tflops')} TF x "
                f"{TF32_PER_BF16:.3f} (nominal tf32/bf16) / 3 MMAs per product (sustained: {peak_sus:.1f} TF, "
                f"frac_sustained); achieved counts algorithmic fp32 flops")
    elif kind == "fp32_simt":
        ach = per_launch_flops / (avg_ms * 1e-3) / 1e12
        peak = N_SM * 128 * 2 * smax * 1e6 / 1e12
        unit, bound = "TFLOP/s", "alu"
        note = f"fp32 FMA peak = 148 SMs x 128 lanes x 2 flop x {smax} MHz (DESIGN.md §5)"
    elif kind == "fp64_simt":
        ach = per_launch_flops / (avg_ms * 1e-3) / 1e12
        peak = N_SM * 64 * 2 * smax * 1e6 / 1e12
        unit, bound = "TFLOP/s", "alu"
        note = f"fp64 FMA peak = 148 SMs x 64 lanes x 2 flop x {smax} MHz (DESIGN.md §5)"
    else:
        ach, peak, unit, bound, note = None, None, None, "latency", "tiny latency-bound kernel"
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                traffic = json.load(f).get(top["name"])
        except Exception:
            traffic = None
    roof = {"kernel": top["name"], "bound": bound, "achieved": ach, "peak": peak, "unit": unit,
            "frac": (ach / peak) if (ach is not None and peak) else None, "traffic": traffic,
            **({"frac_sustained": ach / peak_sus} if kind == "tensor_3xtf32" else {}),
            "avg_launch_ms": avg_ms, "launches": top["launches"],
            "algorithmic_flops_per_launch": per_launch_flops, "algorithmic_bytes_per_launch": per_launch_bytes,
            "peak_source": note}
    return roof, top


def _cpu_baseline(cfg, media, weights):
    """The fp64 oracle as it stands, on the host cores: one Arnoldi step (V-cycle + apply + MGS)."""
    from oracle import rte as O
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    op = O.setup_from_media(cfg, media)
    onet = O.make_mgnet(weights, cfg.M, cfg.L, cfg.C0, cfg.nu)
    b = O.rhs(op)
    t0 = time.perf_counter()
    O.arnoldi_columns(lambda v: O.apply(op, v), b, lambda v: O.vcycle(onet, v), 1)
    dt = time.perf_counter() - t0
    out = {"value": 1.0 / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
           "sample": f"one GMRES inner iteration of the fp64 numpy oracle on the full {cfg.k}-config problem "
                     f"(oracle.arnoldi_columns steps=1: P=I+V-cycle, apply, MGS, norm), {dt:.1f} s wall; "
                     f"BLAS threads={cores}, host cpus={os.cpu_count()}"}
    if cfg.unknowns <= 2 ** 21:  # configs 1-3: also single-threaded (SURVEY §8(d) oracle timing)
        try:
            from threadpoolctl import threadpool_limits
            with threadpool_limits(limits=1):
                t0 = time.perf_counter()
                O.arnoldi_columns(lambda v: O.apply(op, v), b, lambda v: O.vcycle(onet, v), 1)
                out["single_thread_value"] = 1.0 / (time.perf_counter() - t0)
        except Exception:
            pass
    return out


def run_reference(args, cfg):
    """Reference arm: the fp64 CPU oracle (oracle/) on the host cores, same metric and config."""
    dist, rank, ws, _ = _dist()
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    import workloads as W
    from oracle import rte as O
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    media = W.make_media(cfg)
    weights = W.make_weights(cfg)
    op = O.setup_from_media(cfg, media)
    onet = O.make_mgnet(weights, cfg.M, cfg.L, cfg.C0, cfg.nu)
    b = O.rhs(op)
    A = lambda v: O.apply(op, v)
    Pc = lambda v: O.vcycle(onet, v)
    # warm-up: W Arnoldi steps on a small copy of the workload (loads BLAS, touches code paths)
    small = W.small_config(cfg.k, N=min(cfg.N, 32), M=16, n_polar=2, n_azim=8, L=min(cfg.L, 3))
    sm = W.make_media(small)
    sop = O.setup_from_media(small, sm)
    snet = O.make_mgnet(W.make_weights(small), small.M, small.L, small.C0, small.nu)
    O.arnoldi_columns(lambda v: O.apply(sop, v), O.rhs(sop), lambda v: O.vcycle(snet, v), max(1, args.warmup))
    # bounded sample: at most K steps, capped so the run ends within a few minutes
    cap = max(2, int(3e8 // max(cfg.unknowns, 1)))
    steps = max(1, min(args.steps * cfg.restart, cap))  # (inner iterations; a bench step is a cycle)
    t0 = time.perf_counter()
    O.arnoldi_columns(A, b, Pc, steps)
    dt = time.perf_counter() - t0
    val = steps / dt
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / steps * 1e3 * cfg.restart, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": _workload_name(cfg), "unknowns": cfg.unknowns,
                       "step": f"one GMRES({cfg.restart}) restart cycle (timed on a bounded sample of "
                               f"{steps} inner iterations; ms_per_step extrapolated per cycle)"},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{steps} Arnoldi steps (oracle.arnoldi_columns: V-cycle + apply + MGS) "
                                       f"of the fp64 numpy oracle on the full config-{cfg.k} problem "
                                       f"(steps capped from {args.steps} to bound the run)"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def run_ours(args, cfg):
    import torch
    dist, rank, ws, local = _dist()
    import paper_2604_23265_b200 as P
    import workloads as W
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    media = W.make_media(cfg)
    weights = W.make_weights(cfg)
    # batched configs (config 4: independent samples, independent solves) shard the samples across
    # ranks with no data-path collective: total work fixed, "scaling": "strong".
    # B = 1 configs run one replica per rank ("weak").
    sharded = cfg.B > 1 and ws > 1
    lo, hi = benchlib.shard(cfg.B, rank, ws) if sharded else (0, cfg.B)
    if sharded and hi == lo:
        raise SystemExit(f"rank {rank}: no sample to solve (world size {ws} > batch {cfg.B})")
    sl = slice(lo, hi)
    p = P.rte_setup(cfg.N, media.sigma_T[sl], media.sigma_a[sl], media.q[sl], media.eps[sl], media.g[sl],
                    media.inflow[sl], n_polar=cfg.n_polar, n_azim=cfg.n_azim)
    net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, weights)
    coeffnet_ms = None
    if args.coeffnet:  # NEXT-1: the medium-conditioned smoother (setup once per medium, untimed)
        t0 = time.perf_counter()
        P.mgnet_coeffnet(net, media.sigma_T[sl], media.sigma_a[sl], media.eps[sl], W.make_coeffnet_weights(cfg))
        coeffnet_ms = (time.perf_counter() - t0) * 1e3
    b = torch.empty(p.shape, dtype=torch.float32, device=dev)
    P.rte_rhs(p, b)
    x = torch.zeros(p.shape, dtype=torch.float64, device=dev)
    # a step = one whole restart cycle (module docstring): K cycles = K * restart inner iterations
    K, Wm = args.steps * cfg.restart, args.warmup * cfg.restart
    # x0 = 0 (the usual GMRES start): x0_zero sets x to 0 inside the call and skips A x0
    solve = lambda xx, bb, k: P.gmres_solve(p, net, bb, xx, restart=cfg.restart, maxit=k, rtol=1e-300,
                                            history=False, reorth=args.reorth, x0_zero=True)
    # setup: capture the per-Arnoldi-step CUDA graphs once (RTE_NO_GRAPHS=1 disables)
    P.gmres_prepare(p, net, restart=cfg.restart, reorth=args.reorth)
    # warm-up: W inner iterations (one solve), untimed
    solve(x, b, max(Wm, 1))
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()

    # ---- profiled solve (untimed): every launch bracketed by CUDA events -> per-class device
    # times (the "kernels" breakdown) and the dominant class.  The event pairs of every launch
    # cost ~10% of a step, so the timed solve below instruments only the dominant class.
    x.zero_()
    P.rte_timing_enable(True)
    P.rte_timing_filter(None)
    P.rte_timing_reset()
    solve(x, b, K)
    torch.cuda.synchronize()
    all_classes = P.rte_timing_get()
    dominant = max(all_classes, key=lambda c: c["ms"])["name"] if all_classes else None

    # ---- timed region: one solve of exactly K inner iterations --------------------------
    x.zero_()
    sampler = ClockSampler(_device_index(torch, local))
    sampler.start()
    P.rte_launch_count(reset=True)
    P.rte_timing_filter(dominant)  # the dominant kernel's launches are timed live, nothing else
    P.rte_timing_reset()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    rep = solve(x, b, K)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = ev0.elapsed_time(ev1)
    launches = P.rte_launch_count(reset=True)
    classes = P.rte_timing_get()  # the dominant class only, timed inside the timed region
    P.rte_timing_filter(None)
    P.rte_timing_enable(False)
    clocks = sampler.stop()
    iters = sum(r["iterations"] for r in rep) / len(rep)
    assert iters == K, f"solve ran {iters} iterations, expected {K}"
    ms_max = benchlib.max_over_ranks(ms, dist, dev)
    # sharded: the job is K iterations of the whole batch; replicas: ws jobs of K iterations
    value = benchlib.aggregate(K, 1 if sharded else ws, ms_max)

    # ---- e2e: same solve through the public C-ABI call with HOST buffers (gmres_solve_host: b
    # copied in, x copied out inside the call, from/to pinned host memory) --------------------
    b_host = torch.empty(p.shape, dtype=torch.float32, pin_memory=True)
    b_host.copy_(b)
    x_host = torch.empty(p.shape, dtype=torch.float64, pin_memory=True)
    P.gmres_solve_host(p, net, b_host, x_host, restart=cfg.restart, maxit=1, rtol=1e-300, history=False,
                       reorth=args.reorth, x0_zero=True)  # first call allocates the device copies
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    rep_e2e = P.gmres_solve_host(p, net, b_host, x_host, restart=cfg.restart, maxit=K, rtol=1e-300, history=False,
                                 reorth=args.reorth, x0_zero=True)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    assert sum(r["iterations"] for r in rep_e2e) / len(rep_e2e) == K
    ms_e2e = benchlib.max_over_ranks(e0.elapsed_time(e1), dist, dev)
    h2d = b_host.numel() * 4
    d2h = x_host.numel() * 8

    # ---- single-op throughputs (north star: applies/s, V-cycles/s), device events ----------
    ops = {}
    if rank == 0:
        y = torch.empty_like(b)
        z = torch.empty_like(b)
        # input: the seeded iid N(0,1) vector of the parity tests, not the right-hand side -- the operators'
        # speed depends on the data under the power cap (measured at config 5: a V-cycle on the nearly
        # constant rhs takes 1.80 ms, on the random vector 2.03 ms), and Krylov vectors are rough
        xv = torch.from_numpy(W.make_vector(cfg)).to(b.device)
        if xv.shape != b.shape:  # (config-4 sharding: this rank's samples)
            xv = xv.reshape((-1,) + tuple(b.shape[1:]))[:b.shape[0]].contiguous()
        ops["input"] = "seeded iid N(0,1) vector (workloads.make_vector); 20 calls back to back, CUDA events"
        for name, fn in (("rte_apply_per_s", lambda: P.rte_apply(p, xv, y)),
                         ("mgnet_vcycle_per_s", lambda: P.mgnet_vcycle(net, xv, z, True))):
            fn()
            torch.cuda.synchronize()
            reps = 20
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(reps):
                fn()
            a1.record(stream)
            torch.cuda.synchronize()
            ops[name] = reps / (a0.elapsed_time(a1) * 1e-3)

    if rank == 0:
        peaks, src = _peaks()
        roof, top = _roofline(classes, peaks, src)
        if roof is not None:
            roof["timed"] = "live in the timed region (only this class carries CUDA events there)"
        tot_ms = sum(c["ms"] for c in all_classes) or 1.0
        kernels = sorted(({"name": c["name"], "kind": c["kind"], "launches": c["launches"],
                           "ms": round(c["ms"], 4), "share": round(c["ms"] / tot_ms, 4)} for c in all_classes),
                         key=lambda d: -d["ms"])
        roof_apply = None
        app = [c for c in all_classes if c["name"].startswith("apply_f32")]
        if app:
            roof_apply, _ = _roofline(app, peaks, src, top=max(app, key=lambda c: c["ms"]))
            roof_apply["timed"] = "profiled solve (every launch bracketed by CUDA events)"
        roof_v = _composite_roofline(all_classes, lambda n: not n.startswith(_NOT_VCYCLE), peaks,
                                     "MgNet V-cycle (lift, smoother/restriction/prolongation convs, split-K "
                                     "reductions, head + pass-through)")
        roof_v = _vcycle_direct(roof_v, all_classes, ops, ms_max if ws == 1 else None)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "strong" if sharded else "weak",
                "vs_baseline": None,
                "dtype": "f32", "data": "synthetic",
                "config": {"workload": _workload_name(cfg) + (" + CoeffNet-modulated smoother" if args.coeffnet else ""),
                           "unknowns": cfg.unknowns,
                           "step": f"one GMRES({cfg.restart}) restart cycle: {cfg.restart} inner iterations + "
                                   "cycle end (back-solve, x += P(V y), fp64 restart residual)",
                           "restart": cfg.restart, "inner_iterations_timed": K,
                           **({"coeffnet_setup_ms": round(coeffnet_ms, 1)} if args.coeffnet else {}),
                           "l2": "inputs larger than L2 (each vector 4 B x unknowns)" if cfg.unknowns * 4 > 126e6
                           else "working set L2-resident (small config)",
                           "parallelism": (f"{cfg.B} samples sharded over {ws} ranks" if sharded
                                           else f"replicas x{ws}" if ws > 1 else "single GPU"),
                           "precision": "fp32 storage/arithmetic, fp64 iterate, reductions and restart residual",
                           "gram_schmidt": {0: "CGS2", 1: "CGS1", 2: "selective (DGKS)",
                                            3: "DCGS2 (delayed re-orthogonalisation)"}[args.reorth]},
                "roofline": roof, "roofline_apply": roof_apply, "roofline_vcycle": roof_v,
                "e2e": {"value": benchlib.aggregate(K, 1 if sharded else ws, ms_e2e), "unit": UNIT,
                        "h2d_bytes_per_step": h2d / K, "d2h_bytes_per_step": d2h / K,
                        "note": f"one gmres_solve_host call of {K} iterations (C ABI, host buffers): b (fp32) "
                                "copied H2D from pinned host memory inside it, x (fp64) D2H into pinned memory "
                                "(overlapping the closing fp64 residual); bytes amortised per step"},
                "gpu_launches": launches, "clocks": clocks, "ops": ops, "kernels": kernels}
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = _cpu_baseline(cfg, media, weights)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def run_time_to_tol(args, cfg):
    """Time-to-tolerance (north star: "GMRES iterations/s, time-to-tolerance"): the full MgNet-
    preconditioned GMRES(30) solve from x0 = 0 to the config's rtol (configs 1, 2 converge; 3-5 run their
    fixed budgets and report the residual reached), on the device (CUDA events, best of 3 after a warm-up
    solve) and end to end through gmres_solve_host (host wall clock), next to the fp64 oracle's solve on
    the host cores (configs 1-2 only: the cpu_baseline leg).  One JSON line."""
    import torch
    import paper_2604_23265_b200 as P
    import workloads as W
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    media = W.make_media(cfg)
    weights = W.make_weights(cfg)
    p = P.rte_setup(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                    n_polar=cfg.n_polar, n_azim=cfg.n_azim)
    net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, weights)
    b = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_rhs(p, b)
    x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
    P.gmres_prepare(p, net, restart=cfg.restart, reorth=args.reorth)
    kw = dict(restart=cfg.restart, maxit=cfg.maxit, rtol=cfg.rtol, reorth=args.reorth, x0_zero=True, history=False)
    P.gmres_solve(p, net, b, x, **kw)
    torch.cuda.synchronize()
    best, rep = None, None
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rep = P.gmres_solve(p, net, b, x, **kw)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    bh = b.cpu().pin_memory()
    xh = torch.zeros(p.shape, dtype=torch.float64).pin_memory()
    P.gmres_solve_host(p, net, bh, xh, **kw)
    t0 = time.perf_counter()
    P.gmres_solve_host(p, net, bh, xh, **kw)
    e2e_s = time.perf_counter() - t0
    its = [r["iterations"] for r in rep]
    line = {"metric": "time-to-tolerance (s)", "value": best * 1e-3, "unit": "s", "higher_is_better": False,
            "n_gpus": 1, "dtype": "f32", "data": "synthetic",
            "config": {"workload": _workload_name(cfg), "rtol": cfg.rtol, "budget": cfg.maxit,
                       "fixed_budget": cfg.fixed_budget, "restart": cfg.restart,
                       "gram_schmidt": {0: "CGS2", 1: "CGS1", 2: "selective (DGKS)",
                                        3: "DCGS2 (delayed re-orthogonalisation)"}[args.reorth]},
            "iterations": its, "converged": [bool(r["converged"]) for r in rep],
            "relres_true": [r["relres_true"] for r in rep],
            "iter_per_s": sum(its) / len(its) / (best * 1e-3),
            "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes": bh.numel() * 4, "d2h_bytes": xh.numel() * 8,
                    "note": "one gmres_solve_host call (host buffers), host wall clock"}}
    if not cfg.fixed_budget and not args.no_cpu_baseline:
        from oracle import rte as O
        try:
            from threadpoolctl import threadpool_info
            cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
        except Exception:
            cores = os.cpu_count()
        op = O.setup_from_media(cfg, media)
        onet = O.make_mgnet(weights, cfg.M, cfg.L, cfg.C0, cfg.nu)
        b64 = O.rhs(op).astype(np.float32).astype(np.float64)
        t0 = time.perf_counter()
        res = O.gmres(lambda v: O.apply(op, v), b64, P=lambda v: O.vcycle(onet, v), restart=cfg.restart,
                      rtol=cfg.rtol, maxit=cfg.maxit)
        line["cpu_baseline"] = {"value": time.perf_counter() - t0, "unit": "s", "cores": cores, "kind": "oracle",
                                "iterations": res.iterations, "converged": bool(res.converged),
                                "sample": "the whole solve of the fp64 numpy oracle (oracle.gmres with MGS) on the "
                                          "same fp32-rounded b"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3, help="restart cycles timed (x restart inner iterations)")
    ap.add_argument("--warmup", type=int, default=3, help="untimed warm-up cycles")
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--coeffnet", action="store_true",
                    help="NEXT-1: precondition with the CoeffNet-modulated MgNet (DESIGN.md R31-R33)")
    ap.add_argument("--time-to-tol", action="store_true",
                    help="time the full solve to the config's rtol (or its budget) instead of K cycles")
    ap.add_argument("--reorth", type=int, default=3, choices=[0, 1, 2, 3],
                    help="Gram-Schmidt: 3 DCGS2 (default), 0 CGS2, 1 CGS1, 2 selective re-orthogonalisation")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    import workloads as W
    cfg = W.config(args.config)
    if args.impl == "reference":
        run_reference(args, cfg)
    elif args.time_to_tol:
        run_time_to_tol(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
