#!/usr/bin/env python
"""bench.py -- IR time-to-solution on B200 (BASELINE.json configs[1], config 2a).

(--config cfg1|cfg2b|cfg3|cfg4 [--lu-mode tc] measures the other BASELINE
configs the same way; the default line is config 2a.)

Workload (one "step"): the reference's factor-once + refine path on
A = I - 800 G (N = 4096, trapezoid Green's operator, fp64), b ~ N(0,1) seed 0,
<TW,TF,TR> = <fp64, fp32, fp64>, scaled (LPS) corrections, backward-error
stopping rule with ce = 10, litmax = 20:
    MPFactorization ctor work (||A||_1 + demotion + fp32 LU)  + ir_solve_report
A is resident in HBM when the timed region starts (``value``); ``e2e`` goes
through the public C-ABI with pinned HOST buffers, H2D of A and b and D2H of x
inside the timed region.

Metric (BASELINE.json): IR time-to-solution in seconds (lower is better);
the LU GFLOP/s (2N^3/3 over the LU device time) rides along.

--impl reference times the reference's own CPU code path (oracle/_ref: the
unmodified reference headers compiled from /root/reference with its flags),
single-threaded by construction for fp32 factors (mp_structures.hpp:166-167).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess

# more hardware work queues than the default 8 for the LU's concurrent
# streams (see paper_2311_14616_b200/__init__.py); before any CUDA context
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PREC = {0: "f64", 1: "f32", 2: "f16"}
ESZ = {0: 8, 1: 4, 2: 2}
METRIC = "IR time-to-solution & LU GFLOP/s (2N^3/3) vs fp16-TC/fp32 peak"
HBM_FALLBACK = 6650.0
HBM_NOMINAL = 7700.0  # B200_PROFILING.md: HGX B200 HBM3e figure


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--config", default="cfg2a",
                    choices=["cfg1", "cfg2a", "cfg2b", "cfg3", "cfg4", "cfg5a", "cfg5b"],
                    help="BASELINE config (default cfg2a = the headline workload)")
    ap.add_argument("--lu-mode", default="exact", choices=["exact", "tc"],
                    help="tc: tcgen05 trailing update for binary16 factors (cfg3)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--count", type=int, default=4096,
                    help="cfg5b: total independent systems over all ranks")
    ap.add_argument("--dist", action="store_true",
                    help="cfg5a at N=1 through the distributed code path (bench_dist.py)")
    ap.add_argument("--no-also", action="store_true",
                    help="default run only: skip the cfg4 and cfg3-tc lines attached as `also`")
    ap.add_argument("--block-cols", type=int, default=512,
                    help="cfg5a on N>1 GPUs: columns per block of the 1-D block-cyclic layout")
    args = ap.parse_args()
    args.config_given = any(a == "--config" or a.startswith("--config=") for a in sys.argv[1:])
    return args


def workload(args, pinned=False):
    """Seeded host inputs + reference parameters; default cfg 2a.
    pinned: generate A straight into pinned host memory (cfg5a: 34 GB, one copy)."""
    from paper_2311_14616_b200 import configs
    out = None
    if pinned:
        import torch
        n = args.n or configs.FULL_N[args.config]
        out = torch.empty(n * n, dtype=torch.float64).pin_memory().numpy()
    cfg = configs.config(args.config, args.n, out)
    cfg["a_pinned"] = out is not None
    cfg["workload"] = workload_tag(args, cfg)
    return cfg


def workload_tag(args, cfg):
    return (f"{args.config}: N={cfg['n']}, <{PREC[cfg['tw']]},{PREC[cfg['tf']]},"
            f"{PREC[cfg['tr']]}>, ce={cfg['ce']}, litmax={cfg['litmax']}"
            + (", lu_mode=tc (tcgen05 trailing update)" if args.lu_mode == "tc" else ""))


def to_tw(arr64, tw):
    """The facade's one rounding of float64 inputs into TW (runtime.cpp:23-28)."""
    import numpy as np
    return arr64 if tw == 0 else arr64.astype(np.float32)


def measured_peaks():
    for p in (os.path.join(ROOT, "MEASURED_PEAKS.json"), "/root/repo/MEASURED_PEAKS.json"):
        if os.path.exists(p):
            with open(p) as f:
                d = json.load(f)
            return d, "measured"
    return {"hbm_gbs": HBM_FALLBACK}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            import atexit
            atexit.register(self.__exit__)  # never leave nvidia-smi running
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc and self.proc.poll() is None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "nccl" if args.impl == "ours" else "gloo"
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
            # keep NCCL's communicator/transport lines (NVLink, NVLS) in stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group(backend=backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v, world):
    if world <= 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# Reference arm: the reference's CPU path (oracle/_ref), no GPU work.
# ---------------------------------------------------------------------------
def run_reference(args, world, rank):
    if rank != 0:
        return
    from paper_2311_14616_b200 import configs
    n = args.n or configs.FULL_N[args.config]
    if n > SAMPLE_N:  # only the N = 4096 sample is generated (reference_solve)
        cfg = {**configs.config(args.config, SAMPLE_N), "n": n}
        cfg["workload"] = workload_tag(args, cfg)
    else:
        cfg = workload(args)
    a_w, b_w = to_tw(cfg["a"], cfg["tw"]), to_tw(cfg["b"], cfg["tw"])
    times = []
    info = None
    for i in range(args.warmup + args.steps):
        dt, info = reference_solve(args, cfg, a_w, b_w)
        if i >= args.warmup:
            times.append(dt)
    sec = statistics.mean(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": sec, "unit": "s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": f"{PREC[cfg['tw']]}/{PREC[cfg['tf']]}",
        "data": "synthetic (seeded: libstdc++ mt19937_64 generators, SURVEY 8(d))",
        "config": {"workload": cfg["workload"], "n": n},
        "cpu_baseline": {**info, "value": sec},
        "e2e": {"value": sec, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_split_s": info["split_s"],
        "iters": info["iters"], "reason": info["reason"],
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# Our arm
# ---------------------------------------------------------------------------
def lu_work(n, nb):
    """Algorithmic flops of the LU pieces (per factorization)."""
    gemm = trsm = panel = 0.0
    for k0 in range(0, n, nb):
        jb = min(nb, n - k0)
        m = n - k0
        t = n - k0 - jb
        gemm += 2.0 * t * t * jb
        trsm += float(jb) * (jb - 1) * t
        for j in range(jb):
            panel += (m - j - 1) * (1 + 2 * (jb - j - 1))
    return {"gemm": gemm, "trsm": trsm, "panel": panel, "total": 2.0 * n ** 3 / 3.0}


def run_ours(args, world, rank, local):
    import numpy as np
    import torch
    from paper_2311_14616_b200 import _lib as L
    lib = L.lib()
    torch.cuda.set_device(local)
    big = args.config == "cfg5a"
    wl = workload(args, pinned=big)
    n = wl["n"]
    tw, tf, tr = wl["tw"], wl["tf"], wl["tr"]
    a_host, b_host = to_tw(wl["a"], tw), to_tw(wl["b"], tw)
    litmax = wl["litmax"]
    cfg = L.mpirg_config(tw, tf, tr, wl["on_the_fly"], int(wl["resid_term"]),
                         L.LU_TC if args.lu_mode == "tc" else L.LU_EXACT, 0, local)
    tp = L.mpirg_term_params(1.0, wl["ce"], 0.5, litmax)
    a_dev = torch.from_numpy(a_host).cuda()
    b_dev = torch.from_numpy(b_host).cuda()
    sol_dev = torch.empty(n, dtype=b_dev.dtype, device="cuda")
    h = C.c_void_p()
    err = L.mpirg_error()
    L.check(lib.mpirg_factorization_create(C.byref(h), n, C.byref(cfg), a_dev.data_ptr(), 1,
                                           C.byref(err)), err)
    lib.mpirg_factorization_config(h, C.byref(cfg))
    del a_dev  # the handle holds its own copy (a_high); refactor(None) reuses it
    torch.cuda.empty_cache()
    cap = litmax + 1
    rh, dh = (C.c_double * cap)(), (C.c_double * cap)()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    # one CUDA-event pair around the whole step, on the handle's own stream
    # (torch.cuda.Event on torch's current stream would not see it)
    hstream = torch.cuda.ExternalStream(lib.mpirg_factorization_stream(h))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def step(prof=False):
        """One time-to-solution on resident data; returns (device ms between one
        event pair around refactor + solve, factor ms, report)."""
        rep = L.mpirg_report(sol_dev.data_ptr(), 1, rh, dh, cap, 0, 0, 0, 0.0)
        ev0.record(hstream)
        L.check(lib.mpirg_factorization_refactor(h, None, 1, C.byref(err)), err)
        fms = lib.mpirg_factorization_last_factor_ms(h)
        L.check(lib.mpirg_ir_solve(h, b_dev.data_ptr(), 1, C.byref(tp), C.byref(rep),
                                   C.byref(err)), err)
        ev1.record(hstream)
        ev1.synchronize()
        return ev0.elapsed_time(ev1), fms, rep

    # nvidia-smi takes ~0.1 s to start and the cfg 2a timed region lasts ~40 ms:
    # sample from the warm-up through the e2e steps (same load throughout)
    clocks = ClockSampler(local).__enter__()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # Timed region: K steps, L2 flushed between steps (flush excluded from the
    # per-step CUDA-event times), per-kernel event timing on the handle's stream.
    nclass = len(L.KERNEL_CLASSES)
    ms_k = (C.c_double * nclass)()
    cnt_k = (C.c_int * nclass)()
    lib.mpirg_profile_collect(ms_k, cnt_k, nclass)
    step_ms, fac_ms = [], []
    rep = None
    barrier(world)
    torch.cuda.synchronize()
    t_wall0 = time.perf_counter()
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        sms, fms, rep = step()
        step_ms.append(sms)
        fac_ms.append(fms)
    torch.cuda.synchronize()
    barrier(world)
    t_wall = time.perf_counter() - t_wall0
    # Per-kernel split: the same K steps again with a CUDA event pair around
    # every launch on its own stream (mpirg_profile_*). The event records
    # perturb the LU's critical chain (~15% at cfg2a), so these steps are not
    # the ones `value` is taken from; `share_of_step` is against their mean.
    prof_ms = []
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        lib.mpirg_profile_enable(1)
        pms, _, _ = step()
        lib.mpirg_profile_enable(0)
        prof_ms.append(pms)
    torch.cuda.synchronize()
    lib.mpirg_profile_collect(ms_k, cnt_k, nclass)
    kernel_ms = {L.KERNEL_CLASSES[i]: ms_k[i] / args.steps for i in range(nclass)}
    kernel_n = {L.KERNEL_CLASSES[i]: cnt_k[i] / args.steps for i in range(nclass)}
    prof_mean_ms = statistics.mean(prof_ms)
    mean_ms = statistics.mean(step_ms)
    mean_ms = max_over_ranks(mean_ms, world)
    iters = rep.rhist_len - 1
    reason = L.REASONS[rep.reason]

    # e2e: public API with pinned host buffers (H2D of A,b and D2H of x timed).
    e2e = None
    if not args.no_e2e:
        a_pin = (torch.from_numpy(a_host) if wl["a_pinned"] and tw == 0 else
                 torch.from_numpy(a_host).pin_memory())
        b_pin = torch.from_numpy(b_host).pin_memory()
        x_pin = torch.empty(n, dtype=b_dev.dtype).pin_memory()
        e2e_t = []
        # warm-up: the first refactor from this host pointer runs the streamed
        # schedule directly, the second captures it into a graph (replayed after)
        e2e_w = max(3, args.warmup)
        for i in range(e2e_w + args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep2 = L.mpirg_report(x_pin.data_ptr(), 0, rh, dh, cap, 0, 0, 0, 0.0)
            L.check(lib.mpirg_factorization_refactor(h, a_pin.data_ptr(), 0, C.byref(err)), err)
            L.check(lib.mpirg_ir_solve(h, b_pin.data_ptr(), 0, C.byref(tp), C.byref(rep2),
                                       C.byref(err)), err)
            dt = time.perf_counter() - t0
            if i >= e2e_w:
                e2e_t.append(dt)
        e2e_s = max_over_ranks(statistics.mean(e2e_t), world)
        e2e = {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": (n * n + n) * ESZ[tw],
               "d2h_bytes_per_step": n * ESZ[tw] + 3 * 8 * cap}

    clocks.__exit__(None, None, None)
    # Roofline of the dominant kernel class.
    peaks, peak_src = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", HBM_FALLBACK))
    ffma = C.c_double(0.0)
    ffma_ms = C.c_double(0.0)
    lib.mpirg_ffma_peak(C.byref(ffma), C.byref(ffma_ms))
    # panel width as chosen by lu_choose_nb (lu.cu): binary64 factors narrow
    # with n, binary32/16 factors use 64 at every n
    nb = (64 if n <= 4096 else (32 if n <= 8192 else 16)) if tf == 0 else 64
    work = lu_work(n, nb)
    tf_b, tw_b = ESZ[tf], ESZ[tw]
    tc = args.lu_mode == "tc" and tf == 2
    gemm_bound = ("tcgen05 fp16 (fp32 accumulate)" if tc else
                  {0: "fp64 SIMT", 1: "fp32-ffma", 2: "fp16 SIMT (two roundings per term)"}[tf])
    gemm_peak = float(peaks.get("bf16_tflops", 0.0)) if tc else ffma.value
    kernels = {}
    for name in L.KERNEL_CLASSES:
        kms = kernel_ms[name]
        if kms <= 0:
            continue
        d = {"ms_per_step": kms, "launches_per_step": kernel_n[name],
             "share_of_step": kms / prof_mean_ms}
        if name == "gemm":
            d.update(bound=gemm_bound, achieved=work["gemm"] / (kms * 1e-3) / 1e12,
                     unit="TFLOP/s", peak=gemm_peak)
        elif name == "panel":
            d.update(bound="latency (one pivot search per column)", unit="TFLOP/s",
                     achieved=work["panel"] / (kms * 1e-3) / 1e12, peak=ffma.value)
        elif name == "trsm":
            d.update(bound="fp32-ffma", achieved=work["trsm"] / (kms * 1e-3) / 1e12,
                     unit="TFLOP/s", peak=ffma.value)
        elif name == "cast":
            d.update(bound="hbm", achieved=n * n * (tw_b + tf_b) / (kms * 1e-3) / 1e9,
                     unit="GB/s", peak=hbm)
        elif name in ("trsv_lower", "trsv_upper"):
            per = kernel_n[name]
            d.update(bound="hbm", achieved=per * (n * n / 2.0) * tf_b / (kms * 1e-3) / 1e9,
                     unit="GB/s", peak=hbm)
        elif name == "residual":
            per = kernel_n[name]
            d.update(bound="hbm", achieved=per * n * n * tw_b / (kms * 1e-3) / 1e9,
                     unit="GB/s", peak=hbm)
        if "peak" in d and d["peak"]:
            d["frac"] = d["achieved"] / d["peak"]
        if d.get("bound") == "hbm":
            # read-mostly streams can beat the measured copy figure (read+write)
            d["frac_of_nominal_hbm"] = d["achieved"] / HBM_NOMINAL
        kernels[name] = d
    dom = max(kernels, key=lambda k: kernels[k]["ms_per_step"])
    dk = kernels[dom]
    # SURVEY 8(d) units: the LU as a whole (2N^3/3 flops over the factor time,
    # against the FFMA peak for binary32/64 factors -- TF32/tensor cores would
    # change the factor precision -- or the tcgen05 kind::f16 peak in tc mode),
    # the substitution pair and the residual in algorithmic bytes over HBM.
    fac_mean_ms = statistics.mean(fac_ms)
    lu_unit = {"unit": "TFLOP/s", "achieved": work["total"] / (fac_mean_ms * 1e-3) / 1e12,
               "peak": gemm_peak, "bound": "tensor" if tc else gemm_bound,
               "work": "2N^3/3 flops over the refactor device time (cast + LU)",
               "ms": fac_mean_ms}
    if gemm_peak:
        lu_unit["frac"] = lu_unit["achieved"] / gemm_peak
    units = {"lu": lu_unit}
    for nm in ("cast", "trsv_lower", "trsv_upper", "residual", "gemm"):
        if nm in kernels and "frac" in kernels[nm]:
            units[nm] = {k: kernels[nm][k] for k in ("unit", "achieved", "peak", "frac", "bound")}
    # the contract's `roofline` object: the dominant kernel class when it has
    # a 8(d) unit (update, cast, substitution, residual); when the latency-bound
    # panel chain dominates (N = 4096) the LU as a unit, bound named truthfully
    if dom in units:
        rk, ru = dom, units[dom]
    else:
        rk, ru = "lu (panel chain + row moves + U12 solve + trailing update)", lu_unit
    bound_detail = ru.get("bound")
    roof_bound = ("hbm" if bound_detail == "hbm" else
                  "tensor" if (tc and rk != "cast") else
                  "latency" if (rk.startswith("lu") and dom == "panel") else bound_detail)
    peak_note = ("MEASURED_PEAKS.json hbm_gbs" if ru.get("unit") == "GB/s" else
                 "MEASURED_PEAKS.json bf16_tflops (tcgen05 kind::f16 rate)" if tc else
                 "fp32 FFMA microbenchmark (mpirg_ffma_peak) on this GPU; TF32/tensor cores "
                 "excluded by contract")
    roofline = {"kernel": rk, "bound": roof_bound, "bound_detail": bound_detail,
                "dominant_kernel_class": dom,
                "achieved": ru.get("achieved"), "peak": ru.get("peak"), "unit": ru.get("unit"),
                "frac": ru.get("frac"), "traffic": None,
                "traffic_source": None,
                "peak_source": peak_note,
                "peak_kind": peak_src, "units": units}
    tr_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tr_path) and args.n is None and args.lu_mode == "exact":
        trf = json.load(open(tr_path)).get(args.config, {}).get(dom)
        if trf:
            roofline["traffic"] = trf["bytes_per_launch"]
            roofline["traffic_source"] = trf["capture"]
    if roofline["kernel"] != dom:
        roofline["traffic_note"] = "traffic is the dominant class's (%s) per-launch DRAM bytes" % dom
    lu_ms = sum(kernel_ms[k] for k in ("panel", "moves", "trsm", "gemm"))
    # The binary32 trailing-update kernel timed alone (no panel chain sharing
    # the SMs): the K = 128 pass the paired LU steps launch, at this n and at
    # the largest single-GPU LU (cfg4, n = 16384).
    update_alone = []
    if tf == 1:
        for un in sorted({n if n % 4 == 0 else 0, 16384} - {0}):
            tfl, ums = C.c_double(0.0), C.c_double(0.0)
            if lib.mpirg_ubench_gemm_f32(un, 128, 0, 5, C.byref(tfl), C.byref(ums)) == 0:
                update_alone.append({"n": un, "K": 128, "ms": ums.value,
                                     "tflops": tfl.value, "peak_tflops": ffma.value,
                                     "frac": tfl.value / ffma.value})

    # The tcgen05 update timed alone at the three largest node updates of the
    # recursive LU (K = n/2, n/4, n/8 on the first block of each level).
    tc_alone = []
    if tc:
        scratch = (torch.randn(n * n, device="cuda") * 0.01).half()
        for K in (n // 2, n // 4, n // 8):
            if K % 64 or K <= 0:
                continue
            tms = []
            for i in range(4):
                flush.fill_(1.0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                L.check(lib.mpirg_tc_gemm(n, scratch.data_ptr(), K, n, K, n, 0, K, None,
                                          C.byref(err)), err)
                e1.record()
                torch.cuda.synchronize()
                if i:
                    tms.append(e0.elapsed_time(e1))
            tfl = 2.0 * (n - K) ** 2 * K / (min(tms) * 1e-3) / 1e12
            tc_alone.append({"M": n - K, "N": n - K, "K": K, "ms": min(tms), "tflops": tfl,
                             "peak_tflops": gemm_peak,
                             "frac": tfl / gemm_peak if gemm_peak else None,
                             "algorithmic_bytes": 2 * (2 * (n - K) * K) + 4 * (n - K) ** 2})
        try:  # DRAM traffic of the K = n/2 launch from the committed ncu --set full capture
            trf = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
            t4 = trf.get(args.config + "_tc", {}).get("tc_update_K%d" % (n // 2))
            if t4 and tc_alone:
                tc_alone[0]["traffic"] = t4["bytes_per_launch"]
                tc_alone[0]["traffic_source"] = t4["capture"]
        except Exception:
            pass
        del scratch

    checks = None
    if big:
        # Size-independent properties at N = 65536 (the oracle would need hours):
        # no interchanges (A = I - G is diagonally dominant), the reference's
        # stopping reason, and agreement with the continuum solution of
        # u - int g u = 1, u(t) = cos t + (1 - cos 1)/sin 1 * sin t, to the
        # trapezoid rule's O(h^2) discretisation error.
        ipiv = np.zeros(n, dtype=np.int32)
        lib.mpirg_factorization_get_ipiv(h, ipiv.ctypes.data)
        x = sol_dev.double().cpu().numpy()
        t = np.arange(n) / (n - 1.0)
        u = np.cos(t) + (1.0 - np.cos(1.0)) / np.sin(1.0) * np.sin(t)
        checks = {"interchanges": int((ipiv != np.arange(n)).sum()),
                  "max_abs_x_minus_continuum": float(np.abs(x - u).max()),
                  "h2": (1.0 / (n - 1)) ** 2,
                  "max_abs_x_minus_reversed": float(np.abs(x - x[::-1]).max())}
        if rank == 0 and not args.no_cpu_baseline:
            checks.update(host_residual_check(a_host, x, b_host,
                                              lib.mpirg_factorization_a_norm1(h)))
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, wl, a_host, b_host)

    if rank == 0:
        launches = int(round(sum(kernel_n.values())))
        line = {
            "metric": METRIC, "value": mean_ms / 1e3, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_ms,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
            "dtype": f"{PREC[tw]}/{PREC[tf]} (TW={PREC[tw]}, TF={PREC[tf]}, TR={PREC[tr]})",
            "data": "synthetic (seeded: libstdc++ mt19937_64 generators per SURVEY 8(d))",
            "config": {"workload": wl["workload"], "n": n, "nb": nb,
                       "parallelism": "replicas" if world > 1 else "single GPU",
                       "l2": "flushed between steps (256 MiB write), flush excluded",
                       "a_resident_in_hbm": True},
            "lu_gflops": work["total"] / (statistics.mean(fac_ms) * 1e-3) / 1e9,
            "factor_ms": statistics.mean(fac_ms), "lu_kernels_ms": lu_ms,
            "profiled_step_ms": prof_mean_ms,
            "iters": iters, "reason": reason,
            "roofline": roofline, "kernels": kernels,
            "ffma_peak_tflops": ffma.value, "update_kernel_alone": update_alone,
            "tc_update_alone": tc_alone,
            "e2e": e2e, "gpu_launches": launches,
            "clocks": {**clocks.summary(),
                       "window": "warm-up, timed, profiled and e2e steps (nvidia-smi -lms 50)"},
            "wall_s_timed_region": t_wall,
        }
        if checks:
            line["checks"] = checks
        if cpu:
            line["cpu_baseline"] = cpu
    else:
        line = None
    lib.mpirg_factorization_destroy(h)
    del hstream
    torch.cuda.empty_cache()
    return line


SAMPLE_N = 4096  # largest N whose reference solve takes seconds, not hours


def reference_solve(args, wl, a_host, b_host):
    """One reference solve (oracle/_ref, else the restatement) of this workload;
    above SAMPLE_N a bounded sample: the same operator family at N = 4096,
    extrapolated (factor x (N/4096)^3, solve x (N/4096)^2). Returns (s, dict)."""
    import oracle
    n = wl["n"]
    impl = oracle.reference()
    kind = "reference"
    if impl is None:
        impl, kind = oracle.restatement(), "port"
    scale_f = scale_s = 1.0
    if n > SAMPLE_N:
        from paper_2311_14616_b200 import configs
        sw = configs.config(args.config, SAMPLE_N)
        a_host, b_host = to_tw(sw["a"], sw["tw"]), to_tw(sw["b"], sw["tw"])
        scale_f, scale_s = (n / SAMPLE_N) ** 3, (n / SAMPLE_N) ** 2
        ns = SAMPLE_N
    else:
        ns = n
    af = a_host.reshape(ns, ns).T
    t0 = time.perf_counter()
    rep = impl.ir(wl["tw"], wl["tf"], wl["tr"], af, b_host, on_the_fly=wl["on_the_fly"],
                  resid_term=wl["resid_term"], ce=wl["ce"], litmax=wl["litmax"])
    dt = time.perf_counter() - t0
    if ns != n:
        tfac, tsol = rep["t_factor"] or dt, rep["t_solve"] or 0.0
        dt = tfac * scale_f + tsol * scale_s
        sample = (f"one {args.config}-family solve at N={ns} (same operator and parameters) "
                  f"by the compiled reference, factor time x(N/{ns})^3 + solve time "
                  f"x(N/{ns})^2 extrapolated to N={n}; fp32 LU single-threaded "
                  "(mp_structures.hpp:166-167)")
    else:
        sample = (f"one full {args.config} solve (refactor + IR) at N={n}; fp32 LU is "
                  "single-threaded in the reference (mp_structures.hpp:166-167)")
    return dt, {"unit": "s", "cores": 1 if wl["tf"] != 2 else os.cpu_count(), "kind": kind,
                "sample": sample, "iters": len(rep["rhist"]) - 1, "reason": rep["reason"],
                "split_s": {"factor": rep["t_factor"], "solve": rep["t_solve"]}}


def host_residual_check(a_flat, x, b, anorm1):
    """the solution of the N = 65536 system cannot be compared
    with an oracle LU (hours of CPU), so the checker's own compensated
    residual (detail::residual_into, ir_engine.hpp:115-139) is run on the host
    copy of the fp64 matrix and ||r||_inf is held against the reference's
    backward-error rule 10 eps (||b|| + ||A||_1 ||x||). Part of the CPU leg
    (the one place bench.py runs oracle/ code besides the baseline timing)."""
    import numpy as np
    import oracle
    n = x.size
    impl = oracle.reference() or oracle.restatement()
    t0 = time.perf_counter()
    r = impl.residual(0, 0, a_flat.reshape(n, n).T, x, b)
    dt = time.perf_counter() - t0
    rn = float(np.abs(r).max())
    bound = 10.0 * 2.0 ** -52 * (float(np.abs(b).max()) + anorm1 * float(np.abs(x).max()))
    return {"host_residual_inf": rn, "host_residual_bound": bound,
            "host_residual_ok": bool(rn <= bound), "host_residual_seconds": dt}


def cpu_baseline(args, wl, a_host, b_host):
    """The compiled reference (oracle/_ref) on this host: one full solve."""
    try:
        dt, d = reference_solve(args, wl, a_host, b_host)
        d["value"] = dt
        return d
    except Exception as e:  # pragma: no cover
        return {"value": None, "error": str(e)}


def respawn_under_torchrun(args):
    """`python bench.py --gpus N` (N > 1) outside torchrun: start N ranks of this
    script on this node (one process per GPU, NCCL rendezvous on 127.0.0.1)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), "--", os.path.abspath(__file__)] + sys.argv[1:]  # "--": bench's own
    # flags (--n ...) must not be read as abbreviations of torchrun's
    sys.exit(subprocess.call(cmd))


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        respawn_under_torchrun(args)
    world, rank, local = dist_setup(args)
    # N > 1 without an explicit --config: the config that shards,
    # cfg5a's N = 65536 LU in 1-D block-cyclic column blocks over the ranks
    if world > 1 and not args.config_given:
        args.config = "cfg5a"
    if args.config == "cfg5a" and (world > 1 or args.dist) and args.impl == "ours":
        import bench_dist
        line = bench_dist.run_ours(args, world, rank, local)
        if line is not None:
            print(json.dumps(line), flush=True)
    elif args.config == "cfg5b":
        import bench_batch
        if args.impl == "reference":
            bench_batch.run_reference(args, world, rank)
        else:
            bench_batch.run_ours(args, world, rank, local)
    elif args.impl == "reference":
        run_reference(args, world, rank)
    else:
        line = run_ours(args, world, rank, local)
        # The default invocation also times the large single-GPU configs in the
        # same process, so their roofline fractions are driver-timed: cfg4
        # (N = 16384, fp32 LU, pivot-heavy) and cfg3 with the tcgen05 update.
        if (line is not None and world == 1 and not args.config_given and args.n is None
                and args.lu_mode == "exact" and not args.no_also):
            line["also"] = []
            for cfg_name, mode in (("cfg4", "exact"), ("cfg3", "tc")):
                sub = argparse.Namespace(**vars(args))
                sub.config, sub.lu_mode, sub.no_cpu_baseline = cfg_name, mode, True
                sub.steps, sub.warmup = min(args.steps, 3), max(3, min(args.warmup, 3))
                try:
                    extra = run_ours(sub, world, rank, local)
                    for k in ("metric", "data", "clocks", "higher_is_better", "vs_baseline"):
                        extra.pop(k, None)
                    line["also"].append(extra)
                except Exception as e:  # the headline line must survive
                    line["also"].append({"config": {"workload": cfg_name}, "error": repr(e)})
        if line is not None:
            print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
