"""IFGF matvec benchmark (BASELINE.json metric: matvec time & Mpoints/s).

One step = one full operator application as the reference defines it
(ifgf::apply, engine.cpp:260-325): Problem::build (octree + relevant cones) on
the device from device-resident coordinates, then the matvec on
device-resident densities.  `value` = N / step time in Mpoints/s, timed with
CUDA events on the caller stream (the library orders itself after it), L2
flushed between steps.  `e2e` = the same operator through the C ABI
(ifgf_apply) from pinned host buffers, H2D/D2H included.  `apply_only` =
plan reused, matvec only (the iterative-solver case).

Default workload: BASELINE configs[1] (C2, N=1,572,864 sphere, kappa=32pi,
(3,5,5)) on one GPU.  --impl reference times the reference's own CPU
implementation (oracle/_ref, compiled from the reference sources) on a bounded
sample of the same workload with all host threads.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "IFGF matvec throughput (Mpoints/s; N / full apply time incl. device setup)"
UNIT = "Mpoints/s"
# Bounded CPU sample of C2: the same surface and points-per-wavelength density
# at 1/16 of the points (N = 98,304, kappa = 8 pi, i.e. BASELINE configs[0]).
REF_SAMPLE_N = 98_304


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    # the N>1 code path (rank engine + NCCL) at any N, e.g. N=1 on a one-GPU box
    ap.add_argument("--dist", action="store_true")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    # seconds between NVML polls; each poll takes the driver's lock, which the
    # device setup's allocations and syncs then wait on
    INTERVAL = float(os.environ.get("IFGF_CLOCK_INTERVAL", "0.1"))

    def __init__(self, index):
        self.index, self.rows, self._stop = index, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        # NVML in-process (no fork/exec of nvidia-smi inside the timed region)
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            bits = (N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                    N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap)
            while not self._stop.is_set():
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
                pw = N.nvmlDeviceGetPowerUsage(h) / 1e3
                rs = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append([str(sm), str(mx), f"{pw:.1f}", hex(rs)]
                                 + ["Active" if rs & b else "Not Active" for b in bits])
                self._stop.wait(self.INTERVAL)
            return
        except Exception:
            self.rows = []
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 4 + k and r[4 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def load_configs():
    """paper_2112_15198_b200/configs.py loaded by path: the reference leg must
    not import the product package (that would map libifgf_b200.so)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "ifgf_configs", os.path.join(ROOT, "paper_2112_15198_b200", "configs.py"))
    m = importlib.util.module_from_spec(spec)
    sys.modules["ifgf_configs"] = m
    spec.loader.exec_module(m)
    return m


def ref_checker():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from bindings import REF_SO, COracle, Params, RefOracle  # test infra: CPU legs only
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    if os.path.exists(REF_SO):
        return RefOracle(), COracle(), Params(threads=cores), "reference", cores
    return COracle(), COracle(), Params(threads=cores), "port", cores


def cpu_sample_run(steps, warmup):
    """cpu_baseline leg of our arm (rank 0, N=1): the reference's full apply
    (setup + passes) on a bounded sample -- C2's surface and
    points-per-wavelength^2 density at N=98,304 (BASELINE configs[0]);
    seconds per apply.  The like-for-like C2 number is --impl reference."""
    configs = load_configs()
    cfg = configs.scaled(configs.C2, REF_SAMPLE_N)
    chk, gen, params, kind, cores = ref_checker()
    x1, x2, x3, ar, ai = gen.generate(cfg.n, cfg.shape, cfg.c, cfg.dens, cfg.seed)
    if kind == "port":
        gen.lib.oc_set_threads(cores)
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        chk.apply(x1, x2, x3, ar, ai, cfg.kind, cfg.kappa, params)
        if i >= warmup:
            times.append(time.perf_counter() - t0)
    sample = (f"full reference apply (setup+passes) on C2's surface and density at "
              f"N={cfg.n:,} (kappa={cfg.kappa / math.pi:g}pi = BASELINE configs[0]), "
              f"IFGF_SIMD={os.environ.get('IFGF_SIMD', 'avx2')}")
    return cfg.n, times, kind, cores, sample


# reference leg: slices per full matvec (each step runs 1/REF_SLICES of every
# pass; REF_SLICES consecutive steps are exactly one C2 matvec minus setup)
REF_SLICES = int(os.environ.get("IFGF_REF_SLICES", "10"))


def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    reference library compiled from its sources) on OUR arm's workload -- C2
    at full N, all host threads.  Problem::build (single-threaded in the
    reference, ~3 min at C2) runs once outside timing and is reported as
    setup_s; each step then runs the stock passes of apply()
    (engine.cpp:270-315) over slice (step mod S) of their work ranges.  value
    = N / (S x mean step): the apply-only rate, so the driver's ratio against
    our full step (setup included) is a lower bound."""
    rank, _, world = dist_env()
    if rank != 0:
        return
    configs = load_configs()
    cfg = configs.CONFIGS[args.config]
    chk, gen, params, kind, cores = ref_checker()
    x1, x2, x3, ar, ai = gen.generate(cfg.n, cfg.shape, cfg.c, cfg.dens, cfg.seed)
    if kind != "reference":
        raise SystemExit("bench --impl reference: oracle/_ref missing (build on the host with "
                         "/root/reference: python -c 'import __graft_entry__ as g; g.build()')")
    S = max(1, REF_SLICES)
    t0 = time.perf_counter()
    prob = chk.problem(x1, x2, x3, ar, ai, cfg.kind, cfg.kappa,
                       type(params)(depth=cfg.depth, threads=cores))
    setup_s = time.perf_counter() - t0
    depth = prob.depth
    b = prob.bench()
    times, stages = [], {}
    for i in range(args.warmup + args.steps):
        t1 = time.perf_counter()
        st = b.slice(cores, i % S, S)
        dt = time.perf_counter() - t1
        if i >= args.warmup:
            times.append(dt)
            for k, v in st.items():
                stages[k] = stages.get(k, 0.0) + v
    t_matvec = S * statistics.mean(times)
    v = cfg.n / t_matvec / 1e6
    sample = (f"{cfg.name} at full N={cfg.n:,}: the reference's stock passes (apply() minus "
              f"Problem::build) in {S} slices per matvec, {cores} threads, "
              f"IFGF_SIMD={os.environ.get('IFGF_SIMD', 'avx2')}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_matvec * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, DESIGN.md Inputs)",
        "config": {"workload": f"{cfg.label} (BASELINE configs[1]), orders (3,5,5), "
                               f"depth {depth}",
                   "n": cfg.n, "kappa": cfg.kappa, "orders": [3, 5, 5], "depth": depth,
                   "step": f"1/{S} of the reference's apply() passes (rotating slice); "
                           f"ms_per_step = {S} slices = one matvec minus setup"},
        "setup_s": setup_s,
        "full_apply_ms": (setup_s + t_matvec) * 1e3,
        "stages_ms": {k: v2 * 1e3 * S / len(times) for k, v2 in stages.items()},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": sample, "setup_s": setup_s},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_ours(args):
    import numpy as np
    import torch

    import paper_2112_15198_b200 as ifgf
    from paper_2112_15198_b200 import _lib
    from paper_2112_15198_b200.work import count_work

    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    if not ifgf.device_ok():
        raise SystemExit("bench: no usable sm_100 device: " + _lib.last_error())
    cfgd = ifgf.configs.CONFIGS[args.config]
    kcfg = ifgf.KernelConfig(ifgf.KernelKind(cfgd.kind), cfgd.kappa)
    params = ifgf.EngineParams(depth=cfgd.depth, device=local)
    n = cfgd.n
    # each rank owns a full replica (the distributed path lands in dist.py)
    pc = ifgf.generate(n, cfgd.shape, cfgd.c, cfgd.dens, cfgd.seed + 1000 * rank)
    dev = torch.device("cuda", local)
    X = [torch.from_numpy(a).to(dev) for a in (pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im)]
    out = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(2)]
    flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
    s = torch.cuda.Stream(device=dev)
    sh = s.cuda_stream

    def step():
        plan = ifgf.Plan.from_device(X[0].data_ptr(), X[1].data_ptr(), X[2].data_ptr(), n, kcfg,
                                     params, stream=sh)
        rep = plan.apply_device(X[3].data_ptr(), X[4].data_ptr(), out[0].data_ptr(),
                                out[1].data_ptr(), stream=sh)
        # our kernels in this step: setup (plan) + apply; CUB sort/scan launches excluded
        rep.gpu_launches += int(plan.info.setup_launches)
        plan.close()
        return rep, None

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # ---- full operator (setup + apply), device-resident inputs
    for _ in range(args.warmup):
        step()
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    reps = []
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            with torch.cuda.stream(s):
                flush.zero_()
            ev[i][0].record(s)
            reps.append(step()[0])
            ev[i][1].record(s)
        torch.cuda.synchronize()
    barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_step = sum(step_ms) / len(step_ms) / 1e3
    if world > 1:
        tt = torch.tensor([t_step], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_step = float(tt.item())

    # ---- apply only (plan reuse), and an exclusive per-pass timing run
    plan = ifgf.Plan.from_device(X[0].data_ptr(), X[1].data_ptr(), X[2].data_ptr(), n, kcfg,
                                 params, stream=sh)
    for _ in range(2):
        plan.apply_device(X[3].data_ptr(), X[4].data_ptr(), out[0].data_ptr(),
                          out[1].data_ptr(), stream=sh)
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    for i in range(args.steps):
        with torch.cuda.stream(s):
            flush.zero_()
        ev2[i][0].record(s)
        arep = plan.apply_device(X[3].data_ptr(), X[4].data_ptr(), out[0].data_ptr(),
                                 out[1].data_ptr(), stream=sh)
        ev2[i][1].record(s)
    torch.cuda.synchronize()
    t_apply = statistics.mean(a.elapsed_time(b) for a, b in ev2) / 1e3

    # ---- batched right-hand sides (ifgf_plan_apply_batch, plan reused)
    nrhs = 4
    XB = [torch.stack([X[3]] * nrhs).contiguous(), torch.stack([X[4]] * nrhs).contiguous()]
    OB = [torch.empty((nrhs, n), dtype=torch.float64, device=dev) for _ in range(2)]
    for _ in range(2):
        plan.apply_batch_device(nrhs, XB[0].data_ptr(), XB[1].data_ptr(), OB[0].data_ptr(),
                                OB[1].data_ptr(), stream=sh)
    ev3 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(max(2, args.steps // 2))]
    for a, b in ev3:
        with torch.cuda.stream(s):
            flush.zero_()
        a.record(s)
        plan.apply_batch_device(nrhs, XB[0].data_ptr(), XB[1].data_ptr(), OB[0].data_ptr(),
                                OB[1].data_ptr(), stream=sh)
        b.record(s)
    torch.cuda.synchronize()
    t_batch = statistics.mean(a.elapsed_time(b) for a, b in ev3) / 1e3
    batch = {"nrhs": nrhs, "value": nrhs * n / t_batch / 1e6, "unit": "Mpoints*rhs/s",
             "ms_per_batch": t_batch * 1e3, "ms_per_rhs": t_batch * 1e3 / nrhs,
             "note": "setup shared, passes per rhs (kernel-level batching measured: no gain, "
                     "DESIGN.md section 9)"}
    del XB, OB
    plan.set_serial(True)
    serial = []
    for _ in range(3):
        with torch.cuda.stream(s):
            flush.zero_()
        serial.append(plan.apply_device(X[3].data_ptr(), X[4].data_ptr(), out[0].data_ptr(),
                                        out[1].data_ptr(), stream=sh))
    torch.cuda.synchronize()
    work = count_work(plan)
    info = plan.info
    plan.close()

    # ---- measured FP64 peak (not in MEASURED_PEAKS.json)
    import ctypes as C
    pk, pk_ms = C.c_double(), C.c_double()
    ifgf.engine.check(_lib.lib.ifgf_measure_fp64_peak(local, C.byref(pk), C.byref(pk_ms)))
    fp64_peak = pk.value

    # ---- e2e through the C ABI from pinned host buffers
    e2e = None
    if not args.no_e2e:
        host = [torch.from_numpy(a).pin_memory().numpy() for a in
                (pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im)]
        hout = [torch.empty(n, dtype=torch.float64).pin_memory().numpy() for _ in range(2)]
        hpc = ifgf.PointCloud(*host)
        et = []
        for i in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rc = _lib.lib.ifgf_apply(n, _lib.ptr(hpc.x1), _lib.ptr(hpc.x2), _lib.ptr(hpc.x3),
                                     _lib.ptr(hpc.a_re), _lib.ptr(hpc.a_im), int(kcfg.kind),
                                     float(kcfg.wavenumber), C.byref(params.c()),
                                     _lib.ptr(hout[0]), _lib.ptr(hout[1]), None)
            ifgf.engine.check(rc)
            if i >= args.warmup:
                et.append(time.perf_counter() - t0)
        te = statistics.mean(et)
        if world > 1:
            tt = torch.tensor([te], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": world * n / te / 1e6, "unit": UNIT, "h2d_bytes_per_step": 5 * n * 8,
               "d2h_bytes_per_step": 2 * n * 8, "ms_per_step": te * 1e3,
               "api": "ifgf_apply (C ABI, pinned host buffers)"}

    # ---- roofline of the dominant kernel (exclusive serial timings)
    fl = work.flops
    st = {k: statistics.median(getattr(r.seconds, k) for r in serial)
          for k in ("singular", "level_d", "interpolation", "propagation")}
    stage_key = {"near": "singular", "level_d": "level_d", "interpolation": "interpolation",
                 "propagation": "propagation"}
    per_kernel = {}
    for k, sk in stage_key.items():
        t = st[sk]
        per_kernel[k] = {"ms": t * 1e3, "gflop": fl[k] / 1e9,
                         "tflops": fl[k] / t / 1e12 if t > 0 else None,
                         "frac_fp64": (fl[k] / t / 1e12) / fp64_peak if t > 0 else None}
    dom = max(per_kernel, key=lambda k: per_kernel[k]["ms"])
    traffic = None
    summ = os.path.join(ROOT, "profiles", "ncu_summary.json")
    kernel_prefix = {"near": "k_near", "level_d": "k_level_d",
                     "interpolation": "k_interp", "propagation": "k_propagate"}[dom]
    if os.path.exists(summ):
        try:
            # mean DRAM bytes over every launch of the stage's kernels in one
            # captured C2 apply (K3: the four tiled levels and the fly level)
            ls = json.load(open(summ)).get("launches", [])
            hits = [l["dram_read_bytes"] + l["dram_write_bytes"] for l in ls
                    if l["kernel"].startswith(kernel_prefix)]
            traffic = statistics.mean(hits) if hits else None
        except Exception:
            traffic = None
    dk = per_kernel[dom]
    roofline = {"bound": "fp64", "kernel": dom, "achieved": dk["tflops"], "peak": fp64_peak,
                "traffic_note": "mean DRAM bytes per launch of the dominant stage's kernels over "
                                "one C2 apply (ncu dram__bytes_read/write; profiles/ncu_summary.json)",
                "unit": "TFLOP/s", "frac": dk["frac_fp64"], "traffic": traffic,
                "peak_source": "measured in this run: best of DFMA chains and mma.sync m8n8k4 f64 "
                               "over all SMs (ifgf_measure_fp64_peak); MEASURED_PEAKS.json has no FP64 figure",
                "per_kernel": per_kernel,
                "whole_apply_frac": work.total_flops / t_apply / 1e12 / fp64_peak,
                # the fractions are ALGORITHMIC work rates (SURVEY.md 8(d)
                # weights, sincos = 36 flop).  The row kernel reads each node's
                # transfer factor precomputed and K4/K1 use the 12-op table sincos,
                # so the FP64 work actually executed per propagation evaluation
                # is ~380 flop (186 FMA contraction + 4 FMA transfer), not 430.
                # The warp GEMM (fine levels) executes 2 x 80 MMA FMAs per node
                # slot, 89 % of the slots filled: ~360 flop + transfer per
                # evaluation, the same ballpark.
                "flop_model": "algorithmic (SURVEY.md 8(d)); executed ~380 of the 430 "
                              "flop per propagation evaluation (rows; warp GEMM ~370); K4 from the "
                              "plan's locate records executes ~380 of its 429 per evaluation in the "
                              "apply (the kernel factor is computed once, by the setup)",
                "frac_executed_estimate": (dk["frac_fp64"] * 380.0 / 430.0
                                           if dom == "propagation" else None)}

    # ---- setup (Problem::build) against the HBM roofline.
    # Algorithmic bytes: coordinates read for the bounding
    # cube (24 N), Morton keys (36 N), two sort passes (48 N), the sorted
    # gather (52 N), per level the points' box ordinals and coordinates read
    # once by the clause-1 marking (28 N per level), and 2 x 8 B per relevant
    # cone for the bitmap compaction.  The setup is bound by the clause-1
    # locates (one per (point, cousin box) and level, the same count as K4's
    # evaluations), not by HBM: this fraction documents that.
    t_setup = max(t_step - t_apply, 1e-9)
    hbm_peak = None
    try:
        hbm_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        hbm_peak = 6525.6  # B200_PROFILING.md fallback
    n_cones = sum(info.cones[d] for d in range(3, info.depth + 1))
    # plans that keep K4's locate records write them once during the setup
    # (44 B per (point, cousin) pair at kappa > 0): counted as setup bytes
    rec_bytes = int(info.k4_record_bytes)
    setup_bytes = (24 + 36 + 48 + 52 + 28 * info.depth) * n + 16 * n_cones + rec_bytes
    setup_roofline = {"bound": "locate compute (clause 1: one full-precision locate per (point, "
                               "cousin) pair, stored for K4 when the records fit)",
                      "ms": t_setup * 1e3, "k4_record_bytes": rec_bytes,
                      "k4_record_pairs": int(info.k4_record_pairs),
                      "algorithmic_bytes": setup_bytes,
                      "achieved_GBps": setup_bytes / t_setup / 1e9, "peak_GBps": hbm_peak,
                      "frac_hbm": setup_bytes / t_setup / 1e9 / hbm_peak,
                      "clause1_locates": int(sum(work.interp_evals.values())),
                      "clause1_locates_per_s": sum(work.interp_evals.values()) / t_setup,
                      "peak_source": "MEASURED_PEAKS.json hbm_gbs"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cn, ct, kind, cores, sample = cpu_sample_run(1, 0)
        cpu = {"value": cn / statistics.mean(ct) / 1e6, "unit": UNIT, "cores": cores,
               "kind": kind, "sample": sample, "seconds": statistics.mean(ct)}

    if rank == 0:
        r0 = reps[-1]
        line = {
            "metric": METRIC, "value": world * n / t_step / 1e6, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, DESIGN.md Inputs)",
            "config": {"workload": f"{cfgd.label} (BASELINE configs[1]), orders (3,5,5), "
                                   f"depth {info.depth}",
                       "n": n, "kappa": cfgd.kappa, "orders": [3, 5, 5], "depth": info.depth,
                       "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
                       "l2": "flushed between steps (256 MB write)",
                       "step": "Problem::build on device + apply (device-resident inputs)"},
            "apply_only": {"value": world * n / t_apply / 1e6, "unit": UNIT,
                           "ms_per_step": t_apply * 1e3,
                           "stages_ms_overlapped": {k: getattr(arep.seconds, k) * 1e3 for k in
                                                    ("singular", "level_d", "interpolation",
                                                     "propagation")},
                           "stages_ms_serial": {k: v * 1e3 for k, v in st.items()}},
            "setup_ms": (t_step - t_apply) * 1e3,
            "setup_roofline": setup_roofline,
            "apply_batch": batch,
            "gpu_launches": int(r0.gpu_launches),
            "e2e": e2e,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
            "work": work.as_dict(),
            "step_ms_all": step_ms,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_ours_dist(args):
    """N > 1: C2 split across N GPUs (strong scaling) by the C++ rank engine
    (csrc/dist.cu): one process per GPU, NCCL communicator over NVLink;
    every rank builds the structure (replicated setup) and owns its Morton
    interval of points and its cone intervals per level; per-level halo
    exchanges of cone-segment blocks (dist.cpp:241-361).  One step = the rank
    plan build (setup + exchange lists, collective) + the distributed apply
    (full result in the caller's order on every rank), device-resident
    inputs; e2e adds the host copies of the inputs and the result."""
    import torch
    import torch.distributed as dist

    import paper_2112_15198_b200 as ifgf
    from paper_2112_15198_b200.dist import Comm, DistPlan, max_over_ranks, share_comm_id

    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    if not ifgf.device_ok():
        raise SystemExit("bench: no usable sm_100 device: " + ifgf._lib.last_error())
    cfgd = ifgf.configs.CONFIGS[args.config]
    kcfg = ifgf.KernelConfig(ifgf.KernelKind(cfgd.kind), cfgd.kappa)
    params = ifgf.EngineParams(depth=cfgd.depth, device=local)
    n = cfgd.n
    pc = ifgf.generate(n, cfgd.shape, cfgd.c, cfgd.dens, cfgd.seed)
    comm = Comm(share_comm_id(Comm.unique_id), rank, world, local)
    X = [torch.from_numpy(a).to(dev) for a in (pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im)]
    out = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(2)]
    flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device=dev)
    s = torch.cuda.Stream(device=dev)
    sh = s.cuda_stream
    info = {}

    def step():
        plan = DistPlan(comm, X[0].data_ptr(), X[1].data_ptr(), X[2].data_ptr(), n, kcfg, params,
                        stream=sh)
        rep = plan.apply_device(X[3].data_ptr(), X[4].data_ptr(), out[0].data_ptr(),
                                out[1].data_ptr(), stream=sh)
        if not info:
            ri = plan.info()
            info["rank"] = ri
            info["launches"] = int(plan.plan_info().launches)
        plan.close()
        return rep

    def barrier():
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            with torch.cuda.stream(s):
                flush.zero_()
            ev[i][0].record(s)
            step()
            ev[i][1].record(s)
        torch.cuda.synchronize()
    barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_step = max_over_ranks(statistics.mean(step_ms) / 1e3, device=dev)

    # apply only (rank plan reused)
    plan = DistPlan(comm, X[0].data_ptr(), X[1].data_ptr(), X[2].data_ptr(), n, kcfg, params,
                    stream=sh)
    for _ in range(2):
        plan.apply_device(X[3].data_ptr(), X[4].data_ptr(), out[0].data_ptr(),
                          out[1].data_ptr(), stream=sh)
    barrier()
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    for i in range(args.steps):
        with torch.cuda.stream(s):
            flush.zero_()
        ev2[i][0].record(s)
        plan.apply_device(X[3].data_ptr(), X[4].data_ptr(), out[0].data_ptr(),
                          out[1].data_ptr(), stream=sh)
        ev2[i][1].record(s)
    torch.cuda.synchronize()
    t_apply = max_over_ranks(statistics.mean(a.elapsed_time(b) for a, b in ev2) / 1e3,
                             device=dev)
    plan.close()

    # e2e: pinned host inputs in, result out, every step
    e2e = None
    if not args.no_e2e:
        host = [torch.from_numpy(a).pin_memory() for a in (pc.x1, pc.x2, pc.x3, pc.a_re, pc.a_im)]
        hout = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(2)]
        et = []
        for i in range(args.warmup + args.steps):
            barrier()
            t0 = time.perf_counter()
            with torch.cuda.stream(s):
                for d_, h_ in zip(X, host):
                    d_.copy_(h_, non_blocking=True)
            step()
            with torch.cuda.stream(s):
                hout[0].copy_(out[0], non_blocking=True)
                hout[1].copy_(out[1], non_blocking=True)
            s.synchronize()
            if i >= args.warmup:
                et.append(time.perf_counter() - t0)
        te = max_over_ranks(statistics.mean(et), device=dev)
        e2e = {"value": n / te / 1e6, "unit": UNIT, "h2d_bytes_per_step": 5 * n * 8,
               "d2h_bytes_per_step": 2 * n * 8, "ms_per_step": te * 1e3,
               "api": "ifgf_dist_plan_create_device + ifgf_dist_plan_apply_device (C ABI), "
                      "pinned host buffers, every rank"}
    ri = info.get("rank")
    halo = None
    if ri is not None:
        halo = {"rank0_block_bytes": ri.block_bytes,
                "rank0_levels": [{k: lv[k] for k in ("d", "owned_cones", "halo_cones")}
                                 for lv in ri.levels]}
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": n / t_step / 1e6, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, DESIGN.md Inputs)",
            "config": {"workload": f"{cfgd.label} (BASELINE configs[1]) split over {world} GPUs",
                       "n": n, "kappa": cfgd.kappa, "orders": [3, 5, 5],
                       "parallelism": f"rank layout dist.cpp:78-130 x{world}, NCCL halo exchange",
                       "l2": "flushed between steps (256 MB write)",
                       "step": "rank plan build (replicated setup + exchange lists) + "
                               "distributed apply, device-resident inputs"},
            "apply_only": {"value": n / t_apply / 1e6, "unit": UNIT, "ms_per_step": t_apply * 1e3},
            "setup_ms": (t_step - t_apply) * 1e3,
            "partition": halo,
            "e2e": e2e, "gpu_launches": info.get("launches", 0), "roofline": None,
            "cpu_baseline": None, "clocks": clocks.summary(), "step_ms_all": step_ms,
        }), flush=True)
    comm.close()
    dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif dist_env()[2] > 1 or args.dist:
        run_ours_dist(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
