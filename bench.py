#!/usr/bin/env python
"""bench.py -- GPCG hot-path benchmark (BASELINE.json metric) on B200.

A "step" is one full GPCG solve (Algorithm GPCG: every row of
SURVEY.md 8(a) -- GP sweeps a1/a2/a3, CG a4/a5, reductions a6, control a7) of
the configured workload from x0 to tol, inputs resident in HBM.  Default
workload: C3 (BASELINE.json configs[3], 8000^2 = 64M variables, the north_star's
strong-scaling grid; its working set is far larger than the 126 MB L2, so the
sweeps are measured in the HBM regime).  --config C2 runs the paper-size grid.

  value   = reduced Hessian-vector products per second over the K timed solves
            (one per CG iteration: the masked SpMV A_F rho of the CG sweep),
            aggregated over ranks; solve seconds are reported beside it.
  e2e     = the same metric through the C ABI with HOST (pinned) buffers:
            create (H2D of operator, b, l, u) + solve (H2D x0, D2H x) + destroy.
  roofline: the persistent loop with the larger device time (CG or GP), its
            algorithmic bytes per launch (the bytes THIS kernel's
            algorithm must move -- CG: 48 B per free point + 1 B mask per point;
            GP: the speculative sweep's bytes per point, + search and accept
            sweeps for rejected steps) over its CUDA-event-timed duration; SURVEY
            8(d)'s count and the ncu DRAM bytes (profiles/traffic_<config>.json)
            beside it.
  cpu_baseline / --impl reference: the plain-C oracle (oracle/), unmodified, on
            the same workload: reduced HVPs/s of its textbook CG (ora_cg, the
            masked operator Z Z' A Z Z') for a fixed number of iterations -- the
            same unit of work as `value`, independent of the solve's phase.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl reference] [--slabs S] [--xrank]
N > 1 runs under torchrun (one process per GPU): the SAME problem split into N row
slabs (gpcg_create_*_dist: NCCL halo exchange + one allreduce per CG iteration),
i.e. strong scaling; see DESIGN.md "Multi-GPU".  --slabs S (N = 1) splits the
problem into S slabs on the one GPU (the multi-slab persistent loops with fused halo
writes; device-copy halos between the other sweeps).
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "reduced Hessian-vector products/s and HBM GB/s (% of 8 TB/s); GPCG solve s"
UNIT = "reduced HVP/s"

WORKLOADS = {
    "C0": "C0: journal bearing 50x50 (n=2,500), eps=0.1, l=0, u=inf, x0=0, tol 1e-8*||g(x0)|| [BASELINE.json configs[0]]",
    "C1": "C1: 400x400 (n=160,000) noisy faces, Gaussian b, 40%-active two-sided obstacles [configs[1]]",
    "C2": "C2: journal bearing 1600x1600 (n=2,560,000), eps=0.1, l=0, u=inf, x0=0, tol 1e-8*||g(x0)||, "
          "stencil-specialised masked SpMV, 1 B200 [configs[2]]",
    "C3": "C3: 8000x8000 (n=64,000,000) journal bearing with 50%-active two-sided obstacles [configs[3]]",
    "C4": "C4: 256^3 (n=16,777,216) 7-point lognormal CSR, box [-0.01,0.01] [configs[4]]",
}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy_)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def cg_kernel_name(prob, slabs_total=1, ms=False):
    """The CG-iteration kernel libgpcg.so selects for this problem (gpcg.cu run_cg /
    enqueue_cg_iter); slabs_total > 1: the multi-slab persistent loop (ms: slabs of one device, or ranks
    with --xrank), else graph chunks."""
    compact = prob.kind in ("csr", "stencil3d") and slabs_total == 1   # cg_mode 2 -> 3 for small free sets
    if prob.kind == "csr":
        return "k_cg_iter_c<CsrOp> (free-row list, reduced-space vectors) / k_cg_iter<CsrOp>" if compact \
            else "k_cg_iter<CsrOp>"
    if prob.kind == "stencil3d":
        return "k_cg_iter_c<Stencil3Op> / k7_cg_iter" if compact else "k7_cg_iter"
    bc = not prob.wx_ld and not prob.wy_ld and prob.shift is None
    tile = int(os.environ.get("GPCG_TILE", "127") or 127)
    if os.environ.get("GPCG_GENERIC") == "1":
        return "k_cg_iter<StencilOp>"
    if bc and tile & 8:
        if os.environ.get("GPCG_CG_PERSIST", "1") != "0" and slabs_total == 1:
            return "k6_cg_loop (persistent cooperative CG, TMA-fed column march; per-iteration time)"
        if os.environ.get("GPCG_CG_PERSIST", "1") != "0" and ms:
            return "k6_cg_loop_ms (persistent CG over every slab / rank, fused halo writes; per-iteration time)"
        return "k4_cg_iter (TMA-fed column march)"
    if bc and tile & 4:
        return "k3_cg_iter<2> (TMA tile)"
    return "k2_cg_iter (column march)"


def cg_min_bytes_per_free_point(prob):
    """Bytes the stencil CG kernel's 3-vector recurrence must move per free point (read
    rho, p, w; write rho', p', w' = 48 B; + 16 B of full face arrays for C1-type
    operators) -- its own floor, below the 80 B of SURVEY.md 8(d)."""
    if prob.kind == "stencil2d":
        return 48.0 + (16.0 if (prob.wx_ld or prob.wy_ld) else 0.0)
    return cg_bytes_per_free_point(prob)


def cg_bytes_per_free_point(prob):
    """Algorithmic bytes of one k_cg_iter launch per free point:
    5 fp64 vectors read (rho, q, s, p, w) + 5 written = 80 B, plus operator data
    a free row must read: 0 (broadcast face weights, O(nx) cached), 16 B (full
    face arrays: one x- and one y-face weight per point), CSR 8 B row_ptr +
    12 B per stored entry."""
    if prob.kind == "stencil2d":
        return 80.0 + (16.0 if (prob.wx_ld or prob.wy_ld) else 0.0)
    z = prob.val.size / prob.n
    return 80.0 + 8.0 + 12.0 * z


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.limit")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        sm, smax, reasons, pw, plim, capped = [], [], set(), [], [], 0
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.f.read().splitlines():
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
            capped += parts[8].lower().startswith("active")
            try:
                pw.append(float(parts[3]))
                plim.append(float(parts[9]))
            except (ValueError, IndexError):
                pass
        os.unlink(self.f.name)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(smax)) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons),
                "power_w": float(np.median(pw)) if pw else None,
                "power_limit_w": float(np.median(plim)) if plim else None,
                "sw_power_cap_fraction": capped / len(sm) if sm else None}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def oracle_free_set(prob):
    """The free set the oracle's CG rate is measured on: F = {l < P[x0] < u}, or every point if
    that is empty (C2's x0 = 0 = l) -- the masked operator costs the same per row either way."""
    x = np.minimum(np.maximum(prob.x0, prob.l), prob.u)
    fr = ((x > prob.l) & (x < prob.u)).astype(np.uint8)
    if not fr.any():
        fr[:] = 1
    return x, fr


def oracle_cg_rate(prob, iters, A=None, omp=False):
    """The oracle's reduced-HVP rate: `iters` iterations of its textbook CG (ora_cg, one masked
    SpMV Z Z' A Z Z' p per iteration plus the vector updates) on A_F w = -g_F at P[x0], the
    progress test switched off so every call does exactly `iters` iterations.
    -> (iterations, seconds, threads)."""
    from oracle import oracle as O
    A = O.problem_csr(prob) if A is None else A
    x, fr = oracle_free_set(prob)
    g = O.gradient(A, prob.b, x)
    t0 = time.perf_counter()
    it, w, decs = O.cg(A, fr, g, 1e-300, cap=iters, omp=omp)
    secs = time.perf_counter() - t0
    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)) if omp else 1
    return it, secs, threads


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    """--impl reference: the oracle (plain C, 1 thread) timed on the host, same workload/metric:
    each step = a fixed number of its CG iterations (reduced HVPs) on the workload."""
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    from paper_cs_0101018_b200 import problems as P
    prob = P.get(args.config)
    from oracle import oracle as O
    A = O.problem_csr(prob)                      # assembled once (not part of a step)
    # iterations per step: about min(6 s, 150 s / steps) of oracle work, so warm-up + timed steps
    # stay within a few minutes
    _, s1, _ = oracle_cg_rate(prob, 1, A)
    total = args.steps + args.warmup
    iters = max(1, int(min(6.0, 150.0 / max(total, 1)) / max(s1, 1e-6)))
    for _ in range(args.warmup):
        oracle_cg_rate(prob, iters, A)
    its, secs = 0, 0.0
    for _ in range(args.steps):
        it, sec, _ = oracle_cg_rate(prob, iters, A)
        its += it
        secs += sec
    value = its / secs if secs > 0 else 0.0
    sample = (f"each step: {iters} iterations of the oracle's textbook CG (ora_cg: masked SpMV + vector "
              f"updates) on A_F w = -g_F of {args.config} at P[x0] (F = {int(oracle_free_set(prob)[1].sum())} "
              f"points), progress test off; 1 thread, {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / max(args.steps, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": WORKLOADS[args.config], "n": prob.n},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_cs_0101018_b200 import problems as P
    from paper_cs_0101018_b200 import gpcg

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def fresh_nccl_id():
        """A new ncclUniqueId for every communicator this process creates (an id's bootstrap root
        serves one ncclCommInitRank round): rank 0 draws it, torch.distributed broadcasts it."""
        if world == 1:
            return None
        obj = [gpcg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]
    dev = torch.device("cuda", local)
    prob = P.get(args.config)
    stream = torch.cuda.current_stream()
    if world > 1 or args.slabs > 1:
        solver, rb, re, loc = gpcg.Solver.dist(prob, rank, world, fresh_nccl_id(), local_slabs=args.slabs,
                                               stream=stream, device=dev)
        x0_host = loc["x0"]
    else:
        solver = gpcg.Solver.from_problem(prob, stream=stream, device=dev)
        x0_host = prob.x0
        loc = None
    x0 = torch.from_numpy(np.ascontiguousarray(x0_host)).to(dev)
    x_out = torch.empty_like(x0)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)   # 256 MB > 126 MB L2

    for _ in range(args.warmup):
        solver.solve(x0, prob.tol, x_out=x_out)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    tot_ms = 0.0
    agg = {"cg_iters": 0, "gp_iters": 0, "outer_iters": 0, "kernel_launches": 0, "cg_iters_timed": 0,
           "cg_free_iters_timed": 0, "t_cg_timed_ms": 0.0, "t_cg_ms": 0.0, "t_gp_ms": 0.0,
           "gp_spec_rejected": 0}
    last = None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(args.steps):
        flush.zero_()                                   # L2 flushed between timed solves
        torch.cuda.synchronize()
        e0.record(stream)
        rc, _, st = solver.solve(x0, prob.tol, x_out=x_out)
        e1.record(stream)
        torch.cuda.synchronize()
        tot_ms += e0.elapsed_time(e1)
        assert rc == 0, (rc, st)
        for k in agg:
            agg[k] += st[k]
        last = st
    torch.cuda.synchronize()
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    hvps = float(agg["cg_iters"])       # global reduced HVPs (every rank counts the same iterations)
    if world > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    value = hvps / (tot_ms / 1e3)

    # roofline of the dominant kernel (k_cg_iter), steady-state CUDA-event timing
    peak, peak_src = load_peaks()
    bpp = cg_bytes_per_free_point(prob)
    it_t = max(agg["cg_iters_timed"], 1)
    # per launch of this rank's kernel: the global free count split evenly over ranks
    # the mask is read at every point (1 B), except by the free-row-list CG of CSR / 3-D operators
    # with a small free set (cg_mode 2 -> 3), which reads a 4-B list entry per free row instead
    compact = (prob.kind in ("csr", "stencil3d") and world * args.slabs == 1
               and agg["cg_free_iters_timed"] < 0.3 * prob.n * max(agg["cg_iters_timed"], 1))
    per_pt, per_free = (0.0, 4.0) if compact else (1.0, 0.0)
    bytes_per_launch = ((bpp + per_free) * agg["cg_free_iters_timed"]
                        + per_pt * prob.n * agg["cg_iters_timed"]) / it_t / world
    min_bytes_per_launch = ((cg_min_bytes_per_free_point(prob) + per_free) * agg["cg_free_iters_timed"]
                            + per_pt * prob.n * agg["cg_iters_timed"]) / it_t / world
    launch_s = (agg["t_cg_timed_ms"] / 1e3) / it_t
    achieved = bytes_per_launch / launch_s / 1e9 if agg["cg_iters_timed"] else None
    achieved_min = min_bytes_per_launch / launch_s / 1e9 if agg["cg_iters_timed"] else None
    # ncu DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per CG iteration / per GP step
    # on this config, from one `ncu --set full` capture (profiles/traffic_<config>.json)
    traffic = {}
    tr_path = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tr_path):
        tj = json.load(open(tr_path))
        traffic = {"cg": tj.get("cg", {}).get("dram_bytes_per_launch", tj.get("dram_bytes_per_launch")),
                   "gp": tj.get("gp", {}).get("dram_bytes_per_launch")}

    # e2e: through the C ABI with host (pinned) buffers, H2D/D2H inside the timed region
    def pinned(a):
        return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    # e2e steps: 3, or 1 when a solve takes seconds (C3) so that the default run stays minutes long
    e2e_steps = max(1, min(args.steps, 3 if tot_ms / args.steps < 3000.0 else 1))
    if loc is None:
        hp = P.Problem(**{**prob.__dict__})
        for k in ("b", "l", "u", "x0", "wx", "wy", "shift", "row_ptr", "col", "val"):
            setattr(hp, k, pinned(getattr(prob, k)))
        xh = torch.empty(prob.n, dtype=torch.float64).pin_memory()
        make = lambda: gpcg.Solver.from_problem(hp, stream=stream)             # noqa: E731
        h2d = int(prob.input_bytes())
    else:
        # the rank's slab: local_part slices, pinned; create_*_dist uploads them
        hp = P.Problem(**{**prob.__dict__})
        lp = {k: (pinned(v) if isinstance(v, np.ndarray) else v) for k, v in loc.items()}
        xh = torch.empty(loc["n"], dtype=torch.float64).pin_memory()
        make = lambda: gpcg.Solver.dist(prob, rank, world, fresh_nccl_id(), local_slabs=args.slabs,  # noqa: E731
                                        stream=stream, local=lp)[0]
        h2d = int(sum(v.numel() * v.element_size() for v in lp.values() if hasattr(v, "numel")))
    x0h = pinned(np.ascontiguousarray(x0_host))
    s_e2e = make()                                # warm-up of the e2e path (memory pool, module state)
    s_e2e.close()
    e2e_s, e2e_hvps = 0.0, 0
    t_parts = {"create_s": 0.0, "solve_s": 0.0, "destroy_s": 0.0}
    for _ in range(e2e_steps):
        flush.zero_()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        s2 = make()
        t1 = time.perf_counter()
        rc, _, st2 = s2.solve(x0h, prob.tol, x_out=xh)
        t2 = time.perf_counter()
        s2.close()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        e2e_s += t3 - t0
        t_parts["create_s"] += (t1 - t0) / e2e_steps
        t_parts["solve_s"] += (t2 - t1) / e2e_steps
        t_parts["destroy_s"] += (t3 - t2) / e2e_steps
        e2e_hvps += st2["cg_iters"]
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_val = e2e_hvps / e2e_s

    # the GP phase: one GP step = one speculative accept sweep at alpha_0 (k6_gp_loop, 2-D broadcast
    # faces, one slab) whose bytes per point are those the sweep must move: y read,
    # y and the mask written (17 B; the previous mask is recomputed from y, l, u) + l, u unless both
    # are constants (16 B) + b unless every grid row holds the same b (8 B); g is recomputed, never
    # stored.  A step whose speculative sweep was rejected (stats gp_spec_rejected) also ran a search
    # sweep (y [+ l, u] [+ b]) and an accept sweep (y, mask_prev [+ l, u] [+ b] read; y, mask written).
    gp_roof = None
    if agg["gp_iters"] and prob.kind == "stencil2d":
        sb = bool(np.all(prob.l == prob.l[0]) and np.all(prob.u == prob.u[0]))
        bb = bool(np.all(prob.b.reshape(prob.ny, prob.nx) == prob.b[: prob.nx][None, :]))
        spec_b = 17.0 + (0.0 if sb else 16.0) + (0.0 if bb else 8.0)
        srch_b = 8.0 + (0.0 if sb else 16.0) + (0.0 if bb else 8.0)
        acc_b = spec_b + 1.0
        bc_gp = (not prob.wx_ld and not prob.wy_ld and prob.shift is None
                 and os.environ.get("GPCG_GP_PERSIST", "1") != "0")
        persist = bc_gp and world * args.slabs == 1
        persist_ms = bc_gp and ((world == 1 and args.slabs > 1) or (world > 1 and args.xrank))
        rej = agg["gp_spec_rejected"]
        gp_step_s = (agg["t_gp_ms"] / 1e3) / agg["gp_iters"]
        gp_bytes = (spec_b * agg["gp_iters"] + (srch_b + acc_b) * rej) * prob.n / agg["gp_iters"] / world
        ach = gp_bytes / gp_step_s / 1e9
        gp_roof = {"bound": "hbm",
                   "kernel": ("k6_gp_loop (persistent GP phase; speculative accept sweep per step)" if persist
                              else "k6_gp_loop_ms (persistent GP phase over every slab / rank, fused halo writes)"
                              if persist_ms else "k5_search / k5_accept GP graph chunks"),
                   "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                   "frac_of_8TBs": ach / 8000.0, "traffic": traffic.get("gp"), "peak_source": peak_src,
                   "bytes_per_launch": gp_bytes, "us_per_launch": gp_step_s * 1e6,
                   "launch": "one GP step (sweep(s) + grid reduction + stop tests), CUDA events around each GP phase",
                   "algorithmic_bytes": f"{spec_b:.0f} B per point per speculative sweep (sb={sb}, bb={bb}); "
                                        f"+{srch_b + acc_b:.0f} B per point for each of {rej} rejected steps",
                   "survey_8d": {"bytes_per_launch": (74.0 if sb else 122.0) * prob.n / world,
                                 "frac": (74.0 if sb else 122.0) * prob.n / world / gp_step_s / 1e9 / peak,
                                 "what": "SURVEY 8(d): 3 sweeps per GP sub-step (a2, a3, a1)"}}
        if traffic.get("gp"):
            gp_roof["dram_over_algorithmic"] = traffic["gp"] / gp_bytes
    elif agg["gp_iters"] and prob.kind in ("csr", "stencil3d") and os.environ.get("GPCG_GP_SPEC", "1") != "0":
        # CSR / 3-D GP graph: one GP step = a Cauchy sweep (y, g read) + k_spec (y, g, b read; y', g',
        # mask' written), each reading the operator (CSR: 8 B row_ptr + 12 B per stored entry; 3-D:
        # the face / shift arrays, 48 B per point) and l, u unless both are constants (16 B)
        sb = bool(np.all(prob.l == prob.l[0]) and np.all(prob.u == prob.u[0]))
        op_b = (8.0 + 12.0 * prob.val.size / prob.n) if prob.kind == "csr" else 48.0
        bnd = 0.0 if sb else 16.0
        step_b = (16.0 + op_b + bnd) + (24.0 + op_b + bnd + 17.0)
        gp_step_s = (agg["t_gp_ms"] / 1e3) / agg["gp_iters"]
        gp_bytes = step_b * prob.n / world
        ach = gp_bytes / gp_step_s / 1e9
        gp_roof = {"bound": "hbm", "kernel": "k_cauchy + k_spec (GP graph: Cauchy sweep + speculative h = 0 step)",
                   "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                   "frac_of_8TBs": ach / 8000.0, "traffic": traffic.get("gp"), "peak_source": peak_src,
                   "bytes_per_launch": gp_bytes, "us_per_launch": gp_step_s * 1e6,
                   "launch": "one GP step (Cauchy + k_spec sweeps, reductions, k_gp_step; the phase's no-op "
                             "launches included), CUDA events around each GP phase",
                   "algorithmic_bytes": f"{step_b:.0f} B per point per GP step (operator {op_b:.0f} B, sb={sb}), "
                                        f"every step's speculative sweep kept"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        A_o = O.problem_csr(prob)
        _, s1, _ = oracle_cg_rate(prob, 1, A_o)
        iters = max(2, int(args.cpu_budget / max(s1, 1e-6)))
        it1, sec1, _ = oracle_cg_rate(prob, iters, A_o)
        _, s1o, _ = oracle_cg_rate(prob, 1, A_o, omp=True)
        iters_o = max(2, int(args.cpu_budget / max(s1o, 1e-6)))
        ito, seco, thr = oracle_cg_rate(prob, iters_o, A_o, omp=True)
        del A_o
        nf = int(oracle_free_set(prob)[1].sum())
        cpu = {"value": it1 / sec1, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{it1} iterations of the oracle's textbook CG (ora_cg: masked SpMV Z Z' A Z Z' p + "
                         f"vector updates, progress test off) on A_F w = -g_F of {args.config} at P[x0] "
                         f"(|F| = {nf}), 1 host thread; {cpu_model()}",
               "openmp": {"value": ito / seco, "unit": UNIT, "cores": thr, "nproc": os.cpu_count(),
                          "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS"),
                          "sample": f"{ito} iterations, same call, liboracle_omp.so (the same source with "
                                    f"-fopenmp: row and elementwise loops threaded, sums serial; bitwise-equal "
                                    f"results)"}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, paper_cs_0101018_b200/problems.py)",
            "config": {"workload": WORKLOADS[args.config], "n": prob.n,
                       "l2": "flushed (256 MB write) between timed solves; C3's vectors (512 MB each) exceed "
                             "the 126 MB L2 anyway",
                       "parallelism": ("1 GPU, 1 slab" if world == 1 and args.slabs == 1 else
                                       f"{world} GPU(s) x {args.slabs} row slab(s) of one problem "
                                       + ("(persistent loops across ranks over IPC-mapped peer memory)"
                                          if args.xrank and world > 1 else
                                          "(persistent loops over every slab, fused halo writes)"
                                          if world == 1 else
                                          "(halo exchange + one allreduce per CG iteration)"))},
            "solve": {"s_per_solve": tot_ms / args.steps / 1e3, "outer_iters": last["outer_iters"],
                      "gp_iters": last["gp_iters"], "cg_iters": last["cg_iters"],
                      "n_free": last["n_free"], "q": last["q"], "pg_norm": last["pg_norm"],
                      "tau": last["tau"], "t_cg_share": agg["t_cg_ms"] / tot_ms},
            # achieved: the bytes THIS kernel's algorithm must move per CG iteration (DESIGN.md 6:
            # the three-vector recurrence, 48 B per free point + the 1 B mask per point for stencils;
            # the five-vector C-G form for CSR = SURVEY 8(d)'s figure); SURVEY 8(d)'s 80 B figure
            # (which also streams A p and A rho) beside it -- against that count the kernel exceeds
            # the copy peak, because it recomputes A p and A rho from neighbours instead of streaming them.
            "roofline": {"bound": "hbm", "kernel": cg_kernel_name(prob, world * args.slabs,
                                                                  (world == 1 and args.slabs > 1) or
                                                                  (world > 1 and args.xrank)),
                         "achieved": achieved_min, "peak": peak, "unit": "GB/s",
                         "frac": (achieved_min / peak) if achieved_min else None,
                         "frac_of_8TBs": (achieved_min / 8000.0) if achieved_min else None,
                         "traffic": traffic.get("cg"), "peak_source": peak_src,
                         "bytes_per_launch": min_bytes_per_launch, "us_per_launch": launch_s * 1e6,
                         "dram_over_algorithmic": (traffic["cg"] / min_bytes_per_launch) if traffic.get("cg") else None,
                         "launch": "one CG iteration (reduced HVP + vector updates + reduction)",
                         "algorithmic_bytes": (f"{cg_min_bytes_per_free_point(prob) + per_free:.0f} B per free point "
                                               f"(reduced-space vectors, the free rows of A, the list entry)"
                                               if compact else
                                               f"{cg_min_bytes_per_free_point(prob):.0f} B per free point + 1 B mask "
                                               f"per point (DESIGN.md 6: the kernel's three-vector recurrence)"),
                         "survey_8d": {"bytes_per_launch": bytes_per_launch, "achieved": achieved,
                                       "frac": (achieved / peak) if achieved else None,
                                       "what": f"{bpp:.0f} B per free point + 1 B mask per point (SURVEY.md 8(d) "
                                               f"fused C-G CG iteration, 5 vectors; this kernel recomputes A p and "
                                               f"A rho from neighbours instead of streaming them)"}},
            "roofline_gp": gp_roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": UNIT,
                    "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": int(x0.numel() * 8),
                    "what": "gpcg_create (H2D operator,b,l,u from pinned host) + gpcg_solve (H2D x0, "
                            "D2H x) + gpcg_destroy, wall clock, %d steps" % e2e_steps,
                    "per_step": t_parts},
            "gpu_launches": agg["kernel_launches"],
            "clocks": clk,
        }
        # `roofline` is the kernel with the larger device time in the timed solves (CUDA events: the
        # CG calls vs the GP phases); the other persistent loop goes to `roofline_other`
        t_cg, t_gp = agg["t_cg_ms"], agg["t_gp_ms"]
        cg_roof, gp_roof_ = line.pop("roofline"), line.pop("roofline_gp")
        if cg_roof is not None:
            cg_roof["device_time_share"] = t_cg / max(tot_ms, 1e-9)
        if gp_roof_ is not None:
            gp_roof_["device_time_share"] = t_gp / max(tot_ms, 1e-9)
        if gp_roof_ is not None and t_gp > t_cg:
            line["roofline"], line["roofline_other"] = gp_roof_, cg_roof
        else:
            line["roofline"], line["roofline_other"] = cg_roof, gp_roof_
        print(json.dumps(line), flush=True)
    solver.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--slabs", type=int, default=1)
    ap.add_argument("--xrank", action="store_true",
                    help="N > 1: the persistent loops span the ranks over IPC-mapped peer memory (GPCG_XRANK=1; "
                         "DESIGN.md 8) instead of NCCL graph chunks")
    args = ap.parse_args()
    if args.xrank:
        os.environ["GPCG_XRANK"] = "1"      # read at create
    if args.impl == "reference":
        return run_reference(args)
    from paper_cs_0101018_b200 import _build
    _build.build()
    try:
        return run_ours(args)
    except Exception as e:          # one JSON line that says what failed, instead of none
        if int(os.environ.get("RANK", "0")) == 0:
            print(json.dumps({"metric": METRIC, "value": None, "unit": "reduced HVP/s", "n_gpus": args.gpus,
                              "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
                              "config": {"workload": args.config}, "error": f"{type(e).__name__}: {e}"[:400]}),
                  flush=True)
        raise


if __name__ == "__main__":
    sys.exit(main())
