#!/usr/bin/env python
"""Benchmark: full SE potential (real space + Fourier space + self term),
particles/s, on BASELINE.json configs[1] ("cfg2"): triply periodic, fp64,
N = 1,000,000 neutral charges uniform in a cube L = 10, ES (Barnett-Magland)
window P = 8, beta = 2.5 P = 20, M = 128^3, rc = 1.0, xi = sqrt(-ln 1e-8)/rc.
Synthetic seeded inputs (seed = config number).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One process per GPU (torchrun for N > 1).  A step is one total-potential
evaluation of all N particles (strong scaling over ranks: each rank owns a
share of every stage and the grid / potentials are sum-all-reduced over
NCCL).  `value` times device-resident inputs with CUDA events per step
(L2 flushed between steps, outside the events), max over ranks; `e2e` times
the public API (core.total_potential) on pinned host arrays, H2D / D2H
inside.  `--impl reference` times the CPU port of the reference
(oracle/se_oracle.py; the Python reference itself cannot travel to the GPU
box) on bounded samples with all host threads.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

sys.path.insert(0, os.path.join(ROOT, "tools"))
import workloads  # noqa: E402  (seeded BASELINE configs)

FLOP_PER_PAIR = 40  # SURVEY 8d constant per EVALUATED pair: erfc(xi r)/r ~ exp + rational + sqrt + div + fma
DESCR = {
    "cfg1": "cfg1: D=3, N=2000 uniform in L=1, Gaussian P=16, M=32^3, rc=0.3, xi=12.94",
    "cfg2": "cfg2: D=3, N=1e6 uniform in L=10, ES P=8 beta=20, M=128^3, rc=1.0, xi=4.2919",
    "cfg3": "cfg3 (as worded): D=2, N=2e5 in L=5, ES P=8, M=96^2 x 104, s0=4, s=2, nI=10, xi=6",
    "cfg3_tol": "cfg3 (tolerance-meeting): D=2, N=2e5 in L=5, ES P=10, s0=4, s=4, nI=48, xi=6",
    "cfg4": "cfg4: D=1 (cubic embedding L=8 of 4x4x8), N=2e5, Gaussian P=12, M=128, xi=4, s0=2.4674, nI=39",
    "cfg5": "cfg5: D=0, N=5e5 (ball + 32 Gaussian clusters) in L=4, ES P=10 beta=25, M=96, xi=6, kernel path",
    "cfg1_tol": "cfg1 (tolerance-meeting): D=3, N=2000 in L=1, Gaussian P=16, M=40^3, rc=0.3, xi=14.31",
    "cfg2_tol": "cfg2 (tolerance-meeting): D=3, N=1e6 in L=10, ES P=10 beta=25, M=128^3, rc=1.0, xi=4.2919",
    "cfg4_tol": "cfg4 (tolerance-meeting): D=1 (cubic embedding L=8), N=2e5, Gaussian P=16, M=128, xi=4, nI=39",
}
CFG = {}


def load_workload(name):
    w = workloads.ALL[name]()
    CFG.clear()
    CFG.update(w["prm"])
    CFG.update(workload=name, D=w["D"], L=w["L"], N=len(w["q"]), seed=int(name[3]), eps_target=w["prm"]["eps"])
    CFG["_pos"], CFG["_q"] = w["pos"], w["q"]
    return w


def metric():
    return (f"particles/sec, full SE potential ({DESCR[CFG['workload']]}, fp64)")


def make_inputs():
    return CFG["_pos"], CFG["_q"]


def se_params():
    from paper_1712_04732_b200 import SEParams
    keys = ("xi", "rc", "M", "P", "window", "shape", "s0", "s", "nI", "R", "eps")
    return SEParams(**{k: CFG[k] for k in keys if k in CFG})


def peaks():
    """Roofline denominators: MEASURED_PEAKS.json (HBM) + our fp64 / smem
    micro-benchmarks (profiles/peaks_r02.json, tools/peaks.cu).  The fp64
    peak is the larger of the measured DFMA and DMMA rates (the conservative
    denominator: the DFMA micro-benchmark measured below the DMMA one)."""
    out = {"hbm_gbs": 6655.0, "hbm_src": "fallback (B200_PROFILING.md)",
           "fp64_tflops": 37.0, "fp64_src": "fallback (datasheet ~37-40 TF/s)",
           "smem_tbs": None, "redg_gops": None}
    try:
        m = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        out["hbm_gbs"], out["hbm_src"] = float(m["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        pass
    try:
        pp = os.path.join(ROOT, "profiles", "peaks_r02.json")
        if not os.path.exists(pp):
            pp = os.path.join(ROOT, "profiles", "r01", "peaks_r01.json")
        p = json.load(open(pp))
        out["fp64_tflops"] = max(float(p["fp64_fma_tflops"]), float(p.get("fp64_dmma_tflops", 0.0)))
        out["fp64_src"] = (f"measured ({os.path.relpath(pp, ROOT)}: max of DFMA {p['fp64_fma_tflops']} and "
                           f"DMMA {p.get('fp64_dmma_tflops')} TF/s)")
        out["smem_tbs"] = float(p["smem_tbs"])
        out["redg_gops"] = float(p["redg_f64_gops"])
    except Exception:
        pass
    return out


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region.

    One nvidia-smi process per measurement, started BEFORE the warm-up (its
    start-up takes longer than a short timed region) and read by a thread
    that stamps every sample on arrival; `mark()` opens the timed window,
    leaving the `with` block closes it, and only samples that arrived inside
    the window are summarised."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index, period_ms=50):
        self.index = index
        self.period_ms = period_ms
        self.proc = None
        self.samples = []  # (arrival time, line)
        self.t0 = None
        self.t1 = None

    def _read(self):
        try:
            for l in self.proc.stdout:
                if l.strip():
                    self.samples.append((time.perf_counter(), l))
        except Exception:
            pass

    def __enter__(self):
        import threading
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True, bufsize=1)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def mark(self):
        """The timed region starts now."""
        self.t0 = time.perf_counter()

    def __exit__(self, *exc):
        self.t1 = time.perf_counter()
        if self.proc is not None:
            # one more period, so that a sample taken inside a region shorter
            # than the period still arrives (it is stamped on arrival)
            time.sleep(1e-3 * self.period_ms)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                pass
            self.thread.join(timeout=2)
        t0 = self.t0 if self.t0 is not None else -1.0
        self.lines = [l for (t, l) in self.samples if t0 <= t <= self.t1 + 1e-3 * self.period_ms]

    def summary(self):
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except Exception:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------ CPU baselines

def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import se_oracle
    return se_oracle


def cpu_sample(pos, q, threads=1, n_cells=2, n_kspace=20000, seed=0):
    """The reference's CPU path (its port, oracle/se_oracle.py) timed on a
    BOUNDED sample of the workload: real space for every target of
    `n_cells` random occupied rc-cells (the reference's per-home-cell dense
    blocks, realspace.py:100-126), spread + gather of `n_kspace` particles
    (sekspace.py:130-178), the whole k-space stage (precompute excluded, as
    cli.py:110-111) and the self term of all N.

    Returned `value` is the throughput MEASURED on that sample, in the
    metric's unit: particles/s = 1 / (per-target real-space seconds + per-
    particle spread+gather seconds + k-space seconds / N).  `seconds` is the
    wall time the sample actually took (the timed region of one step)."""
    from concurrent.futures import ThreadPoolExecutor

    from threadpoolctl import threadpool_limits

    orc = _oracle()
    N, L, D = len(q), CFG["L"], CFG["D"]
    rng = np.random.default_rng(seed)
    n = max(1, int(L // CFG["rc"]))
    cell = np.minimum((pos / (L / n)).astype(int), n - 1)
    flat = (cell[:, 0] * n + cell[:, 1]) * n + cell[:, 2]
    occupied = np.unique(flat[rng.choice(N, min(N, 64 * n_cells), replace=False)])
    cells = rng.choice(occupied, min(n_cells, len(occupied)), replace=False)
    g = orc.geometry(L, D, CFG["M"], CFG["P"], CFG.get("s0", 1.0), CFG.get("s", 1.0), CFG.get("R", 0.0))
    xi, rc = CFG["xi"], CFG["rc"]
    win, shape = CFG["window"], CFG["shape"]
    if D == 0:
        table, kg = orc.d0_kernel_table(L, CFG["M"], CFG["P"], CFG["s0"], rc)  # precompute: untimed

    def kstage(H):
        if D == 3:
            return orc.kspace_d3(H, g, xi, win, shape)
        if D == 0:
            return orc.kspace_d0_kernel(H, g, xi, win, shape, table, kg["nconv"])
        return orc.kspace_mixed(H, g, xi, win, shape, CFG["nI"])
    tsets = [np.nonzero(flat == c)[0] for c in cells]
    n_t = sum(len(x) for x in tsets)
    sel = rng.choice(N, min(N, n_kspace), replace=False)
    chunks = np.array_split(sel, max(1, threads))
    with threadpool_limits(1):
        t00 = time.perf_counter()
        if threads > 1:
            with ThreadPoolExecutor(threads) as ex:
                list(ex.map(lambda s: orc.realspace(pos, q, L, D, xi, rc, targets=s), tsets))
        else:
            for x in tsets:
                orc.realspace(pos, q, L, D, xi, rc, targets=x)
        t_real = time.perf_counter() - t00
        t0 = time.perf_counter()
        if threads > 1:
            with ThreadPoolExecutor(threads) as ex:
                parts = list(ex.map(lambda s: orc.spread(pos[s], q[s], g, win, shape), chunks))
        else:
            parts = [orc.spread(pos[s], q[s], g, win, shape) for s in chunks]
        H = parts[0]
        for p_ in parts[1:]:
            H = H + p_
        t_spread = time.perf_counter() - t0
        t0 = time.perf_counter()
        Ht = kstage(H)
        t_fft = time.perf_counter() - t0
        t0 = time.perf_counter()
        if threads > 1:
            with ThreadPoolExecutor(threads) as ex:
                list(ex.map(lambda s: orc.gather(Ht, pos[s], g, win, shape), chunks))
        else:
            orc.gather(Ht, pos[sel], g, win, shape)
        t_gather = time.perf_counter() - t0
        t0 = time.perf_counter()
        orc.self_term(q, xi)
        t_self = time.perf_counter() - t0
        seconds = time.perf_counter() - t00
    per_particle = t_real / n_t + (t_spread + t_gather) / len(sel) + (t_fft + t_self) / N
    return {"value": 1.0 / per_particle, "unit": "particles/s", "cores": threads, "kind": "port",
            "sample": (f"oracle/se_oracle.py on {CFG['workload']}, {threads} thread(s): real space for all {n_t} "
                       f"targets of {len(cells)} random rc-cells ({t_real:.2f} s), spread+gather of {len(sel)} "
                       f"particles ({t_spread + t_gather:.2f} s), the whole k-space stage ({t_fft:.2f} s) and self "
                       f"term; value = 1 / (real s per target + spread/gather s per particle + k-space s / N), "
                       f"measured in a {seconds:.1f} s sample"),
            "seconds": seconds}


def config_dict(args, world):
    """The `config` object of the JSON line -- the same for both arms."""
    single = world == 1 and "RANK" not in os.environ
    return {"workload": DESCR[CFG["workload"]], "N": CFG["N"], "seed": CFG["seed"],
            "parallelism": ("single GPU (fused pipeline, CUDA graph)" if single else
                            (f"domain decomposition x{world}: particles partitioned (contiguous "
                             "chunks of the random input order), migrated to x-slabs of "
                             "real-space columns, +x halo with Newton sums returned, touched "
                             "grid planes to the k-space slab owners, slab FFT with two "
                             "all-to-all transposes (D = 3)" if args.mode == "domain" else
                             f"particle-shard x{world} with replicated inputs, {args.kspace} "
                             "k-space")),
            "l2": "flushed (256 MB write) between timed steps, outside the step events"}


def run_reference(args):
    """--impl reference: the reference's CPU path (its port) on the host
    cores.  Each step is one bounded sample of the workload (cpu_sample);
    ms_per_step is the sample's own wall time, value the particles/s
    measured on it (mean over the timed steps)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    load_workload(args.workload)
    pos, q = make_inputs()
    threads = os.cpu_count() or 1
    vals, secs, last = [], [], None
    t_w0 = time.perf_counter()
    for i in range(args.warmup + args.steps):
        if i == args.warmup:
            t_w0 = time.perf_counter()
        r = cpu_sample(pos, q, threads=threads, n_cells=threads, n_kspace=min(len(q), 10000 * max(1, threads // 2)),
                       seed=i)
        if i >= args.warmup:
            vals.append(r["value"])
            secs.append(r["seconds"])
            last = r
    t_wall = time.perf_counter() - t_w0
    value = statistics.mean(vals)
    line = {"impl": "reference", "metric": metric(), "value": value, "unit": "particles/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.mean(secs), "wall_s_timed_region": t_wall,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.md 3.1)",
            "config": config_dict(args, int(os.environ.get("WORLD_SIZE", "1"))),
            "cpu_baseline": {"value": value, "unit": "particles/s", "cores": threads, "kind": "port",
                             "sample": last["sample"]},
            "e2e": {"value": value, "unit": "particles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


# -------------------------------------------------------------- our pipeline

class _PlanGroup:
    """Profiling view over the sharded backend's plans (real space on the
    main stream, the k-space chain on the side stream); `handle` is the
    real-space plan (pair count)."""

    def __init__(self, plans):
        self.plans = plans
        self.handle = plans[0].handle

    def set_profiling(self, on):
        for p in self.plans:
            p.set_profiling(on)

    def grid(self):
        return self.plans[0].grid()

    def launches(self):
        return sum(p.launches() for p in self.plans)

    def kernel_times(self):
        out = {}
        for p in self.plans:
            for k, (ms, n) in p.kernel_times().items():
                a = out.get(k, (0.0, 0))
                out[k] = (a[0] + ms, a[1] + n)
        return out


def realspace_newton(N, L, rc, D):
    """Whether the real-space kernel runs its Newton (half-shell) path, which
    evaluates every unordered in-cutoff pair once -- the rule of cell_bin
    (se_realspace.cu): columns of edge >= rc / reach, reach 3 unless columns
    would hold < 256 particles; minimum-image mode (no Newton) when a
    periodic x / y axis has fewer than 2 reach + 1 columns."""
    reach = 3
    while True:
        nn = min(1024, max(1, int(math.floor(reach * L / rc))))
        if reach == 2 or N / (nn * nn) >= 256.0:
            break
        reach -= 1
    if D >= 1 and rc > L / 2 + 1e-12:
        return False
    return not (D >= 1 and nn < 2 * reach + 1)


def _source_hash(files):
    import hashlib
    h = hashlib.sha256()
    for f in files:
        h.update(open(os.path.join(ROOT, f), "rb").read())
    return h.hexdigest()[:16]


REALSPACE_SOURCES = ("paper_1712_04732_b200/csrc/se_realspace.cu", "paper_1712_04732_b200/csrc/se_erfc_coeffs.h",
                     "paper_1712_04732_b200/csrc/se_common.h", "paper_1712_04732_b200/csrc/se_host.cpp")


def ncu_evidence():
    """The committed ncu --set full summary of the real-space kernel, used
    only if it was captured from the CURRENT sources (profiles/ncu_r02_summary.json
    records the hash of the kernel's source files); otherwise None and a
    warning on stderr -- a stale profile is never attached to a number."""
    path = os.path.join(ROOT, "profiles", "ncu_r02_summary.json")
    try:
        nc = json.load(open(path))
    except Exception:
        return None
    cur = _source_hash(REALSPACE_SOURCES)
    rs = nc.get("realspace", {})
    if rs.get("source_hash") != cur:
        print(f"bench: profiles/ncu_r02_summary.json is of another build of the real-space kernel "
              f"({rs.get('source_hash')} != {cur}); roofline.traffic left null", file=sys.stderr)
        return None
    return rs


def measure(name, args, dev, world, rank, sharded, steps, warmup, extras=True):
    """Time `steps` total-potential evaluations of workload `name` (device-
    resident inputs, L2 flushed between steps outside the events, max over
    ranks) and the same through the public host API (e2e)."""
    import torch
    import torch.distributed as dist

    import paper_1712_04732_b200 as se
    from paper_1712_04732_b200 import device as sedev
    from paper_1712_04732_b200.distributed import NativeBackend, total_potential_domain, total_potential_sharded

    load_workload(name)
    local = dev.index
    peri = se.Periodicity(CFG["D"])
    prm = se_params()
    N, L = CFG["N"], CFG["L"]
    pos_h, q_h = make_inputs()
    pos_p = torch.from_numpy(pos_h).pin_memory()
    q_p = torch.from_numpy(q_h).pin_memory()
    pos_d = pos_p.to(dev)
    q_d = q_p.to(dev)
    phi_d = torch.empty(N, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    lo, hi = N * rank // world, N * (rank + 1) // world
    if sharded:
        backend = NativeBackend(L, prm, peri, dev)
        plan = _PlanGroup(backend.plans)
        if args.mode == "domain":
            # particles partitioned over the ranks: rank r passes the r-th
            # contiguous chunk of the (spatially random) input order
            pos_r, q_r = pos_d[lo:hi].contiguous(), q_d[lo:hi].contiguous()

            def step():
                return total_potential_domain(pos_r, q_r, backend)
        else:
            def step():
                return total_potential_sharded(pos_d, q_d, backend, kspace=args.kspace)
    else:
        plan = sedev.plan(L, prm, peri, dev)

        def step():
            return sedev.total_potential(pos_d, q_d, L, prm, peri, out=phi_d)

    clk = ClockSampler(local)
    clk.__enter__()  # running before the warm-up; the timed window opens at clk.mark()
    plan.set_profiling(True)
    for _ in range(max(3, warmup)):
        step()
    torch.cuda.synchronize(dev)

    import ctypes

    from paper_1712_04732_b200 import _native
    cnt = ctypes.c_int64()
    _native.call("se_realspace_pair_count_dev", plan.handle, _native.ptr(pos_d), _native.ptr(q_d), N,
                 ctypes.byref(cnt))
    pairs = int(cnt.value)

    plan.set_profiling(True)
    launches0 = plan.launches()
    plan.kernel_times()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    if sharded:
        dist.barrier()
    torch.cuda.synchronize(dev)
    try:
        clk.mark()
        t_wall0 = time.perf_counter()
        for i in range(steps):
            flush.zero_()
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize(dev)
        if sharded:
            dist.barrier()
        t_wall = time.perf_counter() - t_wall0
    finally:
        clk.__exit__(None, None, None)
    launches = plan.launches() - launches0
    ktimes = plan.kernel_times()
    plan.set_profiling(False)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if sharded:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms_per_step = float(tot.item()) / steps
    value = N / (ms_per_step * 1e-3)

    # end to end through the public API with pinned host buffers
    if not sharded:
        system = se.ParticleSystem(pos_p.numpy(), q_p.numpy(), L)
        # the same warm-up as the device-resident steps: the host entry's
        # first calls bind its staging buffers and capture its CUDA graph
        for _ in range(max(3, warmup)):
            phi_h = se.total_potential(system, prm, peri)
        t_e = []
        for _ in range(steps):
            t0 = time.perf_counter()
            phi_h = se.total_potential(system, prm, peri)
            t_e.append(time.perf_counter() - t0)
        e2e = {"value": N / statistics.mean(t_e), "unit": "particles/s",
               "h2d_bytes_per_step": pos_h.nbytes + q_h.nbytes, "d2h_bytes_per_step": N * 8,
               "ms_per_step": 1e3 * statistics.mean(t_e),
               "api": "paper_1712_04732_b200.total_potential (se_total_potential_host)"}
    else:
        t_e = []
        domain = args.mode == "domain"
        pos_pr, q_pr = (pos_p[lo:hi].pin_memory(), q_p[lo:hi].pin_memory()) if domain else (pos_p, q_p)
        phi_pin = torch.empty((hi - lo) if domain else N, dtype=torch.float64, pin_memory=True)  # D2H target
        for it in range(max(3, warmup) + max(1, steps)):  # untimed warm-up calls first
            torch.cuda.synchronize(dev)
            dist.barrier()
            t0 = time.perf_counter()
            pd = pos_pr.to(dev, non_blocking=True)
            qd = q_pr.to(dev, non_blocking=True)
            if domain:
                phi_pin.copy_(total_potential_domain(pd, qd, backend), non_blocking=True)
            else:
                phi_pin.copy_(total_potential_sharded(pd, qd, backend, kspace=args.kspace), non_blocking=True)
            torch.cuda.synchronize(dev)
            phi_h = phi_pin.numpy()
            if it >= max(3, warmup):
                t_e.append(time.perf_counter() - t0)
        te = torch.tensor([statistics.mean(t_e)], dtype=torch.float64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        nb = (hi - lo) if domain else N
        e2e = {"value": N / float(te.item()), "unit": "particles/s",
               "h2d_bytes_per_step": 32 * nb, "d2h_bytes_per_step": 8 * nb,
               "h2d_note": "per rank (its own particles)" if domain else "per rank (replicated inputs)",
               "api": ("paper_1712_04732_b200.distributed.total_potential_domain" if domain else
                       "paper_1712_04732_b200.distributed.total_potential_sharded")}
    out = {"name": name, "N": N, "ms_per_step": ms_per_step, "value": value, "e2e": e2e, "ktimes": ktimes,
           "launches": launches, "t_wall": t_wall, "clocks": clk.summary(), "pairs": pairs, "plan": plan,
           "pos_d": pos_d, "q_d": q_d, "phi_d": phi_d, "prm": prm, "peri": peri, "phi_h": phi_h}
    return out


def kspace_vs_direct(name, ntargets=64, seed=11):
    """Relative RMS of the SE k-space potential against the reference's own
    direct Ewald Fourier sum (oracle.py:109-192 as device kernels,
    paper_1712_04732_b200.direct) at `ntargets` sampled targets of the full
    system -- the tolerance the metric names ('at rms tol ...'), measured as
    the reference's CLI does (cli.py:114-118: se_kspace vs kspace_direct)."""
    import paper_1712_04732_b200 as se
    from paper_1712_04732_b200 import direct

    w = workloads.ALL[name]()
    p = se.SEParams(**w["prm"])
    s = se.ParticleSystem(w["pos"], w["q"], w["L"])
    peri = se.Periodicity(w["D"])
    phik = se.se_kspace(s, p, peri)
    sel = np.sort(np.random.default_rng(seed).choice(s.N, ntargets, replace=False))
    kmax = direct.OracleConfig.for_accuracy(p.xi, s.L, 1e-13).kmax
    t0 = time.perf_counter()
    ref = direct.kspace_direct(s, p.xi, peri, kmax, targets=sel)
    return {"rms_vs_direct": float(se.relative_rms_error(phik[sel], ref)), "targets": int(ntargets),
            "kmax": int(kmax), "eps_target": float(w["prm"]["eps"]),
            "meets_tolerance": bool(se.relative_rms_error(phik[sel], ref) <= w["prm"]["eps"]),
            "direct_s": time.perf_counter() - t0}


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # under torchrun (any world size, 1 included) the sharded NCCL pipeline runs
    sharded = "RANK" in os.environ and "WORLD_SIZE" in os.environ
    if sharded:
        dist.init_process_group("nccl", device_id=dev)

    m = measure(args.workload, args, dev, world, rank, sharded, args.steps, args.warmup)
    N, ms_per_step, value, ktimes, plan = m["N"], m["ms_per_step"], m["value"], m["ktimes"], m["plan"]
    pos_d, q_d, phi_d = m["pos_d"], m["q_d"], m["phi_d"]
    from paper_1712_04732_b200 import _native

    pk = peaks()
    real_ms = ktimes["realspace"][0] / max(1, ktimes["realspace"][1])
    pairs = m["pairs"]
    newton = realspace_newton(N, CFG["L"], CFG["rc"], CFG["D"])
    evaluated = pairs // 2 if newton else pairs
    achieved = evaluated * FLOP_PER_PAIR / (real_ms * 1e-3) / 1e12
    kern = {}
    for k, (ms, n) in ktimes.items():
        if n:
            kern[k] = {"ms_per_launch": ms / n, "share_of_step": (ms / n) / ms_per_step}
    P3 = CFG["P"] ** 3
    gshape = plan.grid().shape
    G = gshape[0] * gshape[1] * gshape[2]
    # spreading / gathering measured alone (stage entry points, CUDA events on
    # the plan's stream around each kernel): the SURVEY 8d bounds -- on-chip
    # shared-memory RMW traffic vs the measured smem bandwidth, the update rate
    # vs the measured global fp64 atomic (REDG) rate a direct-to-grid spread
    # would be bound by, and the compulsory HBM traffic vs the HBM copy rate
    spread_gather = None
    if not sharded:
        import torch
        grid_d = torch.empty(G, dtype=torch.float64, device=dev)
        plan.set_profiling(True)
        plan.kernel_times()
        for _ in range(5):
            _native.call("se_spread_dev", plan.handle, _native.ptr(pos_d), _native.ptr(q_d), N, _native.ptr(grid_d))
            _native.call("se_gather_dev", plan.handle, _native.ptr(grid_d), _native.ptr(pos_d), N,
                         _native.ptr(phi_d), 0)
        torch.cuda.synchronize(dev)
        kt = plan.kernel_times()
        plan.set_profiling(False)
        sg = {}
        for k, onchip_b in (("spread", 16), ("gather", 8)):
            ms, n = kt.get(k, (0.0, 0))
            if not n:
                continue
            t = ms / n * 1e-3
            comp = 32 * N + 8 * G + (8 * N if k == "gather" else 0)
            frac = lambda v, peak: v / peak if peak else None  # noqa: E731
            sg[k] = {"ms_per_launch": ms / n, "updates_per_s": N * P3 / t,
                     "onchip_GBps": onchip_b * N * P3 / t / 1e9,
                     "frac_of_smem_peak": frac(onchip_b * N * P3 / t, (pk["smem_tbs"] or 0) * 1e12),
                     "compulsory_hbm_GBps": comp / t / 1e9,
                     "frac_of_hbm": frac(comp / t, pk["hbm_gbs"] * 1e9)}
        spread_gather = {"updates_per_launch": N * P3, **sg,
                         "peaks": {"smem_tbs": pk["smem_tbs"], "hbm_gbs": pk["hbm_gbs"], "source": pk["fp64_src"]}}
    roofline = {"kernel": "realspace_cell_kernel (erfc pair sum, polynomial pair term 1/r - Q(r^2))", "bound": "fp64",
                "achieved": achieved, "peak": pk["fp64_tflops"], "unit": "TFLOP/s",
                "frac": achieved / pk["fp64_tflops"], "traffic": None,
                "peak_source": pk["fp64_src"],
                "algorithmic": (f"{evaluated} evaluated in-cutoff pairs ({pairs} ordered pairs"
                                f"{', Newton: each unordered pair evaluated once' if newton else ''}) x "
                                f"{FLOP_PER_PAIR} flop (SURVEY 8d) per launch"),
                "evaluated_pairs": evaluated, "ms_per_launch": real_ms}
    ev = ncu_evidence()
    if ev is not None and CFG["workload"] == ev.get("workload"):
        roofline["traffic"] = ev.get("dram_bytes")
        roofline["fp64_pipe_pct"] = ev.get("fp64_pipe_pct")
        roofline["issue_active_pct"] = ev.get("issue_active_pct")
        inst = ev.get("inst_executed")
        if inst:
            roofline["inst_per_pair"] = 32.0 * float(inst) / evaluated
        roofline["ncu_source"] = ev.get("source")

    line = {"metric": metric(), "value": value, "unit": "particles/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, BASELINE.md 3.1; no public dataset exists for this path)",
            "config": config_dict(args, world),
            "e2e": m["e2e"], "roofline": roofline, "kernels": kern,
            "spread_gather": spread_gather,
            "kernels_note": ("event spans per stage on the stream it runs on; the k-space pipeline "
                             "(spread, kspace, gather, its sort) runs on a side stream concurrently with "
                             "the real-space kernel, so its spans include waiting for SM resources and "
                             "the shares do not add up to 1"),
            "gpu_launches": m["launches"],
            "gpu_launches_per_step": m["launches"] / args.steps, "wall_s_timed_region": m["t_wall"],
            "clocks": m["clocks"] if rank == 0 else None,
            "pairs_in_cutoff": pairs}
    # the tolerance the metric names: cfg2 (P = 8) misses 1e-8; its
    # tolerance-meeting variant (ES P = 10, beta = 25) on the same inputs
    if world == 1 and not sharded and args.workload == "cfg2" and not args.no_tol:
        line["rms"] = kspace_vs_direct("cfg2")
        t = measure("cfg2_tol", args, dev, world, rank, sharded, args.steps, args.warmup)
        line["cfg2_tol"] = {"workload": DESCR["cfg2_tol"], "value": t["value"], "unit": "particles/s",
                            "ms_per_step": t["ms_per_step"], "e2e": t["e2e"], "clocks": t["clocks"],
                            "gpu_launches": t["launches"], **kspace_vs_direct("cfg2_tol")}
        load_workload(args.workload)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        pos_h, q_h = make_inputs()
        big = args.workload.startswith("cfg2")  # ~12 s of CPU work at cfg2; clustered cfg5 cells stay at 2
        line["cpu_baseline"] = cpu_sample(pos_h, q_h, threads=1, n_cells=6 if big else 2,
                                          n_kspace=60000 if big else 20000)
    if rank == 0:
        emit(line)
    if sharded:
        dist.destroy_process_group()
    return 0


_JSON_FD = None


def emit(line):
    """The one JSON line on the original stdout; everything else (NCCL's
    version banner, library chatter) was redirected to stderr by main()."""
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, data)


def _free_port():
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        return s_.getsockname()[1]


def self_launch(gpus):
    """`bench.py --gpus N` outside torchrun: re-exec this script under
    torch.distributed.run with N ranks on this node (one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    global _JSON_FD
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tol", action="store_true", help="skip the cfg2_tol (tolerance-meeting) companion line")
    ap.add_argument("--kspace", choices=("replicated", "slab"), default="replicated",
                    help="multi-GPU k-space stage (torchrun): replicated after a grid all-reduce, or "
                         "slab-decomposed (D = 3)")
    ap.add_argument("--mode", choices=("domain", "sharded"), default="domain",
                    help="multi-GPU decomposition (torchrun): domain (partitioned particles) or sharded "
                         "(replicated inputs)")
    ap.add_argument("--workload", default="cfg2", choices=sorted(workloads.ALL),
                    help="BASELINE config (default cfg2 = configs[1], the headline)")
    args = ap.parse_args()
    ws = os.environ.get("WORLD_SIZE")
    if ws is None and args.gpus > 1:
        return self_launch(args.gpus)
    if ws is not None and int(ws) != args.gpus:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={ws}", file=sys.stderr)
        return 2
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)  # fd 1 (C and Python writers) -> stderr; the JSON line goes to the saved fd
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
