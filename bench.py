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

FLOP_PER_PAIR = 40  # SURVEY 8d constant: erfc(xi r)/r ~ exp + rational + sqrt + div + fma
DESCR = {
    "cfg1": "cfg1: D=3, N=2000 uniform in L=1, Gaussian P=16, M=32^3, rc=0.3, xi=12.94",
    "cfg2": "cfg2: D=3, N=1e6 uniform in L=10, ES P=8 beta=20, M=128^3, rc=1.0, xi=4.2919",
    "cfg3": "cfg3 (as worded): D=2, N=2e5 in L=5, ES P=8, M=96^2 x 104, s0=4, s=2, nI=10, xi=6",
    "cfg3_tol": "cfg3 (tolerance-meeting): D=2, N=2e5 in L=5, ES P=10, s0=4, s=4, nI=48, xi=6",
    "cfg4": "cfg4: D=1 (cubic embedding L=8 of 4x4x8), N=2e5, Gaussian P=12, M=128, xi=4, s0=2.4674, nI=39",
    "cfg5": "cfg5: D=0, N=5e5 (ball + 32 Gaussian clusters) in L=4, ES P=10 beta=25, M=96, xi=6, kernel path",
}
CFG = {}


def load_workload(name):
    w = workloads.ALL[name]()
    CFG.clear()
    CFG.update(w["prm"])
    CFG.update(workload=name, D=w["D"], L=w["L"], N=len(w["q"]), seed=int(name[3]))
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
    micro-benchmarks (profiles/peaks_r01.json, tools/peaks.cu)."""
    out = {"hbm_gbs": 6655.0, "hbm_src": "fallback (B200_PROFILING.md)",
           "fp64_tflops": 37.0, "fp64_src": "fallback (datasheet ~37-40 TF/s)",
           "smem_tbs": None, "redg_gops": None}
    try:
        m = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        out["hbm_gbs"], out["hbm_src"] = float(m["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        pass
    try:
        p = json.load(open(os.path.join(ROOT, "profiles", "peaks_r01.json")))
        out["fp64_tflops"], out["fp64_src"] = float(p["fp64_fma_tflops"]), "measured (profiles/peaks_r01.json)"
        out["smem_tbs"] = float(p["smem_tbs"])
        out["redg_gops"] = float(p["redg_f64_gops"])
    except Exception:
        pass
    return out


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

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
    """Oracle port of the reference on a bounded sample of the workload,
    extrapolated to the full N: real space on every target of `n_cells`
    random occupied rc-cells (the reference's per-home-cell dense blocks,
    realspace.py:100-126), spread + gather for `n_kspace` particles
    (sekspace.py:130-178), the full k-space stage (precompute excluded, as
    cli.py:110-111), and the self term."""
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
    with threadpool_limits(1):
        t0 = time.perf_counter()
        tsets = [np.nonzero(flat == c)[0] for c in cells]
        if threads > 1:
            with ThreadPoolExecutor(threads) as ex:
                list(ex.map(lambda s: orc.realspace(pos, q, L, D, xi, rc, targets=s), tsets))
        else:
            for s in tsets:
                orc.realspace(pos, q, L, D, xi, rc, targets=s)
        t_real = time.perf_counter() - t0
        n_t = sum(len(s) for s in tsets)
        sel = rng.choice(N, n_kspace, replace=False)
        chunks = np.array_split(sel, max(1, threads))
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
    est = t_real * N / n_t + (t_spread + t_gather) * N / n_kspace + t_fft + t_self
    return {"value": N / est, "unit": "particles/s", "cores": threads, "kind": "port",
            "sample": (f"oracle/se_oracle.py on {CFG['workload']}: real space for all {n_t} targets of "
                       f"{len(cells)} random rc-cells, spread+gather of {n_kspace} particles, full k-space stage, "
                       f"self term; extrapolated to N={N} ({est:.0f} s per evaluation)"),
            "seconds_sampled": t_real + t_spread + t_fft + t_gather + t_self,
            "est_seconds_full": est}


def run_reference(args):
    """--impl reference: the reference's CPU path (its port) on host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    load_workload(args.workload)
    pos, q = make_inputs()
    threads = os.cpu_count() or 1
    vals, last = [], None
    for i in range(args.warmup + args.steps):
        r = cpu_sample(pos, q, threads=threads, n_cells=threads, n_kspace=min(len(q), 20000 * max(1, threads // 2)),
                       seed=i)
        if i >= args.warmup:
            vals.append(r["value"])
            last = r
    value = statistics.mean(vals)
    line = {"impl": "reference", "metric": metric(), "value": value, "unit": "particles/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * CFG["N"] / value, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.md 3.1)",
            "config": {"workload": DESCR[CFG["workload"]], "N": CFG["N"], "seed": CFG["seed"]},
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


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1712_04732_b200 as se
    from paper_1712_04732_b200 import device as sedev
    from paper_1712_04732_b200.distributed import NativeBackend, total_potential_sharded

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # under torchrun (any world size, 1 included) the sharded NCCL pipeline runs
    sharded = "RANK" in os.environ and "WORLD_SIZE" in os.environ
    if sharded:
        dist.init_process_group("nccl", device_id=dev)
    load_workload(args.workload)
    peri = se.Periodicity(CFG["D"])
    prm = se_params()
    N, L = CFG["N"], CFG["L"]
    pos_h, q_h = make_inputs()
    # pinned host copies (e2e inputs) and device-resident copies (value)
    pos_p = torch.from_numpy(pos_h).pin_memory()
    q_p = torch.from_numpy(q_h).pin_memory()
    pos_d = pos_p.to(dev)
    q_d = q_p.to(dev)
    phi_d = torch.empty(N, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    if sharded:
        backend = NativeBackend(L, prm, peri, dev)
        plan = _PlanGroup(backend.plans)

        def step():
            return total_potential_sharded(pos_d, q_d, backend, kspace=args.kspace)
    else:
        plan = sedev.plan(L, prm, peri, dev)

        def step():
            return sedev.total_potential(pos_d, q_d, L, prm, peri, out=phi_d)

    # profiling (per-kernel CUDA events) is on from the warm-up on, so that the
    # CUDA graph of the fused pipeline is captured during warm-up and the timed
    # steps are replays; the counters are reset before the timed region
    plan.set_profiling(True)
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize(dev)

    # pair count for the real-space roofline (untimed)
    npairs = torch.zeros(1, dtype=torch.int64)
    import ctypes
    from paper_1712_04732_b200 import _native
    cnt = ctypes.c_int64()
    _native.call("se_realspace_pair_count_dev", plan.handle, _native.ptr(pos_d), _native.ptr(q_d), N,
                 ctypes.byref(cnt))
    npairs[0] = cnt.value

    plan.set_profiling(True)
    launches0 = plan.launches()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if sharded:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        t_wall0 = time.perf_counter()
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize(dev)
        if sharded:
            dist.barrier()
        t_wall = time.perf_counter() - t_wall0
    launches = plan.launches() - launches0
    ktimes = plan.kernel_times()
    plan.set_profiling(False)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if sharded:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms_per_step = float(tot.item()) / args.steps
    value = N / (ms_per_step * 1e-3)

    # end-to-end through the public API with pinned host buffers (rank 0, N=1)
    e2e = None
    if not sharded:
        system = se.ParticleSystem(pos_p.numpy(), q_p.numpy(), L)
        se.total_potential(system, prm, peri)
        t_e = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            se.total_potential(system, prm, peri)
            t_e.append(time.perf_counter() - t0)
        e2e = {"value": N / statistics.mean(t_e), "unit": "particles/s",
               "h2d_bytes_per_step": pos_h.nbytes + q_h.nbytes, "d2h_bytes_per_step": N * 8,
               "ms_per_step": 1e3 * statistics.mean(t_e),
               "api": "paper_1712_04732_b200.total_potential (se_total_potential_host)"}
    else:
        # sharded runs: host inputs replicated to every rank, phi read back on every rank
        t_e = []
        for _ in range(max(1, args.steps)):
            torch.cuda.synchronize(dev)
            dist.barrier()
            t0 = time.perf_counter()
            pd = pos_p.to(dev, non_blocking=True)
            qd = q_p.to(dev, non_blocking=True)
            phi = total_potential_sharded(pd, qd, backend, kspace=args.kspace).cpu()
            t_e.append(time.perf_counter() - t0)
        te = torch.tensor([statistics.mean(t_e)], dtype=torch.float64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": N / float(te.item()), "unit": "particles/s",
               "h2d_bytes_per_step": pos_h.nbytes + q_h.nbytes, "d2h_bytes_per_step": N * 8,
               "api": "paper_1712_04732_b200.distributed.total_potential_sharded"}

    pk = peaks()
    real_ms = ktimes["realspace"][0] / max(1, ktimes["realspace"][1])
    pairs = int(npairs[0])
    achieved = pairs * FLOP_PER_PAIR / (real_ms * 1e-3) / 1e12
    kern = {}
    for k, (ms, n) in ktimes.items():
        if n:
            kern[k] = {"ms_per_launch": ms / n, "share_of_step": (ms / n) / ms_per_step}
    P3 = CFG["P"] ** 3
    gshape = plan.grid().shape
    G = gshape[0] * gshape[1] * gshape[2]
    for k in ("spread", "gather"):
        if k in kern:
            t = kern[k]["ms_per_launch"] * 1e-3
            onchip = (16 if k == "spread" else 8) * N * P3
            kern[k]["onchip_GBps"] = onchip / t / 1e9
            kern[k]["compulsory_GBps"] = (32 * N + 8 * G) / t / 1e9
            kern[k]["updates_per_s"] = N * P3 / t
    # spreading / gathering measured alone (stage entry points, CUDA events on
    # the plan's stream around each kernel): the SURVEY 8d bounds -- on-chip
    # shared-memory RMW traffic vs the measured smem bandwidth, the update rate
    # vs the measured global fp64 atomic (REDG) rate a direct-to-grid spread
    # would be bound by, and the compulsory HBM traffic vs the HBM copy rate
    spread_gather = None
    if not sharded:
        grid_d = torch.empty(G, dtype=torch.float64, device=dev)
        plan.set_profiling(True)
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
            if k == "spread":  # vs a spread that adds every update straight into the grid (REDG)
                sg[k]["frac_of_redg_peak"] = frac(N * P3 / t, (pk["redg_gops"] or 0) * 1e9)
        spread_gather = {"updates_per_launch": N * P3, **sg,
                         "peaks": {"redg_gops": pk["redg_gops"], "smem_tbs": pk["smem_tbs"],
                                   "hbm_gbs": pk["hbm_gbs"], "source": pk["fp64_src"]}}
    roofline = {"kernel": "realspace_cell_kernel (erfc pair sum)", "bound": "fp64",
                "achieved": achieved, "peak": pk["fp64_tflops"], "unit": "TFLOP/s",
                "frac": achieved / pk["fp64_tflops"], "traffic": None,
                "peak_source": pk["fp64_src"],
                "algorithmic": f"{pairs} ordered in-cutoff pairs x {FLOP_PER_PAIR} flop per launch",
                "ms_per_launch": real_ms}
    try:
        nc = json.load(open(os.path.join(ROOT, "profiles", "ncu_r01_summary.json")))
        roofline["traffic"] = nc.get("realspace", {}).get("dram_bytes")
    except Exception:
        pass

    line = {"metric": metric(), "value": value, "unit": "particles/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, BASELINE.md 3.1; no public dataset exists for this path)",
            "config": {"workload": DESCR[CFG["workload"]], "N": N, "seed": CFG["seed"],
                       "parallelism": (f"particle-shard x{world} (grid + phi sum-all-reduce)"
                                       if args.kspace == "replicated" or world == 1 else
                                       f"particle-shard x{world}, slab k-space (grid reduce-scatter, "
                                       "2 all-to-all, all-gather; phi sum-all-reduce)"),
                       "l2": "flushed (256 MB write) between timed steps, outside the step events"},
            "e2e": e2e, "roofline": roofline, "kernels": kern,
            "spread_gather": spread_gather,
            "kernels_note": ("event spans per stage on the stream it runs on; the k-space pipeline "
                             "(spread, kspace, gather, its sort) runs on a side stream concurrently with "
                             "the real-space kernel, so its spans include waiting for SM resources and "
                             "the shares do not add up to 1"),
            "gpu_launches": launches,
            "gpu_launches_per_step": launches / args.steps, "wall_s_timed_region": t_wall,
            "clocks": clk.summary() if rank == 0 else None,
            "pairs_in_cutoff": pairs}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_sample(pos_h, q_h, threads=1)
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


def main():
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)  # fd 1 (C and Python writers) -> stderr; the JSON line goes to the saved fd
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--kspace", choices=("replicated", "slab"), default="replicated",
                    help="multi-GPU k-space stage (torchrun): replicated after a grid all-reduce, or "
                         "slab-decomposed (D = 3)")
    ap.add_argument("--workload", default="cfg2", choices=sorted(workloads.ALL),
                    help="BASELINE config (default cfg2 = configs[1], the headline)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
