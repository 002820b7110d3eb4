#!/usr/bin/env python
"""HALLaR time-to-1e-5 on B200 — the BASELINE.json headline metric.

Workload (BASELINE.json configs[1]): Lovasz theta on the Hamming graph H(12,2)
(n = 4096 vertices, m = 24,577 constraints), SolverConfig{eps = 1e-5, seed = 0},
all other reference defaults.  One "step" = one full solve.

  value  device time of the persistent solve kernel (instance resident in HBM),
         CUDA events on the launching stream, mean over K steps, max over ranks
  e2e    the same solve through the reference-facing C-ABI with HOST buffers:
         instance built from host edge arrays (H2D), solve, U and p read back (D2H)

`--impl reference` times the reference algorithm's CPU implementation (the
oracle port, oracle/ — the reference itself cannot be built: no Eigen) on the
host cores.  Multi-GPU: the path does not shard at this size — replicas only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time-to-1e-5 rel. precision (s)"
UNIT = "s"
HYPERCUBE_D = 12
WORKLOAD = "theta H(12,2): n=4096, m=24577, eps=1e-5, seed=0 (BASELINE configs[1])"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling via NVML during the timed region."""

    def __init__(self, index=0, period=0.1):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self.index, self.period = index, period

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            names = {
                getattr(pynvml, "nvmlClocksThrottleReasonHwSlowdown", 0x8): "hw_slowdown",
                getattr(pynvml, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
                getattr(pynvml, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
                getattr(pynvml, "nvmlClocksThrottleReasonSwPowerCap", 0x4): "sw_power_cap",
            }

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                        for bit, nm in names.items():
                            if r & bit:
                                self.reasons.add(nm)
                    except Exception:
                        pass
                    time.sleep(self.period)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def cpu_reference_solve():
    from oracle import oracle as O
    inst = O.OracleInstance.hypercube(HYPERCUBE_D)
    t0 = time.perf_counter()
    r = inst.solve(eps=1e-5, seed=0)
    wall = time.perf_counter() - t0
    assert r.status == "optimal", r.status
    return r, wall


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_reference_solve()
    times = []
    last = None
    for _ in range(args.steps):
        last, wall = cpu_reference_solve()
        times.append(last.wall_seconds)
    v = statistics.mean(times)
    cores = os.cpu_count()
    line = {
        "metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": WORKLOAD},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{args.steps} full solves of H(12,2) to 1e-5 (oracle port of lrsdp, "
                                   f"{cores} threads; fista_iters {last.fista_iters})"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "counters": {"outer": last.outer_iters, "fista": last.fista_iters, "eig": last.eig_products,
                     "rank": last.rank, "pval": last.pval},
    }
    print(json.dumps(line), flush=True)


def algorithmic_bytes_grad_pass(n, m_pairs, s):
    # per pair constraint: upper entry (col int32 + p f64) + lower entry (col + p) = 24 B;
    # per row: lo_ptr + up_ptr (16 B), U row read (8s), gradient row write (8s)
    return 24 * m_pairs + 16 * n + 16 * n * s


def large_roofline(H, np, peak, peak_kind, d=23, s=2, iters=10):
    """In-kernel timing of the fused value+gradient pass (A(UU') and (C + A*(q))U,
    one team pass) and of the constraint map on H(d,2), algorithmic bytes per
    SURVEY §8(d) / DESIGN §3; traffic from the committed ncu capture."""
    import time as _t
    t0 = _t.perf_counter()
    inst = H.build_theta_instance(H.make_hypercube(d))
    gen = _t.perf_counter() - t0
    rng = np.random.default_rng(0)
    U = rng.standard_normal((inst.n, s))
    U /= np.linalg.norm(U)
    p = rng.standard_normal(inst.m)
    npairs = inst.m - 1
    out = {"instance": f"theta H({d},2): n={inst.n}, m={inst.m}, s={s}", "gen_s": round(gen, 2),
           "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "bound": "hbm"}
    ns = inst.bench_pass("grad_pass", U, p, beta=10.0, iters=iters)
    alg = algorithmic_bytes_grad_pass(inst.n, npairs, s)
    out["grad_pass"] = {"ns_per_pass": ns, "algorithmic_bytes": alg,
                        "achieved": alg / (ns * 1e-9) / 1e9, "frac": alg / (ns * 1e-9) / 1e9 / peak}
    ns = inst.bench_pass("map_pass", U, p, beta=10.0, iters=iters)
    alg = 16 * npairs + 8 * inst.n * s
    out["map_pass"] = {"ns_per_pass": ns, "algorithmic_bytes": alg,
                       "achieved": alg / (ns * 1e-9) / 1e9, "frac": alg / (ns * 1e-9) / 1e9 / peak}
    ns = inst.bench_pass("lanczos_matvec", U, p, beta=10.0, iters=iters)
    alg = 24 * npairs + 32 * inst.n
    out["lanczos_matvec"] = {"ns_per_pass": ns, "algorithmic_bytes": alg,
                             "achieved": alg / (ns * 1e-9) / 1e9, "frac": alg / (ns * 1e-9) / 1e9 / peak}
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            out["grad_pass"]["traffic"] = json.load(f).get(f"grad_pass_H{d}_s{s}_bytes_per_pass")
    del inst
    return out


def north_star_matcomp(H):
    """Time-to-1e-5 of SURVEY §8 C4, McSpec{400000, 600000, 3, seed 0}
    (n = 1,000,000 rows, m = 124,339,596 samples) on one B200: one device
    solve after a warm-up solve, instance resident in HBM."""
    import time as _t
    t0 = _t.perf_counter()
    inst = H.gen_matrix_completion(H.McSpec(400000, 600000, 3, seed=0))
    gen = _t.perf_counter() - t0
    cfg = H.SolverConfig(eps=1e-5, seed=0)
    H.solve(inst, cfg, fetch=False)
    r = H.solve(inst, cfg, fetch=False)
    out = {"instance": f"matrix completion 400000 x 600000, r=3: n={inst.n}, m={inst.m}",
           "metric": "time-to-1e-5 rel. precision (s)", "status": r.status,
           "device_s": r.device_seconds, "wall_s": r.wall_seconds, "gen_s": round(gen, 2),
           "pval": r.pval, "nuclear_norm": inst.nuclear_norm,
           "rel": [r.rel_pfeas, r.rel_gap, r.rel_dfeas], "rank": r.rank,
           "counters": {"outer": r.outer_iters, "fista": r.fista_iters, "eig": r.eig_products}}
    del inst
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-large", action="store_true", help="skip the H(23,2) pass roofline and the C4 solve")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return

    import numpy as np
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2505_13719_b200 as H

    graph = H.make_hypercube(HYPERCUBE_D)
    inst = H.build_theta_instance(graph)
    cfg = H.SolverConfig(eps=1e-5, seed=0)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        r = H.solve(inst, cfg, fetch=False)
        assert r.status == "optimal", r.status
    barrier()
    clocks = ClockSampler(local).start()
    t_wall = time.perf_counter()
    times, reps = [], []
    for k in range(args.steps):
        flush.fill_(float(k))  # > 126 MB L2: every step starts cold
        torch.cuda.synchronize()
        r = H.solve(inst, cfg, fetch=False)
        assert r.status == "optimal", r.status
        times.append(r.device_seconds)
        reps.append(r)
    barrier()
    wall = time.perf_counter() - t_wall
    clk = clocks.stop()
    value = statistics.mean(times)

    # e2e: the reference-facing call with host buffers, copies inside the region
    edges = None
    ei, ej = inst.pairs()
    e2e_times, h2d, d2h = [], 0, 0
    for k in range(-1, args.steps):  # one untimed warm-up pass (first-use allocations)
        flush.fill_(float(k))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g = H.graph_from_edges(inst.n, np.stack([ei, ej], axis=1))
        inst2 = H.build_theta_instance(g)
        r2 = H.solve(inst2, cfg, fetch=True)
        t1 = time.perf_counter()
        assert r2.status == "optimal"
        if k >= 0:
            e2e_times.append(t1 - t0)
        h2d = inst2.info()["h2d_bytes"]
        d2h = r2.U.nbytes + r2.p.nbytes
        del inst2
    e2e = statistics.mean(e2e_times)

    if dist is not None:
        t = torch.tensor([value, e2e, wall], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        value, e2e, wall = t.tolist()

    # roofline of the dominant phase (fused value+gradient row pass), timed in-kernel
    rng = np.random.default_rng(0)
    s = reps[-1].rank
    U = rng.standard_normal((inst.n, s))
    U /= np.linalg.norm(U)
    p = rng.standard_normal(inst.m)
    ns = inst.bench_pass("grad_pass", U, p, beta=10.0, iters=400)
    ns_sync = inst.bench_pass("sync", U, p, iters=2000)
    ns_red = inst.bench_pass("allreduce", U, p, iters=2000)
    alg = algorithmic_bytes_grad_pass(inst.n, inst.m - 1, s)
    peak, peak_kind = measured_peaks()
    achieved = alg / (ns * 1e-9) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(f"grad_pass_H12_s{s}_bytes_per_pass")

    # the north-star instance (SURVEY §8 C5, H(23,2): n = 8.4M, m = 96.5M): the
    # A / A* passes where HBM bandwidth, not latency, bounds them
    large = None
    c4 = None
    if not args.no_large:
        large = large_roofline(H, np, peak, peak_kind)
        c4 = north_star_matcomp(H)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "l2": "flushed between steps (256 MiB write)",
                   "team_ctas": inst.info()["team_ctas"], "parallelism": f"replicas x{world}"},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "fused (C + A*(p+beta(A(UU')-b)))U row pass + reductions (one team pass)",
                     "algorithmic_bytes": alg, "ns_per_pass": ns, "peak_kind": peak_kind,
                     "team_sync_ns": ns_sync, "team_allreduce_ns": ns_red},
        "roofline_c5": large,
        "solve_c4": c4,
        "clocks": clk,
        "wall_s_timed_region": wall,
        "counters": {"outer": reps[-1].outer_iters, "fista": reps[-1].fista_iters,
                     "eig": reps[-1].eig_products, "rank": reps[-1].rank, "pval": reps[-1].pval,
                     "rel": [reps[-1].rel_pfeas, reps[-1].rel_gap, reps[-1].rel_dfeas]},
    }
    if rank == 0 and not args.no_cpu_baseline:
        cr, cw = cpu_reference_solve()
        line["cpu_baseline"] = {"value": cr.wall_seconds, "unit": UNIT, "cores": os.cpu_count(),
                                "kind": "port",
                                "sample": f"1 full solve of H(12,2) to 1e-5 (oracle port, fista_iters "
                                          f"{cr.fista_iters}, pval {cr.pval:.10g})"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
