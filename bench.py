#!/usr/bin/env python
"""HALLaR time-to-1e-5 on B200 — the BASELINE.json headline metric, on the
largest single-GPU configuration (BASELINE configs[3]).

Workload: matrix completion McSpec{400000, 600000, r = 3, seed = 0} (reference
sampling rule, instances.cpp:123-175): n = 1,000,000 rows of U, m = 124,339,596
samples, SolverConfig{eps = 1e-5, seed = 0}, all other reference defaults.
One "step" = one full solve to 1e-5 relative precision.

  value  device time of the persistent solve kernel, instance resident in HBM
         (6 GB of constraint data, > L2: no flush needed), CUDA events on the
         launching stream, mean over K steps, max over ranks
  e2e    the same solve through the reference-facing C-ABI with HOST buffers:
         cuhallar_matcomp_from_samples(i, j, b from pinned host memory: H2D and
         the pair CSR built on the GPU), the solve, U and p read back (D2H)
  roofline  the fused (C + A*(p + beta(A(UU') - b)))U row pass at C4, s = 3,
         SURVEY §8(d) bytes 16 m + 16 n s, CUDA-event timed (difference of two
         launches of 60 and 10 passes) and CTA-0 globaltimer timed

`--impl reference` runs the reference algorithm's CPU implementation (the oracle
port in oracle/ -- the reference itself cannot be built: no Eigen)
on the host cores: it cannot finish C4 in minutes (hours), so each
step times one apply_map, one C_plus_adjoint at s = 3 and one at s = 1 (the
Lanczos matvec) on the C4 instance and reports the time-to-1e-5 those per-call
costs give on the solve's call counts (A5: 3 maps + 2 fused adjoints per FISTA
iteration, 1 s = 1 matvec per eig product; CGS2, doublings and BLAS-1 ignored, so
it is a lower bound on the CPU time).  Multi-GPU: N independent replicas.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time-to-1e-5 rel. precision (s)"
UNIT = "s"
C4 = dict(n1=400000, n2=600000, r=3, seed=0)
WORKLOAD = ("matrix completion McSpec{400000, 600000, r=3, seed=0}: n=1,000,000, m=124,339,596, "
            "eps=1e-5 (SURVEY C4 / BASELINE configs[3], 1 GPU)")
# call counts of the C4 solve (fast mode; on matrix completion its counters equal
# the oracle's, tests/test_gpu_parity_mode.py) -- profiles/r02_c4_counters.json
COUNTS_FILE = os.path.join(ROOT, "profiles", "r02_c4_counters.json")


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


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


# ------------------------------------------------------------ CPU (oracle) --
def load_counts():
    with open(COUNTS_FILE) as f:
        return json.load(f)


def oracle_c4():
    from oracle import oracle as O
    t0 = time.perf_counter()
    inst = O.OracleInstance.matcomp(C4["n1"], C4["n2"], C4["r"], seed=C4["seed"])
    return inst, time.perf_counter() - t0


def oracle_kernel_sample(inst, np):
    """One apply_map, one C_plus_adjoint at s = 3 and at s = 1 on the C4 instance
    (the oracle's own parallel_for threading: map over constraints, adjoint over
    columns, instances.cpp:27-55)."""
    rng = np.random.default_rng(1)
    U = rng.standard_normal((inst.n, 3))
    U /= np.linalg.norm(U)
    p = rng.standard_normal(inst.m)
    t = {}
    t0 = time.perf_counter(); inst.apply_map(U); t["map_s3"] = time.perf_counter() - t0
    t0 = time.perf_counter(); inst.C_plus_adjoint(p, U); t["c_plus_adjoint_s3"] = time.perf_counter() - t0
    t0 = time.perf_counter(); inst.C_plus_adjoint(p, U[:, :1]); t["matvec_s1"] = time.perf_counter() - t0
    return t


def cpu_time_to_eps(t, counts):
    """A5 accounting on the solve's counters: per FISTA iteration 3 maps + 2 fused
    adjoints (no doublings), per eig product one s = 1 adjoint (CGS2 ignored)."""
    return (counts["fista_iters"] * (3 * t["map_s3"] + 2 * t["c_plus_adjoint_s3"])
            + counts["eig_products"] * t["matvec_s1"])


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    counts = load_counts()
    inst, gen_s = oracle_c4()
    vals, samples = [], []
    for k in range(args.warmup + args.steps):
        t = oracle_kernel_sample(inst, np)
        if k >= args.warmup:
            vals.append(cpu_time_to_eps(t, counts))
            samples.append(t)
    v = statistics.mean(vals)
    cores = os.cpu_count()
    med = {k: statistics.median(s[k] for s in samples) for k in samples[0]}
    line = {
        "metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": WORKLOAD},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": ("per step: 1 apply_map + 1 C_plus_adjoint (s=3) + 1 Lanczos-matvec "
                                    "adjoint (s=1) of the oracle port on C4 (reference threading, "
                                    f"{cores} host threads); value = A5 call counts of the solve "
                                    f"(fista {counts['fista_iters']}, eig {counts['eig_products']}) x "
                                    "per-call time, a lower bound (no doublings / CGS2 / BLAS-1)"),
                         "per_call_s": med, "instance_gen_s": round(gen_s, 1)},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- ours ----
def pass_roofline(H, inst, np, torch, peak, peak_kind, s=3):
    """Dominant phase at C4: the fused value+gradient row pass; and the map."""
    rng = np.random.default_rng(0)
    U = rng.standard_normal((inst.n, s))
    U /= np.linalg.norm(U)
    p = rng.standard_normal(inst.m)
    m, n = inst.m, inst.n
    out = {}
    for kind, alg in (("grad_pass", 16 * m + 16 * n * s), ("map_pass", 16 * m + 8 * n * s),
                      ("lanczos_matvec", 16 * m + 16 * n)):
        ss = 1 if kind == "lanczos_matvec" else s
        Uk = U[:, :ss]
        inst.bench_pass(kind, Uk, p, beta=10.0, iters=2)  # first use: workspace allocation
        ev = []
        for iters in (10, 60):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            ns_k = inst.bench_pass(kind, Uk, p, beta=10.0, iters=iters)
            e1.record()
            torch.cuda.synchronize()
            ev.append(e0.elapsed_time(e1))
        ns_event = (ev[1] - ev[0]) * 1e6 / 50.0
        ach = alg / (ns_event * 1e-9) / 1e9
        out[kind] = {"ns_per_pass_event": ns_event, "ns_per_pass_globaltimer": ns_k,
                     "algorithmic_bytes": alg, "achieved": ach, "frac": ach / peak}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the H(12,2) / H(23,2) extras")
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

    t0 = time.perf_counter()
    inst = H.gen_matrix_completion(H.McSpec(C4["n1"], C4["n2"], C4["r"], seed=C4["seed"]))
    gen_s = time.perf_counter() - t0
    cfg = H.SolverConfig(eps=1e-5, seed=0)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # N > 1: one C4 instance row-sharded over the N GPUs (one process per GPU,
    # peers mapped through CUDA IPC); falls back to N replicas
    # if the sharded solve cannot run on this box
    mode = "replicas"
    handles = None
    if dist is not None:
        try:
            hb = H.shard_export(inst)
            handles = [None] * world
            dist.all_gather_object(handles, hb)
            barrier()
            r = H.solve_rank(inst, world, rank, handles, cfg)
            ok = torch.tensor([1.0 if r.status == "optimal" else 0.0], device="cuda")
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            mode = "sharded" if ok.item() == 1.0 else "replicas"
        except Exception as e:  # noqa: BLE001
            print(f"[rank {rank}] sharded solve unavailable ({e}); replicas", file=sys.stderr)
            mode = "replicas"

    def one_solve():
        if mode == "sharded":
            barrier()
            return H.solve_rank(inst, world, rank, handles, cfg)
        return H.solve(inst, cfg, fetch=False)

    for _ in range(args.warmup):
        r = one_solve()
        assert r.status == "optimal", r.status
    barrier()
    clocks = ClockSampler(local).start()
    t_wall = time.perf_counter()
    times, reps = [], []
    for k in range(args.steps):
        r = one_solve()
        assert r.status == "optimal", r.status
        times.append(r.device_seconds)
        reps.append(r)
    barrier()
    wall = time.perf_counter() - t_wall
    clk = clocks.stop()
    value = statistics.mean(times)
    last = reps[-1]

    # e2e: host sample arrays (pinned) -> cuhallar_matcomp_from_samples -> solve -> U, p back
    ei, ej = inst.pairs()
    hb = inst.b
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    ei, ej, hb = pin(ei), pin(ej), pin(hb)
    tau = inst.tau
    e2e_times, h2d, d2h = [], 0, 0
    for k in range(-1, args.steps):  # one untimed warm-up pass
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        inst2 = H.matcomp_from_samples(C4["n1"], C4["n2"], ei, ej, hb, tau)
        if mode == "sharded":
            h2 = [None] * world
            dist.all_gather_object(h2, H.shard_export(inst2))
            barrier()
            r2 = H.solve_rank(inst2, world, rank, h2, cfg, fetch=True)
        else:
            r2 = H.solve(inst2, cfg, fetch=True)
        t1 = time.perf_counter()
        assert r2.status == "optimal" and r2.fista_iters == last.fista_iters
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

    peak, peak_kind = measured_peaks()
    passes = pass_roofline(H, inst, np, torch, peak, peak_kind, s=3)
    g = passes["grad_pass"]
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("grad_pass_C4_s3_bytes_per_pass")
    counts = {"outer_iters": last.outer_iters, "fw_steps": last.fw_steps, "aipp_iters": last.aipp_iters,
              "fista_iters": last.fista_iters, "eig_products": last.eig_products, "rank": last.rank}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False,
        "scaling": "strong" if mode == "sharded" else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "l2": "inputs > L2 (6 GB of constraint data per step); no flush",
                   "team_ctas": inst.info()["team_ctas"],
                   "parallelism": (f"row-sharded x{world} (one process per GPU, CUDA IPC peer memory)"
                                   if mode == "sharded" else f"replicas x{world}"),
                   "instance_gen_s": round(gen_s, 2), "instance_gen": "device (csrc/devgen.cu)"},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": args.steps,
        "roofline": {"bound": "hbm", "achieved": g["achieved"], "peak": peak, "unit": "GB/s",
                     "frac": g["frac"], "traffic": traffic,
                     "kernel": "fused (C + A*(p+beta(A(UU')-b)))U row pass at C4, s=3 (one team pass of "
                               "the persistent kernel)",
                     "algorithmic_bytes": g["algorithmic_bytes"],
                     "bytes_rule": "SURVEY 8(d) K2: 16 m + 16 n s", "peak_kind": peak_kind,
                     "ns_per_pass": g["ns_per_pass_event"], "passes": passes},
        "clocks": clk,
        "wall_s_timed_region": wall,
        "counters": counts,
        "result": {"status": last.status, "pval": last.pval, "nuclear_norm": inst.nuclear_norm,
                   "rel": [last.rel_pfeas, last.rel_gap, last.rel_dfeas]},
    }
    del inst

    if not args.no_secondary and rank == 0:
        # BASELINE configs[1] (H(12,2)) and the north-star passes at C5 (H(23,2))
        hi = H.build_theta_instance(H.make_hypercube(12))
        rs = [H.solve(hi, cfg, fetch=False) for _ in range(4)][1:]
        line["secondary_h12"] = {"device_s": statistics.mean(x.device_seconds for x in rs),
                                 "fista_iters": rs[-1].fista_iters, "rank": rs[-1].rank,
                                 "pval": rs[-1].pval}
        del hi
        t0 = time.perf_counter()
        h23 = H.build_theta_instance(H.make_hypercube(23))
        g23 = time.perf_counter() - t0
        p23 = pass_roofline(H, h23, np, torch, peak, peak_kind, s=2)
        p23["instance_gen_s"] = round(g23, 2)
        line["roofline_c5"] = p23
        del h23

    if rank == 0 and not args.no_cpu_baseline:
        oi, ogen = oracle_c4()
        t = oracle_kernel_sample(oi, np)
        est = cpu_time_to_eps(t, counts)
        line["cpu_baseline"] = {
            "value": est, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "sample": ("1 apply_map + 1 C_plus_adjoint (s=3) + 1 Lanczos-matvec adjoint (s=1) of the oracle "
                       "port on C4, x this solve's A5 call counts (lower bound on the CPU time-to-1e-5)"),
            "per_call_s": t, "instance_gen_s": round(ogen, 1)}
        del oi
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
