"""Gaussian-measurement phase retrieval (BASELINE configs[2]: n = 10^4, m = 12 n)
to 1e-5 on one B200: instance generation, operator pass timings (forward +
adjoint DMMA GEMMs) and the solve.  python scripts/solve_gauss.py 10000 120000"""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import paper_2505_13719_b200 as H  # noqa: E402

n, m = int(sys.argv[1]), int(sys.argv[2])
tl = float(sys.argv[3]) if len(sys.argv) > 3 else 1200.0
t0 = time.perf_counter()
inst = H.gen_gauss_phase_retrieval(H.GaussPrSpec(n, m, seed=0))
gen = time.perf_counter() - t0
rng = np.random.default_rng(0)
out = {"n": n, "m": m, "gen_s": round(gen, 2), "A_bytes": 16 * n * m}
for s in (1, 2, 4):
    U = rng.standard_normal((2 * n, s)); U /= np.linalg.norm(U)
    p = rng.standard_normal(m)
    inst.bench_pass("map_pass", U, p, beta=1.0, iters=2)
    tmap = inst.bench_pass("map_pass", U, p, beta=1.0, iters=10) / 1e6
    tgrad = inst.bench_pass("grad_pass", U, p, beta=1.0, iters=10) / 1e6
    # map: one streaming of A' (16 m n bytes); grad: forward + adjoint = two
    out[f"s{s}"] = {"map_ms": tmap, "grad_ms": tgrad,
                    "map_GBs": 16 * n * m / (tmap * 1e-3) / 1e9,
                    "grad_GBs": 32 * n * m / (tgrad * 1e-3) / 1e9,
                    "map_TFs": 8 * m * n * 2 * (2 * ((s + 3) // 4) * 4) / 2 / (tmap * 1e-3) / 1e12}
print(json.dumps({k: v for k, v in out.items()}), flush=True)  # pass timings first
cfg = H.SolverConfig(eps=1e-5, seed=0, time_limit=tl, profile=True)
ev = []
t_solve = time.perf_counter()


def sink(e):
    ev.append(e)
    if e.kind == "outer":
        print(json.dumps({"t": round(time.perf_counter() - t_solve, 1), "outer": e.outer_iter, "beta": e.beta,
                          "rank": e.rank, "rel_pfeas": e.rel_pfeas, "rel_gap": e.rel_gap}), file=sys.stderr,
              flush=True)


r = H.solve(inst, cfg, sink=sink)
_, x = inst.gauss_data() if n * m <= 4e7 else (None, None)
out.update({"status": r.status, "device_s": r.device_seconds, "rank": r.rank, "pval": r.pval,
            "rel": [r.rel_pfeas, r.rel_gap, r.rel_dfeas],
            "counters": {"outer": r.outer_iters, "aipp": r.aipp_iters, "fista": r.fista_iters,
                         "eig": r.eig_products}})
if x is not None:
    u = r.U[:n, 0] + 1j * r.U[n:, 0]
    out["overlap"] = float(abs(np.vdot(u, x)) / np.linalg.norm(u) / np.linalg.norm(x))
prof = inst.last_profile()
out["phases"] = {k: {"ms": round(v[0], 1), "n": v[1]} for k, v in prof.items() if v[1]}
print(json.dumps(out), flush=True)
