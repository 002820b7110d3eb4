"""A large solve with the per-FISTA-call debug trace (kind 9) and the phase
profile: where the FISTA iterations go (per outer iteration: FISTA calls,
iterations, status mix, final curvature L), for the north-star H(d,2) runs.

python scripts/solve_large_trace.py H23 --time-limit 2400 [--parity]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
os.environ["CUHALLAR_DEBUG_FISTA"] = "1"
import paper_2505_13719_b200 as H  # noqa: E402


def build(name):
    if name.startswith("H"):
        return H.build_theta_instance(H.make_hypercube(int(name[1:])))
    if name.startswith("mc"):
        n1, n2, r = [int(x) for x in name[2:].split("_")]
        return H.gen_matrix_completion(H.McSpec(n1, n2, r, seed=0))
    if name.startswith("pr"):
        nc, L = [int(x) for x in name[2:].split("_")]
        return H.gen_phase_retrieval(H.PrSpec(nc, L, seed=0))
    raise KeyError(name)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--time-limit", type=float, default=3600.0)
    ap.add_argument("--parity", action="store_true")
    a = ap.parse_args()
    t0 = time.perf_counter()
    inst = build(a.name)
    gen = time.perf_counter() - t0
    ev = []
    t_solve = time.perf_counter()
    fcalls = [0, 0]

    def sink(e):  # live: progress survives a killed run
        ev.append(e)
        if e.kind == "fista_debug":
            fcalls[0] += 1
            fcalls[1] += e.outer_iter
        elif e.kind == "outer":
            print(json.dumps({"t": round(time.perf_counter() - t_solve, 1), "outer": e.outer_iter,
                              "beta": e.beta, "rank": e.rank, "rel_pfeas": e.rel_pfeas,
                              "rel_gap": e.rel_gap, "fista_calls": fcalls[0], "fista_iters": fcalls[1]}),
                  file=sys.stderr, flush=True)

    cfg = H.SolverConfig(eps=1e-5, seed=0, time_limit=a.time_limit, profile=True, parity=a.parity)
    r = H.solve(inst, cfg, sink=sink, fetch=False)
    outer, cur = [], {"calls": 0, "iters": 0, "success": 0, "failure": 0, "limit": 0, "L_max": 0.0,
                      "lambda_min": None}
    for e in ev:
        if e.kind == "fista_debug":
            cur["calls"] += 1
            cur["iters"] += e.outer_iter
            cur[["success", "failure", "limit"][min(e.rank, 2)]] += 1
            cur["L_max"] = max(cur["L_max"], e.gap)
            lam = e.fw_alpha
            cur["lambda_min"] = lam if cur["lambda_min"] is None else min(cur["lambda_min"], lam)
        elif e.kind == "outer":
            cur.update({"outer": e.outer_iter, "beta": e.beta, "eps_inner": e.eps_inner, "rank": e.rank,
                        "rel_pfeas": e.rel_pfeas, "rel_gap": e.rel_gap})
            outer.append(cur)
            cur = {"calls": 0, "iters": 0, "success": 0, "failure": 0, "limit": 0, "L_max": 0.0,
                   "lambda_min": None}
    prof = inst.last_profile()
    print(json.dumps({
        "instance": a.name, "n": inst.n, "m": inst.m, "gen_s": round(gen, 2), "parity": a.parity,
        "status": r.status, "message": r.message, "device_s": r.device_seconds, "wall_s": r.wall_seconds,
        "pval": r.pval, "rel": [r.rel_pfeas, r.rel_gap, r.rel_dfeas], "rank": r.rank,
        "counters": {"outer": r.outer_iters, "fw": r.fw_steps, "aipp": r.aipp_iters, "fista": r.fista_iters,
                     "eig": r.eig_products},
        "per_outer": outer,
        "phases": {k: {"ms": round(v[0], 1), "n": v[1]} for k, v in prof.items() if v[1]},
    }), flush=True)


if __name__ == "__main__":
    main()
