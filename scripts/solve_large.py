"""Time-to-1e-5 on the large north-star instances (one device solve each).

python scripts/solve_large.py H20 H23 mc400000_600000_3 mcp3200000_4800000_3 --time-limit 600 [--profile]
(mcpN1_N2_R: the paper's sampling rule, 40 (n1 + n2) draws with replacement, deduplicated)
Prints one JSON line per instance: generation time, device seconds, counters,
residuals, and (with --profile) the per-phase device-time breakdown.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build(H, name):
    if name.startswith("H"):
        return H.build_theta_instance(H.make_hypercube(int(name[1:])))
    if name.startswith("mcp"):  # the paper's sampling rule: 40 (n1 + n2) draws, deduplicated
        n1, n2, r = [int(x) for x in name[3:].split("_")]
        return H.gen_matrix_completion(H.McSpec(n1, n2, r, seed=0, draws_per_dim=40))
    if name.startswith("mc"):
        n1, n2, r = [int(x) for x in name[2:].split("_")]
        return H.gen_matrix_completion(H.McSpec(n1, n2, r, seed=0))
    if name.startswith("pr"):
        n, L = [int(x) for x in name[2:].split("_")]
        return H.gen_phase_retrieval(H.PrSpec(n, L, seed=0))
    raise KeyError(name)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="+")
    ap.add_argument("--time-limit", type=float, default=600.0)
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--eps", type=float, default=1e-5)
    args = ap.parse_args()
    import paper_2505_13719_b200 as H
    for name in args.names:
        t0 = time.time()
        inst = build(H, name)
        gen = time.time() - t0
        cfg = H.SolverConfig(eps=args.eps, time_limit=args.time_limit, profile=args.profile)
        r = H.solve(inst, cfg, fetch=False)
        row = {"inst": name, "n": inst.n, "m": inst.m, "gen_s": round(gen, 2), "status": r.status,
               "device_s": r.device_seconds, "wall_s": r.wall_seconds, "pval": r.pval, "dval": r.dval,
               "rel": [r.rel_pfeas, r.rel_gap, r.rel_dfeas], "rank": r.rank, "outer": r.outer_iters,
               "fw": r.fw_steps, "aipp": r.aipp_iters, "fista": r.fista_iters, "eig": r.eig_products,
               "hbm_bytes": inst.info()["device_bytes"], "message": r.message}
        if args.profile:
            prof = inst.last_profile()
            row["phases_ms"] = {k: [round(v[0], 2), v[1]] for k, v in prof.items() if v[1]}
        print(json.dumps(row), flush=True)
        del inst


if __name__ == "__main__":
    main()
