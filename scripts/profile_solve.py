"""Per-phase device-time breakdown of a solve (cfg.profile) and a team-size sweep.

python scripts/profile_solve.py H12 mc2000_2000_3 --ctas 0 74 37
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build(H, name):
    if name.startswith("H"):
        return H.build_theta_instance(H.make_hypercube(int(name[1:])))
    if name == "C5":
        return H.build_theta_instance(H.make_cycle(5))
    n1, n2, r = [int(x) for x in name[2:].split("_")]
    return H.gen_matrix_completion(H.McSpec(n1, n2, r, seed=0))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="+")
    ap.add_argument("--ctas", type=int, nargs="+", default=[0])
    args = ap.parse_args()
    import paper_2505_13719_b200 as H
    for name in args.names:
        inst = build(H, name)
        for ct in args.ctas:
            cfg = H.SolverConfig(profile=True, team_ctas=ct)
            H.solve(inst, cfg, fetch=False)
            r = H.solve(inst, cfg, fetch=False)
            prof = inst.last_profile()
            tot = sum(v[0] for v in prof.values())
            row = {"inst": name, "team_ctas": ct, "status": r.status, "device_ms": r.device_seconds * 1e3,
                   "fista": r.fista_iters, "eig": r.eig_products, "profiled_ms": tot,
                   "phases": {k: {"ms": round(v[0], 3), "n": v[1], "us_each": round(1e3 * v[0] / max(1, v[1]), 2)}
                              for k, v in prof.items() if v[1]}}
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
