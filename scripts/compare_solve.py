"""Device solve vs oracle solve on named configs: counters, objective, time.

Usage: python scripts/compare_solve.py H10 H12 mc100 ...   (oracle optional: --no-oracle)
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def make(H, O, name):
    if name.startswith("H"):
        d = int(name[1:])
        return H.build_theta_instance(H.make_hypercube(d)), (lambda: O.OracleInstance.hypercube(d))
    if name == "C5":
        return H.build_theta_instance(H.make_cycle(5)), (lambda: O.OracleInstance.cycle(5))
    if name == "petersen":
        return H.build_theta_instance(H.make_petersen()), O.OracleInstance.petersen
    if name.startswith("mc"):
        n1, n2, r = [int(x) for x in name[2:].split("_")]
        return (H.gen_matrix_completion(H.McSpec(n1, n2, r, seed=0)),
                (lambda: O.OracleInstance.matcomp(n1, n2, r, seed=0)))
    raise KeyError(name)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="+")
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--repeat", type=int, default=2)
    args = ap.parse_args()
    import paper_2505_13719_b200 as H
    from oracle import oracle as O
    for name in args.names:
        t0 = time.time()
        inst, mk = make(H, O, name)
        gen_s = time.time() - t0
        reps = [H.solve(inst) for _ in range(args.repeat)]
        r = reps[-1]
        row = dict(name=name, n=inst.n, m=inst.m, gen_s=round(gen_s, 3), status=r.status, pval=r.pval,
                   rank=r.rank, outer=r.outer_iters, fw=r.fw_steps, aipp=r.aipp_iters, fista=r.fista_iters,
                   eig=r.eig_products, wall_s=[round(x.wall_seconds, 4) for x in reps],
                   dev_s=[round(x.device_seconds, 4) for x in reps],
                   res=[r.rel_pfeas, r.rel_gap, r.rel_dfeas])
        if not args.no_oracle:
            o = mk().solve()
            row["oracle"] = dict(status=o.status, pval=o.pval, rank=o.rank, outer=o.outer_iters, fw=o.fw_steps,
                                 aipp=o.aipp_iters, fista=o.fista_iters, eig=o.eig_products,
                                 wall_s=round(o.wall_seconds, 3))
            row["pval_rel_diff"] = abs(r.pval - o.pval) / max(1.0, abs(o.pval))
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
