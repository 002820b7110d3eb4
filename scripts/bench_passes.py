"""Per-pass device timing (inside one persistent launch) and algorithmic GB/s.

python scripts/bench_passes.py H12 H18 H23 mc2000_2000_3 mc400000_600000_3 --s 1 2 3
Prints one JSON line per (instance, pass, s).  Algorithmic bytes per pass:
  grad_pass       24 B per pair constraint (upper col+p, lower col+p) [+16 B b for MC]
                  + 16 n (row pointers) + 16 n s (own U row read, gradient row write)
  map_pass        16 B per pair (i, j int32 + p) [+8 B b for MC] + 8 n s (U once)
  lanczos_matvec  24 B per pair (col + q, both halves) + 16 n + 16 n (v read, w write)
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
    if name.startswith("mc"):
        n1, n2, r = [int(x) for x in name[2:].split("_")]
        return H.gen_matrix_completion(H.McSpec(n1, n2, r, seed=0))
    raise KeyError(name)


def alg_bytes(kind, n, npairs, s, mc):
    if kind == "grad_pass":
        return (24 + (16 if mc else 0)) * npairs + 16 * n + 16 * n * s
    if kind == "map_pass":
        return (16 + (8 if mc else 0)) * npairs + 8 * n * s
    if kind == "lanczos_matvec":
        return 24 * npairs + 32 * n
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="+")
    ap.add_argument("--s", type=int, nargs="+", default=[2])
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--kinds", nargs="+", default=["sync", "allreduce", "grad_pass", "map_pass", "lanczos_matvec"])
    args = ap.parse_args()
    import numpy as np
    import paper_2505_13719_b200 as H
    peak = 6537.3
    pj = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pj):
        peak = json.load(open(pj)).get("hbm_gbs", peak)
    for name in args.names:
        t0 = time.time()
        inst = build(H, name)
        gen = time.time() - t0
        mc = inst.identity_constraint is None
        npairs = inst.m if mc else inst.m - 1
        rng = np.random.default_rng(0)
        p = rng.standard_normal(inst.m)
        for s in args.s:
            U = rng.standard_normal((inst.n, s))
            U /= np.linalg.norm(U)
            for kind in args.kinds:
                it = args.iters if kind not in ("sync", "allreduce") else 2000
                ns = inst.bench_pass(kind, U, p, beta=10.0, iters=it)
                b = alg_bytes(kind, inst.n, npairs, s, mc)
                row = dict(inst=name, n=inst.n, m=inst.m, s=s, kind=kind, us=ns / 1e3,
                           alg_bytes=b, gbs=(b / (ns * 1e-9) / 1e9) if b else None,
                           frac=(b / (ns * 1e-9) / 1e9 / peak) if b else None, gen_s=round(gen, 2),
                           team_ctas=inst.info()["team_ctas"])
                print(json.dumps(row), flush=True)
        del inst


if __name__ == "__main__":
    main()
