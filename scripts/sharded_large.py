"""Row-sharded solve at full size on one device (world co-resident launches):
python scripts/sharded_large.py mc400000_600000_3 2   -> one JSON line (single vs sharded)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def build(H, name):
    if name.startswith("H"):
        return H.build_theta_instance(H.make_hypercube(int(name[1:])))
    if name.startswith("mcp"):  # the paper's sampling rule
        n1, n2, r = [int(x) for x in name[3:].split("_")]
        return H.gen_matrix_completion(H.McSpec(n1, n2, r, seed=0, draws_per_dim=40))
    n1, n2, r = [int(x) for x in name[2:].split("_")]
    return H.gen_matrix_completion(H.McSpec(n1, n2, r, seed=0))


def main():
    import paper_2505_13719_b200 as H
    name, world = sys.argv[1], int(sys.argv[2])
    insts = [build(H, name) for _ in range(world)]
    cfg = H.SolverConfig(eps=1e-5, seed=0, time_limit=float(os.environ.get("TL", "900")))
    single = H.solve(insts[0], cfg, fetch=False)
    t0 = time.time()
    shard = H.solve_sharded(insts, cfg, fetch=False)
    row = {"inst": name, "world": world, "n": insts[0].n, "m": insts[0].m,
           "single": {"status": single.status, "device_s": single.device_seconds, "pval": single.pval,
                      "fista": single.fista_iters, "rank": single.rank},
           "sharded": {"status": shard.status, "device_s": shard.device_seconds, "pval": shard.pval,
                       "fista": shard.fista_iters, "rank": shard.rank, "wall_s": time.time() - t0,
                       "rel": [shard.rel_pfeas, shard.rel_gap, shard.rel_dfeas]},
           "pval_rel_diff": abs(shard.pval - single.pval) / max(1.0, abs(single.pval))}
    print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
