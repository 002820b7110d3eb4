"""Parity mode vs the CPU oracle: counters and objective side by side.
usage: python scripts/parity_compare.py C5 petersen H4 H10 H12 mc30 mc100 mc2000 ..."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_13719_b200 as H  # noqa: E402
from oracle import oracle as O  # noqa: E402


def pair(name):
    if name == "C5":
        return H.build_theta_instance(H.make_cycle(5)), O.OracleInstance.cycle(5)
    if name == "petersen":
        return H.build_theta_instance(H.make_petersen()), O.OracleInstance.petersen()
    if name.startswith("H"):
        d = int(name[1:])
        return H.build_theta_instance(H.make_hypercube(d)), O.OracleInstance.hypercube(d)
    if name.startswith("mc"):
        spec = {"mc30": (30, 70, 2, 5), "mc100": (100, 210, 3, 0), "mc2000": (2000, 2000, 3, 0),
                "mc300": (300, 700, 3, 0), "mc1000": (1000, 1000, 3, 0)}[name]
        n1, n2, r, seed = spec
        return (H.gen_matrix_completion(H.McSpec(n1, n2, r, seed=seed)),
                O.OracleInstance.matcomp(n1, n2, r, seed=seed))
    raise KeyError(name)


KEYS = ["status", "outer_iters", "fw_steps", "aipp_iters", "fista_iters", "eig_products", "rank"]


def main(names):
  for name in names:
      inst, ref = pair(name)
      t0 = time.perf_counter()
      o = ref.solve(eps=1e-5, seed=0)
      to = time.perf_counter() - t0
      rows = {"name": name, "oracle_s": round(to, 3)}
      for mode in (True, False):
          r = H.solve(inst, H.SolverConfig(eps=1e-5, seed=0, parity=mode))
          tag = "parity" if mode else "fast"
          rows[tag] = {k: getattr(r, k) for k in KEYS}
          rows[tag]["pval"] = r.pval
          rows[tag]["device_s"] = round(r.device_seconds, 4)
          rows[tag]["pval_bitwise"] = r.pval == o.pval
          rows[tag]["counters_equal"] = all(getattr(r, k) == getattr(o, k) for k in KEYS)
      rows["oracle"] = {k: getattr(o, k) for k in KEYS}
      rows["oracle"]["pval"] = o.pval
      rows["oracle"]["message"] = o.message
      print(json.dumps(rows), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
