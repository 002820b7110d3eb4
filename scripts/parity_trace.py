"""First divergence between the parity-mode device trace and the oracle trace.
usage: python scripts/parity_trace.py H12"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_13719_b200 as H  # noqa: E402
from parity_compare import pair  # noqa: E402

FIELDS = ["kind", "outer_iter", "beta", "eps_inner", "gap", "theta", "rank", "al_value", "fw_alpha",
          "rel_pfeas", "rel_gap", "rel_dfeas"]
name = sys.argv[1]
inst, ref = pair(name)
o = ref.solve(eps=1e-5, seed=0, trace=True)
ev = []
r = H.solve(inst, H.SolverConfig(eps=1e-5, seed=0, parity=True), sink=ev.append)
kinds = {"inner_stationary": 0, "inner_rank_step": 1, "outer": 2}
print("oracle events", len(o.trace), "device events", len(ev))
for i, (a, b) in enumerate(zip(o.trace, ev)):
    da = {f: a[f] for f in FIELDS}
    db = {f: getattr(b, f) for f in FIELDS}
    if isinstance(da["kind"], str):
        da["kind"] = kinds[da["kind"]]
    db["kind"] = kinds[db["kind"]] if isinstance(db["kind"], str) else db["kind"]
    diff = [f for f in FIELDS if da[f] != db[f]]
    print(i, da["kind"], da["outer_iter"], "OK" if not diff else "DIFF " + ",".join(diff))
    if diff:
        print(json.dumps({"oracle": da, "device": db}, default=float))
        break
