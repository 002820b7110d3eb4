"""First differing fista() call between the parity-mode device solve and the
oracle (ORC_DEBUG_FISTA / CUHALLAR_DEBUG_FISTA records).
usage: python scripts/parity_fista_debug.py H12"""
import os
import sys
import tempfile

os.environ["CUHALLAR_DEBUG_FISTA"] = "1"
dbg = os.path.join(tempfile.mkdtemp(), "orc_fista.txt")
os.environ["ORC_DEBUG_FISTA"] = dbg
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_13719_b200 as H  # noqa: E402
from parity_compare import pair  # noqa: E402

inst, ref = pair(sys.argv[1])
ref.solve(eps=1e-5, seed=0)
orc = []
with open(dbg) as f:
    for line in f:
        L0, st, it, L, psi, cap = line.split()
        orc.append((float(L0), int(st), int(it), float(L), float(psi), int(cap)))
ev = []
H.solve(inst, H.SolverConfig(eps=1e-5, seed=0, parity=True), sink=ev.append)
dev = [(e.eps_inner, int(e.rank), e.outer_iter, e.gap, e.theta, int(e.fw_alpha)) for e in ev
       if e.kind == "fista_debug"]
print("calls: oracle", len(orc), "device", len(dev))
for i, (a, b) in enumerate(zip(orc, dev)):
    if a != b:
        print("first difference at call", i)
        for j in range(max(0, i - 2), min(i + 3, len(orc), len(dev))):
            print(j, "oracle", orc[j])
            print(j, "device", dev[j])
        break
else:
    print("all common calls identical")
