"""SELL engine vs the row-thread engine: bitwise-equal operator outputs and
in-kernel pass timings at C4 (MC 400k x 600k, s = 3) and C5 (H(23,2), s = 2)."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2505_13719_b200 as H

def build(name, sell):
    if sell:
        os.environ.pop("CUHALLAR_NO_SELL", None)
    else:
        os.environ["CUHALLAR_NO_SELL"] = "1"
    if name == "C4":
        return H.gen_matrix_completion(H.McSpec(400000, 600000, 3, seed=0)), 3
    return H.build_theta_instance(H.make_hypercube(int(name[1:]))), 2

for name in sys.argv[1:]:
    out = {"instance": name}
    res = {}
    for sell in (True, False):
        inst, s = build(name, sell)
        rng = np.random.default_rng(0)
        U = rng.standard_normal((inst.n, s)); U /= np.linalg.norm(U)
        p = rng.standard_normal(inst.m)
        g = inst.al_gradient(U, p, 3.0)
        q = inst.C_plus_adjoint(p, U[:, :1])
        t = {}
        for kind in ("grad_pass", "lanczos_matvec", "map_pass"):
            Uk = U[:, :1] if kind == "lanczos_matvec" else U
            inst.bench_pass(kind, Uk, p, beta=10.0, iters=2)
            t[kind] = inst.bench_pass(kind, Uk, p, beta=10.0, iters=40) / 1e6
        res[sell] = (g, q)
        out["sell" if sell else "rt"] = t
        out["m"], out["n"] = inst.m, inst.n
        del inst
    out["grad_bitwise_equal"] = bool(np.array_equal(res[True][0], res[False][0]))
    out["matvec_bitwise_equal"] = bool(np.array_equal(res[True][1], res[False][1]))
    print(json.dumps(out), flush=True)
os.environ.pop("CUHALLAR_NO_SELL", None)
