"""Command-line solve and JSON report, mirroring the reference CLI's ``solve``
subcommand (tools/main.cpp:541-610) and its report (``report_to_json``,
tools/main.cpp:311-354; schema docs/report-schema.json) — SURVEY §8(f) row 4.

    python -m paper_2505_13719_b200 solve --problem theta --hypercube 10 --json-out r.json
    python -m paper_2505_13719_b200 solve --problem matcomp --n1 2000 --n2 2000 --r 3
    python -m paper_2505_13719_b200 solve --problem theta --graph g.txt --format edge-list
    python -m paper_2505_13719_b200 solve --spec instance.spec

Same flags, the same instance descriptor, ``b_hash`` / ``config_hash`` (FNV-1a,
tools/main.cpp:30-47, 219-228), the same exit codes (0 optimal, 2 iteration or
time limit, 3 numerical failure, 64 usage / input error, 66 I/O;
tools/main.cpp:21-28, 369-377).  The solve runs on the B200 through the C-ABI;
the reference's optional post-hoc ``verify`` block is not produced (the
report's certificate fields come from the device's own final certify,
solver.cpp:175-201)."""
from __future__ import annotations

import argparse
import json
import sys

EXIT_OPTIMAL, EXIT_LIMIT, EXIT_NUMERICAL, EXIT_USAGE, EXIT_NOINPUT = 0, 2, 3, 64, 66
VERSION = "0.1.0"  # lrsdp kVersion (include/lrsdp/types.hpp:29): the report format mirrored


def fnv1a(data: bytes, h: int = 0xCBF29CE484222325) -> int:
    """64-bit FNV-1a (tools/main.cpp:30-37)."""
    for c in data:
        h ^= c
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def hex64(v: int) -> str:
    return "%016x" % v


def vector_hash(b) -> str:
    """FNV-1a over the raw little-endian doubles of b (tools/main.cpp:45-47)."""
    import numpy as np
    return hex64(fnv1a(np.ascontiguousarray(b, dtype="<f8").tobytes()))


def _num(x) -> str:
    """A double as std::ostream prints it by default (precision 6, %g)."""
    return "%g" % x


def config_hash(o: argparse.Namespace) -> str:
    """tools/main.cpp:219-228: FNV-1a of the option string."""
    s = (f"tol={_num(o.tol)};seed={o.seed};time_limit={_num(o.time_limit)}"
         f";deterministic={int(bool(o.deterministic))};beta0={_num(o.beta0)}"
         f";beta_growth={_num(o.beta_growth)};eps0={_num(o.eps0)}"
         f";eps_decay={_num(o.eps_decay)};eps_floor={_num(o.eps_floor)}"
         f";max_outer={o.max_outer};lambda0={_num(o.lambda0)}")
    return hex64(fnv1a(s.encode()))


def read_spec_file(path: str) -> dict:
    """key=value lines, '#' comments (tools/main.cpp:54-80)."""
    try:
        lines = open(path).read().splitlines()
    except OSError as e:
        raise OSError(f"cannot open spec file '{path}'") from e
    out = {}
    for line in lines:
        t = line.strip()
        if not t or t.startswith("#"):
            continue
        if "=" not in t:
            from .api import InputError
            raise InputError(f"spec line without '=': {t}")
        k, v = t.split("=", 1)
        out[k.strip()] = v.strip()
    return out


def spec_from_flags(f: argparse.Namespace) -> dict:
    """tools/main.cpp:273-309."""
    from .api import InputError
    if f.spec:
        return read_spec_file(f.spec)
    if not f.problem:
        raise InputError("one of --problem or --spec is required")
    spec = {"family": f.problem, "seed": str(f.seed)}
    if f.problem == "matcomp":
        if f.n1 is None or f.n2 is None or f.r is None:
            raise InputError("matcomp needs --n1 --n2 --r")
        spec.update(n1=str(f.n1), n2=str(f.n2), r=str(f.r))
    elif f.problem == "phaseret":
        if f.n is None or f.L is None:
            raise InputError("phaseret needs --n --L")
        spec.update(n=str(f.n), L=str(f.L))
    elif f.problem == "theta":
        del spec["seed"]  # theta instances are seed-free
        if f.graph:
            spec.update(graph=f.graph, format=f.format)
        elif f.hypercube is not None:
            spec["hypercube"] = str(f.hypercube)
        elif f.cycle is not None:
            spec["cycle"] = str(f.cycle)
        elif f.petersen:
            spec["petersen"] = "1"
        else:
            raise InputError("theta needs --graph, --hypercube, --cycle or --petersen")
    else:
        raise InputError(f"unknown problem family '{f.problem}'")
    return spec


def build_from_spec(spec: dict):
    """(instance, descriptor) as tools/main.cpp:106-181 builds them."""
    from . import api as H
    fam = spec.get("family")
    if fam == "matcomp":
        ms = H.McSpec(int(spec["n1"]), int(spec["n2"]), int(spec["r"]), seed=int(spec.get("seed", 0)))
        if "tau_safety" in spec:
            ms.tau_safety = float(spec["tau_safety"])
        if "offset_sample_count" in spec:
            ms.offset_sample_count = spec["offset_sample_count"] == "1"
        inst = H.gen_matrix_completion(ms)
        desc = {"family": "matcomp", "n1": ms.n1, "n2": ms.n2, "r": ms.r, "seed": ms.seed,
                "nuclear_norm": inst.nuclear_norm}
    elif fam == "phaseret":
        ps = H.PrSpec(int(spec["n"]), int(spec["L"]), seed=int(spec.get("seed", 0)))
        if "tau_slack" in spec:
            ps.tau_slack = float(spec["tau_slack"])
        inst = H.gen_phase_retrieval(ps)
        desc = {"family": "phaseret", "n": ps.n, "L": ps.L, "seed": ps.seed}
    elif fam == "theta":
        if "graph" in spec:
            fmt = spec.get("format", "edge-list")
            g, src = H.load_graph(spec["graph"], fmt), {"graph": spec["graph"], "format": fmt}
        elif "hypercube" in spec:
            g, src = H.make_hypercube(int(spec["hypercube"])), {"hypercube": int(spec["hypercube"])}
        elif "cycle" in spec:
            g, src = H.make_cycle(int(spec["cycle"])), {"cycle": int(spec["cycle"])}
        elif "petersen" in spec:
            g, src = H.make_petersen(), {"petersen": True}
        else:
            raise H.InputError("theta needs --graph (with --format), or one of hypercube/cycle/petersen")
        inst = H.build_theta_instance(g)
        desc = {"family": "theta", "vertices": inst.n, "edges": inst.m - 1, "source": src}
    else:
        raise H.InputError(f"unknown problem family '{fam}'")
    desc.update(n=inst.n, m=inst.m, tau=inst.tau, b_hash=vector_hash(inst.b))
    return inst, desc


def make_config(o: argparse.Namespace):
    """tools/main.cpp:201-217."""
    from .api import SolverConfig
    return SolverConfig(eps=o.tol, seed=o.seed, threads=o.threads, time_limit=o.time_limit,
                        deterministic=bool(o.deterministic), beta0=o.beta0, beta_growth=o.beta_growth,
                        eps0=o.eps0, eps_decay=o.eps_decay, eps_floor=o.eps_floor, max_outer=o.max_outer,
                        aipp_lambda0=o.lambda0)


def report_to_json(desc: dict, rep, o: argparse.Namespace, threads: int = 1) -> dict:
    """tools/main.cpp:311-354 (without the optional verify block)."""
    j = {
        "version": VERSION,
        "instance": desc,
        "config_hash": config_hash(o),
        "environment": {"threads": max(1, int(threads)), "deterministic": bool(o.deterministic),
                        "version": VERSION},
        "status": rep.status,
        "pval": rep.pval, "dval": rep.dval, "dval_no_theta": rep.dval_no_theta,
        "rel_pfeas": rep.rel_pfeas, "rel_gap": rep.rel_gap, "rel_dfeas": rep.rel_dfeas,
        "rank": rep.rank, "theta": rep.theta, "tau": rep.tau,
        "outer_iters": rep.outer_iters, "fw_steps": rep.fw_steps, "aipp_iters": rep.aipp_iters,
        "fista_iters": rep.fista_iters, "eig_products": rep.eig_products,
        "wall_seconds": rep.wall_seconds,
    }
    if rep.message:
        j["message"] = rep.message
    return j


def status_exit_code(status: str) -> int:
    """tools/main.cpp:369-377."""
    if status == "optimal":
        return EXIT_OPTIMAL
    if status in ("iteration_limit", "time_limit"):
        return EXIT_LIMIT
    return EXIT_NUMERICAL


def _trace_printer(verbose: int):
    """tools/main.cpp:356-367 (stderr progress lines)."""
    if not verbose:
        return None

    def sink(e):
        if e.kind == "outer":
            print(f"[outer] t={e.outer_iter:<3d} beta={e.beta:.3e} eps_t={e.eps_inner:.3e} gap={e.gap:.3e} "
                  f"theta={e.theta:.6f} rank={e.rank} pfeas={e.rel_pfeas:.3e} gap_rel={e.rel_gap:.3e} "
                  f"dfeas={e.rel_dfeas:.3e}", file=sys.stderr)
        elif verbose > 1 and e.kind in ("inner_stationary", "inner_rank_step"):
            tag = "stat" if e.kind == "inner_stationary" else "fw "
            print(f"[inner] t={e.outer_iter:<3d} {tag} gap={e.gap:.3e} theta={e.theta:.6f} rank={e.rank} "
                  f"al={e.al_value:.9e} alpha={e.fw_alpha:.3f}", file=sys.stderr)
    return sink


def parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2505_13719_b200", description="B200 HALLaR low-rank SDP solver")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve", help="solve one instance")
    # family flags (tools/main.cpp:259-272)
    s.add_argument("--problem", choices=["matcomp", "theta", "phaseret"])
    s.add_argument("--spec", default="")
    s.add_argument("--graph", default="")
    s.add_argument("--format", default="edge-list")
    s.add_argument("--hypercube", type=int)
    s.add_argument("--cycle", type=int)
    s.add_argument("--petersen", action="store_true")
    s.add_argument("--n1", type=int)
    s.add_argument("--n2", type=int)
    s.add_argument("--r", type=int)
    s.add_argument("--n", type=int)
    s.add_argument("--L", type=int)
    # common flags (tools/main.cpp:230-245)
    s.add_argument("--tol", type=float, default=1e-5)
    s.add_argument("--seed", type=int, default=0)
    s.add_argument("--threads", type=int, default=0)
    s.add_argument("--time-limit", dest="time_limit", type=float, default=3600.0)
    s.add_argument("--deterministic", action="store_true")
    s.add_argument("--beta0", type=float, default=0.0)
    s.add_argument("--beta-growth", dest="beta_growth", type=float, default=2.0)
    s.add_argument("--eps0", type=float, default=0.0)
    s.add_argument("--eps-decay", dest="eps_decay", type=float, default=0.5)
    s.add_argument("--eps-floor", dest="eps_floor", type=float, default=0.0)
    s.add_argument("--max-outer", dest="max_outer", type=int, default=500)
    s.add_argument("--lambda0", type=float, default=10.0)
    s.add_argument("-v", "--verbose", action="count", default=0)
    s.add_argument("--json-out", dest="json_out", default="")
    return ap


def cmd_solve(o: argparse.Namespace) -> int:
    from . import api as H
    inst, desc = build_from_spec(spec_from_flags(o))
    sink = _trace_printer(o.verbose)
    rep = H.solve(inst, make_config(o), sink=sink)
    j = report_to_json(desc, rep, o, threads=inst.info().get("team_ctas", 1))
    text = json.dumps(j, indent=2)
    if o.json_out:
        try:
            with open(o.json_out, "w") as fh:
                fh.write(text + "\n")
        except OSError:
            print(f"error: cannot write '{o.json_out}'", file=sys.stderr)
            return EXIT_NOINPUT
    print(text)
    return status_exit_code(rep.status)


def main(argv=None) -> int:
    """Exit codes as the reference main (tools/main.cpp:593-610)."""
    try:
        o = parser().parse_args(argv)
    except SystemExit as e:
        return EXIT_USAGE if e.code else EXIT_OPTIMAL
    try:
        from .api import InputError, NumericalError
    except Exception as e:  # the native library is missing: not a usable install
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE
    try:
        return cmd_solve(o)
    except InputError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except NumericalError as e:
        print(f"numerical error: {e}", file=sys.stderr)
        return EXIT_NUMERICAL
    except OSError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_NOINPUT
    except Exception as e:  # tools/main.cpp:605-607
        print(f"error: {e}", file=sys.stderr)
        return EXIT_NUMERICAL
