"""CLI / JSON report parity with the reference's `lrsdp solve` (tools/main.cpp,
docs/report-schema.json).  The pure parts (hashes, spec
handling, report layout, exit codes) run on CPU; the solve itself on the GPU."""
import argparse
import json
import os

import pytest

from paper_2505_13719_b200 import cli

SCHEMA_REQUIRED = ["version", "instance", "config_hash", "environment", "status", "pval", "dval",
                   "dval_no_theta", "rel_pfeas", "rel_gap", "rel_dfeas", "rank", "theta", "tau",
                   "outer_iters", "fw_steps", "aipp_iters", "fista_iters", "eig_products", "wall_seconds"]


def test_fnv1a_known_answers():
    # FNV-1a 64 published test vectors (tools/main.cpp:30-37 is the standard algorithm)
    assert cli.hex64(cli.fnv1a(b"")) == "cbf29ce484222325"
    assert cli.hex64(cli.fnv1a(b"a")) == "af63dc4c8601ec8c"
    assert cli.hex64(cli.fnv1a(b"foobar")) == "85944171f73967e8"


def test_vector_hash_is_over_raw_doubles():
    import numpy as np
    b = np.array([1.0, -2.5, 0.0])
    assert cli.vector_hash(b) == cli.hex64(cli.fnv1a(b.astype("<f8").tobytes()))
    assert len(cli.vector_hash(b)) == 16


def _opts(**kw):
    o = cli.parser().parse_args(["solve"])
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def test_config_hash_string_matches_ostream_format():
    o = _opts()
    s = ("tol=1e-05;seed=0;time_limit=3600;deterministic=0;beta0=0;beta_growth=2;eps0=0"
         ";eps_decay=0.5;eps_floor=0;max_outer=500;lambda0=10")
    assert cli.config_hash(o) == cli.hex64(cli.fnv1a(s.encode()))
    assert cli.config_hash(_opts(tol=1e-6)) != cli.config_hash(o)


def test_spec_from_flags_and_errors(tmp_path):
    from paper_2505_13719_b200 import InputError
    o = _opts(problem="matcomp", n1=20, n2=30, r=2, seed=7)
    assert cli.spec_from_flags(o) == {"family": "matcomp", "seed": "7", "n1": "20", "n2": "30", "r": "2"}
    assert cli.spec_from_flags(_opts(problem="theta", hypercube=5)) == {"family": "theta", "hypercube": "5"}
    with pytest.raises(InputError):
        cli.spec_from_flags(_opts(problem="matcomp", n1=2))
    with pytest.raises(InputError):
        cli.spec_from_flags(_opts(problem="theta"))
    with pytest.raises(InputError):
        cli.spec_from_flags(_opts())
    p = tmp_path / "x.spec"
    p.write_text("# comment\nfamily = theta\ncycle=5\n")
    assert cli.spec_from_flags(_opts(spec=str(p))) == {"family": "theta", "cycle": "5"}
    with pytest.raises(OSError):
        cli.read_spec_file(str(tmp_path / "missing.spec"))


def test_report_layout_and_exit_codes():
    rep = argparse.Namespace(status="optimal", pval=1.0, dval=1.0, dval_no_theta=1.0, rel_pfeas=0.0,
                             rel_gap=0.0, rel_dfeas=0.0, rank=2, theta=0.0, tau=1.0, outer_iters=3,
                             fw_steps=1, aipp_iters=2, fista_iters=9, eig_products=4, wall_seconds=0.1,
                             message="")
    desc = {"family": "theta", "n": 5, "m": 6, "tau": 1.0, "b_hash": "0" * 16}
    j = cli.report_to_json(desc, rep, _opts(), threads=148)
    assert all(k in j for k in SCHEMA_REQUIRED) and "message" not in j
    assert j["environment"] == {"threads": 148, "deterministic": False, "version": "0.1.0"}
    json.dumps(j)
    assert [cli.status_exit_code(s) for s in ("optimal", "iteration_limit", "time_limit", "numerical_failure")] \
        == [0, 2, 2, 3]
    assert cli.main(["solve", "--bogus-flag"]) == 64


@pytest.mark.gpu
def test_cli_solve_petersen(tmp_path, capsys):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = tmp_path / "r.json"
    rc = cli.main(["solve", "--problem", "theta", "--petersen", "--json-out", str(out)])
    assert rc == 0
    j = json.loads(out.read_text())
    assert all(k in j for k in SCHEMA_REQUIRED)
    assert j["status"] == "optimal" and j["instance"]["family"] == "theta"
    assert j["instance"]["vertices"] == 10 and j["instance"]["edges"] == 15 and j["instance"]["m"] == 16
    assert abs(-j["pval"] - 4.0) <= 1e-3  # theta(Petersen) = 4 (acceptance.cpp:226-246)
    assert json.loads(capsys.readouterr().out)["config_hash"] == j["config_hash"]


@pytest.mark.gpu
def test_cli_solve_matcomp_and_graph_file(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = tmp_path / "mc.json"
    assert cli.main(["solve", "--problem", "matcomp", "--n1", "30", "--n2", "70", "--r", "2",
                     "--json-out", str(out)]) == 0
    j = json.loads(out.read_text())
    assert j["instance"]["n"] == 100 and j["rank"] == 2 and j["instance"]["nuclear_norm"] > 0
    g = tmp_path / "c5.txt"
    g.write_text("1 2\n2 3\n3 4\n4 5\n5 1\n")  # edge list, 1-based
    out2 = tmp_path / "c5.json"
    assert cli.main(["solve", "--problem", "theta", "--graph", str(g), "--json-out", str(out2)]) == 0
    assert abs(-json.loads(out2.read_text())["pval"] - 5 ** 0.5) <= 1e-4
    assert cli.main(["solve", "--problem", "theta", "--graph", str(tmp_path / "none.txt")]) == 66
