"""Graph-file ingestion (load_graph, graph.cpp:56-109):
edge-list, Matrix Market (pattern) and GSET files produce the same device
instance as the generator, with the reference's normalisation (1-based ids,
self-loops dropped, duplicates merged, (u, v) sorted) and its error behaviour
(InputError for malformed lines, OSError / status 66 for a missing file)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2505_13719_b200 as H
    return H


def _petersen_edges():
    e = []
    for i in range(5):
        e += [(i, (i + 1) % 5), (i, i + 5), (i + 5, (i + 2) % 5 + 5)]
    return e


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_formats_match_generator(H, tmp_path):
    ref = H.build_theta_instance(H.make_petersen())
    ri, rj = ref.pairs()
    e = _petersen_edges()
    # edge list: comments, blank lines, a self-loop and a duplicate (reversed) edge
    el = "# petersen\n\n" + "".join(f"{u + 1} {v + 1}\n" for u, v in e) + "3 3\n2 1\n"
    mm = "%%MatrixMarket matrix coordinate pattern symmetric\n% comment\n10 10 15\n" + \
         "".join(f"{v + 1} {u + 1}\n" for u, v in e)
    gs = "10 15\n" + "".join(f"{u + 1} {v + 1} 1\n" for u, v in e)
    for fmt, text in (("edge-list", el), ("matrix-market", mm), ("gset", gs)):
        inst = H.build_theta_instance(H.load_graph(_write(tmp_path, fmt + ".txt", text), fmt))
        i, j = inst.pairs()
        assert (inst.n, inst.m) == (ref.n, ref.m)
        assert np.array_equal(i, ri) and np.array_equal(j, rj)
        r = H.solve(inst, H.SolverConfig(eps=1e-5, seed=0))
        assert abs(-r.pval - 4.0) <= 1e-3  # theta(Petersen) = 4 (acceptance.cpp:226-246)


def test_declared_vertex_count_keeps_isolated_vertices(H, tmp_path):
    # Matrix Market size line 12 > max id 10: two isolated vertices (n_hint, graph.cpp:93)
    mm = "%%MatrixMarket matrix coordinate pattern symmetric\n12 12 15\n" + \
         "".join(f"{u + 1} {v + 1}\n" for u, v in _petersen_edges())
    inst = H.build_theta_instance(H.load_graph(_write(tmp_path, "iso.mtx", mm), "matrix-market"))
    assert inst.n == 12 and inst.m == 16


@pytest.mark.parametrize("fmt,text", [
    ("edge-list", "1 2\n0 3\n"),                    # vertex indices are 1-based
    ("edge-list", "1 2\nfoo\n"),                    # expected two vertex indices
    ("gset", "x y\n1 2 1\n"),                       # bad GSET header
    ("matrix-market", "%%MatrixMarket matrix coordinate real symmetric\n3 3 1\n1 2 1.0\n"),  # not pattern
    ("matrix-market", "3 4 1\n1 2\n"),              # adjacency matrix must be square
    ("gset", "3 1\n1 5 1\n"),                       # vertex index exceeds declared count
])
def test_malformed_files_raise_input_error(H, tmp_path, fmt, text):
    with pytest.raises(H.InputError):
        H.build_theta_instance(H.load_graph(_write(tmp_path, "bad.txt", text), fmt))


def test_missing_file_is_io_error(H, tmp_path):
    with pytest.raises(OSError):
        H.build_theta_instance(H.load_graph(str(tmp_path / "nope.txt")))
