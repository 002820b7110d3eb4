"""CPU coverage of the row-sharded (N > 1) path with torch.distributed/gloo,
world_size 2 (the device implementation is team.cuh's
publish_rows / two-level team_reduce_smem and capi.cu's
cuhallar_solve_sharded).

Each rank owns a contiguous block of rows and the upper (edge-order)
constraints of those rows — the device ownership rule — and evaluates the
fused value + gradient row pass of AlFunction::value_and_gradient
(sdp_instance.cpp:115-127) for its rows only, with the reference's per-row
fold order (instances.cpp:45-52: lower entries, then upper, increasing k).
Rows are then published to every rank (all_gather: the peer-row push) and
per-rank partial sums are joined in rank order (the fixed-order cross-rank
reduction).  The assembled gradient must equal the oracle's bit for bit, the
value within 1e-12, and every rank must hold identical results."""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _csr(ei, ej, n):
    """Upper / lower CSR of the pair constraints (capi.cu upload_pairs)."""
    order_lo = np.lexsort((np.arange(len(ei)), ej))  # lower entries of row a sorted by k
    up_ptr = np.zeros(n + 1, dtype=np.int64)
    lo_ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(up_ptr, ei + 1, 1)
    np.add.at(lo_ptr, ej + 1, 1)
    return np.cumsum(up_ptr), np.cumsum(lo_ptr), order_lo


def _row_blocks(up_ptr, lo_ptr, world):
    """Contiguous row blocks balanced by entries (+8 per row), as row_split does."""
    n = len(up_ptr) - 1
    work = up_ptr + lo_ptr + 8 * np.arange(n + 1)
    cuts = [0] + [int(np.searchsorted(work, work[-1] * r / world)) for r in range(1, world)] + [n]
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def _rank_pass(U, p, b, beta, ei, ej, up_ptr, lo_ptr, order_lo, rl, rh):
    """Own rows [rl, rh): h = 0.5 U + fold_k 0.5 q_k U_b (MC: C = I/2), and the
    upper-entry partials p.r, r^2, q(r + b), <h, U>."""
    s = U.shape[1]
    h = np.zeros((rh - rl, s))
    pr = rr = qrb = 0.0
    for a in range(rl, rh):
        acc = 0.5 * U[a].copy()
        ents = [(int(order_lo[e]), int(ei[order_lo[e]])) for e in range(lo_ptr[a], lo_ptr[a + 1])]
        ents += [(k, int(ej[k])) for k in range(up_ptr[a], up_ptr[a + 1])]
        for k, bcol in ents:
            d = 0.0
            for c in range(s):
                t = U[a, c] * U[bcol, c]
                d = t if c == 0 else d + t
            r = d - b[k]
            q = p[k] + beta * r
            if k >= up_ptr[a] and k < up_ptr[a + 1]:  # upper: each constraint once
                pr = pr + p[k] * r
                rr = rr + r * r
                qrb = qrb + q * (r + b[k])
            w = 0.5 * q
            if w == 0.0:
                continue
            for c in range(s):
                acc[c] = acc[c] + w * U[bcol, c]
        h[a - rl] = acc
    hu = float(np.sum(h * U[rl:rh]))
    return h, np.array([hu, pr, rr, qrb])


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        inst = O.OracleInstance.matcomp(30, 70, 2, seed=5)
        ei, ej = inst.pairs()
        ej = ej + 30  # McInstance::omega_j is in [0, n2); rows of V start at n1
        n, m = inst.n, inst.m
        b = inst.b
        up_ptr, lo_ptr, order_lo = _csr(ei, ej, n)
        rng = np.random.default_rng(11)
        U = rng.standard_normal((n, 3)) / np.sqrt(n)
        p = rng.standard_normal(m)
        beta = 2.5
        blocks = _row_blocks(up_ptr, lo_ptr, world)
        rl, rh = blocks[rank]
        h, part = _rank_pass(U, p, b, beta, ei, ej, up_ptr, lo_ptr, order_lo, rl, rh)
        # publish own rows to every rank (the peer push), then rank-ordered reduction
        rows = [None] * world
        dist.all_gather_object(rows, (rl, rh, h))
        parts = [None] * world
        dist.all_gather_object(parts, part)
        H = np.zeros((n, 3))
        for (a0, a1, hh) in rows:
            H[a0:a1] = hh
        tot = parts[0].copy()
        for r in range(1, world):
            tot = tot + parts[r]
        hu, pr, rr, qrb = tot
        value = (hu - qrb) + pr + 0.5 * beta * rr  # sdp_instance.cpp:122-125
        q_full = p + beta * (inst.apply_map(U) - b)
        ref_h = inst.C_plus_adjoint(q_full, U)
        ref_v, ref_g = inst.al_value_and_gradient(U, p, beta)
        q.put((rank, bool(np.array_equal(H, ref_h)), bool(np.array_equal(2.0 * H, ref_g)),
               float(value), float(ref_v), H.tobytes(), float(value)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_row_sharded_value_gradient_world2(orc):
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    res.sort()
    for rank, h_ok, g_ok, v, ref_v, _, _ in res:
        assert h_ok, f"rank {rank}: (C + A*q)U differs from the oracle"
        assert g_ok, f"rank {rank}: gradient differs from the oracle"
        assert abs(v - ref_v) <= 1e-12 * max(1.0, abs(ref_v))
    # every rank holds bit-identical results (replicated control flow)
    assert res[0][5] == res[1][5] and res[0][6] == res[1][6]


def test_row_blocks_cover_rows_and_constraints_once():
    rng = np.random.default_rng(3)
    n = 200
    pairs = {(int(min(u, v)), int(max(u, v))) for u, v in rng.integers(0, n, (900, 2)) if u != v}
    ei, ej = map(np.array, zip(*sorted(pairs)))
    up_ptr, lo_ptr, _ = _csr(ei, ej, n)
    for world in (2, 3, 4, 8):
        blocks = _row_blocks(up_ptr, lo_ptr, world)
        assert blocks[0][0] == 0 and blocks[-1][1] == n
        assert all(blocks[r][1] == blocks[r + 1][0] for r in range(world - 1))
        owned = np.concatenate([np.arange(up_ptr[a0], up_ptr[a1]) for a0, a1 in blocks])
        assert np.array_equal(owned, np.arange(len(ei)))  # each constraint owned exactly once
