"""CPU tier for the row-partitioned path: partition / ghost-zone
/ halo-list invariants, and the communication-avoiding matrix-powers protocol
(one halo exchange, prefix-row levels, one Gram allreduce) emulated in numpy --
in one process and over a real world-size-2 gloo process group -- against the
single-process block (owned rows of Y bit for bit, G to rounding)."""

import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import sscg_oracle as O
from paper_1908_04081_b200 import problems
from paper_1908_04081_b200.partition import (CsrRows, Stencil7Rows, build_local, link_halos,
                                             partition_all, partition_rank, slab_bounds)


def _random_spd_csr(n, seed):
    rng = np.random.default_rng(seed)
    m = sp.random(n, n, density=4.0 / n, random_state=seed, format="csr")
    m = m + m.T + sp.identity(n) * 10
    m = m.tocsr()
    m.sort_indices()
    return CsrRows(n, m.indptr, m.indices.astype(np.int32), m.data)


@pytest.mark.parametrize("world,depth", [(2, 3), (3, 5), (4, 8)])
def test_partition_invariants(world, depth):
    rows_list = [CsrRows.of(problems.make_problem("c1", scale=24).a), _random_spd_csr(300, 7)]
    for rows in rows_list:
        parts = partition_all(rows, world, depth)
        assert [p.row_lo for p in parts] == list(slab_bounds(rows.n, world)[:-1])
        assert parts[-1].row_hi == rows.n
        for p in parts:
            # local CSR reproduces the global rows (columns mapped back)
            ip, cols, vals = rows.rows(p.global_rows[: p.n_rows])
            np.testing.assert_array_equal(p.row_ptr, ip)
            np.testing.assert_array_equal(p.global_rows[p.col_idx], cols)
            np.testing.assert_array_equal(p.values, vals)
            # levels are graph-distance shells around the slab
            assert p.lvl_rows[0] == p.row_hi - p.row_lo
            assert np.all(np.diff(p.lvl_rows) >= 0) and p.n_local == p.lvl_rows[-1]
            owned = set(range(p.row_lo, p.row_hi))
            d1 = set(cols[: ip[p.n_own]].tolist()) - owned
            assert d1 == set(p.global_rows[p.lvl_rows[0]:p.lvl_rows[1]].tolist())
            # halo lists: mine from q == q's list for me, same global rows and order
            for k, q in enumerate(p.peers):
                mine = p.global_rows[p.recv_idx[p.recv_off[k]:p.recv_off[k + 1]]]
                other = parts[q]
                kq = other.peers.index(p.rank)
                theirs = other.send_idx[other.send_off[kq]:other.send_off[kq + 1]] + other.row_lo
                np.testing.assert_array_equal(mine, theirs)
            # every ghost is received exactly once
            assert sorted(p.global_rows[p.recv_idx].tolist()) == sorted(p.global_rows[p.n_own:].tolist())


def test_stencil_rows_match_global_csr():
    a = problems.stencil7(5, 4, 6)
    gen = Stencil7Rows(5, 4, 6)
    ref = CsrRows.of(a)
    idx = np.random.default_rng(0).permutation(a.n)[:50]
    for x, y in zip(gen.rows(idx), ref.rows(idx)):
        np.testing.assert_array_equal(x, y)


def emulate_rank_block(part, ghosts_of, p_glob, r_glob, prm, s):
    """One rank's CA-MPK levels on its local prefix rows, from owned values +
    the ghost values its halo delivered (ghosts_of: local ghost idx -> values)."""
    nl = part.n_local
    mat = sp.csr_matrix((part.values, part.col_idx, part.row_ptr), shape=(part.n_rows, nl))
    P = np.zeros((nl, s + 1))
    R = np.zeros((nl, s))
    P[: part.n_own, 0] = p_glob[part.row_lo:part.row_hi]
    R[: part.n_own, 0] = r_glob[part.row_lo:part.row_hi]
    gi, gp, gr = ghosts_of
    P[gi, 0], R[gi, 0] = gp, gr
    D = part.depth
    for l in range(s):
        for Y, deg, lim_d in ((P, s, D - 1 - l), (R, s - 1, D - 2 - l)):
            if l >= deg:
                continue
            lim = part.lvl_rows[max(lim_d, 0)]
            y = Y[:, l]
            w = mat[:lim] @ y - prm.thetas[l] * y[:lim]
            if l >= 1 and prm.mus[l - 1] != 0.0:
                w = w - prm.mus[l - 1] * Y[:lim, l - 1]
            Y[:lim, l + 1] = w / prm.gammas[l]
    own = np.hstack([P[: part.n_own], R[: part.n_own]])
    return own, own.T @ own


def _problem_and_block(s=6):
    prob = problems.make_problem("c1", scale=20)
    rng = np.random.default_rng(3)
    p, r = rng.standard_normal(prob.a.n), rng.standard_normal(prob.a.n)
    prm = O.params_chebyshev(0.1, 7.9, s)
    mat = O.csr_of(prob.a.n, prob.a.row_ptr, prob.a.col_idx, prob.a.values)
    y = np.hstack([O.krylov_columns(mat, p, s, prm), O.krylov_columns(mat, r, s - 1, prm)])
    return prob, p, r, prm, y, O.gram_matrix(y)


@pytest.mark.parametrize("world", [2, 3, 5])
def test_partitioned_mpk_and_gram_match_single_process(world):
    s = 6
    prob, p, r, prm, y_ref, g_ref = _problem_and_block(s)
    parts = partition_all(CsrRows.of(prob.a), world, depth=s)
    g_sum = np.zeros_like(g_ref)
    for part in parts:
        gi = part.recv_idx
        gg = part.global_rows[gi]
        own, g = emulate_rank_block(part, (gi, p[gg], r[gg]), p, r, prm, s)
        np.testing.assert_array_equal(own, y_ref[part.row_lo:part.row_hi])  # bit for bit
        g_sum += g
    scale = np.sqrt(np.outer(np.diag(g_ref), np.diag(g_ref)))
    assert np.max(np.abs(g_sum - g_ref) / scale) < 1e-13


def _free_port():
    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        return sck.getsockname()[1]


def _gloo_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = 6
    prob, p, r, prm, y_ref, g_ref = _problem_and_block(s)

    def exchange(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    part = partition_rank(CsrRows.of(prob.a), rank, world, s, exchange)
    # the per-outer-loop halo exchange over gloo: p and r of the owned rows each
    # peer needs, received straight into our ghost rows
    ops, recv_bufs = [], []
    own_p, own_r = p[part.row_lo:part.row_hi], r[part.row_lo:part.row_hi]
    for k, q in enumerate(part.peers):
        si = part.send_idx[part.send_off[k]:part.send_off[k + 1]]
        sbuf = torch.from_numpy(np.concatenate([own_p[si], own_r[si]]))
        n_in = int(part.recv_off[k + 1] - part.recv_off[k])
        rbuf = torch.empty(2 * n_in, dtype=torch.float64)
        ops.append(dist.P2POp(dist.isend, sbuf, q))
        ops.append(dist.P2POp(dist.irecv, rbuf, q))
        recv_bufs.append((k, rbuf, n_in))
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    gi_all, gp_all, gr_all = [], [], []
    for k, rbuf, n_in in recv_bufs:
        gi_all.append(part.recv_idx[part.recv_off[k]:part.recv_off[k + 1]])
        v = rbuf.numpy()
        gp_all.append(v[:n_in])
        gr_all.append(v[n_in:])
    ghosts = (np.concatenate(gi_all), np.concatenate(gp_all), np.concatenate(gr_all))
    own, g = emulate_rank_block(part, ghosts, p, r, prm, s)
    gt = torch.from_numpy(g.copy())
    dist.all_reduce(gt)  # the one synchronisation of the outer loop
    np.save(os.path.join(out_dir, f"own{rank}.npy"), own)
    np.save(os.path.join(out_dir, f"g{rank}.npy"), gt.numpy())
    np.save(os.path.join(out_dir, f"lo{rank}.npy"), np.array([part.row_lo, part.row_hi]))
    dist.destroy_process_group()


def test_gloo_world2_partitioned_protocol(tmp_path):
    import torch.multiprocessing as mp

    world = 2
    port = _free_port()
    mp.spawn(_gloo_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    s = 6
    prob, p, r, prm, y_ref, g_ref = _problem_and_block(s)
    g0 = np.load(tmp_path / "g0.npy")
    for rank in range(world):
        lo, hi = np.load(tmp_path / f"lo{rank}.npy")
        np.testing.assert_array_equal(np.load(tmp_path / f"own{rank}.npy"), y_ref[lo:hi])
        np.testing.assert_array_equal(np.load(tmp_path / f"g{rank}.npy"), g0)  # identical on ranks
    scale = np.sqrt(np.outer(np.diag(g_ref), np.diag(g_ref)))
    assert np.max(np.abs(g0 - g_ref) / scale) < 1e-13


@pytest.mark.parametrize("jacobi", [False, True])
def test_varcoef27_rows_match_the_generator(jacobi):
    """The on-demand c4 / c4j rows (what a partitioned rank builds its slab
    from) are the global generator's rows bit for bit, in any order."""
    from paper_1908_04081_b200.partition import Varcoef27Rows
    n = 9
    prob = problems.make_problem("c4j" if jacobi else "c4", scale=n)
    g = Varcoef27Rows(n, jacobi=jacobi)
    ip, cols, vals = g.rows(np.arange(n ** 3))
    np.testing.assert_array_equal(ip, np.asarray(prob.a.row_ptr))
    np.testing.assert_array_equal(cols, np.asarray(prob.a.col_idx))
    np.testing.assert_array_equal(vals, np.asarray(prob.a.values))
    np.testing.assert_array_equal(g.rhs(), prob.b)
    sel = np.array([700, 5, 364, 0, 728])
    for x, y in zip(g.rows(sel), CsrRows.of(prob.a).rows(sel)):
        np.testing.assert_array_equal(x, y)
    parts = partition_all(g, 3, 4)
    for p in parts:  # slabs of whole planes: what the plane-table value stream needs
        assert p.n_local % (n * n) == 0


def test_rank_decision_digests():
    """The cross-rank check of a partitioned solve: identical digests pass, any
    divergence raises (a desynchronised rank would corrupt the halo)."""
    from types import SimpleNamespace

    from paper_1908_04081_b200.dist import RankMismatch, check_ranks_agree, logs_digest
    def fake(alpha):
        s = SimpleNamespace(status=1, total_iters=2, total_outer=1, n_records=1)
        it = np.zeros((4, 10))
        it[:2, 0] = alpha
        return SimpleNamespace(s=s, rec_i=np.zeros((3, 8), np.int32), iters=it)
    a, b = logs_digest(fake(0.5)), logs_digest(fake(0.5))
    check_ranks_agree([a, b])
    with pytest.raises(RankMismatch):
        check_ranks_agree([a, logs_digest(fake(np.nextafter(0.5, 1.0)))])
