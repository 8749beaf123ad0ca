"""World-size-2 (gloo, CPU) model of the sharded dense path.

Each rank holds a contiguous slab of the last mode.  The model runs R-STHOSVD with rho
ending at the last mode exactly as the library's sharded path sequences it:
  modes n < d-1 : partial sketch over the local slab with Omega rows at GLOBAL unfolding
                  columns c_glob = c_loc + offset * prod_{k<d-1, k!=n} I_k  (col_offset_for),
                  allreduce(Y), redundant QR; local B-pass, allreduce(Gram); redundant eig;
                  local shrink (the core stays sharded along the last mode)
  mode d-1      : local rows of Y_d are complete -> allgather by row blocks; redundant QR;
                  partial B_d = Q_d(slab rows)^T G_(d) summed by allreduce; redundant eig;
                  replicated core.
The result must equal the unsharded oracle (Omega identical by construction, only the
reduction order differs: <= 1e-12 relative).  Oracle primitives (unfold, omega_rows, QR,
SVD) serve as the per-rank local steps; the collectives are torch.distributed over gloo."""
import os
import socket

import numpy as np
import pytest

import oracle as O
from workloads import hilbert


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shards(extent, world):
    ext = [extent // world + (1 if r < extent % world else 0) for r in range(world)]
    off = [sum(ext[:r]) for r in range(world)]
    return off, ext


def _allreduce(x):
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    dist.all_reduce(t)
    return t.numpy()


def _allgather(x):
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [o.numpy() for o in out]


def _sharded_rsthosvd(xloc, gdims, off, ext, ext_all, ranks, p, seed, order):
    """Model of run_sthosvd with a sharded last mode (dense.cu)."""
    d = len(gdims)
    assert order[-1] == d - 1
    g = np.asarray(xloc, dtype=np.float64)             # local slab, shape (.., ext)
    cur = list(gdims)
    factors = [None] * d
    for n in order:
        ell, r = O.rank_caps(cur, n, ranks[n], p)
        if n != d - 1:
            gn = O.unfold(g, n)                         # I_n x (local columns)
            lm = int(np.prod([cur[k] for k in range(d - 1) if k != n]))
            cols = np.arange(gn.shape[1], dtype=np.int64) + lm * off   # col_offset_for
            y = _allreduce(gn @ O.omega_rows(seed, n, cols, ell))
            q, _ = np.linalg.qr(y)
            b = q.T @ gn                                # local B (l x local columns)
            gram = _allreduce(b @ b.T)
            w, v = np.linalg.eigh(gram)
            ub = v[:, ::-1][:, :r]
            a = q @ ub
            sg = O.algorithms.canonical_signs(a)
            a, ub = a * sg, ub * sg
            factors[n] = a
            shape = list(g.shape)
            shape[n] = r
            g = O.fold(ub.T @ b, n, tuple(shape))
            cur[n] = r
        else:
            gn = O.unfold(g, n)                         # ext x prod(others): complete local rows
            cols = np.arange(gn.shape[1], dtype=np.int64)
            yloc = gn @ O.omega_rows(seed, n, cols, ell)
            # sketch_last_sharded: local rows placed at the shard offset in a zeroed global
            # buffer with a coverage column of ones, summed over the ranks (x + 0 = x: exact);
            # every row must be covered exactly once
            buf = np.zeros((gdims[n], ell + 1))
            buf[off:off + ext, :ell] = yloc
            buf[off:off + ext, ell] = 1.0
            buf = _allreduce(buf)
            assert np.all(buf[:, ell] == 1.0)
            y = buf[:, :ell]
            q, _ = np.linalg.qr(y)
            bd = _allreduce(q[off:off + ext].T @ gn)   # B_d sums over the sharded index
            w, v = np.linalg.eigh(bd @ bd.T)
            ub = v[:, ::-1][:, :r]
            a = q @ ub
            sg = O.algorithms.canonical_signs(a)
            a, ub = a * sg, ub * sg
            factors[n] = a
            shape = list(g.shape)
            shape[n] = r
            g = O.fold(ub.T @ bd, n, tuple(shape))
            cur[n] = r
    return g, factors


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = hilbert((11, 9, 13), "paper")
        off, ext = _shards(x.shape[2], world)
        core, factors = _sharded_rsthosvd(x[:, :, off[rank]:off[rank] + ext[rank]], x.shape, off[rank], ext[rank],
                                          ext, (3, 4, 5), 2, 7, (0, 1, 2))
        if rank == 0:
            o = O.r_sthosvd(x, (3, 4, 5), 2, 7, (0, 1, 2))
            delta = O.approx_distance(x, (core, factors), (o.core, o.factors))
            q.put(float(delta))
    finally:
        dist.destroy_process_group()


def test_sharded_rsthosvd_matches_unsharded_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    delta = q.get(timeout=5)
    assert delta <= 1e-12, delta


def _sharded_adaptive(xloc, gdims, off, eps, b, seed):
    """Model of run_adaptive with a sharded last mode (adaptive.cu, Alg 5 with reading R8):
    modes n < d: the block sketch W and ||B_i||^2 are allreduced, QR / projections redundant,
    B local, truncation Gram allreduced, local shrink; mode d (last): local rows of W placed at
    the shard offset and summed, B_i = Q_i(slab rows)^T G_(d) allreduced, replicated core."""
    d = len(gdims)
    tau2 = (eps / np.sqrt(d)) ** 2 * float(_allreduce(np.array([np.sum(np.asarray(xloc) ** 2)]))[0])
    g = np.asarray(xloc, dtype=np.float64)
    cur = list(gdims)
    factors = [None] * d
    for n in range(d):
        last = n == d - 1
        gn = O.unfold(g, n)
        gn2 = float(_allreduce(np.array([np.sum(gn * gn)]))[0])
        I = cur[n]
        cap = min(I, int(np.prod([cur[k] for k in range(d) if k != n])))
        q = np.zeros((I, 0))
        bs = []
        e, k = gn2, 0
        while e > tau2 and k < cap:
            bb = min(b, cap - k)
            if not last:
                lm = int(np.prod([cur[kk] for kk in range(d - 1) if kk != n]))
                cols = np.arange(gn.shape[1], dtype=np.int64) + lm * off
                w = _allreduce(gn @ O.omega_rows(seed, n, cols, bb, k0=k))
            else:
                cols = np.arange(gn.shape[1], dtype=np.int64)
                buf = np.zeros((I, bb))
                buf[off:off + gn.shape[0]] = gn @ O.omega_rows(seed, n, cols, bb, k0=k)
                w = _allreduce(buf)
            w = w - q @ (q.T @ w)
            w = w - q @ (q.T @ w)
            qi, _ = np.linalg.qr(w)
            if not last:
                bi = qi.T @ gn
                nb = float(_allreduce(np.array([np.sum(bi * bi)]))[0])
            else:
                bi = _allreduce(qi[off:off + gn.shape[0]].T @ gn)
                nb = float(np.sum(bi * bi))
            q = np.hstack([q, qi])
            bs.append(bi)
            e -= nb
            k += bb
        bm = np.vstack(bs)
        gram = bm @ bm.T if last else _allreduce(bm @ bm.T)
        wv, vv = np.linalg.eigh(gram)
        wv, vv = wv[::-1], vv[:, ::-1]
        r = int(np.nonzero(gn2 - np.cumsum(wv) <= tau2)[0][0]) + 1
        a = q @ vv[:, :r]
        sg = O.algorithms.canonical_signs(a)
        a, u = a * sg, vv[:, :r] * sg
        factors[n] = a
        shape = list(g.shape)
        shape[n] = r
        g = O.fold(u.T @ bm, n, tuple(shape))
        cur[n] = r
    return g, factors


def _ad_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = hilbert((16, 14, 12), "paper")
        off, ext = _shards(x.shape[2], world)
        core, factors = _sharded_adaptive(x[:, :, off[rank]:off[rank] + ext[rank]], x.shape, off[rank], 1e-5, 2, 3)
        if rank == 0:
            o = O.adaptive_r_sthosvd(x, 1e-5, 2, seed=3, order=(0, 1, 2))
            ranks = tuple(f.shape[1] for f in factors)
            delta = O.approx_distance(x, (core, factors), (o.core, o.factors))
            q.put((ranks == o.ranks, float(delta)))
    finally:
        dist.destroy_process_group()


def test_sharded_adaptive_matches_unsharded_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ad_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=180)
        assert pr.exitcode == 0
    same_ranks, delta = q.get(timeout=5)
    assert same_ranks and delta <= 1e-12, (same_ranks, delta)


def _sharded_sp_sthosvd(idx, vals, dims, ranks, p, seed, eta):
    """Model of run_sparse_sthosvd on an nnz partition (sparse.cu): per mode the partial
    sketch of the local nonzeros is summed over the ranks, QR and sRRQR run redundantly on
    every rank, each rank filters its own nonzeros, and the core nonzeros are gathered in rank
    order.  Local steps are oracle primitives."""
    import scipy.sparse as sp
    d = len(dims)
    order = O.auto_order(dims)
    cur = list(dims)
    idx = np.array(idx, dtype=np.int64, copy=True)
    vals = np.asarray(vals, dtype=np.float64).copy()
    sels, facs = [None] * d, [None] * d
    for j in order:
        ell = ranks[j] + p
        cols = O.unfold_columns(cur, j, idx)
        om = O.omega_rows(seed, j, cols, ell) if cols.size else np.zeros((0, ell))
        yl = sp.coo_matrix((vals, (idx[j], np.arange(cols.size))), shape=(cur[j], cols.size)).tocsr() @ om
        y = _allreduce(np.asarray(yl))                    # partial sketches summed over ranks
        q, _ = np.linalg.qr(y)
        sel, _ = O.srrqr_select(q, eta)                   # redundant, identical on every rank
        sels[j], facs[j] = np.asarray(sel), O.oblique_factor(q, sel)
        keep = np.isin(idx[j], sels[j])                   # local filter, no communication
        idx, vals = idx[:, keep], vals[keep]
        idx[j] = np.searchsorted(sels[j], idx[j])
        cur[j] = ell
    import torch
    import torch.distributed as dist
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, (idx, vals))           # rank-order gather of the core
    cidx = np.concatenate([pi for pi, _ in parts], axis=1)
    cval = np.concatenate([pv for _, pv in parts])
    return cidx, cval, sels, facs


def _sp_worker(rank, world, port, q):
    import torch.distributed as dist
    from workloads import sparse_zipf
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dims = (300, 250, 2000, 60)
        idx, vals = sparse_zipf(dims=dims, ndraws=40_000, seed=12)
        nnz = idx.shape[1]
        lo, hi = rank * nnz // world, (rank + 1) * nnz // world   # contiguous nnz partition
        cidx, cval, sels, facs = _sharded_sp_sthosvd(idx[:, lo:hi], vals[lo:hi], dims, (4, 4, 4, 4), 3, 5, 2.0)
        if rank == 0:
            o = O.sp_sthosvd(idx, vals, dims, (4, 4, 4, 4), 3, seed=5)
            same_sel = all(list(a) == list(b) for a, b in zip(sels, o.selections))
            ferr = max(np.linalg.norm(a - b) / np.linalg.norm(b) for a, b in zip(facs, o.factors))
            same_core = np.array_equal(cidx, o.core_idx) and np.array_equal(cval, np.asarray(o.core_vals, dtype=np.float64))
            q.put((same_sel, float(ferr), bool(same_core)))
    finally:
        dist.destroy_process_group()


def test_nnz_partitioned_sp_sthosvd_matches_unsharded_gloo_world2():
    """SP-STHOSVD on an nnz partition over 2 gloo ranks = the unsharded oracle: identical
    selections, identical core (entries in the same order), factors to 1e-12."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sp_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=180)
        assert pr.exitcode == 0
    same_sel, ferr, same_core = q.get(timeout=5)
    assert same_sel and same_core and ferr <= 1e-12, (same_sel, ferr, same_core)


@pytest.mark.parametrize("extent,world", [(800, 8), (13, 2), (7, 4), (1, 1)])
def test_shard_partition(extent, world):
    """Contiguous slabs cover the last mode exactly once (bench.py / library partition)."""
    off, ext = _shards(extent, world)
    assert sum(ext) == extent and off[0] == 0
    assert all(off[r] + ext[r] == off[r + 1] for r in range(world - 1))
    assert max(ext) - min(ext) <= 1


def test_global_column_offset_formula():
    """Omega rows of a slab = rows of the unsharded unfolding at the global columns:
    c_glob = c_loc + offset * prod_{k<d-1, k!=n} I_k for n < d-1 (col_offset_for)."""
    dims = (4, 3, 5, 6)
    x = np.arange(np.prod(dims), dtype=np.float64).reshape(dims, order="F")
    off, e = 2, 3
    for n in range(3):
        full = O.unfold(x, n)
        loc = O.unfold(x[:, :, :, off:off + e], n)
        lm = int(np.prod([dims[k] for k in range(3) if k != n]))
        cols = np.arange(loc.shape[1]) + lm * off
        np.testing.assert_array_equal(full[:, cols], loc)
