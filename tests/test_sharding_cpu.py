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
            # row blocks padded to the largest extent, gathered, unpadded (sketch_last_sharded)
            blocks = _allgather(np.vstack([yloc, np.zeros((max(ext_all) - yloc.shape[0], ell))]))
            y = np.vstack([blk[:e] for blk, e in zip(blocks, ext_all)])
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
