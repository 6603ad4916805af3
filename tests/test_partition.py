"""Host logic of the vertex-domain partition through the C ABI, on
CPU: balanced contiguous block-row ranges, ghost-column lists, and a world-size-2 gloo run of the
distributed SpMV / dot-product data flow (each rank owns its rows, receives exactly its ghost
values, all-reduces its partial dot) reproducing the single-process product and dot."""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import scenes


def _pattern(sc):
    """Node-adjacency CSR (diagonal included) of a scene's tets: the static SpMV pattern."""
    T = np.asarray(sc["tets"], np.int64)
    N = len(sc["rest_x"])
    r = np.repeat(T, 4, axis=1).ravel()
    c = np.tile(T, (1, 4)).ravel()
    A = sp.coo_matrix((np.ones(len(r)), (r, c)), shape=(N, N)).tocsr()
    A.sum_duplicates()
    A.sort_indices()
    A = A + sp.identity(N, format="csr")  # isolated (obstacle) nodes keep their diagonal
    A.sum_duplicates()
    A.sort_indices()
    return A.indptr.astype(np.int32), A.indices.astype(np.int32), N


def _scene():
    return scenes.make_puffer_net(seed=4, nx=4, nz=4, n_balls=1, ball_R=5.0, n_spikes=16, spike_len=4.0)


def test_partition_is_balanced_and_contiguous():
    import paper_2407_00046_b200 as bal
    rp, col, N = _pattern(_scene())
    cost = np.diff(rp).astype(np.int64)
    for world in (1, 2, 3, 4, 8):
        b = bal.bal_partition_rows(cost, world)
        assert b[0] == 0 and b[-1] == N and np.all(np.diff(b) >= 0)
        loads = np.array([cost[b[k]:b[k + 1]].sum() for k in range(world)])
        # each split point is the first row reaching k/W of the total: imbalance below one row's cost
        assert loads.max() - cost.sum() / world <= cost.max() + 1e-9
    with pytest.raises(bal.BalError):
        bal.bal_partition_rows(np.array([1, -1], np.int64), 2)


def test_ghost_columns_match_reference():
    import paper_2407_00046_b200 as bal
    rp, col, N = _pattern(_scene())
    b = bal.bal_partition_rows(np.diff(rp).astype(np.int64), 3)
    for k in range(3):
        r0, r1 = int(b[k]), int(b[k + 1])
        cols = col[rp[r0]:rp[r1]]
        ref = np.unique(cols[(cols < r0) | (cols >= r1)])
        np.testing.assert_array_equal(bal.bal_ghost_columns(rp, col, r0, r1), ref)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2407_00046_b200 as bal
    rp, col, N = _pattern(_scene())
    rng = np.random.default_rng(0)  # same matrix and vector on every rank (replicated assembly)
    vals = rng.normal(size=len(col))
    A = sp.csr_matrix((vals, col, rp), shape=(N, N))
    x = rng.normal(size=N)
    b = bal.bal_partition_rows(np.diff(rp).astype(np.int64), world)
    r0, r1 = int(b[rank]), int(b[rank + 1])
    ghosts = bal.bal_ghost_columns(rp, col, r0, r1)
    # owned slice -> exchange (all-gather of the slices; each rank keeps only its ghost values)
    own = torch.as_tensor(x[r0:r1])
    sizes = [int(b[k + 1] - b[k]) for k in range(world)]
    m = max(sizes)
    pad = torch.zeros(m, dtype=torch.float64)
    pad[:len(own)] = own
    gathered = [torch.zeros(m, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, pad)
    full = np.concatenate([gathered[k].numpy()[:sizes[k]] for k in range(world)])
    xl = np.full(N, np.nan)  # only owned + ghost entries are known locally
    xl[r0:r1] = x[r0:r1]
    xl[ghosts] = full[ghosts]
    y_own = A[r0:r1] @ xl  # NaN if the ghost list missed a needed column
    # partial dot of the owned rows, all-reduced
    d = torch.tensor([float(x[r0:r1] @ y_own)], dtype=torch.float64)
    dist.all_reduce(d)
    out[rank] = (r0, r1, y_own, float(d.item()), len(ghosts))
    dist.barrier()
    dist.destroy_process_group()


def test_distributed_spmv_and_dot_data_flow_gloo():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    rp, col, N = _pattern(_scene())
    rng = np.random.default_rng(0)
    A = sp.csr_matrix((rng.normal(size=len(col)), col, rp), shape=(N, N))
    x = rng.normal(size=N)
    y = A @ x
    y_dist = np.concatenate([out[k][2] for k in range(world)])
    assert out[0][0] == 0 and out[world - 1][1] == N and out[0][1] == out[1][0]
    assert np.all(np.isfinite(y_dist))
    np.testing.assert_allclose(y_dist, y, rtol=1e-13, atol=1e-13)
    for k in range(world):
        assert out[k][3] == pytest.approx(float(x @ y), rel=1e-12)
        assert out[k][4] > 0  # ranks do exchange values


def _aligned_bounds(rp, world, align=64):
    import paper_2407_00046_b200 as bal
    N = len(rp) - 1
    b = bal.bal_partition_rows(np.diff(rp).astype(np.int64), world)
    for k in range(1, world):
        b[k] = max(b[k - 1], min((int(b[k]) + align // 2) // align * align, N))
    return b


def test_halo_plan_matches_reference():
    """bal_halo_plan: the send list of rank k to m is exactly the owned rows of k adjacent to rows
    of m, the receive list of k from m exactly m's rows adjacent to k's rows, and the send list of
    k to m equals the receive list of m from k (the exchange is consistent)."""
    import paper_2407_00046_b200 as bal
    rp, col, N = _pattern(_scene())
    world = 4
    b = _aligned_bounds(rp, world)
    owner = np.searchsorted(b, np.arange(N), side="right") - 1
    plans = [bal.bal_halo_plan(rp, col, b, k) for k in range(world)]
    for k in range(world):
        sp_, si, rpp, ri = plans[k]
        for m in range(world):
            s_km = si[sp_[m]:sp_[m + 1]]
            r_km = ri[rpp[m]:rpp[m + 1]]
            if m == k:
                assert len(s_km) == 0 and len(r_km) == 0
                continue
            rows_k = np.arange(b[k], b[k + 1])
            need = [i for i in rows_k if np.any(owner[col[rp[i]:rp[i + 1]]] == m)]
            np.testing.assert_array_equal(s_km, need)
            ghost = np.unique([j for i in rows_k for j in col[rp[i]:rp[i + 1]] if owner[j] == m])
            np.testing.assert_array_equal(r_km, ghost.astype(np.int32) if len(ghost) else np.zeros(0, np.int32))
            sp2, si2, _rp2, _ri2 = plans[m]
            np.testing.assert_array_equal(r_km, si2[sp2[k]:sp2[k + 1]])


def test_halo_pack_unpack_roundtrip():
    import paper_2407_00046_b200 as bal
    rng = np.random.default_rng(3)
    v = rng.normal(size=30)
    idx = np.array([7, 2, 9], np.int32)
    buf = bal.bal_halo_pack(idx, v)
    np.testing.assert_array_equal(buf, v.reshape(-1, 3)[idx].ravel())
    w = np.zeros(30)
    bal.bal_halo_unpack(idx, buf, w)
    np.testing.assert_array_equal(w.reshape(-1, 3)[idx], v.reshape(-1, 3)[idx])
    assert np.count_nonzero(w) == 9


def _halo_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2407_00046_b200 as bal
    rp, col, N = _pattern(_scene())
    rng = np.random.default_rng(0)
    vals = rng.normal(size=len(col))
    A = sp.csr_matrix((vals, col, rp), shape=(N, N))
    x = rng.normal(size=(N, 3))
    b = _aligned_bounds(rp, world)
    r0, r1 = int(b[rank]), int(b[rank + 1])
    sp_, si, rpp, ri = bal.bal_halo_plan(rp, col, b, rank)
    xl = np.full((N, 3), np.nan)
    xl[r0:r1] = x[r0:r1]
    # the library's halo: pack the owned boundary rows per peer, point-to-point exchange, unpack
    reqs, bufs = [], {}
    for m in range(world):
        if sp_[m + 1] > sp_[m]:
            sb = torch.as_tensor(bal.bal_halo_pack(si[sp_[m]:sp_[m + 1]], xl))
            reqs.append(dist.isend(sb, m))
            bufs[("s", m)] = sb
        if rpp[m + 1] > rpp[m]:
            rb = torch.zeros(3 * int(rpp[m + 1] - rpp[m]), dtype=torch.float64)
            reqs.append(dist.irecv(rb, m))
            bufs[("r", m)] = rb
    for q in reqs:
        q.wait()
    flat = xl.ravel()
    for m in range(world):
        if ("r", m) in bufs:
            bal.bal_halo_unpack(ri[rpp[m]:rpp[m + 1]], bufs[("r", m)].numpy(), flat)
    xl = flat.reshape(N, 3)
    y_own = A[r0:r1] @ xl  # NaN if the plan missed a ghost
    d = torch.tensor([float(np.sum(x[r0:r1] * y_own))], dtype=torch.float64)
    dist.all_reduce(d)
    out[rank] = (r0, r1, y_own, float(d.item()), int(sp_[-1]), int(rpp[-1]))
    dist.barrier()
    dist.destroy_process_group()


def test_halo_exchange_spmv_gloo():
    """World-2 gloo run of the library's own halo plan + pack/unpack (bal_halo_plan, bal_halo_pack,
    bal_halo_unpack): each rank computes its owned rows of A x from owned + received ghost values
    only, and the all-reduced dot equals the single-process one."""
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_halo_worker, args=(world, port, out), nprocs=world, join=True)
    rp, col, N = _pattern(_scene())
    rng = np.random.default_rng(0)
    A = sp.csr_matrix((rng.normal(size=len(col)), col, rp), shape=(N, N))
    x = rng.normal(size=(N, 3))
    y = A @ x
    y_dist = np.concatenate([out[k][2] for k in range(world)])
    assert np.all(np.isfinite(y_dist))
    np.testing.assert_allclose(y_dist, y, rtol=1e-13, atol=1e-13)
    for k in range(world):
        assert out[k][3] == pytest.approx(float(np.sum(x * y)), rel=1e-12)
        assert out[k][4] > 0 and out[k][5] > 0
