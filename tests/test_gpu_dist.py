"""Partitioned multi-GPU solve on the one GPU a gpurun box has:
 * the NCCL path with a world-1 communicator (bal_nccl_unique_id -> bal_init with the id): the
   distributed PCG / warm start kernels, the NCCL all-reduces and the all-gather run, and a C1 step
   matches the oracle;
 * two processes sharing cuda:0 with the library's host transport (gloo underneath): the halo
   plan, pack/exchange/unpack, owned-row SpMV, distributed PCG, warm start and all-gather of a real
   two-rank partition, checked against the oracle and across ranks;
 * bal_spmv_rows: owned-row SpMV over any tile-aligned partition concatenates to the full SpMV
   bitwise (each row is summed in the same fixed order whoever owns it)."""
import os
import socket

import numpy as np
import pytest

import scenes

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import paper_2407_00046_b200 as bal  # noqa: E402

DEV = torch.device("cuda:0")
SYM_R = 64  # kSymR: partition bounds are tile aligned


def _oracle_steps(sc, n):
    from oracle.bal import Oracle
    o = Oracle(sc)
    x, v = sc["x0"], sc["v0"]
    out = []
    for _ in range(n):
        x, v, _s = o.step(x, v)
        out.append(x.copy())
    return out


def _gpu_steps(ctx, sc, n):
    x = torch.as_tensor(sc["x0"].ravel(), device=DEV)
    v = torch.as_tensor(sc["v0"].ravel(), device=DEV)
    xs, st = [], []
    for _ in range(n):
        xn, vn = torch.empty_like(x), torch.empty_like(v)
        st.append(bal.bal_step(ctx, x, v, xn, vn))
        x, v = xn, vn
        xs.append(x.cpu().numpy().reshape(-1, 3).copy())
    return xs, st


def test_world1_nccl_path_matches_oracle():
    sc = scenes.make_cubes(1)
    ctx = bal.bal_init(sc, world=1, nccl_id=bal.bal_nccl_unique_id())
    r0, r1, _hs, _hr = bal.bal_dist_info(ctx)
    assert (r0, r1) == (0, len(sc["rest_x"]))
    xg, _ = _gpu_steps(ctx, sc, 3)
    xo = _oracle_steps(sc, 3)
    for a, b in zip(xg, xo):
        assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-6


def test_spmv_rows_partition_is_bitwise_identical():
    sc = scenes.make_cubes(1)
    ctx = bal.bal_init(sc)
    N = len(sc["rest_x"])
    rng = np.random.default_rng(5)
    xt = torch.as_tensor(sc["x0"].ravel(), device=DEV)
    bal.bal_assemble(ctx, xt, y=sc["x0"] + 0.01 * rng.normal(size=sc["x0"].shape))
    v = torch.as_tensor(rng.normal(size=3 * N), device=DEV)
    y = torch.empty_like(v)
    bal.bal_spmv_rows(ctx, 0, N, v, y)  # the partitioned path's row-range kernel, one part
    yt = torch.empty_like(v)
    bal.bal_spmv(ctx, v, yt)  # single-GPU tile-symmetric kernel: same product, other summation order
    assert torch.allclose(yt, y, rtol=1e-12, atol=1e-12 * float(y.abs().max()))
    for parts in (2, 3, 7):
        cuts = sorted({min(N, SYM_R * int(round(k * N / parts / SYM_R))) for k in range(1, parts)} | {0, N})
        yp = torch.full_like(v, float("nan"))
        for a, b in zip(cuts[:-1], cuts[1:]):
            bal.bal_spmv_rows(ctx, a, b, v, yp)
        assert torch.equal(yp, y), parts


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _host_transport(rank, world):
    def allreduce(a):
        t = torch.as_tensor(a)
        dist.all_reduce(t)
        return t.numpy()

    def exchange(send, scnt, rcnt):
        so = np.concatenate([[0], np.cumsum(scnt)])
        ro = np.concatenate([[0], np.cumsum(rcnt)])
        recv = torch.zeros(int(ro[-1]), dtype=torch.float64)
        reqs = []
        for m in range(world):
            if m == rank:
                continue
            if scnt[m]:
                reqs.append(dist.isend(torch.as_tensor(send[so[m]:so[m + 1]].copy()), m))
            if rcnt[m]:
                reqs.append(dist.irecv(recv[ro[m]:ro[m + 1]], m))
        for q in reqs:
            q.wait()
        return recv.numpy()

    return allreduce, exchange


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = scenes.make_cubes(1)
    ctx = bal.bal_init(sc, rank=rank, world=world, host_transport=_host_transport(rank, world))
    info = bal.bal_dist_info(ctx)
    xs, st = _gpu_steps(ctx, sc, 2)
    info = info[:2] + bal.bal_dist_info(ctx)[2:]
    out[rank] = (info, xs, [(s["newton_iters"], s["pcg_iters"]) for s in st])
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_host_transport_step():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    sc = scenes.make_cubes(1)
    N = len(sc["rest_x"])
    (a0, a1, hs0, hr0), xs0, it0 = out[0]
    (b0, b1, hs1, hr1), xs1, it1 = out[1]
    assert a0 == 0 and a1 == b0 and b1 == N and a1 % SYM_R == 0 and 0 < a1 < N
    assert hs0 > 0 and hr0 > 0 and hs0 == hr1 and hr0 == hs1  # consistent boundary-only halo
    assert hr0 < N - a1  # not an all-gather
    assert it0 == it1  # identical decisions on both ranks (all-reduced scalars)
    for p, q in zip(xs0, xs1):
        assert np.array_equal(p, q)  # replicated state stays bitwise identical
    xo = _oracle_steps(sc, 2)
    for a, b in zip(xs0, xo):
        assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-6
