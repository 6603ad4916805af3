"""paper_2407_00046_b200 -- B200-native BAL inexact Newton-PCG (arXiv 2407.00046).

Thin Python binding over the C ABI of ``libbal.so`` (include/bal.h).  The functions below have
the same names as the C entry points and only marshal arguments: scene dicts (from ``scenes``)
become ``bal_mesh`` / ``bal_params`` structs, torch CUDA tensors become device pointers.  PyTorch
is used for device memory and streams only.  There is no CPU fallback: importing this package
raises when the CUDA library is missing.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import (BAL_ADDITIVE_PRECOND, BAL_PCG_CRIT_I, BAL_PCG_CRIT_II, BAL_PCG_CRIT_III, BAL_CCD_LITERAL, BAL_FP32_MATRIX, BAL_FRICTION_LAGGED, BAL_FRICTION_NO_FREEZE, BAL_PCG_LITERAL_STALL, BAL_NO_AUGLAG, BAL_NO_WARMSTART, BAL_SIGMA_CAP,
                   BAL_SIGMA_MIN, STATUS, bal_bsr_host, bal_contact_state, bal_dist, bal_material, bal_mesh,
                   bal_params, bal_pcg_opts, bal_pcg_stats, bal_step_stats, bal_system_view)

__all__ = ["BalError", "BalCtx", "bal_init", "bal_step", "bal_step_host", "bal_assemble", "bal_spmv", "bal_pcg",
           "bal_load_bsr", "bal_bench_spmv", "bal_destroy", "bal_nccl_unique_id", "bal_dist_info", "bal_spmv_rows",
           "bal_halo_plan", "bal_halo_pack", "bal_halo_unpack", "bal_get_system", "BAL_NO_WARMSTART", "BAL_NO_AUGLAG",
           "BAL_FRICTION_LAGGED", "BAL_SIGMA_CAP", "BAL_SIGMA_MIN", "BAL_FRICTION_NO_FREEZE", "BAL_CCD_LITERAL",
           "BAL_PCG_LITERAL_STALL", "BAL_FP32_MATRIX", "BAL_ADDITIVE_PRECOND", "BAL_PCG_CRIT_I", "BAL_PCG_CRIT_II", "BAL_PCG_CRIT_III", "lib_path"]

lib_path = _lib.LIB_PATH


class BalError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"bal status {status} ({STATUS.get(status, '?')}): {msg}")
        self.status = status


def _check(ctx, st):
    if st != 0:
        msg = _lib.lib.bal_last_error(ctx.handle if ctx is not None else None)
        raise BalError(st, msg.decode() if msg else "")


def _dptr(t, numel=None, ctx=None):
    """Device pointer of a contiguous float64 CUDA tensor (or None); checks dtype, size and device
    so that no kernel reads or writes out of bounds through a mismatched tensor."""
    if t is None:
        return None
    import torch
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("expected a contiguous CUDA tensor")
    if t.dtype != torch.float64:
        raise ValueError(f"expected a float64 tensor, got {t.dtype}")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"expected {numel} elements, got {t.numel()}")
    if ctx is not None and t.device.index != ctx.device:
        raise ValueError(f"tensor on cuda:{t.device.index}, context on cuda:{ctx.device}")
    return C.c_void_p(t.data_ptr())


def _vecs(ctx, *ts):
    """Device pointers of [3N] float64 tensors of ctx's device (None passes through)."""
    return [_dptr(t, 3 * ctx.n_nodes, ctx) for t in ts]


class BalCtx:
    def __init__(self, handle, scene, device=0):
        self.handle = handle
        self.device = device
        self.n_nodes = int(len(scene["rest_x"]))
        self.n_tets = int(len(scene["tets"]))
        self._keep = []

    def __del__(self):
        try:
            bal_destroy(self)
        except Exception:
            pass

    @property
    def kernel_launches(self):
        return int(_lib.lib.bal_kernel_launches(self.handle)) if self.handle else 0


def make_params(p, flags=0):
    prm = bal_params()
    prm.h = p["h"]
    prm.gravity[:] = list(p["gravity"])
    prm.dhat = p["dhat"]
    prm.eps_v = p["eps_v"]
    prm.chi = p["chi"]
    prm.newton_rel_tol = p["newton_rel_tol"]
    prm.pcg_rel_tol = p["pcg_rel_tol"]
    prm.pcg_stall_window = p["pcg_stall_window"]
    prm.pcg_resume_iters = p["pcg_resume_iters"]
    prm.alpha_min = p["alpha_min"]
    prm.ws_rel_tol = p["ws_rel_tol"]
    prm.ws_max_iters = p["ws_max_iters"]
    prm.max_newton = p["max_newton"]
    prm.max_pcg = p["max_pcg"]
    prm.max_constraints = p["max_constraints"]
    prm.flags = flags
    return prm


def bal_nccl_unique_id():
    """128-byte NCCL unique id (rank 0 creates it, the caller broadcasts it)."""
    buf = (C.c_uint8 * 128)()
    st = _lib.lib.bal_nccl_unique_id(buf)
    if st != 0:
        raise BalError(st, "bal_nccl_unique_id")
    return bytes(buf)


def bal_init(scene, device=0, flags=0, params=None, rank=0, world=1, nccl_id=None, host_transport=None):
    """bal_init(mesh, materials, params, dist) from a ``scenes`` dict.  world > 1 (or nccl_id /
    host_transport given) selects the partitioned solve: nccl_id = bal_nccl_unique_id() of rank 0;
    host_transport = (allreduce(np.ndarray) in place, exchange(send, send_counts, recv_counts) ->
    recv) Python callables (tests)."""
    x = np.ascontiguousarray(scene["rest_x"], np.float64).ravel()
    tets = np.ascontiguousarray(scene["tets"], np.int32).ravel()
    fixed = np.ascontiguousarray(scene["node_fixed"], np.uint8)
    mat = np.ascontiguousarray(scene["tet_material"], np.int32)
    ob = np.ascontiguousarray(scene["obstacle_tris"], np.int32).ravel()
    mats = np.ascontiguousarray(scene["materials"], np.float64).reshape(-1, 3)
    m = bal_mesh()
    m.n_nodes = len(fixed)
    m.n_tets = len(tets) // 4
    m.rest_x = _lib.ptr(x, C.c_double)
    m.tets = _lib.ptr(tets, C.c_int32)
    m.node_fixed = _lib.ptr(fixed, C.c_uint8)
    m.tet_material = _lib.ptr(mat, C.c_int32)
    m.n_obstacle_tris = len(ob) // 3
    m.obstacle_tris = _lib.ptr(ob, C.c_int32)
    models = np.asarray(scene.get("material_model", np.zeros(len(mats))), np.int32).reshape(-1)
    ma = (bal_material * len(mats))(*[bal_material(*row, int(mdl)) for row, mdl in zip(mats, models)])
    prm = make_params(params or scene["params"], flags)
    d = bal_dist()
    d.rank, d.world, d.device = int(rank), int(world), int(device)
    keep = []
    if nccl_id is not None:
        idb = C.create_string_buffer(bytes(nccl_id), 128)
        keep.append(idb)
        d.nccl_unique_id = C.cast(idb, C.c_void_p)
    if host_transport is not None:
        ar, ex = host_transport

        def _ar(buf, n, _u):
            try:
                a = np.ctypeslib.as_array(buf, shape=(n,))
                a[:] = ar(a.copy())
                return 0
            except Exception:  # noqa: BLE001  (reported to the library as a transport failure)
                return 1

        def _ex(send, scnt, recv, rcnt, _u):
            try:
                sc = np.ctypeslib.as_array(scnt, shape=(world,)).copy()
                rc = np.ctypeslib.as_array(rcnt, shape=(world,)).copy()
                s_ = np.ctypeslib.as_array(send, shape=(max(int(sc.sum()), 1),))[:int(sc.sum())].copy()
                r_ = ex(s_, sc, rc)
                if int(rc.sum()):
                    np.ctypeslib.as_array(recv, shape=(int(rc.sum()),))[:] = r_
                return 0
            except Exception:  # noqa: BLE001
                return 1

        f1, f2 = _lib.HOST_ALLREDUCE(_ar), _lib.HOST_EXCHANGE(_ex)
        keep += [f1, f2]
        d.host_allreduce, d.host_exchange = f1, f2
    h = C.c_void_p()
    st = _lib.lib.bal_init(C.byref(m), ma, len(mats), C.byref(prm), C.byref(d), C.byref(h))
    if st != 0:
        raise BalError(st, _lib.lib.bal_last_error(None).decode())
    ctx = BalCtx(h, scene, device)
    ctx._keep = keep
    try:  # order library work after torch's work on this device (device tensors come from torch)
        import torch
        if torch.cuda.is_available():
            bal_set_stream(ctx, torch.cuda.current_stream(device))
    except ImportError:
        pass
    return ctx


def bal_destroy(ctx):
    if ctx.handle:
        _lib.lib.bal_destroy(ctx.handle)
        ctx.handle = None


def bal_set_stream(ctx, stream):
    _check(ctx, _lib.lib.bal_set_stream(ctx.handle, C.c_void_p(stream.cuda_stream if stream is not None else 0)))


def bal_step(ctx, x_t, v_t, x_next, v_next=None):
    """One time step on device tensors; returns the stats dict."""
    s = bal_step_stats()
    _check(ctx, _lib.lib.bal_step(ctx.handle, *_vecs(ctx, x_t, v_t, x_next, v_next), C.byref(s)))
    return {f: getattr(s, f) for f, _ in bal_step_stats._fields_}


def bal_frame_begin(ctx, x_t, v_t):
    """Start a time step (setup of Alg. 1) on device tensors; advance it with bal_frame_iterate."""
    _check(ctx, _lib.lib.bal_frame_begin(ctx.handle, *_vecs(ctx, x_t, v_t)))


def bal_frame_iterate(ctx, max_iters):
    """Run up to max_iters inexact-Newton iterations of the frame in progress; True once converged."""
    done = C.c_int32(0)
    _check(ctx, _lib.lib.bal_frame_iterate(ctx.handle, int(max_iters), C.byref(done)))
    return bool(done.value)


def bal_frame_finish(ctx, x_next=None, v_next=None, allow_unconverged=False):
    """Write x_{t+1}, v_{t+1} of the frame in progress; returns the stats dict.  Raises BalError on
    BAL_E_NOT_CONVERGED unless allow_unconverged (x_next is the last accepted iterate either way)."""
    s = bal_step_stats()
    st = _lib.lib.bal_frame_finish(ctx.handle, *_vecs(ctx, x_next, v_next), C.byref(s))
    out = {f: getattr(s, f) for f, _ in bal_step_stats._fields_}
    out["converged"] = st == 0
    if st == -4 and allow_unconverged:
        return out
    _check(ctx, st)
    return out


def bal_frame_stats(ctx):
    """Stats of the frame in progress so far (same fields as bal_step's), without finishing it."""
    s = bal_step_stats()
    _check(ctx, _lib.lib.bal_frame_peek(ctx.handle, C.byref(s)))
    return {f: getattr(s, f) for f, _ in bal_step_stats._fields_}


def bal_step_host(ctx, x_t, v_t, allow_unconverged=False):
    """End-to-end step on host numpy arrays (copies inside the call).  allow_unconverged: return
    the last accepted iterate and the stats on BAL_E_NOT_CONVERGED (stats["converged"] False)."""
    x_t = np.ascontiguousarray(x_t, np.float64).ravel()
    v_t = np.ascontiguousarray(v_t, np.float64).ravel()
    xn = np.empty_like(x_t)
    vn = np.empty_like(v_t)
    s = bal_step_stats()
    st = _lib.lib.bal_step_host(ctx.handle, _lib.ptr(x_t, C.c_double), _lib.ptr(v_t, C.c_double),
                                _lib.ptr(xn, C.c_double), _lib.ptr(vn, C.c_double), C.byref(s))
    out = {f: getattr(s, f) for f, _ in bal_step_stats._fields_}
    out["converged"] = st == 0
    if not (st == -4 and allow_unconverged):
        _check(ctx, st)
    return xn, vn, out


TRACE_FIELDS = ("l", "nA", "nAp", "rebuilt", "dmin", "sigma", "ws_iters", "pcg_iters", "pcg_stop", "alpha_ccd",
                "alpha", "halvings", "resumes", "safeguard", "rel_e")


def bal_get_trace(ctx, max_records=100000):
    """Decision trace of the last bal_step: list of dicts (one per Newton iteration)."""
    out = np.zeros(max_records * len(TRACE_FIELDS))
    n = _lib.lib.bal_get_trace(ctx.handle, _lib.ptr(out, C.c_double), max_records)
    if n < 0:
        raise BalError(n, "bal_get_trace")
    rows = out[:n * len(TRACE_FIELDS)].reshape(n, len(TRACE_FIELDS))
    return [dict(zip(TRACE_FIELDS, r.tolist())) for r in rows]


def bal_pcg_objective_history(ctx, max_n=200000):
    """phi_0 - phi_k (CG objective decrease), k = 0..iters, of the last global PCG solve."""
    out = np.zeros(max_n)
    n = _lib.lib.bal_pcg_objective_history(ctx.handle, _lib.ptr(out, C.c_double), max_n)
    if n < 0:
        raise BalError(n, "bal_pcg_objective_history")
    return out[:n].copy()


def bal_pcg_history(ctx, max_n=200000):
    """||r_k|| of the last global PCG solve, k = 0..iters."""
    out = np.zeros(max_n)
    n = _lib.lib.bal_pcg_history(ctx.handle, _lib.ptr(out, C.c_double), max_n)
    if n < 0:
        raise BalError(n, "bal_pcg_history")
    return out[:n].copy()


def bal_spmv_counters(ctx):
    """(total SpMV kernel ms, launches, algorithmic bytes, full-BSR minimum bytes) since ctx creation."""
    out = np.zeros(4)
    _check(ctx, _lib.lib.bal_spmv_counters(ctx.handle, _lib.ptr(out, C.c_double)))
    return dict(ms=out[0], launches=int(out[1]), bytes_alg=out[2], bytes_moved=out[3])


def _keys_arr(k):
    k = np.ascontiguousarray(np.asarray(k, np.int32).reshape(-1, 5))
    return k, (_lib.ptr(k, C.c_int32) if len(k) else None)


def bal_assemble(ctx, x, active_keys=(), aprime_keys=(), aprime_mu=(), aprime_s=(), sigma=1.0, friction=None,
                 x_t=None, y=None):
    """Assemble at device positions x; returns a dict of torch tensors (copies of the device views)."""
    import torch
    cs = bal_contact_state()
    keep = []
    ak, cs.active_keys = _keys_arr(active_keys)
    cs.n_active = len(ak)
    pk, cs.aprime_keys = _keys_arr(aprime_keys)
    cs.n_aprime = len(pk)
    mu = np.ascontiguousarray(aprime_mu, np.float64)
    s = np.ascontiguousarray(aprime_s, np.float64)
    cs.aprime_mu = _lib.ptr(mu, C.c_double) if len(mu) else None
    cs.aprime_s = _lib.ptr(s, C.c_double) if len(s) else None
    cs.sigma = float(sigma)
    if friction is not None:
        fk, cs.friction_keys = _keys_arr(friction["keys"])
        fg = np.ascontiguousarray(friction["gamma"], np.float64).ravel()
        fn = np.ascontiguousarray(friction["n"], np.float64).ravel()
        fl = np.ascontiguousarray(friction["lam"], np.float64).ravel()
        keep += [fk, fg, fn, fl]
        cs.n_friction = len(fk)
        cs.friction_gamma = _lib.ptr(fg, C.c_double)
        cs.friction_n = _lib.ptr(fn, C.c_double)
        cs.friction_lambda = _lib.ptr(fl, C.c_double)
    if x_t is not None:
        xt = np.ascontiguousarray(x_t, np.float64).ravel()
        keep.append(xt)
        cs.x_t = _lib.ptr(xt, C.c_double)
    if y is not None:
        yy = np.ascontiguousarray(y, np.float64).ravel()
        keep.append(yy)
        cs.y = _lib.ptr(yy, C.c_double)
    v = bal_system_view()
    _check(ctx, _lib.lib.bal_assemble(ctx.handle, *_vecs(ctx, x), C.byref(cs), C.byref(v)))
    return _views(v, x.device)


def bal_detect(ctx, x, max_n=1 << 20):
    """GPU active set at device positions x: (keys int32 [n][5], d float64 [n])."""
    keys = np.zeros((max_n, 5), np.int32)
    d = np.zeros(max_n, np.float64)
    n = C.c_int32(0)
    _check(ctx, _lib.lib.bal_detect(ctx.handle, *_vecs(ctx, x), _lib.ptr(keys, C.c_int32), _lib.ptr(d, C.c_double),
                                    max_n, C.byref(n)))
    return keys[:n.value].copy(), d[:n.value].copy()


def bal_get_system(ctx, device=None):
    """Views of the system the last Newton iteration or bal_assemble assembled (copies, dict of
    torch tensors as bal_assemble returns)."""
    import torch
    v = bal_system_view()
    _check(ctx, _lib.lib.bal_get_system(ctx.handle, C.byref(v)))
    return _views(v, device or torch.device(f"cuda:{ctx.device}"))


def _views(v, device):
    import torch
    N = v.n_nodes

    def view(p, n, dtype):
        if not p or n == 0:
            return torch.zeros(0, dtype=dtype, device=device)
        return _wrap(p, n, dtype, device).clone()

    return dict(
        n_nodes=N,
        static_row_ptr=view(v.static_row_ptr, N + 1, torch.int32),
        static_col=view(v.static_col, v.nnzb_static, torch.int32),
        static_val=view(v.static_val, 9 * v.nnzb_static, torch.float64),
        contact_row_ptr=view(v.contact_row_ptr, N + 1 if v.nnzb_contact else 0, torch.int32),
        contact_col=view(v.contact_col, v.nnzb_contact, torch.int32),
        contact_val=view(v.contact_val, 9 * v.nnzb_contact, torch.float64),
        diag_inv=view(v.diag_inv, 6 * N, torch.float64),
        grad=view(v.grad, 3 * N, torch.float64),
        e_node=view(v.e_node, N, torch.float64),
        group=view(v.group, N, torch.int32),
        elastic_blocks=view(v.elastic_blocks, 90 * v.n_elastic, torch.float64),
        elastic_lbar=view(v.elastic_lbar, v.n_elastic, torch.float64),
        contact_blocks=view(v.contact_blocks, 90 * v.n_contact_stencils, torch.float64),
        contact_lbar=view(v.contact_lbar, v.n_contact_stencils, torch.float64),
        contact_stencil_nodes=view(v.contact_stencil_nodes, 4 * v.n_contact_stencils, torch.int32),
        n_friction_stencils=int(v.n_friction_stencils),
        contact_grad=view(v.contact_grad, 12 * v.n_contact_stencils, torch.float64),
    )


class _CAI:
    def __init__(self, p, n, typestr):
        self.__cuda_array_interface__ = dict(shape=(n,), typestr=typestr, data=(int(p), False), version=3)


def _wrap(p, n, dtype, device):
    import torch
    typestr = {torch.float64: "<f8", torch.int32: "<i4"}[dtype]
    with torch.cuda.device(device):
        return torch.as_tensor(_CAI(p, n, typestr), device=device)


def bal_spmv(ctx, v, y):
    _check(ctx, _lib.lib.bal_spmv(ctx.handle, *_vecs(ctx, v, y)))


def bal_pcg(ctx, rhs, x0, x_out, warm_start=None, rel_tol=None, stall_window=None, max_iters=None,
            ws_rel_tol=None, ws_max_iters=None):
    o = bal_pcg_opts()
    o.warm_start = 1 if warm_start is None else int(warm_start)
    o.rel_tol = 1e-4 if rel_tol is None else rel_tol
    o.stall_window = 100 if stall_window is None else stall_window
    o.max_iters = 20000 if max_iters is None else max_iters
    o.ws_rel_tol = 1e-2 if ws_rel_tol is None else ws_rel_tol
    o.ws_max_iters = 100 if ws_max_iters is None else ws_max_iters
    s = bal_pcg_stats()
    _check(ctx, _lib.lib.bal_pcg(ctx.handle, *_vecs(ctx, rhs, x0, x_out), C.byref(o), C.byref(s)))
    return {f: getattr(s, f) for f, _ in bal_pcg_stats._fields_}


def bal_load_bsr(ctx, row_ptr, col, val, group=None):
    rp = np.ascontiguousarray(row_ptr, np.int32)
    cc = np.ascontiguousarray(col, np.int32)
    vv = np.ascontiguousarray(val, np.float64).ravel()
    b = bal_bsr_host()
    b.n_nodes = len(rp) - 1
    b.nnzb = len(cc)
    b.row_ptr = _lib.ptr(rp, C.c_int32)
    b.col = _lib.ptr(cc, C.c_int32)
    b.val = _lib.ptr(vv, C.c_double)
    g = None
    if group is not None:
        g = np.ascontiguousarray(group, np.int32)
        b.group = _lib.ptr(g, C.c_int32)
    _check(ctx, _lib.lib.bal_load_bsr(ctx.handle, C.byref(b)))


def bal_bench_spmv(ctx, iters):
    us = C.c_double()
    _check(ctx, _lib.lib.bal_bench_spmv(ctx.handle, iters, C.byref(us)))
    return us.value


def bal_dist_info(ctx):
    """(r0, r1, halo_send, halo_recv): owned block rows and the last solve's halo sizes."""
    r0, r1 = C.c_int32(), C.c_int32()
    hs, hr = C.c_int64(), C.c_int64()
    _check(ctx, _lib.lib.bal_dist_info(ctx.handle, C.byref(r0), C.byref(r1), C.byref(hs), C.byref(hr)))
    return r0.value, r1.value, hs.value, hr.value


def bal_spmv_rows(ctx, r0, r1, v, y):
    n3 = 3 * ctx.n_nodes
    _check(ctx, _lib.lib.bal_spmv_rows(ctx.handle, int(r0), int(r1), _dptr(v, n3, ctx), _dptr(y, n3, ctx)))


def bal_halo_plan(row_ptr, col, bounds, rank):
    """Halo plan of `rank` (host): (send_ptr, send_idx, recv_ptr, recv_idx)."""
    rp = np.ascontiguousarray(row_ptr, np.int32)
    cl = np.ascontiguousarray(col, np.int32)
    b = np.ascontiguousarray(bounds, np.int32)
    world = len(b) - 1
    sp_ = np.zeros(world + 1, np.int32)
    rpp = np.zeros(world + 1, np.int32)
    n = len(rp) - 1
    m = _lib.lib.bal_halo_plan(n, _lib.ptr(rp, C.c_int32), _lib.ptr(cl, C.c_int32), world, _lib.ptr(b, C.c_int32),
                               int(rank), _lib.ptr(sp_, C.c_int32), None, _lib.ptr(rpp, C.c_int32), None, 0)
    if m < 0:
        raise BalError(m, "bal_halo_plan")
    si = np.zeros(max(m, 1), np.int32)
    ri = np.zeros(max(m, 1), np.int32)
    _lib.lib.bal_halo_plan(n, _lib.ptr(rp, C.c_int32), _lib.ptr(cl, C.c_int32), world, _lib.ptr(b, C.c_int32),
                           int(rank), _lib.ptr(sp_, C.c_int32), _lib.ptr(si, C.c_int32), _lib.ptr(rpp, C.c_int32),
                           _lib.ptr(ri, C.c_int32), m)
    return sp_, si[:sp_[-1]], rpp, ri[:rpp[-1]]


def bal_halo_pack(idx, v):
    idx = np.ascontiguousarray(idx, np.int32)
    v = np.ascontiguousarray(v, np.float64).ravel()
    buf = np.zeros(3 * max(len(idx), 1))
    _check(None, _lib.lib.bal_halo_pack(len(idx), _lib.ptr(idx, C.c_int32), _lib.ptr(v, C.c_double),
                                        _lib.ptr(buf, C.c_double)))
    return buf[:3 * len(idx)]


def bal_halo_unpack(idx, buf, v):
    """In place: v[3 idx[k] + c] = buf[3k + c]."""
    idx = np.ascontiguousarray(idx, np.int32)
    buf = np.ascontiguousarray(buf, np.float64)
    _check(None, _lib.lib.bal_halo_unpack(len(idx), _lib.ptr(idx, C.c_int32), _lib.ptr(buf, C.c_double),
                                          _lib.ptr(v, C.c_double)))
    return v


def bal_partition_rows(row_cost, world):
    """Contiguous block-row ranges balanced by row_cost; returns bounds (world+1,)."""
    rc = np.ascontiguousarray(row_cost, np.int64)
    b = np.zeros(world + 1, np.int32)
    _check(None, _lib.lib.bal_partition_rows(len(rc), _lib.ptr(rc, C.c_int64), int(world), _lib.ptr(b, C.c_int32)))
    return b


def bal_ghost_columns(row_ptr, col, r0, r1):
    """Sorted unique columns of rows [r0, r1) outside [r0, r1) (the per-SpMV ghost values)."""
    rp = np.ascontiguousarray(row_ptr, np.int32)
    cl = np.ascontiguousarray(col, np.int32)
    n = len(rp) - 1
    m = _lib.lib.bal_ghost_columns(n, _lib.ptr(rp, C.c_int32), _lib.ptr(cl, C.c_int32), int(r0), int(r1), None, 0)
    if m < 0:
        raise BalError(m, "bal_ghost_columns")
    out = np.zeros(max(m, 1), np.int32)
    _lib.lib.bal_ghost_columns(n, _lib.ptr(rp, C.c_int32), _lib.ptr(cl, C.c_int32), int(r0), int(r1),
                               _lib.ptr(out, C.c_int32), m)
    return out[:m]
