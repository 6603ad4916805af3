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
from ._lib import (BAL_FRICTION_LAGGED, BAL_NO_AUGLAG, BAL_NO_WARMSTART, STATUS, bal_bsr_host, bal_contact_state, bal_material,
                   bal_mesh, bal_params, bal_pcg_opts, bal_pcg_stats, bal_step_stats, bal_system_view)

__all__ = ["BalError", "BalCtx", "bal_init", "bal_step", "bal_step_host", "bal_assemble", "bal_spmv", "bal_pcg",
           "bal_load_bsr", "bal_bench_spmv", "bal_destroy", "BAL_NO_WARMSTART", "BAL_NO_AUGLAG", "BAL_FRICTION_LAGGED", "lib_path"]

lib_path = _lib.LIB_PATH


class BalError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"bal status {status} ({STATUS.get(status, '?')}): {msg}")
        self.status = status


def _check(ctx, st):
    if st != 0:
        msg = _lib.lib.bal_last_error(ctx.handle if ctx is not None else None)
        raise BalError(st, msg.decode() if msg else "")


def _dptr(t):
    """Device pointer of a contiguous float64/int32 CUDA tensor (or None)."""
    if t is None:
        return None
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("expected a contiguous CUDA tensor")
    return C.c_void_p(t.data_ptr())


class BalCtx:
    def __init__(self, handle, scene):
        self.handle = handle
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


def bal_init(scene, device=0, flags=0, params=None):
    """bal_init(mesh, materials, params, device) from a ``scenes`` dict."""
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
    ma = (bal_material * len(mats))(*[bal_material(*row) for row in mats])
    prm = make_params(params or scene["params"], flags)
    h = C.c_void_p()
    st = _lib.lib.bal_init(C.byref(m), ma, len(mats), C.byref(prm), device, C.byref(h))
    if st != 0:
        raise BalError(st, _lib.lib.bal_last_error(None).decode())
    ctx = BalCtx(h, scene)
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
    _check(ctx, _lib.lib.bal_step(ctx.handle, _dptr(x_t), _dptr(v_t), _dptr(x_next), _dptr(v_next), C.byref(s)))
    return {f: getattr(s, f) for f, _ in bal_step_stats._fields_}


def bal_frame_begin(ctx, x_t, v_t):
    """Start a time step (setup of Alg. 1) on device tensors; advance it with bal_frame_iterate."""
    _check(ctx, _lib.lib.bal_frame_begin(ctx.handle, _dptr(x_t), _dptr(v_t)))


def bal_frame_iterate(ctx, max_iters):
    """Run up to max_iters inexact-Newton iterations of the frame in progress; True once converged."""
    done = C.c_int32(0)
    _check(ctx, _lib.lib.bal_frame_iterate(ctx.handle, int(max_iters), C.byref(done)))
    return bool(done.value)


def bal_frame_finish(ctx, x_next=None, v_next=None, allow_unconverged=False):
    """Write x_{t+1}, v_{t+1} of the frame in progress; returns the stats dict.  Raises BalError on
    BAL_E_NOT_CONVERGED unless allow_unconverged (x_next is the last accepted iterate either way)."""
    s = bal_step_stats()
    st = _lib.lib.bal_frame_finish(ctx.handle, _dptr(x_next), _dptr(v_next), C.byref(s))
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


def bal_step_host(ctx, x_t, v_t):
    """End-to-end step on host numpy arrays (copies inside the call)."""
    x_t = np.ascontiguousarray(x_t, np.float64).ravel()
    v_t = np.ascontiguousarray(v_t, np.float64).ravel()
    xn = np.empty_like(x_t)
    vn = np.empty_like(v_t)
    s = bal_step_stats()
    _check(ctx, _lib.lib.bal_step_host(ctx.handle, _lib.ptr(x_t, C.c_double), _lib.ptr(v_t, C.c_double),
                                       _lib.ptr(xn, C.c_double), _lib.ptr(vn, C.c_double), C.byref(s)))
    return xn, vn, {f: getattr(s, f) for f, _ in bal_step_stats._fields_}


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
    _check(ctx, _lib.lib.bal_assemble(ctx.handle, _dptr(x), C.byref(cs), C.byref(v)))
    N = v.n_nodes

    def view(p, n, dtype):
        if not p or n == 0:
            return torch.zeros(0, dtype=dtype, device=x.device)
        return _wrap(p, n, dtype, x.device).clone()

    out = dict(
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
    )
    return out


class _CAI:
    def __init__(self, p, n, typestr):
        self.__cuda_array_interface__ = dict(shape=(n,), typestr=typestr, data=(int(p), False), version=3)


def _wrap(p, n, dtype, device):
    import torch
    typestr = {torch.float64: "<f8", torch.int32: "<i4"}[dtype]
    with torch.cuda.device(device):
        return torch.as_tensor(_CAI(p, n, typestr), device=device)


def bal_spmv(ctx, v, y):
    _check(ctx, _lib.lib.bal_spmv(ctx.handle, _dptr(v), _dptr(y)))


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
    _check(ctx, _lib.lib.bal_pcg(ctx.handle, _dptr(rhs), _dptr(x0), _dptr(x_out), C.byref(o), C.byref(s)))
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
