"""Helpers for the GPU parity tests: conversions between the library's device views and the
oracle's scipy / dense representations.  (Test infrastructure; no method arithmetic.)"""
import numpy as np
import scipy.sparse as sp


def bsr_to_csr(row_ptr, col, val, N):
    """Full BSR (3x3 blocks) -> scipy CSR (3N x 3N)."""
    row_ptr = np.asarray(row_ptr, np.int64)
    col = np.asarray(col, np.int64)
    val = np.asarray(val, np.float64).reshape(-1, 3, 3)
    rows = np.repeat(np.arange(N), np.diff(row_ptr))
    r = (3 * rows[:, None, None] + np.arange(3)[None, :, None]).repeat(3, axis=2)
    c = (3 * col[:, None, None] + np.arange(3)[None, None, :]).repeat(3, axis=1)
    return sp.csr_matrix((val.ravel(), (r.ravel(), c.ravel())), shape=(3 * N, 3 * N))


def csr_to_bsr(A, N):
    """scipy CSR (3N x 3N) -> full BSR arrays (row_ptr, col, val (nnzb,9)) with sorted columns."""
    B = sp.bsr_matrix(A, blocksize=(3, 3))
    B.sort_indices()
    return B.indptr.astype(np.int32), B.indices.astype(np.int32), B.data.reshape(-1, 9).copy()


def lower_blocks_to_full(blocks90, k):
    """[10][9] lower blocks (a>=b, index a(a+1)/2+b) -> (3k x 3k) symmetric matrix."""
    b = np.asarray(blocks90).reshape(10, 3, 3)
    H = np.zeros((3 * k, 3 * k))
    for a in range(k):
        for c in range(a + 1):
            blk = b[a * (a + 1) // 2 + c]
            H[3 * a:3 * a + 3, 3 * c:3 * c + 3] = blk
            H[3 * c:3 * c + 3, 3 * a:3 * a + 3] = blk.T
    return H


def dinv_full(d6):
    d = np.asarray(d6).reshape(-1, 6)
    out = np.zeros((len(d), 3, 3))
    out[:, 0, 0], out[:, 0, 1], out[:, 0, 2] = d[:, 0], d[:, 1], d[:, 2]
    out[:, 1, 0], out[:, 1, 1], out[:, 1, 2] = d[:, 1], d[:, 3], d[:, 4]
    out[:, 2, 0], out[:, 2, 1], out[:, 2, 2] = d[:, 2], d[:, 4], d[:, 5]
    return out


def oracle_state(o, x, y=None, sigma=1.0, ap_keys=None, ap_mu=None, ap_s=None):
    return dict(y=(x if y is None else y).copy(), x_t=x.copy(), sigma=sigma,
                ap_keys=np.zeros((0, 5), np.int64) if ap_keys is None else ap_keys,
                ap_mu=np.zeros(0) if ap_mu is None else ap_mu, ap_s=np.zeros(0) if ap_s is None else ap_s,
                fr_keys=None)


def _node_pairs(ids):
    ids = np.asarray(ids, np.int64)
    k = len(ids)
    return np.repeat(ids, k), np.tile(ids, k)


def assembly_bounds(o, x, y, asm, contact_tol=(), friction=None, friction_tol=(), elastic_tol=1e-12):
    """Per-slot and per-node error bounds of an assembled system (SURVEY c.4 "per slot"):
    slot (a, b) may differ by sum_i tol_i ||P_i||_F over the stencils i that write it (each stencil is
    determined to tol_i relative: 1e-12 for tets, the distance-cancellation bound for contact and
    friction), node j's gradient by sum_i tol_i ||g_i|| plus 1e-12 of its inertia term.  Returns
    (slot bound as N x N CSR, node bound [N])."""
    N = o.N
    rows, cols, vals = [], [], []
    gb = np.zeros(N)
    tets = o.mesh.tets
    if "elastic_P" in asm:
        nP = np.linalg.norm(asm["elastic_P"].reshape(len(tets), -1), axis=1)
        ng = np.linalg.norm(asm["elastic_g"].reshape(len(tets), -1), axis=1)
        rows.append(np.repeat(tets, 4, axis=1).ravel())
        cols.append(np.tile(tets, (1, 4)).ravel())
        vals.append(np.repeat(elastic_tol * nP, 16))
        # a near-rest tet's gradient V P(F) Dm^-T is a small difference of large terms: its rounding
        # is ~u |H| |x_a - x_b| (the gradient is ~ H times the edge vectors), not relative to |g|
        xe = x[tets]
        L = np.max(np.linalg.norm(xe[:, :, None, :] - xe[:, None, :, :], axis=-1), axis=(1, 2))
        for k in range(4):
            np.add.at(gb, tets[:, k], elastic_tol * ng + 1e-15 * nP * L)
    for P, g, ids, t in zip(asm.get("contact_P", []), asm.get("contact_g", []), asm.get("contact_ids", []),
                            contact_tol):
        r, c = _node_pairs(ids)
        rows.append(r), cols.append(c), vals.append(np.full(len(r), t * np.linalg.norm(P)))
        gb[np.asarray(ids)] += t * np.linalg.norm(g)
    for (ids, g, H), t in zip(friction or [], friction_tol):
        r, c = _node_pairs(ids)
        rows.append(r), cols.append(c), vals.append(np.full(len(r), t * np.linalg.norm(H)))
        gb[np.asarray(ids)] += t * np.linalg.norm(g)
    mh = o.mesh.mass / o.h ** 2
    # inertia M(x - y)/h^2: x - y carries ~u |x| absolute error per coordinate
    gb += mh * (1e-12 * np.linalg.norm(x - y, axis=1) + 4e-16 * np.abs(x).max())
    rows.append(np.arange(N)), cols.append(np.arange(N)), vals.append(1e-15 * mh)
    B = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(N, N)).tocsr()
    B.sum_duplicates()
    return B, gb


def slot_errors(Ag, Ao, N):
    """Frobenius norm of each 3x3 block of Ag - Ao as an N x N CSR."""
    D = (Ag - Ao).tocsr()
    D2 = D.multiply(D).tocoo()
    S = sp.coo_matrix((D2.data, (D2.row // 3, D2.col // 3)), shape=(N, N)).tocsr()
    S.sum_duplicates()
    S.data = np.sqrt(S.data)
    return S


def check_assembly_bounds(Ag, Ao, ge, go, B, gb, N, fixed):
    """Every slot of Ag within its bound B (entries of B absent from the pattern: exact 0 allowed
    only for the identity rows / columns of fixed nodes, App. C); every free node's gradient within gb.
    Returns the worst ratios (slot, gradient)."""
    S = slot_errors(Ag, Ao, N).tocoo()
    free_pair = ~(fixed[S.row] | fixed[S.col])
    err = S.data[free_pair]
    bnd = np.asarray(B[S.row[free_pair], S.col[free_pair]]).ravel()
    slot_ratio = float(np.max(err / np.maximum(bnd, 1e-300))) if len(err) else 0.0
    dg = np.linalg.norm((np.asarray(ge) - np.asarray(go)).reshape(N, 3), axis=1)
    g_ratio = float(np.max(dg[~fixed] / np.maximum(gb[~fixed], 1e-300))) if np.any(~fixed) else 0.0
    return slot_ratio, g_ratio
