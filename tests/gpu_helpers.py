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
