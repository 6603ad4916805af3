"""Map-based assembly of the Newton system and the stiffness grouping.

TEST INFRASTRUCTURE (see oracle/__init__.py).

A = M/h^2 + sum_i S_i^T P(H_i) S_i  (+ friction stencils, PSD by construction, not projected)
    - PAPER.md:386-389 (projected stencil Hessians), 416-418 (D / L / C storage of the same matrix)
    - fixed DOFs: identity row and column, zero rhs (App. C)
Lambda_rr = m_j/h^2 + sum_{elastic, contact stencils containing j} lambda_bar_i (Q17/Q18)
e_j = Lambda_{3j} + Lambda_{3j+1} + Lambda_{3j+2}, group_j = floor(log10 e_j)  (Q19)

The assembled system is returned as a dict of 3x3 blocks {(row, col): block} summed in ascending
stencil order (tets, then contact keys, then friction), plus a dense/CSR conversion.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

# exact decimal literals 1e-40 .. 1e40 (Q19)
_DECADES = {k: float(f"1e{k}") for k in range(-60, 61)}


def floor_log10(e):
    """Exact floor(log10(e)) for e > 0: start from numpy's log10, then correct against the
    decimal literal table so the decade test is a pure comparison (Q19)."""
    e = np.asarray(e, np.float64)
    g = np.floor(np.log10(e)).astype(np.int64)
    out = g.copy()
    for i in range(len(e)):
        gi = int(g[i])
        while gi > -60 and e[i] < _DECADES[gi]:
            gi -= 1
        while gi < 59 and e[i] >= _DECADES[gi + 1]:
            gi += 1
        out[i] = gi
    return out


class BlockSystem:
    """Dictionary-of-blocks symmetric matrix over N nodes (3x3 blocks)."""

    def __init__(self, N):
        self.N = N
        self.blocks = {}

    def add(self, i, j, B):
        key = (int(i), int(j))
        if key in self.blocks:
            self.blocks[key] = self.blocks[key] + B
        else:
            self.blocks[key] = np.array(B, dtype=np.float64)

    def add_stencil(self, ids, H):
        k = len(ids)
        for a in range(k):
            for b in range(k):
                self.add(ids[a], ids[b], H[3 * a:3 * a + 3, 3 * b:3 * b + 3])

    def finalize_fixed(self, fixed):
        """Drop fixed rows/cols; fixed diagonal -> identity (App. C)."""
        nb = {}
        for (i, j), B in self.blocks.items():
            if fixed[i] or fixed[j]:
                continue
            nb[(i, j)] = B
        for i in np.nonzero(fixed)[0]:
            nb[(int(i), int(i))] = np.eye(3)
        self.blocks = nb

    def to_csr(self):
        rows, cols, vals = [], [], []
        for (i, j), B in self.blocks.items():
            for a in range(3):
                for b in range(3):
                    rows.append(3 * i + a)
                    cols.append(3 * j + b)
                    vals.append(B[a, b])
        return sp.csr_matrix((vals, (rows, cols)), shape=(3 * self.N, 3 * self.N))

    def to_dense(self):
        return self.to_csr().toarray()

    def diag_blocks(self):
        D = np.zeros((self.N, 3, 3))
        for i in range(self.N):
            D[i] = self.blocks.get((i, i), np.zeros((3, 3)))
        return D

    def to_bsr_arrays(self):
        """Full (both-triangle) BSR with rows sorted by column: (row_ptr, col, val (nnzb,3,3))."""
        keys = sorted(self.blocks.keys())
        row_ptr = np.zeros(self.N + 1, np.int64)
        col = np.zeros(len(keys), np.int64)
        val = np.zeros((len(keys), 3, 3))
        for n, (i, j) in enumerate(keys):
            row_ptr[i + 1] += 1
            col[n] = j
            val[n] = self.blocks[(i, j)]
        return np.cumsum(row_ptr), col, val


def stiffness_groups(mass, h, stencil_nodes, stencil_lbar, fixed):
    """Lambda diagonal -> e_j and group ids (free nodes only; fixed nodes get group None=-999)."""
    N = len(mass)
    lam_diag = np.repeat(mass / (h * h), 3).reshape(N, 3).copy()
    for ids, lb in zip(stencil_nodes, stencil_lbar):
        for j in ids:
            lam_diag[j] += lb
    e = lam_diag.sum(axis=1)
    grp = np.full(N, -999, np.int64)
    free = ~fixed
    grp[free] = floor_log10(e[free])
    return e, grp
