"""Mesh precomputation.

TEST INFRASTRUCTURE (see oracle/__init__.py).

 - D_m = [X1-X0, X2-X0, X3-X0], V_e = det(D_m)/6 > 0 (else bad mesh), D_m^{-1}
 - lumped mass m_j = sum_{e ∋ j} rho_e V_e / 4            ("lumped mass matrix")
 - Lamé: mu = E/(2(1+nu)), lambda = E nu/((1+nu)(1-2nu))  (Q1 reading)
 - surface triangles = faces referenced by exactly one tet, oriented outward, plus the listed
   static obstacle triangles; surface edges = unique undirected edges of surface triangles.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class BadMesh(ValueError):
    pass


@dataclass
class Mesh:
    rest_x: np.ndarray        # (N,3)
    tets: np.ndarray          # (T,4) int64
    fixed: np.ndarray         # (N,) bool
    Dm_inv: np.ndarray        # (T,3,3)
    vol: np.ndarray           # (T,)
    mu: np.ndarray            # (T,) Lamé mu per tet
    lam: np.ndarray           # (T,) Lamé lambda per tet
    mass: np.ndarray          # (N,)
    tris: np.ndarray          # (F,3) surface triangles (outward) incl. obstacles
    edges: np.ndarray         # (E,2) unique surface edges (i<j)
    surf_verts: np.ndarray    # (V,) vertices of surface triangles
    arap: np.ndarray = None   # (T,) bool: ARAP tet (NEXT-4, scene["material_model"] == 1), else Neo-Hookean

    @property
    def n(self):
        return len(self.rest_x)


def precompute(scene) -> Mesh:
    X = np.asarray(scene["rest_x"], np.float64)
    tets = np.asarray(scene["tets"], np.int64).reshape(-1, 4)
    fixed = np.asarray(scene["node_fixed"]).astype(bool)
    N = len(X)
    if len(tets) and (tets.min() < 0 or tets.max() >= N):
        raise BadMesh("tet index out of range")
    mats = np.asarray(scene["materials"], np.float64).reshape(-1, 3)
    tm = np.asarray(scene["tet_material"], np.int64)

    Dm = np.stack([X[tets[:, 1]] - X[tets[:, 0]], X[tets[:, 2]] - X[tets[:, 0]],
                   X[tets[:, 3]] - X[tets[:, 0]]], axis=2)  # columns are edge vectors
    detDm = np.linalg.det(Dm) if len(tets) else np.zeros(0)
    if np.any(detDm <= 0):
        raise BadMesh(f"inverted or degenerate rest tet {int(np.argmax(detDm <= 0))}")
    vol = detDm / 6.0
    Dm_inv = np.linalg.inv(Dm) if len(tets) else np.zeros((0, 3, 3))
    E, nu, rho = mats[tm, 0], mats[tm, 1], mats[tm, 2]
    mu = E / (2.0 * (1.0 + nu))
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mass = np.zeros(N)
    for k in range(4):
        np.add.at(mass, tets[:, k], rho * vol / 4.0)

    # boundary faces: referenced exactly once; orient away from the opposite vertex
    faces = []
    opp = []
    for (i, j, k, o) in [(0, 1, 2, 3), (0, 1, 3, 2), (0, 2, 3, 1), (1, 2, 3, 0)]:
        faces.append(tets[:, [i, j, k]])
        opp.append(tets[:, o])
    faces = np.concatenate(faces, axis=0)
    opp = np.concatenate(opp, axis=0)
    key = np.sort(faces, axis=1)
    _, idx, counts = np.unique(key, axis=0, return_index=True, return_counts=True)
    bidx = idx[counts == 1]
    bf = faces[bidx]
    bo = opp[bidx]
    a, b, c = X[bf[:, 0]], X[bf[:, 1]], X[bf[:, 2]]
    nrm = np.cross(b - a, c - a)
    flip = np.einsum("ij,ij->i", nrm, X[bo] - a) > 0
    bf[flip, 1], bf[flip, 2] = bf[flip, 2].copy(), bf[flip, 1].copy()
    obst = np.asarray(scene.get("obstacle_tris", np.zeros((0, 3))), np.int64).reshape(-1, 3)
    if len(obst) and not np.all(fixed[obst]):
        raise BadMesh("obstacle triangle references a free node")
    tris = np.concatenate([bf, obst], axis=0)
    # canonical order for determinism: sort rows by sorted key
    order = np.lexsort(np.sort(tris, axis=1).T[::-1])
    tris = tris[order]
    e = np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [2, 0]]], axis=0)
    e = np.unique(np.sort(e, axis=1), axis=0)
    sv = np.unique(tris.ravel())
    model = np.asarray(scene.get("material_model", np.zeros(len(mats))), np.int64).reshape(-1)
    arap = model[tm] == 1 if len(tets) else np.zeros(0, bool)
    return Mesh(X, tets, fixed, Dm_inv, vol, mu, lam, mass, tris, e, sv, arap)
