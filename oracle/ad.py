"""Batched forward-mode second-order automatic differentiation (value, gradient, Hessian).

TEST INFRASTRUCTURE (see oracle/__init__.py).  Derivatives in the oracle are taken by this AD
over the plain energy expressions, so they are exact to rounding and independent of any
hand-derived closed form used by the CUDA path ("forward-mode second-order
AD ... makes the oracle independent of the GPU's hand-derived closed forms").

A ``D2`` holds, for a batch of B independent evaluations of a scalar function of n inputs:
    v : (B,)        value
    g : (B, n)      gradient
    H : (B, n, n)   Hessian
"""
from __future__ import annotations

import numpy as np


class D2:
    __slots__ = ("v", "g", "H")

    def __init__(self, v, g, H):
        self.v = v
        self.g = g
        self.H = H

    # ---- constructors -------------------------------------------------------
    @staticmethod
    def variables(x):
        """x: (B, n) -> list of n D2 seeds (identity gradients, zero Hessians)."""
        B, n = x.shape
        out = []
        for i in range(n):
            g = np.zeros((B, n))
            g[:, i] = 1.0
            out.append(D2(x[:, i].astype(np.float64), g, np.zeros((B, n, n))))
        return out

    def const_like(self, c):
        B, n = self.g.shape
        return D2(np.broadcast_to(np.asarray(c, np.float64), (B,)).astype(np.float64),
                  np.zeros((B, n)), np.zeros((B, n, n)))

    # ---- arithmetic --------------------------------------------------------
    def __add__(self, o):
        if isinstance(o, D2):
            return D2(self.v + o.v, self.g + o.g, self.H + o.H)
        return D2(self.v + o, self.g, self.H)

    __radd__ = __add__

    def __neg__(self):
        return D2(-self.v, -self.g, -self.H)

    def __sub__(self, o):
        return self + (-o)

    def __rsub__(self, o):
        return (-self) + o

    def __mul__(self, o):
        if isinstance(o, D2):
            outer = self.g[:, :, None] * o.g[:, None, :]
            H = (self.H * o.v[:, None, None] + o.H * self.v[:, None, None]
                 + outer + np.transpose(outer, (0, 2, 1)))
            return D2(self.v * o.v, self.g * o.v[:, None] + o.g * self.v[:, None], H)
        c = np.asarray(o, np.float64)
        if c.ndim == 0:
            return D2(self.v * c, self.g * c, self.H * c)
        return D2(self.v * c, self.g * c[:, None], self.H * c[:, None, None])

    __rmul__ = __mul__

    def _chain(self, f0, f1, f2):
        """Compose a scalar function with value f0, first derivative f1, second f2 (arrays (B,))."""
        H = f1[:, None, None] * self.H + f2[:, None, None] * (self.g[:, :, None] * self.g[:, None, :])
        return D2(f0, f1[:, None] * self.g, H)

    def recip(self):
        v = self.v
        return self._chain(1.0 / v, -1.0 / v ** 2, 2.0 / v ** 3)

    def __truediv__(self, o):
        if isinstance(o, D2):
            return self * o.recip()
        return self * (1.0 / np.asarray(o, np.float64))

    def __rtruediv__(self, o):
        return self.recip() * o

    def log(self):
        v = self.v
        return self._chain(np.log(v), 1.0 / v, -1.0 / v ** 2)

    def sqrt(self):
        s = np.sqrt(self.v)
        return self._chain(s, 0.5 / s, -0.25 / (s * self.v))

    def sq(self):
        return self * self

    def select(self, mask, other):
        """Per-batch select: where mask take self else other."""
        m = np.asarray(mask, bool)
        return D2(np.where(m, self.v, other.v), np.where(m[:, None], self.g, other.g),
                  np.where(m[:, None, None], self.H, other.H))


def dot3(a, b):
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]


def sub3(a, b):
    return [a[0] - b[0], a[1] - b[1], a[2] - b[2]]


def cross3(a, b):
    return [a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]]


def apply_scalar(fn, x):
    """Evaluate D2 of fn over inputs x (B, n) where fn maps a list of n D2 to one D2."""
    return fn(D2.variables(np.asarray(x, np.float64)))
