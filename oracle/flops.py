"""Convention flop counter for timing reports of the oracle.

Not part of the method: it only counts "what the method must compute" so the
oracle's GFLOP/s (bench.py cpu_baseline) uses the same convention as libhm:
  TRUNC, QR route (l < min(m,n)):  2(m+n)l^2 - 4/3 l^3 + l^3/3 + 22 l^3 + 2(m+n) l k
  TRUNC, dense route:              2 m n l + 14 p q^2 + 8 q^3   (p = max, q = min(m,n))
  addeval, dense leaf m'x n':      2 m' n' c ;  low-rank leaf: 2 k' (m'+n') c
  identity expansion (X|ts I):     0 (a copy)
  dense flush add:                 2 m n l
"""
from __future__ import annotations

from .trees import ADM, DENSE


class ConventionCounter:
    def __init__(self):
        self.trunc = 0.0
        self.eval = 0.0
        self.dense = 0.0

    def on_trunc(self, m, n, l, k):
        if l <= 0:
            return
        if l < min(m, n):
            self.trunc += 2.0 * (m + n) * l * l - (4.0 / 3.0) * l ** 3 + l ** 3 / 3.0 + 22.0 * l ** 3 + 2.0 * (m + n) * l * k
        else:
            p, q = max(m, n), min(m, n)
            self.trunc += 2.0 * m * n * l + 14.0 * p * q * q + 8.0 * q ** 3

    def on_eval(self, H, b, c, identity):
        if identity or c == 0:
            return
        stack = [b]
        while stack:
            x = stack.pop()
            if x.kind == DENSE:
                self.eval += 2.0 * x.t.size * x.s.size * c
            elif x.kind == ADM:
                self.eval += 2.0 * H.A[x.id].shape[1] * (x.t.size + x.s.size) * c
            else:
                stack.extend(x.sons)

    def on_dense(self, m, n, l):
        self.dense += 2.0 * m * n * l

    def total_flops(self):
        return self.trunc + self.eval + self.dense
