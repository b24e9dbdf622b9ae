"""O4 — exact rational solve of the precise test, for known-answer tests.

TEST INFRASTRUCTURE ONLY (see oracle/canonical.py header).

Solves PAPER.md Eq. (26) / SPEC.md:460 ``p + s·e1 + t·e2 = q + a·f1 + b·f2`` in
``fractions.Fraction`` arithmetic by Gaussian elimination with exact pivots — an
independent elimination oracle as SPEC.md:468 asks for ("verify ... against
hand-solved linear system [DERIVED: 4×4 solve by independent elimination
oracle]").  On dyadic inputs whose canonical determinants are exact (SURVEY.md
§7.3: ≤ ~11 significant bits per coordinate), the canonical FP64 result equals
the correctly rounded exact result, so this pins the canonical arithmetic.
"""
from __future__ import annotations

from fractions import Fraction


def solve_exact(p, e1, e2, q, f1, f2):
    """Return (s, t, a, b) as Fractions, or None if the system is singular."""
    F = [[Fraction(float(e1[r])), Fraction(float(e2[r])), -Fraction(float(f1[r])),
          -Fraction(float(f2[r])), Fraction(float(q[r])) - Fraction(float(p[r]))] for r in range(4)]
    n = 4
    for col in range(n):
        piv = next((r for r in range(col, n) if F[r][col] != 0), None)
        if piv is None:
            return None
        F[col], F[piv] = F[piv], F[col]
        for r in range(n):
            if r != col and F[r][col] != 0:
                fac = F[r][col] / F[col][col]
                F[r] = [F[r][k] - fac * F[col][k] for k in range(n + 1)]
    return tuple(F[r][n] / F[r][r] for r in range(n))


def det_exact(e1, e2, f1, f2):
    """det[e1, e2, f1, f2] exactly (Leibniz over 24 permutations)."""
    from itertools import permutations

    cols = [[Fraction(float(v[r])) for r in range(4)] for v in (e1, e2, f1, f2)]
    total = Fraction(0)
    for perm in permutations(range(4)):
        sign = 1
        for i in range(4):
            for j in range(i + 1, 4):
                if perm[i] > perm[j]:
                    sign = -sign
        prod = Fraction(sign)
        for c in range(4):
            prod *= cols[c][perm[c]]
        total += prod
    return total


def accepted(sol) -> bool:
    """Exact acceptance: s,t,a,b ≥ 0, s+t ≤ 1, a+b ≤ 1."""
    if sol is None:
        return False
    s, t, a, b = sol
    return s >= 0 and t >= 0 and a >= 0 and b >= 0 and s + t <= 1 and a + b <= 1
