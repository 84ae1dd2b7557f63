"""Exact rational polynomial arithmetic on the reference tetrahedron (test helper).

Independent of the oracle: polynomials are dicts {(a,b,c): Fraction} in x,y,z and
are integrated exactly with  int_T x^a y^b z^c = a! b! c! / (a+b+c+3)!  over
T = {x,y,z >= 0, x+y+z <= 1}.  Used to pin the oracle's element matrices
(exact rationals) and its quadrature rule.
"""
from fractions import Fraction
from math import factorial


def mono_integral(a, b, c):
    return Fraction(factorial(a) * factorial(b) * factorial(c), factorial(a + b + c + 3))


def padd(p, q, s=1):
    r = dict(p)
    for k, v in q.items():
        r[k] = r.get(k, 0) + s * v
    return {k: v for k, v in r.items() if v != 0}


def pmul(p, q):
    r = {}
    for (a1, b1, c1), v1 in p.items():
        for (a2, b2, c2), v2 in q.items():
            k = (a1 + a2, b1 + b2, c1 + c2)
            r[k] = r.get(k, 0) + v1 * v2
    return {k: v for k, v in r.items() if v != 0}


def pscale(p, s):
    return {k: v * s for k, v in p.items() if v * s != 0}


def pdiff(p, d):
    r = {}
    for k, v in p.items():
        if k[d] > 0:
            kk = list(k)
            kk[d] -= 1
            r[tuple(kk)] = r.get(tuple(kk), 0) + v * k[d]
    return r


def pint(p):
    return sum((v * mono_integral(*k) for k, v in p.items()), Fraction(0))


ONE = {(0, 0, 0): Fraction(1)}
X = {(1, 0, 0): Fraction(1)}
Y = {(0, 1, 0): Fraction(1)}
Z = {(0, 0, 1): Fraction(1)}
LAM = [padd(padd(padd(ONE, X, -1), Y, -1), Z, -1), X, Y, Z]
EDGES = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]


def p2_basis_exact():
    out = []
    for m in range(4):
        out.append(pmul(LAM[m], padd(pscale(LAM[m], 2), ONE, -1)))
    for i, j in EDGES:
        out.append(pscale(pmul(LAM[i], LAM[j]), 4))
    return out


def reference_element_matrices(form_full=True):
    """Exact A (30x30, eta=1), B (4x30) on the reference tet; dof = 3 a + c."""
    phi = p2_basis_exact()
    grad = [[pdiff(p, d) for d in range(3)] for p in phi]
    n = 30
    A = [[Fraction(0)] * n for _ in range(n)]
    for a in range(10):
        for c in range(3):
            for b in range(10):
                for d in range(3):
                    # eps(phi_a e_c):eps(phi_b e_d) = 1/2 (delta_cd g_a.g_b + g_a[d] g_b[c])
                    t = {}
                    if c == d:
                        for k in range(3):
                            t = padd(t, pscale(pmul(grad[a][k], grad[b][k]), Fraction(1, 2)))
                    t = padd(t, pscale(pmul(grad[a][d], grad[b][c]), Fraction(1, 2)))
                    if form_full:
                        t = padd(t, pscale(pmul(grad[a][c], grad[b][d]), Fraction(-1, 3)))
                    A[3 * a + c][3 * b + d] = 2 * pint(t)
    B = [[Fraction(0)] * n for _ in range(4)]
    for p in range(4):
        for b in range(10):
            for d in range(3):
                B[p][3 * b + d] = -pint(pmul(LAM[p], grad[b][d]))
    return A, B
