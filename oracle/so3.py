"""SO(3) machinery for the oracle (test infrastructure only; see oracle/__init__.py).

Conventions are DESIGN.md §3 (readings s6-s9 of SURVEY.md §8(c)):
  * real spherical harmonics, component index lm = l*l + l + m, m = -l..l,
    built from Condon-Shortley complex harmonics ("Spherical
    harmonics ... Y_l^m ... basis for the (2l+1)-dimensional irreducible
    representation"); for l=1 this is (y, z, x).
  * complex Clebsch-Gordan coefficients by Racah's closed-form sum, with the
    selection rules of PAPER.md:696-697 ("triangle rule", "m1 + m2 = m3").
  * real coupling C^L_{l1 l2}[M, m1, m2] = basis change of the complex CG,
    rows orthonormal ("component" normalization), overall sign fixed so the
    first entry with |x| > 1e-12 in row-major [M][m1][m2] order is positive.
"""
from fractions import Fraction
from functools import lru_cache
from math import factorial, sqrt

import numpy as np

NONZERO = 1e-12


def lm_index(l, m):
    """Position of component (l, m) in the (lmax+1)^2 feature row (PAPER.md:1528 layout)."""
    return l * l + l + m


# ---------------------------------------------------------------- complex CG
def _f(n):
    return factorial(n)


@lru_cache(maxsize=None)
def cg_complex(j1, m1, j2, m2, J, M):
    """<j1 m1; j2 m2 | J M> by Racah's formula (exact rationals, one final sqrt).

    Zero unless m1 + m2 = M and |j1-j2| <= J <= j1+j2.
    """
    if m1 + m2 != M or not (abs(j1 - j2) <= J <= j1 + j2):
        return 0.0
    if abs(m1) > j1 or abs(m2) > j2 or abs(M) > J:
        return 0.0
    pref = Fraction((2 * J + 1) * _f(J + j1 - j2) * _f(J - j1 + j2) * _f(j1 + j2 - J), _f(j1 + j2 + J + 1))
    pref *= _f(J + M) * _f(J - M) * _f(j1 - m1) * _f(j1 + m1) * _f(j2 - m2) * _f(j2 + m2)
    s = Fraction(0)
    for k in range(0, j1 + j2 - J + 1):
        den = [k, j1 + j2 - J - k, j1 - m1 - k, j2 + m2 - k, J - j2 + m1 + k, J - j1 - m2 + k]
        if min(den) < 0:
            continue
        term = Fraction(1, 1)
        for d in den:
            term /= _f(d)
        s += (-1) ** k * term
    if s == 0:
        return 0.0
    sign = 1.0 if s > 0 else -1.0
    return sign * sqrt(float(pref * s * s))


def cg_complex_block(l1, l2, L):
    """Dense complex-basis block [M][m1][m2] (indices shifted by +l)."""
    out = np.zeros((2 * L + 1, 2 * l1 + 1, 2 * l2 + 1))
    for M in range(-L, L + 1):
        for m1 in range(-l1, l1 + 1):
            m2 = M - m1
            if -l2 <= m2 <= l2:
                out[M + L, m1 + l1, m2 + l2] = cg_complex(l1, m1, l2, m2, L, M)
    return out


# ---------------------------------------------------------- real basis change
def real_from_complex(l):
    """Q_l with Y_real = Q_l @ Y_complex (rows: real m = -l..l; cols: complex m = -l..l).

    Y_{l,m}^real = i/sqrt2 (Y_l^m - (-1)^m Y_l^{-m})   m < 0
                 = Y_l^0                               m = 0
                 = 1/sqrt2 (Y_l^{-m} + (-1)^m Y_l^m)   m > 0
    """
    Q = np.zeros((2 * l + 1, 2 * l + 1), dtype=complex)
    r = 1 / np.sqrt(2)
    for m in range(-l, l + 1):
        row = m + l
        if m < 0:
            Q[row, m + l] += 1j * r
            Q[row, -m + l] += -1j * r * (-1) ** m
        elif m == 0:
            Q[row, l] = 1.0
        else:
            Q[row, -m + l] += r
            Q[row, m + l] += r * (-1) ** m
    return Q


def real_sph_harm(lmax, xyz):
    """Real SH of unit vectors xyz [n,3] -> [n, (lmax+1)^2], DESIGN.md §3 basis.

    Complex Y_l^m from scipy.special.sph_harm_y (Condon-Shortley phase), then Q_l.
    """
    from scipy.special import sph_harm_y

    xyz = np.atleast_2d(np.asarray(xyz, dtype=float))
    theta = np.arccos(np.clip(xyz[:, 2], -1, 1))
    phi = np.arctan2(xyz[:, 1], xyz[:, 0])
    out = np.zeros((xyz.shape[0], (lmax + 1) ** 2))
    for l in range(lmax + 1):
        yc = np.stack([sph_harm_y(l, m, theta, phi) for m in range(-l, l + 1)], axis=1)
        yr = yc @ real_from_complex(l).T
        assert np.abs(yr.imag).max() < 1e-12
        out[:, l * l:(l + 1) ** 2] = yr.real
    return out


# ------------------------------------------------------------------- real CG
@lru_cache(maxsize=None)
def real_cg(l1, l2, L):
    """Real coupling C^L_{l1 l2}[M, m1, m2]; zero block if the triangle rule fails.

    C_real = Q_L  C_complex  (Q_l1^dagger (x) Q_l2^dagger), made real by removing
    the global phase, then signed by the first-nonzero-positive rule.
    """
    if not (abs(l1 - l2) <= L <= l1 + l2):
        return np.zeros((2 * L + 1, 2 * l1 + 1, 2 * l2 + 1))
    C = cg_complex_block(l1, l2, L)
    QL, Q1, Q2 = real_from_complex(L), real_from_complex(l1), real_from_complex(l2)
    Cr = np.einsum("Mn,nab,ia,jb->Mij", QL, C, Q1.conj(), Q2.conj())
    # the coupling is unique up to a complex phase: pick the phase of the largest entry
    flat = Cr.reshape(-1)
    ph = flat[np.argmax(np.abs(flat))]
    Cr = Cr / (ph / abs(ph))
    assert np.abs(Cr.imag).max() < 1e-12
    Cr = Cr.real.copy()
    Cr[np.abs(Cr) < NONZERO] = 0.0
    first = Cr.reshape(-1)[np.nonzero(np.abs(Cr.reshape(-1)) > NONZERO)[0][0]]
    if first < 0:
        Cr = -Cr
    Cr.setflags(write=False)
    return Cr


# ----------------------------------------------------------- Wigner-D (tests)
def wigner_d_fit(l, R, n_samples=200, seed=0):
    """D^l(R) fitted by least squares from Y_l(R r) = D^l(R) Y_l(r) on random r.

    Independent of every CG routine: it only uses real_sph_harm (scipy-backed).
    """
    rng = np.random.default_rng(seed)
    r = rng.normal(size=(n_samples, 3))
    r /= np.linalg.norm(r, axis=1, keepdims=True)
    Y = real_sph_harm(l, r)[:, l * l:]
    YR = real_sph_harm(l, r @ R.T)[:, l * l:]
    # YR^T = D Y^T  ->  Y D^T = YR
    Dt, *_ = np.linalg.lstsq(Y, YR, rcond=None)
    return Dt.T


def random_rotation(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    a, b, c, d = q
    return np.array([
        [a * a + b * b - c * c - d * d, 2 * (b * c - a * d), 2 * (b * d + a * c)],
        [2 * (b * c + a * d), a * a - b * b + c * c - d * d, 2 * (c * d - a * b)],
        [2 * (b * d - a * c), 2 * (c * d + a * b), a * a - b * b - c * c + d * d],
    ])


def block_diag_d(lmax, R):
    """Block-diagonal D(R) acting on a (lmax+1)^2 feature row."""
    n = (lmax + 1) ** 2
    D = np.zeros((n, n))
    for l in range(lmax + 1):
        D[l * l:(l + 1) ** 2, l * l:(l + 1) ** 2] = wigner_d_fit(l, R)
    return D
