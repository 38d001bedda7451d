"""Pins for oracle/so3.py (closed forms, textbook tables, invariants, paper counts)."""
import json
import os

import numpy as np
import pytest

from oracle.so3 import (cg_complex, cg_complex_block, real_cg, real_sph_harm, wigner_d_fit,
                        random_rotation, lm_index)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_sh_closed_forms():
    # Y_0^0 = 1/(2 sqrt(pi)) everywhere; Y_1 at +z = (0, sqrt(3/4pi), 0)
    rng = np.random.default_rng(0)
    r = rng.normal(size=(10, 3))
    r /= np.linalg.norm(r, axis=1, keepdims=True)
    Y = real_sph_harm(1, r)
    assert np.allclose(Y[:, 0], 1 / (2 * np.sqrt(np.pi)), atol=1e-14)
    Yz = real_sph_harm(1, [[0, 0, 1]])[0]
    assert np.allclose(Yz[1:], [0, np.sqrt(3 / (4 * np.pi)), 0], atol=1e-14)
    # l=1 real basis is (y, z, x) with positive coefficient sqrt(3/4pi)
    assert np.allclose(Y[:, 1:4], np.sqrt(3 / (4 * np.pi)) * r[:, [1, 2, 0]], atol=1e-13)


def test_sh_orthonormal_quadrature():
    # Gauss-Legendre x uniform-phi product rule integrates Y_l Y_l' exactly for l, l' <= 3
    x, w = np.polynomial.legendre.leggauss(12)
    phi = np.linspace(0, 2 * np.pi, 24, endpoint=False)
    th = np.arccos(x)
    T, P = np.meshgrid(th, phi, indexing="ij")
    Wt = (w[:, None] * np.full(len(phi), 2 * np.pi / len(phi))[None, :]).reshape(-1)
    pts = np.stack([np.sin(T) * np.cos(P), np.sin(T) * np.sin(P), np.cos(T)], -1).reshape(-1, 3)
    Y = real_sph_harm(3, pts)
    G = (Y * Wt[:, None]).T @ Y
    assert np.allclose(G, np.eye(16), atol=1e-12)


def _val(s):
    return float(eval(s, {"sqrt": np.sqrt}))


def test_cg_complex_textbook():
    gold = json.load(open(os.path.join(GOLD, "cg_textbook.json")))
    for j1, m1, j2, m2, J, M, v in gold["entries"]:
        assert cg_complex(j1, m1, j2, m2, J, M) == pytest.approx(_val(v), abs=1e-15)


def test_cg_complex_unitary_and_selection():
    for l1 in range(4):
        for l2 in range(4):
            # full unitary map (m1,m2) -> (J,M) over all J
            rows = []
            for J in range(abs(l1 - l2), l1 + l2 + 1):
                C = cg_complex_block(l1, l2, J)
                rows.append(C.reshape(2 * J + 1, -1))
                for M in range(-J, J + 1):
                    for m1 in range(-l1, l1 + 1):
                        for m2 in range(-l2, l2 + 1):
                            if m1 + m2 != M:
                                assert C[M + J, m1 + l1, m2 + l2] == 0.0
            U = np.concatenate(rows, 0)
            assert np.allclose(U @ U.T, np.eye(U.shape[0]), atol=1e-14)
            assert np.allclose(U.T @ U, np.eye(U.shape[0]), atol=1e-14)
    assert cg_complex(1, 0, 1, 0, 4, 0) == 0.0   # triangle rule


def test_real_cg_orthonormal_sign_and_diagonal():
    for l1 in range(4):
        for l2 in range(4):
            for L in range(abs(l1 - l2), l1 + l2 + 1):
                C = real_cg(l1, l2, L).reshape(2 * L + 1, -1)
                assert np.allclose(C @ C.T, np.eye(2 * L + 1), atol=1e-12)
                flat = C.reshape(-1)
                assert flat[np.nonzero(np.abs(flat) > 1e-12)[0][0]] > 0     # DESIGN.md §3 sign rule
    for l in range(4):
        # (l,l)->0 = +delta/sqrt(2l+1)
        assert np.allclose(real_cg(l, l, 0)[0], np.eye(2 * l + 1) / np.sqrt(2 * l + 1), atol=1e-14)
    # 1 (x) 1 -> 1 is the cross product (y,z,x ordering): (u x v) in basis (y,z,x), / sqrt(2)
    rng = np.random.default_rng(1)
    u, v = rng.normal(size=3), rng.normal(size=3)   # cartesian
    uy, vy = u[[1, 2, 0]], v[[1, 2, 0]]
    w = np.einsum("Mab,a,b->M", real_cg(1, 1, 1), uy, vy)
    c = np.cross(u, v)[[1, 2, 0]] / np.sqrt(2)
    assert np.allclose(np.abs(w), np.abs(c), atol=1e-14) and (np.allclose(w, c) or np.allclose(w, -c))


def test_cg_density_paper_and_fig5():
    gold = json.load(open(os.path.join(GOLD, "derived_counts.json")))
    nr = nc = 0
    for l1 in range(4):
        for l2 in range(4):
            for L in range(4):
                nr += int((np.abs(real_cg(l1, l2, L)) > 1e-12).sum())
                nc += int((np.abs(cg_complex_block(l1, l2, L)) > 1e-12).sum())
    assert nr / 4096 < 0.20                                   # PAPER.md:547 "less than 20%"
    assert [nr, 4096] == gold["cg_density_real"]
    assert [nc, 4096] == gold["cg_density_complex"]
    C = real_cg(2, 3, 2)                                      # Fig. 5 block
    assert [int((np.abs(C) > 1e-12).sum()), C.size] == gold["fig5_block_nnz"]
    assert [int((np.abs(C[1]) > 1e-12).sum()), C[1].size] == gold["fig5_row_mminus1_nnz"]


def test_wigner_fit_is_a_representation():
    rng = np.random.default_rng(2)
    R1, R2 = random_rotation(rng), random_rotation(rng)
    for l in range(4):
        D1, D2, D12 = wigner_d_fit(l, R1), wigner_d_fit(l, R2), wigner_d_fit(l, R1 @ R2)
        assert np.allclose(D1 @ D1.T, np.eye(2 * l + 1), atol=1e-12)
        assert np.allclose(D12, D1 @ D2, atol=1e-12)
    assert np.allclose(wigner_d_fit(2, np.eye(3)), np.eye(5), atol=1e-12)


def test_real_cg_equivariance():
    rng = np.random.default_rng(3)
    for _ in range(3):
        R = random_rotation(rng)
        D = {l: wigner_d_fit(l, R) for l in range(7)}
        for l1 in range(4):
            for l2 in range(4):
                for L in range(abs(l1 - l2), l1 + l2 + 1):
                    C = real_cg(l1, l2, L)
                    lhs = np.einsum("Mab,ai,bj->Mij", C, D[l1], D[l2])
                    rhs = np.einsum("MN,Nij->Mij", D[L], C)
                    assert np.allclose(lhs, rhs, atol=1e-11), (l1, l2, L)


def test_lm_index_layout():
    seen = sorted(lm_index(l, m) for l in range(4) for m in range(-l, l + 1))
    assert seen == list(range(16))
