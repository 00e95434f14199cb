"""csrc/tn_math.cuh compiled for the host and checked against the CPU oracle's algebra.

No GPU needed: the header is plain inline arithmetic shared by every TensorNet kernel, so a
transcription error in the forward or reverse formulas shows up here first.
"""

import ctypes
import os
import subprocess

import numpy as np
import pytest

from oracle import tensornet_oracle as T
from oracle import neighbors_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def lib(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("host") / "libtnmath.so")
    subprocess.run(["g++", "-O1", "-shared", "-fPIC", "-x", "c++",
                    os.path.join(HERE, "host", "tn_math_host.cpp"), "-o", out], check=True)
    L = ctypes.CDLL(out)
    L.h_frob.restype = ctypes.c_float
    L.h_normalize_fwd.restype = ctypes.c_float
    L.h_silu.restype = ctypes.c_float
    L.h_silu_grad.restype = ctypes.c_float
    L.h_silu.argtypes = [ctypes.c_float]
    L.h_silu_grad.argtypes = [ctypes.c_float]
    L.h_basis.argtypes = [ctypes.c_float] * 3 + [ctypes.c_void_p]
    L.h_hermite.argtypes = [ctypes.c_float, ctypes.c_void_p]
    L.h_normalize_bwd.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_float, ctypes.c_void_p]
    return L


def f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def test_basis_roundtrip_and_dots(lib, rng):
    for _ in range(20):
        c = f32(rng.standard_normal(9))
        m = np.zeros(9, np.float32)
        lib.h_to_full(p(c), p(m))
        assert np.allclose(m.reshape(3, 3), T.to_full(c.astype(np.float64)), atol=1e-6)
        back = np.zeros(9, np.float32)
        lib.h_from_full(p(m), p(back))
        assert np.allclose(back, c, atol=1e-6)
        d = f32(rng.standard_normal(9))
        out = np.zeros(3, np.float32)
        lib.h_dots(p(c), p(d), p(out))
        c64, d64 = c.astype(np.float64), d.astype(np.float64)
        assert np.allclose(out, [T.dot_I(c64, d64), T.dot_A(c64, d64), T.dot_S(c64, d64)], rtol=1e-5, atol=1e-6)
        assert np.isclose(lib.h_frob(p(c), p(d)), (T.to_full(c64) * T.to_full(d64)).sum(), rtol=1e-5, atol=1e-6)


def test_edge_basis(lib, rng):
    u = rng.standard_normal(3)
    u /= np.linalg.norm(u)
    b = np.zeros(9, np.float32)
    lib.h_basis(*[float(x) for x in u], p(b))
    ref = T.edge_basis(u[None, :], np.array([False]))[0]
    assert np.allclose(b, ref, atol=1e-6)
    lib.h_basis(0.0, 0.0, 0.0, p(b))
    assert np.array_equal(b, [1, 0, 0, 0, 0, 0, 0, 0, 0])


def test_node_product_forward_and_reverse(lib, rng):
    for _ in range(10):
        M, Y, GQ = (f32(0.7 * rng.standard_normal(9)) for _ in range(3))
        Q = np.zeros(9, np.float32)
        lib.h_node_product_fwd(p(M), p(Y), p(Q))
        M64, Y64, G64 = (a.astype(np.float64) for a in (M, Y, GQ))
        Pf = T.to_full(M64) @ T.to_full(Y64) + T.to_full(Y64) @ T.to_full(M64)
        Pc = T.from_full(Pf)
        npn = T.frob(Pc, Pc) + 1.0
        assert np.allclose(Q, Pc / npn, rtol=1e-5, atol=1e-6)
        GM, GY = np.zeros(9, np.float32), np.zeros(9, np.float32)
        lib.h_node_product_bwd(p(M), p(Y), p(GQ), p(GM), p(GY))
        G_P = G64 / npn - Pc * (2.0 * T.frob(G64, Pc) / npn**2)
        GPf = T.to_full(G_P)
        refM = T.from_full(GPf @ T.to_full(Y64).T + T.to_full(Y64).T @ GPf)
        refY = T.from_full(T.to_full(M64).T @ GPf + GPf @ T.to_full(M64).T)
        assert np.allclose(GM, refM, rtol=1e-4, atol=1e-6)
        assert np.allclose(GY, refY, rtol=1e-4, atol=1e-6)


def test_residual_and_normalize(lib, rng):
    for _ in range(10):
        Xh, D, G = (f32(0.5 * rng.standard_normal(9)) for _ in range(3))
        Xn = np.zeros(9, np.float32)
        lib.h_residual_fwd(p(Xh), p(D), p(Xn))
        D64 = T.to_full(D.astype(np.float64))
        assert np.allclose(Xn, Xh + D + T.from_full(D64 @ D64), rtol=1e-5, atol=1e-6)
        GD = np.zeros(9, np.float32)
        lib.h_residual_bwd(p(G), p(D), p(GD))
        Gf = T.to_full(G.astype(np.float64))
        assert np.allclose(GD, G + T.from_full(Gf @ D64.T + D64.T @ Gf), rtol=1e-5, atol=1e-6)
        X = f32(rng.standard_normal(9))
        out = np.zeros(9, np.float32)
        n = lib.h_normalize_fwd(p(X), p(out))
        X64 = X.astype(np.float64)
        n64 = T.frob(X64, X64) + 1.0
        assert np.isclose(n, n64, rtol=1e-6) and np.allclose(out, X64 / n64, rtol=1e-5, atol=1e-7)
        GX = np.zeros(9, np.float32)
        lib.h_normalize_bwd(p(G), p(out), ctypes.c_float(n), p(GX))
        G64 = G.astype(np.float64)
        ref = G64 / n64 - X64 * (2.0 * T.frob(G64, X64) / n64**2)
        assert np.allclose(GX, ref, rtol=1e-4, atol=1e-6)


def test_hermite_and_silu(lib):
    w = np.zeros(8, np.float32)
    for t in (0.0, 0.25, 0.5, 1.0):
        lib.h_hermite(t, p(w))
        ref = [2*t**3-3*t**2+1, t**3-2*t**2+t, -2*t**3+3*t**2, t**3-t**2,
               6*t**2-6*t, 3*t**2-4*t+1, -6*t**2+6*t, 3*t**2-2*t]
        assert np.allclose(w, ref, atol=1e-6)
    for x in (-20.0, -3.0, 0.0, 0.7, 15.0):
        assert np.isclose(lib.h_silu(x), O.silu(np.array([x]))[0], rtol=1e-6, atol=1e-9)
        assert np.isclose(lib.h_silu_grad(x), O.silu_grad(np.array([x]))[0], rtol=1e-5, atol=1e-8)
