"""TEST INFRASTRUCTURE ONLY -- ctypes binding of the CPU oracle (oracle.cpp).

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs. The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liboracle.so")


def build():
    subprocess.run(["make", "-C", HERE, "_build/liboracle.so"], check=True, stdout=subprocess.DEVNULL)


def _lib():
    if not os.path.exists(LIB):
        build()
    lib = C.CDLL(LIB)
    lib.orc_create.restype = C.c_void_p
    lib.orc_create.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p,
                               C.c_void_p]
    lib.orc_destroy.argtypes = [C.c_void_p]
    lib.orc_set_dt.argtypes = [C.c_void_p, C.c_double]
    lib.orc_potential.argtypes = [C.c_void_p, C.c_void_p]
    lib.orc_initial_samples.restype = C.c_double
    lib.orc_initial_samples.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p]
    lib.orc_analyze.argtypes = [C.c_void_p, C.c_void_p]
    lib.orc_synthesize.argtypes = [C.c_void_p, C.c_void_p]
    lib.orc_steps.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    lib.orc_l2_norm.restype = C.c_double
    lib.orc_l2_norm.argtypes = [C.c_void_p, C.c_void_p]
    lib.orc_energy.restype = C.c_double
    lib.orc_energy.argtypes = [C.c_void_p, C.c_void_p]
    lib.orc_dft.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int]
    lib.orc_points.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.orc_cbc_exhaustive.argtypes = [C.c_int64, C.c_int, C.c_void_p, C.c_void_p]
    lib.orc_aaset.restype = C.c_int
    lib.orc_aaset.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p]
    return lib


_L = None


def lib():
    global _L
    if _L is None:
        _L = _lib()
    return _L


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def dft(x, sign=-1):
    x = np.ascontiguousarray(x, np.complex128)
    out = np.zeros_like(x)
    lib().orc_dft(_p(x), _p(out), x.size, sign)
    return out


def points(gen, moduli):
    g = np.ascontiguousarray(np.asarray(gen, np.int64))
    n = np.ascontiguousarray(np.asarray(moduli, np.int64))
    r, d = g.shape
    out = np.zeros((int(np.prod(n)), d), np.int64)
    lib().orc_points(d, r, _p(g), _p(n), _p(out))
    return out


def cbc_exhaustive(n, d):
    z = np.zeros(d, np.int64)
    w = np.zeros(d)
    lib().orc_cbc_exhaustive(n, d, _p(z), _p(w))
    return z, w


def aaset(gen, moduli, with_vectors=True, cap=-1.0):
    g = np.ascontiguousarray(np.asarray(gen, np.int64))
    n = np.ascontiguousarray(np.asarray(moduli, np.int64))
    r, d = g.shape
    N = int(np.prod(n))
    norm2 = np.zeros(N, np.uint32)
    h = np.zeros((N, d), np.int16) if with_vectors else None
    rc = lib().orc_aaset(d, r, _p(g), _p(n), cap, _p(norm2), _p(h) if h is not None else None)
    if rc != 0:
        raise RuntimeError("oracle aaset: radius cap reached")
    return norm2, h


class Oracle:
    """Literal SPEC.md Strang propagator on coefficients (CPU)."""

    def __init__(self, gen, moduli, norm2, eps, a, b):
        g = np.ascontiguousarray(np.asarray(gen, np.int64))
        self.moduli = np.ascontiguousarray(np.asarray(moduli, np.int64))
        r, d = g.shape
        self.N = int(np.prod(self.moduli))
        self._norm2 = np.ascontiguousarray(norm2, np.uint32)
        self._a = np.ascontiguousarray(a, np.float64)
        self._b = np.ascontiguousarray(b if d > 1 else [0.0], np.float64)
        self._h = lib().orc_create(d, r, _p(g), _p(self.moduli), _p(self._norm2), eps, _p(self._a), _p(self._b))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_destroy(self._h)
            self._h = None

    def set_dt(self, dt):
        lib().orc_set_dt(self._h, dt)

    def potential(self):
        out = np.zeros(self.N)
        lib().orc_potential(self._h, _p(out))
        return out

    def initial_samples(self, c, p, sigma):
        c = np.ascontiguousarray(c, np.float64)
        p = np.ascontiguousarray(p, np.int32)
        out = np.zeros(self.N, np.complex128)
        lib().orc_initial_samples(self._h, _p(c), _p(p), sigma, _p(out))
        return out

    def analyze(self, u):
        x = np.array(u, np.complex128, copy=True)
        lib().orc_analyze(self._h, _p(x))
        return x

    def synthesize(self, uhat):
        x = np.array(uhat, np.complex128, copy=True)
        lib().orc_synthesize(self._h, _p(x))
        return x

    def steps(self, uhat, n):
        x = np.array(uhat, np.complex128, copy=True)
        lib().orc_steps(self._h, _p(x), n)
        return x

    def l2_norm(self, uhat):
        x = np.ascontiguousarray(uhat, np.complex128)
        return lib().orc_l2_norm(self._h, _p(x))

    def energy(self, uhat):
        x = np.ascontiguousarray(uhat, np.complex128)
        return lib().orc_energy(self._h, _p(x))
