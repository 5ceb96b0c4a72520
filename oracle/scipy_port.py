"""TEST INFRASTRUCTURE ONLY -- the oracle's literal Strang step with its
transforms done by scipy.fft (pocketfft, multi-threaded): the strongest CPU
restatement of the reference's specified solver that this image can run.

Used as bench.py's CPU baseline and `--impl reference` arm (the reference has
no solver of its own), never by the product. Setup (points, v,
initial samples, norm table) comes from the C++ oracle (oracle.cpp); only the
per-step transforms differ, and tests/test_scipy_port.py checks the two
against each other.

  literal  : SPEC.md:336-344 strang_step on coefficients -- synthesize,
             x potH, analyze, x kin, synthesize, x potH, analyze (4 length-N
             DFTs; prime N runs pocketfft's own Bluestein);
  circulant: the same operator as one length-M cyclic convolution per step
             (M = next_fast_len(2N-1)), the half steps merged, as the GPU
             path computes it: a second, faster CPU datapoint.
"""
from __future__ import annotations

import os

import numpy as np
import scipy.fft as sfft


class ScipyPort:
    def __init__(self, orc, moduli, norm2, eps, workers: int | None = None):
        self.shape = tuple(int(m) for m in moduli)
        self.N = int(np.prod(self.shape))
        self.axes = tuple(range(len(self.shape)))
        self.v = orc.potential()
        self.norm2 = np.asarray(norm2, np.float64)
        self.eps = eps
        self.workers = workers or os.cpu_count()

    # analyze = DFT/N, synthesize = unnormalised inverse
    def analyze(self, u):
        return sfft.fftn(u.reshape(self.shape), axes=self.axes, norm="forward", workers=self.workers).reshape(-1)

    def synthesize(self, c):
        return sfft.ifftn(c.reshape(self.shape), axes=self.axes, norm="forward", workers=self.workers).reshape(-1)

    def set_dt(self, dt):
        self.dt = dt
        self.kin = np.exp(1j * (-self.eps * dt * 2.0 * np.pi ** 2 * self.norm2))
        self.potH = np.exp(1j * (-dt * self.v / (2.0 * self.eps)))
        self._circ = None

    # ---- literal
    def steps(self, uhat, n):
        u = np.array(uhat, np.complex128, copy=True)
        for _ in range(n):
            s = self.synthesize(u)
            s *= self.potH
            u = self.analyze(s)
            u *= self.kin
            s = self.synthesize(u)
            s *= self.potH
            u = self.analyze(s)
        return u

    # ---- circulant (rank-1): a <- V . conv_N(k, a), V = potH^2
    def _circ_tables(self):
        if self._circ is None:
            if len(self.shape) != 1:
                raise ValueError("circulant form is rank-1 only")
            N = self.N
            M = sfft.next_fast_len(2 * N - 1)
            k = sfft.ifft(self.kin, workers=self.workers)  # kernel of F^-1 D F (1/N folded in)
            K = np.zeros(M, np.complex128)
            K[:N] = k
            K[M - N + 1:] = k[1:]
            self._circ = (M, sfft.fft(K, workers=self.workers), self.potH * self.potH)
        return self._circ

    def circulant_steps(self, a, n):
        """n merged steps on half-step-advanced samples a = potH * s."""
        M, Kh, V = self._circ_tables()
        N = self.N
        x = np.zeros(M, np.complex128)
        a = np.array(a, np.complex128, copy=True)
        for _ in range(n):
            x[:N] = a
            x[N:] = 0
            y = sfft.ifft(sfft.fft(x, workers=self.workers) * Kh, workers=self.workers)
            a = y[:N] * V
        return a
