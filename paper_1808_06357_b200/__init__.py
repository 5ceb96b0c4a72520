"""lattdse-b200: B200-native Strang-splitting TDSE hot path on rank-1/rank-r lattices.

Python mirror of the C ABI in include/lattdse_c.h (ctypes over the in-tree
liblattdse_b200.so). The names follow the reference's lattice-core
(/root/reference/proj/src/core/lattice.hpp:31-86) and SPEC.md's
cbc / antialias / tdse operations. There is no CPU fallback: importing this
package without the built library raises ImportError.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblattdse_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make -C paper_1808_06357_b200/csrc -j8` "
        "(or __graft_entry__.build()); the package has no CPU fallback"
    )

_lib = C.CDLL(LIB_PATH)

ERRC = [
    "invalid_argument", "non_divisible_moduli", "non_coprime_component", "rank_deficient",
    "point_count_mismatch", "overflow_risk", "radius_exhausted", "spec_mismatch",
    "non_normalizable", "config_error", "reference_too_coarse", "numerical_invariant",
    "io_error", "device_error", "unsupported", "nccl_error",
]


class LattdseError(RuntimeError):
    """Carries the reference's Errc (errors.hpp:8-22) as .code / .name."""

    def __init__(self, code: int, msg: str):
        self.code = code - 1  # Errc ordinal
        self.name = ERRC[self.code] if 0 <= self.code < len(ERRC) else "unknown"
        super().__init__(f"[{self.name}] {msg}")


_lib.lattdse_last_error.restype = C.c_char_p
_lib.lattdse_version.restype = C.c_char_p


def _ck(rc: int) -> None:
    if rc != 0:
        raise LattdseError(rc, _lib.lattdse_last_error().decode())


i64p = C.POINTER(C.c_int64)
dblp = C.POINTER(C.c_double)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


def version() -> str:
    return _lib.lattdse_version().decode()


# ------------------------------------------------------------------ lattice
class Lattice:
    """Canonical rank-r lattice (lattice.hpp:31-86)."""

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.lattdse_lattice_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @staticmethod
    def create(dim: int, rank: int, gen, moduli) -> "Lattice":
        g = _i64(gen).reshape(-1)
        n = _i64(moduli).reshape(-1)
        if g.size != dim * rank or n.size != rank:
            raise LattdseError(1, "generator must have rank columns and rank moduli")
        h = C.c_void_p()
        _ck(_lib.lattdse_lattice_create(dim, rank, _ptr(g, C.c_int64), _ptr(n, C.c_int64), C.byref(h)))
        return Lattice(h)

    @staticmethod
    def rank1(z, n: int) -> "Lattice":
        z = _i64(z).reshape(-1)
        h = C.c_void_p()
        _ck(_lib.lattdse_lattice_rank1(_ptr(z, C.c_int64), int(z.size), C.c_int64(n), C.byref(h)))
        return Lattice(h)

    @staticmethod
    def grid(moduli) -> "Lattice":
        n = _i64(moduli).reshape(-1)
        h = C.c_void_p()
        _ck(_lib.lattdse_lattice_grid(_ptr(n, C.c_int64), int(n.size), C.byref(h)))
        return Lattice(h)

    @staticmethod
    def from_json(text: str) -> "Lattice":
        h = C.c_void_p()
        _ck(_lib.lattdse_lattice_from_json(text.encode(), C.byref(h)))
        return Lattice(h)

    def _info(self):
        d, r, n, L = C.c_int(), C.c_int(), C.c_int64(), C.c_int64()
        _ck(_lib.lattdse_lattice_info(self._h, C.byref(d), C.byref(r), C.byref(n), C.byref(L)))
        return d.value, r.value, n.value, L.value

    def dim(self) -> int:
        return self._info()[0]

    def rank(self) -> int:
        return self._info()[1]

    def n_total(self) -> int:
        return self._info()[2]

    def denom(self) -> int:
        return self._info()[3]

    def generators(self):
        d, r, _, _ = self._info()
        g = np.zeros(r * d, np.int64)
        n = np.zeros(r, np.int64)
        _ck(_lib.lattdse_lattice_generators(self._h, _ptr(g, C.c_int64), _ptr(n, C.c_int64)))
        return g.reshape(r, d), n

    def moduli(self):
        return self.generators()[1]

    def hash(self) -> int:
        v = C.c_uint64()
        _ck(_lib.lattdse_lattice_hash(self._h, C.byref(v)))
        return v.value

    def to_json(self) -> str:
        need = C.c_size_t()
        _ck(_lib.lattdse_lattice_to_json(self._h, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        _ck(_lib.lattdse_lattice_to_json(self._h, buf, need.value, None))
        return buf.value.decode()

    def in_dual(self, h) -> bool:
        h = _i64(h)
        out = C.c_int()
        _ck(_lib.lattdse_lattice_in_dual(self._h, _ptr(h, C.c_int64), C.byref(out)))
        return bool(out.value)

    def residue(self, h):
        h = _i64(h)
        xi = np.zeros(self.rank(), np.int64)
        _ck(_lib.lattdse_lattice_residue(self._h, _ptr(h, C.c_int64), _ptr(xi, C.c_int64), None))
        return xi

    def flat_residue(self, h) -> int:
        h = _i64(h)
        f = C.c_int64()
        _ck(_lib.lattdse_lattice_residue(self._h, _ptr(h, C.c_int64), None, C.byref(f)))
        return f.value

    def point_numerators(self, first: int = 0, count: int | None = None) -> np.ndarray:
        d, _, n, _ = self._info()
        count = n - first if count is None else count
        out = np.zeros((count, d), np.int64)
        _ck(_lib.lattdse_lattice_point_numerators(self._h, C.c_int64(first), C.c_int64(count), _ptr(out, C.c_int64)))
        return out

    def point_coords(self) -> np.ndarray:
        return self.point_numerators() * (1.0 / self.denom())

    def point_index(self, flat_index: int) -> np.ndarray:
        out = np.zeros(self.rank(), np.int64)
        _ck(_lib.lattdse_lattice_point_index(self._h, C.c_int64(flat_index), _ptr(out, C.c_int64)))
        return out

    def __eq__(self, other) -> bool:
        if not isinstance(other, Lattice):
            return NotImplemented
        a, b = self.generators(), other.generators()
        return self._info() == other._info() and np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


# ---------------------------------------------------------------- cbc / aaset
def wce_squared(z, n: int) -> float:
    z = _i64(z)
    out = C.c_double()
    _ck(_lib.lattdse_wce_squared(_ptr(z, C.c_int64), int(z.size), C.c_int64(n), C.byref(out)))
    return out.value


def cbc_construct(n: int, d_max: int):
    """SPEC.md:128-137, prime-n extension; returns (z, criterion per component)."""
    z = np.zeros(d_max, np.int64)
    w = np.zeros(d_max, np.float64)
    _ck(_lib.lattdse_cbc_construct(C.c_int64(n), int(d_max), _ptr(z, C.c_int64), _ptr(w, C.c_double)))
    return z, w


def aaset_build(lat: Lattice, with_vectors: bool = True, cap_radius: float = -1.0):
    """SPEC.md:178-187; returns (norm2[u32], h[n,d] int16 or None, max_norm2)."""
    n = lat.n_total()
    d = lat.dim()
    norm2 = np.zeros(n, np.uint32)
    h = np.zeros((n, d), np.int16) if with_vectors else None
    mx = C.c_uint32()
    _ck(_lib.lattdse_aaset_build(lat.handle, C.c_double(cap_radius), _ptr(norm2, C.c_uint32),
                                 _ptr(h, C.c_int16) if h is not None else None, C.byref(mx)))
    return norm2, h, mx.value


def cbc_construct_device(n: int, d_max: int, device: int = 0):
    """CBC on the GPU (prime n > 64): returns (z[int64], wce[float64]) like cbc_construct."""
    z = np.zeros(d_max, np.int64)
    w = np.zeros(d_max)
    _ck(_lib.lattdse_cbc_construct_device(C.c_int64(n), d_max, device, _ptr(z, C.c_int64), _ptr(w, C.c_double)))
    return z, w


def aaset_norms_device(lat: Lattice, device: int = 0, cap_radius: float = -1.0):
    """The anti-aliasing norm table built on the GPU (rank-1); returns (norm2[u32], max_norm2)."""
    norm2 = np.zeros(lat.n_total(), np.uint32)
    mx = C.c_uint32()
    _ck(_lib.lattdse_aaset_norms_device(lat.handle, device, C.c_double(cap_radius), _ptr(norm2, C.c_uint32),
                                        C.byref(mx)))
    return norm2, mx.value


def problem_draw(seed: int, dim: int, batch: int, c_lo: float, c_hi: float, p_max: int):
    a = np.zeros(dim)
    b = np.zeros(max(dim - 1, 1))
    c = np.zeros(batch * dim)
    p = np.zeros(batch * dim, np.int32)
    _ck(_lib.lattdse_problem_draw(C.c_uint64(seed), dim, C.c_int64(batch), C.c_double(c_lo), C.c_double(c_hi), p_max, _ptr(a, C.c_double),
                                  _ptr(b, C.c_double), _ptr(c, C.c_double), _ptr(p, C.c_int)))
    return a, b[: dim - 1], c.reshape(batch, dim), p.reshape(batch, dim)


# ------------------------------------------------------------------ solver
class _Problem(C.Structure):
    _fields_ = [("eps", C.c_double), ("dim", C.c_int), ("a", dblp), ("b", dblp), ("batch", C.c_int64),
                ("sigma", C.c_double), ("c", dblp), ("p", C.POINTER(C.c_int))]


class _Opts(C.Structure):
    _fields_ = [("device", C.c_int), ("method", C.c_int), ("group", C.c_int64), ("force_M1", C.c_int64),
                ("force_M2", C.c_int64), ("force_M2a", C.c_int64)]


class _Info(C.Structure):
    _fields_ = [("n_total", C.c_int64), ("batch", C.c_int64), ("M", C.c_int64), ("M1", C.c_int64),
                ("M2", C.c_int64), ("group", C.c_int64), ("rank", C.c_int), ("method", C.c_int),
                ("bytes_per_step", C.c_double), ("bytes_per_pass_col", C.c_double),
                ("bytes_per_pass_row", C.c_double), ("launches_per_step", C.c_int), ("M2a", C.c_int64),
                ("row_chunk", C.c_int64), ("pass4", C.c_int)]


METHODS = {"circulant": 0, "bluestein": 1}
SAMPLES, COEFFICIENTS = 0, 1


class Solver:
    """Device Strang propagator over the C ABI."""

    def __init__(self, lat: Lattice, eps: float, a, b, c, p, sigma: float, *, method: str = "circulant",
                 device: int = 0, group: int = 0, norm2=None, geometry=None):
        """geometry: None (automatic), (M1, M2) or three-level (M1, M2a, M2b)."""
        self.lat = lat
        d = lat.dim()
        self._a = np.ascontiguousarray(a, np.float64)
        self._b = np.ascontiguousarray(b if d > 1 else [0.0], np.float64)
        self._c = np.ascontiguousarray(np.asarray(c, np.float64).reshape(-1, d))
        self._p = np.ascontiguousarray(np.asarray(p, np.int32).reshape(-1, d))
        self.batch = self._c.shape[0]
        self.n = lat.n_total()
        prob = _Problem(eps, d, _ptr(self._a, C.c_double), _ptr(self._b, C.c_double), self.batch, sigma,
                        _ptr(self._c, C.c_double), _ptr(self._p, C.c_int))
        g = tuple(geometry or ())
        if g and len(g) not in (2, 3):
            raise ValueError("geometry is (M1, M2) or (M1, M2a, M2b)")
        f1, f2, fa = (g[0], g[1], 0) if len(g) == 2 else ((g[0], g[1] * g[2], g[1]) if g else (0, 0, 0))
        opts = _Opts(device, METHODS[method], group, f1, f2, fa)
        h = C.c_void_p()
        if norm2 is None:
            _ck(_lib.lattdse_solver_create(lat.handle, C.byref(prob), C.byref(opts), C.byref(h)))
        else:
            nv = np.ascontiguousarray(norm2, np.uint32)
            if nv.shape != (self.n,):
                raise LattdseError(ERRC.index("spec_mismatch") + 1,
                                   f"norm table has {nv.size} entries, the lattice {self.n} points")
            _ck(_lib.lattdse_solver_create_with_norms(lat.handle, _ptr(nv, C.c_uint32), C.byref(prob),
                                                      C.byref(opts), C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.lattdse_solver_destroy(h)
            self._h = None

    def close(self):
        self.__del__()

    def set_dt(self, dt: float):
        _ck(_lib.lattdse_solver_set_dt(self._h, C.c_double(dt)))
        self.dt = float(dt)

    def set_watchdog(self, tol: float):
        """propagate raises numerical_invariant when |norm - norm(0)| > tol (0 = off)."""
        _ck(_lib.lattdse_solver_set_watchdog(self._h, C.c_double(tol)))

    def save(self, path: str, step: int = 0, time: float = 0.0, space: int = SAMPLES):
        """Snapshot every member's state (checkpoint)."""
        snapshot_write(self.lat, path, self.get_state(space), space=space, step=step, time=time,
                       dt=getattr(self, "dt", 0.0))

    def load(self, path: str) -> dict:
        """Resume from a snapshot written for the same lattice and batch; returns its metadata."""
        data, meta = snapshot_read(self.lat, path)
        if data.shape[0] != self.batch:
            raise LattdseError(10, f"snapshot holds {data.shape[0]} members, solver has {self.batch}")
        self.set_state(data, meta["space"])
        return meta

    def discretize_initial(self):
        _ck(_lib.lattdse_solver_discretize_initial(self._h))

    def set_state(self, x, space: int = SAMPLES, m0: int = 0):
        x = np.ascontiguousarray(x, np.complex128).reshape(-1, self.n)
        _ck(_lib.lattdse_solver_set_state(self._h, x.ctypes.data_as(dblp), C.c_int64(x.shape[0]), space, C.c_int64(m0)))

    def set_state_ptr(self, ptr: int, count: int, space: int = SAMPLES, m0: int = 0):
        """Host pointer variant (pinned buffers in bench.py)."""
        _ck(_lib.lattdse_solver_set_state(self._h, C.cast(ptr, dblp), C.c_int64(count), space, C.c_int64(m0)))

    def get_state(self, space: int = SAMPLES, m0: int = 0, count: int | None = None) -> np.ndarray:
        count = self.batch - m0 if count is None else count
        out = np.zeros((count, self.n), np.complex128)
        _ck(_lib.lattdse_solver_get_state(self._h, out.ctypes.data_as(dblp), C.c_int64(count), space, C.c_int64(m0)))
        return out

    def get_state_ptr(self, ptr: int, count: int, space: int = SAMPLES, m0: int = 0):
        _ck(_lib.lattdse_solver_get_state(self._h, C.cast(ptr, dblp), C.c_int64(count), space, C.c_int64(m0)))

    def step(self, nsteps: int = 1):
        _ck(_lib.lattdse_solver_step(self._h, C.c_int64(nsteps)))

    def l2_norm(self) -> np.ndarray:
        out = np.zeros(self.batch)
        _ck(_lib.lattdse_solver_l2_norm(self._h, _ptr(out, C.c_double)))
        return out

    def energy(self) -> np.ndarray:
        out = np.zeros(self.batch)
        _ck(_lib.lattdse_solver_energy(self._h, _ptr(out, C.c_double)))
        return out

    def l2_distance(self, ref, space: int = SAMPLES, member: int = 0) -> float:
        r = np.ascontiguousarray(ref, np.complex128).reshape(-1)
        out = C.c_double()
        _ck(_lib.lattdse_solver_l2_distance(self._h, r.ctypes.data_as(dblp), space, C.c_int64(member), C.byref(out)))
        return out.value

    def l2_distance_initial(self, member: int = 0) -> float:
        out = C.c_double()
        _ck(_lib.lattdse_solver_l2_distance_initial(self._h, C.c_int64(member), C.byref(out)))
        return out.value

    def propagate(self, m: int, record_every: int, member: int = 0) -> np.ndarray:
        rows = np.zeros((m // max(record_every, 1) + 2, 4))
        nr = C.c_int64()
        _ck(_lib.lattdse_solver_propagate(self._h, C.c_int64(m), C.c_int64(record_every), C.c_int64(member), _ptr(rows, C.c_double), C.byref(nr)))
        return rows[: nr.value]

    def info(self) -> dict:
        i = _Info()
        _ck(_lib.lattdse_solver_info_get(self._h, C.byref(i)))
        d = {k: getattr(i, k) for k, _ in _Info._fields_}
        d["pass_kernel"] = "fft_pass4_kernel" if d["pass4"] else "fft_pass_kernel"
        return d

    def time_steps(self, nsteps: int) -> float:
        ms = C.c_double()
        _ck(_lib.lattdse_solver_time_steps(self._h, C.c_int64(nsteps), C.byref(ms)))
        return ms.value

    def profile_passes(self, nsteps: int):
        a, b = C.c_double(), C.c_double()
        _ck(_lib.lattdse_solver_profile_passes(self._h, C.c_int64(nsteps), C.byref(a), C.byref(b)))
        return a.value, b.value

    def synchronize(self):
        _ck(_lib.lattdse_solver_synchronize(self._h))

    def flush_l2(self):
        _ck(_lib.lattdse_solver_flush_l2(self._h))

    def kernel_launches(self) -> int:
        v = C.c_int64()
        _ck(_lib.lattdse_solver_kernel_launches(self._h, C.byref(v)))
        return v.value


class DistSolver:
    """One wave function sharded over `world` ranks (include/lattdse/dist.hpp).
    rank=-1: all ranks virtual on `device` (block exchanges by device copies);
    rank>=0: one process per GPU, NCCL exchanges (nccl_id from rank 0)."""

    def __init__(self, lat: Lattice, eps: float, a, b, c, p, sigma: float, *, world: int, rank: int = -1,
                 device: int = 0, nccl_id: bytes | None = None, norm2=None):
        self.lat = lat
        d = lat.dim()
        self._a = np.ascontiguousarray(a, np.float64)
        self._b = np.ascontiguousarray(b if d > 1 else [0.0], np.float64)
        self._c = np.ascontiguousarray(np.asarray(c, np.float64).reshape(-1, d)[:1])
        self._p = np.ascontiguousarray(np.asarray(p, np.int32).reshape(-1, d)[:1])
        self.n = lat.n_total()
        prob = _Problem(eps, d, _ptr(self._a, C.c_double), _ptr(self._b, C.c_double), 1, sigma,
                        _ptr(self._c, C.c_double), _ptr(self._p, C.c_int))
        nv = None if norm2 is None else np.ascontiguousarray(norm2, np.uint32)
        idb = None if nccl_id is None else (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        h = C.c_void_p()
        _ck(_lib.lattdse_dist_create(lat.handle, _ptr(nv, C.c_uint32) if nv is not None else None, C.byref(prob),
                                     world, rank, device, idb, C.byref(h)))
        self._h = h

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _ck(_lib.lattdse_dist_nccl_unique_id(buf))
        return bytes(buf)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.lattdse_dist_destroy(h)
            self._h = None

    def set_dt(self, dt: float):
        _ck(_lib.lattdse_dist_set_dt(self._h, C.c_double(dt)))

    def discretize_initial(self):
        _ck(_lib.lattdse_dist_discretize_initial(self._h))

    def set_state(self, x):
        x = np.ascontiguousarray(x, np.complex128).reshape(-1)
        _ck(_lib.lattdse_dist_set_state(self._h, x.ctypes.data_as(dblp)))

    def get_state(self) -> np.ndarray:
        out = np.zeros(self.n, np.complex128)
        _ck(_lib.lattdse_dist_get_state(self._h, out.ctypes.data_as(dblp)))
        return out

    def step(self, nsteps: int = 1):
        _ck(_lib.lattdse_dist_step(self._h, C.c_int64(nsteps)))

    def l2_norm(self) -> float:
        v = C.c_double()
        _ck(_lib.lattdse_dist_l2_norm(self._h, C.byref(v)))
        return v.value

    def time_steps(self, nsteps: int) -> float:
        v = C.c_double()
        _ck(_lib.lattdse_dist_time_steps(self._h, C.c_int64(nsteps), C.byref(v)))
        return v.value

    def info(self) -> dict:
        M, M1, M2 = C.c_int64(), C.c_int64(), C.c_int64()
        xb = C.c_double()
        _ck(_lib.lattdse_dist_info(self._h, C.byref(M), C.byref(M1), C.byref(M2), C.byref(xb)))
        Ma, Mb = C.c_int64(), C.c_int64()
        _ck(_lib.lattdse_dist_three_level(self._h, C.byref(Ma), C.byref(Mb)))
        pk = C.c_double()
        _ck(_lib.lattdse_dist_table_peak_bytes(self._h, C.byref(pk)))
        return {"M": M.value, "M1": M1.value, "M2": M2.value, "Ma": Ma.value, "Mb": Mb.value,
                "exchange_bytes_per_rank": xb.value, "table_peak_bytes": pk.value}


def snapshot_write(lat: Lattice, path: str, data, *, space: int = SAMPLES, step: int = 0, time: float = 0.0,
                   dt: float = 0.0):
    """Raw little-endian complex128 + JSON sidecar (include/lattdse/snapshot.hpp)."""
    x = np.ascontiguousarray(data, np.complex128).reshape(-1, lat.n_total())
    _ck(_lib.lattdse_snapshot_write(lat.handle, os.fsencode(path), x.ctypes.data_as(dblp), C.c_int64(x.shape[0]),
                                    space, C.c_int64(step), C.c_double(time), C.c_double(dt)))


def snapshot_read(lat: Lattice, path: str):
    """Returns (members x N complex128 array, metadata dict) after checking the sidecar against `lat`."""
    mem, sp, st, t, dt = C.c_int64(), C.c_int(), C.c_int64(), C.c_double(), C.c_double()
    _ck(_lib.lattdse_snapshot_probe(lat.handle, os.fsencode(path), C.byref(mem), C.byref(sp), C.byref(st),
                                    C.byref(t), C.byref(dt)))
    out = np.zeros((mem.value, lat.n_total()), np.complex128)
    _ck(_lib.lattdse_snapshot_read(lat.handle, os.fsencode(path), out.ctypes.data_as(dblp), C.c_int64(out.size)))
    return out, {"members": mem.value, "space": sp.value, "step": st.value, "time": t.value, "dt": dt.value}


def exported_symbols() -> list[str]:
    """Every lattdse_* function declared in include/lattdse_c.h."""
    import re

    hdr = os.path.join(_HERE, "..", "include", "lattdse_c.h")
    with open(hdr) as f:
        txt = f.read()
    return sorted(set(re.findall(r"\b(lattdse_[a-z0-9_]+)\s*\(", txt)))
