"""Edge cases and error behaviour of the device path through the C ABI:
the smallest lattices (N = 2, 3, 5; d = 1), single-point-per-axis rank-2
grids, ragged ensembles (batch not a multiple of the L2 group), call-order
and argument errors mapped to the reference's Errc names, sizes beyond the
compiled transform range, and state round trips in both spaces."""
import numpy as np
import pytest

import paper_1808_06357_b200 as L
from paper_1808_06357_b200 import configs
from oracle.pyoracle import Oracle

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("n,d", [(2, 1), (3, 1), (5, 2), (7, 3), (11, 1)])
def test_tiny_lattices_vs_oracle(n, d):
    z = [1] + [int(x) for x in np.arange(2, d + 1) % n]
    z = [c if c % n else 1 for c in z]
    lat = L.Lattice.rank1(z, n)
    a, b, c, p = L.problem_draw(7 + n, d, 1, 0.4, 0.6, 1)
    norm2, _, _ = L.aaset_build(lat, with_vectors=False)
    gen, moduli = lat.generators()
    orc = Oracle(gen, moduli, norm2, 0.3, a, b)
    orc.set_dt(0.05)
    S = L.Solver(lat, 0.3, a, b, c, p, 0.2, norm2=norm2)
    S.set_dt(0.05)
    S.discretize_initial()
    u0 = orc.analyze(orc.initial_samples(c[0], p[0], 0.2))
    S.step(5)
    assert rel(S.get_state(L.COEFFICIENTS)[0], orc.steps(u0, 5)) <= 1e-12


def test_ragged_ensemble_groups():
    lat, a, b, c, p = configs.small_rank1(3, 1021, seed=8, batch=7)
    norm2, _, _ = L.aaset_build(lat, with_vectors=False)
    outs = []
    for group in (3, 7, 1):  # 3 + 3 + 1: a ragged last group
        S = L.Solver(lat, 0.1, a, b, c, p, 0.1, group=group, norm2=norm2)
        S.set_dt(1 / 64)
        S.discretize_initial()
        S.step(4)
        outs.append(S.get_state())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[1], outs[2])


def test_state_round_trips_both_spaces():
    lat, a, b, c, p = configs.small_rank1(2, 4099, seed=2, batch=2)
    S = L.Solver(lat, 0.1, a, b, c, p, 0.1)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 4099)) + 1j * rng.standard_normal((2, 4099))
    S.set_state(x, L.SAMPLES)
    assert np.array_equal(S.get_state(L.SAMPLES), x)
    S.set_state(x, L.COEFFICIENTS)
    assert rel(S.get_state(L.COEFFICIENTS), x) <= 1e-13
    S.set_state(x[1:], L.SAMPLES, m0=1)  # one member, offset
    assert np.array_equal(S.get_state(L.SAMPLES, m0=1), x[1:])


def test_call_order_and_argument_errors():
    lat, a, b, c, p = configs.small_rank1(2, 55, seed=1)
    S = L.Solver(lat, 0.1, a, b, c, p, 0.1)
    with pytest.raises(L.LattdseError) as e:
        S.step(1)  # no dt yet
    assert e.value.name == "config_error"
    for bad in (0.0, float("nan"), float("inf")):
        with pytest.raises(L.LattdseError) as e:
            S.set_dt(bad)
        assert e.value.name == "invalid_argument"
    S.set_dt(0.01)
    with pytest.raises(L.LattdseError) as e:
        S.get_state(m0=1, count=1)  # member out of range
    assert e.value.name == "invalid_argument"
    with pytest.raises(L.LattdseError) as e:
        S.l2_distance(np.zeros(55, complex), member=3)
    assert e.value.name == "invalid_argument"
    with pytest.raises(L.LattdseError) as e:  # norm table of another lattice
        L.Solver(lat, 0.1, a, b, c, p, 0.1, norm2=np.zeros(54, np.uint32))
    assert e.value.name in ("spec_mismatch", "invalid_argument")
    with pytest.raises(L.LattdseError) as e:
        L.Solver(lat, -1.0, a, b, c, p, 0.1)  # eps must be > 0
    assert e.value.name == "invalid_argument"


def test_sizes_beyond_the_compiled_range():
    # rank-2 grid whose line length has no compiled pass kernel
    lat = L.Lattice.create(2, 2, [[1, 0], [0, 1]], [11, 11])
    a, b, c, p = L.problem_draw(3, 2, 1, 0.4, 0.6, 1)
    with pytest.raises(L.LattdseError) as e:
        L.Solver(lat, 0.1, a, b, c, p, 0.1)
    assert e.value.name == "unsupported"
    # forced three-level geometry that is too small for N
    lat1, a1, b1, c1, p1 = configs.small_rank1(2, 4099, seed=4)
    with pytest.raises(L.LattdseError) as e:
        L.Solver(lat1, 0.1, a1, b1, c1, p1, 0.1, geometry=(4, 4, 4))
    assert e.value.name == "unsupported"
