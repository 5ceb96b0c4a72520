"""The oracle-side case table (oracle/cases.py) and the scipy.fft port
(oracle/scipy_port.py): CPU tests. The case table is an independent
restatement of the configs; it must agree with the product's configs.py
(seeds, lattices, parameters) and its C0 vector must be the exhaustive
oracle CBC. The scipy port must equal the literal C++ oracle."""
import numpy as np
import pytest

import paper_1808_06357_b200 as L
from paper_1808_06357_b200 import configs
from oracle import pyoracle as po
from oracle.cases import CASES, checksum_weights, checksums, subset_indices
from oracle.scipy_port import ScipyPort


@pytest.mark.parametrize("name", ["C0", "C1", "C2", "C3", "C4r"])
def test_cases_match_product_configs(name):
    cs, cfg = CASES[name], configs.CONFIGS[name]
    assert (cs.d, cs.N, cs.eps, cs.T, cs.m, cs.sigma, cs.batch) == (cfg.d, cfg.N, cfg.eps, cfg.T, cfg.m, cfg.sigma,
                                                                    cfg.batch)
    gen, moduli = configs.lattice(cfg).generators()
    assert [list(map(int, g)) for g in gen] == cs.gen and tuple(map(int, moduli)) == cs.moduli
    a, b, c, p = configs.problem(cfg, batch=min(cfg.batch, 3))
    a2, b2, _ = cs.potential_params()
    assert np.array_equal(a, a2) and np.array_equal(b, b2)
    for m in range(c.shape[0]):
        c2, p2 = cs.member(m)
        assert np.array_equal(c[m], c2) and np.array_equal(p[m], p2)


def test_c0_vector_is_exhaustive_oracle_cbc():
    z, _ = po.cbc_exhaustive(4099, 2)
    assert [int(x) for x in z] == CASES["C0"].gen[0]


def test_checksums_are_linear_and_sensitive():
    rng = np.random.default_rng(3)
    u = rng.standard_normal(5000) + 1j * rng.standard_normal(5000)
    e = 1e-11 * (rng.standard_normal(5000) + 1j * rng.standard_normal(5000))
    s0, s1 = checksums(u), checksums(u + e)
    assert np.allclose(checksums(2 * u), 2 * s0)
    # |S_k(e)| ~ ||e||: detects an error at the 1e-11 level
    d = np.abs(s1 - s0)
    assert np.all(d > 1e-3 * np.linalg.norm(e)) and np.all(d < 10 * np.linalg.norm(e))
    w = checksum_weights(5000, 1, 100, 200)
    assert np.allclose(np.abs(w), 1.0) and np.allclose(w, checksum_weights(5000, 1)[100:200])
    idx = subset_indices(5000, 100, 7)
    assert idx[0] == 0 and idx[-1] == 4999 and np.all(np.diff(idx) > 0)


def _c0_oracle():
    cs = CASES["C0"]
    norm2, _ = po.aaset(cs.gen, cs.moduli, with_vectors=False)
    a, b, _ = cs.potential_params()
    orc = po.Oracle(cs.gen, cs.moduli, norm2, cs.eps, a, b)
    orc.set_dt(cs.dt)
    c, p = cs.member(0)
    return cs, norm2, orc, orc.initial_samples(c, p, cs.sigma)


def test_scipy_literal_equals_oracle():
    cs, norm2, orc, g = _c0_oracle()
    port = ScipyPort(orc, cs.moduli, norm2, cs.eps, workers=2)
    port.set_dt(cs.dt)
    u0 = orc.analyze(g)
    assert np.linalg.norm(port.analyze(g) - u0) <= 1e-13 * np.linalg.norm(u0)
    want = orc.steps(u0, 8)
    got = port.steps(u0, 8)
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


def test_scipy_circulant_equals_literal():
    cs, norm2, orc, g = _c0_oracle()
    port = ScipyPort(orc, cs.moduli, norm2, cs.eps, workers=2)
    port.set_dt(cs.dt)
    want = port.synthesize(port.steps(orc.analyze(g), 8))
    got = port.circulant_steps(port.potH * g, 8) / port.potH
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


def test_scipy_literal_rank2():
    lat = configs.rank2_product(16, 8, 4)
    gen, moduli = lat.generators()
    norm2, _ = po.aaset(gen, moduli, with_vectors=False)
    a, b, c, p = L.problem_draw(5, 4, 1, 0.4, 0.6, 2)
    orc = po.Oracle(gen, moduli, norm2, 0.1, a, b)
    orc.set_dt(1 / 32)
    port = ScipyPort(orc, moduli, norm2, 0.1, workers=2)
    port.set_dt(1 / 32)
    u0 = orc.analyze(orc.initial_samples(c[0], p[0], 0.1))
    want = orc.steps(u0, 4)
    assert np.linalg.norm(port.steps(u0, 4) - want) <= 1e-12 * np.linalg.norm(want)


def test_c4r_host_cbc_equals_device_catalog():
    """The C4r generating vector (d = 20, N = 16777259) recomputed by the HOST
    fast CBC (tools/c4r_host_cbc.py, 41 min on 8 cores, committed output)
    equals catalog.json's device-CBC vector bit for bit."""
    import json
    import os

    here = os.path.dirname(__file__)
    host = json.load(open(os.path.join(here, "golden", "c4r_host_cbc.json")))
    cat = json.load(open(os.path.join(here, "..", "paper_1808_06357_b200", "catalog.json")))["C4r"]
    assert host["n"] == cat["n"] == 16777259 and host["d"] == 20
    assert host["z"] == cat["z"] == CASES["C4r"].gen[0]
