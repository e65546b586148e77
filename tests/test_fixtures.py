"""Synthetic-input generator: the uniform generator is the reference's
generate_random_system bit for bit; the config-specific pieces (water geometry,
charge rebalancing, Maxwell-Boltzmann) have the stated properties."""
import ctypes as C

import numpy as np
import pytest

from paper_1309_1889_b200 import fixtures as fx


@pytest.mark.parametrize("n,scheme,sep,seed", [(500, 2, 1.5, 42), (300, 1, 0.0, 3), (64, 0, 2.0, 9), (2000, 2, 1.0, 11)])
def test_uniform_matches_reference_generator(ref, n, scheme, sep, seed):
    import oracle_lib
    box = np.array([40.0, 31.0, 22.0])
    p1, q1 = np.zeros((n, 3)), np.zeros(n)
    buf = C.create_string_buffer(256)
    rc = ref.lib.ref_generate_random_system(n, oracle_lib._p(box), scheme, sep, seed, oracle_lib._p(p1),
                                            oracle_lib._p(q1), buf, 256)
    assert rc == 0
    p2, q2 = fx.uniform(n, box, ["all_plus_one", "alternating", "random_neutral"][scheme], sep, seed)
    assert np.array_equal(p1, p2) and np.array_equal(q1, q2)


def test_water_geometry():
    pos, q, m = fx.water(200, [30.0, 30.0, 30.0], 2.5, 5)
    o, h1, h2 = pos[0::3], pos[1::3], pos[2::3]
    d1 = np.linalg.norm(h1 - o, axis=1)
    d2 = np.linalg.norm(h2 - o, axis=1)
    assert np.allclose(d1, 0.9572, atol=1e-12) and np.allclose(d2, 0.9572, atol=1e-12)
    cosang = np.sum((h1 - o) * (h2 - o), axis=1) / (d1 * d2)
    assert np.allclose(np.degrees(np.arccos(cosang)), 104.52, atol=1e-9)
    assert np.allclose(q[0::3], -0.834) and np.allclose(q[1::3], 0.417)
    assert abs(q.sum()) < 1e-9
    assert np.all(m[0::3] == 16.0) and np.all(m[1::3] == 1.0)
    # O-O min separation honoured
    from scipy.spatial import cKDTree
    assert cKDTree(o).query(o, k=2)[0][:, 1].min() >= 2.5


def test_rebalanced_charges_neutral():
    q = fx.rebalanced_charges(100_000, 3)
    assert q.sum() == 0.0 and set(np.unique(q)) == {-1.0, 1.0}


def test_maxwell_boltzmann_com_and_temperature():
    m = np.full(200_000, 18.0)
    v = fx.maxwell_boltzmann(m, 300.0, 7)
    assert np.abs((m[:, None] * v).sum(0)).max() < 1e-9
    kt = 0.0019872041 * 300.0 * 4.184e-4
    t_est = (m[:, None] * v ** 2).mean() / kt
    assert abs(t_est - 1.0) < 0.01


def test_config_shapes():
    w = fx.config("c1")
    assert w.n == 8192 and tuple(w.box) == (40.0, 40.0, 40.0) and (w.a, w.h, w.levels, w.dt) == (10.0, 2.5, 2, 2.0)
    assert w.q[0] == 1.0 and w.q[1] == -1.0
    w = fx.config("c2", n_override=3000)
    assert w.n == 3000 and w.levels == 6
    w = fx.config("c5", n_override=4096)
    assert w.extra["coarse"] == (8.0, 5.0, 3, 2.0, 25) and w.q.sum() == 0
