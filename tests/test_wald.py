"""Edge significance (Thm 5 / Cor. 10; Bonferroni): the oracle
pinned to the SPEC worked value (tests/golden/wald.json) and to the defining relations, and
libggm's host implementation (include/ggm.h (4); no GPU needed) against the oracle."""
import json
import os

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "wald.json")))


def test_oracle_worked_value():
    z, pr, pb = O.wald_edge(GOLD["psi"], GOLD["d_rest"], GOLD["sigma2"], 1)
    assert abs(z - GOLD["z"]) < 1e-5
    assert abs(pr - GOLD["p_raw"]) < 1e-4
    assert pb == pr


def test_oracle_threshold_is_the_critical_value():
    # at |psi| = tau the Bonferroni p-value is exactly alpha; above it smaller, below larger
    for d_rest, s2, a, m in [(50, 1.0, 0.05, 1), (60000, 1.0, 0.05, 124750), (1000, 0.5, 0.01, 10 ** 6)]:
        tau = O.wald_threshold(d_rest, s2, a, m)
        assert abs(O.wald_edge(tau, d_rest, s2, m)[2] - a) < 1e-9 * max(1.0, a)
        assert O.wald_edge(tau * 1.01, d_rest, s2, m)[2] < a < O.wald_edge(tau * 0.99, d_rest, s2, m)[2]
    # z scales as sqrt(d_rest) sigma^2: tau halves when d_rest quadruples
    assert abs(O.wald_threshold(200, 1.0, 0.05, 7) * 2 - O.wald_threshold(50, 1.0, 0.05, 7)) < 1e-12


@pytest.fixture(scope="module")
def G():
    from paper_2407_19892_b200 import build
    build.build()
    import paper_2407_19892_b200 as G
    return G


@pytest.mark.parametrize("psi,d_rest,s2,m", [(0.4, 50, 1.0, 1), (-0.02, 60000, 1.0, 124750),
                                              (0.003, 2000, 0.5, 10 ** 7), (0.0, 10, 1.0, 3)])
def test_library_edge_matches_oracle(G, psi, d_rest, s2, m):
    got = G.wald_edge(psi, d_rest, s2, m)
    want = O.wald_edge(psi, d_rest, s2, m)
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-300)


@pytest.mark.parametrize("d_rest,s2,a,m", [(50, 1.0, 0.05, 1), (60000, 1.0, 0.05, 124750),
                                           (300 * 200, 1.0, 0.05, 139650), (10, 0.25, 0.2, 45),
                                           (10 ** 6, 1.0, 1e-3, 5 * 10 ** 11)])
def test_library_threshold_matches_oracle(G, d_rest, s2, a, m):
    np.testing.assert_allclose(G.wald_threshold(d_rest, s2, a, m), O.wald_threshold(d_rest, s2, a, m),
                               rtol=1e-12)
