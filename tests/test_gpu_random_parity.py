"""Randomised parity sweep (fixed seed): lattice sizes, particle numbers,
integrators, Taylor orders, time steps and noise targets drawn at random, so
that every step-kernel family and its edge cases (odd and ragged N, N % 4 !=
0, orders > 4, on-site-only noise) meet the oracle.  Same bars as
test_gpu_parity.py: reference bits in exact mode between renormalisations,
1e-13 after them, FMA mode within 1e-12.
"""

import numpy as np
import pytest

from oracle import ctqw_oracle as orc
from tests.test_gpu_parity import assert_stats_match, device_case, pkg, run_evolve, stepper  # noqa: F401

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _cases(count=48, seed=20261017):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        m = int(rng.choice([1, 2, 2, 2, 3]))
        n = int({1: rng.integers(5, 200), 2: rng.integers(5, 140), 3: rng.integers(4, 14)}[m])
        backend = str(rng.choice(["taylor", "taylor", "rk4"]))
        order = int(rng.integers(1, 7)) if backend == "taylor" else 4
        dt = float(rng.uniform(0.01, 0.06))
        steps = int(rng.integers(3, 13))
        target = str(rng.choice(["tunneling", "onsite", "both"]))
        B = int(rng.integers(1, 6))
        out.append((m, n, B, backend, order, round(dt, 4), steps, target))
    return out


CASES = _cases()


@pytest.mark.parametrize("case", CASES, ids=[f"m{c[0]}n{c[1]}B{c[2]}{c[3]}{c[4]}{c[7]}" for c in CASES])
def test_random_case_matches_oracle(pkg, case):
    m, n, B, backend, order, dt, steps, target = case
    h, st, _keep = device_case(m, n, B, target)
    psi0 = np.tile(orc.product_state(m, n), (B, 1))
    mine, stats = run_evolve(h, psi0, B, steps, stepper(backend, order, dt))
    try:
        ref, ostats = orc.evolve_segment(st, psi0.copy(), 0, steps, dt, 1.0, backend, order)
    except orc.NormFailure as failure:
        # a low order at a large step: the same abort, same realization and step
        assert stats.failed
        assert (stats.fail_realization, stats.fail_step) == (failure.realization, failure.step)
        return
    assert not stats.failed
    assert_stats_match(stats, ostats)
    if ostats.event_count == 0:
        np.testing.assert_array_equal(mine, ref)
    else:
        assert np.abs(mine - ref).max() <= 1e-13
    fma, _ = run_evolve(h, psi0, B, steps, stepper(backend, order, dt, exact=False))
    assert np.abs(fma - ref).max() <= 1e-12
