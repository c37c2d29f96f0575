"""Known-answer tests of the device stepping, after the reference's own
propagator and run tests (``test_propagators.py:82-119``,
``test_ensemble.py:251-291``): one step against ``expm`` of the dense
Hamiltonian, the order of accuracy of Taylor-4 and RK4, their coincidence,
and a noiseless ``run()`` against exact propagation.

The dense Hamiltonian is assembled column by column from the oracle stencil
(the same operator the parity tests pin to the reference).
"""

import numpy as np
import pytest
from scipy.linalg import expm

from oracle import ctqw_oracle as orc
from tests.test_gpu_parity import device_case, pkg, run_evolve, stepper  # noqa: F401  (pkg: fixture)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def noisy_pair(hbar=1.0, seed=3):
    """Ring of 6 sites, two particles, U = 1.5, on-site and tunnelling noise
    of +-0.2 (the reference's ``noisy_pair``)."""
    return device_case(2, 6, 1, "both", seed=seed, onsite=0.0, t=1.0, U=1.5, hbar=hbar, levels=(-0.2, 0.2))


def dense(st):
    dim = st.n ** st.m
    cols = [orc.apply_stencil(st, np.eye(dim, dtype=np.complex128)[k][None])[0] for k in range(dim)]
    return np.stack(cols, axis=1)


def random_state(dim, seed):
    rng = np.random.default_rng(seed)
    psi = rng.normal(size=dim) + 1j * rng.normal(size=dim)
    return psi / np.linalg.norm(psi)


def one_step(h, psi, backend, order, dt, exact=True):
    # no renormalisation: the one-step defect itself is measured
    out, stats = run_evolve(h, psi[None], 1, 1, stepper(backend, order, dt, tol_norm=0.2, tol_fail=0.5,
                                                         renormalize=False, exact=exact))
    assert not stats.failed
    return out[0]


@pytest.mark.parametrize("exact", [True, False], ids=["exact", "fma"])
def test_high_order_taylor_matches_expm(pkg, exact):
    h, st, _keep = noisy_pair()
    psi = random_state(36, seed=6)
    out = one_step(h, psi, "taylor", 24, 0.2, exact)
    ref = expm(-1j * dense(st) * 0.2) @ psi
    assert np.abs(out - ref).max() <= 1e-13


@pytest.mark.parametrize("backend,seed", [("taylor", 7), ("rk4", 8)])
def test_fourth_order_accuracy(pkg, backend, seed):
    """Halving dt shrinks the one-step defect by about 2**5."""
    h, st, _keep = noisy_pair()
    psi = random_state(36, seed=seed)
    H = dense(st)
    errors = [np.linalg.norm(one_step(h, psi, backend, 4, dt) - expm(-1j * H * dt) @ psi) for dt in (0.2, 0.1)]
    assert 20 < errors[0] / errors[1] < 45


def test_rk4_coincides_with_taylor4(pkg):
    """Same 4th-degree polynomial in dt*H: agreement to rounding."""
    h, st, _keep = noisy_pair(hbar=1.3)
    psi = random_state(36, seed=9)
    for dt in (0.01, 0.05, 0.25):
        a = one_step(h, psi, "taylor", 4, dt)
        b = one_step(h, psi, "rk4", 4, dt)
        assert np.abs(a - b).max() <= 1e-14


def test_noiseless_run_close_to_exact(pkg):
    """run() with no disorder: the dense rho after 20 Taylor-4 steps of 0.05
    against expm(-i H t) (``test_ensemble.py:266-276``)."""
    p = pkg
    space = p.JointSpace(lattice=p.build_lattice([9]), m=1)
    cfg = p.RunConfig(space=space, noise=p.NoiseSpec(levels=(0.0,), rate=0.0), stepper=p.StepperConfig(dt=0.05),
                      realizations=1, steps=20, post_rate=20, precision="double")
    sinks = p.MemorySinks(dense=True)
    p.run(cfg, sinks)
    psi0 = p.build_initial_state(cfg.initial, space)
    st = orc.make_stencil(1, 9, 0.0, 1.0, 0.0)
    exact = expm(-1j * dense(st) * 1.0) @ psi0
    rho = sinks.densities[-1]
    np.testing.assert_allclose(rho.dense(), np.outer(exact, exact.conj()), atol=1e-5)
    assert rho.time_tag == pytest.approx(1.0)
