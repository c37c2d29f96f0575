"""run() semantics from the reference's tests/test_ensemble.py, on the device:
a zero-step run snapshots the initial state (:278-288), the snapshot cadence
and row names (:290-308), and the master seed changes the output
(:400-411)."""

import numpy as np
import pytest

from tests.test_gpu_parity import pkg  # noqa: F401

pytestmark = pytest.mark.gpu


def small(p, **kw):
    base = dict(space=p.JointSpace(p.build_lattice([11]), 2), noise=p.NoiseSpec(levels=(-0.2, 0.2), rate=1.0),
                stepper=p.StepperConfig(dt=0.05), realizations=3, steps=12, post_rate=4, precision="double")
    base.update(kw)
    return p.RunConfig(**base)


@pytest.mark.parametrize("n", [11, 64, 256])  # generic, resident64 (lazy initial state), band4
def test_zero_steps_snapshots_initial_state(pkg, n):
    p = pkg
    cfg = small(p, space=p.JointSpace(p.build_lattice([n]), 2), steps=0, realizations=4,
                noise=p.NoiseSpec(rate=0.0))
    sinks = p.MemorySinks(dense=n <= 64)
    report = p.run(cfg, sinks)
    assert report.snapshots == 1
    psi0 = p.build_initial_state(cfg.initial, cfg.space)
    pops = np.array([v for _, name, _, v in sinks.rows if name == "population"])
    ref = (np.abs(psi0.reshape(n, n)) ** 2)
    np.testing.assert_allclose(pops, ref.sum(axis=0) + ref.sum(axis=1), atol=1e-14)
    assert {t for t, *_ in sinks.rows} == {0.0}
    if n <= 64:
        np.testing.assert_allclose(sinks.densities[0].diagonal().real, np.abs(psi0) ** 2, atol=1e-14)


def test_snapshot_cadence_and_rows(pkg):
    p = pkg
    cfg = small(p, steps=20, post_rate=6, realizations=2)
    sinks = p.MemorySinks()
    report = p.run(cfg, sinks)
    assert report.snapshots == 4  # steps 6, 12, 18, 20
    assert sorted({t for t, *_ in sinks.rows}) == [pytest.approx(s * 0.05) for s in (6, 12, 18, 20)]
    assert {name for _, name, _, _ in sinks.rows} == {"population", "position_mean", "position_variance",
                                                     "position_wrapped", "purity", "participation_ratio"}


def test_seed_changes_output(pkg):
    p = pkg
    a, b = p.MemorySinks(), p.MemorySinks()
    p.run(small(p, master_seed=1, steps=20, post_rate=20), a)
    p.run(small(p, master_seed=2, steps=20, post_rate=20), b)
    assert [v for *_, v in a.rows] != [v for *_, v in b.rows]
