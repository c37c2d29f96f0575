"""The reference's release gate (``test_acceptance.py``) replayed through this
package's ``run()`` on the device: the criteria that concern the stepping
path and its observables.

Criterion 2 compares against the eigen backend, which is out of scope here
(``DESIGN.md`` §1). Criteria 8–10 time the reference's CPU worker pool.
Criterion 3's spectral check is ``test_gpu_known_answers.py``.
"""

import numpy as np
import pytest

from tests.test_gpu_parity import pkg  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def test_criterion_04_norm_drift_watched_and_fatal(pkg):
    """m=1, N=16, telegraph noise, no rescaling: the 1500-step drift stays
    under the watch tolerance; a tenfold step aborts with exit code 3."""
    p = pkg

    def cfg(dt):
        return p.RunConfig(space=p.JointSpace(p.build_lattice([16]), 1),
                           noise=p.NoiseSpec(levels=(-0.3, 0.3), rate=0.2),
                           stepper=p.StepperConfig(backend="taylor", dt=dt, taylor_order=4, tol_norm=1e-6,
                                                   tol_fail=1e-3, renormalize=False),
                           realizations=2, steps=1500, post_rate=500, master_seed=99, precision="double")

    report = p.run(cfg(0.019), p.MemorySinks(keep_densities=False))
    assert report.max_norm_deviation <= 1e-6
    with pytest.raises(p.NormFailureError) as failure:
        p.run(cfg(0.19), p.MemorySinks(keep_densities=False))
    assert failure.value.exit_code == 3


def test_criterion_05_density_structure_at_every_snapshot(pkg):
    """Order-10 series, 100 realizations, 20 snapshots of the dense rho:
    unit trace, Hermitian by storage, positive semidefinite."""
    p = pkg
    cfg = p.RunConfig(space=p.JointSpace(p.build_lattice([8]), 1),
                      noise=p.NoiseSpec(target="tunneling", levels=(-0.3, 0.3), rate=0.2),
                      stepper=p.StepperConfig(backend="taylor", dt=0.035, taylor_order=10),
                      realizations=100, steps=200, post_rate=10, master_seed=4321, precision="double")
    sinks = p.MemorySinks(dense=True)
    p.run(cfg, sinks)
    assert len(sinks.densities) == 20
    for rho in sinks.densities:
        assert abs(rho.trace() - 1.0) <= 1e-6
        dense = rho.dense()
        assert np.array_equal(dense, dense.conj().T)
        assert float(np.linalg.eigvalsh(dense).min()) >= -1e-8


def spreading(p, levels, rate, realizations, post_rate, precision):
    cfg = p.RunConfig(space=p.JointSpace(p.build_lattice([101]), 1),
                      noise=p.NoiseSpec(levels=levels, rate=rate),
                      stepper=p.StepperConfig(backend="taylor", dt=0.05),
                      realizations=realizations, steps=240, post_rate=post_rate, master_seed=2718,
                      precision=precision, observables=("position_mean_variance",))
    sinks = p.MemorySinks(keep_densities=False)
    p.run(cfg, sinks)
    variances = [(t, v) for t, name, _, v in sinks.rows if name == "position_variance"]
    wrapped = [v for _, name, _, v in sinks.rows if name == "position_wrapped"]
    return variances, wrapped


def test_criteria_06_07_spreading(pkg):
    """Noiseless spreading is ballistic (variance exponent 2 +- 0.05, no
    wrap); telegraph noise (levels +-1, rate 1, 500 realizations) slows it
    below 0.7 of the free variance."""
    variances, wrapped = spreading(pkg, (0.0,), 0.0, 1, 10, "double")
    times = np.array([t for t, _ in variances])
    sigma2 = np.array([v for _, v in variances])
    slope = np.polyfit(np.log(times), np.log(sigma2), 1)[0]
    assert 1.95 <= slope <= 2.05
    assert not any(wrapped)
    noisy, _ = spreading(pkg, (-1.0, 1.0), 1.0, 500, 240, "single")
    assert noisy[-1][1] < 0.7 * variances[-1][1]


def test_criterion_11_repeated_runs_are_identical(pkg):
    """Two runs with the same seed give identical observable rows (m=2,
    N=31, telegraph noise, 100 realizations, 300 steps, a row every 10)."""
    p = pkg
    cfg = p.RunConfig(space=p.JointSpace(p.build_lattice([31]), 2),
                      noise=p.NoiseSpec(levels=(-0.1, 0.1), rate=0.1),
                      stepper=p.StepperConfig(backend="taylor", dt=0.02),
                      realizations=100, steps=300, post_rate=10, master_seed=1234, precision="single")
    rows = []
    for _ in range(2):
        sinks = p.MemorySinks(keep_densities=False)
        p.run(cfg, sinks)
        rows.append(sinks.rows)
    assert len(rows[0]) > 0 and rows[0] == rows[1]
