"""The INTEGRATION.md binding, executed: the reference's own run()
(baseline/_ref, the unmodified package; workers = 1 so segments run
in-process) with ctqw.ensemble._evolve_segment replaced by
integration/ctqw_b200_binding.py, against the same run() unpatched.
Skipped when baseline/_ref is not installed."""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ctqw_ref():
    if not os.path.isdir(os.path.join(REF, "ctqw")):
        pytest.skip("baseline/_ref (the reference package) is not installed")
    sys.path.insert(0, REF)
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    import ctqw

    assert os.path.abspath(os.path.dirname(os.path.dirname(ctqw.__file__))) == os.path.abspath(REF)
    return ctqw


def _run(ctqw, cfg, patched):
    import ctqw_b200_binding as b

    if patched:
        b.install()
    try:
        sinks = ctqw.MemorySinks()
        rep = ctqw.run(cfg, sinks)
    finally:
        b.uninstall()
    return sinks, rep


@pytest.mark.parametrize("backend,target,dt", [("taylor", "tunneling", 0.05), ("rk4", "both", 0.05),
                                               ("taylor", "both", 0.1)])
def test_binding_rows_match_reference_run(ctqw_ref, backend, target, dt):
    ctqw = ctqw_ref
    cfg = ctqw.RunConfig(space=ctqw.JointSpace(ctqw.build_lattice([24]), 2),
                         model=ctqw.CouplingModel(onsite_energy=0.1, interaction=0.5),
                         noise=ctqw.NoiseSpec(target=target, levels=(-0.1, 0.1), rate=0.0),
                         stepper=ctqw.StepperConfig(backend=backend, dt=dt, taylor_order=4),
                         realizations=6, steps=30, post_rate=10, precision="double", workers=1)
    ref, rep_ref = _run(ctqw, cfg, False)
    mine, rep = _run(ctqw, cfg, True)
    assert [(t, n, i) for t, n, i, _ in mine.rows] == [(t, n, i) for t, n, i, _ in ref.rows]
    a = np.array([v for *_, v in mine.rows])
    b = np.array([v for *_, v in ref.rows])
    np.testing.assert_allclose(a, b, rtol=1e-10, atol=1e-13)
    assert rep.norm_corrections == rep_ref.norm_corrections
    assert rep.norm_events == rep_ref.norm_events
    for x, y in zip(mine.densities, ref.densities):
        np.testing.assert_allclose(x.packed, y.packed, rtol=0, atol=1e-13)


def test_binding_falls_through_for_dynamic_noise(ctqw_ref):
    ctqw = ctqw_ref
    cfg = ctqw.RunConfig(space=ctqw.JointSpace(ctqw.build_lattice([9]), 1),
                         noise=ctqw.NoiseSpec(levels=(-0.2, 0.2), rate=1.0), stepper=ctqw.StepperConfig(dt=0.05),
                         realizations=3, steps=12, post_rate=6, precision="double", workers=1)
    ref, _ = _run(ctqw, cfg, False)
    mine, _ = _run(ctqw, cfg, True)
    assert mine.rows == ref.rows
