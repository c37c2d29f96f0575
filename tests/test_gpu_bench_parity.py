"""Parity of the exact kernel specializations the BASELINE configurations and
bench.py run, against the oracle (ensemble.py:445-558 / propagators.py:167-241).

Each case uses the bench's model (t = 1, eps0 = 0, U = 0), noise target,
integrator and lattice size, asserts the compiled variant it ran
(``ctqw_step_variant``), and is sized so the persistent schedule's pieces
cross realization boundaries (more norm blocks than CTAs, not a multiple).
Tolerances: bit-exact in exact mode without renormalisations; 1e-13 absolute
once rescales happen; FMA mode within 1e-12 (the bench's arithmetic).
"""

import os

import numpy as np
import pytest

from oracle import ctqw_oracle as orc
from tests.test_gpu_parity import device_case, pkg, run_evolve, stepper  # noqa: F401

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _check(h, st, m, n, B, backend, dt, steps, variant_exact, variant_fma, expect_rescale):
    psi0 = np.tile(orc.product_state(m, n), (B, 1))
    ref, ostats = orc.evolve_segment(st, psi0.copy(), 0, steps, dt, 1.0, backend, 4)
    assert (ostats.corrections > 0) == expect_rescale
    mine, stats = run_evolve(h, psi0, B, steps, stepper(backend, 4, dt, exact=True))
    assert h.step_variant() == variant_exact
    assert stats.corrections == ostats.corrections
    assert stats.event_count == ostats.event_count
    if ostats.event_count == 0:
        np.testing.assert_array_equal(mine, ref)
    else:
        assert np.abs(mine - ref).max() <= 1e-13
    # FMA-mode RK4 runs as the Taylor-4 kernels (the same polynomial, api.cu
    # scalars_for); CTQW_RK4_STAGES=1 keeps the stage form, checked too
    forms = [(variant_fma.replace("<rk4,", "<rk4=taylor4,"), None)]
    if backend == "rk4":
        forms.append((variant_fma, "1"))
    for var, stages in forms:
        if stages:
            os.environ["CTQW_RK4_STAGES"] = stages
        try:
            fma, fstats = run_evolve(h, psi0, B, steps, stepper(backend, 4, dt, exact=False))
        finally:
            os.environ.pop("CTQW_RK4_STAGES", None)
        assert h.step_variant() == var
        assert fstats.corrections == ostats.corrections
        assert np.abs(fma - ref).max() <= 1e-12
        # per-realization squared norms agree with the oracle's to rounding (norm
        # conservation is judged against the oracle's norm)
        n2 = (np.abs(fma) ** 2).sum(axis=1)
        n2_ref = (np.abs(ref) ** 2).sum(axis=1)
        assert np.abs(n2 - n2_ref).max() <= 1e-12


BAND4_BENCH = [
    # (n, B, backend, dt, steps, target, expect_rescale)
    # configs[1] (bench secondary): 111 realizations x 8 blocks over 4 x 148 CTAs
    (256, 111, "taylor", 0.02, 2, "tunneling", False),
    (256, 111, "taylor", 0.08, 2, "tunneling", True),   # rescale every step (SC loop)
    (256, 111, "rk4", 0.02, 2, "tunneling", False),
    (256, 111, "rk4", 0.08, 2, "tunneling", True),
    # configs[3]: N=512, 19 realizations x 16 blocks over 2 x 148 CTAs
    (512, 19, "taylor", 0.02, 2, "tunneling", False),
    (512, 19, "rk4", 0.02, 2, "tunneling", False),
    (512, 19, "taylor", 0.02, 2, "both", False),
    (512, 19, "rk4", 0.08, 2, "both", True),
    # configs[2] (the bench headline): N=1024, 5 realizations x 32 blocks over 148 CTAs
    (1024, 5, "taylor", 0.02, 2, "both", False),
    (1024, 5, "taylor", 0.02, 2, "tunneling", False),
    (1024, 5, "taylor", 0.08, 2, "both", True),
    (1024, 5, "rk4", 0.02, 2, "both", False),
]


@pytest.mark.parametrize("case", BAND4_BENCH,
                         ids=[f"n{c[0]}B{c[1]}{c[2]}dt{c[3]}{c[5]}" for c in BAND4_BENCH])
def test_band4_bench_variants_match_oracle(pkg, case):
    n, B, backend, dt, steps, target, rescale = case
    h, st, _keep = device_case(2, n, B, target, onsite=0.0, U=0.0)
    site = int(target in ("onsite", "both"))
    var = "band4_kernel<{},napp=4,site={},exact={},NN={},dg=0>"
    _check(h, st, 2, n, B, backend, dt, steps, var.format(backend, site, 1, n), var.format(backend, site, 0, n),
           rescale)


PLANE3_BENCH = [
    # (B, backend, dt, steps, target, expect_rescale): configs[4]'s kernel
    (2, "taylor", 0.015, 2, "tunneling", False),
    (2, "rk4", 0.015, 2, "both", False),
    (1, "rk4", 0.06, 2, "both", True),
]


@pytest.mark.parametrize("case", PLANE3_BENCH, ids=[f"B{c[0]}{c[1]}dt{c[2]}{c[4]}" for c in PLANE3_BENCH])
def test_plane3_bench_variants_match_oracle(pkg, case):
    B, backend, dt, steps, target, rescale = case
    h, st, _keep = device_case(3, 128, B, target, onsite=0.0, U=0.0)
    site = int(target in ("onsite", "both"))
    var = "plane3_kernel<{},napp=4,site={},exact={},NN=128,dg={}>"
    dg = 2 if site else 0  # zero-diagonal form when eps0 = U = 0 and no site noise
    _check(h, st, 3, 128, B, backend, dt, steps, var.format(backend, site, 1, dg), var.format(backend, site, 0, dg),
           rescale)


def test_resident_config0_variant_matches_oracle(pkg):
    """configs[0]'s kernel (N=64, the resident path), 100 realizations."""
    n, B, dt, steps = 64, 100, 0.02, 20
    h, st, _keep = device_case(2, n, B, "tunneling", onsite=0.0, U=0.0)
    psi0 = np.tile(orc.product_state(2, n), (B, 1))
    ref, ostats = orc.evolve_segment(st, psi0.copy(), 0, steps, dt, 1.0, "taylor", 4)
    mine, _ = run_evolve(h, psi0, B, steps, stepper("taylor", 4, dt, exact=True))
    assert h.step_variant() == "resident64_kernel<taylor,order=4,site=0,exact=1,N=64>"
    np.testing.assert_array_equal(mine, ref)
    fma, _ = run_evolve(h, psi0, B, steps, stepper("taylor", 4, dt, exact=False))
    assert h.step_variant() == "resident64_kernel<taylor,order=4,site=0,exact=0,N=64>"
    assert np.abs(fma - ref).max() <= 1e-12


@pytest.mark.parametrize("exact", [True, False], ids=["exact", "fma"])
def test_run_config0_full_length_matches_reference(pkg, exact):
    """configs[0] at full length through the public run() against the rows
    the reference's own run() produced (tests/golden/config0_run.npz: N=64,
    R=100, 1500 steps, 150 snapshots incl. purity), 1e-10 relative."""
    from tests.conftest import load_golden

    p = pkg
    data, meta = load_golden("config0_run.npz")
    cfg = p.RunConfig(space=p.JointSpace(p.build_lattice([meta["n"]]), meta["m"]),
                      noise=p.NoiseSpec(target=meta["target"], levels=tuple(meta["levels"]), rate=0.0),
                      stepper=p.StepperConfig(backend=meta["backend"], dt=meta["dt"], taylor_order=meta["order"]),
                      realizations=meta["R"], steps=meta["steps"], post_rate=meta["post_rate"],
                      master_seed=meta["master_seed"], precision="double", exact=exact)
    sinks = p.MemorySinks(keep_densities=False)
    report = p.run(cfg, sinks)
    assert [(t, nm, i) for t, nm, i, _ in sinks.rows] == [tuple(r) for r in meta["rows"]]
    mine = np.array([v for *_, v in sinks.rows])
    np.testing.assert_allclose(mine, data["rows"], rtol=1e-10, atol=1e-13)
    assert report.norm_corrections == meta["corrections"]
    assert report.snapshots == 150


RESIDENT64 = [
    # (B, backend, order, dt, steps, target, onsite, U, expect_rescale): every
    # template branch of resident64_kernel (zero / uniform / coincidence
    # diagonal, site noise, Taylor orders 1-4, RK4, rescales)
    (7, "taylor", 4, 0.02, 30, "tunneling", 0.0, 0.0, False),
    (7, "taylor", 4, 0.12, 12, "tunneling", 0.0, 0.0, True),
    (5, "taylor", 4, 0.02, 20, "both", 0.2, 0.7, False),
    (5, "taylor", 3, 0.02, 20, "both", 0.2, 0.7, True),
    (5, "taylor", 2, 0.01, 20, "onsite", 0.1, 0.0, True),
    (5, "taylor", 1, 0.002, 10, "both", 0.0, 0.5, True),
    (5, "rk4", 4, 0.02, 25, "both", 0.2, 0.7, False),
    (5, "rk4", 4, 0.12, 10, "tunneling", 0.0, 0.0, True),
    (3, "taylor", 4, 0.1, 15, "both", 0.3, 1.1, True),
]


@pytest.mark.parametrize("case", RESIDENT64, ids=[f"B{c[0]}{c[1]}{c[2]}dt{c[3]}{c[5]}U{c[7]}" for c in RESIDENT64])
def test_resident64_variants_match_oracle(pkg, case):
    B, backend, order, dt, steps, target, onsite, U, rescale = case
    h, st, _keep = device_case(2, 64, B, target, onsite=onsite, U=U)
    psi0 = np.tile(orc.product_state(2, 64), (B, 1))
    ref, ostats = orc.evolve_segment(st, psi0.copy(), 0, steps, dt, 1.0, backend, order)
    assert (ostats.corrections > 0) == rescale
    site = int(target in ("onsite", "both"))
    # (exact, CTQW_RK4_STAGES, integrator label): FMA-mode RK4 runs as
    # Taylor-4 unless the stage form is pinned
    forms = [(True, None, backend), (False, None, "rk4=taylor4" if backend == "rk4" else backend)]
    if backend == "rk4":
        forms.append((False, "1", "rk4"))
    for exact, stages, label in forms:
        if stages:
            os.environ["CTQW_RK4_STAGES"] = stages
        try:
            mine, stats = run_evolve(h, psi0, B, steps, stepper(backend, order, dt, exact=exact))
        finally:
            os.environ.pop("CTQW_RK4_STAGES", None)
        assert h.step_variant() == f"resident64_kernel<{label},order={order},site={site},exact={int(exact)},N=64>"
        assert stats.corrections == ostats.corrections and stats.event_count == ostats.event_count
        if exact and ostats.event_count == 0:
            np.testing.assert_array_equal(mine, ref)
        else:
            assert np.abs(mine - ref).max() <= (1e-13 if exact else 1e-12)


def test_resident64_equals_strip_kernel(pkg, monkeypatch):
    """The 4 x 4-block kernel and the column-strip kernel (CTQW_RESIDENT_STRIP)
    give the same bits in exact mode (same operation order per amplitude)."""
    B, dt, steps = 4, 0.03, 25
    h, st, _keep = device_case(2, 64, B, "both", onsite=0.2, U=0.7)
    psi0 = np.tile(orc.product_state(2, 64), (B, 1))
    a, _ = run_evolve(h, psi0, B, steps, stepper("taylor", 4, dt, exact=True))
    monkeypatch.setenv("CTQW_RESIDENT_STRIP", "1")
    b, _ = run_evolve(h, psi0, B, steps, stepper("taylor", 4, dt, exact=True))
    assert h.step_variant().startswith("resident_kernel<")
    np.testing.assert_array_equal(a, b)
