"""GPU parity: libctqw (through its C ABI) against the oracle and the golden fixtures.

Tolerances: bit-exact for the noise draw (integer work) and, in ``exact``
mode, for every propagation between renormalisation events; 1e-13 absolute
on amplitudes once rescales happen (the squared norm is an einsum in the
reference); 1e-10 relative on observable rows (the north-star bar); FMA mode
within 1e-12.
"""

import json

import numpy as np
import pytest

from oracle import ctqw_oracle as orc
from tests.conftest import load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.fail("gpu test without CUDA")
    import paper_1612_00746_b200 as p
    from paper_1612_00746_b200 import native

    native.load_library()
    return p


def numpy_noise(seed, r0, count, levels, total):
    return np.stack([np.random.default_rng((seed, r)).choice(np.asarray(levels, dtype=float), size=total)
                     for r in range(r0, r0 + count)]) if total else np.zeros((count, 0))


def make_handle(m, n, onsite=0.0, t=1.0, U=0.0, hbar=1.0):
    from paper_1612_00746_b200.native import Handle

    return Handle(m, n, onsite, t, U, hbar, 0)


def device_case(m, n, B, target="both", seed=1234, onsite=0.2, t=1.0, U=0.7, hbar=1.0, levels=(-0.1, 0.1)):
    """Handle + bound device coefficients + oracle stencil for the same noise."""
    h = make_handle(m, n, onsite, t, U, hbar)
    nl = n if target in ("tunneling", "both") else 0
    ns = n if target in ("onsite", "both") else 0
    noise = numpy_noise(seed, 0, B, levels, nl + ns)
    dev = torch.device("cuda:0")
    hop = torch.empty((B, n), dtype=torch.float64, device=dev)
    site = torch.empty((B, n), dtype=torch.float64, device=dev) if ns else None
    nz = torch.as_tensor(noise, device=dev).contiguous() if nl + ns else None
    h.build_coefficients(nz, B, nl, ns, hop, site)
    h.bind(hop, site, B, n)
    st = orc.make_stencil(m, n, onsite, t, U, link=noise[:, :nl] if nl else None,
                          site=noise[:, nl:] if ns else None, batch=B)
    return h, st, (hop, site)


def to_dev(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.complex128), device="cuda:0")


def stepper(backend="taylor", order=4, dt=0.05, tol_norm=1e-6, tol_fail=1e-3, renormalize=True, exact=True):
    from paper_1612_00746_b200.native import make_stepper

    return make_stepper(backend, order, dt, tol_norm, tol_fail, renormalize, exact)


def random_states(B, dim, seed=0):
    rng = np.random.default_rng(seed)
    psi = rng.normal(size=(B, dim)) + 1j * rng.normal(size=(B, dim))
    return psi / np.linalg.norm(psi, axis=1, keepdims=True)


# ---------------------------------------------------------------------------
# noise draw (integer work: bit-exact)


def test_noise_draw_matches_golden(pkg):
    data, meta = load_golden("noise_draws.npz")
    h = make_handle(1, 16)
    for case in meta:
        total = case["n_links"] + case["n_sites"]
        out = torch.empty((1, total), dtype=torch.float64, device="cuda:0")
        h.draw_noise(case["seed"], case["r"], 1, case["levels"], total, out)
        np.testing.assert_array_equal(out.cpu().numpy()[0], data[case["key"]])


def test_noise_draw_stack_matches_numpy(pkg):
    h = make_handle(2, 64)
    for levels in ((-0.1, 0.1), (-0.3, 0.0, 0.3), (1.0, 2.0, 3.0, 4.0, 5.0)):
        out = torch.empty((300, 2048), dtype=torch.float64, device="cuda:0")
        h.draw_noise(1234, 10, 300, levels, 2048, out)
        ref = numpy_noise(1234, 10, 300, levels, 2048)
        np.testing.assert_array_equal(out.cpu().numpy(), ref)


# ---------------------------------------------------------------------------
# single steps vs the reference's own outputs (golden)


@pytest.mark.parametrize("idx", range(5))
def test_apply_and_steps_bit_exact_vs_reference(pkg, idx):
    data, meta = load_golden("stencil_steps.npz")
    c = meta[idx]
    h = make_handle(c["m"], c["n"], c["onsite"], c["tunneling"], c["interaction"], c["hbar"])
    n, b = c["n"], c["b"]
    dev = torch.device("cuda:0")
    noise = torch.as_tensor(np.concatenate([data[f"link{idx}"], data[f"site{idx}"]], axis=1),
                            device=dev).contiguous()
    hop = torch.empty((b, n), dtype=torch.float64, device=dev)
    site = torch.empty((b, n), dtype=torch.float64, device=dev)
    h.build_coefficients(noise, b, n, n, hop, site)
    h.bind(hop, site, b, n)
    psi = to_dev(data[f"psi{idx}"])
    out = torch.empty_like(psi)
    h.apply(psi, out, b, exact=True)
    np.testing.assert_array_equal(out.cpu().numpy(), data[f"apply{idx}"])
    for key, st in ((f"taylor4_{idx}", stepper("taylor", 4, c["dt"])),
                    (f"taylor7_{idx}", stepper("taylor", 7, c["dt"])),
                    (f"rk4_{idx}", stepper("rk4", 4, c["dt"]))):
        h.step(psi, out, b, st)
        np.testing.assert_array_equal(out.cpu().numpy(), data[key], err_msg=key)
    # tunnelling-only coefficients
    hop_t = torch.empty((b, n), dtype=torch.float64, device=dev)
    h.build_coefficients(torch.as_tensor(data[f"link{idx}"], device=dev).contiguous(), b, n, 0, hop_t, None)
    h.bind(hop_t, None, b, n)
    h.step(psi, out, b, stepper("taylor", 4, c["dt"]))
    np.testing.assert_array_equal(out.cpu().numpy(), data[f"taylor4t_{idx}"])


# ---------------------------------------------------------------------------
# evolve: resident (N <= 64), streaming tile (N > 64), generic (m = 1, 3)


def run_evolve(h, psi0, B, n_steps, st, first_step=0):
    psi = to_dev(psi0)
    work = torch.empty_like(psi)
    swapped = h.evolve(psi, work, B, first_step, n_steps, st)
    stats = h.segment_stats(0)
    res = (work if swapped else psi).cpu().numpy()
    return res, stats


def assert_stats_match(stats, ostats):
    assert stats.event_count == ostats.event_count
    assert stats.corrections == ostats.corrections
    # deviation = |n2 - 1|: n2 is a D-term sum, so its rounding is absolute (~sqrt(D) ulp)
    assert stats.max_deviation == pytest.approx(ostats.max_deviation, rel=0, abs=2e-14)
    mine = [(int(e.realization), int(e.step), bool(e.corrected)) for e in stats.events[: stats.n_events]]
    theirs = [(r, s, c) for _, c, r, s in ostats.events]
    assert mine == theirs


CASES = [
    # (m, n, B, backend, order, dt, steps, target)
    (2, 16, 5, "taylor", 4, 0.05, 60, "both"),      # resident, with rescales
    (2, 64, 6, "taylor", 4, 0.02, 40, "tunneling"),  # resident, no rescale
    (2, 64, 4, "rk4", 4, 0.05, 40, "both"),          # resident RK4
    (2, 33, 3, "taylor", 6, 0.05, 30, "onsite"),     # resident, order 6
    (2, 96, 3, "taylor", 4, 0.05, 30, "both"),       # tile, ragged last tile
    (2, 128, 3, "taylor", 4, 0.02, 25, "tunneling"), # tile, exact fit
    (2, 128, 2, "rk4", 4, 0.05, 25, "both"),         # tile RK4
    (2, 80, 2, "taylor", 2, 0.03, 20, "both"),       # tile, order 2
    (2, 600, 1, "taylor", 4, 0.02, 6, "both"),       # band4, runtime N
    (2, 100, 3, "rk4", 4, 0.05, 12, "both"),         # band4, runtime N, RK4
    (2, 160, 2, "taylor", 3, 0.04, 15, "onsite"),    # band4, order 3
    (2, 256, 2, "taylor", 1, 0.005, 15, "both"),     # band4, order 1
    (2, 512, 1, "rk4", 4, 0.03, 4, "tunneling"),     # band4, compile-time N, RK4
    (2, 98, 2, "taylor", 4, 0.05, 12, "both"),       # tile (N % 4 != 0)
    (2, 1100, 1, "rk4", 4, 0.02, 2, "both"),         # tile (N > 1024)
    (2, 72, 2, "taylor", 6, 0.03, 10, "both"),       # generic m=2 (order > 4)
    (1, 40, 4, "taylor", 4, 0.1, 50, "both"),        # generic m=1
    (3, 12, 3, "taylor", 4, 0.04, 30, "both"),       # generic m=3
    (3, 10, 2, "rk4", 4, 0.04, 20, "tunneling"),     # generic m=3 RK4
]


@pytest.mark.parametrize("case", CASES, ids=[f"m{c[0]}n{c[1]}{c[3]}{c[4]}" for c in CASES])
def test_evolve_matches_oracle(pkg, case):
    m, n, B, backend, order, dt, steps, target = case
    h, st, _keep = device_case(m, n, B, target)
    psi0 = np.tile(orc.product_state(m, n), (B, 1))
    mine, stats = run_evolve(h, psi0, B, steps, stepper(backend, order, dt))
    ref, ostats = orc.evolve_segment(st, psi0.copy(), 0, steps, dt, 1.0, backend, order)
    assert not stats.failed
    assert_stats_match(stats, ostats)
    if ostats.event_count == 0:
        np.testing.assert_array_equal(mine, ref)   # exact mode: reference bits
    else:
        assert np.abs(mine - ref).max() <= 1e-13


@pytest.mark.parametrize("case", [CASES[1], CASES[5], CASES[10]], ids=["resident", "tile", "generic"])
def test_fma_mode_close(pkg, case):
    m, n, B, backend, order, dt, steps, target = case
    h, st, _keep = device_case(m, n, B, target)
    psi0 = np.tile(orc.product_state(m, n), (B, 1))
    mine, _ = run_evolve(h, psi0, B, steps, stepper(backend, order, dt, exact=False))
    ref, _ = orc.evolve_segment(st, psi0.copy(), 0, steps, dt, 1.0, backend, order)
    assert np.abs(mine - ref).max() <= 1e-12


def test_segments_compose_and_repeat_bitwise(pkg):
    """Two segments == one segment; a repeat run is bit-identical."""
    for n in (48, 100):
        h, st, _keep = device_case(2, n, 3, "both")
        psi0 = np.tile(orc.product_state(2, n), (3, 1))
        one, _ = run_evolve(h, psi0, 3, 30, stepper(dt=0.05))
        a, _ = run_evolve(h, psi0, 3, 13, stepper(dt=0.05))
        b, _ = run_evolve(h, a, 3, 17, stepper(dt=0.05), first_step=13)
        np.testing.assert_array_equal(one, b)
        again, _ = run_evolve(h, psi0, 3, 30, stepper(dt=0.05))
        np.testing.assert_array_equal(one, again)


def test_norm_failure_matches_reference(pkg):
    data, _ = load_golden("segments.npz")
    fail = json.loads(str(data["failure"]))
    noise = numpy_noise(99, 0, 4, (-0.4, 0.4), 18)
    h = make_handle(2, 9, 0.0, 1.0, 0.0, 1.0)
    dev = torch.device("cuda:0")
    hop = torch.empty((4, 9), dtype=torch.float64, device=dev)
    site = torch.empty((4, 9), dtype=torch.float64, device=dev)
    h.build_coefficients(torch.as_tensor(noise, device=dev).contiguous(), 4, 9, 9, hop, site)
    h.bind(hop, site, 4, 9)
    psi0 = np.zeros((4, 81), dtype=np.complex128)
    psi0[:, 3 * 9 + 4] = 1.0
    _, stats = run_evolve(h, psi0, 4, 50, stepper("taylor", 4, 0.6, renormalize=False))
    assert stats.failed
    assert stats.fail_realization == fail["realization"]
    assert stats.fail_step == fail["step"]
    assert stats.fail_deviation == pytest.approx(fail["deviation"], rel=1e-12)


def test_tile_norm_failure(pkg):
    """Streaming path reports the earliest failing step and the worst row."""
    B, n = 3, 80
    h, st, _keep = device_case(2, n, B, "both", levels=(-0.4, 0.4))
    psi0 = np.tile(orc.product_state(2, n), (B, 1))
    _, stats = run_evolve(h, psi0, B, 40, stepper(dt=0.6, renormalize=False))
    with pytest.raises(orc.NormFailure) as info:
        orc.evolve_segment(st, psi0.copy(), 0, 40, 0.6, renormalize=False)
    assert stats.failed
    assert stats.fail_step == info.value.step
    assert stats.fail_realization == info.value.realization


def test_check_norm_stack_semantics(pkg):
    p = pkg
    rng = np.random.default_rng(14)
    stack = rng.normal(size=(6, 32)) + 1j * rng.normal(size=(6, 32))
    stack /= np.linalg.norm(stack, axis=1, keepdims=True)
    stack[1] *= 1.0 + 2e-4
    stack[4] *= 1.0 - 3e-4
    ref = stack.copy()
    cfg = p.StepperConfig(tol_norm=1e-6, tol_fail=1e-1)
    dev, corr = p.check_norm_stack(stack, cfg)
    odev, ocorr = orc.check_norm_stack(ref, 1e-6, 1e-1)
    assert corr.tolist() == ocorr.tolist() == [False, True, False, False, True, False]
    np.testing.assert_allclose(dev, odev, rtol=1e-12, atol=1e-15)
    assert np.abs(stack - ref).max() <= 1e-15
    stack[2] *= 2.0
    with pytest.raises(p.NormFailureError) as info:
        p.check_norm_stack(stack, cfg)
    assert info.value.realization == 2


# ---------------------------------------------------------------------------
# observables and run()


def _initial(c):
    if c["initial"] == "antisymmetrized_pair":
        n = c["n"]
        x = (n - 2) // 2
        psi = np.zeros(n * n, dtype=np.complex128)
        psi[x * n + x + 1] = 1 / np.sqrt(2.0)
        psi[(x + 1) * n + x] = -1 / np.sqrt(2.0)
        return psi
    return orc.product_state(c["m"], c["n"])


@pytest.mark.parametrize("idx", range(5))
def test_run_rows_match_reference(pkg, idx):
    p = pkg
    data, meta = load_golden("run_rows.npz")
    c = meta[idx]
    cfg = p.RunConfig(
        space=p.JointSpace(p.build_lattice([c["n"]]), c["m"]),
        model=p.CouplingModel(onsite_energy=c["onsite"], tunneling=c["tunneling"], interaction=c["interaction"]),
        noise=p.NoiseSpec(target=c["target"], levels=(-0.1, 0.1), rate=0.0),
        stepper=p.StepperConfig(backend=c["backend"], dt=c["dt"]),
        initial=p.InitialStateSpec(kind=c["initial"]),
        realizations=c["R"], steps=c["steps"], post_rate=c["post_rate"], master_seed=1234,
        precision="double", observables=c["observables"],
    )
    sinks = p.MemorySinks()
    report = p.run(cfg, sinks)
    assert [(t, n, i) for t, n, i, _ in sinks.rows] == [tuple(r) for r in c["rows"]]
    mine = np.array([v for *_, v in sinks.rows])
    np.testing.assert_allclose(mine, data[f"rows{idx}"], rtol=1e-10, atol=1e-13)
    assert report.norm_corrections == c["corrections"]
    assert report.norm_events == c["norm_events"]
    assert report.snapshots == len(cfg.schedule)


@pytest.mark.parametrize("n,R,backend", [(64, 20, "taylor"), (100, 6, "rk4"), (20, 5, "taylor")])
def test_run_matches_oracle_rows(pkg, n, R, backend):
    p = pkg
    obs = ("populations", "position_mean_variance", "purity", "participation_ratio", "joint_distribution")
    cfg = p.RunConfig(space=p.JointSpace(p.build_lattice([n]), 2),
                      model=p.CouplingModel(onsite_energy=0.1, interaction=0.3),
                      noise=p.NoiseSpec(target="both", rate=0.0),
                      stepper=p.StepperConfig(backend=backend, dt=0.04),
                      realizations=R, steps=30, post_rate=10, precision="double", observables=obs)
    sinks = p.MemorySinks()
    p.run(cfg, sinks)
    noise = numpy_noise(1234, 0, R, (-0.1, 0.1), 2 * n)
    st = orc.make_stencil(2, n, 0.1, 1.0, 0.3, link=noise[:, :n], site=noise[:, n:], batch=R)
    out, _, _ = orc.run_rows(st, orc.product_state(2, n), R, 30, 10, 0.04, backend=backend, observables=obs)
    ref = [(t, name, i, v) for t, rr in out for name, i, v in rr]
    assert [r[:3] for r in sinks.rows] == [r[:3] for r in ref]
    np.testing.assert_allclose([r[3] for r in sinks.rows], [r[3] for r in ref], rtol=1e-10, atol=1e-14)


def test_run_norm_failure_names_culprit(pkg):
    p = pkg
    cfg = p.RunConfig(space=p.JointSpace(p.build_lattice([9]), 1), noise=p.NoiseSpec(levels=(0.0,), rate=0.0),
                      stepper=p.StepperConfig(dt=2.5, renormalize=False), realizations=3, steps=10,
                      post_rate=10, precision="double")
    sinks = p.MemorySinks()
    with pytest.raises(p.NormFailureError) as info:
        p.run(cfg, sinks)
    assert info.value.realization is not None and info.value.step is not None
    assert "reduce the time step" in str(info.value)
    assert any(m.startswith("aborted") for m in sinks.messages)


# ---------------------------------------------------------------------------
# size-independent properties at the BASELINE sizes


def test_taylor_rk4_agree_at_n256(pkg):
    B, n = 4, 256
    h, _, _keep = device_case(2, n, B, "tunneling")
    psi0 = np.tile(orc.product_state(2, n), (B, 1))
    a, sa = run_evolve(h, psi0, B, 50, stepper("taylor", 4, 0.02))
    b, sb = run_evolve(h, psi0, B, 50, stepper("rk4", 4, 0.02))
    assert np.abs(a - b).max() <= 1e-13
    norms = (np.abs(a) ** 2).sum(axis=1)
    assert np.all(np.abs(norms - 1.0) < 1e-7)
    assert sa.event_count == 0 and sb.event_count == 0


def test_antisymmetric_exclusion_n512(pkg):
    """Link noise is exchange symmetric: a fermionic pair never doubly occupies."""
    B, n = 2, 512
    h, _, _keep = device_case(2, n, B, "tunneling")
    x = (n - 2) // 2
    psi0 = np.zeros((B, n * n), dtype=np.complex128)
    psi0[:, x * n + x + 1] = 1 / np.sqrt(2.0)
    psi0[:, (x + 1) * n + x] = -1 / np.sqrt(2.0)
    out, _ = run_evolve(h, psi0, B, 20, stepper(dt=0.02))
    diag = out.reshape(B, n, n)[:, np.arange(n), np.arange(n)]
    assert np.abs(diag).max() < 1e-12
    # exchange antisymmetry holds realization by realization
    grid = out.reshape(B, n, n)
    assert np.abs(grid + grid.transpose(0, 2, 1)).max() < 1e-12


def test_realization_independence_of_batching(pkg):
    """A realization's result does not depend on which batch it ran in."""
    B, n = 6, 128
    h, _, _keep = device_case(2, n, B, "both")
    psi0 = np.tile(orc.product_state(2, n), (B, 1))
    full, _ = run_evolve(h, psi0, B, 12, stepper(dt=0.03))
    hop, site = _keep
    h.bind(hop[2:5], site[2:5], 3, n)
    part, _ = run_evolve(h, psi0[2:5], 3, 12, stepper(dt=0.03))
    np.testing.assert_array_equal(full[2:5], part)


# ---------------------------------------------------------------------------
# every streaming kernel family on the same cases (CTQW_STREAM pins one)

FAMILY_CASES = [CASES[4], CASES[6], CASES[8], CASES[10], CASES[11], CASES[12]]


@pytest.mark.parametrize("family", ["band4", "tile"])
@pytest.mark.parametrize("case", FAMILY_CASES, ids=[f"n{c[1]}{c[3]}{c[4]}" for c in FAMILY_CASES])
def test_stream_families_match_oracle(pkg, monkeypatch, family, case):
    m, n, B, backend, order, dt, steps, target = case
    monkeypatch.setenv("CTQW_STREAM", family)
    h, st, _keep = device_case(m, n, B, target)
    psi0 = np.tile(orc.product_state(m, n), (B, 1))
    mine, stats = run_evolve(h, psi0, B, steps, stepper(backend, order, dt))
    ref, ostats = orc.evolve_segment(st, psi0.copy(), 0, steps, dt, 1.0, backend, order)
    assert_stats_match(stats, ostats)
    if ostats.event_count == 0:
        np.testing.assert_array_equal(mine, ref)
    else:
        assert np.abs(mine - ref).max() <= 1e-13


BAND4_CASES = [
    # (n, B, backend, order, dt, steps, target)
    (1024, 1, "taylor", 4, 0.02, 3, "both"),   # 256-thread full row, compile-time N
    (20, 4, "taylor", 4, 0.05, 20, "both"),    # runtime N, one norm block per row ring
    (36, 3, "rk4", 4, 0.05, 15, "onsite"),     # ring rows padded (36 % 8 != 0)
    (96, 300, "taylor", 4, 0.03, 4, "both"),   # persistent pieces cross realizations
    (256, 40, "rk4", 4, 0.02, 3, "tunneling"), # compile-time N, RK4
    (64, 5, "taylor", 3, 0.04, 6, "both"),     # order 3
    (128, 3, "taylor", 2, 0.03, 8, "both"),    # order 2
    (48, 3, "taylor", 1, 0.005, 8, "both"),    # order 1
]


@pytest.mark.parametrize("case", BAND4_CASES, ids=[f"n{c[0]}B{c[1]}{c[2]}{c[3]}" for c in BAND4_CASES])
def test_band4_matches_oracle(pkg, monkeypatch, case):
    n, B, backend, order, dt, steps, target = case
    monkeypatch.setenv("CTQW_STREAM", "band4")
    h, st, _keep = device_case(2, n, B, target)
    psi0 = np.tile(orc.product_state(2, n), (B, 1))
    mine, stats = run_evolve(h, psi0, B, steps, stepper(backend, order, dt))
    assert h.step_kernel() == "band4_kernel"
    ref, ostats = orc.evolve_segment(st, psi0.copy(), 0, steps, dt, 1.0, backend, order)
    assert_stats_match(stats, ostats)
    if ostats.event_count == 0:
        np.testing.assert_array_equal(mine, ref)
    else:
        assert np.abs(mine - ref).max() <= 1e-13
    # FMA mode stays within the north-star tolerance
    fma, _ = run_evolve(h, psi0, B, steps, stepper(backend, order, dt, exact=False))
    assert np.abs(fma - ref).max() <= 1e-12


def test_band4_norm_partials_independent_of_batch(pkg, monkeypatch):
    """Row-block norm partials: a realization's bits do not depend on how the
    persistent schedule cut the batch (here 1 vs 500 realizations)."""
    monkeypatch.setenv("CTQW_STREAM", "band4")
    B, n = 500, 96
    h, _, _keep = device_case(2, n, B, "both")
    psi0 = np.tile(orc.product_state(2, n), (B, 1))
    full, sf = run_evolve(h, psi0, B, 30, stepper(dt=0.05))
    assert sf.corrections > 0  # renormalisation exercised
    hop, site = _keep
    h.bind(hop[137:138], site[137:138], 1, n)
    one, _ = run_evolve(h, psi0[137:138], 1, 30, stepper(dt=0.05))
    np.testing.assert_array_equal(full[137:138], one)


PLANE3_CASES = [
    # (B, backend, dt, steps, target)
    (2, "taylor", 0.015, 3, "both"),     # pieces split realizations across clusters
    (1, "rk4", 0.015, 2, "tunneling"),
    (2, "taylor", 0.06, 3, "both"),      # renormalises every step (rescaled ring reads)
]


@pytest.mark.parametrize("case", PLANE3_CASES, ids=[f"B{c[0]}{c[1]}dt{c[2]}" for c in PLANE3_CASES])
def test_plane3_m3_n128_matches_oracle(pkg, case):
    """m = 3, N = 128 (configs[4]): the 16-CTA cluster kernel against the oracle."""
    B, backend, dt, steps, target = case
    n = 128
    h, st, _keep = device_case(3, n, B, target)
    psi0 = np.tile(orc.product_state(3, n), (B, 1))
    mine, stats = run_evolve(h, psi0, B, steps, stepper(backend, 4, dt))
    assert h.step_kernel() == "plane3_kernel"
    ref, ostats = orc.evolve_segment(st, psi0.copy(), 0, steps, dt, 1.0, backend, 4)
    assert_stats_match(stats, ostats)
    if ostats.event_count == 0:
        np.testing.assert_array_equal(mine, ref)
    else:
        assert np.abs(mine - ref).max() <= 1e-13
    fma, _ = run_evolve(h, psi0, B, steps, stepper(backend, 4, dt, exact=False))
    assert np.abs(fma - ref).max() <= 1e-12


@pytest.mark.parametrize("m,n,B,family", [(3, 128, 2, "plane3"), (2, 256, 300, "band4"), (2, 1024, 6, "band4")])
def test_streaming_kernels_bitwise_repeatable(pkg, monkeypatch, m, n, B, family):
    """Repeat runs with a renormalisation every step are bit-identical (catches
    ordering races in the ring / exchange / norm-partial paths)."""
    monkeypatch.setenv("CTQW_STREAM", family)
    h, _, _keep = device_case(m, n, B, "both")
    psi0 = np.tile(orc.product_state(m, n), (B, 1))
    dt = 0.06 if m == 3 else 0.08
    for exact in (True, False):
        first, s0 = run_evolve(h, psi0, B, 3, stepper("taylor", 4, dt, exact=exact))
        assert s0.corrections > 0
        for _ in range(3):
            again, _ = run_evolve(h, psi0, B, 3, stepper("taylor", 4, dt, exact=exact))
            np.testing.assert_array_equal(first, again)


# ---------------------------------------------------------------------------
# dynamic telegraph noise (rate > 0): device process vs the reference


@pytest.mark.parametrize("ti", range(2))
def test_telegraph_device_process_matches_reference(pkg, ti):
    """Device NoiseProcess (init + advance inside ctqw_evolve) == the
    reference's init_process/advance: values, times, switch counts exact;
    switch times exact up to the rare exp/log1p slow paths (<= 2 ulp)."""
    data, meta = load_golden("telegraph.npz")
    c = meta["trajectories"][ti]
    n, B = c["n"], c["count"]
    h = make_handle(1, n)
    dev = torch.device("cuda:0")
    h.telegraph_init(c["seed"], c["r0"], B, c["levels"], c["n_links"], c["n_sites"], c["rate"])
    hop = torch.empty((B, n), dtype=torch.float64, device=dev)
    site = torch.empty((B, n), dtype=torch.float64, device=dev) if c["n_sites"] else None
    h.build_coefficients_from_ptr(h.telegraph_values_ptr(), B, c["n_links"], c["n_sites"], hop, site)
    h.bind(hop, site, B, n)
    h.telegraph_enable(True)
    total = c["n_links"] + c["n_sites"]
    psi = to_dev(np.tile(orc.product_state(1, n), (B, 1)))
    work = torch.empty_like(psi)
    done = 0
    for k in c["checkpoints"]:
        if k > done:
            if h.evolve(psi, work, B, done, k - done, stepper(dt=c["dt"], tol_fail=0.5)):
                psi, work = work, psi
        done = k
        vals = torch.empty((B, total), dtype=torch.float64, device=dev)
        nxt = torch.empty_like(vals)
        times, sw = h.telegraph_read(B, vals, nxt)
        np.testing.assert_array_equal(vals.cpu().numpy(), data[f"traj{ti}_values_{k}"])
        np.testing.assert_array_equal(np.array(times), data[f"traj{ti}_time_{k}"])
        np.testing.assert_array_equal(np.array(sw), data[f"traj{ti}_switches_{k}"])
        ref = data[f"traj{ti}_next_{k}"]
        mine = nxt.cpu().numpy()
        assert np.all(np.abs(mine - ref) <= 2 * np.spacing(np.abs(ref)))
        # the couplings are a fresh assembly of the current values (hamiltonian.py:131-141)
        if c["n_links"]:
            np.testing.assert_array_equal(hop.cpu().numpy(), 1.0 + data[f"traj{ti}_values_{k}"][:, : c["n_links"]])


@pytest.mark.parametrize("idx", range(2))
def test_run_dynamic_noise_matches_reference(pkg, idx):
    p = pkg
    data, meta = load_golden("telegraph.npz")
    c = meta["runs"][idx]
    cfg = p.RunConfig(
        space=p.JointSpace(p.build_lattice([c["n"]]), c["m"]),
        model=p.CouplingModel(onsite_energy=c["onsite"], tunneling=c["tunneling"], interaction=c["interaction"]),
        noise=p.NoiseSpec(target=c["target"], levels=(-0.1, 0.1), rate=c["rate"]),
        stepper=p.StepperConfig(backend=c["backend"], dt=c["dt"]),
        realizations=c["R"], steps=c["steps"], post_rate=c["post_rate"], master_seed=1234, precision="double",
    )
    sinks = p.MemorySinks()
    report = p.run(cfg, sinks)
    assert [(t, n, i) for t, n, i, _ in sinks.rows] == [tuple(r) for r in c["rows"]]
    np.testing.assert_allclose([v for *_, v in sinks.rows], data[f"run{idx}_rows"], rtol=1e-10, atol=1e-13)
    assert report.switch_count == c["switch_count"]
    assert report.norm_corrections == c["corrections"]


DYN_CASES = [
    # (m, n, B, backend, dt, steps, target, family)
    (2, 40, 3, "taylor", 0.05, 12, "both", None),        # resident, one step per launch
    (2, 96, 4, "taylor", 0.04, 8, "both", "band4"),
    (2, 256, 2, "rk4", 0.03, 5, "tunneling", "band4"),
    (2, 100, 2, "taylor", 0.04, 6, "onsite", "tile"),
    (2, 1000, 1, "taylor", 0.03, 3, "both", None),      # band4, large telegraph total (2000 elements)
    (3, 12, 2, "taylor", 0.04, 6, "both", None),         # generic
    (3, 128, 1, "taylor", 0.03, 3, "both", None),        # plane3
]


@pytest.mark.parametrize("case", DYN_CASES, ids=[f"m{c[0]}n{c[1]}{c[3]}{c[7] or 'auto'}" for c in DYN_CASES])
def test_dynamic_noise_every_kernel_matches_oracle(pkg, monkeypatch, case):
    """Couplings rewritten after every step, on every step-kernel family."""
    from oracle.noise_oracle import TelegraphOracle

    m, n, B, backend, dt, steps, target, family = case
    if family:
        monkeypatch.setenv("CTQW_STREAM", family)
    rate, levels, seed = 3.0, (-0.1, 0.1), 77
    nl = n if target in ("tunneling", "both") else 0
    ns = n if target in ("onsite", "both") else 0
    h = make_handle(m, n, 0.2, 1.0, 0.7, 1.0)
    dev = torch.device("cuda:0")
    h.telegraph_init(seed, 0, B, levels, nl, ns, rate)
    hop = torch.empty((B, n), dtype=torch.float64, device=dev)
    site = torch.empty((B, n), dtype=torch.float64, device=dev) if ns else None
    h.build_coefficients_from_ptr(h.telegraph_values_ptr(), B, nl, ns, hop, site)
    h.bind(hop, site, B, n)
    h.telegraph_enable(True)
    psi0 = np.tile(orc.product_state(m, n), (B, 1))
    mine, stats = run_evolve(h, psi0, B, steps, stepper(backend, 4, dt))
    tg = TelegraphOracle(seed, 0, B, levels, nl, ns, rate)
    st = orc.make_stencil(m, n, 0.2, 1.0, 0.7, link=tg.link_values() if nl else None,
                          site=tg.site_values().copy() if ns else None, batch=B)
    ref, ostats = orc.evolve_segment(st, psi0.copy(), 0, steps, dt, 1.0, backend, 4, noise=tg, tunneling=1.0)
    assert int(tg.switches.sum()) > 0
    assert_stats_match(stats, ostats)
    if ostats.event_count == 0:
        np.testing.assert_array_equal(mine, ref)
    else:
        assert np.abs(mine - ref).max() <= 1e-13


def test_init_process_advance_api_matches_reference(pkg):
    """The reference-facing per-realization API (init_process / advance)."""
    p = pkg
    data, meta = load_golden("telegraph.npz")
    c = meta["trajectories"][0]
    spec = p.NoiseSpec(target=c["target"], levels=c["levels"], rate=c["rate"])
    lat = p.build_lattice([c["n"]])
    procs = [p.init_process(spec, lat, seed=(c["seed"], r)) for r in range(c["r0"], c["r0"] + c["count"])]
    done, switched = 0, 0
    for k in c["checkpoints"]:
        for _ in range(k - done):
            for pr in procs:
                d = p.advance(pr, c["dt"])
                switched += d.switches
        done = k
        np.testing.assert_array_equal(np.stack([pr.values for pr in procs]), data[f"traj0_values_{k}"])
        np.testing.assert_array_equal([pr.switch_count for pr in procs], data[f"traj0_switches_{k}"])
    assert switched == int(data[f"traj0_switches_{c['checkpoints'][-1]}"].sum())


# ---------------------------------------------------------------------------
# dense <rho> (density.py:57-98)


def test_accumulate_density_matches_reference(pkg):
    p = pkg
    data, _ = load_golden("density.npz")
    rho = p.accumulate_density(data["stack"], time_tag=0.25)
    assert rho.dim == 30 and rho.sample_count == 7 and rho.time_tag == 0.25
    np.testing.assert_allclose(rho.packed, data["packed"], rtol=0, atol=1e-15)
    assert rho.trace() == pytest.approx(1.0, abs=1e-14)
    dense = rho.dense()
    np.testing.assert_allclose(dense, dense.conj().T)


def test_run_dense_snapshots_match_reference(pkg):
    """run() with MemorySinks(dense=True): the packed <rho> snapshots of the
    reference's run (dynamic noise, 3 collection points)."""
    p = pkg
    data, meta = load_golden("density.npz")
    cfg = p.RunConfig(space=p.JointSpace(p.build_lattice([meta["n"]]), meta["m"]),
                      model=p.CouplingModel(onsite_energy=0.1, tunneling=1.0, interaction=0.5),
                      noise=p.NoiseSpec(target="both", levels=(-0.1, 0.1), rate=meta["rate"]),
                      stepper=p.StepperConfig(backend="taylor", dt=meta["dt"]), realizations=meta["R"],
                      steps=meta["steps"], post_rate=meta["post_rate"], master_seed=1234, precision="double")
    sinks = p.MemorySinks(dense=True)
    p.run(cfg, sinks)
    assert [(d.time_tag, d.sample_count) for d in sinks.densities] == [tuple(x) for x in meta["snapshots"]]
    for i, d in enumerate(sinks.densities):
        np.testing.assert_allclose(d.packed, data[f"snap{i}"], rtol=0, atol=1e-13)
        assert d.purity == pytest.approx(float(2 * np.sum(np.abs(data[f"snap{i}"]) ** 2)
                                               - np.sum(np.abs(np.diagonal(d.dense())) ** 2)), rel=1e-12)


@pytest.mark.parametrize("dim,R", [(1, 1), (1, 5), (63, 17), (64, 16), (65, 33), (200, 1), (300, 100)])
def test_packed_gram_kernel_matches_numpy(pkg, dim, R):
    """ctqw_packed_gram (the triangle-only kernel) against the reference's
    formula gram = stack.T @ stack.conj(); packed = gram[tril] * (1/R)
    (density.py:91-95), on ragged sizes (tile edges, a single realization,
    R not a multiple of the staging depth)."""
    from paper_1612_00746_b200 import density, native

    rng = np.random.default_rng(dim * 1000 + R)
    stack = rng.standard_normal((R, dim)) + 1j * rng.standard_normal((R, dim))
    dev = torch.as_tensor(stack, device="cuda:0")
    got = density.packed_density_device(dev, R).cpu().numpy()
    gram = stack.T @ stack.conj()
    rows, cols = np.tril_indices(dim)
    ref = gram[rows, cols] * (1.0 / R)
    scale = np.abs(ref).max()
    assert np.abs(got - ref).max() <= 1e-14 * scale * max(1, R / 10)
    raw = torch.empty(dim * (dim + 1) // 2, dtype=torch.complex128, device="cuda:0")
    native.packed_gram(dev, R, raw, 1.0)
    assert np.abs(raw.cpu().numpy() - gram[rows, cols]).max() <= 1e-14 * R * scale * max(1, R / 10)


def test_packed_gram_rejects_empty_stack(pkg):
    from paper_1612_00746_b200 import native

    dev = torch.zeros((1, 8), dtype=torch.complex128, device="cuda:0")
    out = torch.empty(36, dtype=torch.complex128, device="cuda:0")
    with pytest.raises(pkg.ConfigurationError):
        native.packed_gram(dev, 0, out, 1.0)


@pytest.mark.parametrize("count,npoints", [(1, 1), (12, 3), (37, 5), (100, 10), (124, 2), (125, 2), (150, 2)])
def test_overlap_sumsq_points_matches_per_point_and_numpy(pkg, count, npoints):
    """ctqw_overlap_sumsq_points (every point of a schedule group in one
    launch set) gives each point the same bits as a separate
    ctqw_overlap_sumsq call, and sum |<a_i|a_j>|^2 to 1e-13 relative
    (observables.py:86-91 via the Gram of the states)."""
    n = 64
    h = make_handle(2, n)
    dim = n * n
    rng = np.random.default_rng(count * 100 + npoints)
    snap = rng.standard_normal((npoints, count, dim)) + 1j * rng.standard_normal((npoints, count, dim))
    snap /= np.linalg.norm(snap, axis=2, keepdims=True)
    dev = torch.as_tensor(snap, device="cuda:0").contiguous()
    got = torch.empty(npoints, dtype=torch.float64, device="cuda:0")
    h.overlap_sumsq_points(dev, count, npoints, count * dim, got)
    one = torch.empty(npoints, dtype=torch.float64, device="cuda:0")
    for k in range(npoints):
        h.overlap_sumsq(dev[k], count, dev[k], count, one[k:k + 1])
    assert got.cpu().numpy().tobytes() == one.cpu().numpy().tobytes()
    for k in range(npoints):
        g = snap[k].conj() @ snap[k].T
        ref = float(np.sum(np.abs(g) ** 2))
        assert abs(float(got[k]) - ref) <= 1e-13 * ref


def test_overlap_sumsq_points_rejects_bad_arguments(pkg):
    h = make_handle(2, 8)
    dev = torch.zeros((2, 3, 64), dtype=torch.complex128, device="cuda:0")
    out = torch.empty(2, dtype=torch.float64, device="cuda:0")
    with pytest.raises(pkg.ConfigurationError):
        h.overlap_sumsq_points(dev, 3, 0, 3 * 64, out)
    with pytest.raises(pkg.ConfigurationError):
        h.overlap_sumsq_points(dev, 3, 2, 3 * 64 - 1, out)
    with pytest.raises(pkg.ConfigurationError):
        h.overlap_sumsq_points(dev, 0, 2, 3 * 64, out)


# ---------------------------------------------------------------------------
# general lattices (q > 1, k_half > 1, open boundaries): generic kernels


@pytest.mark.parametrize("idx", range(7))
def test_lattice_steps_bit_exact_vs_reference(pkg, idx):
    p = pkg
    data, meta = load_golden("lattices.npz")
    c = meta["steps"][idx]
    lat = p.build_lattice(c["dims"], k_half=c["k_half"], boundary=c["boundary"])
    topo = p.build_topology(p.JointSpace(lat, c["m"]))
    model = p.CouplingModel(onsite_energy=c["onsite"], tunneling=c["tunneling"], interaction=c["interaction"],
                            hbar=c["hbar"])
    values = p.assemble_values(topo, model, link_values=data[f"link{idx}"], site_values=data[f"site{idx}"])
    psi = data[f"psi{idx}"]
    np.testing.assert_array_equal(p.apply_values(topo, values, psi), data[f"apply{idx}"])
    np.testing.assert_array_equal(p.step_taylor_values(topo, values, psi, c["dt"], hbar=c["hbar"], order=4),
                                  data[f"taylor4_{idx}"])
    np.testing.assert_array_equal(p.step_rk4_values(topo, values, psi, c["dt"], hbar=c["hbar"]), data[f"rk4_{idx}"])


@pytest.mark.parametrize("idx", range(3))
def test_lattice_run_rows_match_reference(pkg, idx):
    p = pkg
    data, meta = load_golden("lattices.npz")
    c = meta["runs"][idx]
    lat = p.build_lattice(c["dims"], k_half=c["k_half"], boundary=c["boundary"])
    cfg = p.RunConfig(space=p.JointSpace(lat, c["m"]),
                      model=p.CouplingModel(onsite_energy=0.1, tunneling=1.0, interaction=0.5),
                      noise=p.NoiseSpec(target=c["target"], levels=(-0.1, 0.1), rate=c["rate"]),
                      stepper=p.StepperConfig(backend="taylor", dt=0.05), realizations=c["R"], steps=c["steps"],
                      post_rate=c["post_rate"], master_seed=1234, precision="double")
    sinks = p.MemorySinks()
    report = p.run(cfg, sinks)
    assert [(t, n, i) for t, n, i, _ in sinks.rows] == [tuple(r) for r in c["rows"]]
    np.testing.assert_allclose([v for *_, v in sinks.rows], data[f"run{idx}_rows"], rtol=1e-10, atol=1e-13)
    assert report.switch_count == c["switch_count"]
    assert report.norm_corrections == c["corrections"]


# ---------------------------------------------------------------------------
# NCCL plumbing on the real device (one rank: the box has one GPU)


def test_run_through_nccl_group_matches_single_process(pkg, monkeypatch):
    """run(config, group=<NCCL world of 1>) goes through the NCCL all-reduce of
    the diagonal partials, the object gathers of the norm statistics and the
    state gather for purity; rows equal the group-less run bit for bit."""
    import socket

    import torch.distributed as dist

    p = pkg
    monkeypatch.setenv("CTQW_FORCE_COLLECTIVES", "1")  # run the NCCL calls even on one rank
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda:0"))
    try:
        cfg = p.RunConfig(space=p.JointSpace(p.build_lattice([24]), 2),
                          model=p.CouplingModel(onsite_energy=0.1, interaction=0.3),
                          noise=p.NoiseSpec(target="both", rate=0.3), stepper=p.StepperConfig(dt=0.05),
                          realizations=5, steps=20, post_rate=5, precision="double",
                          observables=("populations", "position_mean_variance", "purity", "participation_ratio"))
        a, b = p.MemorySinks(), p.MemorySinks(dense=True)
        ra = p.run(cfg, a, group=dist.group.WORLD)
        p.run(cfg, b, group=dist.group.WORLD)
        plain = p.MemorySinks()
        rp = p.run(cfg, plain)
        assert a.rows == plain.rows
        assert ra.switch_count == rp.switch_count and ra.norm_corrections == rp.norm_corrections
        np.testing.assert_allclose(b.densities[-1].diagonal().real, plain.densities[-1].diag, rtol=1e-12, atol=1e-15)
    finally:
        dist.destroy_process_group()


def test_evolve_without_second_buffer(pkg):
    """work aliased to psi on a path that needs two buffers: the library uses
    its own second buffer and returns the result in psi."""
    B, n = 3, 96
    h, st, _keep = device_case(2, n, B, "both")
    psi0 = np.tile(orc.product_state(2, n), (B, 1))
    psi = to_dev(psi0)
    swapped = h.evolve(psi, psi, B, 0, 7, stepper(dt=0.05))
    assert not swapped
    ref, _ = orc.evolve_segment(st, psi0.copy(), 0, 7, 0.05)
    assert np.abs(psi.cpu().numpy() - ref).max() <= 1e-13


def test_plane3_in_place_run_capacity(pkg):
    """configs[4] marches in place: one state buffer per realization."""
    p = pkg
    from paper_1612_00746_b200.engine import estimate_memory, marches_in_place

    cfg = p.RunConfig(space=p.JointSpace(p.build_lattice([128]), 3), noise=p.NoiseSpec(rate=0.0),
                      stepper=p.StepperConfig(dt=0.015), realizations=5000, steps=1, post_rate=1,
                      precision="double", memory_budget=200 * 2**30)
    assert marches_in_place(cfg)
    assert estimate_memory(cfg)["state_bytes"] == 5000 * 2**21 * 16


# ---------------------------------------------------------------------------
# exact diagonal accumulation (int64 limbs): bitwise vs the NumPy restatement,
# independent of order and batching


def test_observe_diag_fixed_limbs_bitwise(pkg):
    from tests import fixed_point as fx

    rng = np.random.default_rng(3)
    for R, n in ((37, 24), (5, 256), (300, 16)):
        dim = n * n
        psi = random_states(R, dim, seed=R) * rng.uniform(0.5, 2.0, size=(R, 1))
        h = make_handle(2, n)
        dev = to_dev(psi)
        acc = torch.empty((3, dim), dtype=torch.int64, device="cuda:0")
        h.observe_diag_fixed(dev, R, acc)
        ref = fx.limbs(psi)
        np.testing.assert_array_equal(acc.cpu().numpy(), ref)
        # any order / split of the realizations gives the same limbs
        acc2 = torch.empty_like(acc)
        h.observe_diag_fixed(to_dev(psi[::-1]), R, acc2)
        np.testing.assert_array_equal(acc2.cpu().numpy(), ref)
        h.observe_diag_fixed(to_dev(psi[: R // 2]), R // 2, acc2)
        h.observe_diag_fixed(to_dev(psi[R // 2:]), R - R // 2, acc2, accumulate=True)
        np.testing.assert_array_equal(acc2.cpu().numpy(), ref)
        diag = torch.empty(dim, dtype=torch.float64, device="cuda:0")
        h.fixed_to_double(acc, diag)
        np.testing.assert_array_equal(diag.cpu().numpy(), fx.to_double(ref))
        # the double API is the same sum
        d2 = torch.empty_like(diag)
        h.observe_diag(dev, R, d2)
        np.testing.assert_array_equal(d2.cpu().numpy(), diag.cpu().numpy())
        np.testing.assert_allclose(diag.cpu().numpy(), (np.abs(psi) ** 2).sum(axis=0), rtol=1e-14)
