"""Pin the oracle against fixtures produced by the reference itself (CPU only)."""

import json

import numpy as np
import pytest

from oracle import ctqw_oracle as orc
from oracle.noise_oracle import draw_static_noise
from tests.conftest import load_golden


def test_noise_draws_bit_exact():
    data, meta = load_golden("noise_draws.npz")
    assert len(meta) == 75
    for case in meta:
        total = case["n_links"] + case["n_sites"]
        mine = draw_static_noise(case["seed"], case["r"], case["levels"], total)
        np.testing.assert_array_equal(mine, data[case["key"]])


def _stencil(case, link, site):
    return orc.make_stencil(case["m"], case["n"], case["onsite"], case["tunneling"],
                            case["interaction"], link=link, site=site, batch=case["b"])


@pytest.mark.parametrize("idx", range(5))
def test_apply_and_single_steps_bit_exact(idx):
    data, meta = load_golden("stencil_steps.npz")
    case = meta[idx]
    st = _stencil(case, data[f"link{idx}"], data[f"site{idx}"])
    psi = data[f"psi{idx}"]
    np.testing.assert_array_equal(orc.apply_stencil(st, psi), data[f"apply{idx}"])
    np.testing.assert_array_equal(orc.taylor_step(st, psi, case["dt"], case["hbar"], 4),
                                  data[f"taylor4_{idx}"])
    np.testing.assert_array_equal(orc.taylor_step(st, psi, case["dt"], case["hbar"], 7),
                                  data[f"taylor7_{idx}"])
    np.testing.assert_array_equal(orc.rk4_step(st, psi, case["dt"], case["hbar"]), data[f"rk4_{idx}"])
    st_t = _stencil(case, data[f"link{idx}"], None)
    np.testing.assert_array_equal(orc.taylor_step(st_t, psi, case["dt"], case["hbar"], 4),
                                  data[f"taylor4t_{idx}"])


@pytest.mark.parametrize("idx", range(5))
def test_segments_with_norm_policy(idx):
    data, meta = load_golden("segments.npz")
    c = meta[idx]
    total_links = c["n"] if c["target"] in ("tunneling", "both") else 0
    total_sites = c["n"] if c["target"] in ("onsite", "both") else 0
    noise = np.stack([draw_static_noise(c["seed"], r, (-0.1, 0.1), total_links + total_sites)
                      for r in range(c["b"])])
    link = noise[:, :total_links] if total_links else None
    site = noise[:, total_links:] if total_sites else None
    st = orc.make_stencil(c["m"], c["n"], c["onsite"], c["tunneling"], c["interaction"],
                          link=link, site=site, batch=c["b"])
    psi0 = np.tile(orc.product_state(c["m"], c["n"]), (c["b"], 1))
    psi, stats = orc.evolve_segment(st, psi0, 0, c["steps"], c["dt"], 1.0, c["backend"], c["order"])
    ref = data[f"psi{idx}"]
    # The squared norm is an einsum in the reference; everything else is in
    # reference order, so agreement is at rounding level even after rescales.
    err = np.abs(psi - ref).max()
    assert err <= 1e-14, err
    assert stats.event_count == c["event_count"]
    assert stats.corrections == c["corrections"]
    assert abs(stats.max_deviation - c["max_deviation"]) <= 1e-12 * max(1.0, c["max_deviation"])
    ev = np.array([[d, float(k), r, s] for d, k, r, s in stats.events]).reshape(-1, 4)
    np.testing.assert_array_equal(ev[:, 1:], data[f"ev{idx}"][:, 1:])
    np.testing.assert_allclose(ev[:, 0], data[f"ev{idx}"][:, 0], rtol=1e-9)
    if c["event_count"] == 0:
        np.testing.assert_array_equal(psi, ref)  # no rescale -> bit identical


def test_norm_failure_names_culprit():
    data, _ = load_golden("segments.npz")
    fail = json.loads(str(data["failure"]))
    assert fail is not None
    noise = np.stack([draw_static_noise(99, r, (-0.4, 0.4), 18) for r in range(4)])
    st = orc.make_stencil(2, 9, 0.0, 1.0, 0.0, link=noise[:, :9], site=noise[:, 9:], batch=4)
    psi0 = np.zeros((4, 81), dtype=np.complex128)
    psi0[:, 3 * 9 + 4] = 1.0
    with pytest.raises(orc.NormFailure) as info:
        orc.evolve_segment(st, psi0, 0, 50, 0.6, renormalize=False)
    assert info.value.realization == fail["realization"]
    assert info.value.step == fail["step"]
    assert info.value.deviation == pytest.approx(fail["deviation"], rel=1e-12)


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
def test_run_rows(idx):
    data, meta = load_golden("run_rows.npz")
    c = meta[idx]
    nl = c["n"] if c["target"] in ("tunneling", "both") else 0
    ns = c["n"] if c["target"] in ("onsite", "both") else 0
    noise = np.stack([draw_static_noise(1234, r, (-0.1, 0.1), nl + ns) for r in range(c["R"])])
    st = orc.make_stencil(c["m"], c["n"], c["onsite"], c["tunneling"], c["interaction"],
                          link=noise[:, :nl] if nl else None, site=noise[:, nl:] if ns else None,
                          batch=c["R"])
    out, _, totals = orc.run_rows(st, _initial(c), c["R"], c["steps"], c["post_rate"], c["dt"],
                                  backend=c["backend"], observables=c["observables_resolved"])
    rows = [(t, name, i, v) for t, rr in out for name, i, v in rr]
    assert [(t, n, i) for t, n, i, _ in rows] == [tuple(r) for r in c["rows"]]
    mine = np.array([v for *_, v in rows])
    ref = data[f"rows{idx}"]
    # 1e-10 relative (the north-star bar) on every row; wrap flags exact.
    np.testing.assert_allclose(mine, ref, rtol=1e-10, atol=1e-13)
    assert totals.corrections == c["corrections"]
    assert totals.event_count == c["norm_events"]


# ---------------------------------------------------------------------------
# dynamic telegraph noise (rate > 0)


@pytest.mark.parametrize("ti", range(2))
def test_telegraph_oracle_matches_reference_trajectory(ti):
    """TelegraphOracle == the reference's init_process/advance, bit for bit."""
    from oracle.noise_oracle import TelegraphOracle

    data, meta = load_golden("telegraph.npz")
    c = meta["trajectories"][ti]
    tg = TelegraphOracle(c["seed"], c["r0"], c["count"], c["levels"], c["n_links"], c["n_sites"], c["rate"])
    done = 0
    for k in c["checkpoints"]:
        for _ in range(k - done):
            tg.advance(c["dt"])
        done = k
        np.testing.assert_array_equal(tg.values, data[f"traj{ti}_values_{k}"])
        np.testing.assert_array_equal(tg.next_switch, data[f"traj{ti}_next_{k}"])
        np.testing.assert_array_equal(tg.time, data[f"traj{ti}_time_{k}"])
        np.testing.assert_array_equal(tg.switches, data[f"traj{ti}_switches_{k}"])


@pytest.mark.parametrize("idx", range(2))
def test_run_rows_dynamic_noise(idx):
    """Oracle run with telegraph noise == the reference's run() rows."""
    from oracle.noise_oracle import TelegraphOracle

    data, meta = load_golden("telegraph.npz")
    c = meta["runs"][idx]
    nl = c["n"] if c["target"] in ("tunneling", "both") else 0
    ns = c["n"] if c["target"] in ("onsite", "both") else 0
    tg = TelegraphOracle(1234, 0, c["R"], (-0.1, 0.1), nl, ns, c["rate"])
    st = orc.make_stencil(c["m"], c["n"], c["onsite"], c["tunneling"], c["interaction"],
                          link=tg.link_values() if nl else None, site=tg.site_values().copy() if ns else None,
                          batch=c["R"])
    out, _, totals = orc.run_rows(st, orc.product_state(c["m"], c["n"]), c["R"], c["steps"], c["post_rate"],
                                  c["dt"], backend=c["backend"], noise=tg, tunneling=c["tunneling"])
    rows = [(t, name, i, v) for t, rr in out for name, i, v in rr]
    assert [(t, n, i) for t, n, i, _ in rows] == [tuple(r) for r in c["rows"]]
    np.testing.assert_allclose([v for *_, v in rows], data[f"run{idx}_rows"], rtol=1e-10, atol=1e-13)
    assert int(tg.switches.sum()) == c["switch_count"]
    assert totals.corrections == c["corrections"]


# ---------------------------------------------------------------------------
# general lattices (q > 1, k_half > 1, open boundaries)


@pytest.mark.parametrize("idx", range(7))
def test_lattice_steps_match_reference(idx):
    data, meta = load_golden("lattices.npz")
    c = meta["steps"][idx]
    st = orc.make_lattice_stencil(c["m"], c["dims"], c["k_half"], c["boundary"], c["onsite"], c["tunneling"],
                                  c["interaction"], link=data[f"link{idx}"], site=data[f"site{idx}"],
                                  batch=c["b"])
    psi = data[f"psi{idx}"]
    np.testing.assert_array_equal(orc.apply_stencil(st, psi), data[f"apply{idx}"])
    np.testing.assert_array_equal(orc.taylor_step(st, psi, c["dt"], c["hbar"], 4), data[f"taylor4_{idx}"])
    np.testing.assert_array_equal(orc.rk4_step(st, psi, c["dt"], c["hbar"]), data[f"rk4_{idx}"])


@pytest.mark.parametrize("idx", range(3))
def test_lattice_run_rows(idx):
    from oracle.noise_oracle import TelegraphOracle

    data, meta = load_golden("lattices.npz")
    c = meta["runs"][idx]
    n = int(np.prod(c["dims"]))
    K = sum(c["k_half"])
    nl = n * K if c["target"] in ("tunneling", "both") else 0
    ns = n if c["target"] in ("onsite", "both") else 0
    if c["rate"] > 0:
        tg = TelegraphOracle(1234, 0, c["R"], (-0.1, 0.1), nl, ns, c["rate"])
        noise = tg.values
    else:
        tg = None
        noise = np.stack([draw_static_noise(1234, r, (-0.1, 0.1), nl + ns) for r in range(c["R"])])
    st = orc.make_lattice_stencil(c["m"], c["dims"], c["k_half"], c["boundary"], 0.1, 1.0, 0.5,
                                  link=noise[:, :nl] if nl else None, site=noise[:, nl:].copy() if ns else None,
                                  batch=c["R"])
    out, _, totals = orc.run_rows(st, orc.product_state(c["m"], n), c["R"], c["steps"], c["post_rate"], 0.05,
                                  observables=c["observables_resolved"], noise=tg, tunneling=1.0,
                                  periodic=c["boundary"] == "periodic")
    rows = [(t, name, i, v) for t, rr in out for name, i, v in rr]
    assert [(t, nm, i) for t, nm, i, _ in rows] == [tuple(r) for r in c["rows"]]
    np.testing.assert_allclose([v for *_, v in rows], data[f"run{idx}_rows"], rtol=1e-10, atol=1e-13)


def test_config0_oracle_prefix_matches_reference_run():
    """BASELINE configs[0] (N=64, R=100, tunnelling, Taylor-4, dt=0.02, post
    every 10 steps) through the reference's own run(): the oracle reproduces
    the first 100 steps (10 snapshots) of the committed 1500-step rows (the
    full length is checked on the GPU, tests/test_gpu_bench_parity.py)."""
    data, meta = load_golden("config0_run.npz")
    n, R, dt = meta["n"], meta["R"], meta["dt"]
    noise = np.stack([np.random.default_rng((meta["master_seed"], r)).choice(np.array(meta["levels"]), n)
                      for r in range(R)])
    st = orc.make_stencil(2, n, 0.0, 1.0, 0.0, link=noise, batch=R)
    obs = tuple(meta["observables_resolved"])
    out, _, _ = orc.run_rows(st, orc.product_state(2, n), R, 100, meta["post_rate"], dt, observables=obs)
    mine = np.array([v for _, rows in out for _, _, v in rows])
    ref = data["rows"][: mine.size]
    assert [tuple(r) for r in meta["rows"][: mine.size]] == [(t, nm, i) for t, rows in out for nm, i, _ in rows]
    np.testing.assert_allclose(mine, ref, rtol=1e-12, atol=1e-14)
