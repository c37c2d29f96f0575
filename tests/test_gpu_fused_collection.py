"""ctqw_evolve_observe (diag(rho) fused into the resident step kernel, or a
segment loop with the limb pass elsewhere) and run()'s batched schedule
path against the per-segment path they replace (ensemble.py:722-769,
density.py:91-95): limbs, rows, per-segment events and failures identical."""

import numpy as np
import pytest

from oracle import ctqw_oracle as orc
from tests.test_gpu_parity import device_case, pkg, stepper, to_dev  # noqa: F401

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _segment_loop(h, psi0, B, first, steps, post, st):
    """Reference schedule: ctqw_evolve per segment + ctqw_observe_diag_fixed."""
    psi = to_dev(psi0)
    work = torch.empty_like(psi)
    dim = psi.shape[1]
    last = first + steps
    targets = [g for g in range(first + 1, last + 1) if (g - first) % post == 0 or g == last]
    acc = torch.zeros((len(targets), 3, dim), dtype=torch.int64, device="cuda:0")
    done = first
    for k, t in enumerate(targets):
        if h.evolve(psi, work, B, done, t - done, st):
            psi, work = work, psi
        h.observe_diag_fixed(psi, B, acc[k], accumulate=True)
        done = t
    return acc.cpu().numpy(), psi.cpu().numpy()


CASES = [
    # (m, n, B, backend, dt, first, steps, post, target): resident64 (fused), band4, generic
    (2, 64, 9, "taylor", 0.02, 0, 37, 10, "tunneling"),
    (2, 64, 9, "taylor", 0.12, 5, 23, 4, "both"),      # renormalisations inside the call
    (2, 64, 4, "rk4", 0.05, 10, 12, 5, "both"),
    (2, 256, 5, "taylor", 0.02, 0, 7, 3, "tunneling"),
    (1, 50, 6, "taylor", 0.05, 3, 9, 4, "both"),
]


@pytest.mark.parametrize("case", CASES, ids=[f"m{c[0]}n{c[1]}{c[3]}post{c[7]}" for c in CASES])
def test_evolve_observe_limbs_equal_segment_loop(pkg, case):
    m, n, B, backend, dt, first, steps, post, target = case
    h, st, _keep = device_case(m, n, B, target)
    psi0 = np.tile(orc.product_state(m, n), (B, 1))
    ref_acc, ref_psi = _segment_loop(h, psi0, B, first, steps, post, stepper(backend, 4, dt, exact=True))
    psi = to_dev(psi0)
    work = torch.empty_like(psi)
    acc = torch.full_like(torch.as_tensor(ref_acc, device="cuda:0"), 7)  # the call zeroes it
    swapped = h.evolve_observe(psi, work, B, first, steps, post, acc, stepper(backend, 4, dt, exact=True))
    out = (work if swapped else psi).cpu().numpy()
    np.testing.assert_array_equal(acc.cpu().numpy(), ref_acc)
    np.testing.assert_array_equal(out, ref_psi)
    if m == 2 and n == 64:
        assert h.step_kernel() == "resident64_kernel"
    # batched reduction == per-point fixed_to_double + observe_reduce
    P = ref_acc.shape[0]
    pts = torch.empty((P, n + 3), dtype=torch.float64, device="cuda:0")
    diag = torch.empty((P, n ** m), dtype=torch.float64, device="cuda:0")
    h.observe_points(acc, P, float(B), pts, diag)
    for k in range(P):
        d1 = torch.empty(n ** m, dtype=torch.float64, device="cuda:0")
        h.fixed_to_double(acc[k], d1)
        pops = torch.empty(n, dtype=torch.float64, device="cuda:0")
        sc = torch.empty(3, dtype=torch.float64, device="cuda:0")
        h.observe_reduce(d1, float(B), pops, sc, None)
        np.testing.assert_array_equal(diag[k].cpu().numpy(), d1.cpu().numpy())
        np.testing.assert_array_equal(pts[k, :n].cpu().numpy(), pops.cpu().numpy())
        np.testing.assert_array_equal(pts[k, n:].cpu().numpy(), sc.cpu().numpy())


def _run(p, cfg, fused, monkeypatch):
    from paper_1612_00746_b200 import engine

    if not fused:
        monkeypatch.setattr(engine, "fused_collection_ok", lambda *a: False)
    sinks = p.MemorySinks(keep_densities=False)
    err = None
    try:
        rep = p.run(cfg, sinks)
    except p.NormFailureError as e:
        rep, err = None, (e.realization, e.step, round(e.deviation, 12))
    monkeypatch.undo()
    return sinks, rep, err


@pytest.mark.parametrize("n,steps,post,dt,obs", [
    (64, 150, 10, 0.02, None),                       # configs[0] shape, resident64 fused
    (64, 60, 7, 0.11, ("populations", "participation_ratio", "joint_distribution")),  # rescales, ragged
    (96, 40, 15, 0.05, None),                        # band/tile path, segment loop
    (64, 30, 10, 0.35, None),                        # norm failure mid-run
    (64, 100, 10, 0.02, ("populations", "position_mean_variance", "purity", "participation_ratio")),  # purity
    (64, 45, 7, 0.11, ("purity", "joint_distribution")),  # purity with renormalisations, ragged schedule
])
def test_run_batched_path_equals_segment_path(pkg, monkeypatch, n, steps, post, dt, obs):
    p = pkg
    cfg = p.RunConfig(space=p.JointSpace(p.build_lattice([n]), 2),
                      model=p.CouplingModel(onsite_energy=0.1, interaction=0.5),
                      noise=p.NoiseSpec(target="both", rate=0.0), stepper=p.StepperConfig(dt=dt),
                      realizations=12, steps=steps, post_rate=post, precision="double",
                      observables=obs if obs else ("populations", "position_mean_variance", "participation_ratio"))
    a, ra, ea = _run(p, cfg, True, monkeypatch)
    b, rb, eb = _run(p, cfg, False, monkeypatch)
    assert ea == eb
    assert a.rows == b.rows  # bitwise: the same limbs and reductions
    assert [(e.realization, e.step, e.corrected, e.deviation) for e in a.events] == \
           [(e.realization, e.step, e.corrected, e.deviation) for e in b.events]
    if ra is not None:
        assert (ra.norm_corrections, ra.norm_events, ra.snapshots) == (rb.norm_corrections, rb.norm_events,
                                                                        rb.snapshots)
        assert ra.max_norm_deviation == rb.max_norm_deviation
