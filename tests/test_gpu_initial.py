"""ctqw_set_initial (the lazy np.tile(psi0) of ensemble.py:678): the first
step reading one shared initial state gives the same bits as filling the
stack first, on every kernel family (band4 reads it directly, resident64
too; plane3, tile and the generic kernels fill the stack themselves)."""

import numpy as np
import pytest

from oracle import ctqw_oracle as orc
from tests.test_gpu_parity import device_case, pkg, stepper, to_dev  # noqa: F401

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.mark.parametrize("m,n,B,backend,steps,kernel", [
    (2, 256, 5, "taylor", 3, "band4_kernel"),
    (2, 256, 5, "rk4", 2, "band4_kernel"),
    (2, 1024, 3, "taylor", 2, "band4_kernel"),
    (2, 64, 4, "taylor", 5, "resident64_kernel"),
    (2, 32, 4, "taylor", 5, "resident_kernel"),
    (2, 100, 3, "taylor", 2, "band4_kernel"),        # runtime-N band4 (cp.async ring)
    (2, 102, 3, "taylor", 2, "tile_step_kernel"),    # N % 4 != 0
    (1, 40, 4, "taylor", 3, "taylor_order_kernel"),
    (3, 128, 1, "taylor", 2, "plane3_kernel"),
], ids=lambda c: str(c))
def test_set_initial_equals_filled_stack(pkg, m, n, B, backend, steps, kernel):
    h, st, _keep = device_case(m, n, B, "both")
    psi0 = torch.as_tensor(orc.product_state(m, n), device="cuda:0")
    sp = stepper(backend, 4, 0.03, exact=True)
    # reference: the stack filled first
    a = torch.empty((B, n ** m), dtype=torch.complex128, device="cuda:0")
    wa = torch.empty_like(a)
    h.fill_states(a, B, psi0)
    sa = h.evolve(a, wa, B, 0, steps, sp)
    ref = (wa if sa else a).cpu().numpy()
    # lazy: psi holds garbage, the first step reads psi0
    b = torch.full((B, n ** m), float("nan"), dtype=torch.complex128, device="cuda:0")
    wb = torch.empty_like(b)
    h.set_initial(psi0)
    sb = h.evolve(b, wb, B, 0, steps, sp)
    got = (wb if sb else b).cpu().numpy()
    assert h.step_kernel() == kernel
    np.testing.assert_array_equal(got, ref)


def test_engine_states_before_the_first_step_are_materialised(pkg):
    p = pkg
    from paper_1612_00746_b200 import engine

    cfg = p.RunConfig(space=p.JointSpace(p.build_lattice([64]), 2), noise=p.NoiseSpec(rate=0.0),
                      realizations=3, steps=2, post_rate=2, precision="double", device=0)
    ens = engine.EnsembleState(cfg, 0, 0, 3)
    s = ens.states().cpu().numpy()
    np.testing.assert_array_equal(s, np.tile(orc.product_state(2, 64), (3, 1)))
    ens.release()


def test_pinned_initial_pool_across_state_kinds(pkg):
    """The pooled pinned upload buffer (engine._PINNED) rewrites only the
    nonzeros of closed-form initial states: a sequence of runs with different
    kinds and positions on one pool gives, run for run, the rows of the same
    runs on an empty pool."""
    p = pkg
    from paper_1612_00746_b200 import engine

    n = 16
    rng = np.random.default_rng(5)
    custom = rng.standard_normal(n * n) + 1j * rng.standard_normal(n * n)
    specs = [engine.InitialStateSpec(kind="product", positions=(3, 9)),
             engine.InitialStateSpec(kind="symmetrized_pair", positions=(5, 6)),
             engine.InitialStateSpec(kind="custom_vector", amplitudes=custom),
             engine.InitialStateSpec(kind="antisymmetrized_pair", positions=(1, 12)),
             engine.InitialStateSpec(kind="auto")]

    def run(spec):
        cfg = p.RunConfig(space=p.JointSpace(p.build_lattice([n]), 2), initial=spec,
                          noise=p.NoiseSpec(target="both", rate=0.0), stepper=p.StepperConfig(dt=0.05),
                          realizations=3, steps=6, post_rate=3, precision="double",
                          observables=("populations", "participation_ratio", "joint_distribution"))
        sinks = p.MemorySinks(keep_densities=False)
        p.run(cfg, sinks)
        return sinks.rows

    pooled = [run(s) for s in specs]
    fresh = []
    for s in specs:
        engine._PINNED.clear()
        fresh.append(run(s))
    assert pooled == fresh
    assert all(pooled[k] != pooled[k + 1] for k in range(len(pooled) - 1))  # the states differ
