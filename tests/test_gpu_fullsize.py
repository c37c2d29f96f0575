"""Parity at the BASELINE sizes themselves: the full per-GPU ensembles of
configs[2] (N=1024, 1250 realizations, on-site + tunnelling noise),
configs[3] (N=512, 1000) and a 600-realization configs[4] ensemble (m=3,
N=128) advance on the device through the engine; realizations at the
start, middle and end of the stack (different CTAs, pieces and clusters)
are compared with the oracle on the same seeds (ensemble.py:445-558,
propagators.py:167-241).  Exact mode: bit-exact without renormalisations;
FMA mode (the bench's arithmetic): within 1e-12."""

import numpy as np
import pytest

from oracle import ctqw_oracle as orc
from tests.test_gpu_parity import pkg  # noqa: F401

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _oracle_rows(m, n, target, rows, steps, dt):
    nl = n if target in ("tunneling", "both") else 0
    ns = n if target in ("onsite", "both") else 0
    noise = np.stack([np.random.default_rng((1234, r)).choice(np.array([-0.1, 0.1]), nl + ns) for r in rows])
    st = orc.make_stencil(m, n, 0.0, 1.0, 0.0, link=noise[:, :nl] if nl else None,
                          site=noise[:, nl:] if ns else None, batch=len(rows))
    psi0 = np.tile(orc.product_state(m, n), (len(rows), 1))
    ref, stats = orc.evolve_segment(st, psi0, 0, steps, dt, 1.0, "taylor", 4)
    assert stats.corrections == 0
    return ref


@pytest.mark.parametrize("m,n,R,target,steps,dt,kernel", [
    (2, 1024, 1250, "both", 3, 0.02, "band4_kernel"),
    (2, 512, 1000, "tunneling", 3, 0.02, "band4_kernel"),
    (3, 128, 600, "tunneling", 2, 0.015, "plane3_kernel"),
], ids=["configs2", "configs3", "configs4"])
def test_full_ensemble_rows_match_oracle(pkg, m, n, R, target, steps, dt, kernel):
    p = pkg
    from paper_1612_00746_b200 import engine

    rows = [0, 1, R // 2, R - 2, R - 1]
    ref = _oracle_rows(m, n, target, rows, steps, dt)
    for exact in (True, False):
        cfg = p.RunConfig(space=p.JointSpace(p.build_lattice([n]), m),
                          noise=p.NoiseSpec(target=target, levels=(-0.1, 0.1), rate=0.0),
                          stepper=p.StepperConfig(dt=dt), realizations=R, steps=steps, post_rate=steps,
                          precision="double", memory_budget=170 * 2**30, exact=exact, device=0)
        ens = engine.EnsembleState(cfg, 0, 0, R)
        ens.evolve(0, steps)
        st = ens.stats()
        assert st["failure"] is None and st["corrections"] == 0
        assert ens.handle.step_kernel() == kernel
        mine = ens.states()[rows].cpu().numpy()
        if exact:
            np.testing.assert_array_equal(mine, ref)
        else:
            assert np.abs(mine - ref).max() <= 1e-12
        ens.release()
        del ens
        torch.cuda.empty_cache()
