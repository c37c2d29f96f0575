"""Randomised general-lattice sweep (fixed seed) through the public
single-step API on the device: one- and two-dimensional lattices, periodic
and open boundaries, k_half up to 2, per-direction tunnelling, m = 1..3,
on-site and link noise.  apply / Taylor (orders 1-6) / RK4 must equal the
oracle bit for bit (the reference's operation order; the oracle is pinned
to the reference on seven such lattices in test_oracle_golden.py)."""

import numpy as np
import pytest

from oracle import ctqw_oracle as orc
from tests.test_gpu_parity import pkg  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _lattices(count=24, seed=1612):
    import paper_1612_00746_b200 as p

    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        q = int(rng.integers(1, 3))
        dims = [int(rng.integers(3, 30))] if q == 1 else [int(rng.integers(2, 8)) for _ in range(2)]
        k_half = [int(rng.integers(1, 3)) for _ in range(q)]
        boundary = str(rng.choice(["periodic", "open"]))
        try:
            p.build_lattice(dims, k_half=k_half, boundary=boundary)
        except p.ConfigurationError:
            continue
        n = int(np.prod(dims))
        m = int(rng.integers(1, 4))
        while m > 1 and n ** m > 6000:
            m -= 1
        out.append(dict(dims=dims, k_half=k_half, boundary=boundary, m=m,
                        tunneling=[round(float(v), 3) for v in rng.uniform(0.5, 1.5, q)],
                        onsite=round(float(rng.uniform(-0.5, 0.5)), 3),
                        interaction=round(float(rng.uniform(0.0, 1.5)), 3),
                        order=int(rng.integers(1, 7)), dt=round(float(rng.uniform(0.01, 0.05)), 4),
                        b=int(rng.integers(1, 4)), site=bool(rng.integers(0, 2)), seed=int(rng.integers(1 << 30))))
    return out


CASES = _lattices()


@pytest.mark.parametrize("c", CASES, ids=[f"{'x'.join(map(str, c['dims']))}k{''.join(map(str, c['k_half']))}"
                                          f"{c['boundary'][0]}m{c['m']}" for c in CASES])
def test_random_lattice_matches_oracle(pkg, c):
    p = pkg
    lat = p.build_lattice(c["dims"], k_half=c["k_half"], boundary=c["boundary"])
    topo = p.build_topology(p.JointSpace(lat, c["m"]))
    model = p.CouplingModel(onsite_energy=c["onsite"], tunneling=tuple(c["tunneling"]),
                            interaction=c["interaction"])
    n = lat.n_sites
    K = sum(c["k_half"])
    rng = np.random.default_rng(c["seed"])
    link = 0.1 * rng.normal(size=(c["b"], n * K))
    site = 0.1 * rng.normal(size=(c["b"], n)) if c["site"] else None
    psi = rng.normal(size=(c["b"], n ** c["m"])) + 1j * rng.normal(size=(c["b"], n ** c["m"]))
    psi /= np.linalg.norm(psi, axis=1, keepdims=True)
    st = orc.make_lattice_stencil(c["m"], c["dims"], c["k_half"], c["boundary"], c["onsite"], c["tunneling"],
                                  c["interaction"], link=link, site=site, batch=c["b"])
    values = p.assemble_values(topo, model, link_values=link, site_values=site)
    np.testing.assert_array_equal(p.apply_values(topo, values, psi), orc.apply_stencil(st, psi))
    np.testing.assert_array_equal(p.step_taylor_values(topo, values, psi, c["dt"], order=c["order"]),
                                  orc.taylor_step(st, psi, c["dt"], 1.0, c["order"]))
    np.testing.assert_array_equal(p.step_rk4_values(topo, values, psi, c["dt"]), orc.rk4_step(st, psi, c["dt"], 1.0))
