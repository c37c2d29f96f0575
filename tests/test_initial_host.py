"""Host logic of the initial-state upload (CPU only): the closed-form states'
nonzero entries equal the dense vector the reference builds
(ensemble.py:147-216), and the pooled pinned buffer rewritten in place holds
exactly the new state after any sequence of kinds."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")


def _specs(engine, n):
    rng = np.random.default_rng(3)
    return [engine.InitialStateSpec(kind="product", positions=(2, 7)),
            engine.InitialStateSpec(kind="auto"),
            engine.InitialStateSpec(kind="symmetrized_pair", positions=(4, 5)),
            engine.InitialStateSpec(kind="antisymmetrized_pair", positions=(0, n - 1)),
            engine.InitialStateSpec(kind="symmetrized_pair", positions=(6, 6)),
            engine.InitialStateSpec(kind="custom_vector",
                                    amplitudes=rng.standard_normal(n * n) + 1j * rng.standard_normal(n * n)),
            engine.InitialStateSpec(kind="product", positions=(1, 1))]


def test_entries_match_dense_state():
    import paper_1612_00746_b200 as p
    from paper_1612_00746_b200 import engine

    n = 12
    space = p.JointSpace(p.build_lattice([n]), 2)
    for spec in _specs(engine, n):
        dense = engine.build_initial_state(spec, space)
        entries = engine.initial_state_entries(spec, space)
        if isinstance(entries, np.ndarray):
            np.testing.assert_array_equal(entries, dense)
        else:
            rebuilt = np.zeros(space.dim, dtype=np.complex128)
            for k, v in entries.items():
                rebuilt[k] = v
            np.testing.assert_array_equal(rebuilt, dense)
            assert np.count_nonzero(dense) == len(entries)


def test_pinned_buffer_rewrite_sequence():
    import paper_1612_00746_b200 as p
    from paper_1612_00746_b200 import engine

    n = 12
    space = p.JointSpace(p.build_lattice([n]), 2)
    buf = [torch.full((space.dim,), complex(7.0, -3.0), dtype=torch.complex128), None, None]
    specs = _specs(engine, n)
    for spec in specs + specs[::-1]:
        engine._fill_pinned(buf, engine.initial_state_entries(spec, space))
        np.testing.assert_array_equal(buf[0].numpy(), engine.build_initial_state(spec, space))
