"""Host-side API (no GPU): configuration validation with the reference's error
classes, schedules, initial states, memory estimate, and the C ABI library
loading with every symbol ``include/ctqw.h`` declares."""

import os
import re

import numpy as np
import pytest

import paper_1612_00746_b200 as p
from paper_1612_00746_b200 import native, sharding
from tests.conftest import ROOT


def ring(n, m=1):
    return p.JointSpace(lattice=p.build_lattice([n]), m=m)


def cfg(**kw):
    base = dict(space=ring(9), noise=p.NoiseSpec(levels=(0.0,), rate=0.0),
                stepper=p.StepperConfig(dt=0.05), realizations=1, steps=20, post_rate=20,
                precision="double")
    base.update(kw)
    return p.RunConfig(**base)


def test_exit_codes_match_reference():
    assert p.ConfigurationError.exit_code == 2
    assert p.NumericError.exit_code == 3
    assert p.NormFailureError.exit_code == 3
    assert p.CapacityError.exit_code == 4
    assert p.MemoryBudgetError.exit_code == 4
    assert p.SnapshotFormatError.exit_code == 5
    e = p.NormFailureError(2.5e-3, realization=7, step=12)
    assert "realization 7, step 12" in str(e) and "reduce the time step" in str(e)
    import pickle

    e2 = pickle.loads(pickle.dumps(e))
    assert (e2.deviation, e2.realization, e2.step) == (2.5e-3, 7, 12)


def test_schedule_semantics():
    assert cfg(steps=6, post_rate=2).schedule == (2, 4, 6)
    assert cfg(steps=7, post_rate=3).schedule == (3, 6, 7)
    assert cfg(steps=0, post_rate=10).schedule == (0,)
    assert cfg(steps=1500, post_rate=1500).schedule == (1500,)


@pytest.mark.parametrize("bad", [dict(post_rate=0), dict(steps=10, post_rate=11), dict(realizations=0),
                                 dict(precision="half"), dict(observables=("entropy",)),
                                 dict(observables=()), dict(memory_budget=0)])
def test_run_config_validation(bad):
    with pytest.raises(p.ConfigurationError):
        cfg(**bad)


def test_stepper_and_model_validation():
    with pytest.raises(p.ConfigurationError):
        p.StepperConfig(backend="verlet")
    with pytest.raises(p.ConfigurationError):
        p.StepperConfig(dt=0.0)
    with pytest.raises(p.ConfigurationError):
        p.StepperConfig(taylor_order=0)
    with pytest.raises(p.ConfigurationError):
        p.StepperConfig(tol_norm=1e-3, tol_fail=1e-6)
    with pytest.raises(p.ConfigurationError):
        p.CouplingModel(hbar=0.0)
    with pytest.raises(p.ConfigurationError):
        p.NoiseSpec(target="links")
    with pytest.raises(p.ConfigurationError):
        p.NoiseSpec(levels=())
    with pytest.raises(p.ConfigurationError):
        p.build_lattice([4], k_half=[2])
    # the eigen backend validates but is rejected by the device path
    with pytest.raises(p.ConfigurationError):
        p.StepperConfig(backend="eigen").native()


def test_default_observables_and_position_rule():
    assert cfg().observables == ("populations", "position_mean_variance", "purity", "participation_ratio")
    grid = p.JointSpace(p.build_lattice([3, 3]), 1)
    assert "position_mean_variance" not in p.RunConfig(space=grid, steps=1, post_rate=1).observables
    with pytest.raises(p.ConfigurationError):
        p.RunConfig(space=grid, steps=1, post_rate=1, observables=("position_mean_variance",))


def test_topology_scope():
    assert p.build_topology(ring(7, 2)).dim == 49
    assert p.build_topology(ring(7, 2)).is_ring
    grid = p.build_topology(p.JointSpace(p.build_lattice([3, 4]), 2))
    assert not grid.is_ring and grid.K == 2 and grid.n_links == 24
    chain = p.build_topology(p.JointSpace(p.build_lattice([8], boundary="open"), 1))
    pos, neg, _ = chain.move_tables()
    assert pos[7, 0] == -1 and neg[0, 0] == -1 and pos[3, 0] == 4
    with pytest.raises(p.ConfigurationError):
        p.build_topology(ring(5, 4))


def test_site_move_tables_match_reference_convention():
    """Slots direction-major, distance 1..k_half (hilbert.py:189-224)."""
    lat = p.build_lattice([4, 5], k_half=[1, 2])
    pos, neg, dirs, dist = p.site_move_tables(lat)
    assert list(dirs) == [0, 1, 1] and list(dist) == [1, 1, 2]
    # site (1, 3) = 8: +x0 -> (2, 3) = 13, +x1 by 2 -> (1, 0) = 5 (periodic)
    assert pos[8, 0] == 13 and pos[8, 2] == 5 and neg[8, 1] == 7
    for s in range(3):  # mirror pairing: neg undoes pos
        assert all(neg[pos[x, s], s] == x for x in range(lat.n_sites))


def test_initial_states():
    space = ring(7, 2)
    psi = p.build_initial_state(p.InitialStateSpec(), space)
    assert psi[p.joint_index([2, 3], space)] == 1.0 and np.count_nonzero(psi) == 1
    psi = p.build_initial_state(p.InitialStateSpec(kind="antisymmetrized_pair", positions=(1, 3)), ring(5, 2))
    assert psi[p.joint_index([3, 1], ring(5, 2))] == pytest.approx(-1 / np.sqrt(2))
    with pytest.raises(p.ConfigurationError):
        p.build_initial_state(p.InitialStateSpec(kind="antisymmetrized_pair", positions=(2, 2)), ring(5, 2))
    psi = p.build_initial_state(p.InitialStateSpec(kind="custom_vector", amplitudes=np.array([2, 0, 0, 2j])),
                                ring(4))
    assert np.linalg.norm(psi) == pytest.approx(1.0)
    assert p.build_initial_state(p.InitialStateSpec(), ring(9))[4] == 1.0
    space3 = ring(6, 3)
    psi = p.build_initial_state(p.InitialStateSpec(kind="product", positions=(0, 0, 5)), space3)
    assert psi[p.joint_index([0, 0, 5], space3)] == 1.0


def test_joint_index_roundtrip():
    space = ring(11, 3)
    a = np.arange(space.dim)
    np.testing.assert_array_equal(p.joint_index(p.joint_positions(a, space), space), a)


def test_memory_estimate_and_budget():
    est = p.estimate_memory(cfg(space=ring(256, 2), realizations=1000))
    assert est["state_bytes"] == 2 * 1000 * 65536 * 16
    assert est["topology_bytes"] == 0
    assert p.estimate_memory(cfg(space=ring(256, 2), realizations=1000), world=8)["state_bytes"] == \
        2 * 125 * 65536 * 16


def test_run_rejects_out_of_scope_before_touching_device():
    with pytest.raises(p.MemoryBudgetError):
        p.run(cfg(memory_budget=16))
    with pytest.raises(p.ConfigurationError):
        p.run(cfg(stepper=p.StepperConfig(backend="eigen")))
    with pytest.raises(p.CapacityError):
        p.run(cfg(space=ring(1024, 2), realizations=10000, memory_budget=2**50))


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(p.NativeError):
        p.run(cfg())
    with pytest.raises(p.NativeError):
        native.Handle(2, 16, 0.0, 1.0, 0.0, 1.0)
    with pytest.raises(p.NativeError):
        p.run(cfg(noise=p.NoiseSpec(rate=0.5)))  # dynamic noise is device-only too


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "ctqw.h")).read()
    declared = set(re.findall(r"^\S.*?\b(ctqw_[a-z_0-9]+)\s*\(", header, flags=re.M))
    assert declared == set(native.SIGNATURES), declared ^ set(native.SIGNATURES)
    lib = native.load_library()
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.ctqw_abi_version() == 1
    assert native.exported_symbols() == list(native.SIGNATURES)


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", native.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_handle_create_errors_without_device():
    """ctqw_create validates before touching CUDA."""
    lib = native.load_library()
    import ctypes

    h = ctypes.c_void_p()
    bad = native.Model(4, 16, 1, 1, 0.0, 1.0, 0.0, 1.0)
    assert lib.ctqw_create(ctypes.byref(bad), 0, ctypes.byref(h)) == 2
    bad = native.Model(2, 16, 0, 1, 0.0, 1.0, 0.0, 1.0)  # no move slots
    assert lib.ctqw_create(ctypes.byref(bad), 0, ctypes.byref(h)) == 2
    bad = native.Model(2, 1, 1, 0, 0.0, 1.0, 0.0, 1.0)  # one-site lattice
    assert lib.ctqw_create(ctypes.byref(bad), 0, ctypes.byref(h)) == 2
    bad = native.Model(2, 16, 1, 1, 0.0, 1.0, 0.0, -1.0)
    assert lib.ctqw_create(ctypes.byref(bad), 0, ctypes.byref(h)) == 2
    assert b"hbar" in lib.ctqw_last_error(None)


def test_shard_bounds_cover_realizations():
    for R in (1, 7, 100, 1001):
        for world in (1, 2, 3, 8):
            shards = sharding.all_shards(R, world)
            assert shards[0][0] == 0 and shards[-1][1] == R
            assert all(a[1] == b[0] for a, b in zip(shards, shards[1:]))
            sizes = [hi - lo for lo, hi in shards]
            assert max(sizes) - min(sizes) <= 1


def test_merge_stats_is_split_independent():
    """Failure = earliest step, then largest deviation, then lowest
    realization; events = first MAX_EVENTS in (step, realization) order --
    the same answer a single process gives, whatever the shard split."""
    a = {"event_count": 2, "corrections": 2, "max_deviation": 3e-6, "events": [(3e-6, True, 1, 5)],
         "failure": None}
    b = {"event_count": 1, "corrections": 1, "max_deviation": 2e-6, "events": [(2e-6, True, 9, 2)],
         "failure": (5e-3, 9, 4)}
    c = {"event_count": 0, "corrections": 0, "max_deviation": 0.0, "events": [], "failure": (9e-3, 12, 1)}
    m = sharding.merge_segment_stats([a, b, c])
    assert m["event_count"] == 3 and m["corrections"] == 3
    assert m["max_deviation"] == 3e-6
    assert m["events"] == [(2e-6, True, 9, 2), (3e-6, True, 1, 5)]
    assert m["failure"] == (9e-3, 12, 1)
    # same step: the larger deviation, then the lower realization
    d = {"event_count": 0, "corrections": 0, "max_deviation": 0.0, "events": [], "failure": (9e-3, 3, 1)}
    e = {"event_count": 0, "corrections": 0, "max_deviation": 0.0, "events": [], "failure": (8e-3, 1, 1)}
    assert sharding.merge_segment_stats([c, e, d])["failure"] == (9e-3, 3, 1)
    # order of the ranks does not matter
    assert sharding.merge_segment_stats([c, b, a]) == m


def test_stats_pack_roundtrip():
    st = {"event_count": 250, "corrections": 7, "max_deviation": 1.5e-6,
          "events": [(1e-6 * k, k % 2 == 0, 1000 + k, 3 + k // 10) for k in range(100)],
          "failure": (2e-3, 123456789, 42)}
    rec = sharding.pack_stats(st)
    assert len(rec) == 8 + 4 * sharding.MAX_EVENTS
    assert sharding.unpack_stats(rec) == st
    st2 = dict(st, events=[], failure=None)
    assert sharding.unpack_stats(sharding.pack_stats(st2)) == st2
