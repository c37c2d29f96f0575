"""Multi-process (world_size 2, gloo, CPU) checks of the sharding plumbing that
run() uses over NCCL on GPUs: shard ownership, the all-reduce of per-rank
diagonal partial sums, the all-gather of norm statistics, and the state
gather used for purity.  The per-rank partial sums come from the oracle, so
the distributed reduction must reproduce the single-process observables."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ctqw_oracle as orc
        from paper_1612_00746_b200 import sharding

        n, m, R, steps, dt = 12, 2, 7, 15, 0.05
        lo, hi = sharding.shard_bounds(R, world, rank)
        noise = np.stack([np.random.default_rng((1234, r)).choice(np.array([-0.1, 0.1]), 2 * n)
                          for r in range(lo, hi)])
        st = orc.make_stencil(m, n, 0.1, 1.0, 0.4, link=noise[:, :n], site=noise[:, n:], batch=hi - lo)
        psi = np.tile(orc.product_state(m, n), (hi - lo, 1))
        psi, stats = orc.evolve_segment(st, psi, 0, steps, dt, r0=lo)
        diag = torch.tensor((psi.real ** 2 + psi.imag ** 2).sum(axis=0))
        sharding.allreduce_sum_(diag)
        local = {"event_count": stats.event_count, "corrections": stats.corrections,
                 "max_deviation": stats.max_deviation, "events": stats.events, "failure": None}
        merged = sharding.merge_segment_stats(sharding.gather_stats(local))
        states = sharding.gather_states(torch.tensor(psi))
        if rank == 0:
            out_q.put((diag.numpy(), merged, states.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_reduction_matches_single_process():
    from oracle import ctqw_oracle as orc

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    diag, merged, states = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0

    n, m, R, steps, dt = 12, 2, 7, 15, 0.05
    noise = np.stack([np.random.default_rng((1234, r)).choice(np.array([-0.1, 0.1]), 2 * n)
                      for r in range(R)])
    st = orc.make_stencil(m, n, 0.1, 1.0, 0.4, link=noise[:, :n], site=noise[:, n:], batch=R)
    psi, stats = orc.evolve_segment(st, np.tile(orc.product_state(m, n), (R, 1)), 0, steps, dt)
    np.testing.assert_array_equal(states, psi)   # realizations independent of the partition
    np.testing.assert_allclose(diag / R, orc.joint_distribution(psi), rtol=1e-14, atol=1e-18)
    assert merged["event_count"] == stats.event_count
    assert merged["corrections"] == stats.corrections
    assert merged["max_deviation"] == stats.max_deviation
    assert merged["events"] == sorted(stats.events, key=lambda e: (e[3], e[2]))[:100]


def _limb_worker(rank, world, port, out_q):
    """One rank of the exact-limb reduction run() uses: oracle states of this
    rank's shard -> int64 limbs -> all-reduce (SUM) -> diagonal."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ctqw_oracle as orc
        from paper_1612_00746_b200 import sharding
        from tests import fixed_point as fx

        n, m, R, steps, dt = 10, 2, 11, 12, 0.08
        lo, hi = sharding.shard_bounds(R, world, rank)
        noise = np.stack([np.random.default_rng((1234, r)).choice(np.array([-0.1, 0.1]), 2 * n)
                          for r in range(lo, hi)])
        st = orc.make_stencil(m, n, 0.1, 1.0, 0.4, link=noise[:, :n], site=noise[:, n:], batch=hi - lo)
        psi = np.tile(orc.product_state(m, n), (hi - lo, 1))
        psi, stats = orc.evolve_segment(st, psi, 0, steps, dt, r0=lo)
        acc = torch.tensor(fx.limbs(psi))
        sharding.allreduce_sum_(acc)
        local = {"event_count": stats.event_count, "corrections": stats.corrections,
                 "max_deviation": stats.max_deviation, "events": stats.events, "failure": None}
        merged = sharding.merge_segment_stats(sharding.gather_stats(local))
        if rank == 0:
            out_q.put((fx.to_double(acc.numpy()), merged))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(400)
def test_limb_reduction_bitwise_identical_for_world_1_2_3():
    """The diagonal run() reduces (exact int64 limbs, all-reduced) is the same
    bits for 1, 2 and 3 ranks, and so are the merged norm statistics -- the
    reference's promise across worker counts (pkg/README.md:174-180,
    tests/test_ensemble.py:437-455)."""
    ctx = mp.get_context("spawn")
    results = {}
    for world in (1, 2, 3):
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_limb_worker, args=(r, world, port, q)) for r in range(world)]
        for pr in procs:
            pr.start()
        results[world] = q.get(timeout=300)
        for pr in procs:
            pr.join(timeout=60)
            assert pr.exitcode == 0
    d1, m1 = results[1]
    assert m1["corrections"] > 0  # renormalisations exercised
    for world in (2, 3):
        dw, mw = results[world]
        np.testing.assert_array_equal(dw, d1)
        assert mw == m1
