"""run() sharded over two ranks on the device (gloo process group, both ranks
on cuda:0 -- the box has one GPU), against the single-rank run().

This is the N > 1 path of the bench and of multi-GPU runs: each rank
advances its contiguous realization shard with its own handle and noise
streams seeded (master_seed, r); the collection points all-reduce the
per-rank diagonal sums as exact int64 limbs; norm statistics (one
fixed-size tensor all-gather) and the switch counts are reduced.  The rows
must equal the single-rank rows bit for bit, for 2 and 3 ranks (the
reference's promise across worker counts, pkg/README.md:174-180).
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _config(p, rate, n=24, dt=0.05, purity=True):
    obs = ("populations", "position_mean_variance", "purity", "participation_ratio")
    return p.RunConfig(space=p.JointSpace(p.build_lattice([n]), 2),
                       noise=p.NoiseSpec(target="both", levels=(-0.1, 0.1), rate=rate),
                       stepper=p.StepperConfig(backend="taylor", dt=dt),
                       realizations=7, steps=30, post_rate=10, precision="double",
                       observables=obs if purity else tuple(o for o in obs if o != "purity"))


def _worker(rank, world, port, rate, out_q, kw=None):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1612_00746_b200 as p

        torch.cuda.set_device(0)
        sinks = p.MemorySinks(keep_densities=False)
        report = p.run(_config(p, rate, **(kw or {})), sinks, group=dist.group.WORLD)
        out_q.put((rank, sinks.rows, report.norm_corrections, report.switch_count,
                   [(e.realization, e.step, e.corrected, e.deviation) for e in sinks.events]))
    except Exception as e:  # surface the failure in the parent
        out_q.put((rank, repr(e), None, None, None))
    finally:
        dist.destroy_process_group()


CASES = [
    # (rate, kw): static / telegraph noise with purity (per-segment groups),
    # and the resident N=64 kernel with the collection fused, renormalising
    (0.0, {}), (0.5, {}), (0.0, {"n": 64, "dt": 0.12, "purity": False}),
]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", CASES, ids=["static", "telegraph", "fused-n64-events"])
def test_ranks_match_one_bitwise(case, world):
    import torch.multiprocessing as mp

    import paper_1612_00746_b200 as p

    rate, kw = case
    single = p.MemorySinks(keep_densities=False)
    ref = p.run(_config(p, rate, **kw), single)

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, rate, q, kw)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = dict()
    for _ in range(world):
        rank, rows, corrections, switches, events = q.get(timeout=300)
        results[rank] = (rows, corrections, switches, events)
    for pr in procs:
        pr.join(timeout=60)
    rows, corrections, switches, events = results[0]
    assert not isinstance(rows, str), rows
    assert corrections == ref.norm_corrections
    assert switches == ref.switch_count
    assert events == [(e.realization, e.step, e.corrected, e.deviation) for e in single.events]
    assert len(rows) == len(single.rows)
    for (t0, n0, i0, v0), (t1, n1, i1, v1) in zip(rows, single.rows):
        assert (t0, n0, i0) == (t1, n1, i1)
        assert v0 == v1, (t0, n0, i0, v0, v1)
