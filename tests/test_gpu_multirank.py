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


def _config(p, rate):
    return p.RunConfig(space=p.JointSpace(p.build_lattice([24]), 2),
                       noise=p.NoiseSpec(target="both", levels=(-0.1, 0.1), rate=rate),
                       stepper=p.StepperConfig(backend="taylor", dt=0.05),
                       realizations=7, steps=30, post_rate=10, precision="double",
                       observables=("populations", "position_mean_variance", "purity", "participation_ratio"))


def _worker(rank, world, port, rate, out_q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1612_00746_b200 as p

        torch.cuda.set_device(0)
        sinks = p.MemorySinks(keep_densities=False)
        report = p.run(_config(p, rate), sinks, group=dist.group.WORLD)
        out_q.put((rank, sinks.rows, report.norm_corrections, report.switch_count))
    except Exception as e:  # surface the failure in the parent
        out_q.put((rank, repr(e), None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("rate", [0.0, 0.5], ids=["static", "telegraph"])
def test_ranks_match_one_bitwise(rate, world):
    import torch.multiprocessing as mp

    import paper_1612_00746_b200 as p

    single = p.MemorySinks(keep_densities=False)
    ref = p.run(_config(p, rate), single)

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, rate, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = dict()
    for _ in range(world):
        rank, rows, corrections, switches = q.get(timeout=300)
        results[rank] = (rows, corrections, switches)
    for pr in procs:
        pr.join(timeout=60)
    rows, corrections, switches = results[0]
    assert not isinstance(rows, str), rows
    assert corrections == ref.norm_corrections
    assert switches == ref.switch_count
    assert len(rows) == len(single.rows)
    for (t0, n0, i0, v0), (t1, n1, i1, v1) in zip(rows, single.rows):
        assert (t0, n0, i0) == (t1, n1, i1)
        assert v0 == v1, (t0, n0, i0, v0, v1)
