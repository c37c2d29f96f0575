"""Where the e2e time of bench.py's run() goes (configs[2] shard by default):
one warm run, then a cProfile'd run with the device synchronised at the end."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1612_00746_b200 as p  # noqa: E402

sys.argv = ["bench.py"] + sys.argv[1:]
a = bench.parse()
cfg = bench.make_config(p, a, a.realizations, a.steps, 0)
p.run(bench.make_config(p, a, a.realizations, 3, 0), p.MemorySinks(keep_densities=False))
torch.cuda.synchronize()
for k in range(2):
    t0 = time.perf_counter()
    rep = p.run(cfg, p.MemorySinks(keep_densities=False))
    torch.cuda.synchronize()
    print(f"run {k}: {time.perf_counter() - t0:.4f} s")
pr = cProfile.Profile()
pr.enable()
t0 = time.perf_counter()
rep = p.run(cfg, p.MemorySinks(keep_densities=False))
torch.cuda.synchronize()
pr.disable()
print(f"profiled run: {time.perf_counter() - t0:.4f} s")
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
