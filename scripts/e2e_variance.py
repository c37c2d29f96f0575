import sys, time, gc
sys.path.insert(0, '.')
import torch
import bench
import paper_1612_00746_b200 as p
sys.argv = ['bench.py']
a = bench.parse()
cfg = bench.make_config(p, a, a.realizations, a.steps, 0)
p.run(bench.make_config(p, a, a.realizations, 5, 0), p.MemorySinks(keep_densities=False))
for k in range(8):
    gc.collect(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = p.run(cfg, p.MemorySinks(keep_densities=False))
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    st = rep.profile.as_dict()
    print(f"{t:.4f}", {k2: round(v['seconds'], 4) if isinstance(v, dict) else v for k2, v in st.items()}, round(rep.io_seconds, 4))
