"""Device time of the purity overlap sums (ctqw_overlap_sumsq_points) for a
group of P points of R states of dimension D."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_1612_00746_b200.native import Handle, load_library

load_library()
h = Handle(2, 64, 0.0, 1.0, 0.0, 1.0, 0)
for R, P in ((100, 1), (100, 10), (64, 10), (124, 10), (200, 10)):
    dim = 4096
    x = torch.randn((P, R, dim), dtype=torch.complex128, device="cuda:0")
    out = torch.empty(P, dtype=torch.float64, device="cuda:0")
    for _ in range(3):
        h.overlap_sumsq_points(x, R, P, R * dim, out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20):
        h.overlap_sumsq_points(x, R, P, R * dim, out)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 20
    print(json.dumps({"R": R, "P": P, "us_per_call": round(us, 1), "us_per_point": round(us / P, 2)}))
