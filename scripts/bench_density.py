"""Dense <rho>: the triangle-only packed Gram kernel against its
FP64 roofline and against the library route it replaced (full complex128
GEMM through cuBLAS + a triangle gather).

    python scripts/bench_density.py [--dim 4096] [--realizations 100] [--reps 20]

FP64 peak: measured here as cuBLAS DGEMM throughput (torch float64 matmul,
8192^3), printed beside the nominal figure.  Flops of the packed Gram:
8 per (i, j <= i, r) complex multiply-add.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1612_00746_b200 import density  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def fp64_peak():
    n = 8192
    x = torch.randn(n, n, dtype=torch.float64, device="cuda:0")
    y = torch.randn(n, n, dtype=torch.float64, device="cuda:0")
    ms = timed(lambda: x @ y, 5)
    return 2.0 * n ** 3 / (ms / 1e3) / 1e12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=4096)
    ap.add_argument("--realizations", type=int, default=100)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    D, R = a.dim, a.realizations
    g = torch.Generator(device="cuda:0").manual_seed(7)
    stack = torch.randn((R, D), dtype=torch.complex128, device="cuda:0", generator=g)
    ms = timed(lambda: density.packed_density_device(stack, R), a.reps)
    flops = 8.0 * R * D * (D + 1) / 2

    rows, cols = torch.tril_indices(D, D, device="cuda:0")
    idx = rows * D + cols

    def library():
        gram = stack.transpose(0, 1) @ stack.conj()
        return gram.reshape(-1)[idx] / R

    ms_lib = timed(library, a.reps)
    got = density.packed_density_device(stack, R)
    err = float((got - library()).abs().max() / library().abs().max())
    peak = fp64_peak()
    tflops = flops / (ms / 1e3) / 1e12
    print(json.dumps({
        "kernel": "packed_gram_kernel (csrc/density_gram.cu)", "dim": D, "realizations": R,
        "ms": ms, "fp64_tflops": tflops, "peak_fp64_tflops_dgemm": peak, "frac_of_dgemm_peak": tflops / peak,
        "output_bytes": 16.0 * D * (D + 1) / 2, "output_gbs": 16.0 * D * (D + 1) / 2 / (ms / 1e3) / 1e9,
        "library_route_ms": ms_lib, "speedup_vs_library_route": ms_lib / ms, "max_rel_diff_vs_library": err,
    }))


if __name__ == "__main__":
    main()
