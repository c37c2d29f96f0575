// Dynamic (random-telegraph) noise on the device: the reference's
// NoiseProcess (noise.py:71-206) for rate > 0, bit-compatible with NumPy.
//
// Per realization r the reference keeps a private Generator
// default_rng((master_seed, r)) and
//   init:    values = rng.choice(levels, total)                (noise.py:150)
//            next_switch = rng.exponential(1/rate, total)      (noise.py:157)
//   advance: t_end = time + dt; idx = nonzero(next_switch <= t_end)
//            while idx: values[idx] = rng.choice(levels, |idx|)
//                       next_switch[idx] += rng.exponential(1/rate, |idx|)
//                       idx = idx[next_switch[idx] <= t_end]   (noise.py:186-199)
//            time = t_end
// and the Hamiltonian entries riding changed elements are rewritten
// (hamiltonian.py:164-192; equal to a fresh assembly: hop = t + xi_link,
// site = xi_site).  _evolve_segment advances every realization after each
// step's norm check (ensemble.py:536-544), so step s sees the noise after
// s-1 advances.
//
// One thread per realization initialises; one warp per realization advances:
// the lanes compact the due elements in index order (ballot + prefix), lane 0
// replays the generator calls in the reference's order, and the lanes then
// rewrite the coefficients of elements whose value changed.
#include "ctqw_device.cuh"
#include "kernels.h"
#include "numpy_rng.cuh"

namespace ctqw {

namespace {

using namespace rng;

__global__ void telegraph_init_kernel(uint64_t master_seed, int64_t r0, int64_t count,
                                      const double* __restrict__ levels, int n_levels, int64_t total,
                                      double mean_wait, double* __restrict__ values,
                                      double* __restrict__ next_switch, TelegraphGen* __restrict__ gen) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  Pcg64 g;
  seed_pcg64(master_seed, (uint64_t)(r0 + i), g);
  double* v = values + i * total;
  double* ns = next_switch + i * total;
  U32Cache c{0u, 0};
  if (n_levels == 1) {
    for (int64_t k = 0; k < total; ++k) v[k] = levels[0];
  } else {
    const Bounded32 b((uint32_t)(n_levels - 1));
    for (int64_t k = 0; k < total; ++k) v[k] = levels[b.draw(g, c)];
  }
  for (int64_t k = 0; k < total; ++k) ns[k] = __dmul_rn(mean_wait, standard_exponential(g));
  TelegraphGen t;
  t.state_lo = (uint64_t)g.state;
  t.state_hi = (uint64_t)(g.state >> 64);
  t.inc_lo = (uint64_t)g.inc;
  t.inc_hi = (uint64_t)(g.inc >> 64);
  t.u32 = c.value;
  t.has_u32 = c.has;
  t.time = 0.0;
  t.switches = 0;
  gen[i] = t;
}

constexpr int kAdvWarps = 4;

// Per-realization due lists in a global scratch owned by the handle:
// lists[r] = [current list | original due list] (2 x total ints) and
// oldv[r] = the original values (total doubles), whose comparison with the
// new values decides "changed".  Global (L1/L2-resident) rather than shared
// memory, so any lattice size works (N*K + N elements per realization).
__global__ void __launch_bounds__(32 * kAdvWarps) telegraph_advance_kernel(
    int64_t count, int64_t total, int64_t n_links, int64_t n_sites, int n, double dt,
    const double* __restrict__ levels, int n_levels, double mean_wait, const double* __restrict__ t_slot, int K,
    double* __restrict__ values, double* __restrict__ next_switch, TelegraphGen* __restrict__ gen,
    double* __restrict__ hop, double* __restrict__ site, int64_t hop_stride, int64_t site_stride,
    int* __restrict__ lists, double* __restrict__ oldv_all, const long long* fail) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * kAdvWarps + warp;
  if (r >= count || (fail && *fail != kNoFail)) return;
  int* cur = lists + r * 2 * total;
  int* orig = cur + total;
  double* oldv = oldv_all + r * total;
  TelegraphGen t = gen[r];
  const double t_end = __dadd_rn(t.time, dt);
  double* v = values + r * total;
  double* ns = next_switch + r * total;
  // compact the due elements in index order
  int k = 0;
  for (int64_t base = 0; base < total; base += 32) {
    const int64_t e = base + lane;
    const bool due = e < total && ns[e] <= t_end;
    const unsigned m = __ballot_sync(0xffffffffu, due);
    if (due) {
      const int pos = k + __popc(m & ((1u << lane) - 1u));
      cur[pos] = (int)e;
      orig[pos] = (int)e;
      oldv[pos] = v[e];
    }
    k += __popc(m);
  }
  __syncwarp();
  const int k0 = k;
  if (k0 > 0 && lane == 0) {
    Pcg64 g;
    g.state = ((u128)t.state_hi << 64) | (u128)t.state_lo;
    g.inc = ((u128)t.inc_hi << 64) | (u128)t.inc_lo;
    U32Cache c{t.u32, t.has_u32};
    long long switches = 0;
    while (k > 0) {
      switches += k;
      if (n_levels == 1) {
        for (int q = 0; q < k; ++q) v[cur[q]] = levels[0];
      } else {
        const Bounded32 b((uint32_t)(n_levels - 1));  // one choice() call
        for (int q = 0; q < k; ++q) v[cur[q]] = levels[b.draw(g, c)];
      }
      for (int q = 0; q < k; ++q) {  // one exponential() call, then the in-place add
        const int e = cur[q];
        ns[e] = __dadd_rn(ns[e], __dmul_rn(mean_wait, standard_exponential(g)));
      }
      int kk = 0;
      for (int q = 0; q < k; ++q)
        if (ns[cur[q]] <= t_end) cur[kk++] = cur[q];
      k = kk;
    }
    t.state_lo = (uint64_t)g.state;
    t.state_hi = (uint64_t)(g.state >> 64);
    t.u32 = c.value;
    t.has_u32 = c.has;
    t.switches += switches;
  }
  __syncwarp();
  // coefficients of elements whose value changed over the window
  for (int q = lane; q < k0; q += 32) {
    const int e = orig[q];
    const double nv = v[e];
    if (nv != oldv[q]) {
      if (e < n_links) {
        if (hop) hop[r * hop_stride + e] = __dadd_rn(t_slot[e % K], nv);
      } else if (site) {
        site[r * site_stride + (e - n_links)] = nv;
      }
    }
  }
  if (lane == 0) {
    t.time = t_end;
    gen[r] = t;
  }
}

}  // namespace

cudaError_t launch_telegraph_init(uint64_t master_seed, int64_t r0, int64_t count, const double* levels_dev,
                                  int n_levels, int64_t total, double mean_wait, double* values,
                                  double* next_switch, TelegraphGen* gen, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const int bs = 64;
  telegraph_init_kernel<<<(unsigned)((count + bs - 1) / bs), bs, 0, s>>>(
      master_seed, r0, count, levels_dev, n_levels, total, mean_wait, values, next_switch, gen);
  return cudaGetLastError();
}

cudaError_t launch_telegraph_advance(int64_t count, int64_t total, int64_t n_links, int64_t n_sites, int n,
                                     double dt, const double* levels_dev, int n_levels, double mean_wait,
                                     const double* t_slot, int K, double* values, double* next_switch,
                                     TelegraphGen* gen, double* hop, double* site, int64_t hop_stride,
                                     int64_t site_stride, int* lists, double* oldv, const long long* fail,
                                     cudaStream_t s) {
  if (count <= 0 || total <= 0) return cudaSuccess;
  telegraph_advance_kernel<<<(unsigned)((count + kAdvWarps - 1) / kAdvWarps), 32 * kAdvWarps, 0, s>>>(
      count, total, n_links, n_sites, n, dt, levels_dev, n_levels, mean_wait, t_slot, K, values, next_switch, gen,
      hop, site, hop_stride, site_stride, lists, oldv, fail);
  return cudaGetLastError();
}

}  // namespace ctqw
