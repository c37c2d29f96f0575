// Static-noise draw and stencil-coefficient build (device side).
//
// The reference draws each realization's static disorder on the host with
//   np.random.default_rng((master_seed, r)).choice(levels, size=total)
// (noise.py:150-154, seed from ensemble.py:680-682).  Here one thread runs
// one realization's generator: NumPy's SeedSequence entropy mixing (4-word
// pool), PCG64 (128-bit LCG, XSL-RR output) and Generator.integers' buffered
// 32-bit Lemire bounded draw, so the values are bit-identical to NumPy's.
#include "ctqw_device.cuh"
#include "numpy_rng.cuh"

namespace ctqw {

namespace {

using namespace rng;

__global__ void draw_noise_kernel(uint64_t master_seed, int64_t r0, int64_t count,
                                  const double* __restrict__ levels, int n_levels, int64_t total,
                                  double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double* row = out + i * total;
  if (n_levels == 1) {  // rng == 0: no draws consumed
    for (int64_t k = 0; k < total; ++k) row[k] = levels[0];
    return;
  }
  Pcg64 g;
  seed_pcg64(master_seed, (uint64_t)(r0 + i), g);
  const Bounded32 b((uint32_t)(n_levels - 1));
  U32Cache c{0u, 0};  // a fresh generator has no cached half
  for (int64_t k = 0; k < total; ++k) row[k] = levels[b.draw(g, c)];
}

// hop = t_dir + xi_link (hamiltonian.py:137-141: out[...,1:] = base; += link),
// site = xi_site.  Links are laid out x*K + s (hilbert.py:311); slot s has
// the tunnelling t_slot[s] of its direction.  Without link noise hop = t.
__global__ void build_coef_kernel(const double* __restrict__ noise, int64_t count, int n, int K,
                                  int64_t n_links, int64_t n_sites, const double* __restrict__ t_slot,
                                  double* __restrict__ hop, double* __restrict__ site) {
  const int64_t total = n_links + n_sites;
  const int64_t nk = (int64_t)n * K;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count * nk) return;
  const int64_t r = i / nk, l = i % nk;
  const double* row = noise + r * total;
  const double t = t_slot[l % K];
  hop[i] = n_links ? __dadd_rn(t, row[l]) : t;
  if (n_sites && site && l < n) site[r * n + l] = row[n_links + l];
}

__global__ void fill_states_kernel(double2* __restrict__ psi, int64_t count, int64_t dim,
                                   const double2* __restrict__ psi0) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count * dim) return;
  psi[i] = psi0[i % dim];
}

}  // namespace

cudaError_t launch_draw_noise(uint64_t master_seed, int64_t r0, int64_t count,
                              const double* levels_dev, int n_levels, int64_t total,
                              double* out, cudaStream_t s) {
  if (count <= 0 || total <= 0) return cudaSuccess;
  const int bs = 128;
  draw_noise_kernel<<<(unsigned)((count + bs - 1) / bs), bs, 0, s>>>(master_seed, r0, count,
                                                                      levels_dev, n_levels, total, out);
  return cudaGetLastError();
}

cudaError_t launch_build_coef(const double* noise, int64_t count, int n, int K, int64_t n_links,
                              int64_t n_sites, const double* t_slot, double* hop, double* site,
                              cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const int64_t work = count * n * K;
  const int bs = 256;
  build_coef_kernel<<<(unsigned)((work + bs - 1) / bs), bs, 0, s>>>(noise, count, n, K, n_links, n_sites, t_slot,
                                                                     hop, site);
  return cudaGetLastError();
}

cudaError_t launch_fill_states(double2* psi, int64_t count, int64_t dim, const double2* psi0,
                               cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const int64_t work = count * dim;
  const int bs = 256;
  fill_states_kernel<<<(unsigned)((work + bs - 1) / bs), bs, 0, s>>>(psi, count, dim, psi0);
  return cudaGetLastError();
}

}  // namespace ctqw
