// Static-noise draw and stencil-coefficient build (device side).
//
// The reference draws each realization's static disorder on the host with
//   np.random.default_rng((master_seed, r)).choice(levels, size=total)
// (noise.py:150-154, seed from ensemble.py:680-682).  Here one thread runs
// one realization's generator: NumPy's SeedSequence entropy mixing (4-word
// pool), PCG64 (128-bit LCG, XSL-RR output) and Generator.integers' buffered
// 32-bit Lemire bounded draw, so the values are bit-identical to NumPy's.
#include "ctqw_device.cuh"

namespace ctqw {

namespace {

constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;
constexpr int kXShift = 16;

typedef unsigned __int128 u128;

__device__ __forceinline__ uint32_t hashmix(uint32_t value, uint32_t& hc) {
  value ^= hc;
  hc *= kMultA;
  value *= hc;
  value ^= value >> kXShift;
  return value;
}

__device__ __forceinline__ uint32_t mixw(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  return r ^ (r >> kXShift);
}

// Little-endian 32-bit words of v (0 -> one zero word).
__device__ __forceinline__ int push_words(uint64_t v, uint32_t* w, int n) {
  if (v == 0) {
    w[n++] = 0;
    return n;
  }
  while (v) {
    w[n++] = (uint32_t)(v & 0xffffffffu);
    v >>= 32;
  }
  return n;
}

struct Pcg64 {
  u128 state, inc;

  __device__ __forceinline__ void step() {
    const u128 mult = ((u128)0x2360ed051fc65da4ull << 64) | (u128)0x4385df649fccf645ull;
    state = state * mult + inc;
  }
  __device__ __forceinline__ uint64_t next64() {
    step();
    const unsigned rot = (unsigned)(state >> 122);
    const uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
};

__device__ void seed_pcg64(uint64_t master_seed, uint64_t r, Pcg64& g) {
  uint32_t words[4];
  int nw = push_words(master_seed, words, 0);
  nw = push_words(r, words, nw);
  uint32_t pool[4];
  uint32_t hc = kInitA;
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < nw ? words[i] : 0u, hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mixw(pool[d], hashmix(pool[s], hc));
  // (entropy never exceeds the 4-word pool for two 64-bit seed words)
  uint32_t out32[8];
  uint32_t hb = kInitB;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= kMultB;
    v *= hb;
    v ^= v >> kXShift;
    out32[i] = v;
  }
  uint64_t s64[4];
  for (int k = 0; k < 4; ++k) s64[k] = (uint64_t)out32[2 * k] | ((uint64_t)out32[2 * k + 1] << 32);
  const u128 initstate = ((u128)s64[0] << 64) | (u128)s64[1];
  const u128 initseq = ((u128)s64[2] << 64) | (u128)s64[3];
  g.state = 0;
  g.inc = (initseq << 1) | (u128)1;
  g.step();
  g.state += initstate;
  g.step();
}

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
  const uint32_t rng = (uint32_t)(n_levels - 1);
  const uint32_t excl = rng + 1u;
  const uint32_t threshold = (0xffffffffu - rng) % excl;
  uint64_t buf = 0;
  int have = 0;
  for (int64_t k = 0; k < total; ++k) {
    uint32_t u;
    if (!have) {
      buf = g.next64();
      have = 1;
      u = (uint32_t)buf;
    } else {
      have = 0;
      u = (uint32_t)(buf >> 32);
    }
    uint64_t m = (uint64_t)u * excl;
    uint32_t leftover = (uint32_t)m;
    if (leftover < excl) {
      while (leftover < threshold) {
        if (!have) {
          buf = g.next64();
          have = 1;
          u = (uint32_t)buf;
        } else {
          have = 0;
          u = (uint32_t)(buf >> 32);
        }
        m = (uint64_t)u * excl;
        leftover = (uint32_t)m;
      }
    }
    row[k] = levels[m >> 32];
  }
}

// hop = t + xi_link (hamiltonian.py:137-141: out[...,1:] = base; += link),
// site = xi_site.  Without link noise hop = t exactly.
__global__ void build_coef_kernel(const double* __restrict__ noise, int64_t count, int n,
                                  int64_t n_links, int64_t n_sites, double t,
                                  double* __restrict__ hop, double* __restrict__ site) {
  const int64_t total = n_links + n_sites;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count * n) return;
  const int64_t r = i / n, x = i % n;
  const double* row = noise + r * total;
  hop[i] = n_links ? __dadd_rn(t, row[x]) : t;
  if (n_sites && site) site[i] = row[n_links + x];
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

cudaError_t launch_build_coef(const double* noise, int64_t count, int n, int64_t n_links,
                              int64_t n_sites, double t, double* hop, double* site,
                              cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const int64_t work = count * n;
  const int bs = 256;
  build_coef_kernel<<<(unsigned)((work + bs - 1) / bs), bs, 0, s>>>(noise, count, n, n_links,
                                                                     n_sites, t, hop, site);
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
