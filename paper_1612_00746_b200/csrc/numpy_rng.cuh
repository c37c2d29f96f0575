// NumPy-compatible random streams on the device (shared by noise.cu and
// telegraph.cu): SeedSequence entropy mixing with a 4-word pool, PCG64
// (128-bit LCG, XSL-RR output), Generator.integers' buffered 32-bit Lemire
// bounded draw, and random_standard_exponential's 256-level ziggurat.  The
// published algorithms of NumPy 2.x (numpy/random/bit_generator.pyx,
// src/pcg64/pcg64.h, src/distributions/distributions.c), restated; the
// ziggurat constants are NumPy's own (ziggurat_tables.h).
#pragma once

#include <cstdint>

#include "ziggurat_tables.h"

namespace ctqw {
namespace rng {

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

__device__ __forceinline__ void seed_pcg64(uint64_t master_seed, uint64_t r, Pcg64& g) {
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

// Generator.integers(0, rng + 1) / choice: 32-bit Lemire with rejection on
// next_uint32.  PCG64's next_uint32 hands out the low half of a 64-bit output
// and caches the high half in the bit generator (has_uint32 / uinteger in
// numpy/random/src/pcg64/pcg64.h), so the cache persists across calls and is
// untouched by next_uint64 draws (exponential); callers keep it with the state.
struct U32Cache {
  uint32_t value;
  int has;
};

__device__ __forceinline__ uint32_t next_u32(Pcg64& g, U32Cache& c) {
  if (c.has) {
    c.has = 0;
    return c.value;
  }
  const uint64_t next = g.next64();
  c.has = 1;
  c.value = (uint32_t)(next >> 32);
  return (uint32_t)next;
}

struct Bounded32 {
  uint32_t rng, excl, threshold;
  __device__ __forceinline__ explicit Bounded32(uint32_t r)
      : rng(r), excl(r + 1u), threshold((0xffffffffu - r) % (r + 1u)) {}
  __device__ __forceinline__ uint32_t draw(Pcg64& g, U32Cache& c) const {
    uint64_t m = (uint64_t)next_u32(g, c) * excl;
    uint32_t leftover = (uint32_t)m;
    if (leftover < excl) {
      while (leftover < threshold) {
        m = (uint64_t)next_u32(g, c) * excl;
        leftover = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
};

__device__ __forceinline__ double next_double(Pcg64& g) {
  return (double)(g.next64() >> 11) * (1.0 / 9007199254740992.0);
}

// random_standard_exponential: ziggurat fast path (98.9 %), else the wedge
// test against exp(-x) or, for the base strip, the tail r - log1p(-U).  Every
// product and sum rounded separately, as the x86-64 build of NumPy does.
// exp / log1p are CUDA's (<= 1 ulp); they only enter the rare slow paths.
__device__ __forceinline__ double standard_exponential(Pcg64& g) {
  for (;;) {
    uint64_t ri = g.next64();
    ri >>= 3;
    const int idx = (int)(ri & 0xff);
    ri >>= 8;
    const double x = __dmul_rn((double)ri, kZigWe[idx]);
    if (ri < kZigKe[idx]) return x;
    if (idx == 0) return __dsub_rn(kZigExpR, log1p(-next_double(g)));
    const double f = __dadd_rn(__dmul_rn(__dsub_rn(kZigFe[idx - 1], kZigFe[idx]), next_double(g)), kZigFe[idx]);
    if (f < exp(-x)) return x;
  }
}

}  // namespace rng
}  // namespace ctqw
