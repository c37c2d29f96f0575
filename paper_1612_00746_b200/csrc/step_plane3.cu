// Plane-marching streaming step kernel for m = 3 particles on an N = 128 ring
// (joint dimension 2^21, BASELINE configs[4]).  One thread-block cluster of
// 16 CTAs owns one realization; the cluster marches once down the 128 x0
// planes per time step, every CTA holding an 8-row x1 band of each plane
// (128 x2 columns), so a plane of 16384 amplitudes lives in the cluster's
// distributed shared memory and registers.
//
// Pipeline (as step_band4.cu, with planes for rows): at iteration j stage k
// computes plane j-k+1 from the three-plane register window of stage k-1's
// output (own amplitudes) plus the in-plane neighbours of plane j-k+1 that
// stage k-1 published one iteration earlier.  In-plane neighbours along x2
// and inside the band along x1 come from the CTA's shared memory.  The two
// x1 rows across the band edges are pushed by the neighbouring CTAs straight
// into this CTA's halo rows with st.async (DSMEM), each push counted on this
// CTA's "full" mbarrier, so the data needs no fence to be visible.  Per
// plane: one CTA barrier (own exchange rows) and one relaxed cluster barrier
// (every CTA has consumed the halo rows the next pushes overwrite); the
// release form of the cluster arrive would cost a GPU-scope fence per plane
// (MEMBAR.ALL.GPU + ERRBAR, ~15 % of the time, profiles/r01c).
//
// Threads: 256 per CTA, thread (u, v) owns the 2x2 block x1 = 8c + 2u + {0,1},
// x2 = 2v + {0,1}.  psi planes arrive by TMA (ten 2 KB rows per plane: the
// band plus one halo row on each side, so stage 1 needs no DSMEM), 128B
// swizzled, into a 5-plane ring with one mbarrier per slot.
//
// Arithmetic is the reference's (hamiltonian.py:205-222): diagonal
// base[#coincident pairs] + ((site[x0] + site[x1]) + site[x2]), then for each
// particle p = 0, 1, 2 the +move and the -move; Taylor terms summed in order,
// RK4 stage arithmetic (propagators.py:185-193, 213-240).  EXACT rounds
// every product and sum separately (bit-identical to the reference between
// renormalisations).
#include "ctqw_device.cuh"
#include "kernels.h"

#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

namespace cg = cooperative_groups;

namespace ctqw {

namespace {

constexpr int kN3 = 128;             // lattice sites
constexpr int kCl = 16;              // CTAs per cluster (x1 bands)
constexpr int kBand = kN3 / kCl;     // x1 rows per CTA
constexpr int kTR = kBand + 2;       // ring rows per plane (band + x1 halo)
constexpr int kRing3 = 5;            // psi planes resident
constexpr int kThreads3 = 256;       // 4 x1 pairs x 64 x2 pairs
constexpr int kPB = 16;              // planes per norm block
constexpr int kNblk3 = kN3 / kPB;    // norm blocks per realization per CTA
constexpr int kRowB = kN3 * 16;      // bytes per x1 row (128 complex)
constexpr int kWrap = 4;             // planes re-read at the end of a full-ring march (NAPP)
constexpr int kPlaneB = kTR * kRowB; // ring bytes per plane
// Per-iteration single-thread duties (TMA issue, barrier arming, norm flush)
// go to a thread of an interior warp (u = 1): the edge warps already push
// and await the halo rows, and every warp waits for the slowest at the CTA
// barrier.
constexpr int kDuty3 = 64;

struct Plane3Args {
  CUtensorMap tmap;  // psi_in: (16 doubles, 16 lines, x1, count*N planes), box = one x1 row
  double2* psi_out;
  double2* side;     // in place: [cluster][kWrap][N][N] output planes 0..kWrap-1 parked until the end
  int inplace;       // psi_out == psi_in
  int64_t count;
  Coef coef;
  StencilConst k;
  double ci[4];
  double rkw[4];     // FMA-mode RK4 weights times c: c/2, c/3, c/6 (constant bank operands)
  const double* scl;
  double* partial;
  const long long* fail;
};

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ int swz3(int c) { return c ^ ((c >> 3) & 7); }
__device__ __forceinline__ int wrap3(int r) { return r & (kN3 - 1); }

__device__ __forceinline__ void mbar_wait3(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void st256b(double2* p, double2 a, double2 b) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y)
               : "memory");
}

// the thread's 2x2 block: index q = 2a + b, x1 offset a, x2 offset b
struct Quad {
  double2 c[4];
};

// planes requested ahead of the one consumed: the ring holds psi(j-1 .. j+1)
// at iteration j, RK4 also psi(j-2), and one slot is being refilled
template <bool RK4>
constexpr int pref3() {
  return RK4 ? kRing3 - 3 : kRing3 - 2;
}

// Shared memory (byte offsets from smem3): ring [kRing3][kTR][128] chunks;
// exchange [3 stages][2 parity][kBand][128] chunks; hop2 [N] (hop[y-1],
// hop[y]); site [N]; red [8] per-warp norm partials; mbarriers [kRing3 + 6].
// After the exchange: halo [3 stages][2 parity][2 sides][128] chunks, the x1
// rows across the band edges, pushed there by the neighbouring CTAs.
extern __shared__ __align__(1024) double2 smem3[];
constexpr int kXOff = kRing3 * kTR * kN3;        // exchange, in double2 units
constexpr int kXStage = 2 * kBand * kN3;
constexpr int kHaloOff = kXOff + 3 * kXStage;
constexpr int kHopOff = kHaloOff + 3 * 2 * 2 * kN3;
constexpr int kSiteOff = kHopOff + kN3;          // doubles follow, in double2 units of the base
constexpr int kBars3 = kRing3 + 6;               // ring slots, halo "full" [3 stages][2 parity]
constexpr int kSplit3 = kBars3;                   // + split-phase plane barrier [iteration parity]
constexpr size_t kSmem3 = (size_t)(kSiteOff) * 16 + (size_t)kN3 * 8 + 16 * 8 + (kBars3 + 2) * 8;

__device__ __forceinline__ double* site_tab() { return reinterpret_cast<double*>(smem3 + kSiteOff); }
__device__ __forceinline__ double* red_tab() { return site_tab() + kN3; }
__device__ __forceinline__ uint32_t bar_addr(int slot) { return s_u32(red_tab() + 16) + 8 * slot; }
// halo k (stage output index) of parity p has landed: armed locally with the
// expected bytes, completed by the neighbours' st.async pushes
__device__ __forceinline__ uint32_t full_bar(int k, int p) { return bar_addr(kRing3 + 2 * k + p); }

struct T3 {
  int u, v, c;          // x1 pair, x2 pair, cluster rank (x1 band)
  int x1a, x2a;         // first owned x1 / x2
  double h2[3];         // hop[x2a-1], hop[x2a], hop[x2a+1] (per lane: kept in registers)
  double h1[3];         // hop[x1a-1], hop[x1a], hop[x1a+1] (warp-uniform)
  double s2[2];         // site[x2a + b]
  uint32_t up_nb;       // shared::cluster address of smem3 in rank c-1 (x1 row above the band)
  uint32_t dn_nb;       // ... in rank c+1 (x1 row below the band)
};

__device__ __forceinline__ void mbar_arm3(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

// Push 16 bytes into a neighbour's shared memory; the bytes count toward the
// transaction of its mbarrier, so the data needs no fence to be seen there.
__device__ __forceinline__ void st_async16(uint32_t cluster_addr, double2 v, uint32_t cluster_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                   cluster_addr),
               "d"(v.x), "d"(v.y), "r"(cluster_bar)
               : "memory");
}

struct Piece3 {
  double2* dst;
  double2* side;  // parked planes (in place), else nullptr
  double* part;
  int64_t g0;  // plane coordinate of x0 = 0 for this realization (r * N)
  int j0, ya, yb, last_rho;
  double s;
  bool scale;
  int pend, pend2;
  int iters;  // iterations the loop executes (phase-unrolled by 3); the last pushes nothing
  int it0;    // CTA iteration count before this piece (split barrier phases)
  uint32_t* ph;
};

// Carried state.  Every stage output plane is published in full to the
// CTA's exchange buffer (the neighbours need all of it), so a window keeps
// only its oldest row in registers: the middle row is re-read from the
// exchange buffer (last iteration's parity) and the newest comes from the
// stage that just produced it.
template <int NAPP>
struct Regs3 {
  Quad old[NAPP];  // old[k]: stage-k output, row (plane) j-k-1 at iteration j; old[0] unused
  Quad acc[3];     // running sums, slot = row mod 3 (relative)
  Quad up;
  Quad m1;         // stage-1 output of the last iteration (own block), instead of re-reading it
  double2 h0w[3];  // hop2[] of the planes stage 1 read, slot = iteration phase (stages 2-4 reuse them)
  double nrm;
};

// ring element (row in the 10-row plane tile, x2 column)
__device__ __forceinline__ double2 ring_at(int slot, int row, int col) {
  return smem3[(slot * kTR + row) * kN3 + swz3(col)];
}

template <bool SC>
__device__ __forceinline__ Quad ring_quad(const T3& T, int slot, double s) {
  Quad v;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    v.c[q] = ring_at(slot, 1 + 2 * T.u + (q >> 1), 2 * T.v + (q & 1));
    if (SC) v.c[q] = rmul(s, v.c[q]);
  }
  return v;
}

// In-plane neighbours of the thread's block: x1m[b] (row x1a-1), x1p[b]
// (row x1a+2), x2m[a] (column x2a-1), x2p[a] (column x2a+2).
struct Nb {
  double2 x1m[2], x1p[2], x2m[2], x2p[2];
};

template <bool SC>
__device__ __forceinline__ Nb ring_nb(const T3& T, int slot, double s) {
  Nb nb;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    nb.x1m[t] = ring_at(slot, 2 * T.u, 2 * T.v + t);
    nb.x1p[t] = ring_at(slot, 2 * T.u + 3, 2 * T.v + t);
    nb.x2m[t] = ring_at(slot, 1 + 2 * T.u + t, wrap3(2 * T.v - 1));
    nb.x2p[t] = ring_at(slot, 1 + 2 * T.u + t, wrap3(2 * T.v + 2));
    if (SC) {
      nb.x1m[t] = rmul(s, nb.x1m[t]);
      nb.x1p[t] = rmul(s, nb.x1p[t]);
      nb.x2m[t] = rmul(s, nb.x2m[t]);
      nb.x2p[t] = rmul(s, nb.x2p[t]);
    }
  }
  return nb;
}

// exchange element of stage k (0-based output index), parity buf.  Rows are
// stored even columns first, then odd ones: every access pattern on them
// (columns 2v+b, 2v-1, 2v+2 across a warp) is then bank-conflict free,
// which the TMA swizzle is not for the +-1 shifted ones.
__device__ __forceinline__ int xoff(int k, int buf, int row, int col) {
  return kXOff + k * kXStage + (buf * kBand + row) * kN3 + (col & 1) * (kN3 / 2) + (col >> 1);
}

// halo element: stage k, parity p, side d (0: the x1 row above the band, 1:
// below), x2 column; even columns first as in the exchange rows
__device__ __forceinline__ int hoff(int k, int p, int d, int col) {
  return kHaloOff + ((k * 2 + p) * 2 + d) * kN3 + (col & 1) * (kN3 / 2) + (col >> 1);
}

__device__ __forceinline__ Nb xch_nb(const T3& T, int k, int buf) {
  Nb nb;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    nb.x2m[t] = smem3[xoff(k, buf, 2 * T.u + t, wrap3(2 * T.v - 1))];
    nb.x2p[t] = smem3[xoff(k, buf, 2 * T.u + t, wrap3(2 * T.v + 2))];
    const int cm = 2 * T.v + t;
    // rows across the band edges were pushed into the halo rows by the
    // neighbouring CTAs; u is warp-uniform, so these branches do not diverge
    nb.x1m[t] = T.u > 0 ? smem3[xoff(k, buf, 2 * T.u - 1, cm)] : smem3[hoff(k, buf, 0, cm)];
    nb.x1p[t] = T.u < 3 ? smem3[xoff(k, buf, 2 * T.u + 2, cm)] : smem3[hoff(k, buf, 1, cm)];
  }
  return nb;
}

// Push the band's edge rows of stage k's output (parity p) to the
// neighbours: u == 0 holds band row 0, the row below rank c-1's band; u == 3
// holds row kBand-1, the row above rank c+1's.
__device__ __forceinline__ void halo_push(const T3& T, int k, int p, const Quad& v) {
  if (T.u == 0) {
    const uint32_t bar = T.up_nb + (full_bar(k, p) - s_u32(smem3));
#pragma unroll
    for (int t = 0; t < 2; ++t) st_async16(T.up_nb + 16u * (uint32_t)hoff(k, p, 1, 2 * T.v + t), v.c[t], bar);
  } else if (T.u == 3) {
    const uint32_t bar = T.dn_nb + (full_bar(k, p) - s_u32(smem3));
#pragma unroll
    for (int t = 0; t < 2; ++t) st_async16(T.dn_nb + 16u * (uint32_t)hoff(k, p, 0, 2 * T.v + t), v.c[2 + t], bar);
  }
}

// Before stage k+2 of iteration i reads the halo rows of stage k's output of
// iteration i-1: the edge warps wait for the neighbours' pushes.
__device__ __forceinline__ void halo_wait(const T3& T, int k, int i) {
  if (i >= 1 && (T.u == 0 || T.u == 3)) mbar_wait3(full_bar(k, (i - 1) & 1), ((i - 1) >> 1) & 1);
}

__device__ __forceinline__ Quad xch_own(const T3& T, int k, int buf) {
  Quad v;
#pragma unroll
  for (int q = 0; q < 4; ++q) v.c[q] = smem3[xoff(k, buf, 2 * T.u + (q >> 1), 2 * T.v + (q & 1))];
  return v;
}

__device__ __forceinline__ void xch_put(const T3& T, int k, int buf, const Quad& v) {
#pragma unroll
  for (int q = 0; q < 4; ++q) smem3[xoff(k, buf, 2 * T.u + (q >> 1), 2 * T.v + (q & 1))] = v.c[q];
}

// (H z) on the block at plane r: up / mid / dn = planes r-1, r, r+1.
// out = i*ci*(H z), or with HORN psi + i*ci*(H z) (Horner-form Taylor, as
// step_band4.cu).
template <bool EXACT, bool SITE, bool HORN = false, bool RAW = false, bool ZD = false>
__device__ __forceinline__ void apply3(const T3& T, const StencilConst& K, int r, double2 h0, const Quad& up,
                                       const Quad& mid, const Quad& dn, const Nb& nb, double ci, Quad& out,
                                       const Quad* psi = nullptr) {
  // particle-0 couplings of plane r from the shared table (hop2[y] =
  // (hop[y-1], hop[y])); the x1 / x2 couplings of the thread's block live in
  // registers (T.h1, T.h2: +1.5 % over re-reading them per application)
  const double s0 = SITE ? site_tab()[r] : 0.0;
  const double* h1 = T.h1;
  const double* h2 = T.h2;
  const double* s2 = T.s2;
  double s1[2] = {0.0, 0.0};
  if (SITE) {
    s1[0] = site_tab()[T.x1a];
    s1[1] = site_tab()[T.x1a + 1];
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int a = q >> 1, b = q & 1;
    const int x1 = T.x1a + a, x2 = T.x2a + b;
    const double2 x1p = a == 1 ? nb.x1p[b] : mid.c[2 + b];
    const double2 x1m = a == 0 ? nb.x1m[b] : mid.c[b];
    const double2 x2p = b == 1 ? nb.x2p[a] : mid.c[2 * a + 1];
    const double2 x2m = b == 0 ? nb.x2m[a] : mid.c[2 * a];
    double2 h;
    if constexpr (ZD) {
      // eps0 = U = 0, no site noise: the diagonal is zero, the sum starts at
      // the first neighbour product (0 + x == x: the reference's bits)
      if (EXACT) h = madd<EXACT>(rmul(h0.y, dn.c[q]), h0.x, up.c[q]);
      else h = rmul(h0.x, up.c[q]);
    } else {
      const int cc = (r == x1) + (r == x2) + (x1 == x2);
      double v0 = K.base[cc];
      if (SITE) v0 = __dadd_rn(v0, __dadd_rn(__dadd_rn(s0, s1[a]), s2[b]));
      h = rmul(v0, mid.c[q]);
      if (EXACT) h = madd<EXACT>(h, h0.y, dn.c[q]);  // particle 0 +move (plane r+1), hop[x0]
      h = madd<EXACT>(h, h0.x, up.c[q]);        // particle 0 -move (plane r-1), hop[x0-1]
    }
    h = madd<EXACT>(h, h1[1 + a], x1p);     // particle 1 +move, hop[x1]
    h = madd<EXACT>(h, h1[a], x1m);         // particle 1 -move, hop[x1-1]
    h = madd<EXACT>(h, h2[1 + b], x2p);     // particle 2 +move, hop[x2]
    h = madd<EXACT>(h, h2[b], x2m);         // particle 2 -move, hop[x2-1]
    // FMA mode: plane r+1 last, the one input the previous stage produced in
    // this iteration (as step_band4.cu)
    if (!EXACT) h = madd<EXACT>(h, h0.y, dn.c[q]);
    if constexpr (HORN)
      out.c[q] = ifma(psi->c[q], ci, h);
    else if constexpr (RAW)
      out.c[q] = h;  // FMA-mode RK4: the caller folds i*c into its combinations
    else
      out.c[q] = times_i(ci, h);
  }
}

// FMA-mode Horner stage in two halves around the split CTA barrier: the
// terms from the thread's own registers (plane r-1, r+1 and the in-block
// in-plane neighbours) before the wait, the four in-plane neighbours other
// warps published last iteration after it (same terms as apply3, FMA order).
template <bool SITE, bool ZD>
__device__ __forceinline__ void apply3_own(const T3& T, const StencilConst& K, int r, double2 h0, const Quad& up,
                                           const Quad& mid, const Quad& dn, Quad& h) {
  const double s0 = SITE ? site_tab()[r] : 0.0;
  const double* h1 = T.h1;
  const double* h2 = T.h2;
  const double* s2 = T.s2;
  double s1[2] = {0.0, 0.0};
  if (SITE) {
    s1[0] = site_tab()[T.x1a];
    s1[1] = site_tab()[T.x1a + 1];
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int a = q >> 1, b = q & 1;
    const int x1 = T.x1a + a, x2 = T.x2a + b;
    double2 v;
    if constexpr (ZD) {
      v = rmul(h0.x, up.c[q]);
    } else {
      const int cc = (r == x1) + (r == x2) + (x1 == x2);
      double v0 = K.base[cc];
      if (SITE) v0 = __dadd_rn(v0, __dadd_rn(__dadd_rn(s0, s1[a]), s2[b]));
      v = madd<false>(rmul(v0, mid.c[q]), h0.x, up.c[q]);
    }
    // the in-block neighbours: x1 +move for a = 0, -move for a = 1; x2 likewise
    v = a == 0 ? madd<false>(v, h1[1], mid.c[2 + b]) : madd<false>(v, h1[a], mid.c[b]);
    v = b == 0 ? madd<false>(v, h2[1], mid.c[2 * a + 1]) : madd<false>(v, h2[b], mid.c[2 * a]);
    h.c[q] = madd<false>(v, h0.y, dn.c[q]);
  }
}

__device__ __forceinline__ void apply3_nb(const T3& T, int r, const Nb& nb, const Quad& h, double ci, Quad& out,
                                          const Quad& psi) {
  const double* h1 = T.h1;
  const double* h2 = T.h2;
  (void)r;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int a = q >> 1, b = q & 1;
    double2 v = h.c[q];
    v = a == 1 ? madd<false>(v, h1[1 + a], nb.x1p[b]) : madd<false>(v, h1[a], nb.x1m[b]);
    v = b == 1 ? madd<false>(v, h2[1 + b], nb.x2p[a]) : madd<false>(v, h2[b], nb.x2m[a]);
    out.c[q] = ifma(psi.c[q], ci, v);
  }
}

__device__ __forceinline__ void store3(const T3& T, Piece3& P, int rr, const Quad& o, double& nrm) {
  // in place, output planes 0..kWrap-1 would overwrite psi planes the march
  // reads again at its end (as planes N..N+3): park them
  double2* base = (P.side && rr < kWrap) ? P.side + ((int64_t)rr * kN3 + T.x1a) * kN3 + T.x2a
                                         : P.dst + ((int64_t)rr * kN3 + T.x1a) * kN3 + T.x2a;
  st256b(base, o.c[0], o.c[1]);
  st256b(base + kN3, o.c[2], o.c[3]);
#pragma unroll
  for (int q = 0; q < 4; ++q) nrm += norm2(o.c[q]);
  if ((rr + 1) % kPB == 0) {
    double v = nrm;
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) v += __shfl_down_sync(0xffffffffu, v, o2);
    const int blk = rr / kPB;
    if ((threadIdx.x & 31) == 0) red_tab()[(blk & 1) * 8 + (threadIdx.x >> 5)] = v;
    nrm = 0.0;
    P.pend = blk;
  }
}

// The warp partials of a finished norm block are written in the last stage,
// after the iteration's cluster arrive, so thread 0 adds them up only after
// the next arrive/wait pair: pend -> pend2 -> flushed.
__device__ __forceinline__ void flush_blk3(const T3& T, Piece3& P, int blk) {
  if (blk >= 0 && threadIdx.x == kDuty3) {
    const double* red = red_tab() + (blk & 1) * 8;
    double b = 0.0;
    for (int w = 0; w < kThreads3 / 32; ++w) b += red[w];
    P.part[blk * kCl + T.c] = b;
  }
}
__device__ __forceinline__ void flush3(const T3& T, Piece3& P, bool all = false) {
  flush_blk3(T, P, P.pend2);
  P.pend2 = P.pend;
  P.pend = -1;
  if (all) {
    flush_blk3(T, P, P.pend2);
    P.pend2 = -1;
  }
}

// TMA: the ten x1 rows (x1a_band - 1 .. +8, wrapped) of psi plane y into slot.
__device__ __forceinline__ void load_plane(const Plane3Args& a, const T3& T, const Piece3& P, int rho) {
  if (threadIdx.x != kDuty3) return;
  const int y = wrap3(P.j0 - 1 + rho);
  const int slot = rho % kRing3;
  const uint32_t bar = bar_addr(slot);
  const uint32_t dst0 = s_u32(smem3) + (uint32_t)slot * kPlaneB;
  const int plane = (int)(P.g0 + y);
  // no proxy fence here: the slot's generic accesses are reads, ordered by the
  // barrier every thread passed (a rescale's in-place writes fence themselves,
  // wait_plane)
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kPlaneB) : "memory");
#pragma unroll
  for (int t = 0; t < kTR; ++t) {
    const int x1 = wrap3(T.c * kBand - 1 + t);
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5}], [%6];" ::"r"(dst0 + t * kRowB),
        "l"(&a.tmap), "r"(0), "r"(0), "r"(x1), "r"(plane), "r"(bar)
        : "memory");
  }
}

// Wait for ring plane rho; if the realization carries a pending norm
// correction, scale the landed tile once in shared memory (rmul(s, psi) is
// exactly what the reference's in-place rescale stores), so the compute loop
// has a single variant.  The caller's next __syncthreads publishes the writes.
__device__ __forceinline__ void wait_plane(Piece3& P, int rho) {
  if (rho <= P.last_rho) {
    const int slot = rho % kRing3;
    mbar_wait3(bar_addr(slot), (*P.ph >> slot) & 1u);
    *P.ph ^= 1u << slot;
    if (P.scale) {
      double2* tile = smem3 + slot * kTR * kN3;
      for (int e = threadIdx.x; e < kTR * kN3; e += kThreads3) tile[e] = rmul(P.s, tile[e]);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // before TMA rewrites the slot
    }
  }
}

// End of an iteration.  The CTA barrier orders this CTA's exchange rows for
// its own warps; the halo rows reach the neighbours through st.async and
// their mbarriers, so the cluster barrier only has to say "every read of the
// halo rows pushed one iteration ago has retired" (all of them were consumed
// by this iteration's arithmetic before the arrive): a relaxed arrive, with
// no GPU-scope fence.
__device__ __forceinline__ void cluster_arrive() {
  __syncthreads();
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// Stage K (2..NAPP) of iteration j: plane j-K+1 from (old, mid, dn) =
// stage K-1's planes j-K, j-K+1, j-K+2 and the in-plane neighbours of the
// middle one.  Returns the stage's output (the next stage's dn).
template <int NAPP, bool RK4, bool SITE, bool EXACT, bool ZD, bool SC, int PH, int K>
__device__ __forceinline__ Quad plane3_stage(const Plane3Args& a, const T3& T, Piece3& P, Regs3<NAPP>& R, int i,
                                             int j, const Quad& mid, const Quad& dn, const Nb& nb, double2 h0) {
  constexpr double c16 = 1.0 / 6.0, c13 = 1.0 / 3.0;
  constexpr int s0 = ((PH - K + 1) % 3 + 3) % 3;  // acc slot of plane j-K+1
  const int buf = i & 1;
  const int rr = wrap3(j - K + 1);
  constexpr bool HORN = !RK4 && !EXACT;
  // as step_band4.cu: one DFMA per stage combination (not with on-site noise,
  // whose extra table reads would spill)
  constexpr bool RKF = RK4 && !EXACT && !SITE;
  const double ci = RK4 ? a.ci[0] : (HORN ? a.ci[NAPP - K] : a.ci[K - 1]);
  Quad tk;
  apply3<EXACT, SITE, HORN, RKF, ZD>(T, a.k, rr, h0, R.old[K - 1], mid, dn, nb, ci, tk, &R.acc[s0]);
  R.old[K - 1] = mid;
  Quad nk;
  if constexpr (RKF) {
    if constexpr (K == NAPP) {
      const int jo = j - K + 1;
#pragma unroll
      for (int q = 0; q < 4; ++q) nk.c[q] = ifma(R.acc[s0].c[q], a.rkw[2], tk.c[q]);
      if (jo >= P.ya && jo < P.yb) store3(T, P, rr, nk, R.nrm);
    } else {
      const Quad pm = ring_quad<SC>(T, (i + (K == 2 ? 0 : kRing3 - 1)) % kRing3, P.s);  // psi(j-1) / psi(j-2)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        nk.c[q] = ifma(pm.c[q], K == 2 ? a.rkw[0] : ci, tk.c[q]);
        R.acc[s0].c[q] = ifma(R.acc[s0].c[q], a.rkw[1], tk.c[q]);
      }
      xch_put(T, K - 1, buf, nk);
      if (i < P.iters - 1) halo_push(T, K - 1, buf, nk);
    }
    return nk;
  }
  if constexpr (K == NAPP) {
    const int jo = j - K + 1;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      nk.c[q] = HORN ? tk.c[q] : (RK4 ? cadd(R.acc[s0].c[q], rmul(c16, tk.c[q])) : cadd(R.acc[s0].c[q], tk.c[q]));
    if (jo >= P.ya && jo < P.yb) store3(T, P, rr, nk, R.nrm);
  } else if constexpr (HORN) {
    nk = tk;
    xch_put(T, K - 1, buf, nk);
    if (i < P.iters - 1) halo_push(T, K - 1, buf, nk);
  } else {
    if (RK4) {
      const Quad pm = ring_quad<SC>(T, (i + (K == 2 ? 0 : kRing3 - 1)) % kRing3, P.s);  // psi(j-1) / psi(j-2)
#pragma unroll
      for (int q = 0; q < 4; ++q) nk.c[q] = K == 2 ? cadd(rmul(0.5, tk.c[q]), pm.c[q]) : cadd(tk.c[q], pm.c[q]);
#pragma unroll
      for (int q = 0; q < 4; ++q) R.acc[s0].c[q] = cadd(R.acc[s0].c[q], rmul(c13, tk.c[q]));
    } else {
      nk = tk;
#pragma unroll
      for (int q = 0; q < 4; ++q) R.acc[s0].c[q] = cadd(R.acc[s0].c[q], tk.c[q]);
    }
    xch_put(T, K - 1, buf, nk);
    if (i < P.iters - 1) halo_push(T, K - 1, buf, nk);
  }
  return nk;
}

template <int NAPP, bool RK4, bool SITE, bool EXACT, bool ZD, bool SC, int PH>
__device__ __forceinline__ void plane3_iter(const Plane3Args& a, const T3& T, Piece3& P, Regs3<NAPP>& R, int i) {
  const int j = P.j0 + i;
  wait_plane(P, i + 2);
  // Orders the rescale writes of wait_plane before stage 1 reads the tile
  // (only pieces with a pending rescale pay it), and starts each piece.
  if (i == 0 || P.scale) __syncthreads();
  const int buf = i & 1;
  constexpr double c16 = 1.0 / 6.0;
  constexpr int SM1 = (PH + 2) % 3;
  const int r = wrap3(j);
  const int sl_up = i % kRing3, sl_mid = (i + 1) % kRing3, sl_dn = (i + 2) % kRing3;
  R.up = ring_quad<SC>(T, sl_up, P.s);
  const Quad psi = ring_quad<SC>(T, sl_mid, P.s);
  const Quad dn = ring_quad<SC>(T, sl_dn, P.s);
  const Nb nb = ring_nb<SC>(T, sl_mid, P.s);
  constexpr bool HORN = !RK4 && !EXACT;
  constexpr bool RKF = RK4 && !EXACT && !SITE;
  Quad t;
  // the plane's couplings: stage 1 loads them, stages 2-4 reuse them in the
  // following iterations (slot = iteration phase; stage 4's plane j-3 leaves
  // the window as plane j enters it)
  const double2 h0_4 = R.h0w[PH];
  R.h0w[PH] = smem3[kHopOff + r];
  apply3<EXACT, SITE, HORN, RKF, ZD>(T, a.k, r, R.h0w[PH], R.up, psi, dn, nb, HORN ? a.ci[NAPP - 1] : a.ci[0], t,
                                     &psi);
  const Quad mid1 = R.m1;  // t1 (arg1) of plane j-1
  Quad nt;
  if constexpr (RKF) {
    // t = H psi: arg = psi + k1/2; acc(j) = psi + k1/6 waits in t
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      nt.c[q] = ifma(psi.c[q], a.rkw[0], t.c[q]);
      t.c[q] = ifma(psi.c[q], a.rkw[2], t.c[q]);
    }
  } else if (HORN) {
    R.acc[SM1] = R.up;  // psi(j-1) joins the window for stages 2..4
    nt = t;
  } else if (RK4) {
#pragma unroll
    for (int q = 0; q < 4; ++q) nt.c[q] = cadd(rmul(0.5, t.c[q]), psi.c[q]);
#pragma unroll
    for (int q = 0; q < 4; ++q) t.c[q] = cadd(psi.c[q], rmul(c16, t.c[q]));
  } else {
    // acc(j-1) = psi(j-1) + t1(j-1); stage 2 below is its first update
#pragma unroll
    for (int q = 0; q < 4; ++q) R.acc[SM1].c[q] = cadd(R.up.c[q], mid1.c[q]);
    nt = t;
  }
  // Split-phase synchronisation: stage 1 above read only this CTA's ring.
  // Before anything is published: every thread of the CTA has finished the
  // last iteration (its exchange rows are visible, its ring and exchange
  // reads retired, its norm partials written: the arrive at the end of the
  // iteration, an mbarrier per iteration parity), and every CTA of the
  // cluster has consumed the halo rows this iteration's pushes overwrite
  // (the relaxed cluster barrier).
  // FMA-mode Horner: stage 2's terms from this thread's registers before the
  // wait too (its neighbour terms need the other warps' rows, after it)
  Quad h2own;
  if constexpr (HORN) apply3_own<SITE, ZD>(T, a.k, wrap3(j - 1), R.h0w[(PH + 2) % 3], R.old[1], mid1, nt, h2own);
  if (i > 0) {
    const int G = P.it0 + i - 1;
    mbar_wait3(bar_addr(kSplit3 + (G & 1)), (uint32_t)(G >> 1) & 1u);
    cluster_wait();
  }
  flush3(T, P);
  if (i + pref3<RK4>() + 1 <= P.last_rho) load_plane(a, T, P, i + pref3<RK4>() + 1);
  // arm the barriers that count this iteration's incoming halo pushes (their
  // previous phase, iteration i-2's pushes, was awaited last iteration)
  if (i < P.iters - 1 && threadIdx.x == kDuty3) {
#pragma unroll
    for (int k = 0; k < 3; ++k) mbar_arm3(full_bar(k, buf), 2 * kN3 * 16);
  }
  xch_put(T, 0, buf, nt);
  if (i < P.iters - 1) halo_push(T, 0, buf, nt);
  R.m1 = nt;
  // the halo rows of all three stages were pushed during the neighbours'
  // previous iteration: wait for them together, so the stages below run as
  // one block of straight-line code
  halo_wait(T, 0, i);
  halo_wait(T, 1, i);
  halo_wait(T, 2, i);
  Quad t2;
  if constexpr (HORN) {
    apply3_nb(T, wrap3(j - 1), xch_nb(T, 0, buf ^ 1), h2own, a.ci[NAPP - 2], t2, R.acc[SM1]);
    R.old[1] = mid1;
    xch_put(T, 1, buf, t2);
    if (i < P.iters - 1) halo_push(T, 1, buf, t2);
  } else {
    t2 = plane3_stage<NAPP, RK4, SITE, EXACT, ZD, SC, PH, 2>(a, T, P, R, i, j, mid1, nt, xch_nb(T, 0, buf ^ 1),
                                                             R.h0w[(PH + 2) % 3]);
  }
  const Quad t3 = plane3_stage<NAPP, RK4, SITE, EXACT, ZD, SC, PH, 3>(a, T, P, R, i, j, xch_own(T, 1, buf ^ 1), t2,
                                                                  xch_nb(T, 1, buf ^ 1), R.h0w[(PH + 1) % 3]);
  plane3_stage<NAPP, RK4, SITE, EXACT, ZD, SC, PH, NAPP>(a, T, P, R, i, j, xch_own(T, NAPP - 2, buf ^ 1), t3,
                                                     xch_nb(T, NAPP - 2, buf ^ 1), h0_4);
  if (RK4) R.acc[PH] = t;
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar_addr(kSplit3 + ((P.it0 + i) & 1)))
               : "memory");
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
}

template <int NAPP, bool RK4, bool SITE, bool EXACT, bool ZD, bool SC>
__device__ __forceinline__ void plane3_loop(const Plane3Args& a, const T3& T, Piece3& P, Regs3<NAPP>& R,
                                            int iters) {
#pragma unroll 1
  for (int i = 0; i < iters; i += 3) {
    plane3_iter<NAPP, RK4, SITE, EXACT, ZD, SC, 0>(a, T, P, R, i);
    plane3_iter<NAPP, RK4, SITE, EXACT, ZD, SC, 1>(a, T, P, R, i + 1);
    plane3_iter<NAPP, RK4, SITE, EXACT, ZD, SC, 2>(a, T, P, R, i + 2);
  }
}

template <int NAPP, bool RK4, bool SITE, bool EXACT, bool ZD>
__global__ void __launch_bounds__(kThreads3, 1) plane3_kernel(const __grid_constant__ Plane3Args a) {
  static_assert(NAPP == 4, "plane3 pipelines four applications (Taylor-4 / RK4)");
  cg::cluster_group cluster = cg::this_cluster();
  const bool failed = *a.fail != kNoFail;  // uniform over the grid
  if (failed) return;
  if ((s_u32(smem3) & 1023u) != 0) __trap();  // TMA 128B swizzle needs 1024-byte aligned slots
  T3 T;
  T.c = (int)cluster.block_rank();
  T.u = threadIdx.x >> 6;
  T.v = threadIdx.x & 63;
  T.x1a = T.c * kBand + 2 * T.u;
  T.x2a = 2 * T.v;
  {
    const uint32_t base = s_u32(smem3);
    uint32_t up, dn;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(up) : "r"(base), "r"((T.c + kCl - 1) % kCl));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dn) : "r"(base), "r"((T.c + 1) % kCl));
    T.up_nb = up;
    T.dn_nb = dn;
  }
  uint32_t ph_bits = 0;
  if (threadIdx.x == 0) {
    for (int q = 0; q < kBars3; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar_addr(q)), "r"(1) : "memory");
    for (int q = 0; q < 2; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar_addr(kSplit3 + q)), "r"(kThreads3) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  int it0 = 0;
  // the cluster's run of (realization, x0 block) work items; in place, whole
  // realizations only (a split realization would overwrite another piece's halo)
  const int64_t nclus = gridDim.x / kCl;
  const int64_t gid = blockIdx.x / kCl;
  const int64_t total = a.count * kNblk3;
  int64_t lo, hi;
  if (a.inplace) {
    lo = (a.count * gid / nclus) * kNblk3;
    hi = (a.count * (gid + 1) / nclus) * kNblk3;
  } else {
    lo = total * gid / nclus;
    hi = total * (gid + 1) / nclus;
  }
  double2* hop2 = smem3 + kHopOff;
  double* site = site_tab();
  constexpr int64_t dim = (int64_t)kN3 * kN3 * kN3;
  while (lo < hi) {
    const int64_t r = lo / kNblk3;
    const int b0 = (int)(lo % kNblk3);
    const int nb = (int)std::min<int64_t>(hi - lo, kNblk3 - b0);
    lo += nb;
    Piece3 P;
    P.ya = b0 * kPB;
    P.yb = (b0 + nb) * kPB;
    const double* hop = a.coef.hop + r * a.coef.stride;
    const double* sg = SITE ? a.coef.site + r * a.coef.stride : nullptr;
    cluster_sync_all();  // previous piece finished everywhere (tables, ring, exchange)
    for (int y = threadIdx.x; y < kN3; y += kThreads3) {
      hop2[y] = make_double2(hop[wrap3(y - 1)], hop[y]);
      if (SITE) site[y] = sg[y];
    }
#pragma unroll
    for (int t = 0; t < 3; ++t) T.h2[t] = hop[wrap3(T.x2a - 1 + t)];
#pragma unroll
    for (int t = 0; t < 3; ++t) T.h1[t] = hop[wrap3(T.x1a - 1 + t)];
#pragma unroll
    for (int t = 0; t < 2; ++t) T.s2[t] = SITE ? sg[T.x2a + t] : 0.0;
    P.s = a.scl ? a.scl[r] : 1.0;
    P.scale = P.s != 1.0;
    P.dst = a.psi_out + r * dim;
    P.side = a.inplace ? a.side + gid * (int64_t)kWrap * kN3 * kN3 : nullptr;
    P.part = a.partial + r * (kNblk3 * kCl);
    P.g0 = r * kN3;
    P.pend = -1;
    P.pend2 = -1;
    P.ph = &ph_bits;
    P.j0 = P.ya - NAPP + 1;
    const int iters = (P.yb - P.ya) + 2 * (NAPP - 1);
    P.iters = (iters + 2) / 3 * 3;
    P.it0 = it0;
    it0 += P.iters;
    P.last_rho = iters + 1;
    for (int rho = 0; rho <= pref3<RK4>(); ++rho)
      if (rho <= P.last_rho) load_plane(a, T, P, rho);
    wait_plane(P, 0);
    wait_plane(P, 1);
    __syncthreads();
    Regs3<NAPP> R;
#pragma unroll
    for (int k = 0; k < NAPP; ++k)
#pragma unroll
      for (int q = 0; q < 4; ++q) R.old[k].c[q] = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < 4; ++q) R.m1.c[q] = make_double2(0.0, 0.0);
#pragma unroll
    for (int w = 0; w < 3; ++w)
#pragma unroll
      for (int q = 0; q < 4; ++q) R.acc[w].c[q] = make_double2(0.0, 0.0);
#pragma unroll
    for (int w = 0; w < 3; ++w) R.h0w[w] = make_double2(0.0, 0.0);
    R.nrm = 0.0;
    plane3_loop<NAPP, RK4, SITE, EXACT, ZD, false>(a, T, P, R, iters);  // ring tiles arrive pre-scaled
    cluster_wait();   // completes the last iteration's arrive
    __syncthreads();  // the last stage has written its norm partials
    flush3(T, P, true);
    // every halo push of the piece has been awaited: restart the halo
    // barriers at phase 0 for the next piece (published by its cluster barrier)
    if (threadIdx.x == 0) {
      for (int q = kRing3; q < kBars3; ++q) {
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(bar_addr(q)) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar_addr(q)), "r"(1) : "memory");
      }
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (P.side) {
      // every CTA has read planes 0..kWrap-1 (its band and halo rows) for the
      // last time: move the parked output planes in; each thread copies the
      // elements it parked itself, so program order suffices
      cluster_sync_all();
      for (int pl = 0; pl < kWrap; ++pl)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t off = ((int64_t)pl * kN3 + T.x1a + (q >> 1)) * kN3 + T.x2a + (q & 1);
          P.dst[off] = P.side[off];
        }
    }
  }
  cluster_sync_all();  // no CTA leaves while a neighbour may still read its exchange planes
}

int sm_count3() {
  static int v = 0;
  if (v == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
  }
  return v;
}

cudaError_t encode_planes_map(CUtensorMap* map, const double2* base, int64_t count) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!encode) return cudaErrorNotSupported;
  if (count * kN3 > 0x7fffffffLL) return cudaErrorInvalidValue;
  const cuuint64_t dims[4] = {16, kN3 / 8, kN3, (cuuint64_t)(count * kN3)};
  const cuuint64_t strides[3] = {128, (cuuint64_t)kRowB, (cuuint64_t)kRowB * kN3};
  const cuuint32_t box[4] = {16, kN3 / 8, 1, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double2*>(base), dims, strides, box,
                            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Parking space for the in-place march: kWrap planes per cluster, per device.
double2* side_buffer(int nclus) {
  static double2* buf[64] = {};
  static int cap[64] = {};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (nclus > cap[dev]) {
    if (buf[dev]) cudaFree(buf[dev]);
    buf[dev] = nullptr;
    cap[dev] = 0;
    if (cudaMalloc(&buf[dev], (size_t)nclus * kWrap * kN3 * kN3 * sizeof(double2)) != cudaSuccess) return nullptr;
    cap[dev] = nclus;
  }
  return buf[dev];
}

template <int NAPP, bool RK4, bool SITE, bool EXACT, bool ZD>
cudaError_t launch_p3(Plane3Args a, const double2* psi_in, cudaStream_t s) {
  auto kern = plane3_kernel<NAPP, RK4, SITE, EXACT, ZD>;
  static int nclus_dev[64] = {};
  int& nclus = nclus_dev[current_device() & 63];
  if (nclus == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem3);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kCl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(kCl * 64, 1, 1);
    cfg.blockDim = dim3(kThreads3, 1, 1);
    cfg.dynamicSmemBytes = kSmem3;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
    if (e != cudaSuccess) return e;
    if (n < 1) return cudaErrorInvalidConfiguration;
    nclus = n;
  }
  cudaError_t e = encode_planes_map(&a.tmap, psi_in, a.count);
  if (e != cudaSuccess) return e;
  const int64_t work = a.inplace ? a.count : a.count * kNblk3;
  const int64_t clusters = std::min<int64_t>(nclus, work);
  if (a.inplace) {
    a.side = side_buffer((int)clusters);
    if (!a.side) return cudaErrorMemoryAllocation;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)(clusters * kCl), 1, 1);
  cfg.blockDim = dim3(kThreads3, 1, 1);
  cfg.dynamicSmemBytes = kSmem3;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

}  // namespace

bool plane3_supported(int m, int n, const StepScalars& sc) {
  return m == 3 && n == kN3 && (sc.backend == 1 || sc.order == 4);
}

int plane3_parts() { return kNblk3 * kCl; }

cudaError_t launch_plane3_step(const double2* psi_in, double2* psi_out, int64_t count, const Coef& coef,
                               const StencilConst& k, const StepScalars& sc, bool exact, const double* scl,
                               double* partial, const long long* fail, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  Plane3Args a;
  a.psi_out = psi_out;
  a.inplace = psi_out == psi_in ? 1 : 0;
  a.side = nullptr;
  a.count = count;
  a.coef = coef;
  a.k = k;
  for (int i = 0; i < 4; ++i) a.ci[i] = sc.ci[i];
  a.rkw[0] = 0.5 * sc.ci[0];
  a.rkw[1] = sc.ci[0] * (1.0 / 3.0);
  a.rkw[2] = sc.ci[0] * (1.0 / 6.0);
  a.rkw[3] = 0.0;
  a.scl = scl;
  a.partial = partial;
  a.fail = fail;
  const bool site = coef.site != nullptr;
  const bool rk4 = sc.backend == 1;
  // eps0 = U = 0 and no site noise (configs[4]): zero diagonal
  const bool zd = !site && k.base[0] == 0.0 && k.base[1] == 0.0 && k.base[2] == 0.0 && k.base[3] == 0.0;
  if (rk4) {
    if (site) return exact ? launch_p3<4, true, true, true, false>(a, psi_in, s)
                           : launch_p3<4, true, true, false, false>(a, psi_in, s);
    if (zd) return exact ? launch_p3<4, true, false, true, true>(a, psi_in, s)
                         : launch_p3<4, true, false, false, true>(a, psi_in, s);
    return exact ? launch_p3<4, true, false, true, false>(a, psi_in, s) : launch_p3<4, true, false, false, false>(a, psi_in, s);
  }
  if (site) return exact ? launch_p3<4, false, true, true, false>(a, psi_in, s)
                         : launch_p3<4, false, true, false, false>(a, psi_in, s);
  if (zd) return exact ? launch_p3<4, false, false, true, true>(a, psi_in, s)
                       : launch_p3<4, false, false, false, true>(a, psi_in, s);
  return exact ? launch_p3<4, false, false, true, false>(a, psi_in, s) : launch_p3<4, false, false, false, false>(a, psi_in, s);
}

}  // namespace ctqw
