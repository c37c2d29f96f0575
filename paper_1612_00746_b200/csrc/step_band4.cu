// Row-marching streaming step kernel for m = 2, four columns per thread,
// lag-1 stage pipeline, persistent balanced row-block schedule.
//
// Why another band kernel.  The one- and two-column kernels (step_band.cu,
// step_band2.cu) are bound by shared memory (ncu: 1.5-2.6 wavefronts per
// element-step, L1/TEX 66-85 % busy) and by latency at 8-16 warps/SM.  Here
// each thread owns four adjacent columns, so per stencil application it
// publishes only its two edge values and reads one value from each
// neighbouring thread: 8 B/element of shared-memory traffic per application
// instead of 24-48.  Per step that is ~0.7 wavefronts per element; the FP64
// pipe (56-88 DFMA/DMUL/DADD per element) becomes the on-chip limit, which
// is below the HBM time of 32 B/element.
//
// Pipeline.  At iteration j stage k (1-based) computes row j-k+1, so stage k
// consumes the row stage k-1 produced in the same iteration (from registers,
// own columns) and the neighbour columns of row j-k+1 that stage k-1
// published one iteration earlier (shared memory, double-buffered by
// iteration parity).  One __syncthreads per row.  Each stage input keeps a
// three-row register window (rows r-1, r, r+1) and the running Taylor sum
// keeps three rows; both rotate with period three, so the loop is unrolled
// by three with compile-time register slots and no moves.
//
//   stage 1:  t1(j)   from psi(j-1), psi(j) [registers], psi(j+1) [ring]
//   stage k:  t_k(j-k+1) from t_{k-1}(j-k), t_{k-1}(j-k+1), t_{k-1}(j-k+2)
//   last:     out(j-n+1) = acc + t_n -> HBM, |out|^2 -> norm partial
//
// psi rows stream in through an 8-row cp.async ring: lanes fetch contiguous
// 16-byte chunks (coalesced) and write them XOR-swizzled
// (chunk c -> c ^ ((c >> 3) & 7)) so that a thread's four-column reads and
// the neighbour reads are bank-conflict free.  Finished rows leave from
// registers as two 256-bit stores per thread.
//
// Schedule.  The realization x row space is cut into blocks of kRB rows.  A
// persistent grid (CTAs resident per SM x SMs) takes equal contiguous runs
// of blocks, so there is no tail wave; a run crossing realizations is
// processed as one piece per realization, each piece paying 2(n-1) ramp
// rows.  Norm partials are per row block, summed in a fixed order, so the
// norm does not depend on the schedule (or on the realization count).
//
// Arithmetic is the reference's (hamiltonian.py:205-222,
// propagators.py:185-193 / 213-240): diagonal, +move/-move of particle 0,
// +move/-move of particle 1; Taylor terms summed ((((psi+t1)+t2)+t3)+t4);
// RK4's stage arithmetic with the rounded 1/6, 1/3 constants.  EXACT keeps
// every product and sum separately rounded (bit-identical to the reference
// between renormalisations); otherwise neighbour terms contract into DFMA.
#include "ctqw_device.cuh"
#include "kernels.h"

#include <algorithm>
#include <cstdlib>

namespace ctqw {

namespace {

constexpr int kCols = 4;        // columns per thread
constexpr int kRing4 = 8;       // psi rows resident
constexpr int kPref4 = 5;       // rows requested ahead of the one consumed
constexpr int kRB = 32;         // rows per norm block
constexpr int kMaxThreads4 = 256;

struct Band4Args {
  const double2* psi_in;
  double2* psi_out;
  int n;
  int npad;         // ring row stride in 16-byte chunks (n rounded up to 8)
  int rb;           // rows per norm block
  int nblk;         // norm blocks per realization (= nparts)
  int64_t total;    // count * nblk
  int64_t count;
  Coef coef;
  StencilConst k;
  double ci[4];
  const double* scl;
  double* partial;
  const long long* fail;
};

__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ int swz(int c) { return c ^ ((c >> 3) & 7); }

__device__ __forceinline__ void st256(double2* p, double2 a, double2 b) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x),
               "d"(b.y)
               : "memory");
}

struct Row4 {
  double2 c[kCols];
};

// Compile-time geometry when NN > 0 (the BASELINE lattice sizes), else runtime.
template <int NN>
struct Geo4 {
  int n_, npad_, rb_;
  __device__ __forceinline__ int n() const { return NN > 0 ? NN : n_; }
  __device__ __forceinline__ int np() const { return n() / kCols; }
  __device__ __forceinline__ int npad() const { return NN > 0 ? ((NN + 7) & ~7) : npad_; }
  __device__ __forceinline__ int rb() const { return NN > 0 ? (NN % kRB == 0 ? kRB : NN) : rb_; }
  __device__ __forceinline__ int wrap(int r) const { return r < 0 ? r + n() : (r >= n() ? r - n() : r); }
};

// Per-thread constants and per-piece state.  Shared memory is addressed by
// element offsets into smem4 (32-bit shared addressing).
struct T4 {
  int p, pl, pr;
  int off[kCols];     // swizzled ring offsets of own columns
  int offl, offr;     // swizzled ring offsets of columns 4p-1 and 4p+4
  double hc[kCols];   // hop[x]      (particle 1 +move coupling)
  double hm0;         // hop[4p-1]   (particle 1 -move coupling of column 0)
  double sx[kCols];   // site[x]
};

struct Piece4 {
  const double2* src;
  double2* dst;
  double* part;       // partial + r * nblk
  int j0, ya, yb, last_rho;
  double s;
  bool scale;
  int pend;           // norm block awaiting its flush (-1 none)
};

extern __shared__ __align__(128) double2 smem4[];

// Shared-memory layout (element offsets): ring [kRing4][npad], xl/xr
// [NX][2][NP], hop2 [n], then doubles: site [n], red [64].
template <int NN, int NAPP, bool SITE>
struct Lay4 {
  static constexpr int NX = NAPP > 1 ? NAPP - 1 : 1;
  __device__ __forceinline__ static int xl(const Geo4<NN>& g, int k, int buf) {
    return kRing4 * g.npad() + (k * 2 + buf) * g.np();
  }
  __device__ __forceinline__ static int xr(const Geo4<NN>& g, int k, int buf) {
    return kRing4 * g.npad() + NX * 2 * g.np() + (k * 2 + buf) * g.np();
  }
  __device__ __forceinline__ static int hop2(const Geo4<NN>& g) { return kRing4 * g.npad() + NX * 4 * g.np(); }
  __device__ __forceinline__ static double* site(const Geo4<NN>& g) {
    return reinterpret_cast<double*>(smem4 + hop2(g) + g.n());
  }
  __device__ __forceinline__ static double* red(const Geo4<NN>& g) { return site(g) + (SITE ? g.n() : 0); }
};

template <int NN>
__device__ __forceinline__ Row4 ring_row(const Geo4<NN>& g, const T4& T, int slot, double s, bool scale) {
  const double2* rowp = smem4 + slot * g.npad();
  Row4 v;
#pragma unroll
  for (int q = 0; q < kCols; ++q) {
    v.c[q] = rowp[T.off[q]];
    if (scale) v.c[q] = rmul(s, v.c[q]);
  }
  return v;
}

// (H z)(r, x) for the thread's four columns of row r: up = row r-1,
// mid = row r, dn = row r+1, lf / rt = columns 4p-1 / 4p+4 of row r.
template <bool EXACT, bool SITE>
__device__ __forceinline__ void apply4(const T4& T, const StencilConst& K, int r, double2 hp,
                                       double srow, const Row4& up, const Row4& mid,
                                       const Row4& dn, double2 lf, double2 rt, double ci,
                                       Row4& out) {
  const int d = r - kCols * T.p;  // diagonal column offset within the thread's four
#pragma unroll
  for (int q = 0; q < kCols; ++q) {
    double v0 = d == q ? K.base[1] : K.base[0];
    if (SITE) v0 = __dadd_rn(v0, __dadd_rn(srow, T.sx[q]));  // base + (site[x0] + site[x1])
    const double2 l = q == 0 ? lf : mid.c[q - 1];
    const double2 rr = q == kCols - 1 ? rt : mid.c[q + 1];
    const double hm = q == 0 ? T.hm0 : T.hc[q - 1];
    double2 h = rmul(v0, mid.c[q]);
    h = madd<EXACT>(h, hp.y, dn.c[q]);  // particle 0 +move: row r+1, hop[r]
    h = madd<EXACT>(h, hp.x, up.c[q]);  // particle 0 -move: row r-1, hop[r-1]
    h = madd<EXACT>(h, T.hc[q], rr);    // particle 1 +move
    h = madd<EXACT>(h, hm, l);          // particle 1 -move
    out.c[q] = times_i(ci, h);
  }
}

template <int NAPP>
struct Regs4 {
  Row4 w[NAPP][3];  // w[k], k >= 1: stage-k output window (input of stage k+1); w[0] unused
  Row4 acc[3];      // running sums, slot = row mod 3 (relative)
  Row4 psi;         // psi(j) (own columns, scaled), carried from the previous iteration
  Row4 up;          // psi(j-1): read by stage 1, reused by RK4 stage 2
  double nrm;
};

// Write one finished row (four columns) and fold |out|^2 into the norm; at
// the end of a norm block, reduce the warp's sum into shared memory (thread 0
// adds the warps in order after the next barrier).
template <int NN, int NAPP, bool SITE>
__device__ __forceinline__ void band4_store(const Geo4<NN>& g, const T4& T, Piece4& P, int rr, const Row4& o,
                                            double& nrm) {
  double2* op = P.dst + (int64_t)rr * g.n() + kCols * T.p;
  st256(op, o.c[0], o.c[1]);
  st256(op + 2, o.c[2], o.c[3]);
#pragma unroll
  for (int q = 0; q < kCols; ++q) nrm += norm2(o.c[q]);
  if ((rr + 1) % g.rb() == 0) {
    double v = nrm;
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) v += __shfl_down_sync(0xffffffffu, v, o2);
    const int blk = rr / g.rb();
    if ((T.p & 31) == 0) Lay4<NN, NAPP, SITE>::red(g)[(blk & 1) * 32 + (T.p >> 5)] = v;
    nrm = 0.0;
    P.pend = blk;
  }
}

// Stage K (2..NAPP) of iteration j: row j-K+1 from window K-1 (rows j-K ..
// j-K+2, slot(y) = (y - j0) mod 3) and the neighbour columns stage K-1
// published last iteration.
template <int NN, int NAPP, bool RK4, bool SITE, bool EXACT, int PH, int K>
__device__ __forceinline__ void band4_stage(const Band4Args& a, const Geo4<NN>& g, const T4& T, Piece4& P,
                                            Regs4<NAPP>& R, int i, int j) {
  using L = Lay4<NN, NAPP, SITE>;
  constexpr double c16 = 1.0 / 6.0, c13 = 1.0 / 3.0;
  constexpr int s0 = ((PH - K + 1) % 3 + 3) % 3;  // row j-K+1
  constexpr int sm = (s0 + 2) % 3;                // row j-K
  constexpr int sp = (s0 + 1) % 3;                // row j-K+2
  const int buf = i & 1;
  const int rr = g.wrap(j - K + 1);
  const double2 lf = smem4[L::xr(g, K - 2, buf ^ 1) + T.pl];
  const double2 rt = smem4[L::xl(g, K - 2, buf ^ 1) + T.pr];
  const double ci = RK4 ? a.ci[0] : a.ci[K - 1];
  Row4 tk;
  apply4<EXACT, SITE>(T, a.k, rr, smem4[L::hop2(g) + rr], SITE ? L::site(g)[rr] : 0.0, R.w[K - 1][sm],
                      R.w[K - 1][s0], R.w[K - 1][sp], lf, rt, ci, tk);
  if constexpr (K == NAPP) {
    const int jo = j - K + 1;
    Row4 o;
#pragma unroll
    for (int q = 0; q < kCols; ++q)
      o.c[q] = RK4 ? cadd(R.acc[s0].c[q], rmul(c16, tk.c[q])) : cadd(R.acc[s0].c[q], tk.c[q]);
    if (jo >= P.ya && jo < P.yb) band4_store<NN, NAPP, SITE>(g, T, P, rr, o, R.nrm);
  } else {
    Row4 nk;
    if (RK4) {
      if (K == 2) {  // arg = 0.5*k2 + psi(j-1)
#pragma unroll
        for (int q = 0; q < kCols; ++q) nk.c[q] = cadd(rmul(0.5, tk.c[q]), R.up.c[q]);
      } else {  // K == 3: arg = k3 + psi(j-2)
        const Row4 pm = ring_row(g, T, (i - 1) & (kRing4 - 1), P.s, P.scale);
#pragma unroll
        for (int q = 0; q < kCols; ++q) nk.c[q] = cadd(tk.c[q], pm.c[q]);
      }
#pragma unroll
      for (int q = 0; q < kCols; ++q) R.acc[s0].c[q] = cadd(R.acc[s0].c[q], rmul(c13, tk.c[q]));
    } else {
      nk = tk;
#pragma unroll
      for (int q = 0; q < kCols; ++q) R.acc[s0].c[q] = cadd(R.acc[s0].c[q], tk.c[q]);
    }
    R.w[K][s0] = nk;
    smem4[L::xl(g, K - 1, buf) + T.p] = nk.c[0];
    smem4[L::xr(g, K - 1, buf) + T.p] = nk.c[kCols - 1];
  }
}

template <int NN>
__device__ __forceinline__ void band4_load_row(const Geo4<NN>& g, const T4& T, const Piece4& P, int rho) {
  const int y = g.wrap(g.wrap(P.j0 - 1 + rho));
  double2* slot = smem4 + (rho & (kRing4 - 1)) * g.npad();
  const double2* src = P.src + (int64_t)y * g.n();
  if (NN > 0) {
#pragma unroll
    for (int c0 = 0; c0 < (NN > 0 ? NN : 1); c0 += (NN > 0 ? NN / kCols : 1)) {
      const int c = c0 + T.p;
      cpa16(slot + swz(c), src + c);
    }
  } else {
    for (int c = T.p; c < g.n(); c += g.np()) cpa16(slot + swz(c), src + c);
  }
}

template <int NN, int NAPP, bool SITE>
__device__ __forceinline__ void band4_flush(const Geo4<NN>& g, const T4& T, Piece4& P) {
  if (P.pend >= 0 && T.p == 0) {
    const double* red = Lay4<NN, NAPP, SITE>::red(g) + (P.pend & 1) * 32;
    const int nw = (g.np() + 31) >> 5;
    double b = 0.0;
    for (int w = 0; w < nw; ++w) b += red[w];
    P.part[P.pend] = b;
  }
  P.pend = -1;
}

// One pipeline iteration.  PH = (iteration index) mod 3 selects register
// slots; i = iteration index (j = j0 + i); rho(y) = y - (j0 - 1) is a row's
// ring index.
template <int NN, int NAPP, bool RK4, bool SITE, bool EXACT, int PH>
__device__ __forceinline__ void band4_iter(const Band4Args& a, const Geo4<NN>& g, const T4& T, Piece4& P,
                                           Regs4<NAPP>& R, int i) {
  using L = Lay4<NN, NAPP, SITE>;
  const int j = P.j0 + i;
  // rho = i + 2 (psi(j+1)) must have landed; the barrier also publishes the
  // neighbour columns of the last iteration and retires its ring reads.
  cpa_wait<kPref4 - 2>();
  __syncthreads();
  band4_flush<NN, NAPP, SITE>(g, T, P);
  if (i + kPref4 + 1 <= P.last_rho) band4_load_row(g, T, P, i + kPref4 + 1);
  cpa_commit();
  const int buf = i & 1;
  constexpr double c16 = 1.0 / 6.0;
  constexpr int SM1 = (PH + 2) % 3;  // slot of row j-1

  // ---- stage 1: row j.  psi(j-1) and psi(j+1) come from the ring, psi(j)
  // was carried in registers from the previous iteration.
  const int r = g.wrap(j);
  R.up = ring_row(g, T, i & (kRing4 - 1), P.s, P.scale);
  const Row4 dn = ring_row(g, T, (i + 2) & (kRing4 - 1), P.s, P.scale);
  const double2* rowj = smem4 + ((i + 1) & (kRing4 - 1)) * g.npad();
  double2 lf = rowj[T.offl], rt = rowj[T.offr];
  if (P.scale) {
    lf = rmul(P.s, lf);
    rt = rmul(P.s, rt);
  }
  Row4 t;
  apply4<EXACT, SITE>(T, a.k, r, smem4[L::hop2(g) + r], SITE ? L::site(g)[r] : 0.0, R.up, R.psi, dn, lf, rt,
                      a.ci[0], t);
  if constexpr (NAPP == 1) {
    Row4 o;
#pragma unroll
    for (int q = 0; q < kCols; ++q) o.c[q] = cadd(R.psi.c[q], t.c[q]);
    if (j >= P.ya && j < P.yb) band4_store<NN, NAPP, SITE>(g, T, P, r, o, R.nrm);
    R.psi = dn;
  } else {
    Row4 nt;
    if (RK4) {
#pragma unroll
      for (int q = 0; q < kCols; ++q) nt.c[q] = cadd(rmul(0.5, t.c[q]), R.psi.c[q]);
      // acc(j) = psi(j) + k1/6; slot PH still holds acc(j-3) until the last
      // stage has consumed it, so the row waits in `t`.
#pragma unroll
      for (int q = 0; q < kCols; ++q) t.c[q] = cadd(R.psi.c[q], rmul(c16, t.c[q]));
    } else {
      // acc(j-1) = psi(j-1) + t1(j-1): both are at hand (psi(j-1) was just
      // read, t1(j-1) is window 1), and stage 2 below is its first update.
#pragma unroll
      for (int q = 0; q < kCols; ++q) R.acc[SM1].c[q] = cadd(R.up.c[q], R.w[1][SM1].c[q]);
      nt = t;
    }
    R.w[1][PH] = nt;
    R.psi = dn;
    smem4[L::xl(g, 0, buf) + T.p] = nt.c[0];
    smem4[L::xr(g, 0, buf) + T.p] = nt.c[kCols - 1];
    if constexpr (NAPP >= 2) band4_stage<NN, NAPP, RK4, SITE, EXACT, PH, 2>(a, g, T, P, R, i, j);
    if constexpr (NAPP >= 3) band4_stage<NN, NAPP, RK4, SITE, EXACT, PH, 3>(a, g, T, P, R, i, j);
    if constexpr (NAPP >= 4) band4_stage<NN, NAPP, RK4, SITE, EXACT, PH, 4>(a, g, T, P, R, i, j);
    if (RK4) R.acc[PH] = t;
  }
}

template <int NAPP, bool RK4, bool SITE, bool EXACT, int NN>
__global__ void __launch_bounds__(kMaxThreads4, 1) band4_kernel(const __grid_constant__ Band4Args a) {
  using L = Lay4<NN, NAPP, SITE>;
  if (*a.fail != kNoFail) return;
  Geo4<NN> g;
  g.n_ = a.n;
  g.npad_ = a.npad;
  g.rb_ = a.rb;
  const int n = g.n(), NP = g.np();
  const int p = threadIdx.x;
  const int64_t dim = (int64_t)n * n;
  const int nblk = n / g.rb();

  T4 T;
  T.p = p;
  T.pl = p == 0 ? NP - 1 : p - 1;
  T.pr = p == NP - 1 ? 0 : p + 1;
#pragma unroll
  for (int q = 0; q < kCols; ++q) T.off[q] = swz(kCols * p + q);
  T.offl = swz(g.wrap(kCols * p - 1));
  T.offr = swz(g.wrap(kCols * p + kCols));

  // this CTA's contiguous run of norm blocks
  const int64_t G = gridDim.x;
  const int64_t total = a.count * nblk;
  int64_t lo = total * blockIdx.x / G;
  const int64_t hi = total * (blockIdx.x + 1) / G;
  double2* hop2 = smem4 + L::hop2(g);
  double* site = L::site(g);
  while (lo < hi) {
    const int64_t r = lo / nblk;
    const int b0 = (int)(lo % nblk);
    const int nb = (int)std::min<int64_t>(hi - lo, nblk - b0);
    lo += nb;
    Piece4 P;
    P.ya = b0 * g.rb();
    P.yb = (b0 + nb) * g.rb();
    const double* hop = a.coef.hop + r * a.coef.stride;
    const double* sg = SITE ? a.coef.site + r * a.coef.stride : nullptr;
    __syncthreads();  // previous piece done with the coefficient tables and the ring
    for (int y = p; y < n; y += NP) {
      hop2[y] = make_double2(hop[y == 0 ? n - 1 : y - 1], hop[y]);
      if (SITE) site[y] = sg[y];
    }
#pragma unroll
    for (int q = 0; q < kCols; ++q) {
      T.hc[q] = hop[kCols * p + q];
      T.sx[q] = SITE ? sg[kCols * p + q] : 0.0;
    }
    T.hm0 = hop[g.wrap(kCols * p - 1)];
    P.s = a.scl ? a.scl[r] : 1.0;
    P.scale = P.s != 1.0;
    P.src = a.psi_in + r * dim;
    P.dst = a.psi_out + r * dim;
    P.part = a.partial + r * nblk;
    P.pend = -1;
    P.j0 = P.ya - NAPP + 1;                    // first iteration's stage-1 row
    const int iters = (P.yb - P.ya) + 2 * (NAPP - 1);
    P.last_rho = iters + 1;                    // psi rows j0-1 .. j0+iters
    // prologue: rows rho = 0 .. kPref4 (one commit group each)
#pragma unroll
    for (int rho = 0; rho <= kPref4; ++rho) {
      if (rho <= P.last_rho) band4_load_row(g, T, P, rho);
      cpa_commit();
    }
    cpa_wait<kPref4 - 1>();  // rho 0, 1 landed
    __syncthreads();
    Regs4<NAPP> R;
#pragma unroll
    for (int k = 1; k < NAPP; ++k)
#pragma unroll
      for (int w = 0; w < 3; ++w)
#pragma unroll
        for (int q = 0; q < kCols; ++q) R.w[k][w].c[q] = make_double2(0.0, 0.0);
#pragma unroll
    for (int w = 0; w < 3; ++w)
#pragma unroll
      for (int q = 0; q < kCols; ++q) R.acc[w].c[q] = make_double2(0.0, 0.0);
    R.nrm = 0.0;
    R.psi = ring_row(g, T, 1, P.s, P.scale);  // psi(j0)
#pragma unroll 1
    for (int i = 0; i < iters; i += 3) {
      band4_iter<NN, NAPP, RK4, SITE, EXACT, 0>(a, g, T, P, R, i);
      band4_iter<NN, NAPP, RK4, SITE, EXACT, 1>(a, g, T, P, R, i + 1);
      band4_iter<NN, NAPP, RK4, SITE, EXACT, 2>(a, g, T, P, R, i + 2);
    }
    cpa_wait<0>();
    __syncthreads();
    band4_flush<NN, NAPP, SITE>(g, T, P);
  }
}

struct Band4Plan {
  int threads, npad, rb, nblk, grid;
  size_t smem;
};

int sm_count4() {
  static int v = 0;
  if (v == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
  }
  return v;
}

Band4Plan plan_band4(int n, int napp, bool site, int64_t count) {
  Band4Plan p{};
  p.threads = n / kCols;
  p.npad = (n + 7) & ~7;
  p.rb = (n % kRB == 0) ? kRB : n;
  p.nblk = n / p.rb;
  const int nx = napp > 1 ? napp - 1 : 1;
  p.smem = (size_t)kRing4 * p.npad * sizeof(double2) + (size_t)nx * 4 * p.threads * sizeof(double2) +
           (size_t)n * sizeof(double2) + (size_t)((site ? n : 0) + 64) * sizeof(double);
  return p;
}

template <int NAPP, bool RK4, bool SITE, bool EXACT, int NN>
cudaError_t launch_b4(const Band4Args& args, Band4Plan p, cudaStream_t s) {
  auto kern = band4_kernel<NAPP, RK4, SITE, EXACT, NN>;
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
  }
  // occupancy depends on the block size (= n/4) for the runtime-n variant
  int occ = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, p.threads, p.smem);
  if (e != cudaSuccess) return e;
  per_sm = occ;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  const int64_t slots = (int64_t)occ * sm_count4();
  const int64_t grid = std::min<int64_t>(slots, args.count * p.nblk);
  kern<<<(unsigned)grid, p.threads, p.smem, s>>>(args);
  return cudaGetLastError();
}

template <int NAPP, bool RK4, bool SITE, bool EXACT>
cudaError_t launch_b4_nn(const Band4Args& a, Band4Plan p, cudaStream_t s) {
  // compile-time lattice sizes only for the four-application steps (the
  // BASELINE configurations: Taylor-4 and RK4 at N = 256, 512, 1024)
  if constexpr (NAPP != 4) return launch_b4<NAPP, RK4, SITE, EXACT, 0>(a, p, s);
  switch (a.n) {
    case 256: return launch_b4<NAPP, RK4, SITE, EXACT, 256>(a, p, s);
    case 512: return launch_b4<NAPP, RK4, SITE, EXACT, 512>(a, p, s);
    case 1024: return launch_b4<NAPP, RK4, SITE, EXACT, 1024>(a, p, s);
    default: return launch_b4<NAPP, RK4, SITE, EXACT, 0>(a, p, s);
  }
}

template <int NAPP, bool RK4>
cudaError_t launch_b4_n(const Band4Args& a, Band4Plan p, bool site, bool exact, cudaStream_t s) {
  if (site && exact) return launch_b4_nn<NAPP, RK4, true, true>(a, p, s);
  if (site) return launch_b4_nn<NAPP, RK4, true, false>(a, p, s);
  if (exact) return launch_b4_nn<NAPP, RK4, false, true>(a, p, s);
  return launch_b4_nn<NAPP, RK4, false, false>(a, p, s);
}

}  // namespace

bool band4_supported(int m, int n, const StepScalars& sc) {
  return m == 2 && n % kCols == 0 && n >= 16 && n / kCols <= kMaxThreads4 &&
         (sc.backend == 1 || (sc.order >= 1 && sc.order <= 4));
}

int band4_parts(int n) { return (n % kRB == 0) ? n / kRB : 1; }

cudaError_t launch_band4_step(const double2* psi_in, double2* psi_out, int64_t count, int n,
                              const Coef& coef, const StencilConst& k, const StepScalars& sc,
                              bool exact, const double* scl, double* partial,
                              const long long* fail, cudaStream_t s) {
  const bool site = coef.site != nullptr;
  const int napp = sc.backend == 1 ? 4 : sc.order;
  const Band4Plan p = plan_band4(n, napp, site, count);
  Band4Args a;
  a.psi_in = psi_in;
  a.psi_out = psi_out;
  a.n = n;
  a.npad = p.npad;
  a.rb = p.rb;
  a.nblk = p.nblk;
  a.total = count * p.nblk;
  a.count = count;
  a.coef = coef;
  a.k = k;
  for (int i = 0; i < 4; ++i) a.ci[i] = sc.ci[i];
  a.scl = scl;
  a.partial = partial;
  a.fail = fail;
  if (count == 0) return cudaSuccess;
  if (sc.backend == 1) return launch_b4_n<4, true>(a, p, site, exact, s);
  switch (napp) {
    case 1: return launch_b4_n<1, false>(a, p, site, exact, s);
    case 2: return launch_b4_n<2, false>(a, p, site, exact, s);
    case 3: return launch_b4_n<3, false>(a, p, site, exact, s);
    case 4: return launch_b4_n<4, false>(a, p, site, exact, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ctqw
