// Row-marching streaming step kernel for m = 2, four columns per thread,
// lag-1 stage pipeline, persistent balanced row-block schedule.
//
// Why four columns.  The one- and two-column kernels of round 1 (retired;
// DESIGN.md section 4 has their measurements) were bound by shared memory
// (ncu: 1.5-2.6 wavefronts per element-step, L1/TEX 66-85 % busy) and by
// latency at 8-16 warps/SM.  Here
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
// psi rows stream in through an 8-row ring, XOR-swizzled (chunk c ->
// c ^ ((c >> 3) & 7)) so that a thread's four-column reads and the neighbour
// reads are bank-conflict free: one TMA box per row (128B swizzle, mbarrier
// per slot) at the compile-time sizes N = 256/512/1024, lane-contiguous
// 16-byte cp.async chunks otherwise.  Finished rows leave from registers as
// two 256-bit stores per thread.
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
#include "band4.h"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

namespace ctqw {
namespace b4 {



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

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
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
__device__ __forceinline__ void mbar_arrive4(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Split-phase row barrier for the one-CTA-per-SM size (n = 1024, 8 warps):
// every thread
// arrives at the end of its iteration and waits for everybody's arrival only
// after computing the next iteration's stage 1 (which reads nothing another
// warp writes), so stage 1 fills the time a warp would idle at a
// __syncthreads.  Two mbarriers alternate by iteration parity; a warp can
// be at most one iteration ahead of the slowest, so a parity wait is exact.
// (At n = 512, two CTAs share an SM and hide each other's __syncthreads;
// the mbarrier form measured 7 % slower there.)
template <int NN>
constexpr bool band4_split() {
  return NN >= 1024;
}

// One psi row (n complex = n/8 lines of 128 B) global -> shared through TMA,
// 128B-swizzled: 16-byte chunk c lands at chunk c ^ ((c >> 3) & 7), which is
// swz(c) because the destination slot is 1024-byte aligned.  No proxy fence
// before the copy: the slot's generic-proxy accesses are all reads, bound
// before every thread's barrier arrive (release), and the issuing thread
// passed that barrier; the fence's MEMBAR.ALL.CTA on the issuing warp cost
// 0.9 % of the headline (measured).
__device__ __forceinline__ void tma_row(uint32_t dst, const CUtensorMap* tm, int grow, uint32_t bar,
                                        uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst),
      "l"(tm), "r"(0), "r"(0), "r"(grow), "r"(bar)
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
  // ring row stride in chunks: compile-time sizes use TMA rows, whose slots
  // must be 1024-byte aligned (multiple of 64 chunks)
  __device__ __forceinline__ int npad() const { return NN > 0 ? ((NN + 63) & ~63) : npad_; }
  __device__ __forceinline__ int rb() const { return NN > 0 ? (NN % kRB == 0 ? kRB : NN) : rb_; }
  __device__ __forceinline__ int wrap(int r) const { return r < 0 ? r + n() : (r >= n() ? r - n() : r); }
};

// Per-thread constants and per-piece state.  Shared memory is addressed by
// element offsets into smem4 (32-bit shared addressing).
struct T4 {
  int p, pl, pr;
  int off[kCols];     // swizzled ring offsets of own columns
  int offl, offr;     // swizzled ring offsets of columns 4p-1 and 4p+4
  const double* colc; // smem column couplings: [q][NP] hop[4p+q] (q < 4), hop[4p-1] (q = 4), site[4p+q] (5..8)
  int NP;
  double hc[kCols];   // register copy of the column couplings (kColcRegs)
  double hm0;
  double sx[kCols];   // register copy of site[4p+q] (Taylor with on-site noise)
};

// Column tunnelling couplings: in registers (10 registers, no loads) for the
// Taylor kernels, re-read from shared memory per application for RK4 (which
// carries one more row and would spill).

// Column couplings of the thread's four columns, re-read from shared memory
// at every stencil application (holding them in registers spills).
struct ColC {
  double hc[kCols];   // hop[x]      (particle 1 +move coupling)
  double hm0;         // hop[4p-1]   (particle 1 -move coupling of column 0)
  double sx[kCols];   // site[x]
};

template <bool SITE, bool CREG>
__device__ __forceinline__ ColC load_colc(const T4& T) {
  ColC c;
  if (CREG) {
#pragma unroll
    for (int q = 0; q < kCols; ++q) c.hc[q] = T.hc[q];
    c.hm0 = T.hm0;
  } else {
#pragma unroll
    for (int q = 0; q < kCols; ++q) c.hc[q] = T.colc[q * T.NP + T.p];
    c.hm0 = T.colc[kCols * T.NP + T.p];
  }
#pragma unroll
  for (int q = 0; q < kCols; ++q) c.sx[q] = SITE ? (CREG ? T.sx[q] : T.colc[(kCols + 1 + q) * T.NP + T.p]) : 0.0;
  return c;
}

struct Piece4 {
  const double2* src;
  double2* dst;
  double* part;       // partial + r * nblk
  int j0, ya, yb, last_rho;
  double s;
  bool scale;
  int pend;           // norm block awaiting its flush (-1 none)
  int g0;             // CTA iteration count before this piece (split barrier phases)
  int pend_it;        // iteration whose last stage completed norm block pend
  int64_t grow0;      // TMA row coordinate of psi row 0 of this realization (r * n)
  uint32_t* ph;       // per-slot mbarrier phase bits (TMA path)
};

extern __shared__ __align__(1024) double2 smem4[];

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
  __device__ __forceinline__ static double* colc(const Geo4<NN>& g) { return red(g) + 64; }
  __device__ __forceinline__ static uint64_t* bars(const Geo4<NN>& g) {
    return reinterpret_cast<uint64_t*>(colc(g) + (SITE ? 9 : 5) * g.np());
  }
  // RK4: acc(j) = psi(j) + k1/6 parked from stage 1 to the end of the iteration
  // ([q][NP], private per thread), instead of 16 registers across stages 2-4
  // split-phase row barrier (band4_split): mbarriers [iteration & 1]
  __device__ __forceinline__ static uint64_t* rowbar(const Geo4<NN>& g) { return bars(g) + kRing4; }
  __device__ __forceinline__ static double2* stash(const Geo4<NN>& g) {
    const uintptr_t b = reinterpret_cast<uintptr_t>(bars(g) + kRing4 + 2);
    return reinterpret_cast<double2*>((b + 15) & ~uintptr_t(15));
  }
};


// SC: multiply by the pending rescale s (the CTA's realization had a norm
// correction last step); s == 1.0 otherwise, so skipping is exact.
template <bool SC, int NN>
__device__ __forceinline__ Row4 ring_row(const Geo4<NN>& g, const T4& T, int slot, double s) {
  const double2* rowp = smem4 + slot * g.npad();
  Row4 v;
#pragma unroll
  for (int q = 0; q < kCols; ++q) {
    v.c[q] = rowp[T.off[q]];
    if (SC) v.c[q] = rmul(s, v.c[q]);
  }
  return v;
}

// (H z)(r, x) for the thread's four columns of row r: up = row r-1,
// mid = row r, dn = row r+1, lf / rt = columns 4p-1 / 4p+4 of row r.
// DG: the diagonal carries the coincidence term (base[1] != base[0], U != 0).
// HORN: out = psi + i*ci*(H z) (one DFMA per component, the Horner form of
// the Taylor sum); RAW: out = H z (the caller folds i*ci into its sums);
// otherwise out = i*ci*(H z).
template <bool EXACT, bool SITE, int DG, bool CREG, bool HORN = false, bool RAW = false>
__device__ __forceinline__ void apply4(const T4& T, const StencilConst& K, int r, double2 hp,
                                       double srow, const Row4& up, const Row4& mid,
                                       const Row4& dn, double2 lf, double2 rt, double ci,
                                       Row4& out, const Row4* psi = nullptr) {
  const int d = r - kCols * T.p;  // diagonal column offset within the thread's four
  const ColC C = load_colc<SITE, CREG>(T);
#pragma unroll
  for (int q = 0; q < kCols; ++q) {
    // DG: 0 = zero diagonal base (eps0 = U = 0: no multiply by it), 1 = one
    // base for every amplitude (U = 0), 2 = coincidence term on the diagonal
    double v0 = (DG == 2 && d == q) ? K.base[1] : K.base[0];
    if (SITE) v0 = DG == 0 ? __dadd_rn(srow, C.sx[q]) : __dadd_rn(v0, __dadd_rn(srow, C.sx[q]));  // base + (site[x0] + site[x1])
    const double2 l = q == 0 ? lf : mid.c[q - 1];
    const double2 rr = q == kCols - 1 ? rt : mid.c[q + 1];
    const double hm = q == 0 ? C.hm0 : C.hc[q - 1];
    // a zero diagonal (DG == 0, no site noise) contributes nothing: the sum
    // starts at the first neighbour product (0 + x == x, so exact mode keeps
    // the reference's bits)
    constexpr bool ZD = DG == 0 && !SITE;
    double2 h;
    if constexpr (EXACT) {
      h = ZD ? rmul(hp.y, dn.c[q]) : madd<EXACT>(rmul(v0, mid.c[q]), hp.y, dn.c[q]);  // particle 0 +move: row r+1, hop[r]
      h = madd<EXACT>(h, hp.x, up.c[q]);  // particle 0 -move: row r-1, hop[r-1]
      h = madd<EXACT>(h, C.hc[q], rr);    // particle 1 +move
      h = madd<EXACT>(h, hm, l);          // particle 1 -move
    } else {
      // FMA mode: row r+1 last.  In the pipeline it is the only input the
      // previous stage produced in this same iteration, so everything else
      // can issue before that stage finishes (two dependent DFMAs per stage
      // on the critical path instead of six).
      h = ZD ? rmul(hp.x, up.c[q]) : madd<EXACT>(rmul(v0, mid.c[q]), hp.x, up.c[q]);
      h = madd<EXACT>(h, C.hc[q], rr);
      h = madd<EXACT>(h, hm, l);
      h = madd<EXACT>(h, hp.y, dn.c[q]);
    }
    if constexpr (HORN)
      out.c[q] = ifma(psi->c[q], ci, h);
    else if constexpr (RAW)
      out.c[q] = h;
    else
      out.c[q] = times_i(ci, h);
  }
}

// FMA-mode Taylor (order >= 2) runs in Horner form,
//   psi' = psi + c1 H (psi + c2 H (psi + ... (psi + cn H psi))),  ck = -i dt/(hbar k),
// the same polynomial as the reference's term recursion: stage k applies
// c_{n-k+1}, adds psi of its row, and the running sums are replaced by a
// three-row window of psi (Regs4::acc).  12 FP64 instructions per element
// and application instead of 14.  EXACT keeps the reference's order.
template <int NAPP, bool RK4, bool EXACT>
constexpr bool horner4() {
  return !EXACT && !RK4 && NAPP >= 2;
}

// FMA-mode RK4: the stage returns H z and every stage combination
// (arg = psi + a*k, acc += b*k with k = -i dt/hbar H z) is one DFMA per
// component with the weight a*c or b*c folded in: 14 instead of 20 FP64
// instructions per amplitude and stage.
template <bool RK4, bool EXACT>
constexpr bool rk4fma() {
  return RK4 && !EXACT;
}

template <int NAPP>
struct Regs4 {
  Row4 w[NAPP][3];  // w[k], k >= 1: stage-k output window (input of stage k+1); w[0] unused
  Row4 acc[3];      // running sums (Horner: psi), slot = row mod 3 (relative)
  Row4 up;          // psi(j-1): read by stage 1, reused by RK4 stage 2
  double2 hw[3];    // hop2[] of the rows stage 1 read, slot = iteration phase (stages 2-4 reuse them)
  double nrm;
};

// Write one finished row (four columns) and fold |out|^2 into the norm; at
// the end of a norm block, reduce the warp's sum into shared memory (thread 0
// adds the warps in order after the next barrier).
template <int NN, int NAPP, bool SITE>
__device__ __forceinline__ void band4_store(const Geo4<NN>& g, const T4& T, Piece4& P, int rr, const Row4& o,
                                            double& nrm, int it) {
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
    P.pend_it = it;
  }
}

// Stage K (2..NAPP) of iteration j: row j-K+1 from window K-1 (rows j-K ..
// j-K+2, slot(y) = (y - j0) mod 3) and the neighbour columns stage K-1
// published last iteration.
template <int NN, int NAPP, bool RK4, bool SITE, bool EXACT, bool SC, int DG, int PH, int K, bool PRE = false>
__device__ __forceinline__ void band4_stage(const Band4Args& a, const Geo4<NN>& g, const T4& T, Piece4& P,
                                            Regs4<NAPP>& R, int i, int j, double2 hw4, double2 lf_pre = double2(),
                                            double2 rt_pre = double2()) {
  using L = Lay4<NN, NAPP, SITE>;
  constexpr double c16 = 1.0 / 6.0, c13 = 1.0 / 3.0;
  constexpr int s0 = ((PH - K + 1) % 3 + 3) % 3;  // row j-K+1
  constexpr int sm = (s0 + 2) % 3;                // row j-K
  constexpr int sp = (s0 + 1) % 3;                // row j-K+2
  const int buf = i & 1;
  const int rr = g.wrap(j - K + 1);
  // PRE: the neighbour columns were read before the warp's early arrive
  const double2 lf = PRE ? lf_pre : smem4[L::xr(g, K - 2, buf ^ 1) + T.pl];
  const double2 rt = PRE ? rt_pre : smem4[L::xl(g, K - 2, buf ^ 1) + T.pr];
  constexpr bool HORN = horner4<NAPP, RK4, EXACT>();
  constexpr bool RKF = rk4fma<RK4, EXACT>();
  const double ci = RK4 ? a.ci[0] : (HORN ? a.ci[NAPP - K] : a.ci[K - 1]);
  Row4 tk;
  // the row's couplings: loaded by stage 1 K-1 iterations ago (slot =
  // its phase), stage NAPP's row leaves the window in this iteration (hw4).
  // Without on-site noise only: the on-site variants spill with the window
  // (measured -8.5 % at N = 1024, +3.5 % tunnelling-only at N = 256), and
  // the RK4 stage form (exact mode) spills with it too
  constexpr bool HWIN = !SITE && !RK4;  // RK4 (exact / stage form) spills with it
  const double2 hp = !HWIN ? smem4[L::hop2(g) + rr]
                           : (K == NAPP && NAPP >= 4 ? hw4 : R.hw[((PH - K + 1) % 3 + 3) % 3]);
  apply4<EXACT, SITE, DG, !RK4 || RKF, HORN, RKF>(T, a.k, rr, hp, SITE ? L::site(g)[rr] : 0.0,
                                           R.w[K - 1][sm], R.w[K - 1][s0], R.w[K - 1][sp], lf, rt, ci, tk,
                                           &R.acc[s0]);
  if constexpr (RKF) {
    // tk = H arg; k = i*c*tk
    if constexpr (K == NAPP) {
      const int jo = j - K + 1;
      Row4 o;
#pragma unroll
      for (int q = 0; q < kCols; ++q) o.c[q] = ifma(R.acc[s0].c[q], a.rkw[2], tk.c[q]);
      if (jo >= P.ya && jo < P.yb) band4_store<NN, NAPP, SITE>(g, T, P, rr, o, R.nrm, i);
    } else {
      // arg = psi(row) + k/2 (K = 2) or + k (K = 3), psi re-read from the ring
      const Row4 pm = ring_row<SC>(g, T, (i + (K == 2 ? 0 : -1)) & (kRing4 - 1), P.s);
      Row4 nk;
#pragma unroll
      for (int q = 0; q < kCols; ++q) {
        nk.c[q] = ifma(pm.c[q], K == 2 ? a.rkw[0] : ci, tk.c[q]);
        R.acc[s0].c[q] = ifma(R.acc[s0].c[q], a.rkw[1], tk.c[q]);
      }
      R.w[K][s0] = nk;
      smem4[L::xl(g, K - 1, buf) + T.p] = nk.c[0];
      smem4[L::xr(g, K - 1, buf) + T.p] = nk.c[kCols - 1];
    }
    return;
  }
  if constexpr (K == NAPP) {
    const int jo = j - K + 1;
    Row4 o;
#pragma unroll
    for (int q = 0; q < kCols; ++q)
      o.c[q] = HORN ? tk.c[q] : (RK4 ? cadd(R.acc[s0].c[q], rmul(c16, tk.c[q])) : cadd(R.acc[s0].c[q], tk.c[q]));
    if (jo >= P.ya && jo < P.yb) band4_store<NN, NAPP, SITE>(g, T, P, rr, o, R.nrm, i);
  } else if constexpr (HORN) {
    R.w[K][s0] = tk;
    smem4[L::xl(g, K - 1, buf) + T.p] = tk.c[0];
    smem4[L::xr(g, K - 1, buf) + T.p] = tk.c[kCols - 1];
  } else {
    Row4 nk;
    if (RK4) {
      if (K == 2) {  // arg = 0.5*k2 + psi(j-1) (re-read: keeping it from stage 1 spills)
        const Row4 pm = ring_row<SC>(g, T, i & (kRing4 - 1), P.s);
#pragma unroll
        for (int q = 0; q < kCols; ++q) nk.c[q] = cadd(rmul(0.5, tk.c[q]), pm.c[q]);
      } else {  // K == 3: arg = k3 + psi(j-2)
        const Row4 pm = ring_row<SC>(g, T, (i - 1) & (kRing4 - 1), P.s);
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

// Ring slot rho & 7 <- psi row j0 - 1 + rho.  Compile-time sizes: one TMA
// box issued by thread 0, completion on the slot's mbarrier.  Runtime sizes:
// every thread cp.asyncs n/NP 16-byte chunks (lane-contiguous in global
// memory, XOR-swizzled in shared memory).
template <int NN>
__device__ __forceinline__ void band4_load_row(const Band4Args& a, const Geo4<NN>& g, const T4& T,
                                               const Piece4& P, int rho, uint32_t bars) {
  const int y = g.wrap(g.wrap(P.j0 - 1 + rho));
  const int slot = rho & (kRing4 - 1);
  if constexpr (NN > 0) {
    if (T.p == 0)
      tma_row(smem_u32(smem4 + slot * g.npad()), &a.tmap, (int)(P.grow0 + y), bars + 8 * slot,
              (uint32_t)(NN * sizeof(double2)));
  } else {
    double2* dst = smem4 + slot * g.npad();
    const double2* src = P.src + (int64_t)y * g.n();
    for (int c = T.p; c < g.n(); c += g.np()) cpa16(dst + swz(c), src + c);
  }
}

// Wait until ring row rho has landed (TMA path: the slot's mbarrier phase).
template <int NN>
__device__ __forceinline__ void band4_wait_row(Piece4& P, int rho, uint32_t bars) {
  if constexpr (NN > 0) {
    if (rho <= P.last_rho) {
      const int slot = rho & (kRing4 - 1);
      mbar_wait(bars + 8 * slot, (*P.ph >> slot) & 1u);
      *P.ph ^= 1u << slot;
    }
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
template <int NN, int NAPP, bool RK4, bool SITE, bool EXACT, bool SC, int DG, int PH>
__device__ __forceinline__ void band4_iter(const Band4Args& a, const Geo4<NN>& g, const T4& T, Piece4& P,
                                           Regs4<NAPP>& R, int i, uint32_t bars) {
  using L = Lay4<NN, NAPP, SITE>;
  const int j = P.j0 + i;
  // rho = i + 2 (psi(j+1)) must have landed; the barrier also publishes the
  // neighbour columns of the last iteration and retires its ring reads.
  constexpr bool SPLIT = band4_split<NN>();
  if constexpr (NN > 0) {
    band4_wait_row<NN>(P, i + 2, bars);
  } else {
    cpa_wait<kPref4 - 2>();
  }
  if constexpr (!SPLIT) {
    __syncthreads();
    band4_flush<NN, NAPP, SITE>(g, T, P);
    if (i + kPref4 + 1 <= P.last_rho) band4_load_row(a, g, T, P, i + kPref4 + 1, bars);
  }
  if constexpr (NN == 0) cpa_commit();
  const int buf = i & 1;
  constexpr double c16 = 1.0 / 6.0;
  constexpr int SM1 = (PH + 2) % 3;  // slot of row j-1

  // ---- stage 1: row j; psi(j-1), psi(j), psi(j+1) come from the ring.
  const int r = g.wrap(j);
  R.up = ring_row<SC>(g, T, i & (kRing4 - 1), P.s);
  const Row4 psi = ring_row<SC>(g, T, (i + 1) & (kRing4 - 1), P.s);  // psi(j): re-read, not carried
  const Row4 dn = ring_row<SC>(g, T, (i + 2) & (kRing4 - 1), P.s);
  const double2* rowj = smem4 + ((i + 1) & (kRing4 - 1)) * g.npad();
  double2 lf = rowj[T.offl], rt = rowj[T.offr];
  if (SC) {
    lf = rmul(P.s, lf);
    rt = rmul(P.s, rt);
  }
  constexpr bool HORN = horner4<NAPP, RK4, EXACT>();
  constexpr bool RKF = rk4fma<RK4, EXACT>();
  Row4 t;
  const double2 hw4 = (SITE || RK4) ? double2() : R.hw[PH];  // row j-3 (stage 4's) leaves the window, row j enters
  const double2 hp1 = smem4[L::hop2(g) + r];
  if constexpr (!SITE && !RK4) R.hw[PH] = hp1;
  apply4<EXACT, SITE, DG, !RK4 || RKF, HORN, RKF>(T, a.k, r, hp1, SITE ? L::site(g)[r] : 0.0, R.up, psi,
                                           dn, lf, rt, HORN ? a.ci[NAPP - 1] : a.ci[0], t, &psi);
  if constexpr (NAPP == 1) {
    Row4 o;
#pragma unroll
    for (int q = 0; q < kCols; ++q) o.c[q] = cadd(psi.c[q], t.c[q]);
    if (j >= P.ya && j < P.yb) band4_store<NN, NAPP, SITE>(g, T, P, r, o, R.nrm, i);
  } else {
    Row4 nt;
    if constexpr (RKF) {
      // t = H psi: arg = psi + k1/2, acc(j) = psi + k1/6 (parked as below)
#pragma unroll
      for (int q = 0; q < kCols; ++q) {
        nt.c[q] = ifma(psi.c[q], a.rkw[0], t.c[q]);
        t.c[q] = ifma(psi.c[q], a.rkw[2], t.c[q]);
      }
      if constexpr (stash_fits(NN, SITE)) {
        double2* st = L::stash(g);
#pragma unroll
        for (int q = 0; q < kCols; ++q) st[q * g.np() + T.p] = t.c[q];
      }
    } else if (RK4) {
#pragma unroll
      for (int q = 0; q < kCols; ++q) nt.c[q] = cadd(rmul(0.5, t.c[q]), psi.c[q]);
      // acc(j) = psi(j) + k1/6; slot PH still holds acc(j-3) until the last
      // stage has consumed it, so the row waits in `t` (or in the stash).
#pragma unroll
      for (int q = 0; q < kCols; ++q) t.c[q] = cadd(psi.c[q], rmul(c16, t.c[q]));
      if constexpr (stash_fits(NN, SITE)) {
        double2* st = L::stash(g);
#pragma unroll
        for (int q = 0; q < kCols; ++q) st[q * g.np() + T.p] = t.c[q];
      }
    } else if constexpr (HORN) {
      // psi(j-1) joins the window for stages 2..n (rows j-1 .. j-n+1); its
      // slot held psi(j-4), which the last stage used one iteration ago
      R.acc[SM1] = R.up;
      nt = t;
    } else {
      // acc(j-1) = psi(j-1) + t1(j-1): both are at hand (psi(j-1) was just
      // read, t1(j-1) is window 1), and stage 2 below is its first update.
#pragma unroll
      for (int q = 0; q < kCols; ++q) R.acc[SM1].c[q] = cadd(R.up.c[q], R.w[1][SM1].c[q]);
      nt = t;
    }
    R.w[1][PH] = nt;
    if constexpr (SPLIT) {
      // everybody finished iteration i-1: its exchange rows are published,
      // the exchange buffer this stage overwrites and the ring slot the next
      // TMA refills are no longer read, its norm-block partials are in place
      const int G = P.g0 + i;
      if (i > 0) mbar_wait(smem_u32(L::rowbar(g)) + 8 * ((G - 1) & 1), (uint32_t)((G - 1) >> 1) & 1u);
      // the arrives come before the last stage, so a norm block whose last
      // row was stored in iteration i-1 is complete only at iteration i+1
      if (P.pend >= 0 && P.pend_it <= i - (SITE ? 2 : 1)) band4_flush<NN, NAPP, SITE>(g, T, P);
      if (i + kPref4 + 1 <= P.last_rho) band4_load_row(a, g, T, P, i + kPref4 + 1, bars);
    }
    smem4[L::xl(g, 0, buf) + T.p] = nt.c[0];
    smem4[L::xr(g, 0, buf) + T.p] = nt.c[kCols - 1];
    if constexpr (NAPP >= 2) band4_stage<NN, NAPP, RK4, SITE, EXACT, SC, DG, PH, 2>(a, g, T, P, R, i, j, hw4);
    if constexpr (NAPP >= 3) band4_stage<NN, NAPP, RK4, SITE, EXACT, SC, DG, PH, 3>(a, g, T, P, R, i, j, hw4);
    if constexpr (NAPP >= 4) {
      // early arrive: measured +2 % with on-site noise (the headline) and -7 %
      // without (register allocation of the zero-diagonal variant), so only
      // the on-site variants use it
      if constexpr (SPLIT && SITE) {
        // the last stage publishes nothing and reads neither the ring nor
        // any exchange row but its two neighbour columns: read those, then
        // arrive, so the other warps' waits do not cover this stage too (its
        // norm-block partial is flushed one row later, band4_store)
        const double2 lf4 = smem4[L::xr(g, NAPP - 2, buf ^ 1) + T.pl];
        const double2 rt4 = smem4[L::xl(g, NAPP - 2, buf ^ 1) + T.pr];
        mbar_arrive4(smem_u32(L::rowbar(g)) + 8 * ((P.g0 + i) & 1));
        band4_stage<NN, NAPP, RK4, SITE, EXACT, SC, DG, PH, 4, true>(a, g, T, P, R, i, j, hw4, lf4, rt4);
      } else {
        band4_stage<NN, NAPP, RK4, SITE, EXACT, SC, DG, PH, 4>(a, g, T, P, R, i, j, hw4);
      }
    }
    if constexpr (RK4) {
      if constexpr (stash_fits(NN, SITE)) {
        const double2* st = L::stash(g);
#pragma unroll
        for (int q = 0; q < kCols; ++q) R.acc[PH].c[q] = st[q * g.np() + T.p];
      } else {
        R.acc[PH] = t;
      }
    }
  }
  if constexpr (SPLIT && !SITE) mbar_arrive4(smem_u32(L::rowbar(g)) + 8 * ((P.g0 + i) & 1));
}

template <int NN, int NAPP, bool RK4, bool SITE, bool EXACT, bool SC, int DG>
__device__ __forceinline__ void band4_loop(const Band4Args& a, const Geo4<NN>& g, const T4& T, Piece4& P,
                                           Regs4<NAPP>& R, int iters, uint32_t bars) {
#pragma unroll 1
  for (int i = 0; i < iters; i += 3) {
    band4_iter<NN, NAPP, RK4, SITE, EXACT, SC, DG, 0>(a, g, T, P, R, i, bars);
    band4_iter<NN, NAPP, RK4, SITE, EXACT, SC, DG, 1>(a, g, T, P, R, i + 1, bars);
    band4_iter<NN, NAPP, RK4, SITE, EXACT, SC, DG, 2>(a, g, T, P, R, i + 2, bars);
  }
}

template <int NAPP, bool RK4, bool SITE, bool EXACT, int NN, int DG>
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
  T.colc = L::colc(g);
  T.NP = NP;

  // TMA rows are 128B-swizzled relative to 1024-byte boundaries
  if (NN > 0 && (smem_u32(smem4) & 1023u) != 0) __trap();
  // TMA ring barriers (one per slot) live after the column table
  uint32_t ph_bits = 0;
  const uint32_t bars = smem_u32(L::bars(g));
  if (NN > 0 && p == 0) {
    for (int q = 0; q < kRing4; ++q) mbar_init(bars + 8 * q, 1);
    if (band4_split<NN>()) {
      mbar_init(smem_u32(L::rowbar(g)), NP);
      mbar_init(smem_u32(L::rowbar(g)) + 8, NP);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  int g0 = 0;

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
    {
      double* cc = L::colc(g);
#pragma unroll
      for (int q = 0; q < kCols; ++q) {
        cc[q * NP + p] = hop[kCols * p + q];
        if (SITE) cc[(kCols + 1 + q) * NP + p] = sg[kCols * p + q];
      }
      cc[kCols * NP + p] = hop[g.wrap(kCols * p - 1)];
#pragma unroll
      for (int q = 0; q < kCols; ++q) {
        T.hc[q] = hop[kCols * p + q];
        T.sx[q] = SITE ? sg[kCols * p + q] : 0.0;
      }
      T.hm0 = hop[g.wrap(kCols * p - 1)];
    }
    P.s = a.scl ? a.scl[r] : 1.0;
    P.scale = P.s != 1.0;
    P.src = a.psi_in + (a.bcast ? 0 : r * dim);
    P.dst = a.psi_out + r * dim;
    P.part = a.partial + r * nblk;
    P.pend = -1;
    P.pend_it = 0;
    P.g0 = g0;
    P.grow0 = a.bcast ? 0 : r * n;
    P.ph = &ph_bits;
    P.j0 = P.ya - NAPP + 1;                    // first iteration's stage-1 row
    const int iters = (P.yb - P.ya) + 2 * (NAPP - 1);
    P.last_rho = iters + 1;                    // psi rows j0-1 .. j0+iters
    // prologue: rows rho = 0 .. kPref4 (one commit group each)
#pragma unroll
    for (int rho = 0; rho <= kPref4; ++rho) {
      if (rho <= P.last_rho) band4_load_row(a, g, T, P, rho, bars);
      if constexpr (NN == 0) cpa_commit();
    }
    if constexpr (NN > 0) {
      band4_wait_row<NN>(P, 0, bars);
      band4_wait_row<NN>(P, 1, bars);
    } else {
      cpa_wait<kPref4 - 1>();  // rho 0, 1 landed
    }
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
#pragma unroll
    for (int w = 0; w < 3; ++w) R.hw[w] = make_double2(0.0, 0.0);
    R.nrm = 0.0;
    if constexpr (NN > 0) {  // compile-time sizes: no rescale multiplies unless needed
      if (P.scale) band4_loop<NN, NAPP, RK4, SITE, EXACT, true, DG>(a, g, T, P, R, iters, bars);
      else band4_loop<NN, NAPP, RK4, SITE, EXACT, false, DG>(a, g, T, P, R, iters, bars);
    } else {
      band4_loop<NN, NAPP, RK4, SITE, EXACT, true, DG>(a, g, T, P, R, iters, bars);
    }
    g0 += (iters + 2) / 3 * 3;  // the loop runs whole groups of three iterations
    if constexpr (NN == 0) cpa_wait<0>();
    __syncthreads();
    band4_flush<NN, NAPP, SITE>(g, T, P);
  }
}

inline int sm_count4() {
  static int v = 0;
  if (v == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
  }
  return v;
}

// TMA descriptor of the input state stack: rows of n complex128 viewed as
// n/8 lines of 16 doubles (128 B), one box = one row, 128B swizzle.
inline cudaError_t encode_rows_map(CUtensorMap* map, const double2* base, int n, int64_t count) {
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
  if (n % 64 != 0 || n / 8 > 256 || count * n > 0x7fffffffLL) return cudaErrorInvalidValue;
  const cuuint64_t dims[3] = {16, (cuuint64_t)(n / 8), (cuuint64_t)(count * n)};
  const cuuint64_t strides[2] = {128, (cuuint64_t)n * sizeof(double2)};
  const cuuint32_t box[3] = {16, (cuuint32_t)(n / 8), 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double2*>(base), dims, strides,
                            box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int NAPP, bool RK4, bool SITE, bool EXACT, int NN, int DG>
cudaError_t launch_b4(const Band4Args& args, Band4Plan p, cudaStream_t s) {
  auto kern = band4_kernel<NAPP, RK4, SITE, EXACT, NN, DG>;
  static DeviceOnce once;
  if (once.first()) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
  }
  // occupancy depends on the block size (= n/4) for the runtime-n variant
  int occ = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, p.threads, p.smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  const int64_t slots = (int64_t)occ * sm_count4();
  const int64_t grid = std::min<int64_t>(slots, args.count * p.nblk);
  if constexpr (NN > 0) {
    Band4Args a = args;
    e = encode_rows_map(&a.tmap, a.psi_in, NN, a.bcast ? 1 : a.count);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)grid, p.threads, p.smem, s>>>(a);
  } else {
    kern<<<(unsigned)grid, p.threads, p.smem, s>>>(args);
  }
  return cudaGetLastError();
}

#define CTQW_B4_INST(NAPP, RK4, SITE, EXACT, NN, DG) \
  template cudaError_t launch_b4<NAPP, RK4, SITE, EXACT, NN, DG>(const Band4Args&, Band4Plan, cudaStream_t);

}  // namespace b4
}  // namespace ctqw
