// Internal launch interface between api.cu and the kernel translation units.
#pragma once

#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "ctqw_device.cuh"

namespace ctqw {

constexpr int64_t kMaxGridY = 65535;

inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

// Once-per-device flag: function attributes (cudaFuncSetAttribute) belong to
// a device, and one process may drive a handle per GPU.
struct DeviceOnce {
  std::atomic<uint64_t> done{0};
  bool first() {
    const int d = current_device() & 63;
    const uint64_t bit = 1ull << d;
    return !(done.fetch_or(bit) & bit);
  }
};
constexpr int kMaxParts = 256;  // norm partials per realization

// Diagonal base per coincidence count c: m*eps0 + U*c (hamiltonian.py:132).
struct StencilConst {
  double base[4];
};

// Taylor / RK4 scalars, computed on the host exactly as the reference does
// (coeff = -1j*dt/hbar, coeff/j; propagators.py:185,191).
constexpr int kMaxTaylorOrder = 64;

struct StepScalars {
  int backend;  // 0 taylor, 1 rk4
  int order;    // Taylor order (applications per step); 4 for RK4
  double ci[kMaxTaylorOrder];  // imaginary part of coeff/j, j = 1..order (taylor); ci[0] = coeff (rk4)
  int rk4_horner;  // 1: an FMA-mode RK4 step run as the Taylor-4 kernels (the same polynomial)
};

int generic_parts(int64_t dim);

// noise.cu
cudaError_t launch_draw_noise(uint64_t master_seed, int64_t r0, int64_t count,
                              const double* levels_dev, int n_levels, int64_t total,
                              double* out, cudaStream_t s);
cudaError_t launch_build_coef(const double* noise, int64_t count, int n, int K, int64_t n_links,
                              int64_t n_sites, const double* t_slot, double* hop, double* site,
                              cudaStream_t s);
cudaError_t launch_fill_states(double2* psi, int64_t count, int64_t dim, const double2* psi0,
                               cudaStream_t s);

// telegraph.cu (dynamic noise, rate > 0)
struct TelegraphGen {
  uint64_t state_lo, state_hi, inc_lo, inc_hi;  // PCG64 of the realization's Generator
  uint32_t u32;                                  // PCG64's cached upper half (next_uint32)
  int has_u32;
  double time;                                   // NoiseProcess.time
  long long switches;                            // NoiseProcess.switch_count
};
cudaError_t launch_telegraph_init(uint64_t master_seed, int64_t r0, int64_t count, const double* levels_dev,
                                  int n_levels, int64_t total, double mean_wait, double* values,
                                  double* next_switch, TelegraphGen* gen, cudaStream_t s);
cudaError_t launch_telegraph_advance(int64_t count, int64_t total, int64_t n_links, int64_t n_sites, int n,
                                     double dt, const double* levels_dev, int n_levels, double mean_wait,
                                     const double* t_slot, int K, double* values, double* next_switch,
                                     TelegraphGen* gen, double* hop, double* site, int64_t hop_stride,
                                     int64_t site_stride, int* lists, double* oldv, const long long* fail,
                                     cudaStream_t s);

// stencil_generic.cu
cudaError_t launch_apply(int m, const double2* psi, double2* out, int64_t count, int64_t dim,
                         int n, const Coef& coef, const StencilConst& k, bool exact,
                         cudaStream_t s);
cudaError_t launch_taylor_order(int m, bool exact, bool scale, const double2* term_in,
                                double2* term_out, const double2* acc_in, double2* acc_out,
                                int64_t count, int64_t dim, int n, const Coef& coef,
                                const StencilConst& k, double ci, const double* scl,
                                double* partial, const long long* fail, cudaStream_t s);
cudaError_t launch_rk4_stage(int m, bool exact, bool scale, int stage, const double2* arg_in,
                             const double2* psi, const double2* out_in, double2* arg_out,
                             double2* out_out, int64_t count, int64_t dim, int n,
                             const Coef& coef, const StencilConst& k, double ci,
                             const double* scl, double* partial, const long long* fail,
                             cudaStream_t s);
cudaError_t launch_norm_partial(const double2* psi, int64_t count, int64_t dim, double* partial,
                                cudaStream_t s);

// step_tile.cu (m = 2 fused paths)
struct TileGeom {
  int n;       // ring length
  int nt;      // tiles per axis
  int halo;    // stencil applications per step
};
bool tile_supported(int m, int n, const StepScalars& sc);
bool resident_supported(int m, int n, const StepScalars& sc);
bool resident64_supported(int m, int n, const StepScalars& sc);
cudaError_t launch_resident64(double2* psi, int64_t count, const Coef& coef, const StencilConst& k,
                              const StepScalars& sc, bool exact, const NormPolicy& pol, long long first_step,
                              long long n_steps, RealStat* stats, EventRec* events, long long* fail,
                              cudaStream_t s, unsigned long long* obs = nullptr, long long post_rate = 1,
                              long long origin = 0, long long final_step = 0, const double2* psi0 = nullptr,
                              double2* snap = nullptr);
// Batched post-processing of P collection points from their exact limbs
// acc[P][3][dim]: diag[P][dim] (scratch or the caller's), out[P][n + 3] =
// populations (n) + {sum p, sum p^2, participation ratio}.
cudaError_t launch_observe_points(int m, int n, int64_t dim, const unsigned long long* acc, int64_t npoints,
                                  double total, double* diag, double* out, double* scratch, cudaStream_t s);
int tile_parts(int n, const StepScalars& sc);
cudaError_t launch_tile_step(const double2* psi_in, double2* psi_out, int64_t count, int n,
                             const Coef& coef, const StencilConst& k, const StepScalars& sc,
                             bool exact, const double* scl, double* partial,
                             const long long* fail, cudaStream_t s);
// step_plane3.cu (m = 3, N = 128: one 16-CTA cluster per realization, DSMEM
// plane exchange, TMA plane ring)
bool plane3_supported(int m, int n, const StepScalars& sc);
int plane3_parts();
cudaError_t launch_plane3_step(const double2* psi_in, double2* psi_out, int64_t count, const Coef& coef,
                               const StencilConst& k, const StepScalars& sc, bool exact, const double* scl,
                               double* partial, const long long* fail, cudaStream_t s);
// step_band4.cu (m = 2 row-marching kernel, four columns per thread, lag-1
// pipeline, persistent row-block schedule; the default streaming path)
bool band4_supported(int m, int n, const StepScalars& sc);
int band4_parts(int n);
// bcast_in: psi_in is ONE state, the input of every realization (the first
// step from the initial state, without materialising the stack)
cudaError_t launch_band4_step(const double2* psi_in, double2* psi_out, int64_t count, int n,
                              const Coef& coef, const StencilConst& k, const StepScalars& sc,
                              bool exact, const double* scl, double* partial,
                              const long long* fail, cudaStream_t s, bool bcast_in = false);
cudaError_t launch_resident(double2* psi, int64_t count, int n, const Coef& coef,
                            const StencilConst& k, const StepScalars& sc, bool exact,
                            const NormPolicy& pol, long long first_step, long long n_steps,
                            RealStat* stats, EventRec* events, long long* fail,
                            cudaStream_t s);

// norm_observe.cu
cudaError_t launch_norm_decide(const double* partial, int nparts, int64_t count,
                               long long step, const NormPolicy& pol, double* scl,
                               RealStat* stats, EventRec* events, long long* fail,
                               cudaStream_t s);
cudaError_t launch_rescale(double2* psi, int64_t count, int64_t dim, double* scl,
                           cudaStream_t s);
cudaError_t launch_reset_stats(RealStat* stats, double* scl, int64_t count, long long* fail,
                               cudaStream_t s);
struct Summary {
  long long events;
  long long corrections;
  double max_dev;
  long long fail_step;
  long long fail_row;
  double fail_dev;
};
cudaError_t launch_stats_reduce(const RealStat* stats, int64_t count, Summary* out,
                                cudaStream_t s);
cudaError_t launch_norm_sum(const double* partial, int nparts, int64_t count, double* n2,
                            cudaStream_t s);
cudaError_t launch_scale_rows(double2* psi, int64_t count, int64_t dim, const double* scl,
                              cudaStream_t s);
cudaError_t launch_observe_diag_fixed(const double2* psi, int64_t count, int64_t dim, unsigned long long* acc,
                                      bool accumulate, cudaStream_t s);
cudaError_t launch_fixed_from_double(const double* diag, int64_t dim, unsigned long long* acc, cudaStream_t s);
cudaError_t launch_fixed_to_double(const unsigned long long* acc, int64_t dim, double* diag, cudaStream_t s);
cudaError_t launch_observe_reduce(int m, int n, int64_t dim, const double* diag_sum,
                                  double total, double* pops, double* scalars, double* joint,
                                  double* scratch, cudaStream_t s);
cudaError_t launch_overlap_sumsq(const double2* a, int64_t ra, const double2* b, int64_t rb,
                                 int64_t dim, double* scratch, int64_t scratch_cap,
                                 double* out, cudaStream_t s, int64_t npoints = 1, int64_t pstride = 0);
cudaError_t launch_packed_gram(const double2* psi, int64_t count, int64_t dim, double scale, double2* packed,
                               cudaStream_t s);
int64_t overlap_parts(int64_t ra, int64_t rb, bool same);
int64_t overlap_scratch_doubles(int64_t ra, int64_t rb, bool same, int64_t dim, int64_t npoints = 1);

}  // namespace ctqw
