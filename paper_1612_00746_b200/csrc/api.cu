// C ABI of libctqw.so (declared in include/ctqw.h): handle management,
// validation with the reference's error classes, and the path dispatch of
// ctqw_evolve:
//   m = 2, N <= 64            -> resident kernel (whole segment on chip)
//   m = 2, N > 64, order <= 4 -> streaming tile kernel, one launch per step
//   otherwise (m = 1, 3, ...) -> generic per-application kernels
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ctqw.h"
#include "ctqw_device.cuh"
#include "kernels.h"

using namespace ctqw;

struct ctqw_ctx {
  int device = 0;
  ctqw_model_t model{};
  int m = 0, n = 0;
  int64_t dim = 0;
  StencilConst k{};
  // bound coefficient rows (caller-owned)
  int64_t coef_count = 0;
  const double* hop = nullptr;
  const double* site = nullptr;
  int64_t stride = 0;
  int64_t site_stride = 0;
  // lattice: K stored slots per site; general lattices carry move tables and
  // run on the generic kernels only
  int K = 1;
  bool needs_lattice = false;  // created with k_half != 1 or open boundary
  bool general = false;        // ctqw_set_lattice called
  int* lat_pos = nullptr;
  int* lat_neg = nullptr;
  double* t_slot = nullptr;    // [K] tunnelling per slot (device)
  // library-owned device buffers
  double* levels = nullptr;
  int64_t levels_cap = 0;
  double* partial = nullptr;
  int64_t partial_cap = 0;
  double* scl = nullptr;
  RealStat* stats = nullptr;
  EventRec* events = nullptr;
  int64_t stat_cap = 0;
  long long* fail = nullptr;
  Summary* summary_dev = nullptr;
  Summary* summary_host = nullptr;
  double2* scratch[2] = {nullptr, nullptr};
  double2* scratch_work = nullptr;  // second state buffer when the caller passes none
  int64_t scratch_work_elems = 0;
  int64_t scratch_elems = 0;
  double* n2_dev = nullptr;
  int64_t n2_cap = 0;
  double* small = nullptr;  // observe_reduce scratch (2 x 148 doubles)
  unsigned long long* fixed_acc = nullptr;  // [3][dim] exact diagonal limbs (ctqw_observe_diag)
  int64_t fixed_cap = 0;
  double* overlap_partial = nullptr;
  int64_t overlap_cap = 0;
  const double2* initial = nullptr;  // ctqw_set_initial: the next evolve starts every realization from this state
  double* points_scratch = nullptr;  // ctqw_observe_points: per-point partials (+ diag when the caller gives none)
  int64_t points_cap = 0;
  int64_t last_count = 0;
  std::atomic<long long> launches{0};
  // optional CUDA-event timing of the dominant kernel launches (bench.py)
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  int64_t timed_launches = 0;
  // dynamic telegraph noise (rate > 0): library-owned process state
  double* tg_values = nullptr;      // [count][total]
  double* tg_next = nullptr;        // [count][total] next switch times
  TelegraphGen* tg_gen = nullptr;   // [count] generator, time, switch count
  double* tg_levels = nullptr;
  int64_t tg_cap = 0, tg_gen_cap = 0, tg_count = 0, tg_total = 0, tg_links = 0, tg_sites = 0;
  int tg_nlev = 0;
  double tg_mean_wait = 0.0;
  bool tg_enabled = false;
  long long* tg_sum = nullptr;
  int* tg_lists = nullptr;          // [count][2][total] due lists (advance scratch)
  double* tg_oldv = nullptr;        // [count][total] values before the advance
  int stream_kind = 0;  // CTQW_STREAM: 0 auto, 1 tile, 4 band4, 5 plane3, 6 generic
  const char* stream_kernel = "";  // dominant kernel of the last ctqw_evolve
  char variant[128] = {0};         // its compile-time specialization (ctqw_step_variant)
  std::string err;
};

namespace {

thread_local std::string g_err;

int fail_with(ctqw_ctx* h, int code, const std::string& msg) {
  if (h) h->err = msg;
  g_err = msg;
  return code;
}

int check_cuda(ctqw_ctx* h, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return CTQW_OK;
  return fail_with(h, CTQW_ERR_OTHER, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(h, expr)                                     \
  do {                                                        \
    int _rc = check_cuda((h), (expr), #expr);                 \
    if (_rc != CTQW_OK) return _rc;                           \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

template <typename T>
int ensure(ctqw_ctx* h, T** ptr, int64_t* cap, int64_t want, const char* what) {
  if (want <= *cap && *ptr) return CTQW_OK;
  if (*ptr) cudaFree(*ptr);
  *ptr = nullptr;
  *cap = 0;
  cudaError_t e = cudaMalloc((void**)ptr, (size_t)std::max<int64_t>(want, 1) * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail_with(h, CTQW_ERR_CAPACITY,
                     std::string("cannot allocate ") + what + ": " + cudaGetErrorString(e));
  }
  *cap = want;
  return CTQW_OK;
}

int ensure_stats(ctqw_ctx* h, int64_t count) {
  if (count <= h->stat_cap && h->stats) return CTQW_OK;
  if (h->scl) cudaFree(h->scl);
  if (h->stats) cudaFree(h->stats);
  if (h->events) cudaFree(h->events);
  h->scl = nullptr;
  h->stats = nullptr;
  h->events = nullptr;
  h->stat_cap = 0;
  const int64_t c = std::max<int64_t>(count, 1);
  if (cudaMalloc((void**)&h->scl, c * sizeof(double)) != cudaSuccess ||
      cudaMalloc((void**)&h->stats, c * sizeof(RealStat)) != cudaSuccess ||
      cudaMalloc((void**)&h->events, c * kMaxEvents * sizeof(EventRec)) != cudaSuccess) {
    cudaGetLastError();
    return fail_with(h, CTQW_ERR_CAPACITY, "cannot allocate per-realization statistics");
  }
  h->stat_cap = count;
  return CTQW_OK;
}

int ensure_scratch(ctqw_ctx* h, int64_t elems) {
  if (elems <= h->scratch_elems && h->scratch[0]) return CTQW_OK;
  for (auto& p : h->scratch) {
    if (p) cudaFree(p);
    p = nullptr;
  }
  h->scratch_elems = 0;
  for (auto& p : h->scratch) {
    if (cudaMalloc((void**)&p, (size_t)elems * sizeof(double2)) != cudaSuccess) {
      cudaGetLastError();
      return fail_with(h, CTQW_ERR_CAPACITY, "cannot allocate propagation scratch");
    }
  }
  h->scratch_elems = elems;
  return CTQW_OK;
}

// Record a CUDA event on s (timing mode); returns nullptr when disabled.
cudaEvent_t timing_event(ctqw_ctx* h, cudaStream_t s) {
  if (!h->timing) return nullptr;
  if (h->ev_used == h->ev_pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    h->ev_pool.push_back(e);
  }
  cudaEvent_t e = h->ev_pool[h->ev_used++];
  cudaEventRecord(e, s);
  return e;
}

int validate_stepper(ctqw_ctx* h, const ctqw_stepper_t* st) {
  if (!st) return fail_with(h, CTQW_ERR_CONFIG, "stepper is NULL");
  if (st->backend != CTQW_BACKEND_TAYLOR && st->backend != CTQW_BACKEND_RK4)
    return fail_with(h, CTQW_ERR_CONFIG, "backend must be taylor or rk4 (eigen is not on the B200 path)");
  if (!(std::isfinite(st->dt) && st->dt > 0))
    return fail_with(h, CTQW_ERR_CONFIG, "dt must be positive and finite");
  if (st->backend == CTQW_BACKEND_TAYLOR && (st->order < 1 || st->order > kMaxTaylorOrder))
    return fail_with(h, CTQW_ERR_CONFIG, "taylor_order must be in [1, 64] on the B200 path");
  if (!(0 < st->tol_norm && st->tol_norm < st->tol_fail))
    return fail_with(h, CTQW_ERR_CONFIG, "need 0 < tol_norm < tol_fail");
  return CTQW_OK;
}

// integrator label of a kernel variant string
const char* integ_label(const StepScalars& sc) {
  return sc.rk4_horner ? "rk4=taylor4" : sc.backend == CTQW_BACKEND_RK4 ? "rk4" : "taylor";
}

StepScalars scalars_for(const ctqw_ctx* h, const ctqw_stepper_t* st) {
  StepScalars sc{};
  sc.backend = st->backend;
  // coeff = -1j*dt/hbar has real part 0 and imaginary part -dt/hbar; the
  // Taylor recursion multiplies by coeff/j (propagators.py:185,191).
  const double c = -st->dt / h->model.hbar;
  // For a Hamiltonian constant over the step, classic RK4 is exactly the
  // degree-4 Taylor polynomial: (k1 + 2k2 + 2k3 + k4)/6 = A + A^2/2 + A^3/6 +
  // A^4/24 applied to psi (A = coeff*H; the reference's own tests assert
  // RK4 == Taylor-4, test_propagators.py:112-119).  Exact mode keeps the
  // reference's stage arithmetic bit for bit; FMA mode only promises 1e-12, so
  // it evaluates that polynomial in Horner form with the Taylor kernels (12
  // instead of 14 FP64 instructions per amplitude and stage, no stage stash).
  // CTQW_RK4_STAGES=1 keeps the stage form (A/B and the stage kernels' tests).
  const char* stages = std::getenv("CTQW_RK4_STAGES");
  const bool horner = st->backend == CTQW_BACKEND_RK4 && !st->exact &&
                      !(stages && stages[0] != '\0' && std::strcmp(stages, "0") != 0);
  if (st->backend == CTQW_BACKEND_TAYLOR || horner) {
    if (horner) sc.backend = CTQW_BACKEND_TAYLOR;
    sc.rk4_horner = horner ? 1 : 0;
    sc.order = horner ? 4 : st->order;
    for (int j = 1; j <= sc.order; ++j) sc.ci[j - 1] = c / (double)j;
  } else {
    sc.order = 4;
    sc.ci[0] = c;
  }
  return sc;
}

Coef coef_of(const ctqw_ctx* h) {
  Coef c{h->hop, h->site, h->stride, h->site_stride};
  if (h->general) {
    c.pos = h->lat_pos;
    c.neg = h->lat_neg;
    c.K = h->K;
  }
  return c;
}

int check_bound(ctqw_ctx* h, int64_t count) {
  if (h->needs_lattice && !h->general) return fail_with(h, CTQW_ERR_CONFIG, "no lattice tables (ctqw_set_lattice)");
  if (!h->hop) return fail_with(h, CTQW_ERR_CONFIG, "no coefficients bound (ctqw_bind_coefficients)");
  if (count < 0) return fail_with(h, CTQW_ERR_CONFIG, "negative realization count");
  if (h->stride != 0 && count > h->coef_count)
    return fail_with(h, CTQW_ERR_CONFIG, "more realizations than bound coefficient rows");
  return CTQW_OK;
}

// One generic step (no norm policy when partial == nullptr).
// in/out: Taylor reads `in`, writes `out` (may equal in only when scaled
// lazily through scl and n >= 2); A/C scratch term buffers, B accumulator.
int generic_step(ctqw_ctx* h, const ctqw_stepper_t* st, const StepScalars& sc, const double2* in,
                 double2* out, double2* A, double2* B, double2* C, int64_t count,
                 const double* scl, double* partial, const long long* fail, cudaStream_t s) {
  const Coef coef = coef_of(h);
  const bool exact = st->exact != 0;
  const bool scale = scl != nullptr;
  const bool inplace = (const void*)in == (const void*)out;
  long long launches = 0;
  const int64_t rows_chunks = (count + kMaxGridY - 1) / kMaxGridY;
  if (sc.backend == CTQW_BACKEND_TAYLOR) {
    const int n_ord = sc.order;
    const double2* term_in = in;
    double2* bufs[2] = {A, C};
    int which = 0;
    for (int j = 1; j <= n_ord; ++j) {
      const bool first = j == 1, last = j == n_ord;
      double2* term_out = last ? nullptr : bufs[which];
      const double2* acc_in = first ? in : B;
      double2* acc_out = (last && !(inplace && first)) ? out : B;
      CUDA_TRY(h, launch_taylor_order(h->m, exact, first && scale, term_in, term_out, acc_in,
                                      acc_out, count, h->dim, h->n, coef, h->k, sc.ci[j - 1],
                                      scl, last ? partial : nullptr, fail, s));
      launches += rows_chunks;
      if (!last) {
        term_in = bufs[which];
        which ^= 1;
      }
    }
    if (inplace && n_ord == 1) {
      CUDA_TRY(h, cudaMemcpyAsync(out, B, (size_t)count * h->dim * sizeof(double2),
                                  cudaMemcpyDeviceToDevice, s));
    }
  } else {
    const double ci = sc.ci[0];
    CUDA_TRY(h, launch_rk4_stage(h->m, exact, scale, 1, in, in, nullptr, A, B, count, h->dim,
                                 h->n, coef, h->k, ci, scl, nullptr, fail, s));
    CUDA_TRY(h, launch_rk4_stage(h->m, exact, scale, 2, A, in, B, C, B, count, h->dim, h->n, coef,
                                 h->k, ci, scl, nullptr, fail, s));
    CUDA_TRY(h, launch_rk4_stage(h->m, exact, scale, 3, C, in, B, A, B, count, h->dim, h->n, coef,
                                 h->k, ci, scl, nullptr, fail, s));
    CUDA_TRY(h, launch_rk4_stage(h->m, exact, false, 4, A, in, B, nullptr, out, count, h->dim,
                                 h->n, coef, h->k, ci, scl, partial, fail, s));
    launches += 4 * rows_chunks;
  }
  h->launches += launches;
  return CTQW_OK;
}

// Advance the bound telegraph process by dt and rewrite the couplings of
// switched elements (ensemble.py:536-544); a no-op for static noise.
int telegraph_step(ctqw_ctx* h, int64_t count, double dt, cudaStream_t s) {
  if (!h->tg_enabled) return CTQW_OK;
  if (count > h->tg_count) return fail_with(h, CTQW_ERR_CONFIG, "more realizations than the noise process holds");
  CUDA_TRY(h, launch_telegraph_advance(count, h->tg_total, h->tg_links, h->tg_sites, h->n, dt, h->tg_levels,
                                       h->tg_nlev, h->tg_mean_wait, h->t_slot, h->K, h->tg_values, h->tg_next,
                                       h->tg_gen, const_cast<double*>(h->hop), const_cast<double*>(h->site),
                                       h->stride, h->site_stride, h->tg_lists, h->tg_oldv, h->fail, s));
  h->launches += 1;
  return CTQW_OK;
}

}  // namespace

extern "C" {

int ctqw_abi_version(void) { return CTQW_ABI_VERSION; }

const char* ctqw_last_error(ctqw_handle_t h) { return h ? h->err.c_str() : g_err.c_str(); }

int ctqw_create(const ctqw_model_t* model, int32_t device, ctqw_handle_t* out) {
  if (!model || !out) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL argument");
  *out = nullptr;
  const ctqw_model_t& md = *model;
  if (md.m < 1 || md.m > 3)
    return fail_with(nullptr, CTQW_ERR_CONFIG, "the B200 path supports 1 <= m <= 3 particles");
  if (md.n_sites < 2) return fail_with(nullptr, CTQW_ERR_CONFIG, "the lattice needs n_sites >= 2");
  if (md.k_half < 1) return fail_with(nullptr, CTQW_ERR_CONFIG, "k_half (slots per site) must be >= 1");
  const bool ring = md.k_half == 1 && md.periodic == 1;
  if (ring && md.n_sites < 3)
    return fail_with(nullptr, CTQW_ERR_CONFIG, "ring needs n_sites >= 3 (2*k_half < extent)");
  for (double v : {md.onsite_energy, md.tunneling, md.interaction, md.hbar})
    if (!std::isfinite(v)) return fail_with(nullptr, CTQW_ERR_CONFIG, "model parameters must be finite");
  if (!(md.hbar > 0)) return fail_with(nullptr, CTQW_ERR_CONFIG, "hbar must be > 0");
  double dimd = std::pow((double)md.n_sites, md.m);
  if (dimd > 4.0e12) return fail_with(nullptr, CTQW_ERR_CAPACITY, "joint dimension too large");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail_with(nullptr, CTQW_ERR_OTHER, "no CUDA device available");
  }
  if (device < 0 || device >= ndev) return fail_with(nullptr, CTQW_ERR_CONFIG, "invalid device index");
  DeviceGuard g(device);
  ctqw_ctx* h = new ctqw_ctx();
  h->device = device;
  h->model = md;
  h->m = md.m;
  h->n = md.n_sites;
  h->K = md.k_half;
  h->needs_lattice = !ring;
  h->dim = 1;
  for (int p = 0; p < md.m; ++p) h->dim *= md.n_sites;
  for (int c = 0; c < 4; ++c) {
    // (m*eps0 + U*c), each product rounded as Python/NumPy does (hamiltonian.py:132)
    const double a = (double)md.m * md.onsite_energy;
    const double b = md.interaction * (double)c;
    h->k.base[c] = a + b;
  }
  if (cudaMalloc((void**)&h->fail, sizeof(long long)) != cudaSuccess ||
      cudaMalloc((void**)&h->summary_dev, sizeof(Summary)) != cudaSuccess ||
      cudaMallocHost((void**)&h->summary_host, sizeof(Summary)) != cudaSuccess ||
      cudaMalloc((void**)&h->small, 2 * 160 * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    ctqw_destroy(h);
    return fail_with(nullptr, CTQW_ERR_OTHER, "cannot allocate handle buffers");
  }
  long long nf = kNoFail;
  cudaMemcpy(h->fail, &nf, sizeof(nf), cudaMemcpyHostToDevice);
  // ring slot coupling (one slot, the model's t); ctqw_set_lattice replaces it
  if (cudaMalloc((void**)&h->t_slot, sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    ctqw_destroy(h);
    return fail_with(nullptr, CTQW_ERR_OTHER, "cannot allocate handle buffers");
  }
  cudaMemcpy(h->t_slot, &md.tunneling, sizeof(double), cudaMemcpyHostToDevice);
  if (const char* sk = std::getenv("CTQW_STREAM")) {
    h->stream_kind = std::strcmp(sk, "tile") == 0    ? 1
                     : std::strcmp(sk, "band4") == 0 ? 4
                     : std::strcmp(sk, "plane3") == 0 ? 5
                     : std::strcmp(sk, "generic") == 0 ? 6
                                                     : 0;
  }
  *out = h;
  return CTQW_OK;
}

int ctqw_destroy(ctqw_handle_t h) {
  if (!h) return CTQW_OK;
  DeviceGuard g(h->device);
  for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
  void* dev_ptrs[] = {h->levels, h->partial, h->scl, h->stats, h->events, h->fail,
                      h->summary_dev, h->scratch[0], h->scratch[1], h->n2_dev, h->small,
                      h->overlap_partial, h->tg_values, h->tg_next, h->tg_gen, h->tg_levels, h->tg_sum,
                      h->lat_pos, h->lat_neg, h->t_slot, h->scratch_work, h->fixed_acc,
                      h->tg_lists, h->tg_oldv, h->points_scratch};
  for (void* p : dev_ptrs)
    if (p) cudaFree(p);
  if (h->summary_host) cudaFreeHost(h->summary_host);
  delete h;
  return CTQW_OK;
}

int ctqw_draw_noise(ctqw_handle_t h, uint64_t master_seed, int64_t r0, int64_t count,
                    const double* levels_host, int32_t n_levels, int64_t total, double* noise_dev,
                    void* stream) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  if (n_levels < 1 || !levels_host) return fail_with(h, CTQW_ERR_CONFIG, "noise level set is empty");
  if (r0 < 0 || count < 0 || total < 0) return fail_with(h, CTQW_ERR_CONFIG, "negative sizes");
  for (int i = 0; i < n_levels; ++i)
    if (!std::isfinite(levels_host[i])) return fail_with(h, CTQW_ERR_CONFIG, "noise levels must be finite");
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  int rc = ensure(h, &h->levels, &h->levels_cap, n_levels, "noise levels");
  if (rc) return rc;
  CUDA_TRY(h, cudaMemcpyAsync(h->levels, levels_host, n_levels * sizeof(double),
                              cudaMemcpyHostToDevice, s));
  CUDA_TRY(h, launch_draw_noise(master_seed, r0, count, h->levels, n_levels, total, noise_dev, s));
  // levels_host may be freed by the caller after return
  CUDA_TRY(h, cudaStreamSynchronize(s));
  h->launches += 1;
  return CTQW_OK;
}

int ctqw_telegraph_init(ctqw_handle_t h, uint64_t master_seed, int64_t r0, int64_t count,
                        const double* levels_host, int32_t n_levels, int64_t n_links, int64_t n_sites,
                        double rate, void* stream) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  if (n_levels < 1 || !levels_host) return fail_with(h, CTQW_ERR_CONFIG, "noise level set is empty");
  if (r0 < 0 || count < 0 || n_links < 0 || n_sites < 0) return fail_with(h, CTQW_ERR_CONFIG, "negative sizes");
  if ((n_links != 0 && n_links != (int64_t)h->n * h->K) || (n_sites != 0 && n_sites != h->n))
    return fail_with(h, CTQW_ERR_CONFIG, "noise rows must hold 0 or N*K links and 0 or N sites");
  if (!(rate > 0.0) || !std::isfinite(rate)) return fail_with(h, CTQW_ERR_CONFIG, "telegraph rate must be > 0");
  for (int i = 0; i < n_levels; ++i)
    if (!std::isfinite(levels_host[i])) return fail_with(h, CTQW_ERR_CONFIG, "noise levels must be finite");
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t total = n_links + n_sites;
  int rc = ensure(h, &h->tg_values, &h->tg_cap, count * total, "telegraph values");
  if (rc) return rc;
  if (h->tg_next) cudaFree(h->tg_next);
  h->tg_next = nullptr;
  if (count * total > 0 && cudaMalloc(&h->tg_next, count * total * sizeof(double)) != cudaSuccess)
    return fail_with(h, CTQW_ERR_CAPACITY, "cannot allocate telegraph switch times");
  if (h->tg_gen) cudaFree(h->tg_gen);
  h->tg_gen = nullptr;
  if (count > 0 && cudaMalloc(&h->tg_gen, count * sizeof(TelegraphGen)) != cudaSuccess)
    return fail_with(h, CTQW_ERR_CAPACITY, "cannot allocate telegraph generators");
  for (void** p : {(void**)&h->tg_lists, (void**)&h->tg_oldv}) {
    if (*p) cudaFree(*p);
    *p = nullptr;
  }
  if (count * total > 0 && (cudaMalloc(&h->tg_lists, (size_t)count * total * 2 * sizeof(int)) != cudaSuccess ||
                            cudaMalloc(&h->tg_oldv, (size_t)count * total * sizeof(double)) != cudaSuccess))
    return fail_with(h, CTQW_ERR_CAPACITY, "cannot allocate the telegraph due lists");
  if (h->tg_levels) cudaFree(h->tg_levels);
  h->tg_levels = nullptr;
  if (cudaMalloc(&h->tg_levels, n_levels * sizeof(double)) != cudaSuccess)
    return fail_with(h, CTQW_ERR_CAPACITY, "cannot allocate noise levels");
  CUDA_TRY(h, cudaMemcpyAsync(h->tg_levels, levels_host, n_levels * sizeof(double), cudaMemcpyHostToDevice, s));
  h->tg_count = count;
  h->tg_total = total;
  h->tg_links = n_links;
  h->tg_sites = n_sites;
  h->tg_nlev = n_levels;
  h->tg_mean_wait = 1.0 / rate;  // noise.py:112 (_mean_wait = 1.0 / spec.rate)
  h->tg_enabled = false;
  if (total > 0)
    CUDA_TRY(h, launch_telegraph_init(master_seed, r0, count, h->tg_levels, n_levels, total, h->tg_mean_wait,
                                      h->tg_values, h->tg_next, h->tg_gen, s));
  CUDA_TRY(h, cudaStreamSynchronize(s));  // levels_host may be freed by the caller after return
  h->launches += 1;
  return CTQW_OK;
}

const double* ctqw_telegraph_values(ctqw_handle_t h) { return h ? h->tg_values : nullptr; }

int ctqw_telegraph_advance(ctqw_handle_t h, int64_t count, double dt, void* stream) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  if (!(dt >= 0.0) || !std::isfinite(dt)) return fail_with(h, CTQW_ERR_CONFIG, "advance window dt must be >= 0");
  if (count < 0 || count > h->tg_count) return fail_with(h, CTQW_ERR_CONFIG, "count exceeds the noise process");
  if (h->tg_total == 0 || count == 0) return CTQW_OK;
  DeviceGuard g(h->device);
  const bool coef = h->hop && h->coef_count >= count;
  CUDA_TRY(h, launch_telegraph_advance(count, h->tg_total, h->tg_links, h->tg_sites, h->n, dt, h->tg_levels,
                                       h->tg_nlev, h->tg_mean_wait, h->t_slot, h->K, h->tg_values, h->tg_next,
                                       h->tg_gen, coef ? const_cast<double*>(h->hop) : nullptr,
                                       coef ? const_cast<double*>(h->site) : nullptr, h->stride, h->site_stride,
                                       h->tg_lists, h->tg_oldv, nullptr, (cudaStream_t)stream));
  h->launches += 1;
  return CTQW_OK;
}

int ctqw_telegraph_enable(ctqw_handle_t h, int32_t enable) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  if (enable && h->tg_total > 0 && !h->tg_values)
    return fail_with(h, CTQW_ERR_CONFIG, "no telegraph process (ctqw_telegraph_init)");
  h->tg_enabled = enable != 0 && h->tg_total > 0;
  return CTQW_OK;
}

int ctqw_telegraph_read(ctqw_handle_t h, double* values_dev, double* next_switch_dev, double* times_host,
                        int64_t* switches_host, void* stream) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bytes = (size_t)h->tg_count * h->tg_total * sizeof(double);
  if (values_dev && bytes) CUDA_TRY(h, cudaMemcpyAsync(values_dev, h->tg_values, bytes, cudaMemcpyDeviceToDevice, s));
  if (next_switch_dev && bytes)
    CUDA_TRY(h, cudaMemcpyAsync(next_switch_dev, h->tg_next, bytes, cudaMemcpyDeviceToDevice, s));
  if ((times_host || switches_host) && h->tg_count) {
    std::vector<TelegraphGen> gens(h->tg_count);
    CUDA_TRY(h, cudaMemcpyAsync(gens.data(), h->tg_gen, h->tg_count * sizeof(TelegraphGen), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(h, cudaStreamSynchronize(s));
    for (int64_t i = 0; i < h->tg_count; ++i) {
      if (times_host) times_host[i] = gens[i].time;
      if (switches_host) switches_host[i] = gens[i].switches;
    }
  }
  return CTQW_OK;
}

int ctqw_set_lattice(ctqw_handle_t h, int32_t n_slots, const int32_t* pos_host, const int32_t* neg_host,
                     const double* t_slot_host) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  if (n_slots != h->K) return fail_with(h, CTQW_ERR_CONFIG, "n_slots must equal the model's k_half (slots per site)");
  if (!pos_host || !neg_host || !t_slot_host) return fail_with(h, CTQW_ERR_CONFIG, "NULL lattice table");
  const int64_t nk = (int64_t)h->n * n_slots;
  for (int64_t i = 0; i < nk; ++i)
    if (pos_host[i] < -1 || pos_host[i] >= h->n || neg_host[i] < -1 || neg_host[i] >= h->n)
      return fail_with(h, CTQW_ERR_CONFIG, "lattice move targets out of range");
  for (int s = 0; s < n_slots; ++s)
    if (!std::isfinite(t_slot_host[s])) return fail_with(h, CTQW_ERR_CONFIG, "tunneling amplitudes must be finite");
  DeviceGuard g(h->device);
  for (int** p : {&h->lat_pos, &h->lat_neg}) {
    if (*p) cudaFree(*p);
    *p = nullptr;
    if (cudaMalloc((void**)p, nk * sizeof(int)) != cudaSuccess)
      return fail_with(h, CTQW_ERR_CAPACITY, "cannot allocate lattice tables");
  }
  if (h->t_slot) cudaFree(h->t_slot);
  h->t_slot = nullptr;
  if (cudaMalloc((void**)&h->t_slot, n_slots * sizeof(double)) != cudaSuccess)
    return fail_with(h, CTQW_ERR_CAPACITY, "cannot allocate lattice tables");
  CUDA_TRY(h, cudaMemcpy(h->lat_pos, pos_host, nk * sizeof(int), cudaMemcpyHostToDevice));
  CUDA_TRY(h, cudaMemcpy(h->lat_neg, neg_host, nk * sizeof(int), cudaMemcpyHostToDevice));
  CUDA_TRY(h, cudaMemcpy(h->t_slot, t_slot_host, n_slots * sizeof(double), cudaMemcpyHostToDevice));
  h->general = true;
  return CTQW_OK;
}

int ctqw_build_coefficients(ctqw_handle_t h, const double* noise_dev, int64_t count,
                            int64_t n_links, int64_t n_sites, double* hop_dev, double* site_dev,
                            void* stream) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  if ((n_links != 0 && n_links != (int64_t)h->n * h->K) || (n_sites != 0 && n_sites != h->n))
    return fail_with(h, CTQW_ERR_CONFIG, "noise rows must hold 0 or N*K links and 0 or N sites");
  if (n_sites && !site_dev) return fail_with(h, CTQW_ERR_CONFIG, "site_dev required for on-site noise");
  if ((n_links || n_sites) && !noise_dev) return fail_with(h, CTQW_ERR_CONFIG, "noise_dev is NULL");
  if (h->needs_lattice && !h->general) return fail_with(h, CTQW_ERR_CONFIG, "no lattice tables (ctqw_set_lattice)");
  DeviceGuard g(h->device);
  CUDA_TRY(h, launch_build_coef(noise_dev, count, h->n, h->K, n_links, n_sites, h->t_slot,
                                hop_dev, site_dev, (cudaStream_t)stream));
  h->launches += 1;
  return CTQW_OK;
}

int ctqw_bind_coefficients(ctqw_handle_t h, int64_t count, const double* hop_dev,
                           const double* site_dev, int64_t stride) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  if (!hop_dev) return fail_with(h, CTQW_ERR_CONFIG, "hop_dev is NULL");
  if (stride != 0 && stride != (int64_t)h->n * h->K) return fail_with(h, CTQW_ERR_CONFIG, "stride must be 0 or N*K");
  h->coef_count = count;
  h->hop = hop_dev;
  h->site = site_dev;
  h->stride = stride;
  h->site_stride = stride ? h->n : 0;
  return CTQW_OK;
}

int ctqw_fill_states(ctqw_handle_t h, double* psi_dev, int64_t count, const double* psi0_dev,
                     void* stream) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  DeviceGuard g(h->device);
  CUDA_TRY(h, launch_fill_states((double2*)psi_dev, count, h->dim, (const double2*)psi0_dev,
                                 (cudaStream_t)stream));
  h->launches += 1;
  h->initial = nullptr;
  return CTQW_OK;
}

int ctqw_set_initial(ctqw_handle_t h, const double* psi0_dev) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  h->initial = (const double2*)psi0_dev;
  return CTQW_OK;
}

int ctqw_apply(ctqw_handle_t h, const double* psi_dev, double* out_dev, int64_t count,
               int32_t exact, void* stream) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  int rc = check_bound(h, count);
  if (rc) return rc;
  if (count == 0) return CTQW_OK;
  DeviceGuard g(h->device);
  CUDA_TRY(h, launch_apply(h->m, (const double2*)psi_dev, (double2*)out_dev, count, h->dim, h->n,
                           coef_of(h), h->k, exact != 0, (cudaStream_t)stream));
  h->launches += (count + kMaxGridY - 1) / kMaxGridY;
  return CTQW_OK;
}

int ctqw_step(ctqw_handle_t h, const double* psi_dev, double* out_dev, int64_t count,
              const ctqw_stepper_t* stepper, void* stream) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  int rc = validate_stepper(h, stepper);
  if (rc) return rc;
  rc = check_bound(h, count);
  if (rc) return rc;
  if (psi_dev == out_dev) return fail_with(h, CTQW_ERR_CONFIG, "out must not alias psi");
  if (count == 0) return CTQW_OK;
  DeviceGuard g(h->device);
  rc = ensure_scratch(h, count * h->dim);
  if (rc) return rc;
  const StepScalars sc = scalars_for(h, stepper);
  // Taylor: term buffers scratch[0]/[1], accumulator straight into out.
  return generic_step(h, stepper, sc, (const double2*)psi_dev, (double2*)out_dev, h->scratch[0],
                      (double2*)out_dev, h->scratch[1], count, nullptr, nullptr, nullptr,
                      (cudaStream_t)stream);
}

int ctqw_check_norm(ctqw_handle_t h, double* psi_dev, int64_t count, const ctqw_stepper_t* st,
                    double* deviations_dev, int32_t* corrected_dev, int64_t* fail_row,
                    double* fail_deviation, void* stream) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  if (!st) return fail_with(h, CTQW_ERR_CONFIG, "stepper is NULL");
  if (!(0 < st->tol_norm && st->tol_norm < st->tol_fail))
    return fail_with(h, CTQW_ERR_CONFIG, "need 0 < tol_norm < tol_fail");
  if (count == 0) return CTQW_OK;
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int nparts = generic_parts(h->dim);
  int rc = ensure(h, &h->partial, &h->partial_cap, count * nparts, "norm partials");
  if (rc) return rc;
  rc = ensure(h, &h->n2_dev, &h->n2_cap, 2 * count, "norm scratch");
  if (rc) return rc;
  CUDA_TRY(h, launch_norm_partial((const double2*)psi_dev, count, h->dim, h->partial, s));
  CUDA_TRY(h, launch_norm_sum(h->partial, nparts, count, h->n2_dev, s));
  h->launches += 2;
  std::vector<double> n2(count), dev(count), scale(count, 1.0);
  std::vector<int32_t> corr(count, 0);
  CUDA_TRY(h, cudaMemcpyAsync(n2.data(), h->n2_dev, count * sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(h, cudaStreamSynchronize(s));
  int64_t worst = 0;
  bool failed = false;
  for (int64_t r = 0; r < count; ++r) {
    dev[r] = std::fabs(n2[r] - 1.0);
    if (dev[r] > dev[worst]) worst = r;
    if (dev[r] > st->tol_fail) failed = true;
  }
  if (deviations_dev)
    CUDA_TRY(h, cudaMemcpyAsync(deviations_dev, dev.data(), count * sizeof(double),
                                cudaMemcpyHostToDevice, s));
  if (failed) {
    if (fail_row) *fail_row = worst;
    if (fail_deviation) *fail_deviation = dev[worst];
    if (corrected_dev) CUDA_TRY(h, cudaMemsetAsync(corrected_dev, 0, count * sizeof(int32_t), s));
    CUDA_TRY(h, cudaStreamSynchronize(s));
    char buf[160];
    snprintf(buf, sizeof buf, "norm deviation %.3e exceeds the failure threshold (row %lld)",
             dev[worst], (long long)worst);
    return fail_with(h, CTQW_ERR_NUMERIC, buf);
  }
  bool any = false;
  if (st->renormalize) {
    for (int64_t r = 0; r < count; ++r)
      if (dev[r] > st->tol_norm) {
        corr[r] = 1;
        scale[r] = 1.0 / std::sqrt(n2[r]);
        any = true;
      }
  }
  if (corrected_dev)
    CUDA_TRY(h, cudaMemcpyAsync(corrected_dev, corr.data(), count * sizeof(int32_t),
                                cudaMemcpyHostToDevice, s));
  if (any) {
    CUDA_TRY(h, cudaMemcpyAsync(h->n2_dev + count, scale.data(), count * sizeof(double),
                                cudaMemcpyHostToDevice, s));
    CUDA_TRY(h, launch_scale_rows((double2*)psi_dev, count, h->dim, h->n2_dev + count, s));
    h->launches += 1;
  }
  CUDA_TRY(h, cudaStreamSynchronize(s));
  return CTQW_OK;
}

namespace {

// Fused collection target of ctqw_evolve_observe (resident64 path only).
struct ObsTarget {
  unsigned long long* acc = nullptr;
  long long post_rate = 1;
  long long origin = 0;  // the call's first_step: points at origin + k * post_rate and at final_step
  long long final_step = 0;
  double2* snap = nullptr;  // optional states at each point [point][count][dim]
};

// Does this handle's evolve run the N = 64 block kernel (which can fuse the
// collection into the step)?
bool uses_resident64(const ctqw_ctx* h, const StepScalars& sc) {
  return h->stream_kind == 0 && !h->general && resident_supported(h->m, h->n, sc) &&
         resident64_supported(h->m, h->n, sc) && !std::getenv("CTQW_RESIDENT_STRIP");
}

int evolve_impl(ctqw_ctx* h, double* psi_dev, double* work_dev, int64_t count, int64_t first_step,
                int64_t n_steps, const ctqw_stepper_t* st, int32_t* result_in_work, cudaStream_t s, bool reset,
                const ObsTarget& obs);

}  // namespace

int ctqw_evolve(ctqw_handle_t h, double* psi_dev, double* work_dev, int64_t count,
                int64_t first_step, int64_t n_steps, const ctqw_stepper_t* st,
                int32_t* result_in_work, void* stream) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  int rc = validate_stepper(h, st);
  if (rc) return rc;
  rc = check_bound(h, count);
  if (rc) return rc;
  if (n_steps < 0 || first_step < 0) return fail_with(h, CTQW_ERR_CONFIG, "negative step count");
  DeviceGuard g(h->device);
  return evolve_impl(h, psi_dev, work_dev, count, first_step, n_steps, st, result_in_work, (cudaStream_t)stream,
                     true, ObsTarget{});
}

int ctqw_evolve_observe(ctqw_handle_t h, double* psi_dev, double* work_dev, int64_t count, int64_t first_step,
                        int64_t n_steps, int64_t post_rate, int64_t* acc_dev, double* snap_dev,
                        const ctqw_stepper_t* st, int32_t keep_stats, int32_t* result_in_work, void* stream) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  int rc = validate_stepper(h, st);
  if (rc) return rc;
  rc = check_bound(h, count);
  if (rc) return rc;
  if (n_steps < 1 || first_step < 0 || post_rate < 1)
    return fail_with(h, CTQW_ERR_CONFIG, "evolve_observe needs n_steps >= 1, first_step >= 0, post_rate >= 1");
  if (!acc_dev) return fail_with(h, CTQW_ERR_CONFIG, "NULL limb accumulator");
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t last = first_step + n_steps;
  const int64_t npoints = (n_steps + post_rate - 1) / post_rate;
  CUDA_TRY(h, cudaMemsetAsync(acc_dev, 0, (size_t)npoints * 3 * h->dim * sizeof(int64_t), s));
  if (result_in_work) *result_in_work = 0;
  const StepScalars sc = scalars_for(h, st);
  if (uses_resident64(h, sc)) {
    ObsTarget o;
    o.acc = reinterpret_cast<unsigned long long*>(acc_dev);
    o.post_rate = post_rate;
    o.origin = first_step;
    o.final_step = last;
    o.snap = (double2*)snap_dev;
    return evolve_impl(h, psi_dev, work_dev, count, first_step, n_steps, st, result_in_work, s, !keep_stats, o);
  }
  // every other path: one segment per collection point, then the separate
  // exact-limb pass over the state (the same bits as the fused form)
  double* cur = psi_dev;
  double* other = work_dev;
  int64_t done = first_step;
  for (int64_t idx = 0; idx < npoints; ++idx) {
    const int64_t target = std::min<int64_t>(last, first_step + (idx + 1) * post_rate);
    int32_t swapped = 0;
    rc = evolve_impl(h, cur, other, count, done, target - done, st, &swapped, s, idx == 0 && !keep_stats,
                     ObsTarget{});
    if (rc) return rc;
    if (swapped) std::swap(cur, other);
    done = target;
    CUDA_TRY(h, launch_observe_diag_fixed((const double2*)cur, count, h->dim,
                                          reinterpret_cast<unsigned long long*>(acc_dev) + idx * 3 * h->dim, true,
                                          s));
    h->launches += 1;
    if (snap_dev)
      CUDA_TRY(h, cudaMemcpyAsync(snap_dev + idx * count * h->dim * 2, cur, (size_t)count * h->dim * sizeof(double2),
                                  cudaMemcpyDeviceToDevice, s));
  }
  if (result_in_work) *result_in_work = cur == psi_dev ? 0 : 1;
  return CTQW_OK;
}

namespace {

int evolve_impl(ctqw_ctx* h, double* psi_dev, double* work_dev, int64_t count, int64_t first_step,
                int64_t n_steps, const ctqw_stepper_t* st, int32_t* result_in_work, cudaStream_t s, bool reset,
                const ObsTarget& obs) {
  int rc = CTQW_OK;
  if (result_in_work) *result_in_work = 0;
  rc = ensure_stats(h, count);
  if (rc) return rc;
  h->last_count = count;
  if (reset) {
    CUDA_TRY(h, launch_reset_stats(h->stats, h->scl, count, h->fail, s));
    h->launches += 1;
  }
  if (count == 0 || n_steps == 0) {
    if (h->initial && count > 0) {  // nothing to step: the stack is the initial state
      CUDA_TRY(h, launch_fill_states((double2*)psi_dev, count, h->dim, h->initial, s));
      h->launches += 1;
    }
    h->initial = nullptr;
    return CTQW_OK;
  }
  const StepScalars sc = scalars_for(h, st);
  const NormPolicy pol{st->tol_norm, st->tol_fail, st->renormalize};
  const bool exact = st->exact != 0;
  const Coef coef = coef_of(h);
  double2* psi = (double2*)psi_dev;
  double2* work = (double2*)work_dev;

  if (h->needs_lattice && !h->general) return fail_with(h, CTQW_ERR_CONFIG, "no lattice tables (ctqw_set_lattice)");
  // a pinned streaming family (CTQW_STREAM) bypasses the resident path;
  // general lattices (move tables) run on the generic kernels only
  if (h->stream_kind == 0 && !h->general && resident_supported(h->m, h->n, sc)) {
    // N = 64 with <= 4 applications per step: the 4 x 4-block kernel
    // (resident64.cu); other sizes / orders: the column-strip kernel
    const bool r64 = uses_resident64(h, sc);
    h->stream_kernel = r64 ? "resident64_kernel" : "resident_kernel";
    std::snprintf(h->variant, sizeof(h->variant), "%s<%s,order=%d,site=%d,exact=%d,N=%d>", h->stream_kernel,
                  integ_label(sc), sc.order, coef.site != nullptr ? 1 : 0, exact ? 1 : 0, h->n);
    // a pending initial state: resident64 reads it directly, the strip kernel
    // needs the stack materialised
    const double2* init = h->initial;
    h->initial = nullptr;
    if (init && !r64) {
      CUDA_TRY(h, launch_fill_states(psi, count, h->dim, init, s));
      h->launches += 1;
      init = nullptr;
    }
    // dynamic noise changes the couplings after every step: one step per launch
    const int64_t chunk = h->tg_enabled ? 1 : n_steps;
    for (int64_t j = 0; j < n_steps; j += chunk) {
      timing_event(h, s);
      if (r64)
        CUDA_TRY(h, launch_resident64(psi, count, coef, h->k, sc, exact, pol, first_step + j, chunk, h->stats,
                                      h->events, h->fail, s, obs.acc, obs.post_rate, obs.origin, obs.final_step,
                                      j == 0 ? init : nullptr, obs.snap));
      else
        CUDA_TRY(h, launch_resident(psi, count, h->n, coef, h->k, sc, exact, pol, first_step + j, chunk,
                                    h->stats, h->events, h->fail, s));
      timing_event(h, s);
      h->timed_launches += h->timing ? 1 : 0;
      h->launches += 1;
      rc = telegraph_step(h, count, st->dt, s);
      if (rc) return rc;
    }
    return CTQW_OK;
  }
  // plane3 (m = 3, N = 128) updates psi in place; every other streaming or
  // generic path needs a second buffer: the caller's, or (work NULL / aliased
  // to psi) a library-owned one
  const bool plane3_path = (h->stream_kind == 0 || h->stream_kind == 5) && !h->general &&
                           plane3_supported(h->m, h->n, sc);
  if (!plane3_path && (!work || work == psi)) {
    if (!h->scratch_work || h->scratch_work_elems < count * h->dim) {
      if (h->scratch_work) cudaFree(h->scratch_work);
      h->scratch_work = nullptr;
      h->scratch_work_elems = 0;
      if (cudaMalloc((void**)&h->scratch_work, (size_t)count * h->dim * sizeof(double2)) != cudaSuccess)
        return fail_with(h, CTQW_ERR_CAPACITY, "cannot allocate the second state buffer");
      h->scratch_work_elems = count * h->dim;
    }
    work = h->scratch_work;
  }
  if (!work) work = psi;
  // streaming m = 2 path: the four-column band kernel (N % 4 == 0, N <= 1024);
  // the tile kernel covers the other m = 2 sizes.  CTQW_STREAM pins one
  // family (A/B measurements, per-kernel parity tests); a pinned family that
  // does not support the case falls through to the next one in auto order.
  const int kind = h->general ? 6 : h->stream_kind;
  const bool use_band4 = (kind == 0 || kind == 4) && band4_supported(h->m, h->n, sc);
  const bool use_plane3 = (kind == 0 || kind == 5) && plane3_supported(h->m, h->n, sc);
  const bool use_tile = !use_band4 && kind < 5 && tile_supported(h->m, h->n, sc);
  if (use_plane3 || use_band4 || use_tile) {
    h->stream_kernel = use_plane3 ? "plane3_kernel" : use_band4 ? "band4_kernel" : "tile_step_kernel";
    {
      const int napp = sc.backend == CTQW_BACKEND_RK4 ? 4 : sc.order;
      // band4 compiles N in for the four-application steps at the BASELINE sizes
      const int nn = (use_band4 && napp == 4 && (h->n == 256 || h->n == 512 || h->n == 1024)) ? h->n
                     : use_plane3 ? 128 : 0;
      // band4's zero-diagonal form (eps0 = U = 0) at the compile-time sizes
      const bool zd = h->k.base[0] == 0.0 && h->k.base[1] == 0.0 && h->k.base[2] == 0.0 && h->k.base[3] == 0.0;
      // (plane3: without site noise)
      const int dg = ((use_band4 && nn > 0 && zd) || (use_plane3 && zd && coef.site == nullptr)) ? 0 : 2;
      std::snprintf(h->variant, sizeof(h->variant), "%s<%s,napp=%d,site=%d,exact=%d,NN=%d,dg=%d>", h->stream_kernel,
                    integ_label(sc), napp, coef.site != nullptr ? 1 : 0,
                    exact ? 1 : 0, nn, dg);
    }
    const int nparts = use_plane3 ? plane3_parts()
                       : use_band4 ? band4_parts(h->n)
                                  : tile_parts(h->n, sc);
    rc = ensure(h, &h->partial, &h->partial_cap, count * nparts, "norm partials");
    if (rc) return rc;
    // a pending initial state: band4's first step reads it as one shared
    // input (no materialised stack); plane3 (in place) and tile need the stack
    const double2* init = h->initial;
    h->initial = nullptr;
    if (init && !use_band4) {
      CUDA_TRY(h, launch_fill_states(psi, count, h->dim, init, s));
      h->launches += 1;
      init = nullptr;
    }
    // plane3 marches in place (output planes 0..3 parked until the march ends)
    double2* bufs[2] = {psi, use_plane3 ? psi : work};
    for (int64_t j = 0; j < n_steps; ++j) {
      const bool from_init = j == 0 && init != nullptr;
      const double2* in = from_init ? init : bufs[j & 1];
      double2* out = bufs[(j + 1) & 1];
      timing_event(h, s);
      if (use_plane3)
        CUDA_TRY(h, launch_plane3_step(in, out, count, coef, h->k, sc, exact, h->scl, h->partial, h->fail, s));
      else if (use_band4)
        CUDA_TRY(h, launch_band4_step(in, out, count, h->n, coef, h->k, sc, exact, h->scl, h->partial,
                                      h->fail, s, from_init));
      else
        CUDA_TRY(h, launch_tile_step(in, out, count, h->n, coef, h->k, sc, exact, h->scl, h->partial,
                                     h->fail, s));
      timing_event(h, s);
      h->timed_launches += h->timing ? 1 : 0;
      CUDA_TRY(h, launch_norm_decide(h->partial, nparts, count, (long long)(first_step + j + 1), pol,
                                     h->scl, h->stats, h->events, h->fail, s));
      h->launches += 2 * ((count + kMaxGridY - 1) / kMaxGridY);
      rc = telegraph_step(h, count, st->dt, s);
      if (rc) return rc;
    }
    double2* final_buf = bufs[n_steps & 1];
    if (final_buf != psi && final_buf == h->scratch_work) {  // library-owned second buffer: result back to psi
      CUDA_TRY(h, cudaMemcpyAsync(psi, final_buf, (size_t)count * h->dim * sizeof(double2),
                                  cudaMemcpyDeviceToDevice, s));
      final_buf = psi;
    }
    CUDA_TRY(h, launch_rescale(final_buf, count, h->dim, h->scl, s));
    h->launches += 2;
    if (result_in_work) *result_in_work = final_buf == psi ? 0 : 1;
    return CTQW_OK;
  }
  if (h->initial) {  // the generic kernels step the stack in place
    CUDA_TRY(h, launch_fill_states(psi, count, h->dim, h->initial, s));
    h->launches += 1;
    h->initial = nullptr;
  }
  // generic path: in place on psi; work = term buffer A, library scratch B, C
  h->stream_kernel = sc.backend == CTQW_BACKEND_TAYLOR ? "taylor_order_kernel" : "rk4_stage_kernel";
  std::snprintf(h->variant, sizeof(h->variant), "%s<%sorder=%d,site=%d,exact=%d>", h->stream_kernel,
                sc.rk4_horner ? "rk4=taylor4," : "", sc.order, coef.site != nullptr ? 1 : 0, exact ? 1 : 0);
  rc = ensure_scratch(h, count * h->dim);
  if (rc) return rc;
  const int nparts = generic_parts(h->dim);
  rc = ensure(h, &h->partial, &h->partial_cap, count * nparts, "norm partials");
  if (rc) return rc;
  for (int64_t j = 0; j < n_steps; ++j) {
    timing_event(h, s);
    rc = generic_step(h, st, sc, psi, psi, work, h->scratch[0], h->scratch[1], count, h->scl,
                      h->partial, h->fail, s);
    if (rc) return rc;
    timing_event(h, s);
    h->timed_launches += h->timing ? 1 : 0;
    CUDA_TRY(h, launch_norm_decide(h->partial, nparts, count, (long long)(first_step + j + 1), pol,
                                   h->scl, h->stats, h->events, h->fail, s));
    h->launches += 1;
    rc = telegraph_step(h, count, st->dt, s);
    if (rc) return rc;
  }
  CUDA_TRY(h, launch_rescale(psi, count, h->dim, h->scl, s));
  h->launches += 2;
  return CTQW_OK;
}

}  // namespace

int ctqw_segment_stats(ctqw_handle_t h, int64_t r0, ctqw_segment_stats_t* out, void* stream) {
  if (!h || !out) return fail_with(h, CTQW_ERR_CONFIG, "NULL argument");
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  std::memset(out, 0, sizeof(*out));
  const int64_t count = h->last_count;
  if (count == 0) {
    CUDA_TRY(h, cudaStreamSynchronize(s));
    return CTQW_OK;
  }
  CUDA_TRY(h, launch_stats_reduce(h->stats, count, h->summary_dev, s));
  h->launches += 1;
  CUDA_TRY(h, cudaMemcpyAsync(h->summary_host, h->summary_dev, sizeof(Summary),
                              cudaMemcpyDeviceToHost, s));
  CUDA_TRY(h, cudaStreamSynchronize(s));
  const Summary sm = *h->summary_host;
  out->event_count = sm.events;
  out->corrections = sm.corrections;
  out->max_deviation = sm.max_dev;
  if (sm.events > 0) {
    // First MAX_EVENTS events in (step, realization) order: each
    // realization's own first events are stored in step order.
    std::vector<RealStat> stats(count);
    std::vector<EventRec> evs((size_t)count * kMaxEvents);
    CUDA_TRY(h, cudaMemcpy(stats.data(), h->stats, count * sizeof(RealStat), cudaMemcpyDeviceToHost));
    CUDA_TRY(h, cudaMemcpy(evs.data(), h->events, (size_t)count * kMaxEvents * sizeof(EventRec),
                           cudaMemcpyDeviceToHost));
    struct Item {
      long long step;
      int64_t r;
      double dev;
      int corrected;
    };
    std::vector<Item> items;
    for (int64_t r = 0; r < count; ++r)
      for (int e = 0; e < stats[r].n_ev; ++e) {
        const EventRec& rec = evs[(size_t)r * kMaxEvents + e];
        items.push_back(Item{rec.step_lo, r, rec.dev, rec.corrected});
      }
    const size_t keep = std::min<size_t>(items.size(), CTQW_MAX_EVENTS);
    std::partial_sort(items.begin(), items.begin() + keep, items.end(),
                      [](const Item& a, const Item& b) {
                        return a.step != b.step ? a.step < b.step : a.r < b.r;
                      });
    for (size_t i = 0; i < keep; ++i) {
      out->events[i].deviation = items[i].dev;
      out->events[i].realization = r0 + items[i].r;
      out->events[i].step = items[i].step;
      out->events[i].corrected = items[i].corrected;
    }
    out->n_events = (int32_t)keep;
  }
  if (sm.fail_step != kNoFail) {
    out->failed = 1;
    out->fail_realization = r0 + sm.fail_row;
    out->fail_step = sm.fail_step;
    out->fail_deviation = sm.fail_dev;
    char buf[200];
    snprintf(buf, sizeof buf,
             "norm deviation %.3e exceeds the failure threshold (realization %lld, step %lld); "
             "reduce the time step",
             sm.fail_dev, (long long)(r0 + sm.fail_row), (long long)sm.fail_step);
    return fail_with(h, CTQW_ERR_NUMERIC, buf);
  }
  return CTQW_OK;
}

int ctqw_observe_diag_fixed(ctqw_handle_t h, const double* psi_dev, int64_t count, int64_t* acc_dev,
                            int32_t accumulate, void* stream) {
  if (!h || !acc_dev) return fail_with(h, CTQW_ERR_CONFIG, "NULL argument");
  if (count < 0) return fail_with(h, CTQW_ERR_CONFIG, "negative realization count");
  if (count > 0 && !psi_dev) return fail_with(h, CTQW_ERR_CONFIG, "NULL state stack");
  DeviceGuard g(h->device);
  CUDA_TRY(h, launch_observe_diag_fixed((const double2*)psi_dev, count, h->dim, (unsigned long long*)acc_dev,
                                        accumulate != 0, (cudaStream_t)stream));
  h->launches += 1;
  return CTQW_OK;
}

int ctqw_fixed_to_double(ctqw_handle_t h, const int64_t* acc_dev, double* diag_dev, void* stream) {
  if (!h || !acc_dev || !diag_dev) return fail_with(h, CTQW_ERR_CONFIG, "NULL argument");
  DeviceGuard g(h->device);
  CUDA_TRY(h, launch_fixed_to_double((const unsigned long long*)acc_dev, h->dim, diag_dev, (cudaStream_t)stream));
  h->launches += 1;
  return CTQW_OK;
}

int ctqw_observe_diag(ctqw_handle_t h, const double* psi_dev, int64_t count, double* diag_sum_dev,
                      int32_t accumulate, void* stream) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  int rc = ensure(h, &h->fixed_acc, &h->fixed_cap, 3 * h->dim, "diagonal limbs");
  if (rc) return rc;
  if (accumulate) {
    CUDA_TRY(h, launch_fixed_from_double(diag_sum_dev, h->dim, h->fixed_acc, s));
    h->launches += 1;
  }
  CUDA_TRY(h, launch_observe_diag_fixed((const double2*)psi_dev, count, h->dim, h->fixed_acc, accumulate != 0, s));
  CUDA_TRY(h, launch_fixed_to_double(h->fixed_acc, h->dim, diag_sum_dev, s));
  h->launches += 2;
  return CTQW_OK;
}

int ctqw_observe_reduce(ctqw_handle_t h, const double* diag_sum_dev, double total_count,
                        double* populations_dev, double* scalars_dev, double* joint_dev,
                        void* stream) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  if (!(total_count > 0)) return fail_with(h, CTQW_ERR_CONFIG, "total_count must be > 0");
  DeviceGuard g(h->device);
  CUDA_TRY(h, launch_observe_reduce(h->m, h->n, h->dim, diag_sum_dev, total_count, populations_dev,
                                    scalars_dev, joint_dev, h->small, (cudaStream_t)stream));
  h->launches += populations_dev ? 3 : 2;
  return CTQW_OK;
}

int ctqw_overlap_sumsq(ctqw_handle_t h, const double* a_dev, int64_t count_a, const double* b_dev,
                       int64_t count_b, double* sumsq_dev, void* stream) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  if (count_a <= 0 || count_b <= 0) return fail_with(h, CTQW_ERR_CONFIG, "empty state stack");
  DeviceGuard g(h->device);
  const bool same = a_dev == b_dev && count_a == count_b;
  const int64_t need = overlap_scratch_doubles(count_a, count_b, same, h->dim) + 2;
  int rc = ensure(h, &h->overlap_partial, &h->overlap_cap, need, "overlap partials");
  if (rc) return rc;
  CUDA_TRY(h, launch_overlap_sumsq((const double2*)a_dev, count_a, (const double2*)b_dev, count_b,
                                   h->dim, h->overlap_partial, h->overlap_cap, sumsq_dev,
                                   (cudaStream_t)stream));
  h->launches += 3;
  return CTQW_OK;
}

int ctqw_overlap_sumsq_points(ctqw_handle_t h, const double* stacks_dev, int64_t count, int64_t npoints,
                              int64_t point_stride, double* sumsq_dev, void* stream) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  if (count <= 0) return fail_with(h, CTQW_ERR_CONFIG, "empty state stack");
  if (npoints <= 0 || npoints > 65535) return fail_with(h, CTQW_ERR_CONFIG, "npoints must be in 1..65535");
  if (npoints > 1 && point_stride < count * h->dim)
    return fail_with(h, CTQW_ERR_CONFIG, "point_stride smaller than one state stack");
  DeviceGuard g(h->device);
  const int64_t need = overlap_scratch_doubles(count, count, true, h->dim, npoints) + 2;
  int rc = ensure(h, &h->overlap_partial, &h->overlap_cap, need, "overlap partials");
  if (rc) return rc;
  const double2* a = (const double2*)stacks_dev;
  CUDA_TRY(h, launch_overlap_sumsq(a, count, a, count, h->dim, h->overlap_partial, h->overlap_cap, sumsq_dev,
                                   (cudaStream_t)stream, npoints, point_stride));
  h->launches += 3;
  return CTQW_OK;
}

int ctqw_packed_gram(const double* psi_dev, int64_t count, int64_t dim, double scale, double* packed_dev,
                     int32_t device, void* stream) {
  if (count <= 0) return fail_with(nullptr, CTQW_ERR_CONFIG, "empty state stack");
  if (dim <= 0) return fail_with(nullptr, CTQW_ERR_CONFIG, "dimension must be positive");
  if (!psi_dev || !packed_dev) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL buffer");
  DeviceGuard g(device);
  CUDA_TRY(nullptr, launch_packed_gram((const double2*)psi_dev, count, dim, scale, (double2*)packed_dev,
                                       (cudaStream_t)stream));
  return CTQW_OK;
}

int ctqw_segment_events(ctqw_handle_t h, int64_t r0, int64_t step_lo, int64_t step_hi, ctqw_segment_stats_t* out,
                        void* stream) {
  if (!h || !out) return fail_with(h, CTQW_ERR_CONFIG, "NULL argument");
  DeviceGuard g(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  std::memset(out, 0, sizeof(*out));
  const int64_t count = h->last_count;
  CUDA_TRY(h, cudaStreamSynchronize(s));
  if (count == 0) return CTQW_OK;
  std::vector<RealStat> stats(count);
  std::vector<EventRec> evs((size_t)count * kMaxEvents);
  CUDA_TRY(h, cudaMemcpy(stats.data(), h->stats, count * sizeof(RealStat), cudaMemcpyDeviceToHost));
  CUDA_TRY(h, cudaMemcpy(evs.data(), h->events, (size_t)count * kMaxEvents * sizeof(EventRec),
                         cudaMemcpyDeviceToHost));
  struct Item {
    long long step;
    int64_t r;
    double dev;
    int corrected;
  };
  std::vector<Item> items;
  for (int64_t r = 0; r < count; ++r)
    for (int e = 0; e < stats[r].n_ev; ++e) {
      const EventRec& rec = evs[(size_t)r * kMaxEvents + e];
      if (rec.step_lo > step_lo && rec.step_lo <= step_hi) items.push_back(Item{rec.step_lo, r, rec.dev, rec.corrected});
    }
  const size_t keep = std::min<size_t>(items.size(), CTQW_MAX_EVENTS);
  std::partial_sort(items.begin(), items.begin() + keep, items.end(), [](const Item& a, const Item& b) {
    return a.step != b.step ? a.step < b.step : a.r < b.r;
  });
  for (size_t i = 0; i < keep; ++i) {
    out->events[i].deviation = items[i].dev;
    out->events[i].realization = r0 + items[i].r;
    out->events[i].step = items[i].step;
    out->events[i].corrected = items[i].corrected;
  }
  out->n_events = (int32_t)keep;
  out->event_count = (int64_t)items.size();
  return CTQW_OK;
}

int ctqw_observe_points(ctqw_handle_t h, const int64_t* acc_dev, int64_t npoints, double total_count,
                        double* out_dev, double* diag_dev, void* stream) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  if (npoints < 0 || npoints > 65535) return fail_with(h, CTQW_ERR_CONFIG, "npoints must be in [0, 65535]");
  if (npoints == 0) return CTQW_OK;
  if (!acc_dev || !out_dev) return fail_with(h, CTQW_ERR_CONFIG, "NULL buffer");
  DeviceGuard g(h->device);
  int rc = ensure(h, &h->points_scratch, &h->points_cap, npoints * 148 * 2 + (diag_dev ? 0 : npoints * h->dim),
                  "collection-point scratch");
  if (rc) return rc;
  double* diag = diag_dev ? diag_dev : h->points_scratch + npoints * 148 * 2;
  CUDA_TRY(h, launch_observe_points(h->m, h->n, h->dim, reinterpret_cast<const unsigned long long*>(acc_dev), npoints,
                                    total_count, diag, out_dev, h->points_scratch, (cudaStream_t)stream));
  h->launches += 4;
  return CTQW_OK;
}

int64_t ctqw_launch_count(ctqw_handle_t h) { return h ? (int64_t)h->launches.load() : 0; }

int ctqw_kernel_timing(ctqw_handle_t h, int32_t enable) {
  if (!h) return fail_with(nullptr, CTQW_ERR_CONFIG, "NULL handle");
  h->timing = enable != 0;
  h->ev_used = 0;
  h->timed_launches = 0;
  return CTQW_OK;
}

const char* ctqw_step_kernel(ctqw_handle_t h) { return h ? h->stream_kernel : ""; }
const char* ctqw_step_variant(ctqw_handle_t h) { return h ? h->variant : ""; }

int ctqw_kernel_time(ctqw_handle_t h, double* total_ms, int64_t* launches, void* stream) {
  if (!h || !total_ms || !launches) return fail_with(h, CTQW_ERR_CONFIG, "NULL argument");
  DeviceGuard g(h->device);
  CUDA_TRY(h, cudaStreamSynchronize((cudaStream_t)stream));
  double total = 0.0;
  for (size_t i = 0; i + 1 < h->ev_used; i += 2) {
    float ms = 0.f;
    CUDA_TRY(h, cudaEventElapsedTime(&ms, h->ev_pool[i], h->ev_pool[i + 1]));
    total += ms;
  }
  *total_ms = total;
  *launches = h->timed_launches;
  h->ev_used = 0;
  h->timed_launches = 0;
  return CTQW_OK;
}

}  // extern "C"
