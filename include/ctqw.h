/*
 * ctqw.h -- C ABI of libctqw.so, the B200 (sm_100a) hot path of the noisy
 * many-particle continuous-time-quantum-walk ensemble simulator.
 *
 * Plain C: pointers, sizes, POD structs.  No torch or C++ types cross the
 * boundary, no exceptions, no allocations handed to the caller.  Device
 * pointers (suffix _dev) are caller-owned CUDA allocations on the handle's
 * device (torch tensors in the Python host layer); the library keeps only
 * its own scratch and statistics buffers.  Streams are passed as void*
 * (a cudaStream_t); NULL means the legacy default stream.
 *
 * Every entry point returns a status equal to the reference's
 * CtqwError.exit_code (pkg/src/ctqw/errors.py:8-75):
 *   0 ok, 2 configuration, 3 numeric (norm failure), 4 capacity, 1 other
 *   (CUDA failure).  ctqw_last_error() gives the message.
 *
 * The reference (pkg/src/ctqw, pure Python/NumPy) has no FFI of its own;
 * each entry point below names the Python function whose contract it takes
 * over.  States are complex128 stored as interleaved (re, im) doubles,
 * realization-major, each realization a row-major N^m joint vector with
 * particle 0 the most significant digit (hilbert.py:141-159).
 */
#ifndef CTQW_H
#define CTQW_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CTQW_ABI_VERSION 1

#define CTQW_OK 0
#define CTQW_ERR_OTHER 1
#define CTQW_ERR_CONFIG 2
#define CTQW_ERR_NUMERIC 3
#define CTQW_ERR_CAPACITY 4

#define CTQW_BACKEND_TAYLOR 0
#define CTQW_BACKEND_RK4 1

#define CTQW_MAX_EVENTS 100 /* ensemble.py:119 MAX_EVENTS_PER_SEGMENT */

typedef struct ctqw_ctx *ctqw_handle_t;

/* Geometry + deterministic couplings.  Replaces JointSpace/LatticeTopology
 * (hilbert.py:45-138) and CouplingModel (hamiltonian.py:30-72), 1 <= m <= 3.
 * The ring (k_half = 1, periodic = 1, n_sites >= 3) is complete as created
 * and runs the fused kernels.  Any other lattice (q >= 1 directions, K =
 * sum(k_half) slots per site, periodic or open) passes its move tables with
 * ctqw_set_lattice and runs the generic kernels. */
typedef struct {
  int32_t m;            /* particles */
  int32_t n_sites;      /* lattice sites N = prod(dims) */
  int32_t k_half;       /* K: positive move slots per site (1 for the ring) */
  int32_t periodic;     /* 1 periodic, 0 open */
  double onsite_energy; /* eps0 */
  double tunneling;     /* t */
  double interaction;   /* U, per coinciding pair */
  double hbar;
} ctqw_model_t;

/* Integrator + norm policy.  Mirrors StepperConfig (propagators.py:61-86). */
typedef struct {
  int32_t backend;     /* CTQW_BACKEND_TAYLOR / CTQW_BACKEND_RK4 */
  int32_t order;       /* Taylor order, 1..64 (ignored for RK4) */
  double dt;
  double tol_norm;
  double tol_fail;
  int32_t renormalize;
  int32_t exact;       /* 1: reference operation order, no FMA contraction
                          (bit-identical to the reference between rescales);
                          0: FMA-contracted stencil, Horner-form Taylor
                          (<= 1e-12 from it) */
} ctqw_stepper_t;

/* NormEvent (propagators.py:89-96). */
typedef struct {
  double deviation;
  int64_t realization;
  int64_t step;
  int32_t corrected;
  int32_t reserved;
} ctqw_norm_event_t;

/* _SegmentStats (ensemble.py:414-423) plus the NormFailureError payload
 * (errors.py:26-49, re-tagged as in ensemble.py:509-516). */
typedef struct {
  int64_t event_count;
  int64_t corrections;
  double max_deviation;
  int32_t failed;
  int32_t n_events;
  int64_t fail_realization;
  int64_t fail_step;
  double fail_deviation;
  ctqw_norm_event_t events[CTQW_MAX_EVENTS];
} ctqw_segment_stats_t;

int ctqw_abi_version(void);
const char *ctqw_last_error(ctqw_handle_t h); /* h may be NULL */

/* Bind a model to a device.  Validation follows hilbert.py:58-82,
 * hamiltonian.py:44-63 (exit 2) and the joint-index capacity (exit 4). */
int ctqw_create(const ctqw_model_t *model, int32_t device, ctqw_handle_t *out);
int ctqw_destroy(ctqw_handle_t h);

/* Static noise draw on the device, bit-identical to
 * init_process(spec, lattice, seed=(master_seed, r)).values for
 * r = r0 .. r0+count-1 (noise.py:128-159, ensemble.py:680-682):
 * SeedSequence -> PCG64 -> Generator.choice(levels, total).
 * noise_dev is [count][total] doubles, levels_host has n_levels entries. */
int ctqw_draw_noise(ctqw_handle_t h, uint64_t master_seed, int64_t r0, int64_t count,
                    const double *levels_host, int32_t n_levels, int64_t total,
                    double *noise_dev, void *stream);

/* Stencil coefficients from noise rows [links(n_links) | sites(n_sites)]:
 * hop = t + xi_link (hamiltonian.py:137-141), site = xi_site
 * (hamiltonian.py:134-135).  n_links is 0 or N, n_sites is 0 or N.
 * hop_dev is [count][N]; site_dev is [count][N] and is written only when
 * n_sites == N. */
/* Dynamic (random-telegraph) noise, rate > 0: the reference's NoiseProcess
 * (noise.py:71-206).  ctqw_telegraph_init draws, per realization
 * r0 .. r0+count-1, values = choice(levels, total) and next_switch =
 * exponential(1/rate, total) from default_rng((master_seed, r)) -- bit-exact
 * to NumPy -- into library-owned buffers ([count][n_links + n_sites], links
 * first); ctqw_telegraph_values returns them (device pointer) for
 * ctqw_build_coefficients.  Once enabled, ctqw_evolve advances the process
 * by dt after every step's norm check and rewrites the bound hop/site rows of
 * switched elements (ensemble.py:536-544, hamiltonian.py:164-192).
 * ctqw_telegraph_read copies values / switch times (device to device) and
 * per-realization time and switch counts (to the host); any pointer may be
 * NULL. */
int ctqw_telegraph_init(ctqw_handle_t h, uint64_t master_seed, int64_t r0, int64_t count,
                        const double *levels_host, int32_t n_levels, int64_t n_links, int64_t n_sites,
                        double rate, void *stream);
const double *ctqw_telegraph_values(ctqw_handle_t h);
/* advance(process, dt) for realizations 0 .. count-1 without a step
 * (noise.py:175-206); rewrites bound coefficients of switched elements. */
int ctqw_telegraph_advance(ctqw_handle_t h, int64_t count, double dt, void *stream);
int ctqw_telegraph_enable(ctqw_handle_t h, int32_t enable);
int ctqw_telegraph_read(ctqw_handle_t h, double *values_dev, double *next_switch_dev, double *times_host,
                        int64_t *switches_host, void *stream);

/* Move tables of a general lattice in the reference's slot order
 * (_site_move_tables, hilbert.py:189-224): pos/neg[x*K + s] = target site of
 * the +/- move of slot s from site x, -1 off an open lattice; t_slot[s] =
 * tunnelling of slot s's direction (slot_couplings, hamiltonian.py:92-97).
 * Links are x*K + s (hilbert.py:311), so hop rows hold N*K couplings. */
int ctqw_set_lattice(ctqw_handle_t h, int32_t n_slots, const int32_t *pos_host, const int32_t *neg_host,
                     const double *t_slot_host);

int ctqw_build_coefficients(ctqw_handle_t h, const double *noise_dev, int64_t count,
                            int64_t n_links, int64_t n_sites, double *hop_dev,
                            double *site_dev, void *stream);

/* Bind coefficient rows used by every compute call below: realization i of
 * a call reads hop_dev + i*stride (stride 0 broadcasts one Hamiltonian,
 * like an unbatched `values` table).  site_dev NULL = no on-site noise. */
int ctqw_bind_coefficients(ctqw_handle_t h, int64_t count, const double *hop_dev,
                           const double *site_dev, int64_t stride);

/* psi_dev[r] = psi0_dev for r < count (np.tile, ensemble.py:678). */
int ctqw_fill_states(ctqw_handle_t h, double *psi_dev, int64_t count, const double *psi0_dev,
                     void *stream);

/* Lazy form of ctqw_fill_states (ensemble.py:678, np.tile(psi0)): the next
 * ctqw_evolve / ctqw_evolve_observe on this handle starts every realization
 * from psi0_dev (one state, D complex128, kept alive by the caller until
 * then) without writing the R x D stack first -- the band4 and resident64
 * kernels read it directly in the first step; other paths fill the stack
 * themselves.  Until that call the contents of psi are undefined (call
 * ctqw_fill_states to materialise them); ctqw_fill_states cancels it. */
int ctqw_set_initial(ctqw_handle_t h, const double *psi0_dev);

/* out = H psi for a batch (apply_values, hamiltonian.py:195-223). */
int ctqw_apply(ctqw_handle_t h, const double *psi_dev, double *out_dev, int64_t count,
               int32_t exact, void *stream);

/* One propagation step with no norm policy: step_taylor_values /
 * step_rk4_values (propagators.py:167-241).  out may not alias psi. */
int ctqw_step(ctqw_handle_t h, const double *psi_dev, double *out_dev, int64_t count,
              const ctqw_stepper_t *stepper, void *stream);

/* check_norm_stack (propagators.py:309-328): deviations_dev[count] and
 * corrected_dev[count] are written; the stack is rescaled in place.  On a
 * failure returns 3 with *fail_row (argmax) and *fail_deviation set and
 * leaves the stack untouched.  Synchronises the stream. */
int ctqw_check_norm(ctqw_handle_t h, double *psi_dev, int64_t count,
                    const ctqw_stepper_t *stepper, double *deviations_dev,
                    int32_t *corrected_dev, int64_t *fail_row, double *fail_deviation,
                    void *stream);

/* The segment inner loop (_evolve_segment, ensemble.py:445-558) for static
 * noise: n_steps steps of `count` realizations starting after step
 * first_step, each followed by the norm policy.  work_dev is a caller-owned
 * buffer shaped like psi_dev.  Asynchronous: the advanced stack is in
 * psi_dev, or in work_dev when *result_in_work is set on return.  Statistics
 * of the call are read with ctqw_segment_stats. */
int ctqw_evolve(ctqw_handle_t h, double *psi_dev, double *work_dev, int64_t count,
                int64_t first_step, int64_t n_steps, const ctqw_stepper_t *stepper,
                int32_t *result_in_work, void *stream);

/* Synchronise and reduce the statistics of the last ctqw_evolve call.
 * Realization indices are offset by r0.  Returns 3 when a realization
 * failed (the stats carry the culprit, as NormFailureError does). */
int ctqw_segment_stats(ctqw_handle_t h, int64_t r0, ctqw_segment_stats_t *out, void *stream);

/* diag_sum_dev[alpha] (+)= sum_r |psi_r(alpha)|^2 (the diagonal of
 * accumulate_density's Gram, density.py:91-92, before the division by R).
 * The sum is exact up to one final rounding and independent of the order of
 * the realizations (see ctqw_observe_diag_fixed).  accumulate = 0 overwrites. */
int ctqw_observe_diag(ctqw_handle_t h, const double *psi_dev, int64_t count,
                      double *diag_sum_dev, int32_t accumulate, void *stream);

/* The same sum as exact fixed-point limbs acc_dev[3][N^m] (int64): each
 * term is split deterministically onto the grids 2^-30, 2^-70, 2^-110 and
 * added as integers, so the limbs are bitwise independent of realization
 * order, batching and GPU count; an int64 SUM all-reduce of the limbs across
 * ranks keeps that (observables identical across 1/2/4/8 GPUs, as the
 * reference's are across worker counts, pkg/README.md:174-180).  Holds up to
 * 2^23 realizations.  accumulate = 0 zeroes the limbs first. */
int ctqw_observe_diag_fixed(ctqw_handle_t h, const double *psi_dev, int64_t count, int64_t *acc_dev,
                            int32_t accumulate, void *stream);
/* diag_dev[alpha] = the value of the limbs (carries normalised, then one
 * rounding per limb pair). */
int ctqw_fixed_to_double(ctqw_handle_t h, const int64_t *acc_dev, double *diag_dev, void *stream);

/* From the (all-reduced) diagonal sum and the total realization count:
 * populations_dev[N] (observables.py:40-56) and scalars_dev[3] =
 * {sum_alpha p, sum_alpha p^2, participation ratio} (observables.py:94-101)
 * with p = diag_sum / total_count.  joint_dev (optional, [N^m]) receives p. */
int ctqw_observe_reduce(ctqw_handle_t h, const double *diag_sum_dev, double total_count,
                        double *populations_dev, double *scalars_dev, double *joint_dev,
                        void *stream);

/* sumsq_dev[0] = sum_{i,j} |<a_i|b_j>|^2 over two state stacks: the
 * off-diagonal information purity needs (observables.py:86-91) without the
 * dense rho.  b_dev == a_dev uses the Hermitian symmetry. */
int ctqw_overlap_sumsq(ctqw_handle_t h, const double *a_dev, int64_t count_a,
                       const double *b_dev, int64_t count_b, double *sumsq_dev, void *stream);

/* Purity sums of npoints collection points in one launch set: sumsq_dev[p] =
 * sum_{i,j} |<a_i|a_j>|^2 over the stack stacks_dev + p * point_stride
 * (complex elements, >= count * dim when npoints > 1), count states each
 * (observables.py:86-91 at every point of a schedule group; the snapshots
 * ctqw_evolve_observe writes).  Same result as npoints ctqw_overlap_sumsq
 * calls with b == a. */
int ctqw_overlap_sumsq_points(ctqw_handle_t h, const double *stacks_dev, int64_t count,
                              int64_t npoints, int64_t point_stride, double *sumsq_dev,
                              void *stream);

/* Packed ensemble density matrix (replaces the Gram product of
 * ctqw/density.py:91-95, accumulate_density): packed_dev[i(i+1)/2 + j] =
 * scale * sum_r psi_r[i] conj(psi_r[j]) for j <= i, psi_dev an (R, dim)
 * complex128 stack (interleaved doubles), packed_dev dim(dim+1)/2 complex128.
 * The reference divides by R (scale = 1/R); scale = 1 gives the raw sums
 * (multi-GPU: all-reduce, then scale).  Realizations are summed in stack
 * order.  Needs no model handle; errors go to ctqw_last_error(NULL). */
int ctqw_packed_gram(const double *psi_dev, int64_t count, int64_t dim, double scale, double *packed_dev,
                     int32_t device, void *stream);

/* ctqw_evolve plus the collection points of the schedule, in one call
 * (replaces the _evolve_segment + accumulate_density-diagonal pairs of
 * ensemble.py:722-769 for a run of segments).  Every step g =
 * first_step + k * post_rate (k >= 1) up to first_step + n_steps, and the
 * last one, is a collection point; point idx = ceil((g - first_step) /
 * post_rate) - 1 (ceil(n_steps / post_rate) points) receives the exact int64
 * limbs of sum_r |psi_r(g)|^2 in acc_dev[idx][3][dim] (zeroed by the call; same limbs
 * as ctqw_observe_diag_fixed).  On the resident N = 64 path the sum is
 * fused into the step kernel; elsewhere each segment is followed by the
 * limb pass.  Statistics accumulate over the whole call (ctqw_segment_stats,
 * ctqw_segment_events), and over earlier calls too when keep_stats != 0.
 * snap_dev (optional, [points][count][dim] complex128) receives the states
 * themselves at every point (purity needs them: observables.py:86-91).
 * n_steps >= 1, post_rate >= 1. */
int ctqw_evolve_observe(ctqw_handle_t h, double *psi_dev, double *work_dev, int64_t count, int64_t first_step,
                        int64_t n_steps, int64_t post_rate, int64_t *acc_dev, double *snap_dev,
                        const ctqw_stepper_t *stepper, int32_t keep_stats, int32_t *result_in_work, void *stream);

/* The events of the last evolve / evolve_observe call with step in
 * (step_lo, step_hi], first CTQW_MAX_EVENTS in (step, realization) order
 * (one segment's list, as _evolve_segment reports it); event_count = events
 * in that range still held in the per-realization logs (CTQW_MAX_EVENTS
 * each).  Synchronises the stream. */
int ctqw_segment_events(ctqw_handle_t h, int64_t r0, int64_t step_lo, int64_t step_hi, ctqw_segment_stats_t *out,
                        void *stream);

/* Post-processing of npoints collection points at once from their limbs
 * acc_dev[npoints][3][dim] (all-reduced over ranks beforehand if sharded):
 * out_dev[npoints][N + 3] = populations (N) + {sum p, sum p^2, participation
 * ratio}, p = diag / total_count (observables.py:34-101); diag_dev
 * (optional, [npoints][dim]) receives the diagonal sums.  Four launches for
 * any number of points; the same bits as ctqw_fixed_to_double +
 * ctqw_observe_reduce per point. */
int ctqw_observe_points(ctqw_handle_t h, const int64_t *acc_dev, int64_t npoints, double total_count,
                        double *out_dev, double *diag_dev, void *stream);

/* Kernel launches issued by this handle since creation (for bench.py). */
int64_t ctqw_launch_count(ctqw_handle_t h);

/* Timing mode (bench.py): when enabled, ctqw_evolve brackets each launch of
 * its dominant step kernel with CUDA events on the launch stream;
 * ctqw_kernel_time synchronises, returns the summed elapsed milliseconds and
 * the number of bracketed launches, and clears the record. */
int ctqw_kernel_timing(ctqw_handle_t h, int32_t enable);
int ctqw_kernel_time(ctqw_handle_t h, double *total_ms, int64_t *launches, void *stream);

/* Name of the dominant kernel the last ctqw_evolve on this handle ran
 * ("band4_kernel", "resident_kernel", ...; "" for the generic path). */
const char *ctqw_step_kernel(ctqw_handle_t h);

/* Its compile-time specialization, e.g.
 * "band4_kernel<taylor,napp=4,site=1,exact=0,NN=1024>" (parity tests assert
 * that the variant a BASELINE configuration runs is the one they check). */
const char *ctqw_step_variant(ctqw_handle_t h);

#ifdef __cplusplus
}
#endif

#endif /* CTQW_H */
