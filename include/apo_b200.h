/*
 * apo_b200.h -- C ABI of libapo_b200.so, the B200 (sm_100a) APO hot path.
 *
 * The drop-in boundary is the reference's backend plug-in protocol
 * (/root/reference/pkg/src/protozoa/kernels/__init__.py:47-56): a backend
 * module exposes NAME, max_workers() and run_updates(...).  The reference's
 * only compiled code is the numba dispatcher that run_updates calls
 * (kernels/numba_backend.py:367-371, `_step_parallel(*args)` with the flat
 * argument tuple built at :358-366); apo_run_updates() below takes exactly
 * that tuple, as device pointers, plus sizes and a stream.  The Python
 * backend paper_2510_14982_b200/kernels/cuda_backend.py binds it with
 * ctypes (see INTEGRATION.md for the binding a reference maintainer adds).
 *
 * Conventions
 *  - every pointer argument is a DEVICE pointer unless the parameter name
 *    ends in _host;
 *  - `stream` is a cudaStream_t (NULL = legacy default stream);
 *  - every function returns 0 on success, or a nonzero status whose text is
 *    available from apo_last_error() (thread-local); invalid arguments are
 *    rejected with APO_EINVAL before any launch;
 *  - no function reads or writes its input population (numba_backend.py
 *    :334-337 "Inputs are read only"); callers own all outputs.
 */
#ifndef APO_B200_H
#define APO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define APO_OK 0
#define APO_EINVAL 1
#define APO_ECUDA 2
#define APO_ENOMEM 3

/* Random streams (the `rng` argument of the run entry points).
 * APO_RNG_KEYED: the reference's keyed fmix64 chain (rng.py:79-111) --
 *   oracle mode, bit-identical to the reference.
 * APO_RNG_PHILOX: production mode -- Philox4x32-10 keyed by the seed with
 *   counter (draw slot, protozoon, iteration); same algorithm and slot layout,
 *   statistically (not bitwise) equivalent. */
#define APO_RNG_KEYED 0
#define APO_RNG_PHILOX 1
/* APO_RNG_TABLE: scripted draws (the "identical pre-generated random tensor" oracle mode, replaying
 *   the reference's ScriptedStream, tests/test_acceptance.py:50-80): every draw (individual, counter)
 *   is read from an apo_draw_table; only the *_scripted entries below take it. */
#define APO_RNG_TABLE 2

/* A draw table in DEVICE memory (the struct itself and its arrays): n entries sorted by
 * (individual, counter), value = the uniform in [0, 1) that draw returns.  miss (device, 3 words,
 * zeroed by the caller) receives {1, individual, counter} of the first draw the table lacks; that
 * draw reads 0.0 and the caller must treat the call as failed (engine.step raises LookupError). */
typedef struct apo_draw_table {
    int64_t n;
    const uint64_t *individual;
    const uint64_t *counter;
    const double *value;
    uint64_t *miss;
} apo_draw_table;

/* Objective codes (objectives.py:34-42), plus codes the reference lacks. */
#define APO_OBJ_SPHERE 0
#define APO_OBJ_BENT_CIGAR 1
#define APO_OBJ_ELLIPTIC 2 /* table = elliptic weights (objectives.py:88-102) */
#define APO_OBJ_HGBAT 3
#define APO_OBJ_ROSENBROCK 4
#define APO_OBJ_GRIEWANK 5
#define APO_OBJ_TABLE 6 /* table[round_half_up(x0)] (objectives.py:183-192, 213-219) */
/* Multilevel thresholds (no reference counterpart): dim = k <= 32
 * thresholds in [0, 255]; table = the 515-entry prefix table written by
 * apo_threshold_tables (classes [0,t_0], [t_0+1,t_1], ..., [t_{k-1}+1, 255],
 * the k = 1 case being the reference's class convention, imaging.py:203-223). */
#define APO_OBJ_OTSU_ML 7  /* -(between-class variance) */
#define APO_OBJ_KAPUR_ML 8 /* -(sum of class entropies) */
#define APO_THRESHOLD_TABLE_LEN 515
/* CEC2022 F1..F12: code = APO_OBJ_CEC2022_BASE + F (no reference counterpart,
 * SPEC.md:146; definitions in csrc/apo_cec.cuh, data from cec2022.py). */
#define APO_OBJ_CEC2022_BASE 100

/* An objective as the kernels see it (device pointers). */
typedef struct apo_objective {
    int32_t code;
    int32_t table_len;
    const double *table;    /* elliptic weights / threshold table */
    const double *shift;    /* CEC2022: [ncomp][dim] optima */
    const double *rot_t;    /* CEC2022: [ncomp][dim][dim], rot_t[k][i][j] = M_k[j][i] */
    const int32_t *shuffle; /* CEC2022 hybrids: [dim], 1-based */
    /* CEC2022, optional: rot_t zero-padded to [ncomp][round_up(dim,4)][8*nt]
     * with nt = dim<=16 ? 2 : dim<=32 ? 4 : dim<=56 ? 7 : 13 (dim <= 104).
     * When present, large populations evaluate in the DMMA kernel
     * k_cec_eval; table may then hold the ELLIPS weights 10^(6i/(dim-1)).
     * For the hybrids (F6-F8) its output columns are permuted by the
     * shuffle: rot_pad[0][i][j] = rot_t[0][i][shuffle[j]-1]. */
    const double *rot_pad;
    /* CEC2022 F1-F8 and F10 at dim > 104, optional: the rotated component's
     * rot_t zero-padded to [round_up(dim,16)][round_up(dim,64)] (hybrids: columns
     * permuted like rot_pad).  When present, the device loop rotates all
     * candidates of an iteration as one DMMA GEMM (apo_cec_gemm.cu). */
    const double *rot_gemm;
    /* APO_OBJ_FMA_SMALL_D: with rot_pad present, the device loop may still rotate with lane-per-output
     * FMAs (the one-kernel fused update) at dim <= 32, where that is faster; batches keep the DMMA
     * evaluator at every dim (measured: profiles/r02_c5_rotation_crossover.txt). */
    int32_t flags;
} apo_objective;
#define APO_OBJ_FMA_SMALL_D 1

int apo_abi_version(void);
/* Largest `dim` the update / initialise / evaluate / run entries accept on this device (one warp's
 * shared-memory scratch must fit a CTA: 6403 on a B200).  Needs a device. */
int64_t apo_max_dim(void);
const char *apo_last_error(void);
/* Number of visible CUDA devices (cuda backend max_workers()). */
int apo_device_count(void);

/*
 * One iteration's per-individual phase over a rank-sorted snapshot.
 * Replaces numba_backend.run_updates (kernels/numba_backend.py:323-372):
 * same inputs (positions [ps, dim] row-major, rank r+1 in row r; fitness
 * [ps]; in_dr [ps] bool by rank), same flat scalars (:358-366), same
 * outputs (new positions/fitness in rank order, accepted, warned).
 * p_dr [ps] holds 0.5*(1-cos((1-i/ps)*pi)) per rank (numba_backend.py:
 * 173-175), computed by the host with libm so the decision threshold is
 * bit-identical; warn_count (nullable) receives the number of warned rows.
 */
int apo_run_updates(const double *positions, const double *fitness, const uint8_t *in_dr, double *out_pos,
                    double *out_fit, uint8_t *out_acc, uint8_t *out_warn, int64_t ps, int64_t dim, uint64_t seed,
                    uint64_t key_iteration, int64_t npairs, double lower, double upper, double span, double eps,
                    double p_ah, double f_mult, double decay, int64_t code, const double *table, int64_t table_len,
                    const double *p_dr, unsigned long long *warn_count, void *stream);

/* Same, for any objective descriptor (codes the reference does not have). */
int apo_run_updates_obj(const double *positions, const double *fitness, const uint8_t *in_dr, double *out_pos,
                        double *out_fit, uint8_t *out_acc, uint8_t *out_warn, int64_t ps, int64_t dim, uint64_t seed,
                        uint64_t key_iteration, int64_t npairs, double lower, double upper, double eps, double p_ah,
                        double f_mult, double decay, const apo_objective *objective_host, const double *p_dr,
                        unsigned long long *warn_count, void *stream);
/* apo_run_updates_obj restricted to ranks [rank_lo, rank_hi) (rows of out_pos/out_fit/out_acc outside
 * are not written; every row of positions may still be read as a partner).  warn_count is added to,
 * not reset, so a caller can split one update into chunks -- e.g. to copy finished ranks to the host
 * while the next chunk computes. */
int apo_run_updates_range(const double *positions, const double *fitness, const uint8_t *in_dr, double *out_pos,
                          double *out_fit, uint8_t *out_acc, uint8_t *out_warn, int64_t ps, int64_t dim,
                          uint64_t seed, uint64_t key_iteration, int64_t npairs, double lower, double upper,
                          double eps, double p_ah, double f_mult, double decay, const apo_objective *objective_host,
                          const double *p_dr, unsigned long long *warn_count, int64_t rank_lo, int64_t rank_hi,
                          void *stream);
/* apo_run_updates_range without the snapshot gather (core.py:504-513's row copy): positions/fitness
 * stay in the caller's row order and order[r] (int32, the stable sort's rank -> row map, apo_sort_order)
 * names the row holding rank r; outputs are by rank, as apo_run_updates writes them.  dim <= 256. */
int apo_run_updates_ordered(const double *positions, const double *fitness, const int32_t *order,
                            const uint8_t *in_dr, double *out_pos, double *out_fit, uint8_t *out_acc,
                            uint8_t *out_warn, int64_t ps, int64_t dim, uint64_t seed, uint64_t key_iteration,
                            int64_t npairs, double lower, double upper, double eps, double p_ah, double f_mult,
                            double decay, const apo_objective *objective_host, const double *p_dr,
                            unsigned long long *warn_count, int64_t rank_lo, int64_t rank_hi, void *stream);

/* Batch fitness: out[r] = f(x[r*ld .. r*ld+dim)) (objectives.evaluate_unchecked,
 * objectives.py:222-228). */
int apo_evaluate(const double *x, int64_t n, int64_t dim, int64_t ld, const apo_objective *objective_host, double *out,
                 void *stream);

/* Iteration-0 population (engine.initialize, engine.py:116-139): row s =
 * lower + u(seed, 0, s+1, d) * span, then its fitness. */
int apo_initialize(uint64_t seed, int64_t ps, int64_t dim, int64_t ld, double lower, double span,
                   const apo_objective *objective_host, double *positions, double *fitness, void *stream);

/* Stable ascending argsort of fitness (core.sort_by_fitness, core.py:
 * 504-513): order[r] = row holding rank r+1; ties keep row order,
 * -0.0 == +0.0, NaN last. */
int apo_sort_order(const double *fitness, int64_t n, int32_t *order, void *stream);

/* Coordinator draws (core.py:263-278, engine.py:157-162): in_dr[r] = 1 iff
 * rank r+1 is in this iteration's dormancy/reproduction set.  Returns the
 * set size through count_host (nullable). */
int apo_select_dr(uint64_t seed, uint64_t key_iteration, int64_t ps, double pf_max, uint8_t *in_dr,
                  int64_t *count_host, void *stream);

/* Scripted-draw variants of apo_run_updates_obj and apo_select_dr (APO_RNG_TABLE): `table` is the
 * device address of an apo_draw_table; the coordinator's set size `count` = ceil(ps * pf) is computed by
 * the caller from its scripted pf draw (core.py:263-278).  Same kernels as the keyed entries. */
int apo_run_updates_scripted(const double *positions, const double *fitness, const uint8_t *in_dr, double *out_pos,
                             double *out_fit, uint8_t *out_acc, uint8_t *out_warn, int64_t ps, int64_t dim,
                             const apo_draw_table *table, int64_t npairs, double lower, double upper, double eps,
                             double p_ah, double f_mult, double decay, const apo_objective *objective_host,
                             const double *p_dr, unsigned long long *warn_count, void *stream);
int apo_select_dr_scripted(const apo_draw_table *table, int64_t ps, int64_t count, uint8_t *in_dr, void *stream);

/* Prefix tables of a 256-bin histogram for APO_OBJ_OTSU_ML (method 0) or
 * APO_OBJ_KAPUR_ML (method 1): table[0] = N, table[1+i] = sum_{v<i} count_v,
 * table[258+i] = sum_{v<i} v count_v (Otsu) / sum_{v<i} p_v ln p_v (Kapur),
 * i = 0..256 (generalises imaging.variance_table, imaging.py:226-228). */
int apo_threshold_tables(const int64_t *counts, int method, double *table, void *stream);

/* 256-bin histogram of an 8-bit image (imaging.histogram, imaging.py:197-200). */
int apo_histogram_u8(const uint8_t *pixels, int64_t n, int64_t *counts, void *stream);

/*
 * Device-resident run (engine.run, engine.py:175-212).  The population
 * stays in HBM in slot order; each iteration is a stable key sort (rank ->
 * slot order, no row gather), the coordinator draws and one fused update
 * launch.  sched_host: [max_iterations][3] = (p_ah, f_mult, decay) per
 * iteration; p_dr_host: [ps].  Both are computed by the host with libm
 * exactly as numba_backend.py:357-366 and :173-175 do.
 */
typedef struct apo_run apo_run;
int apo_run_create(apo_run **out, int64_t ps, int64_t dim, int64_t max_iterations, uint64_t seed, int64_t npairs,
                   double pf_max, double lower, double upper, double eps, const apo_objective *objective_host,
                   const double *sched_host, const double *p_dr_host, int rng, void *stream);
int apo_run_initialize(apo_run *run);
/* Checkpoint/resume: load a population (reference row order, [ps][dim]) that
 * has completed `iteration` iterations; the next apo_run_iterate continues the
 * run exactly (every draw is keyed by (seed, iteration, rank, slot)).  Trace
 * entries before `iteration` are not kept. */
int apo_run_load(apo_run *run, const double *positions, const double *fitness, int is_host, int64_t iteration,
                 int64_t warnings);
/* Runs iterations [t, t+n) where t is the number already run. */
int apo_run_iterate(apo_run *run, int64_t n);
/* Trace entries 0..iterations_run as doubles (host buffer of >= n+1). */
int apo_run_trace(apo_run *run, double *trace_host, int64_t n);
/* Current population in reference row order (row r = rank r+1 of the last
 * snapshot, i.e. what engine.step returns), device or host buffers. */
int apo_run_population(apo_run *run, double *positions, double *fitness, int is_host);
/* Best individual (Population.best, core.py:195-196: first argmin in
 * reference row order). */
int apo_run_best(apo_run *run, double *best_fitness_host, double *best_position_host, int64_t *best_row_host);
int apo_run_counters(apo_run *run, int64_t *iterations_run, int64_t *fe_count, int64_t *warnings);
int apo_run_destroy(apo_run *run);
/* Timing hook: when enabled, CUDA events on the run's stream bracket every
 * fused update launch; _read returns their summed duration (ms) and count
 * since the last apo_run_profile call. */
int apo_run_profile(apo_run *run, int enable);
int apo_run_profile_read(apo_run *run, double *update_ms_host, int64_t *launches_host);
/* Same, split at the boundary between the candidate kernel and the CEC2022
 * evaluation kernel (k_cec_eval; evaluate_ms is 0 for fused objectives). */
int apo_run_profile_split(apo_run *run, double *candidates_ms_host, double *evaluate_ms_host, int64_t *launches_host);
/* Which kernels one iteration's update runs: 0 one fused kernel (basic objectives), 1 CEC2022 split
 * (candidates, then the DMMA evaluation kernel), 2 CEC2022 fused (one kernel: candidates + DMMA
 * evaluation + select; opt-in APO_CEC_FUSED=1), 3 CEC2022 at D > 104 (candidates, DMMA GEMM, finish),
 * 4 the reference's six objectives at 33 <= D <= 256 (candidates, then a lane-per-protozoon sequential
 * evaluation + select). */
int apo_run_update_path(apo_run *run, int *path_host);

/*
 * One population sharded by rank across processes (engine.run with the
 * population split over N GPUs, BASELINE config 4).  Each process keeps the
 * whole population in rank order of the previous iteration in caller-owned
 * buffers pos0/pos1 [ps_pad][ld] and fit0/fit1 [ps_pad]; per iteration:
 *   apo_shard_begin          stable sort + coordinator draws (replicated)
 *   apo_shard_update_range   update ranks [lo, hi) into the next buffers
 *   (caller)                 all-gather rows [lo, hi) of the next buffers
 *   apo_shard_end            the next buffers become current
 * Results are identical for every partition (tests/test_shard.py).
 * trace keys / warnings count this process's ranks only: reduce them
 * (MIN / SUM) across processes.  dim <= 256.
 */
typedef struct apo_shard apo_shard;
int apo_shard_create(apo_shard **out, int64_t ps, int64_t dim, int64_t ld, int64_t max_iterations, uint64_t seed,
                     int64_t npairs, double pf_max, double lower, double upper, double eps,
                     const apo_objective *objective_host, const double *sched_host, const double *p_dr_host, int rng,
                     double *pos0, double *pos1, double *fit0, double *fit1, void *stream);
int apo_shard_initialize(apo_shard *shard);
int apo_shard_begin(apo_shard *shard);
int apo_shard_update_range(apo_shard *shard, int64_t lo, int64_t hi);
int apo_shard_end(apo_shard *shard);
/* Device pointers of the current buffers and the iterations run. */
int apo_shard_state(apo_shard *shard, double **pos_dev, double **fit_dev, int64_t *iterations_host);
/* Order-preserving trace keys (entries 0..n; decode like apo_run_trace) and warnings of this process. */
int apo_shard_counters(apo_shard *shard, unsigned long long *trace_keys_host, int64_t n, int64_t *warnings_host);
int apo_shard_destroy(apo_shard *shard);

/*
 * Many independent small runs, one CTA per run, the whole run resident in
 * shared memory for all iterations (BASELINE configs 1-3 and 5: seeds x
 * objectives).  objectives_host: nruns descriptors; seeds: device [nruns].
 * Outputs (device, nullable except best_fit): best_fit [nruns], best_pos
 * [nruns, dim], trace [nruns, n_iters+1], final_pos [nruns, ps, dim] and
 * final_fit [nruns, ps] in reference row order, warnings [nruns].
 * n_iters <= max_iterations is the number of iterations actually run
 * (max_fes budget, engine.py:192-193).
 */
int apo_run_batch(int64_t nruns, const uint64_t *seeds, const apo_objective *objectives_host, int64_t ps,
                  int64_t dim, int64_t max_iterations, int64_t n_iters, int64_t npairs, double pf_max, double lower,
                  double upper, double eps, const double *sched, const double *p_dr, double *best_fit,
                  double *best_pos, double *trace, double *final_pos, double *final_fit, int64_t *warnings,
                  int rng, void *stream);
/* apo_run_batch with an explicit CTA size: threads_per_run = 0 picks the shape (more runs than SMs:
 * one persistent 640-thread CTA per SM claiming runs costliest first; else one 512-thread CTA per
 * run); a multiple of 32 in [32, 640] forces one CTA of that many threads per run -- e.g. 256 when several batches run
 * concurrently on different streams and must share the SMs. */
int apo_run_batch_shaped(int64_t nruns, const uint64_t *seeds, const apo_objective *objectives_host, int64_t ps,
                         int64_t dim, int64_t max_iterations, int64_t n_iters, int64_t npairs, double pf_max,
                         double lower, double upper, double eps, const double *sched, const double *p_dr,
                         double *best_fit, double *best_pos, double *trace, double *final_pos, double *final_fit,
                         int64_t *warnings, int rng, int threads_per_run, void *stream);
/* Device scratch and run buffers freed by the library stay in the current device's stream-ordered
 * pool for reuse (no cudaMalloc/cudaFree per run or step); this returns them to the driver. */
int apo_release_cached_memory(void);
/* Largest ps*dim the batch kernel can hold in shared memory (basic objectives). */
int64_t apo_run_batch_max_elems(int64_t ps, int64_t dim);
/* 1 if a batch of these objectives at (ps, dim) fits the shared-memory batch kernel. */
int apo_run_batch_fits(int64_t ps, int64_t dim, const apo_objective *objectives_host, int64_t nobj);

/* Host-side RNG entry points (no device needed; the kernels use the same
 * code): one Philox4x32-10 block, and the draw u(seed, iteration, individual,
 * counter) of either stream (rng.py:100-111 for APO_RNG_KEYED). */
void apo_philox4x32_10(const uint32_t *ctr4, const uint32_t *key2, uint32_t *out4);
double apo_rng_uniform(int rng, uint64_t seed, uint64_t iteration, uint64_t individual, uint64_t counter);

/* Debug/verification entry: out[k] = device exp_glibc(x[k]). */
int apo_debug_exp(const double *x, double *out, int64_t n, void *stream);
/* Debug/verification entry: out[k] = device cos_glibc(x[k]) (glibc 2.39's cos, griewank). */
int apo_debug_cos(const double *x, double *out, int64_t n, void *stream);

/* Debug/verification entry: out[r] = CEC2022 basic function `basic` (ids of csrc/apo_cec.cuh /
 * oracle/cec_oracle.c; ELLIPS weights from ew, nullable) of row r of z [rows][n], evaluated by the
 * headline kernels' quad evaluator (variant 0) or the warp evaluator (variant 1).  The five basic
 * functions the reference also has replace objectives.py:112-142 / numba_backend.py:93-131. */
int apo_debug_cec_basic(int basic, const double *z, int64_t rows, int64_t n, const double *ew, double *out,
                        int variant, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* APO_B200_H */
