/*
 * psso.h -- C ABI of the B200-native PSSO hot path (libpsso.so).
 *
 * The reference package (arXiv 2110.01470, `sso`) is pure Python and has no
 * FFI of its own; these entry points are what its Python host code binds
 * through ctypes.  Each one replaces one reference
 * interface, cited below as path:line under /root/reference/pkg/src/sso/.
 *
 * Conventions
 *  - Plain C types only.  Device buffers are borrowed raw pointers (the host
 *    owns them, e.g. as torch tensors); `stream` is a cudaStream_t passed as
 *    void* (NULL = legacy default stream).
 *  - Every function returns PSSO_OK (0) or an error code; the message of the
 *    last error is available from psso_last_error(ctx) (ctx may be NULL for
 *    context-free entry points; the message is then thread-local).
 *  - Fitness values (sol_f, p_f, g_f, trajectory) are always float64; the
 *    position matrices use the configured dtype.
 *  - Matrices are particle-major (row i = particle i, contiguous), the layout
 *    the paper calls "stored sequentially" (reference parallel.py:53-60).
 */
#ifndef PSSO_H
#define PSSO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSSO_ABI_VERSION 2  /* 2: 32-byte candidate header, gBest index, communicators, statistics */

/* status codes */
#define PSSO_OK 0
#define PSSO_E_INVALID 1     /* bad argument -> Python ValueError (core.py:69-81) */
#define PSSO_E_CUDA 2        /* CUDA runtime failure */
#define PSSO_E_NONFINITE 3   /* non-finite fitness -> NonFiniteFitnessError (core.py:43-53) */
#define PSSO_E_UNSUPPORTED 4 /* shape/dtype outside what the kernels handle */
#define PSSO_E_NCCL 5        /* NCCL failure (sharded iteration over a communicator) */

/* dtype of the position matrices */
#define PSSO_F64 0
#define PSSO_F32 1

/* random source */
#define PSSO_RNG_REFERENCE 0 /* the reference's keyed SplitMix64 (rng.py:27-92), bit-exact */
#define PSSO_RNG_PHILOX 1    /* Philox4x32-10 counter RNG (benchmark mode) */

/* config flags */
#define PSSO_FLAG_KEEP_SOL_F 1 /* fused steps also write sol_f for every row (phase-API
                                  state parity); default: sol_f is written only for
                                  non-finite rows, saving 8 bytes per row per iteration */

/* objective ids: 1..9 = f1..f9 (benchmarks.py:33); 0 = test probe: Sphere,
 * except +inf where x[0] > probe_level (fault injection for tests). */
#define PSSO_FN_PROBE 0

/* replaces: SsoParams (core.py:56-85) + make_function metadata
 * (benchmarks.py:169-270) + the seed argument of run_parallel (parallel.py:152) */
typedef struct psso_config {
    int32_t fn_id;      /* objective id, see above */
    int32_t dtype;      /* PSSO_F64 | PSSO_F32 */
    int32_t rng_mode;   /* PSSO_RNG_REFERENCE | PSSO_RNG_PHILOX */
    int32_t flags;      /* PSSO_FLAG_* bits */
    int64_t nsol;       /* global swarm size N */
    int64_t nvar;       /* problem dimension D */
    int64_t row_lo;     /* first global particle owned by this context */
    int64_t row_hi;     /* one past the last; [0, nsol) when unsharded */
    double cw, cp, cg;  /* cumulative branch thresholds, 0 <= cw <= cp <= cg <= 1 */
    double var_min, var_max;
    uint64_t seed;      /* masked to 64 bits like rng.py:68 */
    double probe_level; /* PSSO_FN_PROBE only */
} psso_config;

/* replaces: the Swarm dataclass (core.py:88-115).  Device pointers, borrowed. */
typedef struct psso_buffers {
    void* sol;      /* (row_hi-row_lo) x nvar, dtype          -> Swarm.sol    */
    void* pbests;   /* (row_hi-row_lo) x nvar, dtype          -> Swarm.pbests */
    double* sol_f;  /* (row_hi-row_lo) float64, may be NULL   -> Swarm.sol_f  */
    double* p_f;    /* (row_hi-row_lo) float64                -> Swarm.p_f    */
    void* gbest;    /* nvar, dtype                            -> Swarm.gbest  */
    double* g_f;    /* one float64                            -> Swarm.g_f    */
    double* traj;   /* trajectory indexed by absolute iteration t, may be NULL
                       -> RunRecord.trajectory (records.py:46)                  */
} psso_buffers;

typedef struct psso_ctx psso_ctx;

const char* psso_version(void);
const char* psso_last_error(const psso_ctx* ctx);

/* replaces: run_parallel set-up (parallel.py:164-173): validation, layout,
 * partition.  Allocates only small scratch (per-CTA candidate slots). */
int psso_create(const psso_config* cfg, psso_ctx** out);
void psso_destroy(psso_ctx* ctx);

/* Attach the swarm buffers and the stream every later call enqueues on. */
int psso_bind(psso_ctx* ctx, const psso_buffers* bufs, void* stream);

/* replaces: core.initialize (core.py:196-210): INIT draws -> positions ->
 * fitness -> argmin (lowest index) -> gbest/g_f.  Non-finite -> PSSO_E_NONFINITE
 * reported by psso_check with iteration -1. */
int psso_init(psso_ctx* ctx);

/* replaces: one iteration of the run_parallel loop (parallel.py:195-212):
 * fused search + evaluate + pBest kernel, then the gBest stage-2 kernel and
 * trajectory[t] = g_f.  Asynchronous. */
int psso_step(psso_ctx* ctx, int64_t t);

/* replaces: the whole loop `for t in range(t0, t0+niter)` (parallel.py:192-212).
 * Asynchronous.  Small swarms that fit one thread-block cluster (C1, C2
 * shapes) run all iterations in ONE persistent launch (k_swarm: cluster
 * barrier + DSMEM gBest exchange per iteration); larger swarms replay the
 * fused + gBest kernel pair from a captured CUDA graph. */
int psso_run(psso_ctx* ctx, int64_t t0, int64_t niter);

/* replaces: the loop of run_sequential (core.py:222-244), the per-particle
 * asynchronous schedule: particles updated in index order against the LIVE
 * gbest, which moves as soon as a new pbest is <= g_f (core.py:236-241).
 * Same keyed draws as psso_run; trajectory[t] = g_f after iteration t.  Each
 * iteration runs as speculative passes -- all remaining particles computed in
 * parallel against the current gbest, the prefix up to the first gbest move
 * (or non-finite fitness) committed, the next pass starting after it -- so
 * results are bit-identical to the serial loop.  nvar <= 128: ONE launch
 * (k_seq, asynchronous).  Longer rows: a pass loop of device kernels over the
 * resident swarm (search + evaluate into scratch, first-event search, commit,
 * gbest move); the host reads 16 bytes per pass, so the call returns when the
 * iterations are done.  Unsharded contexts (else PSSO_E_INVALID).  Call
 * psso_init first (core.py:220). */
int psso_run_sequential(psso_ctx* ctx, int64_t t0, int64_t niter);

/* Passes k_seq ran in the last psso_run_sequential (iterations + gbest moves
 * when nothing is non-finite).  Synchronizes the stream. */
int psso_sequential_passes(psso_ctx* ctx, int64_t* passes);

/* Name of the iteration kernel psso_run uses for this configuration
 * (k_swarm / k_chain / k_rows / k_fused / k_tile with its template arguments). */
const char* psso_kernel_name(const psso_ctx* ctx);

/* Phase API -- replaces search_phase / evaluate_phase / update_pbests_phase /
 * update_gbest_phase (parallel.py:120-144).  `t < 0` in psso_evaluate means
 * "iteration None" (the evaluation is not attributed to an iteration). */
int psso_search(psso_ctx* ctx, int64_t t);
int psso_evaluate(psso_ctx* ctx, int64_t t);
int psso_update_pbests(psso_ctx* ctx);
int psso_update_gbest(psso_ctx* ctx);

/* Sharded (multi-rank) iteration, split around the gBest exchange.
 * A candidate record is psso_candidate_bytes(cfg) bytes:
 *   float64 p_f, int64 global index, uint64 the shard's first non-finite key
 *   ((t+1) << 40 | i, all ones if none), float64 that fitness value, then nvar
 *   elements of dtype (the row) at offset 32.  Applying the records also
 *   adopts the smallest non-finite key, so every shard stops at the same
 *   iteration and psso_check reports the same first (t, i) on every rank.
 * psso_step_local: fused kernel over this context's rows, then the local
 * stage-2 reduction, writing this rank's record to `cand` (device).
 * psso_apply_candidates: lexicographic (p_f, index) min over `ncand` gathered
 * records, `<=` against g_f, gbest <- winning row, trajectory[t] = g_f.
 * Replaces the per-slice candidates + `min(candidates)` of parallel.py:199-212. */
int64_t psso_candidate_bytes(const psso_config* cfg);
int psso_init_local(psso_ctx* ctx, void* cand);
int psso_step_local(psso_ctx* ctx, int64_t t, void* cand);
int psso_apply_candidates(psso_ctx* ctx, int64_t t, const void* cands, int32_t ncand, int32_t is_init);

/* Sharded iteration over a communicator the library owns (one process per
 * GPU; replaces the per-slice candidates + min() of parallel.py:199-212 across
 * GPUs).  psso_nccl_unique_id: a 128-byte ncclUniqueId made on rank 0 and
 * handed to every rank (e.g. over torch.distributed); psso_comm_create:
 * collective ncclCommInitRank on the current device, rank `rank` of `nranks`
 * (a session resource: create once, attach to every run's context);
 * psso_attach_comm: the context (whose row range must be that rank's shard)
 * borrows it until psso_destroy.  Then
 * psso_init_sharded = initialize (core.py:196-210) over all shards, and
 * psso_run_sharded = iterations t0..t0+niter-1, each: fused iteration kernel on
 * the local rows -> this rank's candidate record -> ncclAllGather of the
 * records over NVLink / NVSwitch -> k_apply (identical selection on every
 * rank, trajectory[t]).  Iterations are replayed from a captured CUDA graph of
 * 16 (kernels + collective), so the host issues one launch per 16 iterations.
 * NCCL is resolved at run time (dlopen "libnccl.so.2", or PSSO_NCCL_LIB). */
typedef struct psso_comm psso_comm;
int psso_nccl_unique_id(void* id /* 128 bytes */);
int psso_comm_create(const void* id, int32_t nranks, int32_t rank, psso_comm** out);
void psso_comm_destroy(psso_comm* comm);
int psso_attach_comm(psso_ctx* ctx, psso_comm* comm);  /* ctx borrows it */
int psso_init_sharded(psso_ctx* ctx);
int psso_run_sharded(psso_ctx* ctx, int64_t t0, int64_t niter);

/* Device-initiated gBest exchange (replaces the NCCL all-gather of the
 * records; SURVEY §8 f #3).  Every rank owns an exchange buffer of
 * psso_p2p_buffer_bytes(cfg, R) bytes ([2][R] epoch flags, [2][R] candidate
 * records: double-buffered by epoch parity, since a rank may run one exchange ahead),
 * allocated with psso_p2p_alloc; peers map it through psso_p2p_handle /
 * psso_p2p_open (CUDA IPC over NVLink P2P).  Per iteration, after
 * psso_step_local / psso_init_local wrote the local record `cand`:
 *   psso_publish_p2p: stores `cand` into slot `rank` of every rank's buffer
 *     (`peer_bufs` = DEVICE array of R buffer pointers, own included) and
 *     raises this rank's flag in each buffer to `epoch` (system-scope release);
 *   psso_apply_p2p: waits until the R flags of this rank's buffer reached
 *     `epoch` (system-scope acquire), then applies the selection exactly like
 *     psso_apply_candidates.
 * `epoch` must increase by at least 1 per exchange (buffers start at 0).
 * No host synchronization and no collective library on the path. */
int64_t psso_p2p_buffer_bytes(const psso_config* cfg, int32_t nranks);
int psso_p2p_alloc(int64_t bytes, void** dev_ptr);
int psso_p2p_free(void* dev_ptr);
int psso_p2p_handle(void* dev_ptr, void* handle /* 64 bytes (cudaIpcMemHandle_t) */);
int psso_p2p_open(const void* handle, void** dev_ptr);
int psso_p2p_close(void* dev_ptr);
int psso_publish_p2p(psso_ctx* ctx, const void* cand, void* const* peer_bufs, int32_t nranks,
                     int32_t rank, uint64_t epoch);
int psso_apply_p2p(psso_ctx* ctx, int64_t t, const void* my_buf, int32_t nranks, uint64_t epoch,
                   int32_t is_init);

/* Iterations t0..t0+niter-1 with the device-initiated exchange, replayed from
 * a captured CUDA graph of 16 iterations (per iteration the fused kernel and
 * ONE exchange kernel: record, publish, wait for every rank's flag, apply;
 * the epoch is t + 2, read from the device iteration counter, so the graph
 * needs no host values).  Initialize with psso_init_local +
 * psso_publish_p2p / psso_apply_p2p at epoch 1.  `peer_bufs` (device array)
 * and `my_buf` as for psso_publish_p2p / psso_apply_p2p.  Asynchronous. */
int psso_run_p2p(psso_ctx* ctx, int64_t t0, int64_t niter, void* const* peer_bufs, const void* my_buf,
                 int32_t nranks, int32_t rank);

/* Synchronizes the stream and reports the first non-finite fitness seen so
 * far as (iteration, particle); iteration -1 = initialization.  Returns
 * PSSO_E_NONFINITE if there was one (core.py:190-193 semantics). */
int psso_check(psso_ctx* ctx, int64_t* bad_t, int64_t* bad_i);

/* replaces: reading Swarm.g_f and the gBest argmin index after a run
 * (parallel.py:208-211 select `best = min(candidates)`; core.py:202 at
 * initialization).  Synchronizes the stream; writes the gBest fitness and the
 * GLOBAL particle index whose pBest row is gbest (-1 before psso_init), and
 * the first non-finite fitness like psso_check.  Any output may be NULL.
 * Returns PSSO_E_NONFINITE (outputs still written) if there was one. */
int psso_result(psso_ctx* ctx, double* g_f, int64_t* g_idx, int64_t* bad_t, int64_t* bad_i);

/* Per-iteration statistics the streaming iteration kernels (k_chain, k_rows)
 * record on the device -- also inside graph replays: for iterations
 * t0..t0+n-1 (n <= 1024, the most recent 1024 iterations are kept), the summed
 * kernel duration (first CTA start to last CTA end, %globaltimer), the number
 * of rows whose pBest improved (parallel.py:108-112; the rho of the roofline's
 * pBest write-back bytes) and how many of the iterations were recorded
 * (0 for kernels without statistics).  Synchronizes the stream. */
int psso_iteration_stats(psso_ctx* ctx, int64_t t0, int64_t n, double* kernel_ms,
                         int64_t* improved_rows, int64_t* timed_iterations);

/* psso_check plus the non-finite fitness value (NonFiniteFitnessError.value,
 * core.py:43-53), also on shards that do not own the failing particle (the
 * value travels in the candidate records).  *value = 0 when there is none. */
int psso_nonfinite(psso_ctx* ctx, int64_t* bad_t, int64_t* bad_i, double* value);

/* Sets the gBest index psso_result reports, for swarm state uploaded by the
 * host (a checkpoint, a Swarm handed to the phase API).  Asynchronous. */
int psso_set_gbest_index(psso_ctx* ctx, int64_t g_idx);

/* Number of kernels this context has launched (for launch accounting). */
int64_t psso_launch_count(const psso_ctx* ctx);

/* Kernel timing for the roofline: while enabled, psso_step / psso_run (which
 * then launches directly instead of replaying its graph) bracket every
 * iteration-kernel launch with CUDA events on the context's stream.
 * psso_profile_read synchronizes, returns the summed kernel time (ms) and the
 * number of iterations those launches covered (one per fused launch, niter per
 * whole-run launch), and resets the record. */
int psso_profile(psso_ctx* ctx, int32_t enable);
int psso_profile_read(psso_ctx* ctx, double* kernel_ms, int64_t* nlaunch);

/* replaces: RngStream.uniform (rng.py:73-87) on device: out[k] =
 * u(seed, stream_key, t, particles[k], variables[k]). */
int psso_rng_uniform(uint64_t seed, uint64_t stream_key, uint64_t t, const uint64_t* particles,
                     const uint64_t* variables, int64_t n, double* out, void* stream);

/* replaces: BenchmarkFn.__call__ (benchmarks.py:86-94) on device: fitness of
 * `rows` contiguous rows of length nvar (dtype) into out (float64). */
int psso_eval_rows(int32_t fn_id, int32_t dtype, int64_t nvar, const void* x, int64_t rows,
                   double* out, double probe_level, void* stream);

/* replaces: run_parallel (parallel.py:152-233) end to end with HOST buffers:
 * allocates device state, initializes, runs niter iterations, copies the
 * trajectory (niter float64), best position (nvar of dtype) and best fitness
 * back, frees.  wall_s = loop-only device time (parallel.py:190,216). */
int psso_solve(const psso_config* cfg, int64_t niter, double* traj, void* best_position,
               double* best_fitness, double* wall_s);

/* replaces: the reference's multi-seed protocol -- one run_parallel per seed
 * (harness.py:148-163, 217-263: seed = base_seed + run_id) -- as ONE device
 * job: nseeds independent swarms of cfg (cfg->seed ignored), each with its own
 * keyed RNG seed, run side by side by the whole-run kernel.  Per swarm the
 * results are bit-identical to psso_solve with that seed.  Outputs (host):
 * traj nseeds x niter, best_position nseeds x nvar (dtype), best_fitness
 * nseeds.  wall_s = loop-only device time of the whole batch.  Needs
 * nvar <= 128 and nsol*nvar <= 2^22 (else PSSO_E_UNSUPPORTED). */
int psso_solve_batch(const psso_config* cfg, const uint64_t* seeds, int32_t nseeds, int64_t niter,
                     double* traj, void* best_position, double* best_fitness, double* wall_s);

/* replaces: one run_sequential per seed (harness.py:148-163 with
 * ScheduleKind.SEQUENTIAL) as ONE device job: nseeds swarms of cfg initialized
 * together, then the sequential loop of all of them in one k_seq launch (one
 * CTA per swarm).  Per swarm bit-identical to run_sequential with that seed.
 * Same buffers, limits and errors as psso_solve_batch. */
int psso_solve_sequential_batch(const psso_config* cfg, const uint64_t* seeds, int32_t nseeds,
                                int64_t niter, double* traj, void* best_position,
                                double* best_fitness, double* wall_s);

/* The non-finite failure of this thread's last psso_solve_batch /
 * psso_solve_sequential_batch (NonFiniteFitnessError's fields, core.py:43-53):
 * the failing swarm's position in `seeds`, the iteration (-1 = initialization),
 * the particle and the fitness value.  PSSO_E_NONFINITE if that call failed so,
 * else PSSO_OK with *swarm = -1. */
int psso_batch_failure(int64_t* swarm, int64_t* iteration, int64_t* particle, double* value);

#ifdef __cplusplus
}
#endif

#endif /* PSSO_H */
