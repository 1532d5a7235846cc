/*
 * psso_oracle.c -- CPU restatement of the reference PSSO hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library; the
 * product package (paper_2110_01470_b200/) never does.  It is the checker the
 * CUDA path is compared against, and the "port" CPU baseline.
 *
 * Parity pinning: tests/test_oracle_golden.py checks every function here
 * against fixtures produced by running the reference package itself
 * (tests/golden/make_golden.py).  Bitwise: the keyed RNG, positions, and
 * f1-f5, f7, f9 fitness (numpy order, no FMA, glibc cos/sin/sqrt).  Within a
 * few ulps: f6 (numpy's SIMD exp) and f8 (numpy's SIMD pow).
 *
 * Reference anchors (paths under /root/reference/pkg/src/sso/):
 *   rng.py:27-31   constants; rng.py:34-39 SubStream keys
 *   rng.py:48-58   _mix / _fold (SplitMix64 finalizer chain)
 *   rng.py:67-87   RngStream._root / uniform  (u = (h >> 11) * 2^-53)
 *   core.py:118-135 step_update_variable (keep -> pbest -> gbest -> fresh)
 *   core.py:138-173 _draw_update_fields / _compose_update
 *   core.py:196-210 initialize
 *   parallel.py:93-117 search / evaluate / pbest / gbest-candidate slices
 *   parallel.py:192-212 run_parallel loop body
 *   benchmarks.py:109-166 objective bodies; numpy's pairwise add.reduce
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off -fopenmp).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define GAMMA 0x9E3779B97F4A7C15ULL
#define MIX1 0xBF58476D1CE4E5B9ULL
#define MIX2 0x94D049BB133111EBULL
#define STREAM_BRANCH 0x243F6A8885A308D3ULL
#define STREAM_FRESH 0x13198A2E03707344ULL
#define STREAM_INIT 0xA4093822299F31D0ULL

static const double TWO_PI = 6.283185307179586;      /* 2.0 * np.pi, benchmarks.py:52 */
static const double EULER_E = 2.718281828459045;     /* np.e */
static const double SCHWEFEL = 418.9829;            /* benchmarks.py:53 */

/* ---------------------------------------------------------------- RNG ---- */

static inline uint64_t mix64(uint64_t z) { /* rng.py:48-52 */
    z = (z ^ (z >> 30)) * MIX1;
    z = (z ^ (z >> 27)) * MIX2;
    return z ^ (z >> 31);
}

static inline uint64_t fold64(uint64_t h, uint64_t f) { /* rng.py:55-58 */
    return mix64(h ^ (GAMMA * (f + 1)));
}

static inline uint64_t root64(uint64_t seed, uint64_t stream, uint64_t t) { /* rng.py:67-69 */
    return fold64(mix64(seed ^ stream), t);
}

static inline double to_unit(uint64_t h) { /* rng.py:87 */
    return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

double oracle_u(uint64_t seed, uint64_t stream, uint64_t t, uint64_t i, uint64_t j) {
    return to_unit(fold64(fold64(root64(seed, stream, t), i), j));
}

void oracle_u_batch(uint64_t seed, uint64_t stream, uint64_t t, const uint64_t* i,
                    const uint64_t* j, int64_t n, double* out) {
    uint64_t r = root64(seed, stream, t);
    for (int64_t k = 0; k < n; ++k) out[k] = to_unit(fold64(fold64(r, i[k]), j[k]));
}

/* Philox4x32-10 (Salmon et al., SC'11) -- the benchmark-mode generator of the
 * device path; restated here only for its known-answer test. */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* ------------------------------------------------- numpy pairwise sum ---- */
/* numpy's add.reduce over a contiguous axis: blocks of <= 128 with eight
 * strided accumulators, recursive halving (split rounded down to a multiple
 * of 8) above that; blocks shorter than 8 are summed from 0.0 left to right. */
static double pw_sum(const double* a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res = res + a[i];
        return res;
    }
    if (n <= 128) {
        double r[8];
        for (int k = 0; k < 8; ++k) r[k] = a[k];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int k = 0; k < 8; ++k) r[k] = r[k] + a[i + k];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res = res + a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pw_sum(a, n2) + pw_sum(a + n2, n - n2);
}

double oracle_pairwise_sum(const double* a, int64_t n) { return pw_sum(a, n); }

/* ------------------------------------------------------- objectives ---- */
/* benchmarks.py:109-166; scratch must hold >= D doubles. */
static double fitness_row(int fid, int64_t D, const double* x, double* s) {
    switch (fid) {
    case 1: /* sum(x * x) */
        for (int64_t j = 0; j < D; ++j) s[j] = x[j] * x[j];
        return pw_sum(s, D);
    case 2: /* sum(weights * x * x), weights = 1..D */
        for (int64_t j = 0; j < D; ++j) s[j] = ((double)(j + 1) * x[j]) * x[j];
        return pw_sum(s, D);
    case 3: { /* c = cumsum(x); sum(c * c) */
        double c = 0.0;
        for (int64_t j = 0; j < D; ++j) {
            c = (j == 0) ? x[0] : c + x[j];
            s[j] = c * c;
        }
        return pw_sum(s, D);
    }
    case 4: /* sum(100 d d + (1 - h)^2), d = x[1:] - h*h, h = x[:-1] */
        for (int64_t j = 0; j + 1 < D; ++j) {
            double h = x[j];
            double d = x[j + 1] - h * h;
            double o = 1.0 - h;
            s[j] = (100.0 * d) * d + o * o;
        }
        return pw_sum(s, D - 1);
    case 5: /* 10 D + sum(x*x - 10 cos(2 pi x)) */
        for (int64_t j = 0; j < D; ++j) s[j] = x[j] * x[j] - 10.0 * cos(TWO_PI * x[j]);
        return 10.0 * (double)D + pw_sum(s, D);
    case 6: { /* Ackley */
        for (int64_t j = 0; j < D; ++j) s[j] = x[j] * x[j];
        double rms = sqrt(pw_sum(s, D) / (double)D);
        for (int64_t j = 0; j < D; ++j) s[j] = cos(TWO_PI * x[j]);
        double mc = pw_sum(s, D) / (double)D;
        return ((-20.0 * exp(-0.2 * rms) - exp(mc)) + 20.0) + EULER_E;
    }
    case 7: { /* Griewank: sum(x*x)/4000 - prod(cos(x * inv)) + 1, inv = 1/sqrt(1..D) */
        for (int64_t j = 0; j < D; ++j) s[j] = x[j] * x[j];
        double q = pw_sum(s, D) / 4000.0;
        double p = 1.0;
        for (int64_t j = 0; j < D; ++j) p = p * cos(x[j] * (1.0 / sqrt((double)(j + 1))));
        return (q - p) + 1.0;
    }
    case 8: { /* Powell singular, first 4*floor(D/4) coordinates */
        int64_t g = D / 4;
        for (int64_t k = 0; k < g; ++k) {
            double a = x[4 * k], b = x[4 * k + 1], c = x[4 * k + 2], d = x[4 * k + 3];
            double t1 = a + 10.0 * b;
            double t2 = c - d;
            double t3 = b - 2.0 * c;
            double t4 = a - d;
            s[k] = ((t1 * t1 + 5.0 * (t2 * t2)) + pow(t3, 4.0)) + 10.0 * pow(t4, 4.0);
        }
        return pw_sum(s, g);
    }
    case 9: /* 418.9829 D - sum(x sin(sqrt|x|)) */
        for (int64_t j = 0; j < D; ++j) s[j] = x[j] * sin(sqrt(fabs(x[j])));
        return SCHWEFEL * (double)D - pw_sum(s, D);
    default:
        return NAN;
    }
}

int oracle_eval(int fid, int64_t D, const double* x, int64_t rows, double* out, int threads) {
    if (fid < 1 || fid > 9 || D < 1) return -1;
    (void)threads;
#pragma omp parallel num_threads(threads > 0 ? threads : 1)
    {
        double* s = (double*)malloc(sizeof(double) * (size_t)D);
#pragma omp for schedule(static)
        for (int64_t r = 0; r < rows; ++r) out[r] = fitness_row(fid, D, x + r * D, s);
        free(s);
    }
    return 0;
}

/* ----------------------------------------------------------- engine ---- */

typedef struct oracle_cfg {
    int32_t fid;
    int32_t threads;      /* OpenMP threads for the row loops (results independent) */
    int64_t nsol, nvar;   /* nsol = rows held in the arrays */
    int64_t row_lo;       /* global index of array row 0 (shards); 0 when unsharded */
    double cw, cp, cg, var_min, var_max;
    uint64_t seed;
} oracle_cfg;

/* Exact equivalent of (h >> 11) * 2^-53 < c: k < ceil(c * 2^53). */
static inline uint64_t thresh53(double c) {
    double y = ceil(c * 9007199254740992.0);
    if (y <= 0.0) return 0;
    if (y >= 9007199254740992.0) return (uint64_t)1 << 53;
    return (uint64_t)y;
}

static int argmin_lex(const double* f, int64_t n) { /* np.argmin: lowest index */
    int64_t best = 0;
    for (int64_t i = 1; i < n; ++i)
        if (f[i] < f[best]) best = i;
    return (int)best;
}

static int64_t argmin64(const double* f, int64_t n) {
    int64_t best = 0;
    for (int64_t i = 1; i < n; ++i)
        if (f[i] < f[best]) best = i;
    return best;
}

/* core.py:196-210.  Returns 0, or 1 with *bad_i set on a non-finite fitness. */
int oracle_init(const oracle_cfg* c, double* X, double* P, double* sol_f, double* p_f,
                double* gbest, double* g_f, int64_t* bad_i) {
    const int64_t N = c->nsol, D = c->nvar;
    const double span = c->var_max - c->var_min;
    const uint64_t r0 = root64(c->seed, STREAM_INIT, 0);
#pragma omp parallel num_threads(c->threads > 0 ? c->threads : 1)
    {
        double* s = (double*)malloc(sizeof(double) * (size_t)(D + 4));
#pragma omp for schedule(static)
        for (int64_t i = 0; i < N; ++i) {
            uint64_t hi = fold64(r0, (uint64_t)(c->row_lo + i));
            double* x = X + i * D;
            for (int64_t j = 0; j < D; ++j) x[j] = c->var_min + span * to_unit(fold64(hi, (uint64_t)j));
            memcpy(P + i * D, x, sizeof(double) * (size_t)D);
            sol_f[i] = fitness_row(c->fid, D, x, s);
            p_f[i] = sol_f[i];
        }
        free(s);
    }
    for (int64_t i = 0; i < N; ++i)
        if (!isfinite(sol_f[i])) { *bad_i = i; return 1; }
    int64_t b = argmin64(sol_f, N);
    memcpy(gbest, X + b * D, sizeof(double) * (size_t)D);
    *g_f = sol_f[b];
    return 0;
}

/* parallel.py:93-98 + core.py:138-173 for rows [lo, hi): rewrites X only. */
static void search_rows(const oracle_cfg* c, int64_t t, double* X, const double* P,
                        const double* gbest, int64_t lo, int64_t hi) {
    const int64_t D = c->nvar;
    const double span = c->var_max - c->var_min;
    const uint64_t kw = thresh53(c->cw), kp = thresh53(c->cp), kg = thresh53(c->cg);
    const uint64_t rb = root64(c->seed, STREAM_BRANCH, (uint64_t)t);
    const uint64_t rf = root64(c->seed, STREAM_FRESH, (uint64_t)t);
    for (int64_t i = lo; i < hi; ++i) {
        uint64_t gi = (uint64_t)(c->row_lo + i);
        uint64_t hb = fold64(rb, gi), hf = fold64(rf, gi);
        double* x = X + i * D;
        const double* p = P + i * D;
        for (int64_t j = 0; j < D; ++j) {
            uint64_t k = fold64(hb, (uint64_t)j) >> 11;
            double v;
            if (k < kw) v = x[j];
            else if (k < kp) v = p[j];
            else if (k < kg) v = gbest[j];
            else v = c->var_min + span * to_unit(fold64(hf, (uint64_t)j));
            x[j] = v;
        }
    }
}

int oracle_search(const oracle_cfg* c, int64_t t, double* X, const double* P, const double* gbest) {
#pragma omp parallel for num_threads(c->threads > 0 ? c->threads : 1) schedule(static)
    for (int64_t i = 0; i < c->nsol; ++i) search_rows(c, t, X, P, gbest, i, i + 1);
    return 0;
}

/* One full iteration (parallel.py:195-212).  Returns 0, or 1 with *bad_i. */
int oracle_step(const oracle_cfg* c, int64_t t, double* X, double* P, double* sol_f,
                double* p_f, double* gbest, double* g_f, int64_t* bad_i) {
    const int64_t N = c->nsol, D = c->nvar;
    /* search reads P and gbest as they stood at phase entry: rows are disjoint
       and gbest is only written below, so the live arrays are the snapshot */
#pragma omp parallel num_threads(c->threads > 0 ? c->threads : 1)
    {
        double* s = (double*)malloc(sizeof(double) * (size_t)(D + 4));
#pragma omp for schedule(static)
        for (int64_t i = 0; i < N; ++i) {
            search_rows(c, t, X, P, gbest, i, i + 1);
            sol_f[i] = fitness_row(c->fid, D, X + i * D, s);
            if (sol_f[i] <= p_f[i]) { /* parallel.py:109 */
                memcpy(P + i * D, X + i * D, sizeof(double) * (size_t)D);
                p_f[i] = sol_f[i];
            }
        }
        free(s);
    }
    for (int64_t i = 0; i < N; ++i)
        if (!isfinite(sol_f[i])) { *bad_i = i; return 1; }
    /* NB: a non-finite sol_f never reaches P: NaN <= x is false, +inf <= finite false */
    int64_t b = argmin64(p_f, N);
    if (p_f[b] <= *g_f) { /* parallel.py:209-211 */
        *g_f = p_f[b];
        memcpy(gbest, P + b * D, sizeof(double) * (size_t)D);
    }
    return 0;
}

/* Shard-local iteration for sharded drivers: search + evaluate + pbest over
 * this shard's rows, then its (p_f, global index) candidate (parallel.py:115-117). */
int oracle_step_local(const oracle_cfg* c, int64_t t, double* X, double* P, double* sol_f,
                      double* p_f, const double* gbest, double* cand_f, int64_t* cand_i,
                      int64_t* bad_i) {
    const int64_t N = c->nsol, D = c->nvar;
    double* s = (double*)malloc(sizeof(double) * (size_t)(D + 4));
    for (int64_t i = 0; i < N; ++i) {
        if (t >= 0) {
            search_rows(c, t, X, P, gbest, i, i + 1);
        }
        sol_f[i] = fitness_row(c->fid, D, X + i * D, s);
        if (t < 0 || sol_f[i] <= p_f[i]) {
            if (t >= 0) memcpy(P + i * D, X + i * D, sizeof(double) * (size_t)D);
            p_f[i] = sol_f[i];
        }
    }
    free(s);
    for (int64_t i = 0; i < N; ++i)
        if (!isfinite(sol_f[i])) { *bad_i = c->row_lo + i; return 1; }
    int64_t b = argmin64(p_f, N);
    *cand_f = p_f[b];
    *cand_i = c->row_lo + b;
    return 0;
}

int oracle_run(const oracle_cfg* c, int64_t t0, int64_t niter, double* X, double* P,
               double* sol_f, double* p_f, double* gbest, double* g_f, double* traj,
               int64_t* bad_t, int64_t* bad_i) {
    for (int64_t t = t0; t < t0 + niter; ++t) {
        if (oracle_step(c, t, X, P, sol_f, p_f, gbest, g_f, bad_i)) { *bad_t = t; return 1; }
        traj[t - t0] = *g_f;
    }
    return 0;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* unused helper kept static-clean */
int oracle_argmin(const double* f, int64_t n) { return argmin_lex(f, n); }

/* ------------------------------------------------ sequential schedule ---- */
/* run_sequential loop body (core.py:224-243): the same keyed draws as the
 * parallel schedule (_draw_update_fields over all rows, core.py:225), but
 * particles are updated one at a time in index order against the LIVE gbest,
 * and gbest moves as soon as a particle's new pbest is <= g_f (core.py:236-241).
 * Non-finite fitness: the row is already in X (core.py:231), nothing else is
 * written, and the first such particle is reported (core.py:233-234).
 * Returns 0, or 1 with *bad_i set (sol_f[*bad_i] holds the value). */
int oracle_step_seq(const oracle_cfg* c, int64_t t, double* X, double* P, double* sol_f,
                    double* p_f, double* gbest, double* g_f, int64_t* bad_i) {
    const int64_t N = c->nsol, D = c->nvar;
    double* s = (double*)malloc(sizeof(double) * (size_t)(D + 4));
    for (int64_t i = 0; i < N; ++i) {
        search_rows(c, t, X, P, gbest, i, i + 1);
        const double fx = fitness_row(c->fid, D, X + i * D, s);
        sol_f[i] = fx;
        if (!isfinite(fx)) { *bad_i = i; free(s); return 1; }
        if (fx <= p_f[i]) {
            memcpy(P + i * D, X + i * D, sizeof(double) * (size_t)D);
            p_f[i] = fx;
            if (fx <= *g_f) {
                memcpy(gbest, P + i * D, sizeof(double) * (size_t)D);
                *g_f = fx;
            }
        }
    }
    free(s);
    return 0;
}

/* run_sequential's loop (core.py:222-244); traj[t - t0] = g_f after iteration t. */
int oracle_run_seq(const oracle_cfg* c, int64_t t0, int64_t niter, double* X, double* P,
                   double* sol_f, double* p_f, double* gbest, double* g_f, double* traj,
                   int64_t* bad_t, int64_t* bad_i) {
    for (int64_t t = t0; t < t0 + niter; ++t) {
        if (oracle_step_seq(c, t, X, P, sol_f, p_f, gbest, g_f, bad_i)) { *bad_t = t; return 1; }
        traj[t - t0] = *g_f;
    }
    return 0;
}
