// psso_device.cuh -- sm_100a device code of the PSSO hot path.
//
// One templated tile kernel (k_tile) implements, selected by a warp-uniform
// mode mask, every per-particle stage of the reference phased engine:
//   INIT   core.py:196-210   positions from the INIT stream, pbests = sol
//   SEARCH core.py:138-173   keyed branch draw + four-way select (+ fresh draw)
//   EVAL   core.py:176-193   per-row fitness in numpy's reduction order
//   PBEST  parallel.py:108-112  sol_f <= p_f -> pbest row written from smem
//   CAND   parallel.py:115-117  per-CTA lexicographic (p_f, index) candidate
// The fused hot path is SEARCH|EVAL|PBEST|CAND: X and P are read once and X
// written once per iteration; pbest rows are written from the smem copy of the
// new positions (no re-read of X); gBest stage 2 is k_gbest (psso_api.cu).
//
// Compiled with --fmad=false: every position and fitness expression rounds
// exactly like numpy's separate multiply and add.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <math_constants.h>

#include "psso_trig.cuh"

namespace psso {

constexpr int NT = 256;            // threads per CTA of k_tile
#ifndef PSSO_U
#define PSSO_U 4  // phase-A chunks loaded per thread before compute
#endif
#ifndef PSSO_MINB
#define PSSO_MINB 4  // resident CTAs per SM the register budget is sized for
#endif
constexpr int MAX_LEAVES = 64;     // pairwise-sum leaves per row (D <= ~8192)
constexpr int MAX_OPS = 2 * MAX_LEAVES;

constexpr uint64_t GAMMA = 0x9E3779B97F4A7C15ULL;  // rng.py:28
constexpr uint64_t MIX1 = 0xBF58476D1CE4E5B9ULL;   // rng.py:29
constexpr uint64_t MIX2 = 0x94D049BB133111EBULL;   // rng.py:30
constexpr uint64_t STREAM_BRANCH = 0x243F6A8885A308D3ULL;  // rng.py:37
constexpr uint64_t STREAM_FRESH = 0x13198A2E03707344ULL;   // rng.py:38
constexpr uint64_t STREAM_INIT = 0xA4093822299F31D0ULL;    // rng.py:39

enum Mode : int {
  M_INIT = 1,
  M_SEARCH = 2,
  M_EVAL = 4,
  M_PBEST = 8,
  M_CAND = 16,
  M_LOAD = 32,  // EVAL without SEARCH/INIT: positions are loaded from X
  M_SOLF = 64,  // write sol_f for every row (otherwise only non-finite rows)
};

// numpy add.reduce pairwise plan for one row of n terms (host-built, see
// build_plan in psso_api.cu): leaves of <= 128 terms, combined in the
// recursion's post-order (ops >= 0 push leaf, -1 add top two).
struct Plan {
  int32_t n;
  int32_t nleaves;
  int32_t nops;
  int32_t pad;
  int32_t leaf_off[MAX_LEAVES];
  int32_t leaf_len[MAX_LEAVES];
  int8_t ops[MAX_OPS];
};

// q = n / d for 0 <= n < 2^31 (Granlund-Montgomery, round-up multiplier).
struct FastDiv {
  uint32_t d, m, s;
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return (__umulhi(n, m) + n) >> s;
  }
};

struct TileParams {
  void* X;             // local rows x D (dtype T)
  void* P;
  double* sol_f;       // may be null
  double* p_f;
  const void* gbest;   // D (dtype T)
  int64_t rows;        // local rows
  int64_t row_lo;      // global index of local row 0
  int32_t D;
  int32_t R;           // rows per tile
  int32_t G;           // phase-B threads per row (8 per leaf)
  int32_t S;           // smem row stride in elements
  int32_t cpr;         // vector chunks per row (D / V)
  int32_t mode;
  FastDiv div_cpr;
  FastDiv div_G;
  FastDiv div_D;
  FastDiv div_n;               // by the row's term count (plan.n)
  int32_t fn_pad;
  uint64_t seed;
  uint64_t Kw, Kp, Kg;         // reference mode: branch k = h >> 11 compared < K
  uint64_t Kw32, Kp32, Kg32;   // philox mode: 32-bit word compared < K32
  uint32_t Kw32u, Kp32u, Kg32u;  // the same as 32-bit values (K32 < 2^32) ...
  uint32_t K32on;                // ... bit b clear when threshold b is 1.0 (K32 = 2^32: never)
  double var_min, span;
  double span53;               // span * 2^-53 (fresh = var_min + k * span53, exact rescale)
  double span64;               // span * 2^-64 (see fresh_offset)
  double span32;               // span * 2^-32 (fp32 Philox fresh draw)
  double probe_level;
  int64_t t_arg;
  const int64_t* t_dev;        // if non-null, the iteration is read from here
  double* slot_f;              // per-CTA candidates (M_CAND)
  int64_t* slot_i;
  unsigned long long* bad;     // first non-finite key ((t+1) << 40 | i)
  const double* aux;           // f7: 1/sqrt(1..D) table
  int32_t off_xs, off_scr, off_gb, off_hb, off_hf, off_leaf, off_rowf, off_flag, off_red;
  int32_t pre;                 // heavy terms precomputed by all threads (see tile_fitness)
  int32_t off_bar;             // k_fused: two mbarriers; stages start at off_xs
  int32_t stage_bytes;         // k_fused: bytes of one stage (X tile + P tile)
  int32_t pad3;
  unsigned long long* stats;   // per-iteration ring [STATS_CAP][3] (see iter_stats) or null
  Plan plan;
};

// ---- per-iteration kernel statistics (psso_iteration_stats) ---------------
// The streaming iteration kernels (k_chain, k_rows) record, per iteration t,
// the launch's first CTA start and last CTA end (%globaltimer, ns) and the
// number of rows whose pBest improved (parallel.py:108-112: the pBest
// write-back bytes of the roofline's rho term).  Slot t & (STATS_CAP-1) is
// reset by the gBest kernel of iteration t-1.  Recorded inside graph replays
// too, where per-launch CUDA events cannot be.
constexpr int STATS_CAP = 1024;

// Programmatic dependent launch (PSSO_PDL): the iteration kernels and k_gbest
// are launched so that each may be scheduled while its predecessor drains;
// every read of a predecessor's output sits behind griddepcontrol.wait.
#ifndef PSSO_PDL
#define PSSO_PDL 0
#endif
__device__ __forceinline__ void pdl_wait() {
#if PSSO_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_trigger() {
#if PSSO_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// whole CTA calls, after its last global store; nimp = this thread's improved rows
__device__ __forceinline__ void iter_stats(unsigned long long* stats, int64_t t,
                                           unsigned long long t_start, int nimp) {
  if (!stats || t < 0) return;
  unsigned long long* st = stats + 3 * (t & (STATS_CAP - 1));
  const int w = __reduce_add_sync(0xffffffffu, (unsigned)nimp);
  if ((threadIdx.x & 31) == 0 && w) atomicAdd(st + 2, (unsigned long long)w);
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicMin(st, t_start);
    atomicMax(st + 1, gtimer());
  }
}

// ------------------------------------------------------------------ RNG ----

__device__ __forceinline__ uint64_t xs30(uint64_t z) { return z ^ (z >> 30); }
// z * C mod 2^64 in three IMADs (lo*Clo wide, then the two cross terms added
// straight into the high word); the C++ form costs a fourth (IADD) but has a
// shorter dependency chain
template <uint64_t C>
__device__ __forceinline__ uint64_t mul64c(uint64_t z) {
  uint64_t r;
  asm("{\n\t.reg .u32 rl, rh;\n\t"
      "mul.wide.u32 %0, %1, %3;\n\t"
      "mov.b64 {rl, rh}, %0;\n\t"
      "mad.lo.u32 rh, %1, %4, rh;\n\t"
      "mad.lo.u32 rh, %2, %3, rh;\n\t"
      "mov.b64 %0, {rl, rh};\n\t}"
      : "=l"(r)
      : "r"((uint32_t)z), "r"((uint32_t)(z >> 32)), "n"((uint32_t)C), "n"((uint32_t)(C >> 32)));
  return r;
}
// mix64 after its first xorshift: mix64(z) == mix64_tail(xs30(z))
// LEAN: the three-IMAD multiplies (fewer instructions, longer chain).  Measured
// (sustained 500-iteration runs, where the board's power cap binds): faster
// for fp64 at every M (C3 0.565 -> 0.559 ms, C4) and for M <= 8; slower for
// fp32 at M = 16 (issue-bound: the four-IMAD form's parallel pair wins).
template <bool LEAN = false>
__device__ __forceinline__ uint64_t mix64_tail(uint64_t z) {
  if constexpr (LEAN) {
    z = mul64c<MIX1>(z);
    z = mul64c<MIX2>(z ^ (z >> 27));
  } else {
    z *= MIX1;
    z = (z ^ (z >> 27)) * MIX2;
  }
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // rng.py:48-52 (SplitMix64 finalizer)
  return mix64_tail(xs30(z));
}
// (h >> 11) * span * 2^-53 for h = mix64_tail(z), computed as
// (h & ~0x7ff) * (span * 2^-64): the masked value converts to double exactly
// and the power-of-two rescale is exact, so this equals the reference's
// var_min + span*u offset bit for bit with the final shift folded away.
template <bool LEAN = false>
__device__ __forceinline__ double fresh_offset(uint64_t z, double span64) {
  return __dmul_rn((double)(mix64_tail<LEAN>(z) & ~0x7ffull), span64);
}
__device__ __forceinline__ uint64_t fold64(uint64_t h, uint64_t f) {  // rng.py:55-58
  return mix64(h ^ (GAMMA * (f + 1)));
}
__device__ __forceinline__ uint64_t root64(uint64_t seed, uint64_t stream, uint64_t t) {
  return fold64(mix64(seed ^ stream), t);  // rng.py:67-69
}
__device__ __forceinline__ double unit53(uint64_t h) {  // rng.py:87, exact
  return __dmul_rn((double)(h >> 11), 1.1102230246251565e-16);
}

struct Philox4 { uint32_t w[4]; };

// Benchmark-mode keying: one Philox4x32-10 call per PAIR of coordinates
// {16a + b, 16a + b + 8} (b < 8) of a particle -- the two coordinates one lane
// of the chain mapping holds at m = 2a and 2a + 1 -- so each call's four words
// serve two coordinates: word h = branch draw, word 2 + h = fresh draw of the
// pair's half h (INIT: words 2h, 2h+1 = one 64-bit draw).
// counter = (pair, i_lo, i_hi, t or 0xFFFFFFFF for INIT), key = seed.
__device__ __forceinline__ uint32_t philox_pair(int j) { return (uint32_t)(((j >> 4) << 3) | (j & 7)); }
__device__ __forceinline__ int philox_half(int j) { return (j >> 3) & 1; }

// Philox4x32-10 (Salmon et al. 2011).
__device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2,
                                                 uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  Philox4 o; o.w[0] = c0; o.w[1] = c1; o.w[2] = c2; o.w[3] = c3;
  return o;
}

// Two independent Philox4x32-10 calls with their rounds interleaved (same key):
// twice the instruction-level parallelism of one serial 10-round chain.
__device__ __forceinline__ void philox4x32_10_x2(uint32_t a0, uint32_t b0, uint32_t c1, uint32_t c2,
                                                 uint32_t c3, uint32_t k0, uint32_t k1, Philox4& wa,
                                                 Philox4& wb) {
  uint32_t A0 = a0, A1 = c1, A2 = c2, A3 = c3;
  uint32_t B0 = b0, B1 = c1, B2 = c2, B3 = c3;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t ha0 = __umulhi(0xD2511F53u, A0), la0 = 0xD2511F53u * A0;
    const uint32_t ha1 = __umulhi(0xCD9E8D57u, A2), la1 = 0xCD9E8D57u * A2;
    const uint32_t hb0 = __umulhi(0xD2511F53u, B0), lb0 = 0xD2511F53u * B0;
    const uint32_t hb1 = __umulhi(0xCD9E8D57u, B2), lb1 = 0xCD9E8D57u * B2;
    A0 = ha1 ^ A1 ^ k0; A2 = ha0 ^ A3 ^ k1; A1 = la1; A3 = la0;
    B0 = hb1 ^ B1 ^ k0; B2 = hb0 ^ B3 ^ k1; B1 = lb1; B3 = lb0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  wa.w[0] = A0; wa.w[1] = A1; wa.w[2] = A2; wa.w[3] = A3;
  wb.w[0] = B0; wb.w[1] = B1; wb.w[2] = B2; wb.w[3] = B3;
}

// Four independent calls, rounds interleaved (PSSO_PHILOX_X2 == 4).
__device__ __forceinline__ void philox4x32_10_x4(const uint32_t (&a)[4], uint32_t c1, uint32_t c2,
                                                 uint32_t c3, uint32_t k0, uint32_t k1, Philox4 (&w)[4]) {
  uint32_t X0[4], X1[4], X2[4], X3[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) { X0[q] = a[q]; X1[q] = c1; X2[q] = c2; X3[q] = c3; }
#pragma unroll
  for (int r = 0; r < 10; ++r) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t h0 = __umulhi(0xD2511F53u, X0[q]), l0 = 0xD2511F53u * X0[q];
      const uint32_t h1 = __umulhi(0xCD9E8D57u, X2[q]), l1 = 0xCD9E8D57u * X2[q];
      X0[q] = h1 ^ X1[q] ^ k0; X2[q] = h0 ^ X3[q] ^ k1; X1[q] = l1; X3[q] = l0;
    }
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) { w[q].w[0] = X0[q]; w[q].w[1] = X1[q]; w[q].w[2] = X2[q]; w[q].w[3] = X3[q]; }
}

// ---------------------------------------------------------- vector I/O ----

template <typename T, int V>
struct alignas(sizeof(T) * V) VecT { T v[V]; };

// streaming (evict-first) global loads/stores: X and P are touched once per
// iteration and are far larger than L2 at the roofline configs
template <typename T, int V> struct StreamIO;
template <> struct StreamIO<double, 2> {
  static __device__ __forceinline__ VecT<double, 2> ld(const double* p) {
    VecT<double, 2> r;
    asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(r.v[0]), "=d"(r.v[1]) : "l"(p));
    return r;
  }
  static __device__ __forceinline__ void st(double* p, const VecT<double, 2>& r) {
    asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(r.v[0]), "d"(r.v[1]) : "memory");
  }
};
template <> struct StreamIO<double, 1> {
  static __device__ __forceinline__ VecT<double, 1> ld(const double* p) {
    VecT<double, 1> r;
    asm volatile("ld.global.cs.f64 %0, [%1];" : "=d"(r.v[0]) : "l"(p));
    return r;
  }
  static __device__ __forceinline__ void st(double* p, const VecT<double, 1>& r) {
    asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(r.v[0]) : "memory");
  }
};
template <> struct StreamIO<float, 4> {
  static __device__ __forceinline__ VecT<float, 4> ld(const float* p) {
    VecT<float, 4> r;
    asm volatile("ld.global.cs.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]) : "l"(p));
    return r;
  }
  static __device__ __forceinline__ void st(float* p, const VecT<float, 4>& r) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(r.v[0]), "f"(r.v[1]),
                 "f"(r.v[2]), "f"(r.v[3]) : "memory");
  }
};
template <> struct StreamIO<float, 1> {
  static __device__ __forceinline__ VecT<float, 1> ld(const float* p) {
    VecT<float, 1> r;
    asm volatile("ld.global.cs.f32 %0, [%1];" : "=f"(r.v[0]) : "l"(p));
    return r;
  }
  static __device__ __forceinline__ void st(float* p, const VecT<float, 1>& r) {
    asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(r.v[0]) : "memory");
  }
};

template <typename T, int V>
__device__ __forceinline__ VecT<T, V> ldg_stream(const T* p) {
  return StreamIO<T, V>::ld(p);
}
template <typename T, int V>
__device__ __forceinline__ void stg_stream(T* p, const VecT<T, V>& v) {
  StreamIO<T, V>::st(p, v);
}

// ----------------------------------------------------------- objectives ----
// Terms follow benchmarks.py:109-166 in numpy's elementwise order.

// ---------------------------------------------------------- sin / cos ----
// The objectives' sin/cos: the branch-free forms of psso_trig.cuh wherever
// they are valid (|argument| <= trig_max: every position inside a box the
// chain kernels accept), libdevice beyond.  Every kernel family -- chain,
// rows, swarm, sequential, tile, fused and psso_eval_rows -- evaluates an
// objective term with the same instructions, so re-evaluating a position on
// the device returns its in-run fitness bit for bit (the reference's
// `fn(best_position) == best_fitness`, test_core.py:168-174).
template <typename T>
__host__ __device__ constexpr double trig_max() {
  return sizeof(T) == 8 ? kChainTrigMaxAbs : kChainTrigMaxAbsF32;
}
template <typename T>
__device__ __forceinline__ T obj_cos(T y) {
  if constexpr (sizeof(T) == 8) return fabs(y) <= trig_max<T>() ? Trig<T>::cos_(y) : cos(y);
  else return fabsf(y) <= (float)trig_max<T>() ? Trig<T>::cos_(y) : cosf(y);
}
template <typename T>
__device__ __forceinline__ T obj_sin(T y) {
  if constexpr (sizeof(T) == 8) return fabs(y) <= trig_max<T>() ? Trig<T>::sin_(y) : sin(y);
  else return fabsf(y) <= (float)trig_max<T>() ? Trig<T>::sin_(y) : sinf(y);
}

template <typename T> struct Num;
template <> struct Num<double> {
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double cos_(double a) { return obj_cos(a); }
  static __device__ __forceinline__ double sin_(double a) { return obj_sin(a); }
  static __device__ __forceinline__ double exp_(double a) { return exp(a); }
  static __device__ __forceinline__ double sqrt_(double a) { return __dsqrt_rn(a); }
  static __device__ __forceinline__ double pow4(double a) { return pow(a, 4.0); }
  static constexpr double TWO_PI = 6.283185307179586;
};
template <> struct Num<float> {
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
  static __device__ __forceinline__ float cos_(float a) { return obj_cos(a); }
  static __device__ __forceinline__ float sin_(float a) { return obj_sin(a); }
  static __device__ __forceinline__ float exp_(float a) { return expf(a); }
  static __device__ __forceinline__ float sqrt_(float a) { return __fsqrt_rn(a); }
  static __device__ __forceinline__ float pow4(float a) { float s = a * a; return s * s; }
  static constexpr float TWO_PI = 6.2831855f;
};

// Rastrigin's term x*x - 10*cos(2*pi*x) (benchmarks.py:128-131) as
// x*x + (-+10)*|cos(2*pi*x)| with the exact reduction of 2x, and Ackley's
// cos(2*pi*x) (:132-140): the chain kernels' forms (no range check: their
// box is inside trig_max), and the range-checked forms of the other kernels
// (the same instructions inside trig_max, numpy's cos(fl(2*pi*x)) beyond).
template <typename T>
__device__ __forceinline__ T f5_term_in_range(T x) {
  uint32_t odd;
  const T p = Trig<T>::cos2pi_abs(x, odd);
  const T c = Trig<T>::flip((T)-10, odd);
  if constexpr (sizeof(T) == 8) return __fma_rn(p, c, __dmul_rn(x, x));
  else return __fmaf_rn(p, c, __fmul_rn(x, x));
}
template <typename T>
__device__ __forceinline__ T f5_term(T x) {
  using N = Num<T>;
  if (fabs((double)x) <= trig_max<T>()) return f5_term_in_range(x);
  const T c = sizeof(T) == 8 ? (T)cos((double)N::mul((T)N::TWO_PI, x)) : (T)cosf((float)N::mul((T)N::TWO_PI, x));
  return N::sub(N::mul(x, x), N::mul((T)10, c));
}
template <typename T>
__device__ __forceinline__ T cos2pi_term(T x) {
  using N = Num<T>;
  if (fabs((double)x) <= trig_max<T>()) return Trig<T>::cos2pi(x);
  return sizeof(T) == 8 ? (T)cos((double)N::mul((T)N::TWO_PI, x)) : (T)cosf((float)N::mul((T)N::TWO_PI, x));
}

// Objective terms, in numpy's elementwise order (benchmarks.py:109-166).
// "Heavy" terms (transcendentals) may be precomputed by all threads into a
// term buffer before the chain pass when the chains alone would leave threads
// idle; cheap terms are always formed inside the chains.
template <int FN>
__host__ __device__ constexpr bool heavy_terms() { return FN == 5 || FN == 6 || FN == 8 || FN == 9; }
__host__ __device__ constexpr bool two_sums(int FN) { return FN == 6; }

template <typename T, int FN>
__device__ __forceinline__ T heavy_term(const T* x, int e) {
  using N = Num<T>;
  if constexpr (FN == 5) {
    return f5_term(x[e]);
  } else if constexpr (FN == 6) {
    return cos2pi_term(x[e]);
  } else if constexpr (FN == 8) {
    const T a = x[4 * e], b = x[4 * e + 1], c = x[4 * e + 2], d = x[4 * e + 3];
    const T t1 = N::add(a, N::mul((T)10, b));
    const T t2 = N::sub(c, d);
    const T t3 = N::sub(b, N::mul((T)2, c));
    const T t4 = N::sub(a, d);
    return N::add(N::add(N::add(N::mul(t1, t1), N::mul((T)5, N::mul(t2, t2))), N::pow4(t3)),
                  N::mul((T)10, N::pow4(t4)));
  } else if constexpr (FN == 9) {
    const T v = x[e];
    return N::mul(v, N::sin_(N::sqrt_(fabs(v))));
  } else {
    return (T)0;
  }
}

// term #e of the row's first pairwise sum; `buf` holds precomputed terms
// (f3 always, heavy objectives when `pre`).
template <typename T, int FN>
__device__ __forceinline__ T term1(const T* x, const T* buf, int e, bool pre) {
  using N = Num<T>;
  if constexpr (FN == 1 || FN == 0 || FN == 6 || FN == 7) {
    return N::mul(x[e], x[e]);
  } else if constexpr (FN == 2) {
    return N::mul(N::mul((T)(e + 1), x[e]), x[e]);
  } else if constexpr (FN == 3) {
    return buf[e];
  } else if constexpr (FN == 4) {
    const T h = x[e];
    const T d = N::sub(x[e + 1], N::mul(h, h));
    const T o = N::sub((T)1, h);
    return N::add(N::mul(N::mul((T)100, d), d), N::mul(o, o));
  } else {  // 5, 8, 9
    return pre ? buf[e] : heavy_term<T, FN>(x, e);
  }
}

template <typename T, int FN>
__device__ __forceinline__ T term2(const T* x, const T* buf, int e, bool pre) {  // f6 only
  return pre ? buf[e] : heavy_term<T, 6>(x, e);
}

// Final per-row fitness from the pairwise sums (s2 only for f6; prod for f7).
template <typename T, int FN>
__device__ __forceinline__ double finish(T s1, T s2, T prod, int D, const T* x, double probe) {
  using N = Num<T>;
  if constexpr (FN == 5) {
    return (double)N::add(N::mul((T)10, (T)D), s1);
  } else if constexpr (FN == 6) {
    const T rms = N::sqrt_(N::div(s1, (T)D));
    const T mc = N::div(s2, (T)D);
    const T a = N::mul((T)-20, N::exp_(N::mul((T)-0.2, rms)));
    return (double)N::add(N::add(N::sub(a, N::exp_(mc)), (T)20), (T)2.718281828459045);
  } else if constexpr (FN == 7) {
    return (double)N::add(N::sub(N::div(s1, (T)4000), prod), (T)1);
  } else if constexpr (FN == 9) {
    return (double)N::sub(N::mul((T)418.9829, (T)D), s1);
  } else if constexpr (FN == 0) {
    return ((double)x[0] > probe) ? CUDART_INF : (double)s1;
  } else {
    return (double)s1;
  }
}

__device__ __forceinline__ bool lex_less(double fa, int64_t ia, double fb, int64_t ib) {
  return fa < fb || (fa == fb && ia < ib);
}

// ------------------------------------------------------------ phase B ----
// Fitness of the Rt rows held in smem (row r at x + r*SX; term buffer rows at
// buf + r*S), numpy order: each leaf of >= 8 terms is reduced by 8
// consecutive lanes (lane k owns the strided accumulator r[k] = t[k] + t[k+8]
// + ..., summed in order), the 8 accumulators combine as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) through xor shuffles (commutative, so
// bit-identical), the leader lane adds the leaf's tail sequentially, and the
// row leader combines leaves in recursion order.  `pre`: heavy terms are
// first computed by all NTH threads into `buf`.
template <typename T, int FN, int NTH>
__device__ void tile_fitness(const TileParams& p, const T* xsrc, int SX, T* buf, double* leafv,
                             double* rowf, int Rt, bool pre) {
  using N = Num<T>;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Plan& pl = p.plan;
  const int NL = pl.nleaves, S = p.S, D = p.D;

  if constexpr (FN == 3) {  // c = cumsum(x) sequentially (numpy), terms c*c
    for (int r = tid; r < Rt; r += NTH) {
      const T* x = xsrc + r * SX;
      T c = x[0];
      buf[r * S] = N::mul(c, c);
      for (int j = 1; j < D; ++j) {
        c = N::add(c, x[j]);
        buf[r * S + j] = N::mul(c, c);
      }
    }
    __syncthreads();
  }
  if constexpr (heavy_terms<FN>()) {
    if (pre) {  // all threads: heavy terms -> buf (row-major, padded stride)
      const int n = Rt * pl.n;
      for (int e = tid; e < n; e += NTH) {
        const int r = (int)p.div_n.div((uint32_t)e);
        const int j = e - r * pl.n;
        buf[r * S + j] = heavy_term<T, FN>(xsrc + r * SX, j);
      }
      __syncthreads();
    }
  }

  const int total = Rt * p.G;
  for (int base = warp * 32; base < total; base += NTH) {
    const int c = base + lane;
    const bool active = c < total;
    int row = 0, leaf = 0, k = 0, off = 0, len = 0;
    T a1 = (T)0, a2 = (T)0;
    if (active) {
      row = (int)p.div_G.div((uint32_t)c);
      const int q = c - row * p.G;
      leaf = q >> 3;
      k = q & 7;
      off = pl.leaf_off[leaf];
      len = pl.leaf_len[leaf];
      const T* x = xsrc + row * SX;
      const T* bb = buf + row * S;
      const int mlen = len >> 3;  // chain length (leaves >= 8)
      if (mlen > 0) {
        a1 = term1<T, FN>(x, bb, off + k, pre);
        if constexpr (two_sums(FN)) a2 = term2<T, FN>(x, bb, off + k, pre);
        for (int m = 1; m < mlen; ++m) {
          a1 = N::add(a1, term1<T, FN>(x, bb, off + k + 8 * m, pre));
          if constexpr (two_sums(FN)) a2 = N::add(a2, term2<T, FN>(x, bb, off + k + 8 * m, pre));
        }
      }
    }
    a1 = N::add(a1, __shfl_xor_sync(0xffffffffu, a1, 1));
    a1 = N::add(a1, __shfl_xor_sync(0xffffffffu, a1, 2));
    a1 = N::add(a1, __shfl_xor_sync(0xffffffffu, a1, 4));
    if constexpr (two_sums(FN)) {
      a2 = N::add(a2, __shfl_xor_sync(0xffffffffu, a2, 1));
      a2 = N::add(a2, __shfl_xor_sync(0xffffffffu, a2, 2));
      a2 = N::add(a2, __shfl_xor_sync(0xffffffffu, a2, 4));
    }
    if (active && k == 0) {
      const T* x = xsrc + row * SX;
      const T* bb = buf + row * S;
      T r1 = (len >= 8) ? a1 : (T)0;
      T r2 = (len >= 8) ? a2 : (T)0;
      const int tail0 = off + (len & ~7) * (len >= 8 ? 1 : 0);
      for (int e = tail0; e < off + len; ++e) {
        r1 = N::add(r1, term1<T, FN>(x, bb, e, pre));
        if constexpr (two_sums(FN)) r2 = N::add(r2, term2<T, FN>(x, bb, e, pre));
      }
      leafv[(row * NL + leaf) * 2] = (double)r1;
      leafv[(row * NL + leaf) * 2 + 1] = (double)r2;
    }
  }

  if constexpr (FN == 7) {  // factors cos(x * inv) for the sequential product
    const int n = Rt * D;
    for (int e = tid; e < n; e += NTH) {
      const int r = (int)p.div_D.div((uint32_t)e);
      const int j = e - r * D;
      buf[r * S + j] = N::cos_(N::mul(xsrc[r * SX + j], (T)p.aux[j]));
    }
  }
  __syncthreads();

  for (int r = tid; r < Rt; r += NTH) {
    T s1, s2 = (T)0, prod = (T)1;
    const double* lv = leafv + r * NL * 2;
    if (NL == 1) {
      s1 = (T)lv[0];
      s2 = (T)lv[1];
    } else {
      T st1[8], st2[8];
      int sp = 0;
      for (int o = 0; o < pl.nops; ++o) {
        const int op = pl.ops[o];
        if (op >= 0) {
          st1[sp] = (T)lv[op * 2];
          st2[sp] = (T)lv[op * 2 + 1];
          ++sp;
        } else {
          st1[sp - 2] = N::add(st1[sp - 2], st1[sp - 1]);
          st2[sp - 2] = N::add(st2[sp - 2], st2[sp - 1]);
          --sp;
        }
      }
      s1 = st1[0];
      s2 = st2[0];
    }
    if constexpr (FN == 7) {
      const T* f = buf + r * S;
      for (int j = 0; j < D; ++j) prod = N::mul(prod, f[j]);
    }
    rowf[r] = finish<T, FN>(s1, s2, prod, D, xsrc + r * SX, p.probe_level);
  }
}

// ------------------------------------------------------- phase A chunk ----
// One V-wide chunk of one row: the keyed branch draw and four-way select of
// core.py:138-173, branch-free.  Both the branch hash and the fresh hash are
// evaluated for every coordinate (a warp executes the fresh path whenever any
// lane needs it, so predication is free), and the cumulative thresholds turn
// the select chain into three monotone compares:
//   k >= Kw -> pbest, k >= Kp -> gbest, k >= Kg -> fresh   (else keep x)
// The four-way select (core.py:160-173) from one half of a Philox pair:
// branch word w[h] against the 32-bit thresholds, fresh = var_min + span * w[2+h] 2^-32.
#ifndef PSSO_PHILOX_U32CMP
#define PSSO_PHILOX_U32CMP 0
#endif
// fp32 (benchmark mode has no bitwise contract): the fresh draw in fp32,
// var_min + w * (span 2^-32) in one FMA, instead of five fp64 operations.
template <typename T>
__device__ __forceinline__ T philox_select(const TileParams& p, const Philox4& w, int h, T x, T pb,
                                           T gv) {
  const uint32_t kb = h ? w.w[1] : w.w[0];
  const uint32_t wf = h ? w.w[3] : w.w[2];
  T fresh;
  if constexpr (sizeof(T) == 4) {
    fresh = __fmaf_rn((float)wf, (float)p.span32, (float)p.var_min);
  } else {
    const double raw = __dmul_rn((double)wf, 2.3283064365386963e-10);
    fresh = __dadd_rn(p.var_min, __dmul_rn(p.span, raw));
  }
  T a = x;
  if constexpr (sizeof(T) == 4 || PSSO_PHILOX_U32CMP) {  // 32-bit compares (fp32: C3 -1 %)
    a = ((p.K32on & 1) && kb >= p.Kw32u) ? pb : a;
    a = ((p.K32on & 2) && kb >= p.Kp32u) ? gv : a;
    a = ((p.K32on & 4) && kb >= p.Kg32u) ? fresh : a;
  } else {  // fp64: the 64-bit form measured 0.8 % faster at C4 / C5
    a = kb >= p.Kw32 ? pb : a;
    a = kb >= p.Kp32 ? gv : a;
    a = kb >= p.Kg32 ? fresh : a;
  }
  return a;
}

template <typename T, int V, int RNG>
__device__ __forceinline__ VecT<T, V> search_chunk(const TileParams& p, const VecT<T, V>& x,
                                                   const VecT<T, V>& pb, const VecT<T, V>& gv,
                                                   uint64_t hr, uint64_t fr, int col, uint64_t gi,
                                                   int64_t t, uint64_t seed) {
  VecT<T, V> nv;
  if constexpr (RNG == 0) {
    uint64_t g = GAMMA * (uint64_t)(col + 1);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const uint64_t kb = mix64(hr ^ g) >> 11;
      const double fresh = __dadd_rn(p.var_min, __dmul_rn(p.span, unit53(mix64(fr ^ g))));
      T a = x.v[v];
      a = kb >= p.Kw ? pb.v[v] : a;
      a = kb >= p.Kp ? gv.v[v] : a;
      a = kb >= p.Kg ? (T)fresh : a;
      nv.v[v] = a;
      g += GAMMA;
    }
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int j = col + v;
      const Philox4 w = philox4x32_10(philox_pair(j), (uint32_t)gi, (uint32_t)(gi >> 32), (uint32_t)t,
                                      (uint32_t)seed, (uint32_t)(seed >> 32));
      nv.v[v] = philox_select<T>(p, w, philox_half(j), x.v[v], pb.v[v], gv.v[v]);
    }
  }
  return nv;
}

// Initial positions var_min + span * u(INIT, 0, i, j) (core.py:198-199).
template <typename T, int V, int RNG>
__device__ __forceinline__ VecT<T, V> init_chunk(const TileParams& p, uint64_t hr, int col,
                                                 uint64_t gi) {
  VecT<T, V> nv;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    uint64_t h;
    if constexpr (RNG == 0) {
      h = mix64(hr ^ (GAMMA * (uint64_t)(col + v + 1)));
    } else {
      const int j = col + v;
      Philox4 w = philox4x32_10(philox_pair(j), (uint32_t)gi, (uint32_t)(gi >> 32),
                                0xFFFFFFFFu, (uint32_t)p.seed, (uint32_t)(p.seed >> 32));
      const int s = philox_half(j) * 2;
      h = ((uint64_t)w.w[s] << 32) | w.w[s + 1];
    }
    nv.v[v] = (T)__dadd_rn(p.var_min, __dmul_rn(p.span, unit53(h)));
  }
  return nv;
}

// -------------------------------------------------------------- k_tile ----
// FUSED = the hot path (SEARCH|EVAL|PBEST|CAND known at compile time);
// otherwise the mode mask comes from the launch (init, phase API, evaluation).

template <typename T, int FN, int RNG, int V, bool FUSED>
__global__ void __launch_bounds__(NT, PSSO_MINB) k_tile(const __grid_constant__ TileParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* xs = reinterpret_cast<T*>(smem + p.off_xs);
  double* scr = reinterpret_cast<double*>(smem + p.off_scr);
  T* gb = reinterpret_cast<T*>(smem + p.off_gb);
  uint64_t* hbs = reinterpret_cast<uint64_t*>(smem + p.off_hb);
  uint64_t* hfs = reinterpret_cast<uint64_t*>(smem + p.off_hf);
  double* leafv = reinterpret_cast<double*>(smem + p.off_leaf);
  double* rowf = reinterpret_cast<double*>(smem + p.off_rowf);
  int* flag = reinterpret_cast<int*>(smem + p.off_flag);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  const int mode = FUSED ? (M_SEARCH | M_EVAL | M_PBEST | M_CAND | (p.mode & M_SOLF)) : p.mode;
  const int D = p.D, S = p.S, cpr = p.cpr;
  // a non-finite fitness already stopped the run (core.py:190-193 raises at
  // the first one): later iterations leave the state as it was
  if ((mode & M_SEARCH) && p.bad && *(volatile unsigned long long*)p.bad != ~0ull) return;
  const int64_t t = p.t_dev ? *p.t_dev : p.t_arg;
  T* __restrict__ X = reinterpret_cast<T*>(p.X);
  T* __restrict__ P = reinterpret_cast<T*>(p.P);

  uint64_t rootb = 0, rootf = 0;
  if constexpr (RNG == 0) {
    if (mode & M_INIT) {
      rootb = root64(p.seed, STREAM_INIT, 0);
    } else if (mode & M_SEARCH) {
      rootb = root64(p.seed, STREAM_BRANCH, (uint64_t)t);
      rootf = root64(p.seed, STREAM_FRESH, (uint64_t)t);
    }
  }
  if (mode & M_SEARCH) {  // stage the phase-entry gbest once per CTA
    const T* g = reinterpret_cast<const T*>(p.gbest);
    for (int j = tid; j < D; j += NT) gb[j] = g[j];
  }

  double best_f = CUDART_INF;
  int64_t best_i = INT64_MAX;
  const int64_t ntiles = (p.rows + p.R - 1) / p.R;

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * p.R;
    const int Rt = (int)min((int64_t)p.R, p.rows - r0);
    const int64_t gi0 = p.row_lo + r0;
    __syncthreads();  // previous tile's smem (xs, flags, hashes) fully consumed

    if constexpr (RNG == 0) {
      if (mode & (M_INIT | M_SEARCH)) {
        for (int r = tid; r < Rt; r += NT) {
          hbs[r] = fold64(rootb, (uint64_t)(gi0 + r));
          if (mode & M_SEARCH) hfs[r] = fold64(rootf, (uint64_t)(gi0 + r));
        }
      }
    }
    __syncthreads();

    // ---- phase A: positions (coalesced V-wide chunks over the whole tile)
    T* Xt = X + r0 * (int64_t)D;
    T* Pt = P + r0 * (int64_t)D;
    const int nch = Rt * cpr;
    constexpr int U = PSSO_U;  // chunks in flight per thread
    for (int c0 = tid; c0 < nch; c0 += U * NT) {
      VecT<T, V> xv[U], pv[U];
      int rows[U], cols[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + u * NT;
        const int row = (int)p.div_cpr.div((uint32_t)c);
        rows[u] = row;
        cols[u] = (c - row * cpr) * V;
        if (c < nch && (mode & (M_SEARCH | M_LOAD))) {
          xv[u] = ldg_stream<T, V>(Xt + row * D + cols[u]);
          if (mode & M_SEARCH) pv[u] = ldg_stream<T, V>(Pt + row * D + cols[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (c0 + u * NT >= nch) break;
        const int row = rows[u], col = cols[u];
        VecT<T, V> nv;
        if (mode & M_INIT) {
          nv = init_chunk<T, V, RNG>(p, RNG == 0 ? hbs[row] : 0, col, (uint64_t)(gi0 + row));
          stg_stream<T, V>(Pt + row * D + col, nv);
        } else if (mode & M_SEARCH) {
          const VecT<T, V> gv = *reinterpret_cast<const VecT<T, V>*>(gb + col);
          nv = search_chunk<T, V, RNG>(p, xv[u], pv[u], gv, RNG == 0 ? hbs[row] : 0,
                                       RNG == 0 ? hfs[row] : 0, col, (uint64_t)(gi0 + row), t, p.seed);
        } else {
          nv = xv[u];  // M_LOAD: evaluate existing positions
        }
        if (mode & (M_INIT | M_SEARCH)) stg_stream<T, V>(Xt + row * D + col, nv);
        if (mode & M_EVAL) *reinterpret_cast<VecT<T, V>*>(xs + row * S + col) = nv;
      }
    }
    if (!(mode & M_EVAL)) continue;  // warp-uniform: search-only phase
    __syncthreads();

    // ---- phase B: fitness in numpy order
    tile_fitness<T, FN, NT>(p, xs, S, reinterpret_cast<T*>(scr), leafv, rowf, Rt, p.pre != 0);
    __syncthreads();

    // ---- phase C: bookkeeping per row, pbest rows from smem
    for (int r = tid; r < Rt; r += NT) {
      const double f = rowf[r];
      const int64_t gi = gi0 + r;
      if (!isfinite(f) && p.bad)
        atomicMin(p.bad, ((unsigned long long)(t + 1) << 40) | (unsigned long long)gi);
      if (p.sol_f && ((mode & M_SOLF) || !isfinite(f))) p.sol_f[r0 + r] = f;
      double pf = f;
      int imp = 0;
      if (mode & M_INIT) {
        p.p_f[r0 + r] = f;
      } else if (mode & M_PBEST) {
        pf = p.p_f[r0 + r];
        imp = (f <= pf);  // parallel.py:109, ties refresh
        if (imp) { p.p_f[r0 + r] = f; pf = f; }
      } else if (mode & M_CAND) {
        pf = p.p_f[r0 + r];
      }
      flag[r] = imp;
      if ((mode & M_CAND) && lex_less(pf, gi, best_f, best_i)) { best_f = pf; best_i = gi; }
    }
    if (mode & M_PBEST) {  // improved rows only, warp per row, straight from smem
      __syncthreads();
      for (int r = warp; r < Rt; r += NW) {
        if (!flag[r]) continue;
        for (int ch = lane; ch < cpr; ch += 32)
          stg_stream<T, V>(Pt + r * D + ch * V, *reinterpret_cast<const VecT<T, V>*>(xs + r * S + ch * V));
      }
    }
  }

  if (mode & M_CAND) {  // deterministic CTA argmin -> one slot, no atomics
    double* red_f = reinterpret_cast<double*>(smem + p.off_red);
    int64_t* red_i = reinterpret_cast<int64_t*>(smem + p.off_red + 8 * NW);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double of = __shfl_xor_sync(0xffffffffu, best_f, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, best_i, o);
      if (lex_less(of, oi, best_f, best_i)) { best_f = of; best_i = oi; }
    }
    __syncthreads();
    if (lane == 0) { red_f[warp] = best_f; red_i[warp] = best_i; }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < NW; ++w)
        if (lex_less(red_f[w], red_i[w], best_f, best_i)) { best_f = red_f[w]; best_i = red_i[w]; }
      p.slot_f[blockIdx.x] = best_f;
      p.slot_i[blockIdx.x] = best_i;
    }
  }
}

// ------------------------------------------------ TMA bulk-copy helpers ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// --------------------------------------------------------------- k_fused ----
// The hot path: one fused PSSO iteration (SEARCH|EVAL|PBEST|CAND) as a
// persistent kernel whose X and P tiles stream through a two-stage ring in
// shared memory filled by TMA bulk copies (cp.async.bulk + mbarrier).  While
// the CTA computes tile k, tile k+1 is already in flight, so HBM reads are
// decoupled from the register file and the compute phases.  New positions are
// written in place into the X stage (the smem copy phases B/C read) and
// streamed to global X from registers; improved rows go to P from smem.
template <typename T, int FN, int RNG, int V>
__global__ void __launch_bounds__(NT, 2) k_fused(const __grid_constant__ TileParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  T* buf = reinterpret_cast<T*>(smem + p.off_scr);
  T* gb = reinterpret_cast<T*>(smem + p.off_gb);
  uint64_t* hbs = reinterpret_cast<uint64_t*>(smem + p.off_hb);
  uint64_t* hfs = reinterpret_cast<uint64_t*>(smem + p.off_hf);
  double* leafv = reinterpret_cast<double*>(smem + p.off_leaf);
  double* rowf = reinterpret_cast<double*>(smem + p.off_rowf);
  int* flag = reinterpret_cast<int*>(smem + p.off_flag);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + p.off_bar);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  const int mode = M_SEARCH | M_EVAL | M_PBEST | M_CAND | (p.mode & M_SOLF);
  const int D = p.D, cpr = p.cpr;
  if (p.bad && *(volatile unsigned long long*)p.bad != ~0ull) return;  // run already failed
  const int64_t t = p.t_dev ? *p.t_dev : p.t_arg;
  T* __restrict__ X = reinterpret_cast<T*>(p.X);
  T* __restrict__ P = reinterpret_cast<T*>(p.P);
  const int64_t ntiles = (p.rows + p.R - 1) / p.R;
  const uint32_t tile_elems = (uint32_t)p.R * (uint32_t)D;

  auto stage_x = [&](int s) { return reinterpret_cast<T*>(smem + p.off_xs + s * p.stage_bytes); };
  auto stage_p = [&](int s) {
    return reinterpret_cast<T*>(smem + p.off_xs + s * p.stage_bytes) + tile_elems;
  };
  auto issue = [&](int64_t tile, int s) {  // one thread: X and P tiles -> stage s
    if (tile >= ntiles) return;
    const int64_t r0 = tile * p.R;
    const uint32_t rt = (uint32_t)min((int64_t)p.R, p.rows - r0);
    const uint32_t bytes = rt * (uint32_t)D * (uint32_t)sizeof(T);
    mbar_expect_tx(&bar[s], 2 * bytes);
    bulk_g2s(stage_x(s), X + r0 * D, bytes, &bar[s]);
    bulk_g2s(stage_p(s), P + r0 * D, bytes, &bar[s]);
  };

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
    issue(blockIdx.x, 0);
    issue(blockIdx.x + gridDim.x, 1);
  }
  uint64_t rootb = 0, rootf = 0;
  if constexpr (RNG == 0) {
    rootb = root64(p.seed, STREAM_BRANCH, (uint64_t)t);
    rootf = root64(p.seed, STREAM_FRESH, (uint64_t)t);
  }
  {
    const T* g = reinterpret_cast<const T*>(p.gbest);
    for (int j = tid; j < D; j += NT) gb[j] = g[j];
  }
  __syncthreads();  // barriers initialized before anyone waits on them

  double best_f = CUDART_INF;
  int64_t best_i = INT64_MAX;
  int k = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
    const int s = k & 1;
    const uint32_t parity = (k >> 1) & 1;
    const int64_t r0 = tile * p.R;
    const int Rt = (int)min((int64_t)p.R, p.rows - r0);
    const int64_t gi0 = p.row_lo + r0;
    T* Xs = stage_x(s);
    const T* Ps = stage_p(s);

    double pf_row = 0.0;  // this thread's row p_f, loaded early (used in phase C)
    if (tid < Rt) pf_row = p.p_f[r0 + tid];
    if constexpr (RNG == 0) {
      for (int r = tid; r < Rt; r += NT) {
        hbs[r] = fold64(rootb, (uint64_t)(gi0 + r));
        hfs[r] = fold64(rootf, (uint64_t)(gi0 + r));
      }
    }
    mbar_wait(&bar[s], parity);
    __syncthreads();

    // ---- phase A: select in place in the X stage, stream new X to HBM
    T* Xt = X + r0 * (int64_t)D;
    const int nch = Rt * cpr;
    for (int c = tid; c < nch; c += NT) {
      const int row = (int)p.div_cpr.div((uint32_t)c);
      const int col = (c - row * cpr) * V;
      const int e = row * D + col;
      const VecT<T, V> xv = *reinterpret_cast<const VecT<T, V>*>(Xs + e);
      const VecT<T, V> pv = *reinterpret_cast<const VecT<T, V>*>(Ps + e);
      const VecT<T, V> gv = *reinterpret_cast<const VecT<T, V>*>(gb + col);
      const VecT<T, V> nv = search_chunk<T, V, RNG>(p, xv, pv, gv, RNG == 0 ? hbs[row] : 0,
                                                   RNG == 0 ? hfs[row] : 0, col,
                                                   (uint64_t)(gi0 + row), t, p.seed);
      *reinterpret_cast<VecT<T, V>*>(Xs + e) = nv;
      stg_stream<T, V>(Xt + e, nv);
    }
    __syncthreads();

    // ---- phase B: fitness in numpy order (rows contiguous in the X stage)
    tile_fitness<T, FN, NT>(p, Xs, D, buf, leafv, rowf, Rt, p.pre != 0);
    __syncthreads();

    // ---- phase C: pbest <= test, candidate, improved rows -> P
    if (tid < Rt) {
      const int r = tid;
      const double f = rowf[r];
      const int64_t gi = gi0 + r;
      if (!isfinite(f) && p.bad)
        atomicMin(p.bad, ((unsigned long long)(t + 1) << 40) | (unsigned long long)gi);
      if (p.sol_f && ((mode & M_SOLF) || !isfinite(f))) p.sol_f[r0 + r] = f;
      const int imp = (f <= pf_row);  // parallel.py:109, ties refresh
      double pf = pf_row;
      if (imp) { p.p_f[r0 + r] = f; pf = f; }
      flag[r] = imp;
      if (lex_less(pf, gi, best_f, best_i)) { best_f = pf; best_i = gi; }
    }
    __syncthreads();
    T* Pt = P + r0 * (int64_t)D;
    for (int r = warp; r < Rt; r += NW) {
      if (!flag[r]) continue;
      for (int ch = lane; ch < cpr; ch += 32)
        stg_stream<T, V>(Pt + r * D + ch * V, *reinterpret_cast<const VecT<T, V>*>(Xs + r * D + ch * V));
    }
    __syncthreads();  // stage s fully consumed -> refill it with tile k+2
    if (tid == 0) {
      fence_proxy_async();
      issue(tile + 2 * (int64_t)gridDim.x, s);
    }
  }

  double* red_f = reinterpret_cast<double*>(smem + p.off_red);
  int64_t* red_i = reinterpret_cast<int64_t*>(smem + p.off_red + 8 * NW);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double of = __shfl_xor_sync(0xffffffffu, best_f, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, best_i, o);
    if (lex_less(of, oi, best_f, best_i)) { best_f = of; best_i = oi; }
  }
  if (lane == 0) { red_f[warp] = best_f; red_i[warp] = best_i; }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < NW; ++w)
      if (lex_less(red_f[w], red_i[w], best_f, best_i)) { best_f = red_f[w]; best_i = red_i[w]; }
    p.slot_f[blockIdx.x] = best_f;
    p.slot_i[blockIdx.x] = best_i;
  }
}

// --------------------------------------------------------------- k_chain ----
// Hot path for rows whose objective is one pairwise leaf (n <= 128 terms):
// C1-C4 and every objective at D <= 128.
//
// "Chain mapping": 8 consecutive lanes own one particle; lane k holds the
// positions j = k + 8m (m < M) in registers -- exactly the elements numpy's
// accumulator r[k] sums, in the same order -- so the whole iteration is
// register-resident and barrier-free:
//   load X, P (j = k + 8m)  -> keyed draw + select -> stream new X to HBM
//   -> term(j) -> r[k] += term in order -> xor-shuffle combine (numpy's
//   ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))) -> tail terms summed in order
//   -> fitness (identical on the 8 lanes) -> pbest <= test -> improved rows
//   written to P from registers.
// A warp runs 4 particles at a time, persistent over the swarm; no
// __syncthreads in the loop.  f4's neighbour x[j+1] comes from lane k+1
// (same m) or, for k = 7, from lane 0 at m+1, with a single shuffle.  The
// objectives with sequential or grouped terms go through a per-warp smem row:
// f3 (cumsum, benchmarks.py:117-119) and f7's product (:143-148) are formed
// left to right by the segment's lane 0 exactly like numpy; f8's grouped
// terms (:151-162) are read from the row by the chain lanes.
template <int FN>
__host__ __device__ constexpr bool chain_smem_fn() { return FN == 3 || FN == 7 || FN == 8; }

template <typename T, int FN>
__device__ __forceinline__ T chain_term1(T x, T nb, int e) {
  using N = Num<T>;
  if constexpr (FN == 2) {
    return N::mul(N::mul((T)(e + 1), x), x);
  } else if constexpr (FN == 4) {
    const T d = N::sub(nb, N::mul(x, x));
    const T o = N::sub((T)1, x);
    return N::add(N::mul(N::mul((T)100, d), d), N::mul(o, o));
  } else if constexpr (FN == 5) {  // x*x - 10*cos(2*pi*x) as x*x + (-+10)*|cos|
    return f5_term_in_range(x);
  } else if constexpr (FN == 9) {
    return N::mul(x, Trig<T>::sin_(N::sqrt_(fabs(x))));
  } else {  // 0, 1, 6, 7 (the x*x sum)
    return N::mul(x, x);
  }
}

#ifndef PSSO_CHAIN_NT
#define PSSO_CHAIN_NT 256
#endif
#ifndef PSSO_CHAIN_MINB
#define PSSO_CHAIN_MINB 2
#endif
#ifndef PSSO_CHAIN_MINB_F32
#define PSSO_CHAIN_MINB_F32 PSSO_CHAIN_MINB  // resident CTAs per SM for the fp32 chain kernels
#endif
#ifndef PSSO_PHILOX_X2
#define PSSO_PHILOX_X2 1  // chain / rows kernels: two Philox calls with interleaved rounds
                          // (C3 fp32 0.342 -> 0.331 ms; same stream)
#endif
#ifndef PSSO_SWARM_PVJIT
#define PSSO_SWARM_PVJIT 1  // k_swarm / k_seq with resident rows: pbests read from shared memory at
                            // their use (C2 f4 7.5 -> 6.8 us, f6 7.5 -> 7.2, f7 10.5 -> 10.2, C1 3.1 -> 3.0
                            // per iteration)
#endif
#ifndef PSSO_CHAIN_PF
#define PSSO_CHAIN_PF 1  // FULL iteration kernel: TMA prefetch of the next group
#endif


// Shared-memory row stride of the chain / rows kernels' per-warp prefetch
// buffers.  The four 8-lane segments of a warp read the same columns of four
// rows (or leaves): with dense rows (stride a multiple of 128 B) all four hit
// the same banks -- 2x (fp64) / 4x (fp32) the minimum LDS wavefronts, 17 M /
// 136 M conflicts per C3 / C4 launch.  PSSO_ROW_PAD=1 pads each row by half a
// wavefront's width per segment (64 B fp64, 32 B fp32), which puts the
// segments on disjoint banks at the price of one bulk copy per row instead of
// one per group.  Measured (round 2, interleaved A/B): the padded
// layout is SLOWER on every workload -- C3 0.551 vs 0.536-0.544 ms, C3 fp32
// Philox 0.363 vs 0.342 ms, C4 5.29 vs 4.84 ms, C5 1.293 vs 1.276 ms -- the
// four times more, four times smaller TMA copies cost more than the extra LDS
// wavefronts, which the kernels hide.  Dense (0) is the default.
#ifndef PSSO_ROW_PAD
#define PSSO_ROW_PAD 0
#endif
template <typename T>
__host__ __device__ constexpr int row_pad() { return PSSO_ROW_PAD ? (sizeof(T) == 8 ? 64 : 32) : 0; }
template <typename T, int M>
__host__ __device__ constexpr int chain_row_stride() { return 8 * M * (int)sizeof(T) + row_pad<T>(); }
// PSSO_CHAIN_DB: double-buffered prefetch for rows of at most 512 B (see k_chain)
#ifndef PSSO_CHAIN_DB
#define PSSO_CHAIN_DB 0
#endif
template <typename T, int M>
__host__ __device__ constexpr bool chain_db() { return PSSO_CHAIN_DB && 8 * M * (int)sizeof(T) <= 512; }

// Row store of the chain step: streaming global store, or a plain store when
// the swarm is resident in shared memory (RES, k_swarm).
template <typename T, bool RES>
__device__ __forceinline__ void st_row(T* p, T v) {
  if constexpr (RES) *p = v;
  else stg_stream<T, 1>(p, VecT<T, 1>{{v}});
}

// Per-launch constants of the chain step (per swarm in the batched kernel).
struct ChainEnv {
  void* X;                // rows x D positions / pbests of this swarm (shard)
  void* P;
  double* p_f;
  double* sol_f;          // may be null
  unsigned long long* bad;
  int64_t row_lo;         // global index of local row 0
  uint64_t seed;
  uint64_t rootb, rootf;  // keyed roots of the BRANCH/FRESH (or INIT) streams at t
  int64_t t;
  int D, n, mlen, tail;   // row length, terms, full chains, tail terms
  const double* aux;      // f7: 1/sqrt(j+1), staged in shared memory by the kernel
};

// f7's 1/sqrt(j+1) table (benchmarks.py:216) in shared memory for the chain
// kernels (D <= 128): read once per launch instead of once per coordinate
// per iteration from global memory.  The whole block must call it.
template <int FN>
__device__ __forceinline__ const double* stage_aux(const double* aux, int D) {
  if constexpr (FN == 7) {
    __shared__ double aux_s[128];
    for (int j = threadIdx.x; j < D; j += blockDim.x) aux_s[j] = aux[j];
    __syncthreads();
    return aux_s;
  } else {
    return aux;
  }
}

// One group step of the chain mapping: the segment's row r (rv: r exists;
// x holds the loaded positions, pv the pbests unless INIT).  Positions, X
// store, fitness in numpy order, pbest/p_f/sol_f bookkeeping and the
// lexicographic candidate.  The whole warp must call it (shuffles).
// PVJIT: the pbests are read at their use from `pjit` (a shared-memory row,
// k_swarm's resident swarm) instead of from the pv registers.
template <typename T, int FN, int RNG, int M, bool INIT, bool FULL, bool RES = false, bool PVJIT = false>
__device__ __forceinline__ bool chain_step(const TileParams& p, const ChainEnv& ev, const T* gb,
                                           const uint64_t* xg, T* scr, int64_t r, bool rv,
                                           T (&x)[M], const T (&pv)[M], double pf_row,
                                           double& best_f, int64_t& best_i, int& best_new,
                                           const T* pjit = nullptr) {
  using N = Num<T>;
  const int lane = threadIdx.x & 31, k = lane & 7, seg = lane & ~7;
  const int D = ev.D;
  const int64_t gi = ev.row_lo + r;
  T* __restrict__ xr = reinterpret_cast<T*>(ev.X) + r * (int64_t)D;
  T* __restrict__ pr = reinterpret_cast<T*>(ev.P) + r * (int64_t)D;
  const int mode = INIT ? (M_INIT | M_EVAL | M_CAND | M_SOLF)
                        : (M_SEARCH | M_EVAL | M_PBEST | M_CAND | (p.mode & M_SOLF));

  // fitness accumulators: lane k sums terms k, k+8, ... in order (numpy's r[k])
  T a1 = (T)0, a2 = (T)0, t1 = (T)0, t2 = (T)0;
  auto add_term = [&](int m, T v1, T v2) {
    if (m < ev.mlen) {
      a1 = (m == 0) ? v1 : N::add(a1, v1);
      if constexpr (two_sums(FN)) a2 = (m == 0) ? v2 : N::add(a2, v2);
    } else if (m == ev.mlen && k < ev.tail) {
      t1 = v1;
      t2 = v2;
    }
  };
  // position-local objectives: each coordinate's terms right after its draw,
  // interleaving the integer-heavy hash with the fp64-heavy terms.  Measured:
  // a win for latency-bound rows (k_swarm, C2: 7.9 -> 7.6 us/iteration), a
  // loss for the HBM-streaming FULL kernels (C3 0.548 -> 0.561 ms), which
  // keep the two-phase schedule.
  constexpr bool FUSE = !INIT && !FULL && FN != 4 && !chain_smem_fn<FN>();

  // ---- positions
  if constexpr (INIT) {
    uint64_t hb = 0;
    if constexpr (RNG == 0) hb = fold64(ev.rootb, (uint64_t)gi);
    uint64_t g = GAMMA * (uint64_t)(k + 1);
    Philox4 w;  // RNG 1: one call per pair (m even, m + 1), see philox_pair
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int j = k + 8 * m;
      if constexpr (RNG != 0) {
        if ((m & 1) == 0)
          w = philox4x32_10(philox_pair(j), (uint32_t)gi, (uint32_t)(gi >> 32), 0xFFFFFFFFu,
                            (uint32_t)ev.seed, (uint32_t)(ev.seed >> 32));
      }
      if (rv && (FULL || j < D)) {
        uint64_t h;
        if constexpr (RNG == 0) {
          h = mix64(hb ^ g);
        } else {
          h = (m & 1) ? (((uint64_t)w.w[2] << 32) | w.w[3]) : (((uint64_t)w.w[0] << 32) | w.w[1]);
        }
        const T v = (T)__dadd_rn(p.var_min, __dmul_rn(p.span, unit53(h)));
        st_row<T, RES>(pr + j, v);
        x[m] = v;
        st_row<T, RES>(xr + j, v);
      } else {
        x[m] = (T)0;
      }
      g += GAMMA * 8ull;
    }
  } else {
    // core.py:138-173, branch-free (see search_chunk).  Reference RNG:
    // mix64(h ^ g) = mix64_tail(xs30(h) ^ xs30(g)) since the first
    // xorshift is linear over xor; xs30(g_j) comes from the CTA's table.
    uint64_t xb = 0, xf = 0;
    if constexpr (RNG == 0) {
      xb = xs30(fold64(ev.rootb, (uint64_t)gi));
      xf = xs30(fold64(ev.rootf, (uint64_t)gi));
    }
    Philox4 w4[4];  // PSSO_PHILOX_X2 == 4 only (unused otherwise)
    Philox4 w, w_next;  // RNG 1: one call per pair (m even, m + 1), see philox_pair;
                        // PSSO_PHILOX_X2: pairs (m, m+2) computed together every 4 coordinates
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int j = k + 8 * m;
      // rows shorter than 8M (C2: D = 100 in M = 16) skip the empty tail
      // columns with a warp-uniform branch instead of computing and dropping them
      if (!FULL && 8 * m >= D) break;
      T v;
      if constexpr (RNG != 0) {
        if constexpr (PSSO_PHILOX_X2 == 4 && FULL && M % 8 == 0) {
          if ((m & 7) == 0) {
            const uint32_t a[4] = {philox_pair(j), philox_pair(j + 16), philox_pair(j + 32),
                                   philox_pair(j + 48)};
            philox4x32_10_x4(a, (uint32_t)gi, (uint32_t)(gi >> 32), (uint32_t)ev.t, (uint32_t)ev.seed,
                             (uint32_t)(ev.seed >> 32), w4);
          }
          if ((m & 1) == 0) w = w4[(m & 7) >> 1];
        } else if constexpr (PSSO_PHILOX_X2 && FULL && M % 4 == 0) {
          if ((m & 3) == 0)
            philox4x32_10_x2(philox_pair(j), philox_pair(j + 16), (uint32_t)gi, (uint32_t)(gi >> 32),
                             (uint32_t)ev.t, (uint32_t)ev.seed, (uint32_t)(ev.seed >> 32), w, w_next);
          else if ((m & 3) == 2)
            w = w_next;
        } else if ((m & 1) == 0) {
          w = philox4x32_10(philox_pair(j), (uint32_t)gi, (uint32_t)(gi >> 32), (uint32_t)ev.t,
                            (uint32_t)ev.seed, (uint32_t)(ev.seed >> 32));
        }
      }
      if constexpr (RNG == 0) {
        const uint64_t gx = xg[j];
        const uint64_t kb = mix64_tail<(M <= 8 || sizeof(T) == 8)>(xb ^ gx) >> 11;
        const double fresh = __dadd_rn(p.var_min, fresh_offset<(M <= 8 || sizeof(T) == 8)>(xf ^ gx, p.span64));
        v = x[m];
        v = kb >= p.Kw ? (PVJIT ? (j < D ? pjit[j] : (T)0) : pv[m]) : v;
        v = kb >= p.Kp ? gb[j] : v;
        v = kb >= p.Kg ? (T)fresh : v;
      } else {
        v = philox_select<T>(p, w, m & 1, x[m], PVJIT ? (j < D ? pjit[j] : (T)0) : pv[m], gb[j]);
      }
      x[m] = v;
      if (rv && (FULL || j < D)) st_row<T, RES>(xr + j, v);
      if constexpr (FUSE) {
        const T v1 = chain_term1<T, FN>(v, (T)0, j);
        T v2 = (T)0;
        if constexpr (two_sums(FN)) v2 = Trig<T>::cos2pi(v);
        add_term(m, v1, v2);
      }
    }
  }

  // ---- sequential / grouped objectives: the segment's row in smem
  T* row = scr + (lane >> 3) * (8 * M);
  T prod = (T)1;
  if constexpr (FN == 7) {
    // prod(cos(x_j / sqrt(j+1))) left to right (benchmarks.py:143-148): the
    // factors to the segment's smem row, then lane 0 of the segment runs the
    // dependent multiplies over 16-byte loads issued ahead (4 loads per 8
    // factors instead of 8 shuffles in every lane: C2 f7 10.2 -> 10.0 us per
    // iteration) and shares the result
#pragma unroll
    for (int m = 0; m < M; ++m) {
      if (!FULL && 8 * m >= D) break;
      const int j = k + 8 * m;
      if (FULL || j < D) row[j] = Trig<T>::cos_(N::mul(x[m], (T)ev.aux[j]));
    }
    __syncwarp();
    if (k == 0) {
      using V4 = VecT<T, 16 / sizeof(T)>;
      constexpr int PER = 16 / (int)sizeof(T);
#pragma unroll
      for (int g = 0; g < M; ++g) {
        if (8 * g >= D) break;
        T v[8];
#pragma unroll
        for (int h = 0; h < 8 / PER; ++h) {
          const V4 q = reinterpret_cast<const V4*>(row + 8 * g)[h];
#pragma unroll
          for (int e = 0; e < PER; ++e) v[h * PER + e] = q.v[e];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (8 * g + u < D) prod = N::mul(prod, v[u]);
      }
    }
    prod = __shfl_sync(0xffffffffu, prod, seg);
  } else if constexpr (chain_smem_fn<FN>()) {
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int j = k + 8 * m;
      if (FULL || j < D) row[j] = x[m];
    }
    __syncwarp();
    if constexpr (FN == 3) {  // c = cumsum(x) left to right, terms c*c in place, in
      // lane 0 of the segment; operands loaded 8 at a time ahead of the
      // dependent adds so only the fp64 latency of the chain is exposed
      if (k == 0) {
        T c = (T)0;
#pragma unroll
        for (int g = 0; g < M; ++g) {
          if (8 * g >= D) break;
          T v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = (8 * g + u < D) ? row[8 * g + u] : (T)0;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int j = 8 * g + u;
            if (j < D) {
              c = j == 0 ? v[0] : N::add(c, v[u]);
              row[j] = N::mul(c, c);
            }
          }
        }
      }
      __syncwarp();
    }
  }

  // ---- fitness terms (INIT, f4's neighbour, the smem-row objectives)
  if constexpr (!FUSE) {
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int e = k + 8 * m;
      T nb = (T)0;
      if constexpr (FN == 4) {
        const T nxt = (m + 1 < M) ? x[m + 1 < M ? m + 1 : m] : (T)0;
        const T prov = (k == 0) ? nxt : x[m];
        nb = __shfl_sync(0xffffffffu, prov, k < 7 ? lane + 1 : lane - 7);
      }
      if (m < ev.mlen || (m == ev.mlen && k < ev.tail)) {
        T v1;
        if constexpr (FN == 3) v1 = row[e];
        else if constexpr (FN == 8) v1 = heavy_term<T, 8>(row, e);
        else v1 = chain_term1<T, FN>(x[m], nb, e);
        T v2 = (T)0;
        if constexpr (two_sums(FN)) v2 = Trig<T>::cos2pi(x[m]);
        add_term(m, v1, v2);
      }
    }
  }
  if constexpr (chain_smem_fn<FN>()) __syncwarp();  // row reads done before the next group
  a1 = N::add(a1, __shfl_xor_sync(0xffffffffu, a1, 1));
  a1 = N::add(a1, __shfl_xor_sync(0xffffffffu, a1, 2));
  a1 = N::add(a1, __shfl_xor_sync(0xffffffffu, a1, 4));
  if constexpr (two_sums(FN)) {
    a2 = N::add(a2, __shfl_xor_sync(0xffffffffu, a2, 1));
    a2 = N::add(a2, __shfl_xor_sync(0xffffffffu, a2, 2));
    a2 = N::add(a2, __shfl_xor_sync(0xffffffffu, a2, 4));
  }
  T s1 = ev.mlen > 0 ? a1 : (T)0;
  T s2 = ev.mlen > 0 ? a2 : (T)0;
  for (int q = 0; q < ev.tail; ++q) {  // numpy adds the tail left to right
    s1 = N::add(s1, __shfl_sync(0xffffffffu, t1, seg + q));
    if constexpr (two_sums(FN)) s2 = N::add(s2, __shfl_sync(0xffffffffu, t2, seg + q));
  }
  const T x0 = __shfl_sync(0xffffffffu, x[0], seg);
  const double f = finish<T, FN>(s1, s2, prod, D, &x0, p.probe_level);

  // ---- bookkeeping (identical on the 8 lanes; lane k == 0 writes)
  bool improved = false;
  if (rv) {
    if (k == 0) {
      if (!isfinite(f) && ev.bad)
        atomicMin(ev.bad, ((unsigned long long)(ev.t + 1) << 40) | (unsigned long long)gi);
      if (ev.sol_f && ((mode & M_SOLF) || !isfinite(f))) ev.sol_f[r] = f;
    }
    double pf = f;
    bool fresh_row = INIT;  // the row's pbest was (re)written now
    if (INIT) {
      if (k == 0) ev.p_f[r] = f;
    } else {
      const bool imp = f <= pf_row;  // parallel.py:109, ties refresh
      pf = imp ? f : pf_row;
      fresh_row = imp;
      improved = imp;
      if (imp) {
        if (k == 0) ev.p_f[r] = f;
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const int j = k + 8 * m;
          if (FULL || j < D) st_row<T, RES>(pr + j, x[m]);
        }
      }
    }
    if (k == 0 && lex_less(pf, gi, best_f, best_i)) {
      best_f = pf;
      best_i = gi;
      best_new = fresh_row;
    }
  }
  return improved;  // the row's pBest was rewritten (same on the segment's 8 lanes)
}

// Deterministic CTA argmin of the per-thread candidates -> slot (no atomics).
template <int NW>
__device__ __forceinline__ void cta_candidate(double best_f, int64_t best_i, double* red_f,
                                              int64_t* red_i, double* slot_f, int64_t* slot_i) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double of = __shfl_xor_sync(0xffffffffu, best_f, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, best_i, o);
    if (lex_less(of, oi, best_f, best_i)) { best_f = of; best_i = oi; }
  }
  if (lane == 0) { red_f[warp] = best_f; red_i[warp] = best_i; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < NW; ++w)
      if (lex_less(red_f[w], red_i[w], best_f, best_i)) { best_f = red_f[w]; best_i = red_i[w]; }
    *slot_f = best_f;
    *slot_i = best_i;
  }
}

// Shared memory of the chain kernels (offsets in TileParams, host: chain_layout):
//   off 0      gbest (D of T)
//   off_red    warp reduction (16 * NW bytes) + xs30(gamma*(j+1)) table (8 * 8M)
//   off_bar    per-warp mbarriers
//   off_xs     per-warp prefetch buffers (FULL iteration kernel): [X 4 rows][P 4 rows]
//   off_scr    per-warp smem rows [4][8M] (f3, f7, f8)
template <typename T, int FN, int RNG, int M, bool INIT, bool FULL>
__global__ void __launch_bounds__(PSSO_CHAIN_NT, sizeof(T) == 4 ? PSSO_CHAIN_MINB_F32 : PSSO_CHAIN_MINB)
    k_chain(const __grid_constant__ TileParams p) {
  constexpr int NTC = PSSO_CHAIN_NT;
  constexpr int NW = NTC / 32;
  extern __shared__ __align__(128) unsigned char smem[];
  T* gb = reinterpret_cast<T*>(smem);
  double* red_f = reinterpret_cast<double*>(smem + p.off_red);
  int64_t* red_i = reinterpret_cast<int64_t*>(smem + p.off_red + 8 * NW);
  uint64_t* xg = reinterpret_cast<uint64_t*>(smem + p.off_red + 16 * NW);  // [8M]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = lane & 7;
  T* scr = reinterpret_cast<T*>(smem + p.off_scr) + warp * 4 * (8 * M);
  pdl_trigger();
  pdl_wait();
  const unsigned long long t_start = gtimer();
  if (!INIT && p.bad && *(volatile unsigned long long*)p.bad != ~0ull) return;

  ChainEnv ev;
  ev.aux = stage_aux<FN>(p.aux, p.D);
  ev.X = p.X;
  ev.P = p.P;
  ev.p_f = p.p_f;
  ev.sol_f = p.sol_f;
  ev.bad = p.bad;
  ev.row_lo = p.row_lo;
  ev.seed = p.seed;
  ev.t = p.t_dev ? *p.t_dev : p.t_arg;
  ev.D = p.D;
  // FULL: D == 8*M, so the chain lengths and the tail are compile-time
  // (f4 has D-1 terms: M-1 full chains and a 7-term tail)
  ev.n = FULL ? (FN == 4 ? 8 * M - 1 : FN == 8 ? 2 * M : 8 * M) : p.plan.n;
  ev.mlen = ev.n >= 8 ? (ev.n >> 3) : 0;
  ev.tail = ev.n - 8 * ev.mlen;
  ev.rootb = ev.rootf = 0;
  if constexpr (RNG == 0) {
    if (INIT) {
      ev.rootb = root64(p.seed, STREAM_INIT, 0);
    } else {
      ev.rootb = root64(p.seed, STREAM_BRANCH, (uint64_t)ev.t);
      ev.rootf = root64(p.seed, STREAM_FRESH, (uint64_t)ev.t);
    }
  }
  if (!INIT) {
    const T* g = reinterpret_cast<const T*>(p.gbest);
    for (int j = tid; j < ev.D; j += NTC) gb[j] = g[j];
    for (int q = tid; q < 8 * M; q += NTC) xg[q] = xs30(GAMMA * (uint64_t)(q + 1));  // q = j
    __syncthreads();
  }

  const int64_t rows = p.rows;
  const int64_t ngroups = (rows + 3) >> 2;
  double best_f = CUDART_INF;
  int64_t best_i = INT64_MAX;
  int nimp = 0;

  // PF: each warp streams its next group of 4 rows (X and P) into a private
  // shared-memory buffer with TMA bulk copies while it computes the current
  // group from registers, so HBM reads overlap the hash/select/fitness work
  // without costing registers.
  constexpr bool PF = FULL && !INIT && PSSO_CHAIN_PF;
  constexpr int RS = chain_row_stride<T, M>();
  // DB: two buffers per warp (rows of <= 512 B: C4's fp64 M = 8, fp32 M = 16),
  // so the pbests are read from the buffer at their use instead of being held
  // in M registers, and the next group still streams in behind the current one
  constexpr bool DB = PF && chain_db<T, M>();
  uint64_t* wbar0 = reinterpret_cast<uint64_t*>(smem + p.off_bar) + 2 * warp;
  unsigned char* wbuf0 = smem + p.off_xs + (size_t)warp * (DB ? 2 : 1) * (8 * RS);
  uint64_t* wbar = wbar0;
  unsigned char* wbuf = wbuf0;
  const int64_t gstride = (int64_t)gridDim.x * NW;
  uint32_t wphase = 0, wphase1 = 0;
  auto prefetch = [&](int64_t g) {  // whole warp calls; one lane issues both copies
    if (g >= ngroups) return;
    if (lane == 0) {
      const int nr = (int)min((int64_t)4, rows - 4 * g);
      const uint32_t rb = (uint32_t)(8 * M * sizeof(T));
      const T* xg0 = reinterpret_cast<const T*>(p.X) + 4 * g * (int64_t)(8 * M);
      const T* pg0 = reinterpret_cast<const T*>(p.P) + 4 * g * (int64_t)(8 * M);
      mbar_expect_tx(wbar, 2 * nr * rb);
      if constexpr (row_pad<T>() == 0) {
        bulk_g2s(wbuf, xg0, nr * rb, wbar);
        bulk_g2s(wbuf + 4 * RS, pg0, nr * rb, wbar);
      } else {
        for (int q = 0; q < nr; ++q) {
          bulk_g2s(wbuf + q * RS, xg0 + q * (8 * M), rb, wbar);
          bulk_g2s(wbuf + (4 + q) * RS, pg0 + q * (8 * M), rb, wbar);
        }
      }
    }
  };
  if constexpr (PF) {
    if (lane == 0) {
      mbar_init(wbar0, 1);
      if constexpr (DB) mbar_init(wbar0 + 1, 1);
      mbar_fence_init();
    }
    __syncwarp();
    prefetch((int64_t)blockIdx.x * NW + warp);
  }

  int it = 0;
  for (int64_t grp = (int64_t)blockIdx.x * NW + warp; grp < ngroups; grp += gstride, ++it) {
    const int64_t r = 4 * grp + (lane >> 3);
    const bool rv = r < rows;
    // rows past the end (last group only) compute on a clamped row and store nothing
    const int64_t rl = rv ? r : rows - 1;
    double pf_row = 0.0;
    if (!INIT) pf_row = p.p_f[rl];

    T x[M];
    T pv[DB ? 1 : M];
    const T* ps_cur = nullptr;
    if constexpr (DB) {
      const int b = it & 1;  // this group's buffer; the other one takes the next group
      uint32_t& ph = b ? wphase1 : wphase;
      mbar_wait(wbar0 + b, ph);
      ph ^= 1;
      __syncwarp();  // the other buffer's reads (previous group) are done ...
      fence_proxy_async();
      wbar = wbar0 + (b ^ 1);
      wbuf = wbuf0 + (b ^ 1) * (8 * RS);
      prefetch(grp + gstride);  // ... before TMA refills it
      const int sr = (int)(rl - 4 * grp);
      const unsigned char* cur = wbuf0 + b * (8 * RS);
      const T* xs = reinterpret_cast<const T*>(cur + sr * RS);
      ps_cur = reinterpret_cast<const T*>(cur + 4 * RS + sr * RS);
#pragma unroll
      for (int m = 0; m < M; ++m) x[m] = xs[k + 8 * m];
    } else if constexpr (PF) {
      mbar_wait(wbar, wphase);
      wphase ^= 1;
      const int sr = (int)(rl - 4 * grp);  // clamped row within the group
      const T* xs = reinterpret_cast<const T*>(wbuf + sr * RS);
      const T* ps = reinterpret_cast<const T*>(wbuf + 4 * RS + sr * RS);
#pragma unroll
      for (int m = 0; m < M; ++m) {
        x[m] = xs[k + 8 * m];
        pv[DB ? 0 : m] = ps[k + 8 * m];
      }
      __syncwarp();  // the whole buffer is in registers before it is refilled
      fence_proxy_async();
      prefetch(grp + gstride);
    } else if constexpr (!INIT) {
      const T* xl = reinterpret_cast<const T*>(p.X) + rl * (int64_t)ev.D;
      const T* pl = reinterpret_cast<const T*>(p.P) + rl * (int64_t)ev.D;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int j = k + 8 * m;
        if (FULL || j < ev.D) {
          x[m] = ldg_stream<T, 1>(xl + j).v[0];
          pv[DB ? 0 : m] = ldg_stream<T, 1>(pl + j).v[0];
        } else {
          x[m] = (T)0;
          pv[DB ? 0 : m] = (T)0;
        }
      }
      __syncwarp();  // clamped last-row loads precede the valid segment's stores
    } else {
#pragma unroll
      for (int m = 0; m < M; ++m) pv[DB ? 0 : m] = (T)0;
    }
    int best_new = 0;
    bool imp;
    if constexpr (DB)
      imp = chain_step<T, FN, RNG, M, INIT, FULL, false, true>(p, ev, gb, xg, scr, r, rv, x, x, pf_row,
                                                               best_f, best_i, best_new, ps_cur);
    else
      imp = chain_step<T, FN, RNG, M, INIT, FULL>(p, ev, gb, xg, scr, r, rv, x,
                                                  reinterpret_cast<const T(&)[M]>(pv), pf_row,
                                                  best_f, best_i, best_new);
    nimp += (imp && k == 0) ? 1 : 0;
  }
  cta_candidate<NW>(best_f, best_i, red_f, red_i, p.slot_f + blockIdx.x, p.slot_i + blockIdx.x);
  if (!INIT) iter_stats(p.stats, ev.t, t_start, nimp);
}

// ---------------------------------------------------------------- k_rows ----
// Hot path for long rows (C5: D = 4096): D = 512*W, W in {1, 2, 4, 8}, whose
// numpy reduction is a balanced pairwise tree of 4W leaves of 128 terms
// (add.reduce splits at n/2, a multiple of 8, down to 128).  Each row is
// owned by W warps of one CTA (8/W rows per CTA round); warp slice sw holds
// leaves 4sw..4sw+3, one per 8-lane segment, with the chain mapping of
// k_chain inside the leaf (lane k: j = 128*leaf + k + 8m, m < 16), so the
// positions of the whole row stay in registers until the pBest decision:
//   TMA-prefetched X/P slice -> keyed draw + select -> X streamed to HBM ->
//   leaf chains + xor-shuffle combine -> leaf values to smem -> every warp
//   of the row combines the 4W leaves with a butterfly (xor 1, 2, ..., 2W:
//   exactly the balanced tree, fp add being commutative) -> fitness, `<=`
//   -> its slice of an improved row written to P from registers; warp 0 of
//   the row writes p_f and tracks the candidate.
// One CTA barrier per round (leaf slots double-buffered); no atomics.  Objectives with position-local
// terms (f1, f2, f5, f6, f9, probe).
template <int FN>
__host__ __device__ constexpr bool rows_fn() {
  return FN == 0 || FN == 1 || FN == 2 || FN == 5 || FN == 6 || FN == 9;
}

// PSSO_ROWS_JIT: pBest values read from the prefetch buffer just in time
// (not held in 32 registers), the next row's prefetch issued after the draw,
// gbest read through L1 instead of staged in shared memory -- 85 registers and
// ~67 KB of shared memory per CTA, so 3 CTAs per SM.
#ifndef PSSO_ROWS_JIT
#define PSSO_ROWS_JIT 0
#endif
// PSSO_ROWS_ONEFINISH: only the row's first warp combines the leaves and
// evaluates the objective; the others take its decision after a second barrier.
#ifndef PSSO_ROWS_ONEFINISH
#define PSSO_ROWS_ONEFINISH 0
#endif
template <typename T, int FN, int RNG, int W>
__global__ void __launch_bounds__(256, PSSO_ROWS_JIT ? 3 : 2) k_rows(const __grid_constant__ TileParams p) {
  using N = Num<T>;
  constexpr int NW = 8, RPC = NW / W, M = 16, D = 512 * W, NL = 4 * W;
  constexpr int RS = chain_row_stride<T, M>();
  extern __shared__ __align__(128) unsigned char smem[];
  T* gb = reinterpret_cast<T*>(smem);
  double* red_f = reinterpret_cast<double*>(smem + p.off_red);
  int64_t* red_i = reinterpret_cast<int64_t*>(smem + p.off_red + 8 * NW);
  double* leafv = reinterpret_cast<double*>(smem + p.off_leaf);  // [2][RPC][2 NL + 1]
  int* rflag = reinterpret_cast<int*>(smem + p.off_flag);          // [2][RPC] (PSSO_ROWS_ONEFINISH)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = lane & 7, s = lane >> 3;
  const int slot = warp / W, sw = warp % W;
  const int mode = M_SEARCH | M_EVAL | M_PBEST | M_CAND | (p.mode & M_SOLF);
  pdl_trigger();
  pdl_wait();
  const unsigned long long t_start = gtimer();
  if (p.bad && *(volatile unsigned long long*)p.bad != ~0ull) return;
  const int64_t t = p.t_dev ? *p.t_dev : p.t_arg;
  T* __restrict__ X = reinterpret_cast<T*>(p.X);
  T* __restrict__ P = reinterpret_cast<T*>(p.P);

  uint64_t rootb = 0, rootf = 0;
  if constexpr (RNG == 0) {
    rootb = root64(p.seed, STREAM_BRANCH, (uint64_t)t);
    rootf = root64(p.seed, STREAM_FRESH, (uint64_t)t);
  }
  if constexpr (!PSSO_ROWS_JIT) {  // gbest padded by 8 elements per leaf: the segments' reads hit disjoint banks
    const T* g = reinterpret_cast<const T*>(p.gbest);
    constexpr int U = D / 256;  // loads batched ahead of the stores (not one round trip each)
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = g[tid + 256 * u];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = tid + 256 * u;
      gb[j + ((j >> 7) << 3)] = v[u];
    }
  }
  const int jb = 512 * sw + 128 * s + k;  // this lane's first element; j = jb + 8m
  const T* gbl = PSSO_ROWS_JIT ? reinterpret_cast<const T*>(p.gbest)  // gbest of this lane's leaf: gbl[j]
                               : gb + 8 * (4 * sw + s);
  const uint64_t g0 = GAMMA * (uint64_t)(jb + 1);

  const int64_t rows = p.rows;
  const int64_t rstride = (int64_t)gridDim.x * RPC;
  uint64_t* wbar = reinterpret_cast<uint64_t*>(smem + p.off_bar) + warp;
  unsigned char* wbuf = smem + p.off_xs + (size_t)warp * (8 * RS);
  uint32_t wphase = 0;
  auto prefetch = [&](int64_t row) {  // this warp's slice of `row`; one lane issues
    if (row >= rows) return;
    if (lane == 0) {
      constexpr uint32_t SB = (uint32_t)(512 * sizeof(T));  // bytes per slice
      mbar_expect_tx(wbar, 2 * SB);
      const int64_t off = row * (int64_t)D + 512 * sw;
      if constexpr (row_pad<T>() == 0) {
        bulk_g2s(wbuf, X + off, SB, wbar);
        bulk_g2s(wbuf + 4 * RS, P + off, SB, wbar);
      } else {  // one copy per leaf, padded (see chain_row_stride)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          bulk_g2s(wbuf + q * RS, X + off + 128 * q, SB / 4, wbar);
          bulk_g2s(wbuf + (4 + q) * RS, P + off + 128 * q, SB / 4, wbar);
        }
      }
    }
  };
  if (lane == 0) {
    mbar_init(wbar, 1);
    mbar_fence_init();
  }
  __syncthreads();  // gbest staged, barriers initialised
  prefetch((int64_t)blockIdx.x * RPC + slot);

  double best_f = CUDART_INF;
  int64_t best_i = INT64_MAX;
  int round = 0;
  int nimp = 0;
  for (int64_t r0 = (int64_t)blockIdx.x * RPC; r0 < rows; r0 += rstride, ++round) {  // CTA-uniform
    const int64_t r = r0 + slot;
    const bool rv = r < rows;
    const int64_t gi = p.row_lo + r;
    const int par = round & 1;
    double* lv = leafv + (par * RPC + slot) * (2 * NL + 1);  // [s1 leaves][s2 leaves][x0]
    T x[M];
    const double pf_row = rv ? p.p_f[r] : 0.0;  // needed after barrier A
    if (rv) {
      T pv[PSSO_ROWS_JIT ? 1 : M];
      mbar_wait(wbar, wphase);
      wphase ^= 1;
      const T* xs = reinterpret_cast<const T*>(wbuf + s * RS);
      const T* ps = reinterpret_cast<const T*>(wbuf + 4 * RS + s * RS);
      if constexpr (!PSSO_ROWS_JIT) {
#pragma unroll
        for (int m = 0; m < M; ++m) {
          x[m] = xs[k + 8 * m];
          pv[PSSO_ROWS_JIT ? 0 : m] = ps[k + 8 * m];
        }
        __syncwarp();
        fence_proxy_async();
        prefetch(r + rstride);
      } else {
#pragma unroll
        for (int m = 0; m < M; ++m) x[m] = xs[k + 8 * m];
      }
      auto pbest = [&](int m) -> T { return PSSO_ROWS_JIT ? ps[k + 8 * m] : pv[PSSO_ROWS_JIT ? 0 : m]; };

      // ---- positions (core.py:138-173; see k_chain), each followed at once
      // by its objective terms and the in-order chain adds of leaf 4sw+s
      // (lane k: r[k]) -- interleaving the integer-heavy draw with the
      // fp64-heavy terms keeps both pipes busy
      T* xr = X + r * (int64_t)D;
      T a1 = (T)0, a2 = (T)0;
      auto accumulate = [&](int m, T v) {
        const T v1 = chain_term1<T, FN>(v, (T)0, jb + 8 * m);
        a1 = m == 0 ? v1 : N::add(a1, v1);
        if constexpr (two_sums(FN)) {
          const T v2 = Trig<T>::cos2pi(v);
          a2 = m == 0 ? v2 : N::add(a2, v2);
        }
      };
      if constexpr (RNG == 0) {
        const uint64_t xb = xs30(fold64(rootb, (uint64_t)gi)), xf = xs30(fold64(rootf, (uint64_t)gi));
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const int j = jb + 8 * m;
          const uint64_t gx = xs30(g0 + GAMMA * (uint64_t)(8 * m));
          const uint64_t kb = mix64_tail<(sizeof(T) == 8)>(xb ^ gx) >> 11;
          const double fresh = __dadd_rn(p.var_min, fresh_offset<(sizeof(T) == 8)>(xf ^ gx, p.span64));
          T v = x[m];
          v = kb >= p.Kw ? pbest(m) : v;
          v = kb >= p.Kp ? gbl[j] : v;
          v = kb >= p.Kg ? (T)fresh : v;
          x[m] = v;
          stg_stream<T, 1>(xr + j, VecT<T, 1>{{v}});
          accumulate(m, v);
        }
      } else {
        Philox4 w, w_next;  // one call per pair (m even, m + 1): jb is k mod 16
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const int j = jb + 8 * m;
          if constexpr (PSSO_PHILOX_X2) {  // pairs (m, m+2) together (M = 16)
            if ((m & 3) == 0)
              philox4x32_10_x2(philox_pair(j), philox_pair(j + 16), (uint32_t)gi, (uint32_t)(gi >> 32),
                               (uint32_t)t, (uint32_t)p.seed, (uint32_t)(p.seed >> 32), w, w_next);
            else if ((m & 3) == 2)
              w = w_next;
          } else if ((m & 1) == 0) {
            w = philox4x32_10(philox_pair(j), (uint32_t)gi, (uint32_t)(gi >> 32), (uint32_t)t,
                              (uint32_t)p.seed, (uint32_t)(p.seed >> 32));
          }
          x[m] = philox_select<T>(p, w, m & 1, x[m], pbest(m), gbl[j]);
          stg_stream<T, 1>(xr + j, VecT<T, 1>{{x[m]}});
          accumulate(m, x[m]);
        }
      }
      if constexpr (PSSO_ROWS_JIT) {  // this row's slice is consumed: refill with the next row's
        __syncwarp();
        fence_proxy_async();
        prefetch(r + rstride);
      }

#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        a1 = N::add(a1, __shfl_xor_sync(0xffffffffu, a1, o));
        if constexpr (two_sums(FN)) a2 = N::add(a2, __shfl_xor_sync(0xffffffffu, a2, o));
      }
      if (k == 0) {
        lv[4 * sw + s] = (double)a1;
        lv[NL + 4 * sw + s] = (double)a2;
      }
      if (sw == 0 && lane == 0) lv[2 * NL] = (double)x[0];
    }
    // (A) all leaves of the CTA's rows are in smem.  The only barrier per
    // round: leaf slots are double-buffered by round parity, and every warp of
    // a row combines the leaves itself, so nobody waits for a decision.
    __syncthreads();

    bool imp = false;
    if (rv && (!PSSO_ROWS_ONEFINISH || sw == 0)) {  // balanced tree over the 4W leaves
      const T x0 = (T)lv[2 * NL];
      T s1 = (T)0, s2 = (T)0;
      if (lane < NL) {
        s1 = (T)lv[lane];
        s2 = (T)lv[NL + lane];
      }
#pragma unroll
      for (int o = 1; o < NL; o <<= 1) {
        s1 = N::add(s1, __shfl_xor_sync(0xffffffffu, s1, o));
        if constexpr (two_sums(FN)) s2 = N::add(s2, __shfl_xor_sync(0xffffffffu, s2, o));
      }
      // lanes < 4W hold the row sums after the butterfly; lane 0 decides for all
      const double f = finish<T, FN>(s1, s2, (T)1, D, &x0, p.probe_level);
      imp = __shfl_sync(0xffffffffu, (int)(f <= pf_row), 0) != 0;  // parallel.py:109
      if (PSSO_ROWS_ONEFINISH && lane == 0) rflag[par * RPC + slot] = imp;
      if (sw == 0 && lane == 0) {
        if (!isfinite(f) && p.bad)
          atomicMin(p.bad, ((unsigned long long)(t + 1) << 40) | (unsigned long long)gi);
        if (p.sol_f && ((mode & M_SOLF) || !isfinite(f))) p.sol_f[r] = f;
        const double pf = imp ? f : pf_row;
        if (imp) p.p_f[r] = f;
        nimp += imp ? 1 : 0;
        if (lex_less(pf, gi, best_f, best_i)) { best_f = pf; best_i = gi; }
      }
    }
    if constexpr (PSSO_ROWS_ONEFINISH) {  // (B) the row's decision, from its first warp
      __syncthreads();
      imp = rv && rflag[par * RPC + slot];
    }
    if (imp) {  // this warp's slice of pbests[i] = sol[i], from registers
      T* pr = P + r * (int64_t)D;
#pragma unroll
      for (int m = 0; m < M; ++m) stg_stream<T, 1>(pr + jb + 8 * m, VecT<T, 1>{{x[m]}});
    }
  }

#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double of = __shfl_xor_sync(0xffffffffu, best_f, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, best_i, o);
    if (lex_less(of, oi, best_f, best_i)) { best_f = of; best_i = oi; }
  }
  if (lane == 0) { red_f[warp] = best_f; red_i[warp] = best_i; }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < NW; ++w)
      if (lex_less(red_f[w], red_i[w], best_f, best_i)) { best_f = red_f[w]; best_i = red_i[w]; }
    p.slot_f[blockIdx.x] = best_f;
    p.slot_i[blockIdx.x] = best_i;
  }
  iter_stats(p.stats, t, t_start, nimp);
}

}  // namespace psso
