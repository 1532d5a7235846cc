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

namespace psso {

constexpr int NT = 256;            // threads per CTA of k_tile
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
  int32_t fn_pad;
  uint64_t seed;
  uint64_t Kw, Kp, Kg;         // reference mode: branch k = h >> 11 compared < K
  uint64_t Kw32, Kp32, Kg32;   // philox mode: 32-bit word compared < K32
  double var_min, span;
  double probe_level;
  int64_t t_arg;
  const int64_t* t_dev;        // if non-null, the iteration is read from here
  double* slot_f;              // per-CTA candidates (M_CAND)
  int64_t* slot_i;
  unsigned long long* bad;     // first non-finite key ((t+1) << 40 | i)
  const double* aux;           // f7: 1/sqrt(1..D) table
  int32_t off_xs, off_scr, off_gb, off_hb, off_hf, off_leaf, off_rowf, off_flag, off_red;
  int32_t pad2;
  Plan plan;
};

// ------------------------------------------------------------------ RNG ----

__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // rng.py:48-52
  z = (z ^ (z >> 30)) * MIX1;
  z = (z ^ (z >> 27)) * MIX2;
  return z ^ (z >> 31);
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

// Philox4x32-10 (Salmon et al. 2011); counter = (pair, i_lo, i_hi, t), key = seed.
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

template <typename T> struct Num;
template <> struct Num<double> {
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double cos_(double a) { return cos(a); }
  static __device__ __forceinline__ double sin_(double a) { return sin(a); }
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
  static __device__ __forceinline__ float cos_(float a) { return cosf(a); }
  static __device__ __forceinline__ float sin_(float a) { return sinf(a); }
  static __device__ __forceinline__ float exp_(float a) { return expf(a); }
  static __device__ __forceinline__ float sqrt_(float a) { return __fsqrt_rn(a); }
  static __device__ __forceinline__ float pow4(float a) { float s = a * a; return s * s; }
  static constexpr float TWO_PI = 6.2831855f;
};

// term #e of the row's first (and, for f6, second) pairwise sum.
template <typename T, int FN>
__device__ __forceinline__ T term1(const T* x, int e) {
  using N = Num<T>;
  if constexpr (FN == 1 || FN == 0 || FN == 6 || FN == 7) {
    return N::mul(x[e], x[e]);
  } else if constexpr (FN == 2) {
    return N::mul(N::mul((T)(e + 1), x[e]), x[e]);
  } else if constexpr (FN == 3) {
    return x[e];  // f3 sums precomputed c*c terms (scratch passed as x)
  } else if constexpr (FN == 4) {
    T h = x[e];
    T d = N::sub(x[e + 1], N::mul(h, h));
    T o = N::sub((T)1, h);
    return N::add(N::mul(N::mul((T)100, d), d), N::mul(o, o));
  } else if constexpr (FN == 5) {
    T v = x[e];
    return N::sub(N::mul(v, v), N::mul((T)10, N::cos_(N::mul((T)N::TWO_PI, v))));
  } else if constexpr (FN == 8) {
    T a = x[4 * e], b = x[4 * e + 1], c = x[4 * e + 2], d = x[4 * e + 3];
    T t1 = N::add(a, N::mul((T)10, b));
    T t2 = N::sub(c, d);
    T t3 = N::sub(b, N::mul((T)2, c));
    T t4 = N::sub(a, d);
    return N::add(N::add(N::add(N::mul(t1, t1), N::mul((T)5, N::mul(t2, t2))), N::pow4(t3)),
                  N::mul((T)10, N::pow4(t4)));
  } else {  // FN == 9
    T v = x[e];
    return N::mul(v, N::sin_(N::sqrt_(fabs(v))));
  }
}

template <typename T, int FN>
__device__ __forceinline__ T term2(const T* x, int e) {  // f6 only
  using N = Num<T>;
  return N::cos_(N::mul((T)N::TWO_PI, x[e]));
}

__host__ __device__ constexpr bool two_sums(int FN) { return FN == 6; }

// Final per-row fitness from the pairwise sums (s2 only for f6; prod for f7).
template <typename T, int FN>
__device__ __forceinline__ double finish(T s1, T s2, T prod, int D, const T* x, double probe) {
  using N = Num<T>;
  if constexpr (FN == 5) {
    return (double)N::add(N::mul((T)10, (T)D), s1);
  } else if constexpr (FN == 6) {
    T rms = N::sqrt_(N::div(s1, (T)D));
    T mc = N::div(s2, (T)D);
    T a = N::mul((T)-20, N::exp_(N::mul((T)-0.2, rms)));
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
// Fitness of the Rt rows held in smem (row r at xs + r*S), numpy order:
// each leaf of >= 8 terms is reduced by 8 consecutive lanes (lane k owns the
// strided accumulator r[k] = t[k] + t[k+8] + ..., summed in order), the 8
// accumulators combine as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) through xor
// shuffles (commutative, so bit-identical), the leader lane adds the leaf's
// tail sequentially, and the row leader combines leaves in recursion order.
template <typename T, int FN>
__device__ void tile_fitness(const TileParams& p, const T* xs, double* scr, double* leafv,
                             double* rowf, int Rt) {
  using N = Num<T>;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Plan& pl = p.plan;
  const int NL = pl.nleaves, S = p.S, D = p.D;
  T* tscr = reinterpret_cast<T*>(scr);

  if constexpr (FN == 3) {  // c = cumsum(x) sequentially (numpy), terms c*c
    for (int r = tid; r < Rt; r += NT) {
      const T* x = xs + r * S;
      T c = x[0];
      tscr[r * S] = N::mul(c, c);
      for (int j = 1; j < D; ++j) {
        c = N::add(c, x[j]);
        tscr[r * S + j] = N::mul(c, c);
      }
    }
    __syncthreads();
  }
  const T* src = (FN == 3) ? tscr : xs;

  const int total = Rt * p.G;
  for (int base = warp * 32; base < total; base += NT) {
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
      const T* x = src + row * S;
      const int mlen = len >> 3;  // chain length (leaves >= 8)
      if (mlen > 0) {
        a1 = term1<T, FN>(x, off + k);
        if constexpr (two_sums(FN)) a2 = term2<T, FN>(x, off + k);
        for (int m = 1; m < mlen; ++m) {
          a1 = N::add(a1, term1<T, FN>(x, off + k + 8 * m));
          if constexpr (two_sums(FN)) a2 = N::add(a2, term2<T, FN>(x, off + k + 8 * m));
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
      const T* x = src + row * S;
      T r1 = (len >= 8) ? a1 : (T)0;
      T r2 = (len >= 8) ? a2 : (T)0;
      const int tail0 = off + (len & ~7) * (len >= 8 ? 1 : 0);
      for (int e = tail0; e < off + len; ++e) {
        r1 = N::add(r1, term1<T, FN>(x, e));
        if constexpr (two_sums(FN)) r2 = N::add(r2, term2<T, FN>(x, e));
      }
      leafv[(row * NL + leaf) * 2] = (double)r1;
      leafv[(row * NL + leaf) * 2 + 1] = (double)r2;
    }
  }

  if constexpr (FN == 7) {  // factors cos(x * inv) for the sequential product
    const int n = Rt * D;
    for (int e = tid; e < n; e += NT) {
      const int r = (int)p.div_D.div((uint32_t)e);
      const int j = e - r * D;
      tscr[r * S + j] = N::cos_(N::mul(xs[r * S + j], (T)p.aux[j]));
    }
  }
  __syncthreads();

  for (int r = tid; r < Rt; r += NT) {
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
      const T* f = tscr + r * S;
      for (int j = 0; j < D; ++j) prod = N::mul(prod, f[j]);
    }
    rowf[r] = finish<T, FN>(s1, s2, prod, D, xs + r * S, p.probe_level);
  }
}

// -------------------------------------------------------------- k_tile ----

template <typename T, int FN, int RNG, int V>
__global__ void __launch_bounds__(NT) k_tile(const __grid_constant__ TileParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* xs = reinterpret_cast<T*>(smem + p.off_xs);
  double* scr = reinterpret_cast<double*>(smem + p.off_scr);
  T* gb = reinterpret_cast<T*>(smem + p.off_gb);
  uint64_t* hbs = reinterpret_cast<uint64_t*>(smem + p.off_hb);
  uint64_t* hfs = reinterpret_cast<uint64_t*>(smem + p.off_hf);
  double* leafv = reinterpret_cast<double*>(smem + p.off_leaf);
  double* rowf = reinterpret_cast<double*>(smem + p.off_rowf);
  int* flag = reinterpret_cast<int*>(smem + p.off_flag);

  const int tid = threadIdx.x;
  const int mode = p.mode;
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
    constexpr int U = 4;
    for (int c0 = tid; c0 < nch; c0 += U * NT) {
      VecT<T, V> xv[U], pv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + u * NT;
        if (c < nch && (mode & (M_SEARCH | M_LOAD))) {
          const int row = (int)p.div_cpr.div((uint32_t)c);
          const int col = (c - row * cpr) * V;
          xv[u] = ldg_stream<T, V>(Xt + row * D + col);
          if (mode & M_SEARCH) pv[u] = ldg_stream<T, V>(Pt + row * D + col);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + u * NT;
        if (c >= nch) break;
        const int row = (int)p.div_cpr.div((uint32_t)c);
        const int col = (c - row * cpr) * V;
        VecT<T, V> nv;
        if (mode & M_INIT) {
          if constexpr (RNG == 0) {
            const uint64_t hr = hbs[row];
#pragma unroll
            for (int v = 0; v < V; ++v) {
              const uint64_t h = mix64(hr ^ (GAMMA * (uint64_t)(col + v + 1)));
              nv.v[v] = (T)__dadd_rn(p.var_min, __dmul_rn(p.span, unit53(h)));
            }
          } else {
            const uint64_t gi = (uint64_t)(gi0 + row);
#pragma unroll
            for (int v = 0; v < V; ++v) {
              const int j = col + v;
              Philox4 w = philox4x32_10((uint32_t)(j >> 1), (uint32_t)gi, (uint32_t)(gi >> 32),
                                        0xFFFFFFFFu, (uint32_t)p.seed, (uint32_t)(p.seed >> 32));
              const int s = (j & 1) * 2;
              const uint64_t h = ((uint64_t)w.w[s] << 32) | w.w[s + 1];
              nv.v[v] = (T)__dadd_rn(p.var_min, __dmul_rn(p.span, unit53(h)));
            }
          }
          *reinterpret_cast<VecT<T, V>*>(Pt + row * D + col) = nv;
        } else if (mode & M_SEARCH) {
          const VecT<T, V> gv = *reinterpret_cast<const VecT<T, V>*>(gb + col);
          if constexpr (RNG == 0) {
            const uint64_t hr = hbs[row], fr = hfs[row];
#pragma unroll
            for (int v = 0; v < V; ++v) {
              const uint64_t g = GAMMA * (uint64_t)(col + v + 1);
              const uint64_t kb = mix64(hr ^ g) >> 11;
              T val;
              if (kb < p.Kw) val = xv[u].v[v];
              else if (kb < p.Kp) val = pv[u].v[v];
              else if (kb < p.Kg) val = gv.v[v];
              else val = (T)__dadd_rn(p.var_min, __dmul_rn(p.span, unit53(mix64(fr ^ g))));
              nv.v[v] = val;
            }
          } else {
            const uint64_t gi = (uint64_t)(gi0 + row);
            Philox4 w;
#pragma unroll
            for (int v = 0; v < V; ++v) {
              const int j = col + v;
              if (v == 0 || (j & 1) == 0)
                w = philox4x32_10((uint32_t)(j >> 1), (uint32_t)gi, (uint32_t)(gi >> 32),
                                  (uint32_t)t, (uint32_t)p.seed, (uint32_t)(p.seed >> 32));
              const uint64_t kb = w.w[j & 1];
              T val;
              if (kb < p.Kw32) val = xv[u].v[v];
              else if (kb < p.Kp32) val = pv[u].v[v];
              else if (kb < p.Kg32) val = gv.v[v];
              else {
                const double raw = __dmul_rn((double)w.w[2 + (j & 1)], 2.3283064365386963e-10);
                val = (T)__dadd_rn(p.var_min, __dmul_rn(p.span, raw));
              }
              nv.v[v] = val;
            }
          }
        } else {
          nv = xv[u];  // M_LOAD: evaluate existing positions
        }
        if (mode & (M_INIT | M_SEARCH))
          stg_stream<T, V>(Xt + row * D + col, nv);
        if (mode & M_EVAL) *reinterpret_cast<VecT<T, V>*>(xs + row * S + col) = nv;
      }
    }
    if (!(mode & M_EVAL)) continue;  // warp-uniform: search-only phase
    __syncthreads();

    // ---- phase B: fitness in numpy order
    tile_fitness<T, FN>(p, xs, scr, leafv, rowf, Rt);
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
    if (mode & M_PBEST) {
      __syncthreads();
      for (int c = tid; c < nch; c += NT) {
        const int row = (int)p.div_cpr.div((uint32_t)c);
        if (!flag[row]) continue;
        const int col = (c - row * cpr) * V;
        stg_stream<T, V>(Pt + row * D + col, *reinterpret_cast<const VecT<T, V>*>(xs + row * S + col));
      }
    }
  }

  if (mode & M_CAND) {  // deterministic CTA argmin -> one slot, no atomics
    double* red_f = reinterpret_cast<double*>(smem + p.off_red);
    int64_t* red_i = reinterpret_cast<int64_t*>(smem + p.off_red + 8 * (NT / 32));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double of = __shfl_xor_sync(0xffffffffu, best_f, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, best_i, o);
      if (lex_less(of, oi, best_f, best_i)) { best_f = of; best_i = oi; }
    }
    __syncthreads();
    if ((tid & 31) == 0) { red_f[tid >> 5] = best_f; red_i[tid >> 5] = best_i; }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < NT / 32; ++w)
        if (lex_less(red_f[w], red_i[w], best_f, best_i)) { best_f = red_f[w]; best_i = red_i[w]; }
      p.slot_f[blockIdx.x] = best_f;
      p.slot_i[blockIdx.x] = best_i;
    }
  }
}

}  // namespace psso
