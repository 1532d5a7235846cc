// psso_swarm.cuh -- the whole run of small swarms in ONE launch.
//
// Small swarms (C1: 100 x 30, C2: 1024 x 100, the paper's own Table 3.10
// scale) are latency-bound: one iteration is a few microseconds of work, so
// the per-iteration kernel pair (fused + gBest) of the streaming path costs
// more in launch gaps than in compute.  k_swarm keeps the swarm's CTAs
// resident for all iterations of run_parallel (parallel.py:192-212):
//
//   per iteration t:  chain_step over this CTA's row groups (search +
//   evaluate + pBest, registers only) -> CTA candidate (p_f, index) + the
//   candidate's pbest row published to slot[t&1][cta] -> swarm barrier ->
//   every CTA reduces the G slots lexicographically (deterministic, no
//   atomics on data), applies `<=` against its copy of the incumbent and
//   stages the winner row as its smem gbest -> trajectory[t].
//
// Slots are double-buffered by iteration parity, so one barrier per
// iteration suffices: a CTA can only overwrite parity p after every CTA has
// passed the next barrier, i.e. finished reading parity p.  The barrier is an
// arrival counter per swarm (release/acquire at gpu scope); G = 1 swarms use
// __syncthreads only.  blockIdx.y indexes independent swarms (seeds) of a
// batch -- the reference's multi-seed protocol (harness.py:217-263) as one
// launch.  The same keyed RNG and numpy-order fitness as the streaming path,
// so results are bit-identical to it.
#pragma once

#include "psso_device.cuh"

namespace psso {

struct SwarmParams {
  int64_t t0, niter;
  int64_t rows;             // rows per swarm
  int32_t G;                // CTAs per swarm (gridDim.x)
  int32_t do_init;          // run initialize() (core.py:196-210) first
  unsigned int* bar;        // [B] arrival counters, zero at launch
  double* slot_f;           // [B][2][G]
  int64_t* slot_i;          // [B][2][G]
  void* slot_row;           // [B][2][G][D]
  double* traj;             // [B][traj_stride] or null
  int64_t traj_stride;
  double* g_f;              // [B]
  void* gbest;              // [B][D]
  const uint64_t* seeds;    // [B]
  double* sol_f;            // [B][rows] or null
  unsigned long long* bad;  // [B]
};

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// All G CTAs of a swarm: everything written before is visible after.
__device__ __forceinline__ void swarm_barrier(unsigned int* ctr, int G, unsigned int& epoch) {
  ++epoch;
  __syncthreads();
  if (G > 1 && threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    const unsigned int target = (unsigned int)G * epoch;
    while (ld_acquire_u32(ctr) < target) __nanosleep(20);
    __threadfence();
  }
  __syncthreads();
}

template <typename T, int FN, int RNG, int M>
__global__ void __launch_bounds__(PSSO_CHAIN_NT, 1)
    k_swarm(const __grid_constant__ TileParams p, const __grid_constant__ SwarmParams sp) {
  constexpr int NTC = PSSO_CHAIN_NT;
  constexpr int NW = NTC / 32;
  extern __shared__ __align__(128) unsigned char smem[];
  T* gb = reinterpret_cast<T*>(smem);
  double* red_f = reinterpret_cast<double*>(smem + p.off_red);
  int64_t* red_i = reinterpret_cast<int64_t*>(smem + p.off_red + 8 * NW);
  uint64_t* xg = reinterpret_cast<uint64_t*>(smem + p.off_red + 16 * NW);  // [8M]
  double* win_f = reinterpret_cast<double*>(smem + p.off_bar);              // winner (f, i, slot)
  int64_t* win_i = reinterpret_cast<int64_t*>(smem + p.off_bar + 8);
  int* win_c = reinterpret_cast<int*>(smem + p.off_bar + 16);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = lane & 7;
  const int b = blockIdx.y, c = blockIdx.x, G = sp.G;
  const int D = p.D;
  T* scr = reinterpret_cast<T*>(smem + p.off_scr) + warp * 4 * (8 * M);

  ChainEnv ev;
  ev.X = reinterpret_cast<T*>(p.X) + (int64_t)b * sp.rows * D;
  ev.P = reinterpret_cast<T*>(p.P) + (int64_t)b * sp.rows * D;
  ev.p_f = p.p_f + (int64_t)b * sp.rows;
  ev.sol_f = sp.sol_f ? sp.sol_f + (int64_t)b * sp.rows : nullptr;
  ev.bad = sp.bad + b;
  ev.row_lo = 0;
  ev.seed = sp.seeds[b];
  ev.D = D;
  ev.n = p.plan.n;
  ev.mlen = ev.n >= 8 ? (ev.n >> 3) : 0;
  ev.tail = ev.n - 8 * ev.mlen;
  ev.rootf = 0;
  const T* Pb = reinterpret_cast<const T*>(ev.P);
  T* gbp = reinterpret_cast<T*>(sp.gbest) + (int64_t)b * D;
  double* sf = sp.slot_f + (int64_t)b * 2 * G;
  int64_t* si = sp.slot_i + (int64_t)b * 2 * G;
  T* srow = reinterpret_cast<T*>(sp.slot_row) + (int64_t)b * 2 * G * D;
  unsigned int* bar = sp.bar + b;

  for (int q = tid; q < 8 * M; q += NTC) xg[q] = xs30(GAMMA * (uint64_t)(q + 1));
  for (int j = tid; j < D; j += NTC) gb[j] = gbp[j];
  double gf = sp.g_f[b];  // incumbent, identical in every thread of every CTA
  __syncthreads();

  const int64_t rows = sp.rows;
  const int64_t ngroups = (rows + 3) >> 2;
  unsigned int epoch = 0;

  // CTA candidate + its pbest row -> slot[par][c]; barrier; every CTA takes the
  // lexicographic winner (`<=` against the incumbent unless initialising).
  auto exchange = [&](double best_f, int64_t best_i, bool is_init, int64_t t) {
    const int par = (int)(epoch & 1);
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
      sf[par * G + c] = best_f;
      si[par * G + c] = best_i;
      red_i[0] = best_i;
    }
    __syncthreads();
    const int64_t bi = red_i[0];
    if (bi != INT64_MAX)
      for (int j = tid; j < D; j += NTC) srow[((int64_t)par * G + c) * D + j] = Pb[bi * D + j];
    swarm_barrier(bar, G, epoch);
    if (warp == 0) {
      double wf = CUDART_INF;
      int64_t wi = INT64_MAX;
      int wc = 0;
      for (int q = lane; q < G; q += 32) {
        const double f = __ldcg(sf + par * G + q);
        const int64_t i = __ldcg(si + par * G + q);
        if (lex_less(f, i, wf, wi)) { wf = f; wi = i; wc = q; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double of = __shfl_xor_sync(0xffffffffu, wf, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, wi, o);
        const int oc = __shfl_xor_sync(0xffffffffu, wc, o);
        if (lex_less(of, oi, wf, wi)) { wf = of; wi = oi; wc = oc; }
      }
      if (lane == 0) { *win_f = wf; *win_i = wi; *win_c = wc; }
    }
    __syncthreads();
    const double wf = *win_f;
    const bool take = *win_i != INT64_MAX && (is_init || wf <= gf);  // parallel.py:209
    if (take) {
      const T* src = srow + ((int64_t)par * G + *win_c) * D;
      for (int j = tid; j < D; j += NTC) gb[j] = __ldcg(src + j);
      gf = wf;
    }
    if (!is_init && c == 0 && tid == 0 && sp.traj) sp.traj[b * sp.traj_stride + t] = gf;  // :212
    __syncthreads();
  };

  if (sp.do_init) {  // core.py:196-210: INIT draws, evaluate, argmin -> gbest
    ev.t = -1;
    if constexpr (RNG == 0) ev.rootb = root64(ev.seed, STREAM_INIT, 0);
    double best_f = CUDART_INF;
    int64_t best_i = INT64_MAX;
    for (int64_t grp = (int64_t)c * NW + warp; grp < ngroups; grp += (int64_t)G * NW) {
      const int64_t r = 4 * grp + (lane >> 3);
      T x[M], pv[M];
#pragma unroll
      for (int m = 0; m < M; ++m) pv[m] = (T)0;
      chain_step<T, FN, RNG, M, true, false>(p, ev, gb, xg, scr, r, r < rows, x, pv, 0.0, best_f, best_i);
    }
    exchange(best_f, best_i, true, -1);
  }

  for (int64_t it = 0; it < sp.niter; ++it) {
    // a non-finite fitness stops the run (core.py:190-193); every CTA reads the
    // flag after the same barrier, so all leave at the same iteration
    if (*(volatile unsigned long long*)ev.bad != ~0ull) break;
    const int64_t t = sp.t0 + it;
    ev.t = t;
    if constexpr (RNG == 0) {
      ev.rootb = root64(ev.seed, STREAM_BRANCH, (uint64_t)t);
      ev.rootf = root64(ev.seed, STREAM_FRESH, (uint64_t)t);
    }
    double best_f = CUDART_INF;
    int64_t best_i = INT64_MAX;
    for (int64_t grp = (int64_t)c * NW + warp; grp < ngroups; grp += (int64_t)G * NW) {
      const int64_t r = 4 * grp + (lane >> 3);
      const bool rv = r < rows;
      const int64_t rl = rv ? r : rows - 1;
      const double pf_row = ev.p_f[rl];
      const T* xl = reinterpret_cast<const T*>(ev.X) + rl * (int64_t)D;
      const T* pl = Pb + rl * (int64_t)D;
      T x[M], pv[M];
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int j = k + 8 * m;
        x[m] = j < D ? xl[j] : (T)0;
        pv[m] = j < D ? pl[j] : (T)0;
      }
      chain_step<T, FN, RNG, M, false, false>(p, ev, gb, xg, scr, r, rv, x, pv, pf_row, best_f,
                                               best_i);
    }
    exchange(best_f, best_i, false, t);
  }

  if (c == 0) {  // the swarm's final gbest and g_f
    for (int j = tid; j < D; j += NTC) gbp[j] = gb[j];
    if (tid == 0) sp.g_f[b] = gf;
  }
}

}  // namespace psso
