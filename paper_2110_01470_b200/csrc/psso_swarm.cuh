// psso_swarm.cuh -- the whole run of small swarms in ONE launch.
//
// Small swarms (C1: 100 x 30, C2: 1024 x 100, the paper's own Table 3.10
// scale) are latency-bound: one iteration is a few microseconds of work, so
// the per-iteration kernel pair (fused + gBest) of the streaming path costs
// more in launch gaps than in compute.  k_swarm keeps the swarm's G CTAs
// resident for all iterations of run_parallel (parallel.py:192-212):
//
//   per iteration t:  chain_step over this CTA's row groups (search +
//   evaluate + pBest, registers only) -> CTA candidate (p_f, index, "row
//   rewritten now") + the candidate's pbest row published to slot[t&1][cta]
//   -> every CTA waits for all G slots of the epoch and reduces them
//   lexicographically (deterministic, no atomics on data), applies `<=`
//   against its copy of the incumbent and stages the winner row as its smem
//   gbest (skipped when the winner is the incumbent particle with an
//   unchanged row) -> trajectory[t].
//
// The slots carry an epoch tag written with release semantics after the data;
// waiting for all G tags of the epoch IS the swarm barrier (one L2 round trip
// instead of counter + data).  Slots are double-buffered by parity: a CTA can
// only overwrite parity p after every CTA published the next epoch, i.e.
// finished reading parity p.  RES: the CTA's rows (X, P, p_f) live in shared
// memory for the whole launch and go back to HBM once at the end.
// blockIdx.y indexes independent swarms (seeds) of a batch -- the reference's
// multi-seed protocol (harness.py:217-263) as one launch.  Same keyed RNG and
// numpy-order fitness as the streaming path: results are bit-identical to it.
#pragma once

#include <cooperative_groups.h>

#include "psso_device.cuh"

namespace psso {

#ifndef PSSO_SWARM_NT
#define PSSO_SWARM_NT 512  // 16 warps: four per scheduler to hide the chain latency
#endif

struct SwarmParams {
  int64_t t0, niter;
  int64_t rows;             // rows per swarm
  int32_t G;                // CTAs per swarm (gridDim.x)
  int32_t do_init;          // run initialize() (core.py:196-210) first
  int32_t gpc;              // row groups (4 rows) per CTA, contiguous (RES) or strided
  int32_t pad;
  unsigned int* epoch;      // [B][2][G] slot epoch tags, zero at launch
  double* slot_f;           // [B][2][G]
  int64_t* slot_i;          // [B][2][G]
  int32_t* slot_new;        // [B][2][G] candidate row rewritten in that epoch
  void* slot_row;           // [B][2][G][D]
  double* traj;             // [B][traj_stride] or null
  int64_t traj_stride;
  double* g_f;              // [B]
  void* gbest;              // [B][D]
  const uint64_t* seeds;    // [B]
  double* sol_f;            // [B][rows] or null
  unsigned long long* bad;  // [B]
  unsigned long long* trace;  // PSSO_SWARM_TRACE builds: [niter][4] phase timestamps of CTA 0
  int64_t* g_idx;           // [B] gBest particle index (parallel.py:208-211) or null
};

#ifndef PSSO_SWARM_TRACE
#define PSSO_SWARM_TRACE 0
#endif
#define PSSO_TRACE(it, k)                                                            \
  do {                                                                               \
    if (PSSO_SWARM_TRACE && sp.trace && c == 0 && b == 0 && tid == 0 && (it) >= 0)   \
      sp.trace[(it) * 4 + (k)] = gtimer();                                           \
  } while (0)

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// CL (G <= 16 CTAs form one thread-block cluster): each CTA publishes its
// candidate record and row in its OWN shared memory, one hardware cluster
// barrier (barrier.cluster arrive.release / wait.acquire) replaces the
// epoch tags, and the records and the winner row are read over DSMEM.
//
// Shared memory (offsets in TileParams, host: swarm layout in psso_create):
//   0        gbest (D of T)
//   off_red  warp reduction (16 * NW) + xs30(gamma*(j+1)) table (8 * 8M)
//   off_bar  winner record (f, i, slot, new: 24 B) + per-warp "new" flags + stop
//   off_scr  per-warp smem rows [4][8M] (f3, f7, f8)
//   off_leaf CL: published records [2][f, i, new|bad] + rows [2][D]
//   off_xs   RES: X rows [4 gpc][D], P rows [4 gpc][D], p_f [4 gpc]
template <typename T, int FN, int RNG, int M, bool RES, bool CL>
__global__ void __launch_bounds__(PSSO_SWARM_NT, 1)
    k_swarm(const __grid_constant__ TileParams p, const __grid_constant__ SwarmParams sp) {
  constexpr int NTC = PSSO_SWARM_NT;
  constexpr int NW = NTC / 32;
  extern __shared__ __align__(128) unsigned char smem[];
  T* gb = reinterpret_cast<T*>(smem);
  double* red_f = reinterpret_cast<double*>(smem + p.off_red);
  int64_t* red_i = reinterpret_cast<int64_t*>(smem + p.off_red + 8 * NW);
  uint64_t* xg = reinterpret_cast<uint64_t*>(smem + p.off_red + 16 * NW);  // [8M]
  double* win_f = reinterpret_cast<double*>(smem + p.off_bar);              // winner record
  int64_t* win_i = reinterpret_cast<int64_t*>(smem + p.off_bar + 8);
  int* win_c = reinterpret_cast<int*>(smem + p.off_bar + 16);
  int* win_n = reinterpret_cast<int*>(smem + p.off_bar + 20);
  int* red_n = reinterpret_cast<int*>(smem + p.off_bar + 24);

  double* pub_f = reinterpret_cast<double*>(smem + p.off_leaf);       // CL: [2]
  int64_t* pub_i = reinterpret_cast<int64_t*>(smem + p.off_leaf + 16);
  int* pub_n = reinterpret_cast<int*>(smem + p.off_leaf + 32);
  T* pub_row = reinterpret_cast<T*>(smem + p.off_leaf + 64);          // CL: [2][D]
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = lane & 7;
  const int b = blockIdx.y, c = blockIdx.x, G = sp.G;
  const int D = p.D;
  T* scr = reinterpret_cast<T*>(smem + p.off_scr) + warp * 4 * (8 * M);

  const int64_t rows = sp.rows;
  const int64_t ngroups = (rows + 3) >> 2;
  T* Xg = reinterpret_cast<T*>(p.X) + (int64_t)b * rows * D;  // this swarm in HBM
  T* Pg = reinterpret_cast<T*>(p.P) + (int64_t)b * rows * D;
  double* pfg = p.p_f + (int64_t)b * rows;
  // rows of this CTA: RES -> the contiguous block [r0, r0 + nr) held in smem
  const int64_t r0 = RES ? (int64_t)c * sp.gpc * 4 : 0;
  const int nr = RES ? (int)max((int64_t)0, min((int64_t)sp.gpc * 4, rows - r0)) : 0;
  T* Xs = reinterpret_cast<T*>(smem + p.off_xs);
  T* Ps = Xs + (size_t)sp.gpc * 4 * D;
  double* pfs = reinterpret_cast<double*>(Ps + (size_t)sp.gpc * 4 * D);

  ChainEnv ev;
  ev.aux = stage_aux<FN>(p.aux, p.D);
  ev.X = RES ? (void*)Xs : (void*)Xg;
  ev.P = RES ? (void*)Ps : (void*)Pg;
  ev.p_f = RES ? pfs : pfg;
  ev.row_lo = r0;
  ev.sol_f = sp.sol_f ? sp.sol_f + (int64_t)b * rows + r0 : nullptr;
  ev.bad = sp.bad + b;
  ev.seed = sp.seeds[b];
  ev.D = D;
  ev.n = p.plan.n;
  ev.mlen = ev.n >= 8 ? (ev.n >> 3) : 0;
  ev.tail = ev.n - 8 * ev.mlen;
  ev.rootf = 0;
  const T* Pb = reinterpret_cast<const T*>(ev.P);
  T* gbp = reinterpret_cast<T*>(sp.gbest) + (int64_t)b * D;
  const size_t so = (size_t)b * 2 * G;  // this swarm's slots
  unsigned int* sep = sp.epoch + so;
  double* sf = sp.slot_f + so;
  int64_t* si = sp.slot_i + so;
  int32_t* sn = sp.slot_new + so;
  T* srow = reinterpret_cast<T*>(sp.slot_row) + so * D;

  for (int q = tid; q < 8 * M; q += NTC) xg[q] = xs30(GAMMA * (uint64_t)(q + 1));
  for (int j = tid; j < D; j += NTC) gb[j] = gbp[j];
  if constexpr (RES) {
    if (!sp.do_init) {  // the CTA's rows -> smem (initialize() writes them itself)
      for (int64_t e = tid; e < (int64_t)nr * D; e += NTC) {
        Xs[e] = Xg[r0 * D + e];
        Ps[e] = Pg[r0 * D + e];
      }
      for (int r = tid; r < nr; r += NTC) pfs[r] = pfg[r0 + r];
    }
  }
  double gf = sp.g_f[b];   // incumbent, identical in every thread of every CTA
  int64_t gi_inc = -1;     // incumbent particle (unknown at launch: first take copies)
  int64_t g_idx = sp.g_idx ? sp.g_idx[b] : -1;  // the reported gBest index
  __syncthreads();

  unsigned int epoch = 0;
  // CTA candidate + its pbest row -> slot[par][c] (tagged with the epoch);
  // every CTA waits for the G tags, takes the lexicographic winner (`<=`
  // against the incumbent unless initialising, parallel.py:209).  The record
  // also carries "this CTA has seen the run's non-finite flag": the OR over
  // the epoch's records is the same in every CTA, so all stop together
  // (a direct read of the flag could differ between CTAs and deadlock).
  // Returns that stop decision.  t < 0: no trajectory entry.
  int64_t trace_it = -1;
  auto exchange = [&](double best_f, int64_t best_i, int best_new, bool is_init, int64_t t) -> bool {
    ++epoch;
    const int par = (int)(epoch & 1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double of = __shfl_xor_sync(0xffffffffu, best_f, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, best_i, o);
      const int on = __shfl_xor_sync(0xffffffffu, best_new, o);
      if (lex_less(of, oi, best_f, best_i)) { best_f = of; best_i = oi; best_new = on; }
    }
    if (lane == 0) { red_f[warp] = best_f; red_i[warp] = best_i; red_n[warp] = best_new; }
    __syncthreads();
    if (warp == 0) {  // the CTA's NW warp candidates, reduced by warp 0 with shuffles
      best_f = lane < NW ? red_f[lane] : CUDART_INF;
      best_i = lane < NW ? red_i[lane] : INT64_MAX;
      best_new = lane < NW ? red_n[lane] : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double of = __shfl_xor_sync(0xffffffffu, best_f, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, best_i, o);
        const int on = __shfl_xor_sync(0xffffffffu, best_new, o);
        if (lex_less(of, oi, best_f, best_i)) { best_f = of; best_i = oi; best_new = on; }
      }
    }
    if (tid == 0) {
      const int seen_bad = *(volatile unsigned long long*)ev.bad != ~0ull;
      if constexpr (CL) {
        pub_f[par] = best_f;
        pub_i[par] = best_i;
        pub_n[par] = (best_new & 1) | (seen_bad << 1);
      } else {
        sf[par * G + c] = best_f;
        si[par * G + c] = best_i;
        sn[par * G + c] = (best_new & 1) | (seen_bad << 1);
      }
      red_i[0] = best_i;
    }
    if constexpr (CL) {
      __syncthreads();
      const int64_t bi = red_i[0];
      if (bi != INT64_MAX)
        for (int j = tid; j < D; j += NTC) pub_row[par * D + j] = Pb[(bi - r0) * D + j];
      PSSO_TRACE(trace_it, 1);
      cluster.sync();  // every CTA's record and row are published
      if (warp == 0) {
        double wf = CUDART_INF;
        int64_t wi = INT64_MAX;
        int wc = 0, wn = 0, stop = 0;
        if (lane < G) {
          const double* rf = cluster.map_shared_rank(pub_f, lane);
          const int64_t* ri = cluster.map_shared_rank(pub_i, lane);
          const int* rn = cluster.map_shared_rank(pub_n, lane);
          wf = rf[par];
          wi = ri[par];
          wn = rn[par];
          wc = lane;
          stop = wn >> 1;
          wn &= 1;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double of = __shfl_xor_sync(0xffffffffu, wf, o);
          const int64_t oi = __shfl_xor_sync(0xffffffffu, wi, o);
          const int oc = __shfl_xor_sync(0xffffffffu, wc, o);
          const int on = __shfl_xor_sync(0xffffffffu, wn, o);
          stop |= __shfl_xor_sync(0xffffffffu, stop, o);
          if (lex_less(of, oi, wf, wi)) { wf = of; wi = oi; wc = oc; wn = on; }
        }
        if (lane == 0) { *win_f = wf; *win_i = wi; *win_c = wc; *win_n = wn; red_n[NW] = stop; }
      }
      PSSO_TRACE(trace_it, 2);
      __syncthreads();
      const double wf = *win_f;
      const int64_t wi = *win_i;
      const bool take = wi != INT64_MAX && (is_init || wf <= gf);
      if (take) {
        if (wi != gi_inc || *win_n) {
          const T* src = cluster.map_shared_rank(pub_row, *win_c) + par * D;
          for (int j = tid; j < D; j += NTC) gb[j] = src[j];
        }
        gf = wf;
        gi_inc = wi;
        g_idx = wi;
      }
      if (t >= 0 && c == 0 && tid == 0 && sp.traj) sp.traj[b * sp.traj_stride + t] = gf;  // :212
      const bool stop = red_n[NW] != 0;
      __syncthreads();
      return stop;
    }
    __syncthreads();
    const int64_t bi = red_i[0];
    if (bi != INT64_MAX)
      for (int j = tid; j < D; j += NTC) srow[((int64_t)par * G + c) * D + j] = Pb[(bi - r0) * D + j];
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release_u32(sep + par * G + c, epoch);
    }
    PSSO_TRACE(trace_it, 1);
    if (warp == 0) {  // wait for the epoch's G records (the swarm barrier) and reduce
      double wf = CUDART_INF;
      int64_t wi = INT64_MAX;
      int wc = 0, wn = 0, stop = 0;
      for (int q = lane; q < G; q += 32) {
        while (ld_acquire_u32(sep + par * G + q) != epoch) __nanosleep(16);
        const double f = __ldcg(sf + par * G + q);
        const int64_t i = __ldcg(si + par * G + q);
        const int n = __ldcg(sn + par * G + q);
        stop |= n >> 1;
        if (lex_less(f, i, wf, wi)) { wf = f; wi = i; wc = q; wn = n & 1; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double of = __shfl_xor_sync(0xffffffffu, wf, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, wi, o);
        const int oc = __shfl_xor_sync(0xffffffffu, wc, o);
        const int on = __shfl_xor_sync(0xffffffffu, wn, o);
        stop |= __shfl_xor_sync(0xffffffffu, stop, o);
        if (lex_less(of, oi, wf, wi)) { wf = of; wi = oi; wc = oc; wn = on; }
      }
      if (lane == 0) { *win_f = wf; *win_i = wi; *win_c = wc; *win_n = wn; red_n[NW] = stop; }
      __threadfence();
    }
    PSSO_TRACE(trace_it, 2);
    __syncthreads();
    const double wf = *win_f;
    const int64_t wi = *win_i;
    const bool take = wi != INT64_MAX && (is_init || wf <= gf);
    if (take) {
      // the row only changes if another particle wins or the winner's pbest
      // was rewritten this epoch
      if (wi != gi_inc || *win_n) {
        const T* src = srow + ((int64_t)par * G + *win_c) * D;
        for (int j = tid; j < D; j += NTC) gb[j] = __ldcg(src + j);
      }
      gf = wf;
      gi_inc = wi;
      g_idx = wi;
    }
    if (t >= 0 && c == 0 && tid == 0 && sp.traj) sp.traj[b * sp.traj_stride + t] = gf;  // :212
    const bool stop = red_n[NW] != 0;
    __syncthreads();
    return stop;
  };

  const int64_t gbeg = RES ? (int64_t)c * sp.gpc : (int64_t)c * NW;
  const int64_t gend = RES ? min(ngroups, (int64_t)(c + 1) * sp.gpc) : ngroups;
  const int64_t gstep = RES ? NW : (int64_t)G * NW;
  const int64_t gfirst = gbeg + warp;

  // a flag raised before this launch: every CTA reads it before any CTA can
  // compute, and the start-up exchange makes the decision common
  bool stop = exchange(CUDART_INF, INT64_MAX, 0, false, -1);
  if (sp.do_init && !stop) {  // core.py:196-210: INIT draws, evaluate, argmin -> gbest
    ev.t = -1;
    if constexpr (RNG == 0) ev.rootb = root64(ev.seed, STREAM_INIT, 0);
    double best_f = CUDART_INF;
    int64_t best_i = INT64_MAX;
    int best_new = 0;
    for (int64_t grp = gfirst; grp < gend; grp += gstep) {
      const int64_t r = 4 * grp + (lane >> 3);  // swarm row
      T x[M], pv[M];
#pragma unroll
      for (int m = 0; m < M; ++m) pv[m] = (T)0;
      chain_step<T, FN, RNG, M, true, false, RES>(p, ev, gb, xg, scr, r - r0, r < rows, x, pv, 0.0,
                                                  best_f, best_i, best_new);
    }
    stop = exchange(best_f, best_i, best_new, true, -1);
  }

  // a non-finite fitness stops the run (core.py:190-193) at the end of the
  // iteration whose exchange reports it; the first (t, i) stays in the flag
  for (int64_t it = 0; it < sp.niter && !stop; ++it) {
    const int64_t t = sp.t0 + it;
    ev.t = t;
    trace_it = it;
    PSSO_TRACE(it, 0);
    if constexpr (RNG == 0) {
      ev.rootb = root64(ev.seed, STREAM_BRANCH, (uint64_t)t);
      ev.rootf = root64(ev.seed, STREAM_FRESH, (uint64_t)t);
    }
    double best_f = CUDART_INF;
    int64_t best_i = INT64_MAX;
    int best_new = 0;
    for (int64_t grp = gfirst; grp < gend; grp += gstep) {
      const int64_t r = 4 * grp + (lane >> 3);
      const bool rv = r < rows;
      const int64_t rl = (rv ? r : rows - 1) - r0;  // local row
      const double pf_row = ev.p_f[rl];
      const T* xl = reinterpret_cast<const T*>(ev.X) + rl * (int64_t)D;
      const T* pl = Pb + rl * (int64_t)D;
      // (f5 keeps its pbests in registers: 7.1 vs 7.2 us per C2 iteration)
      T x[M], pv[PSSO_SWARM_PVJIT && RES && FN != 5 ? 1 : M];
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int j = k + 8 * m;
        x[m] = j < D ? xl[j] : (T)0;
        if constexpr (!(PSSO_SWARM_PVJIT && RES && FN != 5)) pv[m] = j < D ? pl[j] : (T)0;
      }
      // a segment past the last row reads the (clamped) last row, which the
      // valid segment of the same warp rewrites below: loads before stores
      // (PVJIT: its pbest reads precede the row's pBest write-back, which
      // follows the warp-synchronous fitness shuffles)
      __syncwarp();
      if constexpr (PSSO_SWARM_PVJIT && RES && FN != 5)
        chain_step<T, FN, RNG, M, false, false, RES, true>(p, ev, gb, xg, scr, r - r0, rv, x, x, pf_row,
                                                           best_f, best_i, best_new, pl);
      else
        chain_step<T, FN, RNG, M, false, false, RES>(p, ev, gb, xg, scr, r - r0, rv, x,
                                                     reinterpret_cast<const T(&)[M]>(pv), pf_row,
                                                     best_f, best_i, best_new);
    }
    stop = exchange(best_f, best_i, best_new, false, t);
    PSSO_TRACE(it, 3);
  }

  if constexpr (RES) {  // the CTA's rows back to HBM
    for (int64_t e = tid; e < (int64_t)nr * D; e += NTC) {
      Xg[r0 * D + e] = Xs[e];
      Pg[r0 * D + e] = Ps[e];
    }
    for (int r = tid; r < nr; r += NTC) pfg[r0 + r] = pfs[r];
  }
  if (c == 0) {  // the swarm's final gbest and g_f
    for (int j = tid; j < D; j += NTC) gbp[j] = gb[j];
    if (tid == 0) {
      sp.g_f[b] = gf;
      if (sp.g_idx) sp.g_idx[b] = g_idx;
    }
  }
  if constexpr (CL) cluster.sync();  // no CTA leaves while its smem may still be read
}

}  // namespace psso
