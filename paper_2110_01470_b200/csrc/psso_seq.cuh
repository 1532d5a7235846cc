// psso_seq.cuh -- the reference's SEQUENTIAL (per-particle asynchronous)
// schedule, run_sequential (core.py:213-258), on device.
//
// The schedule is serial by definition: particle i is updated against the
// gbest left by particles 0..i-1 of the same iteration, and gbest moves the
// moment a particle's new pbest is <= g_f (core.py:236-241).  The draws do not
// depend on the state (keyed RNG, core.py:225), so the only serial coupling is
// gbest, and gbest moves rarely (a few dozen times per run, SURVEY appendix A
// / tests/golden/seq_runs.json).  k_seq therefore runs the iteration as
// SPECULATIVE PASSES with rollback:
//
//   pass from row lo: every row r >= lo is computed in parallel against the
//   current gbest (chain_step: draw + select + fitness in numpy order) into a
//   scratch row Xn[r] and fn[r] -- nothing of the swarm is written;
//   the first event r* >= lo = first row whose fitness is non-finite or is a
//   gbest move (fn <= p_f and fn <= g_f) -- a block-wide min;
//   rows lo..r* are exactly what the serial loop would produce (none of them
//   saw a gbest change), so they are committed (X, sol_f, pBest <=); the
//   gbest move of r* is applied; the next pass starts at r* + 1.
//
// An iteration costs 1 + (gbest moves in it) passes; the results are
// bit-identical to the serial loop.  One thread-block cluster of G <= 16
// CTAs per swarm (blockIdx.y = swarm of a batch): CTA c owns a contiguous
// block of rows; per pass each CTA finds its own first event, publishes it
// (row index, fitness, the row itself) in its shared memory, one hardware
// cluster barrier, and every CTA takes the lowest-index event over DSMEM --
// records double-buffered by pass parity, so one barrier per pass suffices.
// The swarm's rows stay in global memory (L2-resident at the sizes this
// schedule is used at), gbest in each CTA's shared memory.
#pragma once

#include <cooperative_groups.h>

#include "psso_device.cuh"

namespace psso {

#ifndef PSSO_SEQ_NT
#define PSSO_SEQ_NT 512
#endif

struct SeqParams {
  int64_t t0, niter;
  int64_t rows;             // rows per swarm
  void* Xn;                 // [B][rows][D] speculative rows (scratch)
  double* fn;               // [B][rows] speculative fitness (scratch)
  double* pfn;              // [B][rows] scratch for chain_step's p_f writes (unused values)
  double* traj;             // [B][traj_stride] (indexed by t) or null
  int64_t traj_stride;
  double* g_f;              // [B]
  void* gbest;              // [B][D]
  const uint64_t* seeds;    // [B]
  double* sol_f;            // [B][rows] or null
  unsigned long long* bad;  // [B]: min((t+1) << 40 | i) of the first non-finite fitness
  int64_t* passes;          // [B] passes run (diagnostic) or null
  int64_t rpc;              // rows per CTA of the cluster (multiple of 4)
  int64_t* g_idx;           // [B] gBest particle index or null
};

// Shared memory (offsets in TileParams):
//   0        gbest (8M entries of T; entries past D are read and discarded)
//   off_red  warp reduction (16 * NW) + xs30(gamma*(j+1)) table (8 * 8M)
//   off_bar  first-event reduction: NW int64 + 2
//   off_scr  per-warp smem rows [4][8M] (f3, f7, f8)
//   off_leaf published event records [2][row index, fitness] + rows [2][D]
//   off_xs   RES: this CTA's rows resident for the launch: X, P, Xn [rpc][D], p_f, fn [rpc]
template <typename T, int FN, int RNG, int M, bool RES>
__global__ void __launch_bounds__(PSSO_SEQ_NT, 1)
    k_seq(const __grid_constant__ TileParams p, const __grid_constant__ SeqParams q) {
  constexpr int NTC = PSSO_SEQ_NT;
  constexpr int NW = NTC / 32;
  extern __shared__ __align__(128) unsigned char smem[];
  T* gb = reinterpret_cast<T*>(smem);
  uint64_t* xg = reinterpret_cast<uint64_t*>(smem + p.off_red + 16 * NW);  // [8M]
  int64_t* red = reinterpret_cast<int64_t*>(smem + p.off_bar);            // [NW + 2]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = lane & 7;
  const int b = blockIdx.y, c = blockIdx.x, G = gridDim.x;
  const int D = p.D;
  const int64_t rows = q.rows;
  const int64_t r0 = (int64_t)c * q.rpc, r1 = min(rows, r0 + q.rpc);  // this CTA's rows
  T* scr = reinterpret_cast<T*>(smem + p.off_scr) + warp * 4 * (8 * M);
  int64_t* pub_i = reinterpret_cast<int64_t*>(smem + p.off_leaf);     // [2]
  double* pub_f = reinterpret_cast<double*>(smem + p.off_leaf + 16);  // [2]
  T* pub_row = reinterpret_cast<T*>(smem + p.off_leaf + 32);          // [2][D]
  namespace cgx = cooperative_groups;
  cgx::cluster_group cluster = cgx::this_cluster();

  T* Xg = reinterpret_cast<T*>(p.X) + (int64_t)b * rows * D;
  T* Pg = reinterpret_cast<T*>(p.P) + (int64_t)b * rows * D;
  double* pfg = p.p_f + (int64_t)b * rows;
  // RES: the CTA's rows live in shared memory for the whole launch (indexed
  // from base = r0); else everything stays in global memory (base = 0)
  const int64_t base = RES ? r0 : 0;
  const int64_t nres = RES ? (int64_t)q.rpc : 0;
  T* Xs = reinterpret_cast<T*>(smem + p.off_xs);
  T* X = RES ? Xs : Xg;
  T* P = RES ? Xs + nres * D : Pg;
  T* Xn = RES ? Xs + 2 * nres * D : reinterpret_cast<T*>(q.Xn) + (int64_t)b * rows * D;
  double* pf = RES ? reinterpret_cast<double*>(Xs + 3 * nres * D) : pfg;
  double* fn = RES ? pf + nres : q.fn + (int64_t)b * rows;
  double* sf = q.sol_f ? q.sol_f + (int64_t)b * rows : nullptr;
  T* gbp = reinterpret_cast<T*>(q.gbest) + (int64_t)b * D;
  unsigned long long* bad = q.bad + b;
  // a flag raised before the launch: every CTA of the cluster sees it and leaves
  if (*(volatile unsigned long long*)bad != ~0ull) return;

  // chain_step writes its row to ev.X (and, when it improves, again to ev.P),
  // its fitness to ev.sol_f and improved fitness to ev.p_f: all scratch here
  ChainEnv ev;
  ev.aux = stage_aux<FN>(p.aux, p.D);
  ev.X = Xn;
  ev.P = Xn;
  ev.p_f = q.pfn + (int64_t)b * rows + base;
  ev.sol_f = fn;
  ev.bad = nullptr;
  ev.row_lo = base;
  ev.seed = q.seeds[b];
  ev.D = D;
  ev.n = p.plan.n;
  ev.mlen = ev.n >= 8 ? (ev.n >> 3) : 0;
  ev.tail = ev.n - 8 * ev.mlen;
  ev.rootb = ev.rootf = 0;

  for (int q8 = tid; q8 < 8 * M; q8 += NTC) {
    xg[q8] = xs30(GAMMA * (uint64_t)(q8 + 1));
    gb[q8] = q8 < D ? gbp[q8] : (T)0;
  }
  if constexpr (RES) {  // this CTA's rows -> shared memory
    for (int64_t e = tid; e < (r1 - r0) * D; e += NTC) {
      X[e] = Xg[r0 * D + e];
      P[e] = Pg[r0 * D + e];
    }
    for (int64_t r = tid; r < r1 - r0; r += NTC) pf[r] = pfg[r0 + r];
  }
  double gf = q.g_f[b];
  int64_t g_idx = q.g_idx ? q.g_idx[b] : -1;
  int64_t npass = 0;
  int par = 0;
  bool stop = false;
  __syncthreads();

  for (int64_t it = 0; it < q.niter && !stop; ++it) {
    const int64_t t = q.t0 + it;
    ev.t = t;
    if constexpr (RNG == 0) {
      ev.rootb = root64(ev.seed, STREAM_BRANCH, (uint64_t)t);
      ev.rootf = root64(ev.seed, STREAM_FRESH, (uint64_t)t);
    }
    int64_t lo = 0;
    while (lo < rows) {
      ++npass;
      const int64_t a0 = max(lo, r0);  // this CTA's rows of the pass: [a0, r1)
      // ---- speculative pass (core.py:227-232 for every remaining row at once)
      double best_f = CUDART_INF;
      int64_t best_i = INT64_MAX;
      int best_new = 0;
      for (int64_t grp = (a0 >> 2) + warp; 4 * grp < r1; grp += NW) {
        const int64_t r = 4 * grp + (lane >> 3);
        const bool rv = r < r1 && r >= a0;
        const int64_t rl = r < r1 ? r : r1 - 1;
        const double pf_row = pf[rl - base];
        const T* xl = X + (rl - base) * (int64_t)D;
        const T* pl = P + (rl - base) * (int64_t)D;
        T x[M], pv[PSSO_SWARM_PVJIT && RES ? 1 : M];
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const int j = k + 8 * m;
          x[m] = j < D ? xl[j] : (T)0;
          if constexpr (!(PSSO_SWARM_PVJIT && RES)) pv[m] = j < D ? pl[j] : (T)0;
        }
        if constexpr (PSSO_SWARM_PVJIT && RES)  // pbests from the resident rows at their use
          chain_step<T, FN, RNG, M, false, false, true, true>(p, ev, gb, xg, scr, r - base, rv, x, x,
                                                              pf_row, best_f, best_i, best_new, pl);
        else
          chain_step<T, FN, RNG, M, false, false, true>(p, ev, gb, xg, scr, r - base, rv, x,
                                                        reinterpret_cast<const T(&)[M]>(pv), pf_row,
                                                        best_f, best_i, best_new);
      }
      __syncthreads();  // Xn / fn of the pass visible to the CTA
      // ---- this CTA's first event: non-finite (core.py:233) or a gbest move (core.py:236-241)
      int64_t ev_r = INT64_MAX;
      for (int64_t r = a0 + tid; r < r1; r += NTC) {
        const double f = fn[r - base];
        if (!isfinite(f) || (f <= pf[r - base] && f <= gf)) { ev_r = r; break; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ev_r = min(ev_r, __shfl_xor_sync(0xffffffffu, ev_r, o));
      if (lane == 0) red[warp] = ev_r;
      __syncthreads();
      if (warp == 0) {
        int64_t v = lane < NW ? red[lane] : INT64_MAX;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0) {
          pub_i[par] = v;
          pub_f[par] = v != INT64_MAX ? fn[v - base] : 0.0;
          red[NW] = v;
        }
      }
      __syncthreads();
      {  // publish the event row (read by every CTA after the barrier)
        const int64_t v = red[NW];
        if (v != INT64_MAX)
          for (int j = tid; j < D; j += NTC) pub_row[par * D + j] = Xn[(v - base) * (int64_t)D + j];
      }
      cluster.sync();  // every CTA's record of this pass is published
      if (warp == 0) {  // lowest-index event over the cluster (DSMEM)
        int64_t v = INT64_MAX;
        int own = 0;
        if (lane < G) {
          v = cluster.map_shared_rank(pub_i, lane)[par];
          own = lane;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const int64_t ov = __shfl_xor_sync(0xffffffffu, v, o);
          const int oo = __shfl_xor_sync(0xffffffffu, own, o);
          if (ov < v) { v = ov; own = oo; }
        }
        if (lane == 0) { red[NW] = v; red[NW + 1] = own; }
      }
      __syncthreads();
      const int64_t rs = red[NW];
      const int own = (int)red[NW + 1];
      const int64_t hi = min(rs, r1 - 1);  // last committed row of this CTA
      // ---- commit this CTA's rows a0..hi: X always (core.py:231), pBest on `<=` (:236-238)
      for (int64_t r = a0 + warp; r <= hi; r += NW) {
        const double f = fn[r - base];
        const bool imp = isfinite(f) && f <= pf[r - base];
        const T* src = Xn + (r - base) * (int64_t)D;
        for (int j = lane; j < D; j += 32) {
          const T v = src[j];
          X[(r - base) * (int64_t)D + j] = v;
          if (imp) P[(r - base) * (int64_t)D + j] = v;
        }
      }
      __syncthreads();  // pBest rows copied before p_f moves
      for (int64_t r = a0 + tid; r <= hi; r += NTC) {
        const double f = fn[r - base];
        if (sf) sf[r] = f;
        if (isfinite(f) && f <= pf[r - base]) pf[r - base] = f;
      }
      if (rs != INT64_MAX) {
        const double f = cluster.map_shared_rank(pub_f, own)[par];
        if (!isfinite(f)) {
          if (c == 0 && tid == 0) *bad = ((unsigned long long)(t + 1) << 40) | (unsigned long long)rs;
          stop = true;
        } else {  // gbest <- pbests[r*] (core.py:239-241)
          const T* src = cluster.map_shared_rank(pub_row, own) + par * D;
          for (int j = tid; j < D; j += NTC) gb[j] = src[j];
          gf = f;
          g_idx = rs;
        }
      }
      __syncthreads();
      par ^= 1;
      if (stop) break;
      lo = rs != INT64_MAX ? rs + 1 : rows;
    }
    if (!stop && c == 0 && tid == 0 && q.traj) q.traj[b * q.traj_stride + t] = gf;  // core.py:242
  }
  if constexpr (RES) {  // the CTA's rows back to global memory
    __syncthreads();
    for (int64_t e = tid; e < (r1 - r0) * D; e += NTC) {
      Xg[r0 * D + e] = X[e];
      Pg[r0 * D + e] = P[e];
    }
    for (int64_t r = tid; r < r1 - r0; r += NTC) pfg[r0 + r] = pf[r];
  }
  if (c == 0) {
    for (int j = tid; j < D; j += NTC) gbp[j] = gb[j];
    if (tid == 0) {
      q.g_f[b] = gf;
      if (q.g_idx) q.g_idx[b] = g_idx;
      if (q.passes) q.passes[b] = npass;
    }
  }
  cluster.sync();  // no CTA leaves while its shared memory may still be read
}

}  // namespace psso
