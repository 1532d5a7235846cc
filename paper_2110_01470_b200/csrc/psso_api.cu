// psso_api.cu -- C ABI (include/psso.h) of the PSSO hot path, plus the small
// kernels around the fused tile kernel: gBest stage 2, the sharded candidate
// records, the unfused phase kernels, the keyed RNG and launch bookkeeping.
//
// Reference anchors (/root/reference/pkg/src/sso/): run_parallel
// parallel.py:152-233; phases parallel.py:120-144; initialize core.py:196-210;
// RngStream.uniform rng.py:73-87; BenchmarkFn.__call__ benchmarks.py:86-94.
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>

#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "psso.h"
#include "psso_device.cuh"
#include "psso_registry.h"
#include "psso_seq.cuh"
#include "psso_swarm.cuh"

using namespace psso;

namespace {

thread_local std::string g_err;
struct BatchFailure { int64_t swarm = -1, t = 0, i = -1; double value = 0.0; };
thread_local BatchFailure g_batch_fail;  // the last psso_solve_*batch non-finite failure

constexpr int GB_THREADS = 256;
constexpr int GRAPH_CHUNK = 16;  // iterations per captured graph
#ifndef PSSO_SWARM_MAX_ELEMS
#define PSSO_SWARM_MAX_ELEMS (1 << 22)  // N*D up to which psso_run uses the whole-run kernel
#endif

// NCCL, resolved at run time from the process (torch loads its bundled
// libnccl.so.2; C callers put it on the library path or name it in
// PSSO_NCCL_LIB), so libpsso.so has no link-time NCCL dependency.  Only the
// five entry points the sharded iteration uses.
struct NcclUid { char internal[128]; };  // ncclUniqueId (nccl.h NCCL_UNIQUE_ID_BYTES)
struct NcclApi {
  bool ok = false;
  std::string err;
  int (*get_unique_id)(NcclUid*) = nullptr;
  int (*comm_init_rank)(void**, int, NcclUid, int) = nullptr;
  int (*all_gather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*comm_destroy)(void*) = nullptr;
  const char* (*error_string)(int) = nullptr;
};
constexpr int NCCL_UINT8 = 1;  // ncclUint8

const NcclApi& nccl() {
  static NcclApi a = [] {
    NcclApi r;
    const char* env = std::getenv("PSSO_NCCL_LIB");
    void* h = nullptr;
    for (const char* name : {env, "libnccl.so.2", "libnccl.so"}) {
      if (name && *name && (h = dlopen(name, RTLD_NOW | RTLD_GLOBAL)) != nullptr) break;
    }
    if (!h) { r.err = "libnccl.so.2 not found (import torch first or set PSSO_NCCL_LIB)"; return r; }
    r.get_unique_id = (int (*)(NcclUid*))dlsym(h, "ncclGetUniqueId");
    r.comm_init_rank = (int (*)(void**, int, NcclUid, int))dlsym(h, "ncclCommInitRank");
    r.all_gather = (int (*)(const void*, void*, size_t, int, void*, cudaStream_t))dlsym(h, "ncclAllGather");
    r.comm_destroy = (int (*)(void*))dlsym(h, "ncclCommDestroy");
    r.error_string = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
    r.ok = r.get_unique_id && r.comm_init_rank && r.all_gather && r.comm_destroy && r.error_string;
    if (!r.ok) r.err = "libnccl lacks a required entry point";
    return r;
  }();
  return a;
}

// Launch plan of the whole-run kernel (k_swarm); see plan_swarm.
struct SwarmPlan {
  const void* fn = nullptr;
  int G = 0, gpc = 0;
  bool res = false, cl = false;
  size_t smem = 0;
  int off_bar = 0, off_scr = 0, off_pub = 0, off_xs = 0;
};

struct Layout {
  int V, R, G, S, NL;
  bool pre;
  size_t smem;
  int off_xs, off_scr, off_gb, off_hb, off_hf, off_leaf, off_rowf, off_flag, off_red, off_bar;
  int stage_bytes;
  Plan plan;
};

FastDiv make_div(uint32_t d) {
  FastDiv f;
  f.d = d;
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  f.s = l;
  f.m = (uint32_t)(((1ull << 32) * ((1ull << l) - d)) / d + 1);
  return f;
}

// numpy add.reduce recursion (pairwise blocks of <= 128, split at n/2 rounded
// down to a multiple of 8) flattened into leaves + a post-order program.
bool build_plan(int64_t n, Plan& p, std::string& err) {
  std::memset(&p, 0, sizeof(p));
  p.n = (int32_t)n;
  struct Rec {
    static bool go(Plan& p, int64_t off, int64_t n) {
      if (n <= 128) {
        if (p.nleaves >= MAX_LEAVES || p.nops >= MAX_OPS) return false;
        p.leaf_off[p.nleaves] = (int32_t)off;
        p.leaf_len[p.nleaves] = (int32_t)n;
        p.ops[p.nops++] = (int8_t)p.nleaves;
        p.nleaves++;
        return true;
      }
      int64_t n2 = n / 2;
      n2 -= n2 % 8;
      if (!go(p, off, n2) || !go(p, off + n2, n - n2)) return false;
      if (p.nops >= MAX_OPS) return false;
      p.ops[p.nops++] = -1;
      return true;
    }
  };
  if (!Rec::go(p, 0, n)) {
    err = "row reduction needs more than " + std::to_string(MAX_LEAVES) + " pairwise leaves";
    return false;
  }
  return true;
}

int64_t terms_of(int fn, int64_t D) {
  if (fn == 4) return D - 1;
  if (fn == 8) return D / 4;
  return D;
}

size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

constexpr bool heavy_fn(int fn) { return fn == 5 || fn == 6 || fn == 8 || fn == 9; }

// Shared-memory layout of a tile kernel.  k_tile (fused=false): padded xs
// tile + optional term buffer.  k_fused (fused=true): two TMA stages of
// contiguous X and P tiles + optional term buffer, sized for two CTAs per SM.
bool make_layout(int fn, int dtype, int64_t D, bool fused, Layout& L, std::string& err) {
  const int es = dtype == PSSO_F64 ? 8 : 4;
  if (!build_plan(terms_of(fn, D), L.plan, err)) return false;
  L.NL = L.plan.nleaves;
  L.G = 8 * L.NL;
  L.V = dtype == PSSO_F64 ? (D % 2 == 0 ? 2 : 1) : (D % 4 == 0 ? 4 : 1);
  const int mod = dtype == PSSO_F64 ? 16 : 32;
  int64_t S = D;
  while (S % mod != 8 % mod || S % L.V) ++S;  // chain reads conflict-free
  L.S = (int)S;
  auto needs_buf = [&](int R) { return fn == 3 || fn == 7 || (heavy_fn(fn) && R * L.G < NT); };
  auto smem_for = [&](int R) {
    size_t s = fused ? 2 * align16((size_t)2 * R * D * es) : align16((size_t)R * S * es);
    s += needs_buf(R) ? align16((size_t)R * S * es) : 0;  // term buffer
    s += align16(D * es);                                  // gbest
    s += 2 * align16((size_t)R * 8);                       // hashes
    s += align16((size_t)R * L.NL * 16);                   // leaf values
    s += align16((size_t)R * 8) + align16((size_t)R * 4) + 128 + 16;
    return s;
  };
  int R = 1;
  while (2 * R * L.G <= NT) R *= 2;  // chains of R rows fill at most one CTA
  const size_t cap = fused ? 110 * 1024 : 200 * 1024;
  while (R > 1 && smem_for(R) > cap) R /= 2;
  if (smem_for(R) > 227 * 1024) {
    err = "nvar " + std::to_string(D) + " too large for the shared-memory row tile";
    return false;
  }
  L.R = R;
  L.pre = heavy_fn(fn) && R * L.G < NT;
  const bool buf = needs_buf(R);
  size_t o = 0;
  L.stage_bytes = (int)align16((size_t)2 * R * D * es);
  L.off_xs = (int)o; o += fused ? 2 * (size_t)L.stage_bytes : align16((size_t)R * S * es);
  L.off_scr = (int)o; o += buf ? align16((size_t)R * S * es) : 0;
  L.off_gb = (int)o; o += align16(D * es);
  L.off_hb = (int)o; o += align16((size_t)R * 8);
  L.off_hf = (int)o; o += align16((size_t)R * 8);
  L.off_leaf = (int)o; o += align16((size_t)R * L.NL * 16);
  L.off_rowf = (int)o; o += align16((size_t)R * 8);
  L.off_flag = (int)o; o += align16((size_t)R * 4);
  L.off_red = (int)o; o += 128;
  L.off_bar = (int)o; o += 16;
  L.smem = o;
  return true;
}

// chain_row_stride<T, M>() (psso_device.cuh) for a runtime element size and M
size_t host_row_stride(int es, int M) {
  return (size_t)8 * M * es + (size_t)(es == 8 ? row_pad<double>() : row_pad<float>());
}

uint64_t k53(double c) {  // (h >> 11) * 2^-53 < c  <=>  (h >> 11) < ceil(c * 2^53)
  double y = std::ceil(c * 9007199254740992.0);
  if (y <= 0.0) return 0;
  if (y >= 9007199254740992.0) return 1ull << 53;
  return (uint64_t)y;
}
uint64_t k32(double c) {
  double y = std::ceil(c * 4294967296.0);
  if (y <= 0.0) return 0;
  if (y >= 4294967296.0) return 1ull << 32;
  return (uint64_t)y;
}

// ------------------------------------------------------------ kernels ----

struct GbParams {
  const double* slot_f;
  const int64_t* slot_i;
  int32_t nslots;
  int32_t D;
  const void* P;         // local pbests
  int64_t row_lo;
  void* gbest;
  double* g_f;
  double* traj;          // may be null
  int64_t t_arg;
  int64_t* t_dev;        // if non-null: t read here and incremented
  int32_t is_init;
  int32_t pad;
  int64_t* g_idx;        // gBest particle index (parallel.py:208-211), may be null
  unsigned long long* bad;  // this shard's first non-finite key ((t+1) << 40 | i)
  const double* sol_f;      // this shard's sol_f (the non-finite value), may be null
  double* bad_val;          // value of the run's first non-finite fitness (sharded runs)
  int64_t row_hi;           // one past this shard's last row
  unsigned long long* stats;  // per-iteration kernel stats ring (iter_stats), may be null
};

// gBest kernels reset the stats slot of the next iteration (thread 0)
__device__ __forceinline__ void reset_stats(unsigned long long* stats, int64_t t_next) {
  if (!stats || t_next < 0) return;
  unsigned long long* st = stats + 3 * (t_next & (STATS_CAP - 1));
  st[0] = ~0ull;
  st[1] = 0;
  st[2] = 0;
}

// Candidate record of a shard (psso_candidate_bytes): the exchange payload of
// parallel.py:199-208 plus the shard's non-finite state, so that every shard
// stops at the same iteration and reports the same first (t, i)
// (core.py:190-193 over the whole swarm, not per shard).
constexpr int64_t REC_HDR = 32;  // f64 p_f | i64 index | u64 non-finite key | f64 its value | row

// Row copy by one CTA with the loads batched ahead of the stores: a plain
// `dst[j] = src[j]` loop issues one load, waits for it, stores, and repeats --
// for C5's 4096-element rows that was 16 dependent HBM round trips per
// thread (k_gbest took ~10 us per iteration).  `fn(j, v)` receives each element.
template <typename T, typename F>
__device__ __forceinline__ void copy_row(const T* __restrict__ src, int D, F&& fn) {
  constexpr int U = 16;
  for (int base = 0; base < D; base += U * (int)blockDim.x) {
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = base + u * (int)blockDim.x + (int)threadIdx.x;
      if (j < D) v[u] = __ldcg(src + j);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = base + u * (int)blockDim.x + (int)threadIdx.x;
      if (j < D) fn(j, v[u]);
    }
  }
}

template <typename T>
__device__ void block_argmin(const double* f, const int64_t* idx, int n, double& bf, int64_t& bi,
                             double* sf, int64_t* si) {
  bf = CUDART_INF;
  bi = INT64_MAX;
  for (int k = threadIdx.x; k < n; k += blockDim.x)
    if (lex_less(f[k], idx[k], bf, bi)) { bf = f[k]; bi = idx[k]; }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double of = __shfl_xor_sync(0xffffffffu, bf, o);
    int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (lex_less(of, oi, bf, bi)) { bf = of; bi = oi; }
  }
  if ((threadIdx.x & 31) == 0) { sf[threadIdx.x >> 5] = bf; si[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (lex_less(sf[w], si[w], sf[0], si[0])) { sf[0] = sf[w]; si[0] = si[w]; }
  }
  __syncthreads();
  bf = sf[0];
  bi = si[0];
}

// gBest stage 2 (parallel.py:208-212): deterministic lexicographic min over
// the per-CTA slots, `<=` against the incumbent, winner row -> gbest.
template <typename T>
__global__ void __launch_bounds__(GB_THREADS) k_gbest(const __grid_constant__ GbParams g) {
  __shared__ double sf[GB_THREADS / 32];
  __shared__ int64_t si[GB_THREADS / 32];
  pdl_trigger();
  pdl_wait();
  double bf;
  int64_t bi;
  block_argmin<T>(g.slot_f, g.slot_i, g.nslots, bf, bi, sf, si);
  const double inc = *g.g_f;
  const bool take = bi != INT64_MAX && (g.is_init || bf <= inc);
  if (take) {
    const T* src = reinterpret_cast<const T*>(g.P) + (bi - g.row_lo) * (int64_t)g.D;
    T* dst = reinterpret_cast<T*>(g.gbest);
    copy_row<T>(src, g.D, [&](int j, T v) { dst[j] = v; });
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double gf = take ? bf : inc;
    if (take) *g.g_f = gf;
    if (take && g.g_idx) *g.g_idx = bi;
    const int64_t t = g.t_dev ? *g.t_dev : g.t_arg;
    if (g.traj && t >= 0) g.traj[t] = gf;
    if (g.t_dev) *g.t_dev = t + 1;
    reset_stats(g.stats, t + 1);
  }
}

// Local stage 2 for sharded runs: this rank's (p_f, index, row) record,
// written to `n` destinations (dst[q] + off): the local record, or straight
// into every rank's exchange buffer slot (the P2P device loop).
template <typename T>
__device__ __forceinline__ void local_cand_to(const GbParams& g, unsigned char* const* dst, int n,
                                              int64_t off) {
  __shared__ double sf[GB_THREADS / 32];
  __shared__ int64_t si[GB_THREADS / 32];
  double bf;
  int64_t bi;
  block_argmin<T>(g.slot_f, g.slot_i, g.nslots, bf, bi, sf, si);
  if (bi != INT64_MAX) {
    const T* src = reinterpret_cast<const T*>(g.P) + (bi - g.row_lo) * (int64_t)g.D;
    copy_row<T>(src, g.D, [&](int j, T v) {
      for (int q = 0; q < n; ++q) reinterpret_cast<T*>(dst[q] + off + REC_HDR)[j] = v;
    });
  }
  if (threadIdx.x == 0) {
    const unsigned long long key = g.bad ? *g.bad : ~0ull;
    double v = 0.0;
    if (key != ~0ull) {
      const int64_t i = (int64_t)(key & ((1ull << 40) - 1));
      if (g.sol_f && i >= g.row_lo && i < g.row_hi) v = g.sol_f[i - g.row_lo];  // the owner's
      else if (g.bad_val) v = *g.bad_val;                       // learnt from an exchange
    }
    for (int q = 0; q < n; ++q) {
      unsigned char* rec = dst[q] + off;
      *reinterpret_cast<double*>(rec) = bf;
      *reinterpret_cast<int64_t*>(rec + 8) = bi;
      *reinterpret_cast<unsigned long long*>(rec + 16) = key;
      *reinterpret_cast<double*>(rec + 24) = v;
    }
  }
}

template <typename T>
__device__ __forceinline__ void local_cand_body(const GbParams& g, unsigned char* rec) {
  local_cand_to<T>(g, &rec, 1, 0);
}

template <typename T>
__global__ void __launch_bounds__(GB_THREADS) k_local_cand(const __grid_constant__ GbParams g,
                                                           unsigned char* rec) {
  local_cand_body<T>(g, rec);
}

// the run's first non-finite fitness over the gathered records: the minimum
// key, adopted by this shard (so its later iterations are no-ops, like the
// owner's) together with its value
__device__ __forceinline__ void adopt_nonfinite(const GbParams& g, const unsigned char* recs,
                                                int64_t rec_bytes, int n, bool cg) {
  unsigned long long kmin = ~0ull;
  double v = 0.0;
  for (int k = 0; k < n; ++k) {
    const unsigned char* r = recs + k * rec_bytes;
    const unsigned long long key = cg ? (unsigned long long)__ldcg(reinterpret_cast<const long long*>(r + 16))
                                      : *reinterpret_cast<const unsigned long long*>(r + 16);
    if (key < kmin) {
      kmin = key;
      v = cg ? __ldcg(reinterpret_cast<const double*>(r + 24)) : *reinterpret_cast<const double*>(r + 24);
    }
  }
  if (kmin != ~0ull && g.bad && kmin <= *g.bad) {
    *g.bad = kmin;
    if (g.bad_val) *g.bad_val = v;
  }
}

// Global stage 2 over gathered records (one per rank, in rank order).
template <typename T>
__global__ void __launch_bounds__(GB_THREADS) k_apply(const __grid_constant__ GbParams g,
                                                      const unsigned char* recs, int64_t rec_bytes,
                                                      int ncand) {
  __shared__ int winner;
  __shared__ int take_s;
  if (threadIdx.x == 0) {
    double bf = CUDART_INF;
    int64_t bi = INT64_MAX;
    int w = 0;
    for (int k = 0; k < ncand; ++k) {
      const unsigned char* r = recs + k * rec_bytes;
      double f = *reinterpret_cast<const double*>(r);
      int64_t i = *reinterpret_cast<const int64_t*>(r + 8);
      if (lex_less(f, i, bf, bi)) { bf = f; bi = i; w = k; }
    }
    adopt_nonfinite(g, recs, rec_bytes, ncand, false);
    const double inc = *g.g_f;
    take_s = bi != INT64_MAX && (g.is_init || bf <= inc);
    winner = w;
    const double gf = take_s ? bf : inc;
    if (take_s) *g.g_f = gf;
    if (take_s && g.g_idx) *g.g_idx = bi;
    const int64_t t = g.t_dev ? *g.t_dev : g.t_arg;
    if (g.traj && t >= 0) g.traj[t] = gf;
    if (g.t_dev) *g.t_dev = t + 1;
    reset_stats(g.stats, g.is_init ? 0 : t + 1);
  }
  __syncthreads();
  if (take_s) {
    const T* src = reinterpret_cast<const T*>(recs + winner * rec_bytes + REC_HDR);
    T* dst = reinterpret_cast<T*>(g.gbest);
    copy_row<T>(src, g.D, [&](int j, T v) { dst[j] = v; });
  }
}

// per-CTA argmin of p_f over local rows (update_gbest_phase, parallel.py:138-144)
// Device-initiated gBest exchange (SURVEY §8 f #3).  Exchange buffer of a
// rank: [2][R] epoch flags (u64, padded to 16 B), [2][R] candidate records,
// both indexed by epoch parity.
// k_publish stores this rank's record into slot `rank` of EVERY rank's buffer
// (peer pointers: CUDA-IPC / NVLink P2P mappings, or plain pointers for
// virtual ranks on one GPU), then raises its flag in each buffer with a
// system-scope release; k_apply_p2p waits for all R flags of its own buffer
// (system-scope acquire) and applies the selection exactly like k_apply.
// One rank (R == 1): the exchange buffer is touched by this GPU only, so the
// flags need GPU scope; any peer (another GPU, or another process's context)
// needs system scope.
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v, bool sys) {
  if (sys) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p, bool sys) {
  unsigned long long v;
  if (sys) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Graph-replayed loops take the epoch from the device iteration counter:
// epoch = t + 2 (initialization: 1), so a captured graph needs no host value.
__device__ __forceinline__ unsigned long long p2p_epoch(unsigned long long epoch, const int64_t* t_dev) {
  return t_dev ? (unsigned long long)(*t_dev + 2) : epoch;
}

__device__ __forceinline__ void publish_body(const unsigned char* cand, unsigned char* const* bufs,
                                             int R, int rank, unsigned long long epoch,
                                             int64_t rec_bytes, int64_t flag_bytes) {
  const uint64_t* src = reinterpret_cast<const uint64_t*>(cand);
  const int64_t words = rec_bytes / 8;
  const int slot = (int)(epoch & 1) * R + rank;  // records double-buffered by epoch parity
  for (int q = 0; q < R; ++q) {
    uint64_t* dst = reinterpret_cast<uint64_t*>(bufs[q] + flag_bytes + (int64_t)slot * rec_bytes);
    for (int64_t w = threadIdx.x; w < words; w += blockDim.x) dst[w] = src[w];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // the block's record stores happen-before this thread's release through the
    // barrier, and release is cumulative: no separate system-wide fence (which
    // measured ~5 us per exchange) is needed
    for (int q = 0; q < R; ++q)
      st_release_u64(reinterpret_cast<unsigned long long*>(bufs[q]) + slot, epoch, R > 1);
  }
}

__global__ void __launch_bounds__(GB_THREADS) k_publish(const unsigned char* cand,
                                                        unsigned char* const* bufs, int R, int rank,
                                                        unsigned long long epoch_arg, int64_t rec_bytes,
                                                        int64_t flag_bytes, const int64_t* t_dev) {
  publish_body(cand, bufs, R, rank, p2p_epoch(epoch_arg, t_dev), rec_bytes, flag_bytes);
}

// The device loop's record + publish: this rank's record (as k_local_cand),
// stored into every rank's buffer, then the epoch flags.  Up to 8 peers (a node's GPUs) travel by value in the launch parameters, so
// the kernel starts without a dependent load of the peer table.
struct PeerPtrs {
  unsigned char* p[8];
  int32_t n;  // 0: read the device table instead
};

template <typename T>
__device__ __forceinline__ void local_cand_publish_body(const GbParams& g, unsigned char* const* bufs,
                                                        const PeerPtrs& pp, int R, int rank,
                                                        int64_t rec_bytes, int64_t flag_bytes,
                                                        unsigned long long epoch) {
  const int slot = (int)(epoch & 1) * R + rank;  // records double-buffered by epoch parity
  // the record straight into this rank's slot of every buffer (R <= 64 ranks)
  __shared__ unsigned char* dst_s[64];
  unsigned char* const* dst = pp.p;
  if (pp.n == 0) {
    for (int q = threadIdx.x; q < R && q < 64; q += blockDim.x) dst_s[q] = bufs[q];
    __syncthreads();
    dst = dst_s;
  }
  local_cand_to<T>(g, dst, R < 64 ? R : 64, flag_bytes + (int64_t)slot * rec_bytes);
  __syncthreads();  // every store of the record precedes the releases (cumulativity)
  if (threadIdx.x == 0)
    for (int q = 0; q < R; ++q)
      st_release_u64(reinterpret_cast<unsigned long long*>(dst[q]) + slot, epoch, R > 1);
}

template <typename T>
__device__ __forceinline__ void apply_p2p_body(const GbParams& g, const unsigned char* buf, int R,
                                               unsigned long long epoch, int64_t rec_bytes,
                                               int64_t flag_bytes) {
  __shared__ int winner;
  __shared__ int take_s;
  // a rank can publish epoch e+1 before a slower rank applied epoch e, never
  // e+2 (that needs the slower rank's e+1 record): parity buffers suffice
  const int par = (int)(epoch & 1);
  const unsigned char* recs = buf + flag_bytes + (int64_t)par * R * rec_bytes;
  if (threadIdx.x == 0) {
    const double inc = *g.g_f;  // this rank's own state: loaded while the flags are polled
    const unsigned long long* flags = reinterpret_cast<const unsigned long long*>(buf) + par * R;
    for (int q = 0; q < R; ++q)
      while (ld_acquire_u64(flags + q, R > 1) < epoch) __nanosleep(32);
    double bf = CUDART_INF;
    int64_t bi = INT64_MAX;
    int w = 0;
    for (int k = 0; k < R; ++k) {
      const unsigned char* r = recs + k * rec_bytes;
      const double f = __ldcg(reinterpret_cast<const double*>(r));
      const int64_t i = __ldcg(reinterpret_cast<const long long*>(r + 8));
      if (lex_less(f, i, bf, bi)) { bf = f; bi = i; w = k; }
    }
    adopt_nonfinite(g, recs, rec_bytes, R, true);
    take_s = bi != INT64_MAX && (g.is_init || bf <= inc);  // parallel.py:209
    winner = w;
    const double gf = take_s ? bf : inc;
    if (take_s) *g.g_f = gf;
    if (take_s && g.g_idx) *g.g_idx = bi;
    const int64_t t = g.t_dev ? *g.t_dev : g.t_arg;
    if (g.traj && t >= 0) g.traj[t] = gf;
    if (g.t_dev) *g.t_dev = t + 1;
    reset_stats(g.stats, g.is_init ? 0 : t + 1);
    __threadfence_block();
  }
  __syncthreads();
  if (take_s) {
    const T* src = reinterpret_cast<const T*>(recs + winner * rec_bytes + REC_HDR);
    T* dst = reinterpret_cast<T*>(g.gbest);
    copy_row<T>(src, g.D, [&](int j, T v) { dst[j] = v; });
  }
}

template <typename T>
__global__ void __launch_bounds__(GB_THREADS) k_apply_p2p(const __grid_constant__ GbParams g,
                                                          const unsigned char* buf, int R,
                                                          unsigned long long epoch_arg, int64_t rec_bytes,
                                                          int64_t flag_bytes) {
  apply_p2p_body<T>(g, buf, R, p2p_epoch(epoch_arg, g.t_dev), rec_bytes, flag_bytes);
}

// The device loop's whole exchange in ONE kernel: this rank's record, stored
// into every rank's buffer with the epoch flags, then (same CTA) the wait for
// every rank's flag, the lexicographic minimum and the gBest update.  Each
// rank publishes before it waits, so the ranks' kernels cannot wait on each
// other in a cycle; one launch per iteration fewer than publish + apply.
template <typename T>
__global__ void __launch_bounds__(GB_THREADS) k_p2p_exchange(const __grid_constant__ GbParams g,
                                                             unsigned char* const* bufs,
                                                             const __grid_constant__ PeerPtrs pp,
                                                             const unsigned char* my_buf, int R, int rank,
                                                             int64_t rec_bytes, int64_t flag_bytes) {
  const unsigned long long epoch = p2p_epoch(0, g.t_dev);  // before apply advances t_dev
  local_cand_publish_body<T>(g, bufs, pp, R, rank, rec_bytes, flag_bytes, epoch);
  __syncthreads();
  apply_p2p_body<T>(g, my_buf, R, epoch, rec_bytes, flag_bytes);
}

__global__ void k_argmin(const double* f, int64_t n, int64_t row_lo, double* slot_f,
                         int64_t* slot_i) {
  __shared__ double sf[32];
  __shared__ int64_t si[32];
  double bf = CUDART_INF;
  int64_t bi = INT64_MAX;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    if (lex_less(f[k], row_lo + k, bf, bi)) { bf = f[k]; bi = row_lo + k; }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double of = __shfl_xor_sync(0xffffffffu, bf, o);
    int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (lex_less(of, oi, bf, bi)) { bf = of; bi = oi; }
  }
  if ((threadIdx.x & 31) == 0) { sf[threadIdx.x >> 5] = bf; si[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (lex_less(sf[w], si[w], bf, bi)) { bf = sf[w]; bi = si[w]; }
    slot_f[blockIdx.x] = bf;
    slot_i[blockIdx.x] = bi;
  }
}

// update_pbests_phase (parallel.py:132-135): sol_f <= p_f -> copy row.
template <typename T>
__global__ void k_pbest(const T* X, T* P, const double* sol_f, double* p_f, int64_t rows, int D) {
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const bool imp = sol_f[r] <= p_f[r];
    if (!imp) continue;
    for (int j = threadIdx.x; j < D; j += blockDim.x) P[r * D + j] = X[r * D + j];
    __syncthreads();
    if (threadIdx.x == 0) p_f[r] = sol_f[r];
  }
}

__global__ void k_rng(uint64_t seed, uint64_t stream, uint64_t t, const uint64_t* ii,
                      const uint64_t* jj, int64_t n, double* out) {
  const uint64_t root = root64(seed, stream, t);
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = unit53(fold64(fold64(root, ii[k]), jj[k]));
}


__global__ void k_set(int64_t* p, int64_t v) { *p = v; }
__global__ void k_set_u64(unsigned long long* p, unsigned long long v) { *p = v; }

// ---- the sequential schedule for rows beyond the chain mapping (nvar > 128):
// the same speculative passes as k_seq (psso_seq.cuh), as a pass loop of
// kernels over the HBM-resident swarm.  ctl = [lo, first event, failed].
// First event in [lo, N): a non-finite fitness (core.py:233) or a pBest `<=`
// that is also `<=` g_f (core.py:236-241).  One CTA; lowest index wins.
__global__ void __launch_bounds__(1024) k_seq_event(const double* fn, const double* p_f,
                                                    const double* g_f, int64_t* ctl, int64_t N) {
  __shared__ int64_t red[32];
  const int64_t lo = ctl[0];
  const double gf = *g_f;
  int64_t ev = INT64_MAX;
  for (int64_t r = lo + threadIdx.x; r < N; r += blockDim.x) {
    const double f = fn[r];
    if (!isfinite(f) || (f <= p_f[r] && f <= gf)) { ev = r; break; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ev = min(ev, (int64_t)__shfl_xor_sync(0xffffffffu, ev, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ev;
  __syncthreads();
  if (threadIdx.x < 32) {
    ev = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : INT64_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ev = min(ev, (int64_t)__shfl_xor_sync(0xffffffffu, ev, o));
    if (threadIdx.x == 0) ctl[1] = ev == INT64_MAX ? N : ev;
  }
}

// commit rows lo..min(ev, N-1): X always (core.py:231), pBest on `<=` (:236-238)
template <typename T>
__global__ void k_seq_commit(T* X, T* P, const T* Xn, const double* fn, double* p_f, double* sol_f,
                             const int64_t* ctl, int64_t N, int D) {
  const int64_t lo = ctl[0], hi = min(ctl[1], N - 1);
  for (int64_t r = lo + blockIdx.x; r <= hi; r += gridDim.x) {
    const double f = fn[r];
    const bool imp = isfinite(f) && f <= p_f[r];
    const T* src = Xn + r * (int64_t)D;
    copy_row<T>(src, D, [&](int j, T v) {
      X[r * (int64_t)D + j] = v;
      if (imp) P[r * (int64_t)D + j] = v;
    });
    __syncthreads();  // every thread read p_f[r] before it moves
    if (threadIdx.x == 0) {
      if (sol_f) sol_f[r] = f;
      if (imp) p_f[r] = f;
    }
  }
}

// the event: gbest <- pbests[r*] (core.py:239-241) or the non-finite stop;
// next pass from r* + 1; trajectory[t] once the iteration is complete (:242)
template <typename T>
__global__ void k_seq_move(T* gbest, const T* Xn, const double* fn, double* g_f, int64_t* g_idx,
                           unsigned long long* bad, double* traj, int64_t t, int64_t* ctl,
                           int64_t* passes, int64_t N, int D) {
  __shared__ int stop;
  const int64_t ev = ctl[1];
  if (threadIdx.x == 0) stop = ev < N && !isfinite(fn[ev]);
  __syncthreads();
  if (ev < N && !stop)
    copy_row<T>(Xn + ev * (int64_t)D, D, [&](int j, T v) { gbest[j] = v; });
  if (threadIdx.x == 0) {
    if (passes) *passes += 1;
    if (stop) {
      if (bad) atomicMin(bad, ((unsigned long long)(t + 1) << 40) | (unsigned long long)ev);
      ctl[2] = 1;
      ctl[0] = N;
    } else {
      if (ev < N) {
        *g_f = fn[ev];
        if (g_idx) *g_idx = ev;
      }
      ctl[0] = ev < N ? ev + 1 : N;
      if (ctl[0] >= N && traj) traj[t] = *g_f;
    }
  }
}

}  // namespace

// ------------------------------------------------------------- context ----

struct psso_comm {  // an NCCL communicator on one device (rank `rank` of `nranks`)
  void* comm;
  int32_t nranks, rank;
  int device;
};

struct psso_ctx {
  psso_config cfg;
  psso_buffers buf;
  bool bound;
  cudaStream_t stream;
  int device, num_sms;
  Layout L;   // k_tile
  Layout LF;  // fused kernel (k_fused when rows vectorize, else k_tile<fused>)
  const void* tile_fn;   // runtime-mode tile kernel (init, phases, evaluation)
  const void* fused_fn;  // fused iteration kernel (the hot path)
  const void* init_fn;   // initialization kernel (k_chain<INIT> or k_tile)
  bool chain;            // fused/init run the register-resident chain kernel
  int rows_w;            // >0: the fused iteration is k_rows with W = rows_w warps per row
  int grid;
  int fused_grid;
  int init_grid;
  size_t init_smem;      // dynamic smem of the chain init kernel (no prefetch buffers)
  int argmin_grid;
  int nslots;
  double* slot_f;
  int64_t* slot_i;
  unsigned long long* bad;
  int64_t* t_dev;
  int64_t* g_idx;        // gBest particle index, -1 before initialization
  double* bad_val;       // first non-finite value learnt from a candidate exchange
  unsigned long long* stats;  // per-iteration kernel stats ring [STATS_CAP][3]
  double* aux;
  uint64_t Kw, Kp, Kg, Kw32, Kp32, Kg32;
  int64_t launches;
  cudaGraphExec_t graph;
  // kernel timing (psso_profile): event pairs around each fused tile launch
  bool profiling;
  std::vector<cudaEvent_t> ev;
  size_t ev_used;
  int64_t prof_iters;    // iterations covered by the timed launches
  // whole-run kernel for small swarms (psso_swarm.cuh); null: streaming path
  const void* swarm_fn;   // == swarm.fn
  SwarmPlan swarm;
  unsigned int* sw_epoch;
  double* sw_slot_f;
  int64_t* sw_slot_i;
  int32_t* sw_slot_new;
  void* sw_slot_row;
  uint64_t* sw_seed;
  // sequential schedule (psso_seq.cuh), allocated on first use
  void* seq_xn;          // rows x D speculative rows
  double* seq_fn;        // rows speculative fitness
  double* seq_pfn;       // rows scratch
  uint64_t* seq_seed;
  int64_t* seq_passes;
  int64_t* seq_ctl;      // long-row sequential passes: [lo, event, failed, -]
  int64_t* seq_ctl_host; // pinned copy
  // sharded iteration over a library-owned NCCL communicator (psso_attach_nccl)
  void* comm;            // ncclComm_t, borrowed from a psso_comm
  int32_t nranks, rank;
  unsigned char* cand;   // this rank's candidate record
  unsigned char* gathered;  // [nranks] records, rank order
  cudaGraphExec_t sgraph;   // GRAPH_CHUNK sharded iterations
  cudaGraphExec_t pgraph;   // GRAPH_CHUNK P2P-exchange iterations (psso_run_p2p)
  const void* pg_peers;     // the arguments pgraph was captured with
  const void* pg_buf;
  int32_t pg_R, pg_rank;
  PeerPtrs pp;              // psso_run_p2p's peer table by value (<= 8 ranks) ...
  const void* pp_src;       // ... read from this device table
  int32_t pp_R;
  std::string kname;     // the iteration kernel psso_run launches (psso_kernel_name)
  std::string err;
};

namespace {

int fail(psso_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  g_err = msg;
  return code;
}

int cuda_fail(psso_ctx* c, cudaError_t e, const char* where) {
  return fail(c, PSSO_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(ctx, call)                                  \
  do {                                                 \
    cudaError_t e_ = (call);                           \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
  } while (0)

int validate(const psso_config* c, std::string& err) {
  if (!c) { err = "null config"; return PSSO_E_INVALID; }
  if (c->fn_id < 0 || c->fn_id > 9) { err = "unknown function id " + std::to_string(c->fn_id); return PSSO_E_INVALID; }
  if (c->dtype != PSSO_F64 && c->dtype != PSSO_F32) { err = "dtype must be PSSO_F64 or PSSO_F32"; return PSSO_E_INVALID; }
  if (c->rng_mode != PSSO_RNG_REFERENCE && c->rng_mode != PSSO_RNG_PHILOX) { err = "unknown rng_mode"; return PSSO_E_INVALID; }
  if (!(0.0 <= c->cw && c->cw <= c->cp && c->cp <= c->cg && c->cg <= 1.0)) {
    char b[160];
    std::snprintf(b, sizeof b, "thresholds must satisfy 0 <= cw <= cp <= cg <= 1, got (%.17g, %.17g, %.17g)", c->cw, c->cp, c->cg);
    err = b;
    return PSSO_E_INVALID;
  }
  if (!(c->var_min < c->var_max)) { err = "need var_min < var_max"; return PSSO_E_INVALID; }
  if (c->nsol < 1) { err = "nsol must be a positive integer"; return PSSO_E_INVALID; }
  if (c->nvar < 1) { err = "nvar must be a positive integer"; return PSSO_E_INVALID; }
  if (c->fn_id == 4 && c->nvar < 2) { err = "f4 needs dimension >= 2"; return PSSO_E_INVALID; }
  if (c->fn_id == 8 && c->nvar < 4) { err = "f8 needs at least 4 variables"; return PSSO_E_INVALID; }
  if (!(0 <= c->row_lo && c->row_lo < c->row_hi && c->row_hi <= c->nsol)) { err = "row range must satisfy 0 <= row_lo < row_hi <= nsol"; return PSSO_E_INVALID; }
  if (c->nvar > (1 << 20)) { err = "nvar too large"; return PSSO_E_UNSUPPORTED; }
  if (c->flags & ~PSSO_FLAG_KEEP_SOL_F) { err = "unknown flags"; return PSSO_E_INVALID; }
  return PSSO_OK;
}

TileParams tile_params(psso_ctx* c, int mode, int64_t t, const int64_t* t_dev, bool fused = false) {
  TileParams p;
  std::memset(&p, 0, sizeof(p));
  const Layout& L = fused ? c->LF : c->L;
  p.X = c->buf.sol;
  p.P = c->buf.pbests;
  p.sol_f = c->buf.sol_f;
  p.p_f = c->buf.p_f;
  p.gbest = c->buf.gbest;
  p.rows = c->cfg.row_hi - c->cfg.row_lo;
  p.row_lo = c->cfg.row_lo;
  p.D = (int32_t)c->cfg.nvar;
  p.R = L.R;
  p.G = L.G;
  p.S = L.S;
  p.cpr = (int32_t)(c->cfg.nvar / L.V);
  p.mode = mode;
  p.div_cpr = make_div((uint32_t)p.cpr);
  p.div_G = make_div((uint32_t)L.G);
  p.div_D = make_div((uint32_t)c->cfg.nvar);
  p.seed = c->cfg.seed;
  p.Kw = c->Kw; p.Kp = c->Kp; p.Kg = c->Kg;
  p.Kw32 = c->Kw32; p.Kp32 = c->Kp32; p.Kg32 = c->Kg32;
  p.Kw32u = (uint32_t)std::min<uint64_t>(c->Kw32, 0xFFFFFFFFull);
  p.Kp32u = (uint32_t)std::min<uint64_t>(c->Kp32, 0xFFFFFFFFull);
  p.Kg32u = (uint32_t)std::min<uint64_t>(c->Kg32, 0xFFFFFFFFull);
  p.K32on = (c->Kw32 >> 32 ? 0u : 1u) | (c->Kp32 >> 32 ? 0u : 2u) | (c->Kg32 >> 32 ? 0u : 4u);
  p.var_min = c->cfg.var_min;
  p.span = c->cfg.var_max - c->cfg.var_min;
  p.span53 = std::ldexp(p.span, -53);
  p.span64 = std::ldexp(p.span, -64);
  p.span32 = std::ldexp(p.span, -32);
  p.probe_level = c->cfg.probe_level;
  p.t_arg = t;
  p.t_dev = t_dev;
  p.slot_f = c->slot_f;
  p.slot_i = c->slot_i;
  p.bad = c->bad;
  p.aux = c->aux;
  p.off_xs = L.off_xs; p.off_scr = L.off_scr; p.off_gb = L.off_gb; p.off_hb = L.off_hb;
  p.off_hf = L.off_hf; p.off_leaf = L.off_leaf; p.off_rowf = L.off_rowf; p.off_flag = L.off_flag;
  p.off_red = L.off_red;
  p.off_bar = L.off_bar;
  p.stage_bytes = L.stage_bytes;
  p.pre = L.pre ? 1 : 0;
  p.div_n = make_div((uint32_t)L.plan.n);
  p.plan = L.plan;
  p.stats = c->stats;
  return p;
}

// A launch that may overlap its predecessor's drain (PSSO_PDL); only kernels
// that read predecessor output behind griddepcontrol.wait are launched so.
cudaError_t launch_pdl(const void* fn, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t s) {
  cudaLaunchConfig_t lc = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  lc.attrs = at;
  lc.numAttrs = PSSO_PDL ? 1 : 0;
  return cudaLaunchKernelExC(&lc, fn, args);
}

int launch_tile(psso_ctx* c, const TileParams& p, bool fused = false) {
  void* args[] = {(void*)&p};
  if (fused && (c->chain || c->rows_w)) {  // k_chain / k_rows wait on their predecessor
    CK(c, launch_pdl(c->fused_fn, dim3(c->fused_grid), dim3(NT), args, c->LF.smem, c->stream));
  } else {
    CK(c, cudaLaunchKernel(fused ? c->fused_fn : c->tile_fn, dim3(fused ? c->fused_grid : c->grid),
                           dim3(NT), args, fused ? c->LF.smem : c->L.smem, c->stream));
  }
  c->launches++;
  return PSSO_OK;
}

GbParams gb_params(psso_ctx* c, int64_t t, int64_t* t_dev, int is_init, int nslots) {
  GbParams g;
  std::memset(&g, 0, sizeof(g));
  g.slot_f = c->slot_f;
  g.slot_i = c->slot_i;
  g.nslots = nslots;
  g.D = (int32_t)c->cfg.nvar;
  g.P = c->buf.pbests;
  g.row_lo = c->cfg.row_lo;
  g.gbest = c->buf.gbest;
  g.g_f = c->buf.g_f;
  g.traj = c->buf.traj;
  g.t_arg = t;
  g.t_dev = t_dev;
  g.is_init = is_init;
  g.g_idx = c->g_idx;
  g.bad = c->bad;
  g.sol_f = c->buf.sol_f;
  g.bad_val = c->bad_val;
  g.row_hi = c->cfg.row_hi;
  g.stats = c->stats;
  return g;
}

int launch_gbest(psso_ctx* c, const GbParams& g) {
  void* args[] = {(void*)&g};
  const void* fn = c->cfg.dtype == PSSO_F64 ? (const void*)k_gbest<double> : (const void*)k_gbest<float>;
  CK(c, launch_pdl(fn, dim3(1), dim3(GB_THREADS), args, 0, c->stream));
  c->launches++;
  return PSSO_OK;
}

// Every context entry point runs on the context's device (the one current at
// psso_create), whatever device the calling thread has current; the caller's
// device is restored on return.
struct DevGuard {
  int prev = -1;
  explicit DevGuard(const psso_ctx* c) {
    if (c && cudaGetDevice(&prev) == cudaSuccess && prev != c->device) cudaSetDevice(c->device);
    else prev = -1;
  }
  ~DevGuard() { if (prev >= 0) cudaSetDevice(prev); }
};
#define DEV_GUARD(c) DevGuard dev_guard_(c)

// NVTX ranges (domain "psso") around the entry points that issue device work:
// nvtx3 is header-only and does nothing unless a tool injects itself, so the
// ranges cost one predictable branch per call.  Under ncu they scope captures
// (`ncu --nvtx --nvtx-include "psso@psso_run/"`), under a timeline tool they
// label the host spans of init / run / solve / exchange calls.
struct NvtxRange {
  static nvtxDomainHandle_t domain() {
    static const nvtxDomainHandle_t d = nvtxDomainCreateA("psso");
    return d;
  }
  explicit NvtxRange(const char* name) {
    nvtxEventAttributes_t a = {};
    a.version = NVTX_VERSION;
    a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
    a.messageType = NVTX_MESSAGE_TYPE_ASCII;
    a.message.ascii = name;
    nvtxDomainRangePushEx(domain(), &a);
  }
  ~NvtxRange() { nvtxDomainRangePop(domain()); }
};
#define TRACE(name) NvtxRange nvtx_range_(name)

int need_bound(psso_ctx* c) {
  if (!c) return fail(nullptr, PSSO_E_INVALID, "null context");
  if (!c->bound) return fail(c, PSSO_E_INVALID, "context has no buffers bound (psso_bind)");
  return PSSO_OK;
}

int fused_mode(const psso_ctx* c) {
  return M_SEARCH | M_EVAL | M_PBEST | M_CAND | ((c->cfg.flags & PSSO_FLAG_KEEP_SOL_F) ? M_SOLF : 0);
}

// the fused tile kernel, bracketed by timing events while profiling
int launch_fused(psso_ctx* c, int64_t t, int64_t* t_dev) {
  const bool timed = c->profiling && !t_dev;
  if (timed) {
    if (c->ev_used + 2 > c->ev.size()) {
      for (int k = 0; k < 64; ++k) {
        cudaEvent_t e;
        CK(c, cudaEventCreate(&e));
        c->ev.push_back(e);
      }
    }
    CK(c, cudaEventRecord(c->ev[c->ev_used], c->stream));
  }
  int rc = launch_tile(c, tile_params(c, fused_mode(c), t, t_dev, true), true);
  if (rc) return rc;
  if (timed) {
    CK(c, cudaEventRecord(c->ev[c->ev_used + 1], c->stream));
    c->ev_used += 2;
    c->prof_iters += 1;
  }
  return PSSO_OK;
}

int fused_step(psso_ctx* c, int64_t t, int64_t* t_dev) {
  if (int rc = launch_fused(c, t, t_dev)) return rc;
  return launch_gbest(c, gb_params(c, t, t_dev, 0, c->fused_grid));
}

// Launch plan of the whole-run kernel for B swarms of this configuration:
// RES (rows in smem, gpc row groups per CTA) when the tiles fit and the
// B x G CTAs can be co-resident; else rows in HBM, one row group per warp.
// G = 1 needs no co-residency (the swarm barrier is __syncthreads).
// Launch plan of the whole-run kernel for B swarms of this configuration.
// Preferred: CL -- one thread-block cluster of G <= 16 CTAs per swarm, rows
// resident in smem, exchange over DSMEM (clusters are independent, so any
// number of swarms).  Else the global-memory exchange: RES when the tiles fit
// and the B x G CTAs can be co-resident; else rows in HBM.  G = 1 needs no
// co-residency.
// Dynamic shared memory cap of a kernel.  The attribute is per function and
// process-wide, so concurrent contexts (host threads running cells or seeds
// side by side) would race if each set its own size: every caller sets the
// device's opt-in maximum instead (the launch's own size decides occupancy),
// after checking that its need fits.
cudaError_t allow_smem(const void* f, size_t need) {
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  cudaFuncAttributes fa;
  if ((e = cudaFuncGetAttributes(&fa, f)) != cudaSuccess) return e;
  const int cap = optin - (int)fa.sharedSizeBytes;  // dynamic + static <= opt-in maximum
  if (need > (size_t)cap) return cudaErrorInvalidValue;
  return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
}

bool plan_swarm(psso_ctx* c, int64_t B, SwarmPlan& sp, cudaError_t& e) {
  const psso_config* cfg = &c->cfg;
  const int64_t rows = cfg->row_hi - cfg->row_lo, D = cfg->nvar;
  const int M = D <= 32 ? 4 : D <= 64 ? 8 : 16;
  const int es = cfg->dtype == PSSO_F64 ? 8 : 4;
  const int nw = PSSO_SWARM_NT / 32;
  const bool smem_fn = cfg->fn_id == 3 || cfg->fn_id == 7 || cfg->fn_id == 8;
  const int64_t ngroups = (rows + 3) / 4;
  sp.off_bar = (int)align16((size_t)c->LF.off_red + 16 * nw + 64 * M);
  sp.off_scr = (int)align16((size_t)sp.off_bar + 24 + 4 * (nw + 1));
  sp.off_pub = (int)align16((size_t)sp.off_scr + (smem_fn ? (size_t)nw * 4 * (8 * M) * es : 0));
  sp.off_xs = (int)align16((size_t)sp.off_pub + 64 + 2 * (size_t)D * es);
  e = cudaSuccess;
  auto res_smem = [&](int64_t gpc) { return (size_t)sp.off_xs + (size_t)gpc * 4 * (D * 2 * es + 8); };
  const char* nc = std::getenv("PSSO_SWARM_NO_CLUSTER");
  if (!(nc && *nc && *nc != '0')) {
    const char* gs = std::getenv("PSSO_SWARM_G");
    // about half the warps of each CTA busy: shorter per-CTA chains beat fewer CTAs
    int64_t G = std::max<int64_t>(1, std::min<int64_t>(16, (ngroups + 7) / 8));
    // a batch: no more clusters than fit one wave (B * G <= SMs) while the
    // CTA's rows still fit in shared memory -- a second wave doubles the time
    if (B > 1)
      while (G > 1 && B * G > c->num_sms && res_smem((ngroups + G - 2) / (G - 1)) <= 227 * 1024) --G;
    if (gs && *gs) G = std::max<int64_t>(1, std::min<int64_t>(16, std::atoll(gs)));
    const int64_t gpc = (ngroups + G - 1) / G;
    G = (ngroups + gpc - 1) / gpc;
    const size_t smem = res_smem(gpc);
    const void* f = swarm_kernel(cfg->dtype, cfg->rng_mode, cfg->fn_id, M, true, true);
    if (f && smem <= 227 * 1024) {
      if ((e = allow_smem(f, smem)) != cudaSuccess ||
          (G > 8 && (e = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess))
        return false;
      cudaLaunchConfig_t lc = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = (unsigned)G;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.gridDim = dim3((unsigned)G, 1, 1);
      lc.blockDim = dim3(PSSO_SWARM_NT, 1, 1);
      lc.dynamicSmemBytes = smem;
      lc.attrs = at;
      lc.numAttrs = 1;
      int nclusters = 0;
      if ((e = cudaOccupancyMaxActiveClusters(&nclusters, f, &lc)) != cudaSuccess) {
        e = cudaSuccess;  // cluster size not schedulable: fall through
        cudaGetLastError();
      } else if (nclusters >= 1) {
        sp.fn = f; sp.G = (int)G; sp.gpc = (int)gpc; sp.res = true; sp.cl = true; sp.smem = smem;
        return true;
      }
    }
  }
  auto try_plan = [&](bool res, int64_t gpc, int64_t G) -> bool {
    const size_t smem = res ? res_smem(gpc) : (size_t)sp.off_xs;
    if (smem > 227 * 1024) return false;
    const void* f = swarm_kernel(cfg->dtype, cfg->rng_mode, cfg->fn_id, M, res, false);
    if (!f) return false;
    int per_sm = 0;
    if ((e = allow_smem(f, smem)) != cudaSuccess ||
        (e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, PSSO_SWARM_NT, smem)) != cudaSuccess)
      return false;
    const int64_t cap = (int64_t)per_sm * c->num_sms;
    if (per_sm < 1 || (G > 1 && G * B > cap)) return false;
    sp.fn = f; sp.G = (int)G; sp.gpc = (int)gpc; sp.res = res; sp.cl = false; sp.smem = smem;
    return true;
  };
  const char* g = std::getenv("PSSO_SWARM_GPC");
  const int64_t gpc = std::max<int64_t>(1, std::min<int64_t>(ngroups, g && *g ? std::atoll(g) : nw));
  if (try_plan(true, gpc, (ngroups + gpc - 1) / gpc)) return true;   // resident, co-resident
  if (e != cudaSuccess) return false;
  if (try_plan(true, ngroups, 1)) return true;                       // resident, one CTA per swarm
  if (e != cudaSuccess) return false;
  int per_sm = 0;                                                     // rows in HBM
  const void* f = swarm_kernel(cfg->dtype, cfg->rng_mode, cfg->fn_id, M, false, false);
  if (!f) return false;
  if ((e = allow_smem(f, sp.off_xs)) != cudaSuccess ||
      (e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, PSSO_SWARM_NT, sp.off_xs)) != cudaSuccess || per_sm < 1)
    return false;
  const int64_t cap = (int64_t)per_sm * c->num_sms;
  int64_t G = std::max<int64_t>(1, std::min<int64_t>((ngroups + nw - 1) / nw, cap / B));
  if (G * B > cap) G = 1;
  sp.fn = f; sp.G = (int)G; sp.gpc = nw; sp.res = false; sp.cl = false; sp.smem = sp.off_xs;
  return true;
}

// Launch B swarms of the plan (grid G x B; clusters of G, or cooperative).
cudaError_t launch_swarm(const SwarmPlan& pl, int64_t B, void** args, cudaStream_t s) {
  if (pl.cl) {
    cudaLaunchConfig_t lc = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)pl.G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.gridDim = dim3((unsigned)pl.G, (unsigned)B, 1);
    lc.blockDim = dim3(PSSO_SWARM_NT, 1, 1);
    lc.dynamicSmemBytes = pl.smem;
    lc.stream = s;
    lc.attrs = at;
    lc.numAttrs = 1;
    return cudaLaunchKernelExC(&lc, pl.fn, args);
  }
  if (pl.G > 1)  // co-residency of the swarm's CTAs is required by its barrier
    return cudaLaunchCooperativeKernel(pl.fn, dim3(pl.G, (unsigned)B), dim3(PSSO_SWARM_NT), args, pl.smem, s);
  return cudaLaunchKernel(pl.fn, dim3(1, (unsigned)B), dim3(PSSO_SWARM_NT), args, pl.smem, s);
}

// One persistent stream per host thread (and device) for the one-shot entry
// points: blocks freed on a stream are reusable by the next call's
// allocations on the SAME stream without any cross-stream dependency, so
// repeated calls never map fresh HBM (with a new stream per call every other
// 16 GiB call paid ~0.7 s of mapping).
cudaError_t solve_stream(cudaStream_t* s) {
  thread_local cudaStream_t st[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!st[dev] && (e = cudaStreamCreateWithFlags(&st[dev], cudaStreamNonBlocking)) != cudaSuccess) return e;
  *s = st[dev];
  return cudaSuccess;
}

// Stream-ordered allocations for the one-shot host-buffer entry points
// (psso_solve, psso_solve_batch): the device's default memory pool keeps
// freed blocks cached (release threshold = max), so repeated calls do not
// pay for mapping and unmapping gigabytes of HBM.
cudaError_t pool_alloc(void** p, size_t bytes, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    configured = true;
  }
  return cudaMallocAsync(p, bytes, s);
}

}  // namespace

// ------------------------------------------------------------- C ABI ----

extern "C" {

const char* psso_version(void) { return "psso-b200 2 (sm_100a)"; }

const char* psso_kernel_name(const psso_ctx* ctx) { return ctx ? ctx->kname.c_str() : ""; }

const char* psso_last_error(const psso_ctx* ctx) {
  if (ctx && !ctx->err.empty()) return ctx->err.c_str();
  return g_err.c_str();
}

int psso_create(const psso_config* cfg, psso_ctx** out) {
  std::string err;
  if (!out) return fail(nullptr, PSSO_E_INVALID, "null output pointer");
  *out = nullptr;
  int rc = validate(cfg, err);
  if (rc) return fail(nullptr, rc, err);
  psso_ctx* c = new psso_ctx();
  c->cfg = *cfg;
  c->bound = false;
  c->stream = nullptr;
  c->graph = nullptr;
  c->launches = 0;
  c->profiling = false;
  c->ev_used = 0;
  if (!make_layout(cfg->fn_id, cfg->dtype, cfg->nvar, false, c->L, err)) {
    delete c;
    return fail(nullptr, PSSO_E_UNSUPPORTED, err);
  }
  {  // the TMA kernel needs 16-byte rows (vectorized V > 1); else the fused k_tile
    const bool tma = c->L.V > 1;
    if (!make_layout(cfg->fn_id, cfg->dtype, cfg->nvar, tma, c->LF, err)) {
      delete c;
      return fail(nullptr, PSSO_E_UNSUPPORTED, err);
    }
  }
  c->tile_fn = tile_kernel(cfg->dtype, cfg->rng_mode, cfg->fn_id, c->L.V, false);
  c->fused_fn = tile_kernel(cfg->dtype, cfg->rng_mode, cfg->fn_id, c->L.V, true);
  c->init_fn = c->tile_fn;
  c->chain = false;
  {  // register-resident chain kernel: one pairwise leaf of position-local terms
    const int64_t D = cfg->nvar;
    const int M = D <= 32 ? 4 : D <= 64 ? 8 : D <= 128 ? 16 : 0;
    const char* off = std::getenv("PSSO_NO_CHAIN");
    // the chain kernel's branch-free trig (psso_trig.cuh) is valid for
    // positions in a box of moderate size; wider boxes take the tile kernels
    const double box = std::max(std::fabs(cfg->var_min), std::fabs(cfg->var_max));
    const bool trig_ok = box <= (cfg->dtype == PSSO_F64 ? kChainTrigMaxAbs : kChainTrigMaxAbsF32);
    if (M && terms_of(cfg->fn_id, D) <= 128 && trig_ok && !(off && *off && *off != '0')) {
      const bool full = D == 8 * M;
      const void* f = chain_kernel(cfg->dtype, cfg->rng_mode, cfg->fn_id, M, false, full);
      const void* i = chain_kernel(cfg->dtype, cfg->rng_mode, cfg->fn_id, M, true, false);
      if (f && i) {
        c->fused_fn = f;
        c->init_fn = i;
        c->chain = true;
        const int es = cfg->dtype == PSSO_F64 ? 8 : 4;
        // gbest | warp reduction + xs30(gamma*(j+1)) table | per-warp mbarriers |
        // per-warp prefetch buffers (FULL iteration kernel, psso_device.cuh)
        // | per-warp smem rows (f3, f7, f8)
        const int nw = PSSO_CHAIN_NT / 32;
        const bool smem_fn = cfg->fn_id == 3 || cfg->fn_id == 7 || cfg->fn_id == 8;
        // (gbest padded to 8M entries: rows shorter than 8M read, and discard,
        // gbest past D in the branch-free select)
        c->LF.off_red = (int)align16((size_t)8 * M * es);
        c->LF.off_bar = (int)align16((size_t)c->LF.off_red + 128 + 64 * M);
        c->LF.off_xs = (int)((c->LF.off_bar + 16 * nw + 127) & ~127);  // two mbarriers per warp
        const bool db = PSSO_CHAIN_DB && 8 * M * es <= 512;  // chain_db<T, M>()
        c->LF.off_scr = (int)align16((size_t)c->LF.off_xs +
                                     (full && PSSO_CHAIN_PF ? (size_t)nw * (db ? 2 : 1) * 8 *
                                      host_row_stride(es, M) : 0));
        c->LF.smem = (size_t)c->LF.off_scr + (smem_fn ? (size_t)nw * 4 * (8 * M) * es : 0);
        c->init_smem = c->LF.smem;
      }
    }
  }
  c->rows_w = 0;
  {  // long rows (C5): D = 512*W, a balanced tree of 4W leaves -> k_rows
    const int64_t D = cfg->nvar;
    const int W = D == 512 ? 1 : D == 1024 ? 2 : D == 2048 ? 4 : D == 4096 ? 8 : 0;
    const char* off = std::getenv("PSSO_NO_ROWS");
    const double box = std::max(std::fabs(cfg->var_min), std::fabs(cfg->var_max));
    const bool trig_ok = box <= (cfg->dtype == PSSO_F64 ? kChainTrigMaxAbs : kChainTrigMaxAbsF32);
    const void* f = W && trig_ok && !(off && *off && *off != '0')
                        ? rows_kernel(cfg->dtype, cfg->rng_mode, cfg->fn_id, W) : nullptr;
    if (f) {
      c->fused_fn = f;
      c->rows_w = W;
      const int es = cfg->dtype == PSSO_F64 ? 8 : 4;
      // gbest | warp reduction | leaf values | mbarriers | prefetch buffers
      c->LF.off_red = PSSO_ROWS_JIT ? 0 : (int)align16((size_t)(D + D / 16) * es);  // gbest padded per leaf
      c->LF.off_leaf = c->LF.off_red + 128;  // leaf values [2][8/W][2*4W + 1] doubles
      c->LF.off_flag = c->LF.off_leaf + (int)align16(2 * (size_t)(8 / W) * (8 * W + 1) * 8);
      c->LF.off_bar = (int)align16((size_t)c->LF.off_flag + 64);  // flags [2][8/W] ints
      c->LF.off_xs = (int)((c->LF.off_bar + 64 + 127) & ~127);
      c->LF.smem = (size_t)c->LF.off_xs + 8 * 8 * host_row_stride(es, 16);
    }
  }
  if (!c->tile_fn || !c->fused_fn) {
    delete c;
    return fail(nullptr, PSSO_E_UNSUPPORTED, "no kernel instantiation for this configuration");
  }
  cudaError_t e;
  if ((e = cudaGetDevice(&c->device)) != cudaSuccess ||
      (e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device)) != cudaSuccess ||
      (e = allow_smem(c->tile_fn, c->L.smem)) != cudaSuccess ||
      (e = allow_smem(c->fused_fn, c->LF.smem)) != cudaSuccess ||
      (c->chain && (e = allow_smem(c->init_fn, c->init_smem)) != cudaSuccess)) {
    delete c;
    return cuda_fail(nullptr, e, "psso_create");
  }
  int per_sm = 0, per_sm_fused = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, c->tile_fn, NT, c->L.smem)) != cudaSuccess ||
      (e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_fused, c->fused_fn, NT, c->LF.smem)) != cudaSuccess ||
      per_sm < 1 || per_sm_fused < 1) {
    delete c;
    return e != cudaSuccess ? cuda_fail(nullptr, e, "occupancy") : fail(nullptr, PSSO_E_UNSUPPORTED, "tile kernel cannot be resident");
  }
  const int64_t rows = cfg->row_hi - cfg->row_lo;
  const int64_t ntiles = (rows + c->L.R - 1) / c->L.R;
  c->grid = (int)std::min<int64_t>(ntiles, (int64_t)per_sm * c->num_sms);
  const int64_t ntiles_f = (rows + c->LF.R - 1) / c->LF.R;
  c->fused_grid = (int)std::min<int64_t>(ntiles_f, (int64_t)per_sm_fused * c->num_sms);
  c->init_grid = c->grid;
  if (c->chain) {  // 4 particles per warp, 8 warps per CTA
    int per_sm_init = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_init, c->init_fn, NT, c->init_smem)) != cudaSuccess ||
        per_sm_init < 1) {
      delete c;
      return e != cudaSuccess ? cuda_fail(nullptr, e, "occupancy") : fail(nullptr, PSSO_E_UNSUPPORTED, "chain kernel cannot be resident");
    }
    const int64_t nctas = (rows + 4 * (NT / 32) - 1) / (4 * (NT / 32));
    int sms = c->num_sms;  // PSSO_FUSED_SMS (diagnostic): persistent grid over fewer SMs
    if (const char* f = std::getenv("PSSO_FUSED_SMS"))
      if (*f) sms = std::max(1, std::min(c->num_sms, std::atoi(f)));
    c->fused_grid = (int)std::min<int64_t>(nctas, (int64_t)per_sm_fused * sms);
    c->init_grid = (int)std::min<int64_t>(nctas, (int64_t)per_sm_init * c->num_sms);
  }
  if (c->rows_w) {  // 8 / W rows per CTA round
    const int rpc = 8 / c->rows_w;
    c->fused_grid = (int)std::min<int64_t>((rows + rpc - 1) / rpc, (int64_t)per_sm_fused * c->num_sms);
  }
  c->swarm_fn = nullptr;
  if (c->chain && cfg->row_lo == 0 && cfg->row_hi == cfg->nsol &&
      rows * cfg->nvar <= PSSO_SWARM_MAX_ELEMS) {  // small swarm: the whole run in one launch
    const char* off = std::getenv("PSSO_NO_SWARM");
    SwarmPlan sp;
    if (!(off && *off && *off != '0')) {
      if (!plan_swarm(c, 1, sp, e) && e != cudaSuccess) {
        delete c;
        return cuda_fail(nullptr, e, "psso_create swarm kernel");
      }
      // measured (scripts/swarm_crossover.py): the whole-run kernel beats the
      // graph-replayed streaming kernels only in its cluster form with at most
      // one row group per warp (C1, C2); the global-exchange forms are slower
      // and serve batches of many swarms (psso_solve_batch) only
      if (sp.fn && sp.cl && sp.gpc <= PSSO_SWARM_NT / 32) {
        c->swarm_fn = sp.fn;
        c->swarm = sp;
      }
    }
  }
  {
    const char* tn = cfg->dtype == PSSO_F64 ? "double" : "float";
    const char* rn = cfg->rng_mode == PSSO_RNG_REFERENCE ? "ref" : "philox";
    const int64_t D = cfg->nvar;
    const int M = D <= 32 ? 4 : D <= 64 ? 8 : 16;
    char b[160];
    if (c->swarm_fn)
      std::snprintf(b, sizeof b, "k_swarm<%s,f%d,%s,M=%d%s> x%d CTAs", tn, cfg->fn_id, rn, M,
                    c->swarm.cl ? ",cluster" : c->swarm.res ? ",smem-resident" : "", c->swarm.G);
    else if (c->rows_w)
      std::snprintf(b, sizeof b, "k_rows<%s,f%d,%s,W=%d>", tn, cfg->fn_id, rn, c->rows_w);
    else if (c->chain)
      std::snprintf(b, sizeof b, "k_chain<%s,f%d,%s,M=%d%s>", tn, cfg->fn_id, rn, M, D == 8 * M ? ",full" : "");
    else
      std::snprintf(b, sizeof b, "%s<%s,f%d,%s>", c->LF.V > 1 ? "k_fused" : "k_tile", tn, cfg->fn_id, rn);
    c->kname = b;
  }
  c->argmin_grid = (int)std::min<int64_t>((rows + 255) / 256, 4 * c->num_sms);
  c->nslots = std::max(std::max(std::max(c->grid, c->fused_grid), c->init_grid), c->argmin_grid);
  c->Kw = k53(cfg->cw); c->Kp = k53(cfg->cp); c->Kg = k53(cfg->cg);
  c->Kw32 = k32(cfg->cw); c->Kp32 = k32(cfg->cp); c->Kg32 = k32(cfg->cg);
  c->aux = nullptr;
  if ((e = cudaMalloc(&c->slot_f, sizeof(double) * c->nslots)) != cudaSuccess ||
      (e = cudaMalloc(&c->slot_i, sizeof(int64_t) * c->nslots)) != cudaSuccess ||
      (e = cudaMalloc(&c->bad, sizeof(unsigned long long))) != cudaSuccess ||
      (e = cudaMalloc(&c->t_dev, sizeof(int64_t))) != cudaSuccess ||
      (e = cudaMalloc(&c->g_idx, sizeof(int64_t))) != cudaSuccess ||
      (e = cudaMalloc(&c->bad_val, sizeof(double))) != cudaSuccess ||
      (e = cudaMalloc(&c->stats, 3 * STATS_CAP * sizeof(unsigned long long))) != cudaSuccess ||
      (e = cudaMemset(c->g_idx, 0xff, sizeof(int64_t))) != cudaSuccess ||
      (e = cudaMemset(c->bad, 0xff, sizeof(unsigned long long))) != cudaSuccess) {
    psso_destroy(c);
    return cuda_fail(nullptr, e, "psso_create alloc");
  }
  {
    std::vector<unsigned long long> st(3 * STATS_CAP, 0ull);
    for (int q = 0; q < STATS_CAP; ++q) st[3 * q] = ~0ull;
    if ((e = cudaMemcpy(c->stats, st.data(), st.size() * 8, cudaMemcpyHostToDevice)) != cudaSuccess) {
      psso_destroy(c);
      return cuda_fail(nullptr, e, "psso_create stats");
    }
  }
  if (c->swarm_fn) {
    const size_t es = cfg->dtype == PSSO_F64 ? 8 : 4;
    const size_t G = (size_t)c->swarm.G;
    const uint64_t seed = cfg->seed;
    if ((e = cudaMalloc(&c->sw_epoch, 2 * G * sizeof(unsigned int))) != cudaSuccess ||
        (e = cudaMalloc(&c->sw_slot_f, 2 * G * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&c->sw_slot_i, 2 * G * sizeof(int64_t))) != cudaSuccess ||
        (e = cudaMalloc(&c->sw_slot_new, 2 * G * sizeof(int32_t))) != cudaSuccess ||
        (e = cudaMalloc(&c->sw_slot_row, 2 * G * (size_t)cfg->nvar * es)) != cudaSuccess ||
        (e = cudaMalloc(&c->sw_seed, sizeof(uint64_t))) != cudaSuccess ||
        (e = cudaMemcpy(c->sw_seed, &seed, sizeof seed, cudaMemcpyHostToDevice)) != cudaSuccess) {
      psso_destroy(c);
      return cuda_fail(nullptr, e, "psso_create swarm buffers");
    }
  }
  if (cfg->fn_id == 7) {
    if ((e = cudaMalloc(&c->aux, sizeof(double) * cfg->nvar)) != cudaSuccess) {
      psso_destroy(c);
      return cuda_fail(nullptr, e, "psso_create aux");
    }
    // 1.0 / np.sqrt(np.arange(1, D+1)) (benchmarks.py:216): IEEE sqrt and division
    // are correctly rounded on host and device alike; copied, not computed on the
    // device, so context creation never synchronizes the whole device
    std::vector<double> inv((size_t)cfg->nvar);
    for (int64_t j = 0; j < cfg->nvar; ++j) inv[(size_t)j] = 1.0 / std::sqrt((double)(j + 1));
    if ((e = cudaMemcpy(c->aux, inv.data(), inv.size() * sizeof(double), cudaMemcpyHostToDevice)) !=
        cudaSuccess) {
      psso_destroy(c);
      return cuda_fail(nullptr, e, "psso_create aux init");
    }
  }
  *out = c;
  return PSSO_OK;
}

void psso_destroy(psso_ctx* c) {
  if (!c) return;
  DEV_GUARD(c);
  if (c->graph) cudaGraphExecDestroy(c->graph);
  if (c->sgraph) cudaGraphExecDestroy(c->sgraph);
  if (c->pgraph) cudaGraphExecDestroy(c->pgraph);
  if (c->comm && c->stream) cudaStreamSynchronize(c->stream);  // the communicator is borrowed
  cudaFree(c->cand);
  cudaFree(c->gathered);
  for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
  cudaFree(c->slot_f);
  cudaFree(c->slot_i);
  cudaFree(c->bad);
  cudaFree(c->t_dev);
  cudaFree(c->g_idx);
  cudaFree(c->bad_val);
  cudaFree(c->stats);
  cudaFree(c->aux);
  cudaFree(c->sw_epoch);
  cudaFree(c->sw_slot_new);
  cudaFree(c->sw_slot_f);
  cudaFree(c->sw_slot_i);
  cudaFree(c->sw_slot_row);
  cudaFree(c->sw_seed);
  cudaFree(c->seq_xn);
  cudaFree(c->seq_fn);
  cudaFree(c->seq_pfn);
  cudaFree(c->seq_seed);
  cudaFree(c->seq_passes);
  cudaFree(c->seq_ctl);
  if (c->seq_ctl_host) cudaFreeHost(c->seq_ctl_host);
  delete c;
}

int psso_bind(psso_ctx* c, const psso_buffers* b, void* stream) {
  DEV_GUARD(c);
  if (!c) return fail(nullptr, PSSO_E_INVALID, "null context");
  if (!b || !b->sol || !b->pbests || !b->p_f || !b->gbest || !b->g_f)
    return fail(c, PSSO_E_INVALID, "sol, pbests, p_f, gbest and g_f buffers are required");
  const uintptr_t al = 16;
  if (((uintptr_t)b->sol | (uintptr_t)b->pbests | (uintptr_t)b->gbest) % al)
    return fail(c, PSSO_E_INVALID, "position buffers must be 16-byte aligned");
  c->buf = *b;
  c->stream = (cudaStream_t)stream;
  c->bound = true;
  if (c->graph) { cudaGraphExecDestroy(c->graph); c->graph = nullptr; }
  if (c->sgraph) { cudaGraphExecDestroy(c->sgraph); c->sgraph = nullptr; }
  if (c->pgraph) { cudaGraphExecDestroy(c->pgraph); c->pgraph = nullptr; }
  return PSSO_OK;
}

// initialization kernel: positions from the INIT stream, fitness, candidates
static int launch_init(psso_ctx* c) {
  if (!c->chain) return launch_tile(c, tile_params(c, M_INIT | M_EVAL | M_CAND | M_SOLF, -1, nullptr));
  TileParams p = tile_params(c, M_INIT | M_EVAL | M_CAND | M_SOLF, -1, nullptr, true);
  void* args[] = {(void*)&p};
  CK(c, cudaLaunchKernel(c->init_fn, dim3(c->init_grid), dim3(NT), args, c->init_smem, c->stream));
  c->launches++;
  return PSSO_OK;
}

// The loop's CUDA graph (GRAPH_CHUNK fused iterations, t read from t_dev),
// captured once per binding.  psso_init captures it already, so host-side
// capture never lands inside a timed loop (the reference's timer starts
// after initialize, parallel.py:190).
static int ensure_graph(psso_ctx* c) {
  if (c->graph || c->swarm_fn || c->stream == nullptr) return PSSO_OK;
  cudaGraph_t g;
  CK(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  const int64_t saved = c->launches;
  for (int k = 0; k < GRAPH_CHUNK; ++k) {
    int rc = fused_step(c, 0, c->t_dev);
    if (rc) { cudaStreamEndCapture(c->stream, &g); return rc; }
  }
  c->launches = saved;
  CK(c, cudaStreamEndCapture(c->stream, &g));
  cudaError_t e = cudaGraphInstantiate(&c->graph, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaGraphInstantiate");
  return PSSO_OK;
}

int psso_init(psso_ctx* c) {
  DEV_GUARD(c);
  TRACE("psso_init");
  if (int rc = need_bound(c)) return rc;
  k_set_u64<<<1, 1, 0, c->stream>>>(c->bad, ~0ull);
  c->launches++;
  int rc = launch_init(c);
  if (rc) return rc;
  GbParams g = gb_params(c, -1, nullptr, 1, c->chain ? c->init_grid : c->grid);
  g.traj = nullptr;
  if ((rc = launch_gbest(c, g))) return rc;
  return c->profiling ? PSSO_OK : ensure_graph(c);
}

int psso_step(psso_ctx* c, int64_t t) {
  DEV_GUARD(c);
  TRACE("psso_step");
  if (int rc = need_bound(c)) return rc;
  if (t < 0) return fail(c, PSSO_E_INVALID, "iteration must be >= 0");
  return fused_step(c, t, nullptr);
}

// the whole loop as one k_swarm launch (small swarms)
static int swarm_run(psso_ctx* c, int64_t t0, int64_t niter) {
  TileParams p = tile_params(c, fused_mode(c), t0, nullptr, true);
  p.off_bar = c->swarm.off_bar;
  p.off_scr = c->swarm.off_scr;
  p.off_leaf = c->swarm.off_pub;
  p.off_xs = c->swarm.off_xs;
  SwarmParams sp;
  std::memset(&sp, 0, sizeof sp);
  sp.t0 = t0;
  sp.niter = niter;
  sp.rows = c->cfg.row_hi - c->cfg.row_lo;
  sp.G = c->swarm.G;
  sp.gpc = c->swarm.gpc;
  sp.do_init = 0;
  sp.epoch = c->sw_epoch;
  sp.slot_f = c->sw_slot_f;
  sp.slot_i = c->sw_slot_i;
  sp.slot_new = c->sw_slot_new;
  sp.slot_row = c->sw_slot_row;
  sp.traj = c->buf.traj;
  sp.traj_stride = 0;
  sp.g_f = c->buf.g_f;
  sp.g_idx = c->g_idx;
  sp.gbest = c->buf.gbest;
  sp.seeds = c->sw_seed;
  sp.sol_f = c->buf.sol_f;
  sp.bad = c->bad;
  CK(c, cudaMemsetAsync(c->sw_epoch, 0, 2 * (size_t)c->swarm.G * sizeof(unsigned int), c->stream));
  const bool timed = c->profiling;
  if (timed) {
    if (c->ev_used + 2 > c->ev.size()) {
      for (int k = 0; k < 8; ++k) {
        cudaEvent_t e;
        CK(c, cudaEventCreate(&e));
        c->ev.push_back(e);
      }
    }
    CK(c, cudaEventRecord(c->ev[c->ev_used], c->stream));
  }
#if PSSO_SWARM_TRACE
  unsigned long long* trace = nullptr;
  CK(c, cudaMalloc(&trace, (size_t)niter * 4 * sizeof(unsigned long long)));
  sp.trace = trace;
#endif
  void* args[] = {(void*)&p, (void*)&sp};
  CK(c, launch_swarm(c->swarm, 1, args, c->stream));
  c->launches++;
#if PSSO_SWARM_TRACE
  {  // phase breakdown of CTA 0 (diagnostic builds only)
    std::vector<unsigned long long> h((size_t)niter * 4);
    CK(c, cudaStreamSynchronize(c->stream));
    CK(c, cudaMemcpy(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost));
    cudaFree(trace);
    double ph[3] = {0, 0, 0}, tot = 0;
    for (int64_t i = 0; i < niter; ++i) {
      for (int k = 0; k < 3; ++k) ph[k] += (double)(h[i * 4 + k + 1] - h[i * 4 + k]);
      tot += (double)(h[i * 4 + 3] - h[i * 4]);
    }
    std::fprintf(stderr, "[swarm trace] G=%d niter=%lld per iteration (ns): compute+publish %.0f  wait %.0f  "
                 "take+sync %.0f  total %.0f\n", c->swarm.G, (long long)niter, ph[0] / niter, ph[1] / niter,
                 ph[2] / niter, tot / niter);
  }
#endif
  if (timed) {
    CK(c, cudaEventRecord(c->ev[c->ev_used + 1], c->stream));
    c->ev_used += 2;
    c->prof_iters += niter;
  }
  return PSSO_OK;
}

int psso_run(psso_ctx* c, int64_t t0, int64_t niter) {
  DEV_GUARD(c);
  TRACE("psso_run");
  if (int rc = need_bound(c)) return rc;
  if (t0 < 0 || niter < 0) return fail(c, PSSO_E_INVALID, "t0 and niter must be >= 0");
  if (niter == 0) return PSSO_OK;
  if (c->swarm_fn) return swarm_run(c, t0, niter);
  int64_t done = 0;
  if (c->stream != nullptr && niter >= GRAPH_CHUNK && !c->profiling) {
    if (int rc = ensure_graph(c)) return rc;
    k_set<<<1, 1, 0, c->stream>>>(c->t_dev, t0);
    c->launches++;
    for (; done + GRAPH_CHUNK <= niter; done += GRAPH_CHUNK) {
      CK(c, cudaGraphLaunch(c->graph, c->stream));
      c->launches += 2 * GRAPH_CHUNK;
    }
  }
  for (; done < niter; ++done) {
    int rc = fused_step(c, t0 + done, nullptr);
    if (rc) return rc;
  }
  return PSSO_OK;
}

// k_seq launch for B swarms stacked along the row axis (psso_seq.cuh layout):
// one cluster of G CTAs per swarm, G = ceil(rows / 64) up to 16: about one
// row group per warp, which beats fewer CTAs with more groups per warp even
// at C1 (100 rows: G = 2 6.2 ms, G = 1 9.6 ms per 1000 iterations);
// PSSO_SEQ_G overrides.  Rows are split in blocks of rpc.
static cudaError_t launch_seq(psso_ctx* c, int M, SeqParams q, int64_t B, cudaStream_t s) {
  const psso_config* cfg = &c->cfg;
  const int es = cfg->dtype == PSSO_F64 ? 8 : 4;
  const int nw = PSSO_SEQ_NT / 32;
  const bool smem_fn = cfg->fn_id == 3 || cfg->fn_id == 7 || cfg->fn_id == 8;
  int64_t G = std::max<int64_t>(1, std::min<int64_t>(16, (q.rows + 63) / 64));
  if (const char* g = std::getenv("PSSO_SEQ_G"))
    if (*g) G = std::max<int64_t>(1, std::min<int64_t>(16, std::atoll(g)));
  q.rpc = ((q.rows + G - 1) / G + 3) / 4 * 4;
  G = (q.rows + q.rpc - 1) / q.rpc;
  TileParams p = tile_params(c, M_SOLF, q.t0, nullptr, false);
  p.off_red = (int)align16((size_t)8 * M * es);
  p.off_bar = (int)align16((size_t)p.off_red + 16 * nw + 64 * M);
  p.off_scr = (int)align16((size_t)p.off_bar + 8 * (nw + 2));
  p.off_leaf = (int)align16((size_t)p.off_scr + (smem_fn ? (size_t)nw * 4 * (8 * M) * es : 0));
  size_t smem = (size_t)p.off_leaf + 32 + 2 * (size_t)cfg->nvar * es;
  // RES: the CTA's rows (X, P, speculative rows, p_f, fitness) resident in
  // shared memory when they fit (C2 shape: 64 rows x 100), else global memory
  p.off_xs = (int)align16(smem);
  const size_t smem_res = (size_t)p.off_xs + 3 * (size_t)q.rpc * cfg->nvar * es + 16 * (size_t)q.rpc;
  const char* nr = std::getenv("PSSO_SEQ_NO_RES");
  const bool res = smem_res <= 227 * 1024 && !(nr && *nr && *nr != '0');
  if (res) smem = smem_res;
  const void* f = seq_kernel(cfg->dtype, cfg->rng_mode, cfg->fn_id, M, res);
  if (!f) return cudaErrorInvalidDeviceFunction;
  cudaError_t e = allow_smem(f, smem);
  if (e == cudaSuccess && G > 8) e = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t lc = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.gridDim = dim3((unsigned)G, (unsigned)B, 1);
  lc.blockDim = dim3(PSSO_SEQ_NT, 1, 1);
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  lc.attrs = at;
  lc.numAttrs = 1;
  void* args[] = {(void*)&p, (void*)&q};
  e = cudaLaunchKernelExC(&lc, f, args);
  if (e == cudaSuccess) c->launches++;
  return e;
}

// run_sequential (core.py:213-258): one k_seq launch for the whole loop
// (speculative passes with rollback, psso_seq.cuh).
// run_sequential (core.py:222-244) for rows the chain mapping does not take
// (nvar > 128): per iteration, speculative passes until the swarm's end --
// every remaining row searched and evaluated against the current gbest into
// scratch (X -> Xn copy, then the tile kernel's search + evaluate on Xn; the
// non-finite flag is not touched speculatively), the first event found,
// rows up to it committed, gbest moved -- all on the device; the host reads
// back 16 bytes per pass (where the next pass starts, whether the run failed).
// Bit-identical to the serial loop for the same reason as k_seq.
static int run_sequential_rows(psso_ctx* c, int64_t t0, int64_t niter) {
  const psso_config* cfg = &c->cfg;
  const int64_t N = cfg->nsol, D = cfg->nvar;
  const int es = cfg->dtype == PSSO_F64 ? 8 : 4;
  if (!c->seq_xn) {
    CK(c, cudaMalloc(&c->seq_xn, (size_t)N * D * es));
    CK(c, cudaMalloc(&c->seq_fn, (size_t)N * sizeof(double)));
    CK(c, cudaMalloc(&c->seq_passes, sizeof(int64_t)));
    CK(c, cudaMemset(c->seq_passes, 0, sizeof(int64_t)));
  }
  if (!c->seq_ctl) {
    CK(c, cudaMalloc(&c->seq_ctl, 4 * sizeof(int64_t)));
    CK(c, cudaMallocHost(&c->seq_ctl_host, 4 * sizeof(int64_t)));
  }
  {  // a run that already failed stays stopped (like the kernels' early exit)
    unsigned long long key = ~0ull;
    CK(c, cudaMemcpyAsync(&key, c->bad, sizeof key, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    if (key != ~0ull) return PSSO_OK;
  }
  CK(c, cudaMemsetAsync(c->seq_passes, 0, sizeof(int64_t), c->stream));
  CK(c, cudaMemsetAsync(c->seq_ctl, 0, 4 * sizeof(int64_t), c->stream));
  const int commit_grid = (int)std::min<int64_t>(N, 8 * c->num_sms);
  unsigned char* X = (unsigned char*)c->buf.sol;
  unsigned char* Xn = (unsigned char*)c->seq_xn;
  for (int64_t t = t0; t < t0 + niter; ++t) {
    int64_t lo = 0;
    k_set<<<1, 1, 0, c->stream>>>(c->seq_ctl, 0);
    c->launches++;
    while (lo < N) {
      const int64_t a = lo - lo % 4;  // 16-byte aligned first row for any nvar / dtype
      CK(c, cudaMemcpyAsync(Xn + (size_t)a * D * es, X + (size_t)a * D * es, (size_t)(N - a) * D * es,
                            cudaMemcpyDeviceToDevice, c->stream));
      TileParams p = tile_params(c, M_SEARCH | M_EVAL | M_SOLF, t, nullptr, false);
      p.X = Xn + (size_t)a * D * es;
      p.P = (unsigned char*)c->buf.pbests + (size_t)a * D * es;
      p.p_f = c->buf.p_f + a;
      p.sol_f = c->seq_fn + a;
      p.rows = N - a;
      p.row_lo = a;
      p.bad = nullptr;  // speculative: a non-finite row counts only if it is the first event
      if (int rc = launch_tile(c, p)) return rc;
      k_seq_event<<<1, 1024, 0, c->stream>>>(c->seq_fn, c->buf.p_f, c->buf.g_f, c->seq_ctl, N);
      if (cfg->dtype == PSSO_F64) {
        k_seq_commit<double><<<commit_grid, 256, 0, c->stream>>>((double*)c->buf.sol, (double*)c->buf.pbests,
            (const double*)c->seq_xn, c->seq_fn, c->buf.p_f, c->buf.sol_f, c->seq_ctl, N, (int)D);
        k_seq_move<double><<<1, 256, 0, c->stream>>>((double*)c->buf.gbest, (const double*)c->seq_xn,
            c->seq_fn, c->buf.g_f, c->g_idx, c->bad, c->buf.traj, t, c->seq_ctl, c->seq_passes, N, (int)D);
      } else {
        k_seq_commit<float><<<commit_grid, 256, 0, c->stream>>>((float*)c->buf.sol, (float*)c->buf.pbests,
            (const float*)c->seq_xn, c->seq_fn, c->buf.p_f, c->buf.sol_f, c->seq_ctl, N, (int)D);
        k_seq_move<float><<<1, 256, 0, c->stream>>>((float*)c->buf.gbest, (const float*)c->seq_xn,
            c->seq_fn, c->buf.g_f, c->g_idx, c->bad, c->buf.traj, t, c->seq_ctl, c->seq_passes, N, (int)D);
      }
      c->launches += 3;
      CK(c, cudaGetLastError());
      CK(c, cudaMemcpyAsync(c->seq_ctl_host, c->seq_ctl, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost,
                            c->stream));
      CK(c, cudaStreamSynchronize(c->stream));
      if (c->seq_ctl_host[2]) return PSSO_OK;  // non-finite: reported by psso_check
      lo = c->seq_ctl_host[0];
    }
  }
  return PSSO_OK;
}

int psso_run_sequential(psso_ctx* c, int64_t t0, int64_t niter) {
  DEV_GUARD(c);
  TRACE("psso_run_sequential");
  if (int rc = need_bound(c)) return rc;
  if (t0 < 0 || niter < 0) return fail(c, PSSO_E_INVALID, "t0 and niter must be >= 0");
  const psso_config* cfg = &c->cfg;
  if (cfg->row_lo != 0 || cfg->row_hi != cfg->nsol)
    return fail(c, PSSO_E_INVALID, "the sequential schedule runs unsharded swarms only");
  if (!c->chain) return run_sequential_rows(c, t0, niter);
  const int64_t rows = cfg->nsol, D = cfg->nvar;
  const int M = D <= 32 ? 4 : D <= 64 ? 8 : 16;
  const int es = cfg->dtype == PSSO_F64 ? 8 : 4;
  if (!seq_kernel(cfg->dtype, cfg->rng_mode, cfg->fn_id, M, false))
    return fail(c, PSSO_E_UNSUPPORTED, "no sequential kernel for this configuration");
  if (!c->seq_xn) {
    const uint64_t seed = cfg->seed;
    CK(c, cudaMalloc(&c->seq_xn, (size_t)rows * D * es));
    CK(c, cudaMalloc(&c->seq_fn, (size_t)rows * sizeof(double)));
    CK(c, cudaMalloc(&c->seq_pfn, (size_t)rows * sizeof(double)));
    CK(c, cudaMalloc(&c->seq_seed, sizeof(uint64_t)));
    CK(c, cudaMalloc(&c->seq_passes, sizeof(int64_t)));
    CK(c, cudaMemcpy(c->seq_seed, &seed, sizeof seed, cudaMemcpyHostToDevice));
    CK(c, cudaMemset(c->seq_passes, 0, sizeof(int64_t)));
  }
  if (niter == 0) return PSSO_OK;
  SeqParams q;
  std::memset(&q, 0, sizeof q);
  q.t0 = t0;
  q.niter = niter;
  q.rows = rows;
  q.Xn = c->seq_xn;
  q.fn = c->seq_fn;
  q.pfn = c->seq_pfn;
  q.traj = c->buf.traj;
  q.traj_stride = 0;
  q.g_f = c->buf.g_f;
  q.g_idx = c->g_idx;
  q.gbest = c->buf.gbest;
  q.seeds = c->seq_seed;
  q.sol_f = c->buf.sol_f;
  q.bad = c->bad;
  q.passes = c->seq_passes;
  CK(c, launch_seq(c, M, q, 1, c->stream));
  return PSSO_OK;
}

int psso_sequential_passes(psso_ctx* c, int64_t* passes) {
  DEV_GUARD(c);
  if (!c || !passes) return fail(c, PSSO_E_INVALID, "null argument");
  *passes = 0;
  if (!c->seq_passes) return PSSO_OK;
  CK(c, cudaStreamSynchronize(c->stream));
  CK(c, cudaMemcpy(passes, c->seq_passes, sizeof(int64_t), cudaMemcpyDeviceToHost));
  return PSSO_OK;
}

int psso_search(psso_ctx* c, int64_t t) {
  DEV_GUARD(c);
  TRACE("psso_search");
  if (int rc = need_bound(c)) return rc;
  return launch_tile(c, tile_params(c, M_SEARCH, t, nullptr));
}

int psso_evaluate(psso_ctx* c, int64_t t) {
  DEV_GUARD(c);
  TRACE("psso_evaluate");
  if (int rc = need_bound(c)) return rc;
  if (!c->buf.sol_f) return fail(c, PSSO_E_INVALID, "evaluate needs a sol_f buffer");
  return launch_tile(c, tile_params(c, M_LOAD | M_EVAL | M_SOLF, t < 0 ? -1 : t, nullptr));
}

int psso_update_pbests(psso_ctx* c) {
  DEV_GUARD(c);
  TRACE("psso_update_pbests");
  if (int rc = need_bound(c)) return rc;
  if (!c->buf.sol_f) return fail(c, PSSO_E_INVALID, "update_pbests needs a sol_f buffer");
  const int64_t rows = c->cfg.row_hi - c->cfg.row_lo;
  const int grid = (int)std::min<int64_t>(rows, 8 * c->num_sms);
  if (c->cfg.dtype == PSSO_F64)
    k_pbest<double><<<grid, 128, 0, c->stream>>>((const double*)c->buf.sol, (double*)c->buf.pbests,
                                                 c->buf.sol_f, c->buf.p_f, rows, (int)c->cfg.nvar);
  else
    k_pbest<float><<<grid, 128, 0, c->stream>>>((const float*)c->buf.sol, (float*)c->buf.pbests,
                                                c->buf.sol_f, c->buf.p_f, rows, (int)c->cfg.nvar);
  c->launches++;
  CK(c, cudaGetLastError());
  return PSSO_OK;
}

int psso_update_gbest(psso_ctx* c) {
  DEV_GUARD(c);
  TRACE("psso_update_gbest");
  if (int rc = need_bound(c)) return rc;
  const int64_t rows = c->cfg.row_hi - c->cfg.row_lo;
  k_argmin<<<c->argmin_grid, 256, 0, c->stream>>>(c->buf.p_f, rows, c->cfg.row_lo, c->slot_f, c->slot_i);
  c->launches++;
  CK(c, cudaGetLastError());
  GbParams g = gb_params(c, -1, nullptr, 0, c->argmin_grid);
  g.traj = nullptr;
  return launch_gbest(c, g);
}

int64_t psso_candidate_bytes(const psso_config* cfg) {
  if (!cfg) return -1;
  const int64_t es = cfg->dtype == PSSO_F64 ? 8 : 4;
  return REC_HDR + ((cfg->nvar * es + 15) / 16) * 16;
}

static int local_cand(psso_ctx* c, void* cand, int nslots) {
  GbParams g = gb_params(c, -1, nullptr, 0, nslots);
  unsigned char* rec = (unsigned char*)cand;
  if (c->cfg.dtype == PSSO_F64)
    k_local_cand<double><<<1, GB_THREADS, 0, c->stream>>>(g, rec);
  else
    k_local_cand<float><<<1, GB_THREADS, 0, c->stream>>>(g, rec);
  c->launches++;
  CK(c, cudaGetLastError());
  return PSSO_OK;
}

int psso_init_local(psso_ctx* c, void* cand) {
  DEV_GUARD(c);
  TRACE("psso_init_local");
  if (int rc = need_bound(c)) return rc;
  if (!cand) return fail(c, PSSO_E_INVALID, "null candidate buffer");
  k_set_u64<<<1, 1, 0, c->stream>>>(c->bad, ~0ull);
  c->launches++;
  int rc = launch_init(c);
  if (rc) return rc;
  return local_cand(c, cand, c->chain ? c->init_grid : c->grid);
}

int psso_step_local(psso_ctx* c, int64_t t, void* cand) {
  DEV_GUARD(c);
  TRACE("psso_step_local");
  if (int rc = need_bound(c)) return rc;
  if (!cand) return fail(c, PSSO_E_INVALID, "null candidate buffer");
  if (int rc = launch_fused(c, t, nullptr)) return rc;
  return local_cand(c, cand, c->fused_grid);
}

int psso_apply_candidates(psso_ctx* c, int64_t t, const void* cands, int32_t ncand, int32_t is_init) {
  DEV_GUARD(c);
  TRACE("psso_apply_candidates");
  if (int rc = need_bound(c)) return rc;
  if (!cands || ncand < 1) return fail(c, PSSO_E_INVALID, "need at least one candidate record");
  GbParams g = gb_params(c, t, nullptr, is_init, 0);
  if (is_init) g.traj = nullptr;
  const int64_t rb = psso_candidate_bytes(&c->cfg);
  if (c->cfg.dtype == PSSO_F64)
    k_apply<double><<<1, GB_THREADS, 0, c->stream>>>(g, (const unsigned char*)cands, rb, ncand);
  else
    k_apply<float><<<1, GB_THREADS, 0, c->stream>>>(g, (const unsigned char*)cands, rb, ncand);
  c->launches++;
  CK(c, cudaGetLastError());
  return PSSO_OK;
}

// ---- sharded iteration over a library-owned NCCL communicator -----------
int psso_nccl_unique_id(void* id) {
  if (!id) return fail(nullptr, PSSO_E_INVALID, "null id buffer");
  const NcclApi& n = nccl();
  if (!n.ok) return fail(nullptr, PSSO_E_UNSUPPORTED, n.err);
  NcclUid u;
  const int r = n.get_unique_id(&u);
  if (r) return fail(nullptr, PSSO_E_NCCL, std::string("ncclGetUniqueId: ") + n.error_string(r));
  std::memcpy(id, &u, sizeof u);
  return PSSO_OK;
}

int psso_comm_create(const void* id, int32_t nranks, int32_t rank, psso_comm** out) {
  if (!out) return fail(nullptr, PSSO_E_INVALID, "null output pointer");
  *out = nullptr;
  if (!id || nranks < 1 || rank < 0 || rank >= nranks) return fail(nullptr, PSSO_E_INVALID, "bad communicator arguments");
  const NcclApi& n = nccl();
  if (!n.ok) return fail(nullptr, PSSO_E_UNSUPPORTED, n.err);
  psso_comm* m = new psso_comm();
  if (cudaGetDevice(&m->device) != cudaSuccess) { delete m; return fail(nullptr, PSSO_E_CUDA, "cudaGetDevice"); }
  NcclUid u;
  std::memcpy(&u, id, sizeof u);
  const int r = n.comm_init_rank(&m->comm, nranks, u, rank);  // collective over the ranks
  if (r) { delete m; return fail(nullptr, PSSO_E_NCCL, std::string("ncclCommInitRank: ") + n.error_string(r)); }
  m->nranks = nranks;
  m->rank = rank;
  *out = m;
  return PSSO_OK;
}

void psso_comm_destroy(psso_comm* m) {
  if (!m) return;
  if (m->comm) nccl().comm_destroy(m->comm);
  delete m;
}

int psso_attach_comm(psso_ctx* c, psso_comm* m) {
  DEV_GUARD(c);
  if (int rc = need_bound(c)) return rc;
  if (!m || !m->comm) return fail(c, PSSO_E_INVALID, "null communicator");
  if (m->device != c->device) return fail(c, PSSO_E_INVALID, "communicator and context are on different devices");
  const int64_t rb = psso_candidate_bytes(&c->cfg);
  if (!c->cand) CK(c, cudaMalloc(&c->cand, (size_t)rb));
  if (c->gathered && c->nranks != m->nranks) { cudaFree(c->gathered); c->gathered = nullptr; }
  if (!c->gathered) CK(c, cudaMalloc(&c->gathered, (size_t)rb * m->nranks));
  if (c->sgraph) { cudaGraphExecDestroy(c->sgraph); c->sgraph = nullptr; }
  c->comm = m->comm;
  c->nranks = m->nranks;
  c->rank = m->rank;
  return PSSO_OK;
}

// one exchange: this rank's record -> all-gather (NVLink / NVSwitch) -> apply
static int sharded_exchange(psso_ctx* c, int64_t t, int64_t* t_dev, int is_init) {
  const int64_t rb = psso_candidate_bytes(&c->cfg);
  const int r = nccl().all_gather(c->cand, c->gathered, (size_t)rb, NCCL_UINT8, c->comm, c->stream);
  if (r) return fail(c, PSSO_E_NCCL, std::string("ncclAllGather: ") + nccl().error_string(r));
  GbParams g = gb_params(c, t, t_dev, is_init, 0);
  if (is_init) g.traj = nullptr;
  if (c->cfg.dtype == PSSO_F64)
    k_apply<double><<<1, GB_THREADS, 0, c->stream>>>(g, c->gathered, rb, c->nranks);
  else
    k_apply<float><<<1, GB_THREADS, 0, c->stream>>>(g, c->gathered, rb, c->nranks);
  c->launches++;
  CK(c, cudaGetLastError());
  return PSSO_OK;
}

static int ensure_sgraph(psso_ctx* c);

int psso_init_sharded(psso_ctx* c) {
  DEV_GUARD(c);
  TRACE("psso_init_sharded");
  if (int rc = need_bound(c)) return rc;
  if (!c->comm) return fail(c, PSSO_E_INVALID, "no communicator (psso_attach_comm)");
  k_set_u64<<<1, 1, 0, c->stream>>>(c->bad, ~0ull);
  c->launches++;
  if (int rc = launch_init(c)) return rc;
  if (int rc = local_cand(c, c->cand, c->chain ? c->init_grid : c->grid)) return rc;
  if (int rc = sharded_exchange(c, -1, nullptr, 1)) return rc;
  return c->profiling ? PSSO_OK : ensure_sgraph(c);
}

static int sharded_step(psso_ctx* c, int64_t t, int64_t* t_dev) {
  if (int rc = launch_fused(c, t, t_dev)) return rc;
  if (int rc = local_cand(c, c->cand, c->fused_grid)) return rc;
  return sharded_exchange(c, t, t_dev, 0);
}

// GRAPH_CHUNK x (fused kernel, record, all-gather, apply), t from t_dev;
// captured by psso_init_sharded already (see ensure_graph)
static int ensure_sgraph(psso_ctx* c) {
  if (c->sgraph || c->stream == nullptr) return PSSO_OK;
  cudaGraph_t g;
  CK(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  const int64_t saved = c->launches;
  for (int k = 0; k < GRAPH_CHUNK; ++k) {
    int rc = sharded_step(c, 0, c->t_dev);
    if (rc) { cudaStreamEndCapture(c->stream, &g); return rc; }
  }
  c->launches = saved;
  CK(c, cudaStreamEndCapture(c->stream, &g));
  cudaError_t e = cudaGraphInstantiate(&c->sgraph, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaGraphInstantiate (sharded)");
  return PSSO_OK;
}

int psso_run_sharded(psso_ctx* c, int64_t t0, int64_t niter) {
  DEV_GUARD(c);
  TRACE("psso_run_sharded");
  if (int rc = need_bound(c)) return rc;
  if (!c->comm) return fail(c, PSSO_E_INVALID, "no communicator (psso_attach_comm)");
  if (t0 < 0 || niter < 0) return fail(c, PSSO_E_INVALID, "t0 and niter must be >= 0");
  int64_t done = 0;
  if (c->stream != nullptr && niter >= GRAPH_CHUNK && !c->profiling) {
    if (int rc = ensure_sgraph(c)) return rc;
    k_set<<<1, 1, 0, c->stream>>>(c->t_dev, t0);
    c->launches++;
    for (; done + GRAPH_CHUNK <= niter; done += GRAPH_CHUNK) {
      CK(c, cudaGraphLaunch(c->sgraph, c->stream));
      c->launches += 3 * GRAPH_CHUNK;
    }
  }
  for (; done < niter; ++done)
    if (int rc = sharded_step(c, t0 + done, nullptr)) return rc;
  return PSSO_OK;
}

int64_t psso_p2p_buffer_bytes(const psso_config* cfg, int32_t nranks) {
  if (!cfg || nranks < 1) return 0;
  return (int64_t)align16((size_t)nranks * 16) + 2 * (int64_t)nranks * psso_candidate_bytes(cfg);
}

int psso_p2p_alloc(int64_t bytes, void** dev_ptr) {
  if (!dev_ptr || bytes <= 0) return fail(nullptr, PSSO_E_INVALID, "bad p2p buffer size");
  cudaError_t e = cudaMalloc(dev_ptr, (size_t)bytes);
  if (e == cudaSuccess) e = cudaMemset(*dev_ptr, 0, (size_t)bytes);
  return e == cudaSuccess ? PSSO_OK : cuda_fail(nullptr, e, "psso_p2p_alloc");
}

int psso_p2p_free(void* dev_ptr) {
  cudaError_t e = cudaFree(dev_ptr);
  return e == cudaSuccess ? PSSO_OK : cuda_fail(nullptr, e, "psso_p2p_free");
}

int psso_p2p_handle(void* dev_ptr, void* handle) {
  if (!dev_ptr || !handle) return fail(nullptr, PSSO_E_INVALID, "null pointer");
  cudaError_t e = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle), dev_ptr);
  return e == cudaSuccess ? PSSO_OK : cuda_fail(nullptr, e, "psso_p2p_handle");
}

int psso_p2p_open(const void* handle, void** dev_ptr) {
  if (!dev_ptr || !handle) return fail(nullptr, PSSO_E_INVALID, "null pointer");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? PSSO_OK : cuda_fail(nullptr, e, "psso_p2p_open");
}

int psso_p2p_close(void* dev_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  return e == cudaSuccess ? PSSO_OK : cuda_fail(nullptr, e, "psso_p2p_close");
}

int psso_publish_p2p(psso_ctx* c, const void* cand, void* const* peer_bufs, int32_t nranks,
                     int32_t rank, uint64_t epoch) {
  DEV_GUARD(c);
  TRACE("psso_publish_p2p");
  if (int rc = need_bound(c)) return rc;
  if (!cand || !peer_bufs || nranks < 1 || rank < 0 || rank >= nranks || epoch == 0)
    return fail(c, PSSO_E_INVALID, "bad p2p publish arguments");
  const int64_t rb = psso_candidate_bytes(&c->cfg);
  k_publish<<<1, GB_THREADS, 0, c->stream>>>((const unsigned char*)cand, (unsigned char* const*)peer_bufs,
                                             nranks, rank, epoch, rb, (int64_t)align16((size_t)nranks * 16),
                                             nullptr);
  c->launches++;
  CK(c, cudaGetLastError());
  return PSSO_OK;
}

int psso_apply_p2p(psso_ctx* c, int64_t t, const void* my_buf, int32_t nranks, uint64_t epoch,
                   int32_t is_init) {
  DEV_GUARD(c);
  TRACE("psso_apply_p2p");
  if (int rc = need_bound(c)) return rc;
  if (!my_buf || nranks < 1 || epoch == 0) return fail(c, PSSO_E_INVALID, "bad p2p apply arguments");
  GbParams g = gb_params(c, t, nullptr, is_init, 0);
  if (is_init) g.traj = nullptr;
  g.t_arg = is_init ? -1 : t;
  const int64_t rb = psso_candidate_bytes(&c->cfg), fb = (int64_t)align16((size_t)nranks * 16);
  if (c->cfg.dtype == PSSO_F64)
    k_apply_p2p<double><<<1, GB_THREADS, 0, c->stream>>>(g, (const unsigned char*)my_buf, nranks, epoch, rb, fb);
  else
    k_apply_p2p<float><<<1, GB_THREADS, 0, c->stream>>>(g, (const unsigned char*)my_buf, nranks, epoch, rb, fb);
  c->launches++;
  CK(c, cudaGetLastError());
  return PSSO_OK;
}

// one P2P exchange step with t (and the epoch) from the device counter
static int p2p_step_dev(psso_ctx* c, const void* peer_bufs, const PeerPtrs& pp, const void* my_buf,
                        int32_t nranks, int32_t rank) {
  if (int rc = launch_fused(c, 0, c->t_dev)) return rc;
  const int64_t rb = psso_candidate_bytes(&c->cfg), fb = (int64_t)align16((size_t)nranks * 16);
  GbParams gl = gb_params(c, 0, c->t_dev, 0, c->fused_grid);
  const auto bufs = (unsigned char* const*)peer_bufs;
  const auto mine = (const unsigned char*)my_buf;
  if (c->cfg.dtype == PSSO_F64)
    k_p2p_exchange<double><<<1, GB_THREADS, 0, c->stream>>>(gl, bufs, pp, mine, nranks, rank, rb, fb);
  else
    k_p2p_exchange<float><<<1, GB_THREADS, 0, c->stream>>>(gl, bufs, pp, mine, nranks, rank, rb, fb);
  c->launches += 1;
  CK(c, cudaGetLastError());
  return PSSO_OK;
}

int psso_run_p2p(psso_ctx* c, int64_t t0, int64_t niter, void* const* peer_bufs, const void* my_buf,
                 int32_t nranks, int32_t rank) {
  DEV_GUARD(c);
  TRACE("psso_run_p2p");
  if (int rc = need_bound(c)) return rc;
  if (!peer_bufs || !my_buf || nranks < 1 || rank < 0 || rank >= nranks || t0 < 0 || niter < 0)
    return fail(c, PSSO_E_INVALID, "bad p2p loop arguments");
  if (nranks > 64) return fail(c, PSSO_E_UNSUPPORTED, "the P2P device loop takes up to 64 ranks");
  if (!c->cand) CK(c, cudaMalloc(&c->cand, (size_t)psso_candidate_bytes(&c->cfg)));
  if (c->pgraph && (c->pg_peers != peer_bufs || c->pg_buf != my_buf || c->pg_R != nranks || c->pg_rank != rank)) {
    cudaGraphExecDestroy(c->pgraph);
    c->pgraph = nullptr;
  }
  if (niter == 0) return PSSO_OK;
  if (c->pp_src != peer_bufs || c->pp_R != nranks) {  // the peer table by value for up to 8 ranks,
    std::memset(&c->pp, 0, sizeof c->pp);               // read once per table (never during capture)
    if (nranks <= 8) {
      CK(c, cudaMemcpy(c->pp.p, peer_bufs, sizeof(void*) * (size_t)nranks, cudaMemcpyDeviceToHost));
      c->pp.n = nranks;
    }
    c->pp_src = peer_bufs;
    c->pp_R = nranks;
  }
  const PeerPtrs& pp = c->pp;
  k_set<<<1, 1, 0, c->stream>>>(c->t_dev, t0);
  c->launches++;
  int64_t done = 0;
  const bool graph = c->stream != nullptr && !c->profiling;
  if (graph && niter >= GRAPH_CHUNK) {
    if (!c->pgraph) {  // GRAPH_CHUNK x (fused kernel, record + publish + wait + apply)
      cudaGraph_t gr;
      CK(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
      const int64_t saved = c->launches;
      for (int k = 0; k < GRAPH_CHUNK; ++k) {
        int rc = p2p_step_dev(c, peer_bufs, pp, my_buf, nranks, rank);
        if (rc) { cudaStreamEndCapture(c->stream, &gr); return rc; }
      }
      c->launches = saved;
      CK(c, cudaStreamEndCapture(c->stream, &gr));
      cudaError_t e = cudaGraphInstantiate(&c->pgraph, gr, 0);
      cudaGraphDestroy(gr);
      if (e != cudaSuccess) return cuda_fail(c, e, "cudaGraphInstantiate (p2p)");
      c->pg_peers = peer_bufs;
      c->pg_buf = my_buf;
      c->pg_R = nranks;
      c->pg_rank = rank;
    }
    for (; done + GRAPH_CHUNK <= niter; done += GRAPH_CHUNK) {
      CK(c, cudaGraphLaunch(c->pgraph, c->stream));
      c->launches += 2 * GRAPH_CHUNK;
    }
  }
  for (; done < niter; ++done)  // same kernels, launched directly
    if (int rc = p2p_step_dev(c, peer_bufs, pp, my_buf, nranks, rank)) return rc;
  return PSSO_OK;
}

int psso_check(psso_ctx* c, int64_t* bad_t, int64_t* bad_i) {
  DEV_GUARD(c);
  if (!c) return fail(nullptr, PSSO_E_INVALID, "null context");
  unsigned long long key = ~0ull;
  CK(c, cudaStreamSynchronize(c->stream));
  CK(c, cudaMemcpy(&key, c->bad, sizeof key, cudaMemcpyDeviceToHost));
  if (key == ~0ull) {
    if (bad_t) *bad_t = 0;
    if (bad_i) *bad_i = -1;
    return PSSO_OK;
  }
  if (bad_t) *bad_t = (int64_t)(key >> 40) - 1;
  if (bad_i) *bad_i = (int64_t)(key & ((1ull << 40) - 1));
  return fail(c, PSSO_E_NONFINITE, "non-finite fitness");
}

int psso_iteration_stats(psso_ctx* c, int64_t t0, int64_t n, double* kernel_ms, int64_t* improved,
                         int64_t* timed) {
  DEV_GUARD(c);
  if (int rc = need_bound(c)) return rc;
  if (t0 < 0 || n < 0 || n > STATS_CAP) return fail(c, PSSO_E_INVALID, "need 0 <= n <= 1024 iterations from t0 >= 0");
  std::vector<unsigned long long> st(3 * STATS_CAP);
  CK(c, cudaStreamSynchronize(c->stream));
  CK(c, cudaMemcpy(st.data(), c->stats, st.size() * 8, cudaMemcpyDeviceToHost));
  double ns = 0.0;
  int64_t imp = 0, cnt = 0;
  for (int64_t t = t0; t < t0 + n; ++t) {
    const unsigned long long* q = &st[3 * (t & (STATS_CAP - 1))];
    if (q[0] == ~0ull || q[1] < q[0]) continue;  // not recorded (kernel without stats)
    ns += (double)(q[1] - q[0]);
    imp += (int64_t)q[2];
    ++cnt;
  }
  if (kernel_ms) *kernel_ms = ns * 1e-6;
  if (improved) *improved = imp;
  if (timed) *timed = cnt;
  return PSSO_OK;
}

int psso_nonfinite(psso_ctx* c, int64_t* bad_t, int64_t* bad_i, double* value) {
  DEV_GUARD(c);
  if (!c) return fail(nullptr, PSSO_E_INVALID, "null context");
  int64_t bt = 0, bi = -1;
  int rc = psso_check(c, &bt, &bi);
  if (rc != PSSO_OK && rc != PSSO_E_NONFINITE) return rc;
  double v = 0.0;
  if (rc == PSSO_E_NONFINITE) {
    if (c->bound && c->buf.sol_f && bi >= c->cfg.row_lo && bi < c->cfg.row_hi)
      CK(c, cudaMemcpy(&v, c->buf.sol_f + (bi - c->cfg.row_lo), sizeof v, cudaMemcpyDeviceToHost));
    else
      CK(c, cudaMemcpy(&v, c->bad_val, sizeof v, cudaMemcpyDeviceToHost));
  }
  if (bad_t) *bad_t = bt;
  if (bad_i) *bad_i = bi;
  if (value) *value = v;
  return rc;
}

int psso_result(psso_ctx* c, double* g_f, int64_t* g_idx, int64_t* bad_t, int64_t* bad_i) {
  DEV_GUARD(c);
  if (int rc = need_bound(c)) return rc;
  CK(c, cudaStreamSynchronize(c->stream));
  if (g_f) CK(c, cudaMemcpy(g_f, c->buf.g_f, sizeof(double), cudaMemcpyDeviceToHost));
  if (g_idx) CK(c, cudaMemcpy(g_idx, c->g_idx, sizeof(int64_t), cudaMemcpyDeviceToHost));
  return psso_check(c, bad_t, bad_i);
}

int psso_set_gbest_index(psso_ctx* c, int64_t g_idx) {
  DEV_GUARD(c);
  if (int rc = need_bound(c)) return rc;
  if (g_idx < -1 || g_idx >= c->cfg.nsol) return fail(c, PSSO_E_INVALID, "gBest index out of range");
  k_set<<<1, 1, 0, c->stream>>>(c->g_idx, g_idx);
  c->launches++;
  CK(c, cudaGetLastError());
  return PSSO_OK;
}

int64_t psso_launch_count(const psso_ctx* c) { return c ? c->launches : -1; }

int psso_profile(psso_ctx* c, int32_t enable) {
  if (!c) return fail(nullptr, PSSO_E_INVALID, "null context");
  c->profiling = enable != 0;
  c->ev_used = 0;
  c->prof_iters = 0;
  return PSSO_OK;
}

int psso_profile_read(psso_ctx* c, double* kernel_ms, int64_t* nlaunch) {
  DEV_GUARD(c);
  if (!c) return fail(nullptr, PSSO_E_INVALID, "null context");
  CK(c, cudaStreamSynchronize(c->stream));
  double tot = 0.0;
  for (size_t k = 0; k + 1 < c->ev_used; k += 2) {
    float ms = 0.f;
    CK(c, cudaEventElapsedTime(&ms, c->ev[k], c->ev[k + 1]));
    tot += ms;
  }
  if (kernel_ms) *kernel_ms = tot;
  if (nlaunch) *nlaunch = c->prof_iters;
  c->ev_used = 0;
  c->prof_iters = 0;
  return PSSO_OK;
}

int psso_rng_uniform(uint64_t seed, uint64_t stream_key, uint64_t t, const uint64_t* particles,
                     const uint64_t* variables, int64_t n, double* out, void* stream) {
  if (n < 0 || (n > 0 && (!particles || !variables || !out)))
    return fail(nullptr, PSSO_E_INVALID, "bad rng arguments");
  if (n == 0) return PSSO_OK;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 4096);
  k_rng<<<grid, 256, 0, (cudaStream_t)stream>>>(seed, stream_key, t, particles, variables, n, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PSSO_OK : cuda_fail(nullptr, e, "psso_rng_uniform");
}

int psso_eval_rows(int32_t fn_id, int32_t dtype, int64_t nvar, const void* x, int64_t rows,
                   double* out, double probe_level, void* stream) {
  TRACE("psso_eval_rows");
  psso_config cfg;
  std::memset(&cfg, 0, sizeof cfg);
  cfg.fn_id = fn_id;
  cfg.dtype = dtype;
  cfg.rng_mode = PSSO_RNG_REFERENCE;
  cfg.nsol = rows > 0 ? rows : 1;
  cfg.nvar = nvar;
  cfg.row_lo = 0;
  cfg.row_hi = cfg.nsol;
  cfg.cw = 0.3; cfg.cp = 0.6; cfg.cg = 0.8;
  cfg.var_min = -1; cfg.var_max = 1;
  cfg.probe_level = probe_level;
  if (rows == 0) return PSSO_OK;
  if (rows < 0 || !x || !out) return fail(nullptr, PSSO_E_INVALID, "bad eval arguments");
  if ((uintptr_t)x % 16) return fail(nullptr, PSSO_E_INVALID, "input rows must be 16-byte aligned");
  psso_ctx* c = nullptr;
  int rc = psso_create(&cfg, &c);
  if (rc) return rc;
  psso_buffers b;
  std::memset(&b, 0, sizeof b);
  c->buf = b;
  c->buf.sol = const_cast<void*>(x);
  c->buf.sol_f = out;
  c->bound = true;
  c->stream = (cudaStream_t)stream;
  TileParams p = tile_params(c, M_LOAD | M_EVAL | M_SOLF, -1, nullptr);
  p.bad = nullptr;
  rc = launch_tile(c, p);
  if (rc == PSSO_OK) {
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) rc = cuda_fail(nullptr, e, "psso_eval_rows");
  }
  psso_destroy(c);
  return rc;
}

int psso_solve(const psso_config* cfg, int64_t niter, double* traj, void* best_position,
               double* best_fitness, double* wall_s) {
  TRACE("psso_solve");
  // PSSO_SOLVE_TRACE=1: host time of each phase to stderr (diagnostic)
  const char* tr_env = std::getenv("PSSO_SOLVE_TRACE");
  const bool trace = tr_env && *tr_env && *tr_env != '0';
  auto tp = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!trace) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[psso_solve] %-10s %9.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - tp).count());
    tp = now;
  };
  std::string err;
  int rc = validate(cfg, err);
  if (rc) return fail(nullptr, rc, err);
  if (niter < 1) return fail(nullptr, PSSO_E_INVALID, "niter must be a positive integer");
  if (cfg->row_lo != 0 || cfg->row_hi != cfg->nsol) return fail(nullptr, PSSO_E_INVALID, "psso_solve runs the whole swarm");
  const size_t es = cfg->dtype == PSSO_F64 ? 8 : 4;
  const size_t N = (size_t)cfg->nsol, D = (size_t)cfg->nvar;
  psso_buffers b;
  std::memset(&b, 0, sizeof b);
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  psso_ctx* c = nullptr;
  cudaError_t e = cudaSuccess;
  auto cleanup = [&]() {
    if (c) psso_destroy(c);
    mark("destroy");
    for (void* q : {b.sol, b.pbests, (void*)b.p_f, b.gbest, (void*)b.g_f, (void*)b.traj})
      if (q) cudaFreeAsync(q, s);
    mark("freeasync");
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (s) { cudaStreamSynchronize(s); mark("streamsync"); }
  };
  if ((e = solve_stream(&s)) != cudaSuccess ||
      (e = cudaEventCreate(&e0)) != cudaSuccess || (e = cudaEventCreate(&e1)) != cudaSuccess ||
      (e = pool_alloc(&b.sol, N * D * es, s)) != cudaSuccess ||
      (e = pool_alloc(&b.pbests, N * D * es, s)) != cudaSuccess ||
      (e = pool_alloc((void**)&b.p_f, N * 8, s)) != cudaSuccess ||
      (e = pool_alloc(&b.gbest, D * es, s)) != cudaSuccess ||
      (e = pool_alloc((void**)&b.g_f, 8, s)) != cudaSuccess ||
      (e = pool_alloc((void**)&b.traj, (size_t)niter * 8, s)) != cudaSuccess) {
    cleanup();
    return cuda_fail(nullptr, e, "psso_solve alloc");
  }
  mark("alloc");
  if ((rc = psso_create(cfg, &c)) != PSSO_OK) { c = nullptr; cleanup(); return rc; }
  mark("create");
  if ((rc = psso_bind(c, &b, s)) || (rc = psso_init(c))) { cleanup(); return rc; }
  int64_t bt, bi;
  if ((rc = psso_check(c, &bt, &bi)) != PSSO_OK) {
    g_err = "non-finite fitness at particle " + std::to_string(bi) + " during initialization";
    cleanup();
    return rc;
  }
  mark("init");
  cudaEventRecord(e0, s);
  if ((rc = psso_run(c, 0, niter)) != PSSO_OK) { cleanup(); return rc; }
  cudaEventRecord(e1, s);
  mark("enqueue");
  if ((rc = psso_check(c, &bt, &bi)) != PSSO_OK) {
    g_err = "non-finite fitness at particle " + std::to_string(bi) + " at iteration " + std::to_string(bt);
    cleanup();
    return rc;
  }
  mark("loop+sync");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  if (traj) e = cudaMemcpy(traj, b.traj, (size_t)niter * 8, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && best_position) e = cudaMemcpy(best_position, b.gbest, D * es, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && best_fitness) e = cudaMemcpy(best_fitness, b.g_f, 8, cudaMemcpyDeviceToHost);
  if (wall_s) *wall_s = ms * 1e-3;
  mark("copy-back");
  cleanup();
  mark("cleanup");
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "psso_solve copy-back");
  return PSSO_OK;
}

}  // extern "C"

// Many swarms of cfg (one per seed), initialized together by the whole-run
// kernel (do_init), then the loop of the parallel schedule (k_swarm) or of the
// sequential schedule (k_seq, one CTA per swarm) -- one launch for all seeds.
static int solve_batch(const psso_config* cfg, const uint64_t* seeds, int32_t nseeds, int64_t niter,
                       double* traj, void* best_position, double* best_fitness, double* wall_s,
                       bool sequential) {
  std::string err;
  int rc = validate(cfg, err);
  if (rc) return fail(nullptr, rc, err);
  if (niter < 1) return fail(nullptr, PSSO_E_INVALID, "niter must be a positive integer");
  if (nseeds < 1 || !seeds) return fail(nullptr, PSSO_E_INVALID, "need at least one seed");
  if (cfg->row_lo != 0 || cfg->row_hi != cfg->nsol) return fail(nullptr, PSSO_E_INVALID, "psso_solve_batch runs whole swarms");
  psso_ctx* c = nullptr;
  if ((rc = psso_create(cfg, &c)) != PSSO_OK) return rc;
  if (!c->chain || cfg->nsol * cfg->nvar > PSSO_SWARM_MAX_ELEMS) {
    psso_destroy(c);
    return fail(nullptr, PSSO_E_UNSUPPORTED, "batched runs need nvar <= 128 and nsol*nvar <= 2^22 (whole-run kernel)");
  }
  const size_t es = cfg->dtype == PSSO_F64 ? 8 : 4;
  const size_t B = (size_t)nseeds, N = (size_t)cfg->nsol, D = (size_t)cfg->nvar;
  SwarmPlan pl;
  cudaError_t e = cudaSuccess;
  if (!plan_swarm(c, (int64_t)B, pl, e)) {
    psso_destroy(c);
    return e != cudaSuccess ? cuda_fail(nullptr, e, "psso_solve_batch plan")
                            : fail(nullptr, PSSO_E_UNSUPPORTED, "no whole-run kernel for this batch");
  }
  const int G = pl.G;
  struct Buf { void* p = nullptr; } X, P, pf, gb, gf, tr, ep, sf, si, sn, sr, sd, bad, xn, fn, pfn, solf;
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  auto cleanup = [&]() {
    for (Buf* b : {&X, &P, &pf, &gb, &gf, &tr, &ep, &sf, &si, &sn, &sr, &sd, &bad, &xn, &fn, &pfn, &solf})
      if (b->p) cudaFreeAsync(b->p, s);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (s) cudaStreamSynchronize(s);
    psso_destroy(c);
  };
  if ((e = solve_stream(&s)) != cudaSuccess ||
      (e = cudaEventCreate(&e0)) != cudaSuccess || (e = cudaEventCreate(&e1)) != cudaSuccess ||
      (e = pool_alloc(&X.p, B * N * D * es, s)) != cudaSuccess ||
      (e = pool_alloc(&P.p, B * N * D * es, s)) != cudaSuccess ||
      (e = pool_alloc(&pf.p, B * N * 8, s)) != cudaSuccess ||
      (e = pool_alloc(&gb.p, B * D * es, s)) != cudaSuccess ||
      (e = pool_alloc(&gf.p, B * 8, s)) != cudaSuccess ||
      (e = pool_alloc(&tr.p, B * (size_t)niter * 8, s)) != cudaSuccess ||
      (e = pool_alloc(&ep.p, B * 2 * G * sizeof(unsigned int), s)) != cudaSuccess ||
      (e = pool_alloc(&sf.p, B * 2 * G * 8, s)) != cudaSuccess ||
      (e = pool_alloc(&si.p, B * 2 * G * 8, s)) != cudaSuccess ||
      (e = pool_alloc(&sn.p, B * 2 * G * 4, s)) != cudaSuccess ||
      (e = pool_alloc(&sr.p, B * 2 * G * D * es, s)) != cudaSuccess ||
      (e = pool_alloc(&sd.p, B * 8, s)) != cudaSuccess ||
      (e = pool_alloc(&bad.p, B * 8, s)) != cudaSuccess ||
      (e = pool_alloc(&solf.p, B * N * 8, s)) != cudaSuccess ||  // non-finite values
      (e = cudaMemcpyAsync(sd.p, seeds, B * 8, cudaMemcpyHostToDevice, s)) != cudaSuccess ||
      (e = cudaMemsetAsync(bad.p, 0xff, B * 8, s)) != cudaSuccess) {
    cleanup();
    return cuda_fail(nullptr, e, "psso_solve_batch alloc");
  }
  psso_buffers pb;
  std::memset(&pb, 0, sizeof pb);
  pb.sol = X.p; pb.pbests = P.p; pb.p_f = (double*)pf.p; pb.gbest = gb.p; pb.g_f = (double*)gf.p;
  c->buf = pb;
  c->stream = s;
  c->bound = true;
  TileParams p = tile_params(c, fused_mode(c), 0, nullptr, true);
  p.off_bar = pl.off_bar;
  p.off_scr = pl.off_scr;
  p.off_leaf = pl.off_pub;
  p.off_xs = pl.off_xs;
  SwarmParams sp;
  std::memset(&sp, 0, sizeof sp);
  sp.rows = (int64_t)N;
  sp.G = G;
  sp.gpc = pl.gpc;
  sp.epoch = (unsigned int*)ep.p;
  sp.slot_f = (double*)sf.p;
  sp.slot_i = (int64_t*)si.p;
  sp.slot_new = (int32_t*)sn.p;
  sp.slot_row = sr.p;
  sp.traj = (double*)tr.p;
  sp.traj_stride = niter;
  sp.g_f = (double*)gf.p;
  sp.gbest = gb.p;
  sp.seeds = (const uint64_t*)sd.p;
  sp.bad = (unsigned long long*)bad.p;
  sp.sol_f = (double*)solf.p;
  auto launch = [&]() -> cudaError_t {
    cudaError_t r = cudaMemsetAsync(ep.p, 0, B * 2 * G * sizeof(unsigned int), s);
    if (r != cudaSuccess) return r;
    void* args[] = {(void*)&p, (void*)&sp};
    return launch_swarm(pl, (int64_t)B, args, s);
  };
  sp.do_init = 1;  // initialize (core.py:196-210), outside the timed loop (parallel.py:190)
  sp.niter = 0;
  if ((e = launch()) != cudaSuccess) { cleanup(); return cuda_fail(nullptr, e, "psso_solve_batch init"); }
  sp.do_init = 0;
  sp.t0 = 0;
  sp.niter = niter;
  if (sequential) {  // speculative-pass scratch of k_seq, then its loop
    const int M = D <= 32 ? 4 : D <= 64 ? 8 : 16;
    if (!seq_kernel(cfg->dtype, cfg->rng_mode, cfg->fn_id, M, false)) {
      cleanup();
      return fail(nullptr, PSSO_E_UNSUPPORTED, "no sequential kernel for this configuration");
    }
    if ((e = pool_alloc(&xn.p, B * N * D * es, s)) != cudaSuccess ||
        (e = pool_alloc(&fn.p, B * N * 8, s)) != cudaSuccess ||
        (e = pool_alloc(&pfn.p, B * N * 8, s)) != cudaSuccess) {
      cleanup();
      return cuda_fail(nullptr, e, "psso_solve_sequential_batch alloc");
    }
    SeqParams q;
    std::memset(&q, 0, sizeof q);
    q.t0 = 0;
    q.niter = niter;
    q.rows = (int64_t)N;
    q.Xn = xn.p;
    q.fn = (double*)fn.p;
    q.pfn = (double*)pfn.p;
    q.traj = (double*)tr.p;
    q.traj_stride = niter;
    q.g_f = (double*)gf.p;
    q.gbest = gb.p;
    q.seeds = (const uint64_t*)sd.p;
    q.bad = (unsigned long long*)bad.p;
    q.sol_f = (double*)solf.p;
    cudaEventRecord(e0, s);
    if ((e = launch_seq(c, M, q, (int64_t)B, s)) != cudaSuccess) {
      cleanup();
      return cuda_fail(nullptr, e, "psso_solve_sequential_batch run");
    }
    cudaEventRecord(e1, s);
  } else {
    cudaEventRecord(e0, s);
    if ((e = launch()) != cudaSuccess) { cleanup(); return cuda_fail(nullptr, e, "psso_solve_batch run"); }
    cudaEventRecord(e1, s);
  }
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) { cleanup(); return cuda_fail(nullptr, e, "psso_solve_batch"); }
  std::vector<unsigned long long> bk(B);
  g_batch_fail = BatchFailure();
  e = cudaMemcpy(bk.data(), bad.p, B * 8, cudaMemcpyDeviceToHost);
  for (size_t q = 0; e == cudaSuccess && q < B; ++q)
    if (bk[q] != ~0ull) {
      const int64_t bt = (int64_t)(bk[q] >> 40) - 1, bi = (int64_t)(bk[q] & ((1ull << 40) - 1));
      g_batch_fail.swarm = (int64_t)q;
      g_batch_fail.t = bt;
      g_batch_fail.i = bi;
      cudaMemcpy(&g_batch_fail.value, (double*)solf.p + q * N + bi, 8, cudaMemcpyDeviceToHost);
      g_err = "non-finite fitness in swarm " + std::to_string(q) + " (seed " + std::to_string(seeds[q]) +
              ") at particle " + std::to_string(bi) +
              (bt < 0 ? std::string(" during initialization") : " at iteration " + std::to_string(bt));
      cleanup();
      return PSSO_E_NONFINITE;
    }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  if (e == cudaSuccess && traj) e = cudaMemcpy(traj, tr.p, B * (size_t)niter * 8, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && best_position) e = cudaMemcpy(best_position, gb.p, B * D * es, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && best_fitness) e = cudaMemcpy(best_fitness, gf.p, B * 8, cudaMemcpyDeviceToHost);
  if (wall_s) *wall_s = ms * 1e-3;
  cleanup();
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "psso_solve_batch copy-back");
  return PSSO_OK;
}

extern "C" {

int psso_batch_failure(int64_t* swarm, int64_t* iteration, int64_t* particle, double* value) {
  if (swarm) *swarm = g_batch_fail.swarm;
  if (iteration) *iteration = g_batch_fail.t;
  if (particle) *particle = g_batch_fail.i;
  if (value) *value = g_batch_fail.value;
  return g_batch_fail.swarm >= 0 ? PSSO_E_NONFINITE : PSSO_OK;
}

int psso_solve_batch(const psso_config* cfg, const uint64_t* seeds, int32_t nseeds, int64_t niter,
                     double* traj, void* best_position, double* best_fitness, double* wall_s) {
  TRACE("psso_solve_batch");
  return solve_batch(cfg, seeds, nseeds, niter, traj, best_position, best_fitness, wall_s, false);
}

int psso_solve_sequential_batch(const psso_config* cfg, const uint64_t* seeds, int32_t nseeds,
                                int64_t niter, double* traj, void* best_position,
                                double* best_fitness, double* wall_s) {
  TRACE("psso_solve_sequential_batch");
  return solve_batch(cfg, seeds, nseeds, niter, traj, best_position, best_fitness, wall_s, true);
}

}  // extern "C"
