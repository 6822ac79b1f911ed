// brm_kernels.cuh -- sm_100a kernels of the nested-MC engine (templates).
//
//   walk_units   persistent CTAs over (unit, chunk) work items; a unit is a
//                pricing block (pricer.py:154-164), a CMC training point
//                (_core.pyx:515-550) or a stopped_sums call (_core.pyx:402-430)
//   finish_units fixed-order fold of chunk partials -> unit sums / labels
//   iz_probes    one thread-block cluster per I&Z probe: the cluster's CTAs
//                split the inner paths, reduce through distributed shared
//                memory and iterate the fixed-point or bisection solve
//                without leaving the kernel (_core.pyx:433-512)
//   decisions, sample_points, raw/normal fills, key derivation
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <type_traits>

#include "brm_internal.h"
#include "brm_walk.cuh"
#include "brm_walk_log.cuh"

namespace cg = cooperative_groups;

namespace brm {

// ---------------------------------------------------------------- walk ----
#ifndef BRM_LOG_MINB
#define BRM_LOG_MINB 2
#endif
template <int D, bool FAST, int SPEC = WALK_GENERIC>
__global__ void __launch_bounds__(kWalkThreads, SPEC == WALK_CMC_LOG ? BRM_LOG_MINB : ((FAST && D < 20) ? 3 : 2))
    walk_units(WalkParams P) {
  constexpr bool kLog = SPEC == WALK_CMC_LOG;  // log-price state and log-threshold tables (brm_walk_log.cuh)
  static_assert(!kLog || (!FAST && D > 1), "the log-price walker is a parity instance for d > 1");
  constexpr int TG = FAST ? 1 : TailGroup<D>::G;
  __shared__ double s_tq_buf[(kWalkThreads / 32) * 32 * TG];
  __shared__ unsigned short s_tq_idx[(kWalkThreads / 32) * 32 * TG];
  const TailQueue tq{s_tq_buf + (threadIdx.x >> 5) * 32 * TG, s_tq_idx + (threadIdx.x >> 5) * 32 * TG};
  using R = RealT<FAST>;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double s_red[2 * (kWalkThreads / 32)];
  __shared__ int s_next;
  __shared__ R s_start[kMaxD];
  __shared__ unsigned char s_stopm[kLog ? kMaxChunk : 1];  // log-price walker: stop date per path slot
  const Model<R> M = load_model<R, kLog>(P.hdr, P.blob, smem);
  [[maybe_unused]] const float4 *cc_rows = nullptr;
  if constexpr (SPEC == WALK_CMC_COLCONST) cc_rows = pack_colconst_rows<D>(M);
  if constexpr (SPEC == WALK_CMC_UNIT && FAST && D > 1)
    cc_rows = reinterpret_cast<const float4 *>(pack_unit_rows<D>(M));
  double *vals = reinterpret_cast<double *>(smem + P.vals_offset);
  const int d = M.d;
  [[maybe_unused]] const double log_strike = kLog ? log(P.hdr.strike) : 0.0;
  // the specialised instances never run on supplied normals (host check)
  const NormalSrc ns = SPEC == WALK_GENERIC ? NormalSrc{P.normals, P.nrm_base, P.nrm_count} : NormalSrc{nullptr, 0, 0};

  // work items are claimed from a counter (the first one is the CTA's own
  // index): items differ in length with their unit's moneyness, and a static
  // stride leaves the last CTAs ~3 sigma of an item-sum behind the mean
  __shared__ int s_item;
  for (int item = blockIdx.x; item < P.n_items; item = s_item) {
    const int u = item / P.chunks_per_unit;
    const int c = item - u * P.chunks_per_unit;
    const int64_t cnt64 = P.total_paths - (int64_t)u * P.per_unit;
    const int cnt = (int)(cnt64 < P.per_unit ? cnt64 : P.per_unit);
    const int p0 = c * P.chunk;
    const int p1 = min(p0 + P.chunk, cnt);
    uint64_t key, stream;
    if (P.keys) {
      key = P.keys[u];
      stream = P.streams[u];
    } else {
      derive_words(P.seed, (uint64_t)P.phase, (uint64_t)(P.item_base + u), (uint64_t)P.key_date, key, stream);
    }
    if (threadIdx.x < d) {
      const R s = P.starts ? (R)P.starts[(size_t)u * P.start_stride + threadIdx.x] : M.s0[threadIdx.x];
      if constexpr (kLog) s_start[threadIdx.x] = log(s);
      else s_start[threadIdx.x] = s;
    }
    if (threadIdx.x == 0) s_next = p0 + blockDim.x;
    __syncthreads();
    if (p0 < p1) {
      const uint64_t base0 = unit_base<FAST>(P.draw_base, P.normals != nullptr);
      double *pout = P.path_out ? P.path_out + (size_t)u * P.per_unit : nullptr;
      int32_t *sout = P.stop_out ? P.stop_out + (size_t)u * P.per_unit : nullptr;
      if constexpr (kLog) {
        walk_paths_log<(D > 1 ? D : 2)>(M, s_start, log_strike, P.m_start, P.n_steps, key, stream, base0, p0, p1, vals,
                                        s_stopm, &s_next, P.steps, tq);
        __syncthreads();
        finish_log_values(M, P.m_start, p0, p1 - p0, vals, s_stopm, pout, sout);
      } else
        walk_paths<D, FAST, SPEC>(M, s_start, P.m_start, P.n_steps, key, stream, base0, p0, p1, ns, vals, &s_next, pout,
                                  sout, P.steps, tq, cc_rows);
    }
    __syncthreads();
    double s = 0.0, q = 0.0;
    fold_values(vals, p1 > p0 ? p1 - p0 : 0, s_red, s, q);
    if (threadIdx.x == 0) {
      P.partials[2 * (size_t)item] = s;
      P.partials[2 * (size_t)item + 1] = q;
      s_item = P.next_item ? (int)gridDim.x + atomicAdd(P.next_item, 1) : item + (int)gridDim.x;
    }
    __syncthreads();  // the next item is known, and this one is finished with s_start / vals / s_next
  }
}

// ------------------------------------------------------------ I&Z probes ----
// Probe state for the payoff-driving scalar x (_core.pyx:476-483): the probed
// asset at x, other assets at their seeds pulled to x - 0.01K when above x.
// iz_space 1 (geometric put) sets the last asset so the state's geometric
// mean is x.  Returns the probed asset's price.
__device__ inline double probe_state(const ModelHdr &h, const double *seed, int asset, double x, double *st) {
  const int d = h.d;
  if (h.iz_space == 1) {
    double sl = 0.0;
    for (int j = 0; j < d - 1; ++j) {
      st[j] = seed[j];
      sl = __dadd_rn(sl, log(seed[j]));
    }
    st[d - 1] = exp(__dsub_rn(__dmul_rn((double)d, log(x)), sl));
    return st[d - 1];
  }
  int j = 0;
  for (int i = 0; i < d; ++i) {
    if (i == asset) {
      st[i] = x;
    } else {
      st[i] = seed[j] <= x ? seed[j] : __dsub_rn(x, __dmul_rn(0.01, h.strike));
      ++j;
    }
  }
  return x;
}

// Fixed-order sums of vals[0..n) in chunks of kIzFoldChunk paths into
// s_chunk[]: warp w folds chunks w, w + 8, ...; lane l adds the chunk's
// values l, l + 32, ... in order, then a fixed shuffle tree.  One barrier.
__device__ __forceinline__ void fold_chunks(const double *vals, int n, double *s_chunk) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nck = (n + kIzFoldChunk - 1) / kIzFoldChunk;
  for (int c = warp; c < nck; c += blockDim.x >> 5) {
    const double *v = vals + c * kIzFoldChunk;
    const int len = min(kIzFoldChunk, n - c * kIzFoldChunk);
    double s = 0.0;
    for (int j = lane; j < len; j += 32) s = __dadd_rn(s, v[j]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, off));
    if (lane == 0) s_chunk[c] = s;
  }
  __syncthreads();
}

// Rank 0 of a probe cluster: the chunk sums of every CTA of the cluster, fetched
// over distributed shared memory by the lanes of warp 0 in parallel (one
// thread fetching them one after the other pays a remote round trip per
// chunk), into s_all in path order.  The caller's thread 0 then adds them in
// that order, so the sum does not depend on the cluster size.  Warp 0 only.
__device__ __forceinline__ int gather_chunk_sums(cg::cluster_group &cluster, double *s_chunk, int csize, int per_cta,
                                                 int n_inner, double *s_all) {
  const int per_cta_chunks = per_cta / kIzFoldChunk;
  const int n_chunks = (n_inner + kIzFoldChunk - 1) / kIzFoldChunk;
  for (int g = threadIdx.x; g < n_chunks; g += 32) {
    const int r = g / per_cta_chunks;
    s_all[g] = cluster.map_shared_rank(s_chunk, r)[g - r * per_cta_chunks];
  }
  __syncwarp();
  return n_chunks;
}

// fold_chunks for n_cand value arrays (vals + t * stride -> s_chunk + t * kIzMaxChunks): the
// (candidate, chunk) pairs go round the warps, one barrier for all of them.
__device__ __forceinline__ void fold_chunks_multi(const double *vals, int stride, int n_cand, int n, double *s_chunk) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nck = (n + kIzFoldChunk - 1) / kIzFoldChunk;
  for (int q = warp; q < n_cand * nck; q += blockDim.x >> 5) {
    const int t = q / nck, c = q - t * nck;
    const double *v = vals + (size_t)t * stride + c * kIzFoldChunk;
    const int len = min(kIzFoldChunk, n - c * kIzFoldChunk);
    double s = 0.0;
    for (int j = lane; j < len; j += 32) s = __dadd_rn(s, v[j]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, off));
    if (lane == 0) s_chunk[t * kIzMaxChunks + c] = s;
  }
  __syncthreads();
}

// GMODE 1: the geometric-put instance (walk_paths' GEO step; launched only for
// that payoff).  GMODE 2: the geometric put on log-prices (walk_paths_log's
// LOG_GEOPUT_IZ; parity mode, log-space I&Z surface, independent assets).
// GMODE 3: GMODE 2 with the bisection draw cache (P.rec): the first pass
// records the paths' increments, the others replay them.
template <int D, bool FAST, int GMODE = 0>
__global__ void __launch_bounds__(kWalkThreads, 2) iz_probes(IzParams P) {
  constexpr int GEOK = GMODE == 3 ? 2 : GMODE;
  static_assert(GEOK != 2 || (!FAST && D > 1), "the log-price probe walker is a parity instance for d > 1");
  [[maybe_unused]] const double log_strike = GEOK == 2 ? log(P.hdr.strike) : 0.0;
  constexpr int TG = FAST ? 1 : TailGroup<D>::G;
  __shared__ double s_tq_buf[(kWalkThreads / 32) * 32 * TG];
  __shared__ unsigned short s_tq_idx[(kWalkThreads / 32) * 32 * TG];
  const TailQueue tq{s_tq_buf + (threadIdx.x >> 5) * 32 * TG, s_tq_idx + (threadIdx.x >> 5) * 32 * TG};
  using R = RealT<FAST>;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int csize = (int)cluster.num_blocks();
  // tree mode: clusters (probe, node slot) of the bisection tree; else one cluster per probe
  const int n_slots = P.tree_levels > 1 ? (1 << P.tree_levels) - 1 : 1;
  const int probe = (int)(blockIdx.x / csize) / n_slots;
  const int probe_slot = (int)(blockIdx.x / csize) % n_slots;

  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_next;
  __shared__ R s_start[kMaxD];
  __shared__ double s_state[kMaxD];
  constexpr int kCand = GMODE == 3 ? kIzReplayCand : 1;  // candidate levels a pass evaluates
  __shared__ double s_chunk[kCand * kIzMaxChunks];  // this CTA's 256-path chunk sums (per candidate)
  __shared__ double s_all[kIzMaxChunks * 8];  // rank 0: every CTA's chunk sums in path order
  __shared__ double s_x, s_lo, s_hi;        // rank 0: solver state
  __shared__ int s_done, s_it, s_armed, s_conv;
  const Model<R> M = load_model<R>(P.hdr, P.blob, smem);
  double *vals = reinterpret_cast<double *>(smem + P.vals_offset);
  double *hist = reinterpret_cast<double *>(smem + P.hist_offset);
  const int d = P.hdr.d;
  const NormalSrc ns{P.normals, P.nrm_base, P.nrm_count};
  const double K = P.hdr.strike;
  const bool call_like = P.hdr.call_like != 0;

  uint64_t key, stream;
  if (P.keys) {
    key = P.keys[probe];
    stream = P.streams[probe];
  } else {
    derive_words(P.seed, 1 /* IZ_CALC */, (uint64_t)(P.item_base + probe), (uint64_t)P.m, key, stream);
  }
  const double *seedp = P.seeds + (size_t)probe * P.seed_stride;
  const int asset = P.assets ? P.assets[probe] : 0;
  const int per_cta = iz_per_cta(P.n_inner, csize);
  const int p0 = rank * per_cta;
  const int p1 = min(p0 + per_cta, P.n_inner);
  const uint64_t per_path = (uint64_t)P.n_steps * (uint64_t)d;
  const uint64_t slab = (uint64_t)P.n_inner * per_path;

  if (threadIdx.x == 0 && rank == 0) {
    s_x = P.solver == 0 ? K : 0.5 * (P.lo + P.hi);
    s_lo = P.lo;
    s_hi = P.hi;
    s_done = P.solver == 1 ? !(P.hi - P.lo > P.tol && P.max_iter > 0) : (P.max_iter <= 0);
    s_it = 0;
    s_armed = 0;
    s_conv = 0;
    hist[0] = K;
  }
  cluster.sync();
  double *x_remote = cluster.map_shared_rank(&s_x, 0);
  int *done_remote = cluster.map_shared_rank(&s_done, 0);

  if (P.tree_levels > 1) {
    // ---- bisection tree (solver 1, cooperative launch) --------------------
    // Cluster (probe, slot) evaluates node `slot` of a complete binary tree
    // of tree_levels bisection levels below the probe's current bracket,
    // every node with the same draws (common random numbers, draw_base 0).
    // After a grid barrier every cluster of the probe walks the tree with
    // the nodes' continuation values and takes the bracket binary bisection
    // would reach after those levels: the same midpoints (the same fp64
    // operations), decisions, iteration count and bits, in 1 / tree_levels
    // of the sequential passes.
    cg::grid_group grid = cg::this_grid();
    const int kt = (1 << P.tree_levels) - 1;
    const int slot = probe_slot;
    for (int pass = 0; pass < P.tree_passes; ++pass) {
      if (rank == 0 && threadIdx.x == 0 && !s_done) {
        // the slot's midpoint: descend from the bracket along the heap path
        double l = s_lo, h = s_hi;
        const int path = slot + 1;
        const int depth = 31 - __clz(path);
        for (int t = depth - 1; t >= 0; --t) {
          const double xm = __dmul_rn(0.5, __dadd_rn(l, h));
          if ((path >> t) & 1) l = xm;
          else h = xm;
        }
        s_x = __dmul_rn(0.5, __dadd_rn(l, h));
      }
      cluster.sync();
      const bool done = *done_remote != 0;
      if (!done) {
        const double x = *x_remote;
        if (threadIdx.x == 0) probe_state(P.hdr, seedp, asset, x, s_state);
        __syncthreads();
        if (threadIdx.x < d) s_start[threadIdx.x] = GEOK == 2 ? (R)log(s_state[threadIdx.x]) : (R)s_state[threadIdx.x];
        if (threadIdx.x == 0) s_next = p0 + blockDim.x;
        __syncthreads();
        const uint64_t base0 = unit_base<FAST>(0, P.normals != nullptr);
        if (p0 < p1) {
          if constexpr (GEOK == 2)
            walk_paths_log<(D > 1 ? D : 2), LOG_GEOPUT_IZ>(M, s_start, log_strike, P.m, P.n_steps, key, stream, base0,
                                                           p0, p1, vals, nullptr, &s_next, P.steps, tq);
          else
            walk_paths<D, FAST, GEOK ? WALK_GEO : WALK_GENERIC>(M, s_start, P.m, P.n_steps, key, stream, base0, p0,
                                                                p1, ns, vals, &s_next, nullptr, nullptr, P.steps, tq);
        }
        __syncthreads();
        fold_chunks(vals, p1 > p0 ? p1 - p0 : 0, s_chunk);
      }
      cluster.sync();
      double *cont_buf = P.tree_cont + (size_t)(pass & 1) * P.n_probes * kt + (size_t)probe * kt;
      if (rank == 0 && threadIdx.x < 32 && !done) {
        const int n_chunks = gather_chunk_sums(cluster, s_chunk, csize, per_cta, P.n_inner, s_all);
        if (threadIdx.x == 0) {
          double total = 0.0;
          for (int g = 0; g < n_chunks; ++g) total = __dadd_rn(total, s_all[g]);
          cont_buf[slot] = __ddiv_rn(total, (double)P.n_inner);
        }
      }
      grid.sync();  // (double-buffered by pass: a cluster may publish pass p+1 while another reads pass p)
      if (rank == 0 && threadIdx.x == 0 && !s_done) {
        double l = s_lo, h = s_hi;
        int j = 0, n_it = s_it;
        bool fin = false;
        for (int t = 0; t < P.tree_levels && !fin; ++t) {
          const double xm = __dmul_rn(0.5, __dadd_rn(l, h));
          double st[kMaxD];
          probe_state(P.hdr, seedp, asset, xm, st);
          Model<double> Md{};
          Md.d = d;
          Md.payoff = P.hdr.payoff;
          Md.strike = K;
          const double pay = payoff<0>(Md, st);
          const bool exercise = __dsub_rn(pay, __ldcg(cont_buf + j)) > 0.0;
          if (call_like == exercise) {
            h = xm;
            j = 2 * j + 1;
          } else {
            l = xm;
            j = 2 * j + 2;
          }
          ++n_it;
          fin = !(__dsub_rn(h, l) > P.tol) || n_it >= P.max_iter;
        }
        s_lo = l;
        s_hi = h;
        s_it = n_it;
        s_done = fin ? 1 : 0;
      }
    }
    if (rank == 0 && threadIdx.x == 0 && slot == 0) {
      double st[kMaxD];
      P.out_level[probe] = probe_state(P.hdr, seedp, asset, __dmul_rn(0.5, __dadd_rn(s_lo, s_hi)), st);
      P.out_iter[probe] = s_it;
      P.out_conv[probe] = !(__dsub_rn(s_hi, s_lo) > P.tol);
    }
    cluster.sync();
    return;
  }

  if constexpr (GMODE == 3) {
    // ---- sequential bisection over a draw cache (solver 1, geometric put) ----
    // Bisection evaluates every candidate level with the same draws, so pass 0
    // walks the paths once from the first midpoint and records them
    // (walk_paths_log's RECORD), and every later pass replays the record for
    // the 2^L - 1 midpoints of the next L bisection levels at once
    // (replay_geoput_log) and then takes those L decisions: the same
    // midpoints (the same fp64 operations), continuation values, decisions
    // and iteration count as one level per pass, in 1 + (levels - 1) / L passes.
    constexpr int DL = D > 1 ? D : 2;
    constexpr int TL = kIzReplayLevels, T = kIzReplayCand;
    __shared__ double s_xl0[T], s_xm[T], s_pay[T], s_cont[T];
    double *rec = P.rec + (size_t)probe * P.n_steps * P.n_inner * 3;
    double *lo_remote = cluster.map_shared_rank(&s_lo, 0), *hi_remote = cluster.map_shared_rank(&s_hi, 0);
    for (int pass = 0;; ++pass) {
      if (*done_remote) break;
      const double lo = *lo_remote, hi = *hi_remote;  // rank 0 moves the bracket between the two barriers below only
      const int n_cand = pass == 0 ? 1 : T;
      if ((int)threadIdx.x < n_cand) {
        // node t of the complete tree of midpoints below (lo, hi), by the heap path
        double l = lo, h = hi;
        const int path = (int)threadIdx.x + 1;
        for (int tt = 31 - __clz(path) - 1; tt >= 0; --tt) {
          const double xm = __dmul_rn(0.5, __dadd_rn(l, h));
          if ((path >> tt) & 1) l = xm;
          else h = xm;
        }
        const double xm = __dmul_rn(0.5, __dadd_rn(l, h));
        double st[kMaxD];
        probe_state(P.hdr, seedp, asset, xm, st);
        s_xm[threadIdx.x] = xm;
        s_xl0[threadIdx.x] = log(st[d - 1]);
        {
          Model<double> Md{};
          Md.d = d;
          Md.payoff = P.hdr.payoff;
          Md.strike = K;
          s_pay[threadIdx.x] = payoff<0>(Md, st);  // the level's exercise value (the bisection's other side)
        }
        if (pass == 0)
          for (int i = 0; i < d; ++i) s_state[i] = st[i];
      }
      __syncthreads();
      if (pass == 0) {
        if (threadIdx.x < d) s_start[threadIdx.x] = log(s_state[threadIdx.x]);
        if (threadIdx.x == 0) s_next = p0 + blockDim.x;
        __syncthreads();
        if (p0 < p1)
          walk_paths_log<DL, LOG_GEOPUT_IZ, true>(M, s_start, log_strike, P.m, P.n_steps, key, stream,
                                                  unit_base<FAST>(0, false), p0, p1, vals, nullptr, &s_next, P.steps,
                                                  tq, rec, P.n_inner);
      } else if (p0 < p1) {
        replay_geoput_log<DL, T>(M, log_strike, P.m, P.n_steps, rec, P.n_inner, p0, p1, s_xl0, n_cand, vals, per_cta);
      }
      __syncthreads();
      fold_chunks_multi(vals, per_cta, n_cand, p1 > p0 ? p1 - p0 : 0, s_chunk);
      cluster.sync();
      if (rank == 0 && threadIdx.x < 32) {
        // every candidate's chunk sums over DSMEM, all remote loads in flight together when they
        // fit s_all (candidate-major), else candidate by candidate
        const int n_chunks = (P.n_inner + kIzFoldChunk - 1) / kIzFoldChunk;
        const int per_cta_chunks = per_cta / kIzFoldChunk;
        const bool together = n_cand * n_chunks <= kIzMaxChunks * 8;
        if (together) {
          for (int q = threadIdx.x; q < n_cand * n_chunks; q += 32) {
            const int t = q / n_chunks, g = q - t * n_chunks, r = g / per_cta_chunks;
            s_all[q] = cluster.map_shared_rank(s_chunk, r)[t * kIzMaxChunks + g - r * per_cta_chunks];
          }
          __syncwarp();
        }
        for (int t = 0; t < n_cand; ++t) {
          if (!together) gather_chunk_sums(cluster, s_chunk + t * kIzMaxChunks, csize, per_cta, P.n_inner, s_all);
          if (threadIdx.x == 0) {
            const double *cs = together ? s_all + t * n_chunks : s_all;
            double total = 0.0;
            for (int g = 0; g < n_chunks; ++g) total = __dadd_rn(total, cs[g]);
            s_cont[t] = __ddiv_rn(total, (double)P.n_inner);
          }
          __syncwarp();
        }
        if (threadIdx.x == 0) {
          double l = s_lo, h = s_hi;
          int j = 0, n_it = s_it;
          bool fin = false;
          for (int lev = 0; lev < (pass == 0 ? 1 : TL) && !fin; ++lev) {
            const double xm = s_xm[j];  // == 0.5 (l + h): the node's midpoint
            const bool exercise = __dsub_rn(s_pay[j], s_cont[j]) > 0.0;
            if (call_like == exercise) {
              h = xm;
              j = 2 * j + 1;
            } else {
              l = xm;
              j = 2 * j + 2;
            }
            ++n_it;
            fin = !(__dsub_rn(h, l) > P.tol) || n_it >= P.max_iter;
          }
          s_lo = l;
          s_hi = h;
          s_it = n_it;
          if (fin) s_done = 1;
        }
      }
      cluster.sync();
    }
  } else
  for (int it = 0;; ++it) {
    if (*done_remote) break;
    const double x = *x_remote;
    if (threadIdx.x == 0) probe_state(P.hdr, seedp, asset, x, s_state);
    __syncthreads();
    if (threadIdx.x < d) s_start[threadIdx.x] = GEOK == 2 ? (R)log(s_state[threadIdx.x]) : (R)s_state[threadIdx.x];
    if (threadIdx.x == 0) s_next = p0 + blockDim.x;
    __syncthreads();
    // fixed point: fresh slab per iteration; bisection: common random numbers
    const uint64_t draw_base = P.solver == 0 ? (uint64_t)it * slab : 0;
    const uint64_t base0 = unit_base<FAST>(draw_base, P.normals != nullptr);
    if (p0 < p1) {
      if constexpr (GMODE == 3) {
        // (handled by the draw-cache solver above)
      } else if constexpr (GEOK == 2) {
        walk_paths_log<(D > 1 ? D : 2), LOG_GEOPUT_IZ>(M, s_start, log_strike, P.m, P.n_steps, key, stream, base0, p0,
                                                       p1, vals, nullptr, &s_next, P.steps, tq);
      } else {
        walk_paths<D, FAST, GEOK ? WALK_GEO : WALK_GENERIC>(M, s_start, P.m, P.n_steps, key, stream, base0, p0, p1,
                                                            ns, vals, &s_next, nullptr, nullptr, P.steps, tq);
      }
    }
    __syncthreads();
    // fixed-order fold in 256-path chunks: the chunk sums are added in path
    // order by rank 0, so the continuation value does not depend on the
    // cluster size (i.e. on how many probes share the GPU)
    fold_chunks(vals, p1 > p0 ? p1 - p0 : 0, s_chunk);
    cluster.sync();
    int n_chunks = 0;
    if (rank == 0 && threadIdx.x < 32) n_chunks = gather_chunk_sums(cluster, s_chunk, csize, per_cta, P.n_inner, s_all);
    if (rank == 0 && threadIdx.x == 0) {
      double total = 0.0;
      for (int g = 0; g < n_chunks; ++g) total = __dadd_rn(total, s_all[g]);
      const double cont = __ddiv_rn(total, (double)P.n_inner);
      const int n_it = it + 1;
      s_it = n_it;
      if (P.solver == 0) {
        const double xn = call_like ? __dadd_rn(K, cont) : __dsub_rn(K, cont);
        const double step = __dsub_rn(xn, x);
        if (!s_armed && (call_like ? step <= 0.0 : step >= 0.0)) s_armed = 1;
        s_x = xn;
        hist[n_it] = xn;
        if (s_armed && fabs(step) < P.eps) {
          s_conv = 1;
          s_done = 1;
        } else if (n_it >= P.max_iter) {
          s_done = 1;
        }
      } else {
        double pay;
        {
          Model<double> Md{};
          Md.d = d;
          Md.payoff = P.hdr.payoff;
          Md.strike = K;
          pay = payoff<0>(Md, s_state);
        }
        const bool exercise = __dsub_rn(pay, cont) > 0.0;
        if (call_like == exercise) s_hi = x;
        else s_lo = x;
        s_x = __dmul_rn(0.5, __dadd_rn(s_lo, s_hi));
        if (!(__dsub_rn(s_hi, s_lo) > P.tol) || n_it >= P.max_iter) s_done = 1;
      }
    }
    cluster.sync();
  }
  if (rank == 0 && threadIdx.x == 0) {
    double level;
    if (P.solver == 0) {
      const int n_it = s_it;
      const int n_avg = P.avg_window < n_it + 1 ? P.avg_window : n_it + 1;
      double acc = 0.0;
      for (int i = n_it + 1 - n_avg; i <= n_it; ++i) acc = __dadd_rn(acc, hist[i]);
      level = __ddiv_rn(acc, (double)n_avg);
    } else {
      level = __dmul_rn(0.5, __dadd_rn(s_lo, s_hi));
    }
    double st[kMaxD];
    P.out_level[probe] = probe_state(P.hdr, seedp, asset, level, st);
    P.out_iter[probe] = s_it;
    P.out_conv[probe] = P.solver == 0 ? s_conv : !(__dsub_rn(s_hi, s_lo) > P.tol);
  }
  cluster.sync();  // keep rank 0's shared memory alive until every CTA is done reading it
}

// ------------------------------------------------------------- decisions ----
template <int D, bool FAST>
__global__ void __launch_bounds__(256) decisions(DecisionParams P) {
  using R = RealT<FAST>;
  extern __shared__ __align__(16) unsigned char smem[];
  const Model<R> M = load_model<R>(P.hdr, P.blob, smem);
  __syncthreads();
  const int d = M.d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P.n; i += (int64_t)gridDim.x * blockDim.x) {
    R v[D > 0 ? D : kMaxD];
    #pragma unroll
    for (int a = 0; a < dim_of<D>(d); ++a) v[a] = (R)P.states[i * d + a];
    R agg;
    const R pay = payoff_agg<D>(M, v, agg);
    P.out[i] = (pay > (R)0 && rule_stop<D>(M, P.m, v, agg)) ? 1 : 0;
  }
}

}  // namespace brm
