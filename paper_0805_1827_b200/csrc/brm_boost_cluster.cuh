// brm_boost_cluster.cuh -- parity-mode AdaBoost spread over the GPU: one
// thread-block CLUSTER per feature (boosting.py:126-206).
//
// The exact parallel cumsum of brm_boost_exact.cuh, with every per-round
// pass split across the CL CTAs of a feature's cluster and the pieces joined
// through distributed shared memory (DSMEM):
//
//   weights   CTA r owns a contiguous run of numpy's pairwise leaves and keeps
//             those weights in its shared memory: it reweights / normalises
//             its run, publishes its leaf sums (every CTA combines all of them
//             up numpy's tree, so s = w.sum() and total have the same bits
//             everywhere), and serves its weights to the other CTAs' gathers
//             over DSMEM;
//   chains    CTA r owns sorted positions [r B, (r+1) B) of each cluster tile
//             (B = kCbThreads x qt, qt <= kCbQ sized so the CTAs share the
//             positions evenly), their codes preloaded in shared memory:
//             block scans, then the CTAs' totals in rank order over DSMEM give
//             every CTA its prefix bases; the events of all CTAs are pushed in
//             order into CTA 0, whose two walker threads do the exact fp64
//             adds; every CTA then reads its bases back and forms its
//             positions' chain values;
//   splits    per-CTA argmin (with the candidate's threshold), merged by CTA 0;
//   grid      ONE grid barrier per round, then every CTA picks the same winner.
//
// The cumsum bits, the pairwise sums and the tie rules are those of
// brm_boost_exact.cuh (and of numpy); only the work split differs.
#pragma once

namespace brm {

#ifndef BRM_CB_THREADS
#define BRM_CB_THREADS 256  // variant builds time other CTA sizes (tools/build_variant.sh)
#endif
constexpr int kCbThreads = BRM_CB_THREADS;
constexpr int kCbQ = 8;                      // sorted positions per thread per tile
constexpr int kCbBlock = kCbThreads * kCbQ;  // positions per CTA per cluster tile
constexpr int kCbEvents = 512;               // events per chain per cluster tile (else serial)
constexpr int kCbMaxCluster = 8;

struct CbParams {
  int n, F, rounds, raw, cl;
  const double *xsorted;   // [F][n]
  const unsigned *code;    // [F][n] (kCodeNeg / kCodeBrk / id)
  const double *xt;        // [F][n] columns in sample order
  const double *y;         // [n]
  const double *w0;        // [n]
  double *chain_g;         // [F][2][n] multi-tile / fallback chain values
  double *wsub;            // [F*CL][n] constant-stump fallback scratch
  const int2 *leaves;
  int n_leaves;
  const int2 *children;
  const int *level_end;
  int n_levels, root;
  int qt;                  // sorted positions per thread per tile (<= kCbQ): a CTA covers qt x kCbThreads
  int slice_cap;           // elements of the largest CTA leaf run (weight slice)
  int pos_cap;             // sorted positions of a CTA over all cluster tiles
  int margin;
  double *feat_err;        // [2][F]
  int *feat_pos;           // [2][F]
  double *feat_thr;        // [2][F] the candidate's threshold (boosting.py:148)
  long long *feat_ierr;    // [2][F] fast mode: the candidate's fixed-point error
  int *out_feat;
  double *out_thr, *out_pol, *out_alpha, *out_err;
  int *out_count;
  double *out_intercept;
  const int *n_pos;
  long long *timing;       // optional per-phase clock64 totals (cluster 0, CTA 0, thread 0)
  int *n_events;           // optional: events of cluster 0, summed over rounds
  unsigned long long *n_fallback;
};

struct CbScanL {
  long long p0, p1;
  int e0, e1;
};

struct CbShared {
  // merged event lists of the cluster tile (used in CTA 0)
  long long ev_P[2][kCbEvents];
  double ev_v[2][kCbEvents];
  double ev_s[2][kCbEvents];
  // this CTA's totals over its positions (read by higher ranks)
  double tot_d[2];
  CbScanL tot_l;
  // CTA 0: exact chain values before the current cluster tile, then after it
  double carry[2];
  Cand cand;
  double cand_thr;
  double s_d[128];
  CbScanL s_l[64];
  int elo[kCbMaxCluster + 1];       // first element of each CTA's weight slice
  const double *rw[kCbMaxCluster];  // each CTA's weight slice (DSMEM), indexed by element id
};

// leaves [lo, hi) of CTA r out of cl
__host__ __device__ __forceinline__ void cb_leaf_run(int L, int cl, int r, int &lo, int &hi) {
  lo = (int)((long long)r * L / cl);
  hi = (int)((long long)(r + 1) * L / cl);
}

__device__ __forceinline__ int cb_owner(int l, int L, int cl) {
  // inverse of cb_leaf_run: the r with lo(r) <= l < lo(r+1)
  int r = (int)(((long long)l * cl) / L);
  while (r + 1 < cl && (long long)(r + 1) * L / cl <= l) ++r;
  while (r > 0 && (long long)r * L / cl > l) --r;
  return r;
}

// a / b with the bits of IEEE division: the straight-line fast path of
// __ddiv_rn (div_nb) when no operand is near the exponent limits
__device__ __forceinline__ double cb_div(double a, double b) {
  const double fa = fabs(a), fb = fabs(b);
  return (fa >= 0x1p-900 && fa <= 0x1p900 && fb >= 0x1p-100 && fb <= 0x1p100) ? div_nb(a, b) : __ddiv_rn(a, b);
}

// weight of sample id, from the CTA whose slice holds it (DSMEM)
__device__ __forceinline__ double cb_weight(const CbShared &sh, int cl, int id) {
  int o = 0;
#pragma unroll
  for (int k = 1; k < kCbMaxCluster; ++k) o += (k < cl && id >= sh.elo[k]) ? 1 : 0;
  return sh.rw[o][id];
}

// numpy's tree over the leaf sums in s_node[0..L), combined by one warp
// (a __syncwarp per level instead of a CTA barrier); every thread gets the root.
__device__ __forceinline__ double cb_tree_warp(const PwView &T, double *s_node) {
  __syncthreads();
  if (threadIdx.x < 32) {
    const int L = T.L;
    int lo = 0;
    for (int h = 0; h < T.n_levels; ++h) {
      const int hi = T.level_end[h];
      for (int j = lo + (int)threadIdx.x; j < hi; j += 32) {
        const int2 c = T.children[j];
        s_node[L + j] = __dadd_rn(s_node[c.x], s_node[c.y]);
      }
      lo = hi;
      __syncwarp();
    }
  }
  __syncthreads();
  return s_node[T.root];
}

// Gather every leaf sum of the cluster (leaf l from its owner's s_leaf) into
// s_node[0..L) and combine numpy's tree.  Every thread gets the root.  The
// callers alternate two s_leaf buffers, so a CTA that runs ahead never
// overwrites leaf sums another CTA is still reading (consecutive uses of one
// buffer are separated by the other buffer's cluster barrier).
__device__ __forceinline__ double cb_tree(cg::cluster_group &cluster, const PwView &T, double *s_leaf,
                                          double *s_node, int cl) {
  cluster.sync();  // every CTA has published its leaf sums
  for (int l = threadIdx.x; l < T.L; l += blockDim.x) {
    const int o = cb_owner(l, T.L, cl);
    s_node[l] = *cluster.map_shared_rank(s_leaf + l, o);
  }
  return cb_tree_warp(T, s_node);
}

// Block-wide exclusive scans of two fp64 values per thread sharing the
// barriers.  As ex_scan: the exclusive value sums EARLIER elements only, so
// each rounding error is relative to the exclusive prefix.
__device__ __forceinline__ void cb_scan_d2(double &x0, double &x1, double *s_w, double &t0, double &t1) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double a = x0, b = x1;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double oa = __shfl_up_sync(0xffffffffu, a, off), ob = __shfl_up_sync(0xffffffffu, b, off);
    if (lane >= off) {
      a = a + oa;
      b = b + ob;
    }
  }
  if (lane == 31) {
    s_w[wid] = a;
    s_w[32 + wid] = b;
  }
  __syncthreads();
  if (wid == 0) {
    double ta = lane < nw ? s_w[lane] : 0.0, tb = lane < nw ? s_w[32 + lane] : 0.0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const double oa = __shfl_up_sync(0xffffffffu, ta, off), ob = __shfl_up_sync(0xffffffffu, tb, off);
      if (lane >= off) {
        ta = ta + oa;
        tb = tb + ob;
      }
    }
    if (lane < nw) {
      s_w[64 + lane] = ta;
      s_w[96 + lane] = tb;
    }
  }
  __syncthreads();
  const double ba = wid > 0 ? s_w[64 + wid - 1] : 0.0, bb = wid > 0 ? s_w[96 + wid - 1] : 0.0;
  t0 = s_w[64 + nw - 1];
  t1 = s_w[96 + nw - 1];
  const double ia = __shfl_up_sync(0xffffffffu, a, 1), ib = __shfl_up_sync(0xffffffffu, b, 1);
  x0 = lane == 0 ? ba : ba + ia;
  x1 = lane == 0 ? bb : bb + ib;
}

__device__ __forceinline__ CbScanL cb_shfl_up(const CbScanL &a, int off) {
  CbScanL o;
  o.p0 = __shfl_up_sync(0xffffffffu, a.p0, off);
  o.p1 = __shfl_up_sync(0xffffffffu, a.p1, off);
  o.e0 = __shfl_up_sync(0xffffffffu, a.e0, off);
  o.e1 = __shfl_up_sync(0xffffffffu, a.e1, off);
  return o;
}

__device__ __forceinline__ void cb_add(CbScanL &a, const CbScanL &b) {
  a.p0 += b.p0;
  a.p1 += b.p1;
  a.e0 += b.e0;
  a.e1 += b.e1;
}

// Block-wide exclusive scan of the integer increments and event counts.
__device__ __forceinline__ CbScanL cb_scan_l(const CbScanL &x, CbScanL *s_w, CbScanL &tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  CbScanL a = x;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const CbScanL o = cb_shfl_up(a, off);
    if (lane >= off) cb_add(a, o);
  }
  if (lane == 31) s_w[wid] = a;
  __syncthreads();
  if (wid == 0) {
    CbScanL t = lane < nw ? s_w[lane] : CbScanL{0, 0, 0, 0};
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const CbScanL o = cb_shfl_up(t, off);
      if (lane >= off) cb_add(t, o);
    }
    if (lane < nw) s_w[32 + lane] = t;
  }
  __syncthreads();
  CbScanL e = wid > 0 ? s_w[32 + wid - 1] : CbScanL{0, 0, 0, 0};
  tot = s_w[32 + nw - 1];
  const CbScanL in = cb_shfl_up(a, 1);
  if (lane > 0) cb_add(e, in);
  return e;
}

__global__ void __launch_bounds__(kCbThreads, 1) boost_cluster_kernel(CbParams P) {
  cg::grid_group grid = cg::this_grid();
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ CbShared sh;
  __shared__ Cand s_cand[kCbThreads / 32];
  __shared__ double s_cthr[kCbThreads / 32];
  __shared__ int s_stop, s_feat;
  __shared__ double s_alpha, s_thr, s_pol, s_err;

  const int n = P.n, F = P.F, cl = P.cl;
  const int r = (int)cluster.block_rank();
  const int f = blockIdx.x / cl;
  const int n_pos_all = *P.n_pos;
  if (one_class_exit(P.raw, n, n_pos_all, P.out_count, P.out_intercept)) return;
  const int L = P.n_leaves;
  const int qt = P.qt;
  const int cblock = qt * kCbThreads;  // positions per CTA per cluster tile
  const int ctile = cl * cblock;       // positions per cluster tile
  const int n_tiles = (n + ctile - 1) / ctile;
  // dynamic shared memory: s_node[2L] | s_leaf[2][L] | weight slice | codes | y slice | tree tables
  double *s_node = reinterpret_cast<double *>(smem_raw);
  double *s_leaf = s_node + 2 * L;  // [2][L]: alternating buffers (see cb_tree)
  double *s_leaf_b = s_leaf + L;
  double *wsl = s_leaf + 2 * L;
  unsigned *s_code = reinterpret_cast<unsigned *>(wsl + P.slice_cap);
  signed char *s_y = reinterpret_cast<signed char *>(s_code + P.pos_cap);
  int2 *s_leaves = reinterpret_cast<int2 *>(smem_raw + ((sizeof(double) * (4 * (size_t)L + P.slice_cap) +
                                                         sizeof(unsigned) * P.pos_cap + P.slice_cap + 15) &
                                                        ~(size_t)15));
  int2 *s_children = s_leaves + L;
  int *s_level = reinterpret_cast<int *>(s_children + max(L - 1, 0));
  for (int i = threadIdx.x; i < L; i += blockDim.x) s_leaves[i] = P.leaves[i];
  for (int i = threadIdx.x; i < L - 1; i += blockDim.x) s_children[i] = P.children[i];
  for (int i = threadIdx.x; i < P.n_levels; i += blockDim.x) s_level[i] = P.level_end[i];
  const PwView T{s_leaves, s_children, s_level, L, P.n_levels, P.root};
  int l_lo, l_hi;
  cb_leaf_run(L, cl, r, l_lo, l_hi);
  const int e_lo = l_lo < L ? P.leaves[l_lo].x : n;  // this CTA's elements [e_lo, e_hi)
  const int e_hi = l_hi > l_lo ? P.leaves[l_hi - 1].x + P.leaves[l_hi - 1].y : e_lo;
  double *wloc = wsl - e_lo;  // indexed by element id within [e_lo, e_hi)
  const unsigned *code = P.code + (size_t)f * n;
  double *chain = P.chain_g + (size_t)f * 2 * n;
  const bool multi = n_tiles > 1;
  // this CTA's sorted positions of every tile, and its slice's labels
  for (int t = 0; t < n_tiles; ++t)
    for (int j = threadIdx.x; j < cblock; j += blockDim.x) {
      const int i = t * ctile + r * cblock + j;
      if (i < n) s_code[t * cblock + j] = __ldg(code + i);
    }
  for (int i = e_lo + (int)threadIdx.x; i < e_hi; i += blockDim.x) s_y[i - e_lo] = P.y[i] > 0.0 ? 1 : -1;
  if (threadIdx.x <= kCbMaxCluster) {
    const int o = threadIdx.x;
    int lo = 0, hi = 0;
    cb_leaf_run(L, cl, min(o, cl - 1), lo, hi);
    sh.elo[o] = o >= cl ? n : (lo < L ? P.leaves[lo].x : n);
    if (o < cl) sh.rw[o] = cluster.map_shared_rank(wsl, o) - sh.elo[o];
  }
  CbShared *sh0 = cluster.map_shared_rank(&sh, 0);
  const long long margin = P.margin;
  int count = 0;
  __syncthreads();

  const bool timed = P.timing && blockIdx.x == 0 && threadIdx.x == 0;
  long long t_mark = timed ? clock64() : 0, tacc[16] = {0};
#define BRM_CB_T(k)                   \
  if (timed) {                        \
    const long long now_ = clock64(); \
    tacc[k] += now_ - t_mark;         \
    t_mark = now_;                    \
  }

  // round 0: the given weights; total = w.sum() (pairwise)
  pw_leaf_sums(T, P.w0, l_lo, l_hi, s_leaf, PwIdentity{}, [&](int i, double v) { wloc[i] = v; });
  double total = cb_tree(cluster, T, s_leaf, s_node, cl);
  BRM_CB_T(5);

  for (int round = 0; round < P.rounds; ++round) {
    // ---- chains and splits of feature f over the cluster -----------------
    Cand best{__longlong_as_double(0x7ff0000000000000LL), 0x7fffffff};
    bool via_global = multi;
    for (int t0 = 0, tile = 0; t0 < n; t0 += ctile, ++tile) {
      double cin0 = 0.0, cin1 = 0.0;
      if (tile > 0) {
        cluster.sync();  // CTA 0's carry of this tile is final
        cin0 = sh0->carry[0];
        cin1 = sh0->carry[1];
      }
      const int i0 = t0 + r * cblock + threadIdx.x * qt;
      const int q = max(0, min(qt, n - i0));
      const unsigned *tc = s_code + tile * cblock + threadIdx.x * qt;
      double v[kCbQ];
      unsigned neg_mask = 0, brk_mask = 0;
#pragma unroll
      for (int k = 0; k < kCbQ; ++k) {
        v[k] = 0.0;
        if (k < q) {
          const unsigned c = tc[k];
          v[k] = cb_weight(sh, cl, (int)(c & kCodeId));
          if (c & kCodeNeg) neg_mask |= 1u << k;
          if (c & kCodeBrk) brk_mask |= 1u << k;
        }
      }
      double x0 = 0.0, x1 = 0.0;
#pragma unroll
      for (int k = 0; k < kCbQ; ++k) {
        if ((neg_mask >> k) & 1u) x1 += v[k];
        else x0 += v[k];
      }
      double td0, td1;
      cb_scan_d2(x0, x1, sh.s_d, td0, td1);
      if (threadIdx.x == 0) {
        sh.tot_d[0] = td0;
        sh.tot_d[1] = td1;
      }
      BRM_CB_T(6);
      cluster.sync();
      BRM_CB_T(7);
      // approximate prefix bases: lower ranks' totals in rank order (every
      // term is a sum of earlier elements, so the error bound holds)
      double b0 = cin0, b1 = cin1;
      for (int o = 0; o < r; ++o) {
        const CbShared *so = cluster.map_shared_rank(&sh, o);
        b0 += so->tot_d[0];
        b1 += so->tot_d[1];
      }
      const double as0 = b0 + x0, as1 = b1 + x1;
      // plain elements, integer increments, event counts
      unsigned plain_mask = 0;
      CbScanL mine{0, 0, 0, 0};
      {
        double a0 = as0, a1 = as1;
#pragma unroll
        for (int k = 0; k < kCbQ; ++k) {
          if (k < q) {
            const bool ng = (neg_mask >> k) & 1u;
            const double a = ng ? a1 : a0;
            const double b = a + v[k];
            bool plain = ex_certain(a, margin) && ex_certain(b, margin) && ex_expo(a) == ex_expo(b);
            long long ri = 0;
            if (plain) {
              const double t = ex_scaled(v[k], a);
              plain = (t - floor(t)) != 0.5;
              ri = __double2ll_rn(t);
            }
            if (plain) {
              plain_mask |= 1u << k;
              if (ng) mine.p1 += ri;
              else mine.p0 += ri;
            } else if (ng) {
              ++mine.e1;
            } else {
              ++mine.e0;
            }
            if (ng) a1 = b;
            else a0 = b;
          }
        }
      }
      CbScanL tl;
      const CbScanL ex = cb_scan_l(mine, sh.s_l, tl);
      if (threadIdx.x == 0) sh.tot_l = tl;
      BRM_CB_T(8);
      cluster.sync();
      BRM_CB_T(9);
      CbScanL base{0, 0, 0, 0}, all{0, 0, 0, 0};
      for (int o = 0; o < cl; ++o) {
        const CbScanL to = cluster.map_shared_rank(&sh, o)->tot_l;
        if (o < r) cb_add(base, to);
        cb_add(all, to);
      }
      const long long P0 = base.p0 + ex.p0, P1 = base.p1 + ex.p1;
      const int E0 = base.e0 + ex.e0, E1 = base.e1 + ex.e1;
      if (all.e0 > kCbEvents || all.e1 > kCbEvents) {
        // event-list overflow (rare): CTA 0 walks the tile serially into chain_g
        if (r == 0 && threadIdx.x == 0) {
          double s0 = cin0, s1 = cin1;
          for (int i = t0; i < min(t0 + ctile, n); ++i) {
            const unsigned cd = code[i];
            const double w = cb_weight(sh, cl, (int)(cd & kCodeId));
            if (cd & kCodeNeg) s1 = __dadd_rn(s1, w);
            else s0 = __dadd_rn(s0, w);
            chain[i] = s0;
            chain[n + i] = s1;
          }
          sh.carry[0] = s0;
          sh.carry[1] = s1;
          if (P.n_fallback) atomicAdd(P.n_fallback, 1ull);
        }
        via_global = true;
        cluster.sync();  // carry (and chain_g) published
        continue;
      }
      // push this CTA's events, in order, into CTA 0's lists
      {
        double a0 = as0, a1 = as1;
        long long p0 = P0, p1 = P1;
        int e0 = E0, e1 = E1;
#pragma unroll
        for (int k = 0; k < kCbQ; ++k) {
          if (k < q) {
            const bool ng = (neg_mask >> k) & 1u;
            const double a = ng ? a1 : a0;
            if ((plain_mask >> k) & 1u) {
              const long long ri = __double2ll_rn(ex_scaled(v[k], a));
              if (ng) p1 += ri;
              else p0 += ri;
            } else if (ng) {
              sh0->ev_P[1][e1] = p1;
              sh0->ev_v[1][e1++] = v[k];
            } else {
              sh0->ev_P[0][e0] = p0;
              sh0->ev_v[0][e0++] = v[k];
            }
            if (ng) a1 = a + v[k];
            else a0 = a + v[k];
          }
        }
      }
      BRM_CB_T(10);
      cluster.sync();
      BRM_CB_T(11);
      // CTA 0: walk the tile's events, one thread per chain
      if (r == 0 && (threadIdx.x & 31) == 0 && threadIdx.x < 64) {
        const int c = threadIdx.x >> 5;
        const int ne = c ? all.e1 : all.e0;
        double s = c ? cin1 : cin0;
        long long pp = 0;
        long long p_next = ne > 0 ? sh.ev_P[c][0] : 0;
        double v_next = ne > 0 ? sh.ev_v[c][0] : 0.0;
        for (int k = 0; k < ne; ++k) {
          const long long p = p_next;
          const double vk = v_next;
          if (k + 1 < ne) {  // the next event's operands load under this one's adds
            p_next = sh.ev_P[c][k + 1];
            v_next = sh.ev_v[c][k + 1];
          }
          if (p != pp) s = __dadd_rn(s, __dmul_rn((double)(p - pp), ex_ulp(s)));
          s = __dadd_rn(s, vk);
          sh.ev_s[c][k] = s;
          pp = p;
        }
        const long long pt = c ? all.p1 : all.p0;
        if (pt != pp) s = __dadd_rn(s, __dmul_rn((double)(pt - pp), ex_ulp(s)));
        sh.carry[c] = s;
        if (P.n_events && blockIdx.x == 0) atomicAdd(P.n_events + c, ne);
      }
      BRM_CB_T(12);
      cluster.sync();
      BRM_CB_T(13);
      // this CTA's positions
      const double tot_neg = sh0->carry[1];  // the final negative chain value when this is the only tile
      double bs0 = cin0, bs1 = cin1;
      long long bp0 = 0, bp1 = 0;
      if (E0 > 0) {
        bs0 = sh0->ev_s[0][E0 - 1];
        bp0 = sh0->ev_P[0][E0 - 1];
      }
      if (E1 > 0) {
        bs1 = sh0->ev_s[1][E1 - 1];
        bp1 = sh0->ev_P[1][E1 - 1];
      }
      long long p0 = P0, p1 = P1;
      int e0 = E0, e1 = E1;
      double cur0 = p0 != bp0 ? __dadd_rn(bs0, __dmul_rn((double)(p0 - bp0), ex_ulp(bs0))) : bs0;
      double cur1 = p1 != bp1 ? __dadd_rn(bs1, __dmul_rn((double)(p1 - bp1), ex_ulp(bs1))) : bs1;
#pragma unroll
      for (int k = 0; k < kCbQ; ++k) {
        if (k < q) {
          const bool ng = (neg_mask >> k) & 1u;
          if ((plain_mask >> k) & 1u) {
            if (ng) {
              p1 += __double2ll_rn(ex_scaled(v[k], bs1));
              cur1 = __dadd_rn(bs1, __dmul_rn((double)(p1 - bp1), ex_ulp(bs1)));
            } else {
              p0 += __double2ll_rn(ex_scaled(v[k], bs0));
              cur0 = __dadd_rn(bs0, __dmul_rn((double)(p0 - bp0), ex_ulp(bs0)));
            }
          } else if (ng) {
            cur1 = bs1 = sh0->ev_s[1][e1];
            bp1 = p1;
            ++e1;
          } else {
            cur0 = bs0 = sh0->ev_s[0][e0];
            bp0 = p0;
            ++e0;
          }
          const int i = i0 + k;
          if (multi) {
            chain[i] = cur0;
            chain[n + i] = cur1;
          } else if (((brk_mask >> k) & 1u) && i < n - 1) {
            ex_split_at(i, cur0, cur1, tot_neg, total, best);
          }
        }
      }
    }
    BRM_CB_T(0);
    if (via_global) {
      cluster.sync();  // every chain value is in chain_g; CTA 0's carry is final
      best = Cand{__longlong_as_double(0x7ff0000000000000LL), 0x7fffffff};
      const double tot_neg = sh0->carry[1];
      // this CTA's share of the positions, ascending
      const int per = (n + cl - 1) / cl;
      for (int i = r * per + threadIdx.x; i < min((r + 1) * per, n - 1); i += blockDim.x)
        if (__ldg(code + i) & kCodeBrk) ex_split_at(i, __ldcg(chain + i), __ldcg(chain + n + i), tot_neg, total, best);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      Cand o;
      o.err = __shfl_down_sync(0xffffffffu, best.err, off);
      o.key = __shfl_down_sync(0xffffffffu, best.key, off);
      if (cand_less(o, best)) best = o;
    }
    if ((threadIdx.x & 31) == 0) {
      s_cand[threadIdx.x >> 5] = best;
      // the warp's candidate threshold, midpoint of the sorted values (boosting.py:148)
      if (best.key != 0x7fffffff) {
        const double *xf = P.xsorted + (size_t)f * n;
        const int i = best.key >> 1;
        s_cthr[threadIdx.x >> 5] = __dmul_rn(0.5, __dadd_rn(__ldg(xf + i), __ldg(xf + i + 1)));
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double thr = s_cthr[0];
      for (int wi = 1; wi < (int)blockDim.x / 32; ++wi)
        if (cand_less(s_cand[wi], best)) {
          best = s_cand[wi];
          thr = s_cthr[wi];
        }
      sh.cand = best;
      sh.cand_thr = thr;
    }
    cluster.sync();
    if (r == 0 && threadIdx.x == 0) {
      Cand b = sh.cand;
      double thr = sh.cand_thr;
      for (int o = 1; o < cl; ++o) {
        const CbShared *so = cluster.map_shared_rank(&sh, o);
        const Cand co = so->cand;
        if (cand_less(co, b)) {
          b = co;
          thr = so->cand_thr;
        }
      }
      // double-buffered by round: with one grid barrier per round a cluster
      // may publish round r+1 while another still reads round r
      P.feat_err[(round & 1) * F + f] = b.err;
      P.feat_pos[(round & 1) * F + f] = b.key;
      P.feat_thr[(round & 1) * F + f] = thr;
    }
    BRM_CB_T(1);
    grid.sync();
    BRM_CB_T(2);
    // ---- the winner (every CTA, same answer) -----------------------------
    double be = __longlong_as_double(0x7ff0000000000000LL), bt = 0.0;
    int bf = 0x7fffffff, bk = 0;
    if (threadIdx.x < 32) {
      for (int g = threadIdx.x; g < F; g += 32) {
        const int pos = __ldcg(P.feat_pos + (round & 1) * F + g);
        const double e = __ldcg(P.feat_err + (round & 1) * F + g);
        const double tg = __ldcg(P.feat_thr + (round & 1) * F + g);
        if (pos != 0x7fffffff && e < be) {
          be = e;
          bf = g;
          bk = pos;
          bt = tg;
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double oe = __shfl_down_sync(0xffffffffu, be, off);
        const int of = __shfl_down_sync(0xffffffffu, bf, off);
        const int ok = __shfl_down_sync(0xffffffffu, bk, off);
        const double ot = __shfl_down_sync(0xffffffffu, bt, off);
        if (oe < be || (oe == be && of < bf)) {
          be = oe;
          bf = of;
          bk = ok;
          bt = ot;
        }
      }
    }
    if (threadIdx.x == 0) {
      if (bf == 0x7fffffff) {
        s_stop = 2;
        s_feat = 0;
        s_thr = __longlong_as_double(0xfff0000000000000LL);
      } else {
        s_feat = bf;
        s_thr = bt;
        s_pol = (bk & 1) ? -1.0 : 1.0;
        s_err = be;
        s_stop = 0;
      }
    }
    __syncthreads();
    if (s_stop == 2) {
      // every feature constant (boosting.py:166-170): pol = +1 iff sum(w*y) >= 0,
      // err = sum(w[y != pol]), both in numpy's pairwise order -- by every CTA
      // over the cluster's weights (rare path)
      double *ws = P.wsub + (size_t)blockIdx.x * n;
      for (int i = threadIdx.x; i < n; i += blockDim.x) ws[i] = __dmul_rn(cb_weight(sh, cl, i), P.y[i]);
      __syncthreads();
      pw_leaf_sums(T, ws, 0, L, s_node, PwIdentity{});
      const double swy = cb_tree_warp(T, s_node);
      const double pol = swy >= 0.0 ? 1.0 : -1.0;
      if (threadIdx.x == 0) {
        int k = 0;
        for (int i = 0; i < n; ++i)
          if (P.y[i] != pol) ws[k++] = cb_weight(sh, cl, i);
        s_pol = pol;
        s_err = pw_serial(ws, k);
        s_stop = 0;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const double err = s_err;
      if (P.raw) {
        if (blockIdx.x == 0) {
          P.out_feat[0] = s_feat;
          P.out_thr[0] = s_thr;
          P.out_pol[0] = s_pol;
          P.out_alpha[0] = 1.0;
          P.out_err[0] = err;
        }
        s_stop = 3;
      } else if (err >= 0.5) {
        s_stop = 1;
      } else {
        const double a = __dmul_rn(0.5, log(__ddiv_rn(__dsub_rn(1.0, err), err > 1e-10 ? err : 1e-10)));
        s_alpha = a;
        if (blockIdx.x == 0) {
          P.out_feat[count] = s_feat;
          P.out_thr[count] = s_thr;
          P.out_pol[count] = s_pol;
          P.out_alpha[count] = a;
          P.out_err[count] = err;
        }
        s_stop = err <= 0.0 ? 3 : 0;
      }
    }
    __syncthreads();
    if (s_stop == 1) break;
    ++count;
    if (s_stop == 3 || round + 1 == P.rounds) break;
    BRM_CB_T(3);
    // ---- reweight this CTA's leaf run; w /= w.sum() -----------------------
    {
      const double a = s_alpha, thr = s_thr, pol = s_pol;
      const double *xcol = P.xt + (size_t)s_feat * n;
      const double e_agree = exp(-a), e_miss = exp(a);
      pw_leaf_sums(
          T, wloc, l_lo, l_hi, s_leaf_b,
          [&](int i, double x) {
            const double pred = __ldg(xcol + i) > thr ? pol : -pol;
            return __dmul_rn(x, ((double)s_y[i - e_lo] * pred > 0.0) ? e_agree : e_miss);
          },
          [&](int i, double v) { wloc[i] = v; });
      BRM_CB_T(14);
      const double s = cb_tree(cluster, T, s_leaf_b, s_node, cl);
      BRM_CB_T(15);
      pw_leaf_sums(
          T, wloc, l_lo, l_hi, s_leaf, [&](int, double x) { return cb_div(x, s); },
          [&](int i, double v) { wloc[i] = v; });
      total = cb_tree(cluster, T, s_leaf, s_node, cl);
    }
    BRM_CB_T(4);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) write_result(count, n, n_pos_all, P.out_count, P.out_intercept);
  if (timed)
    for (int k = 0; k < 16; ++k) P.timing[k] = tacc[k];
#undef BRM_CB_T
  cluster.sync();  // keep this CTA's shared memory alive until the cluster is done with it
}

// Dynamic shared memory of boost_cluster_kernel.
inline size_t cb_smem_bytes(int L, int n_children, int n_levels, int slice_cap, int pos_cap) {
  const size_t head = sizeof(double) * (4 * (size_t)L + slice_cap) + sizeof(unsigned) * pos_cap + slice_cap;
  return ((head + 15) & ~(size_t)15) + sizeof(int2) * (L + n_children) + sizeof(int) * n_levels;
}

// ------------------------------------------------------------- fast mode ----
// BRM_MODE_FAST AdaBoost on the same cluster layout: the split search scans
// weights quantised to 62-bit fixed point (W_i = rint(w_i / s 2^62)), so every
// prefix is an exact integer scan -- no events, no walker -- and the result
// is identical for any schedule.  The first weight sum s is numpy's pairwise
// order over the leaves (every CTA combines the same leaf sums); after a round
// the reweighted weights sum to e^-a (1 - err) + e^a err with err the winner's
// error over the quantised weights, so every CTA forms the next s from the
// integers it already holds -- no pass over the weights, no leaf exchange --
// and the fit does not depend on the cluster size.  Statistically equivalent
// to the reference, not bit-identical to numpy
// (tests/test_gpu_config_parity.py, fast mode).
constexpr double kFixC = 4611686018427387904.0;  // 2^62

struct CbFastCand {
  long long dmin, dmax;
  int kmin, kmax;
};

// MINB = 2 (many features, C4: F > SMs / 8): two CTAs per SM, so a feature's cluster is twice as
// wide and a round covers the sorted positions in half as many tiles; MINB = 1 elsewhere (the
// 128-register cap costs the small fits 2-4%).
template <int MINB>
__global__ void __launch_bounds__(kCbThreads, MINB) boost_fast_cluster_kernel(CbParams P) {
  cg::grid_group grid = cg::this_grid();
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ CbShared sh;
  __shared__ CbFastCand s_fc[kCbThreads / 32];
  __shared__ CbFastCand s_ccand;
  __shared__ double s_cthr[2];
  __shared__ int s_stop, s_feat;
  __shared__ double s_alpha, s_thr, s_pol, s_err;
  __shared__ double s_eag, s_emi, s_sum;  // exp(-alpha), exp(alpha), the reweighted weights' sum
  __shared__ long long s_be;
  __shared__ int s_bf;

  const int n = P.n, F = P.F, cl = P.cl;
  const int r = (int)cluster.block_rank();
  const int f = blockIdx.x / cl;
  const int n_pos_all = *P.n_pos;
  if (one_class_exit(P.raw, n, n_pos_all, P.out_count, P.out_intercept)) return;
  const int L = P.n_leaves;
  const int qt = P.qt;
  const int cblock = qt * kCbThreads;
  const int ctile = cl * cblock;
  const int n_tiles = (n + ctile - 1) / ctile;
  double *s_node = reinterpret_cast<double *>(smem_raw);
  double *s_leaf = s_node + 2 * L;
  double *wsl = s_leaf + 2 * L;
  unsigned *s_code = reinterpret_cast<unsigned *>(wsl + P.slice_cap);
  signed char *s_y = reinterpret_cast<signed char *>(s_code + P.pos_cap);
  int2 *s_leaves = reinterpret_cast<int2 *>(smem_raw + ((sizeof(double) * (4 * (size_t)L + P.slice_cap) +
                                                         sizeof(unsigned) * P.pos_cap + P.slice_cap + 15) &
                                                        ~(size_t)15));
  int2 *s_children = s_leaves + L;
  int *s_level = reinterpret_cast<int *>(s_children + max(L - 1, 0));
  for (int i = threadIdx.x; i < L; i += blockDim.x) s_leaves[i] = P.leaves[i];
  for (int i = threadIdx.x; i < L - 1; i += blockDim.x) s_children[i] = P.children[i];
  for (int i = threadIdx.x; i < P.n_levels; i += blockDim.x) s_level[i] = P.level_end[i];
  const PwView T{s_leaves, s_children, s_level, L, P.n_levels, P.root};
  int l_lo, l_hi;
  cb_leaf_run(L, cl, r, l_lo, l_hi);
  const int e_lo = l_lo < L ? P.leaves[l_lo].x : n;
  const int e_hi = l_hi > l_lo ? P.leaves[l_hi - 1].x + P.leaves[l_hi - 1].y : e_lo;
  double *wloc = wsl - e_lo;
  const unsigned *code = P.code + (size_t)f * n;
  for (int t = 0; t < n_tiles; ++t)
    for (int j = threadIdx.x; j < cblock; j += blockDim.x) {
      const int i = t * ctile + r * cblock + j;
      if (i < n) s_code[t * cblock + j] = __ldg(code + i);
    }
  for (int i = e_lo + (int)threadIdx.x; i < e_hi; i += blockDim.x) s_y[i - e_lo] = P.y[i] > 0.0 ? 1 : -1;
  if (threadIdx.x <= kCbMaxCluster) {
    const int o = threadIdx.x;
    int lo = 0, hi = 0;
    cb_leaf_run(L, cl, min(o, cl - 1), lo, hi);
    sh.elo[o] = o >= cl ? n : (lo < L ? P.leaves[lo].x : n);
    if (o < cl) sh.rw[o] = cluster.map_shared_rank(wsl, o) - sh.elo[o];
  }
  int count = 0;
  __syncthreads();
  pw_leaf_sums(T, P.w0, l_lo, l_hi, s_leaf, PwIdentity{}, [&](int i, double v) { wloc[i] = v; });
  double ssum = cb_tree(cluster, T, s_leaf, s_node, cl);

  for (int round = 0; round < P.rounds; ++round) {
    const double inv_s = 1.0 / ssum;
    // ---- integer split scan of feature f over the cluster -----------------
    long long dmin = LLONG_MAX, dmax = LLONG_MIN;
    int kmin = INT_MAX, kmax = INT_MAX;
    long long carry_p = 0, carry_n = 0;
    for (int t0 = 0, tile = 0; t0 < n; t0 += ctile, ++tile) {
      const int i0 = t0 + r * cblock + threadIdx.x * qt;
      const int q = max(0, min(qt, n - i0));
      const unsigned *tc = s_code + tile * cblock + threadIdx.x * qt;
      long long W[kCbQ];
      unsigned neg_mask = 0, brk_mask = 0;
      CbScanL mine{0, 0, 0, 0};
#pragma unroll
      for (int k = 0; k < kCbQ; ++k) {
        W[k] = 0;
        if (k < q) {
          const unsigned c = tc[k];
          W[k] = __double2ll_rn(cb_weight(sh, cl, (int)(c & kCodeId)) * inv_s * kFixC);
          if (c & kCodeNeg) {
            neg_mask |= 1u << k;
            mine.p1 += W[k];
          } else {
            mine.p0 += W[k];
          }
          if (c & kCodeBrk) brk_mask |= 1u << k;
        }
      }
      CbScanL tl;
      const CbScanL ex = cb_scan_l(mine, sh.s_l, tl);
      if (threadIdx.x == 0) sh.tot_l = tl;
      cluster.sync();
      long long bp = carry_p, bn = carry_n, ap = 0, an = 0;
      for (int o = 0; o < cl; ++o) {
        const CbScanL to = cluster.map_shared_rank(&sh, o)->tot_l;
        if (o < r) {
          bp += to.p0;
          bn += to.p1;
        }
        ap += to.p0;
        an += to.p1;
      }
      long long cp = bp + ex.p0, cn = bn + ex.p1;
#pragma unroll
      for (int k = 0; k < kCbQ; ++k) {
        if (k < q) {
          if ((neg_mask >> k) & 1u) cn += W[k];
          else cp += W[k];
          const int i = i0 + k;
          if (((brk_mask >> k) & 1u) && i < n - 1) {
            const long long dd = cp - cn;
            if (dd < dmin) dmin = dd, kmin = 2 * i;  // positions ascend: first hit keeps the lowest key
            if (dd > dmax) dmax = dd, kmax = 2 * i + 1;
          }
        }
      }
      carry_p += ap;
      carry_n += an;
      // tot_l is reused by the next tile (after the last one, the next write is a grid barrier away)
      if (t0 + ctile < n) cluster.sync();
    }
    const long long tot_pos = carry_p, tot_neg = carry_n, total = tot_pos + tot_neg;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const long long o1 = __shfl_down_sync(0xffffffffu, dmin, off), o2 = __shfl_down_sync(0xffffffffu, dmax, off);
      const int k1 = __shfl_down_sync(0xffffffffu, kmin, off), k2 = __shfl_down_sync(0xffffffffu, kmax, off);
      if (o1 < dmin || (o1 == dmin && k1 < kmin)) dmin = o1, kmin = k1;
      if (o2 > dmax || (o2 == dmax && k2 < kmax)) dmax = o2, kmax = k2;
    }
    if ((threadIdx.x & 31) == 0) s_fc[threadIdx.x >> 5] = CbFastCand{dmin, dmax, kmin, kmax};
    __syncthreads();
    if (threadIdx.x == 0) {
      CbFastCand c = s_fc[0];
      for (int w = 1; w < (int)blockDim.x / 32; ++w) {
        const CbFastCand o = s_fc[w];
        if (o.dmin < c.dmin || (o.dmin == c.dmin && o.kmin < c.kmin)) c.dmin = o.dmin, c.kmin = o.kmin;
        if (o.dmax > c.dmax || (o.dmax == c.dmax && o.kmax < c.kmax)) c.dmax = o.dmax, c.kmax = o.kmax;
      }
      s_ccand = c;
    }
    cluster.sync();
    if (r == 0 && threadIdx.x == 0) {
      CbFastCand c = s_ccand;
      for (int o = 1; o < cl; ++o) {
        const CbFastCand oc = *cluster.map_shared_rank(&s_ccand, o);
        if (oc.dmin < c.dmin || (oc.dmin == c.dmin && oc.kmin < c.kmin)) c.dmin = oc.dmin, c.kmin = oc.kmin;
        if (oc.dmax > c.dmax || (oc.dmax == c.dmax && oc.kmax < c.kmax)) c.dmax = oc.dmax, c.kmax = oc.kmax;
      }
      // err+ = d + tot_neg, err- = tot_pos - d; lowest key at equal error
      long long best_err = LLONG_MAX;
      int best_key = INT_MAX;
      if (c.kmin != INT_MAX) best_err = c.dmin + tot_neg, best_key = c.kmin;
      if (c.kmax != INT_MAX) {
        const long long em = tot_pos - c.dmax;
        if (em < best_err || (em == best_err && c.kmax < best_key)) best_err = em, best_key = c.kmax;
      }
      double thr = 0.0;
      if (best_key != INT_MAX) {
        const double *xf = P.xsorted + (size_t)f * n;
        const int i = best_key >> 1;
        thr = 0.5 * (xf[i] + xf[i + 1]);
      }
      P.feat_ierr[(round & 1) * F + f] = best_err;
      P.feat_pos[(round & 1) * F + f] = best_key;
      P.feat_thr[(round & 1) * F + f] = thr;
    }
    grid.sync();
    // ---- the winner (every CTA, same answer): lowest error, lowest feature at equal error ----
    if (threadIdx.x < 32) {
      const long long *ferr = P.feat_ierr + (round & 1) * F;
      long long e = LLONG_MAX;
      int g = INT_MAX;
      for (int q = threadIdx.x; q < F; q += 32) {
        const long long eq = __ldcg(ferr + q);
        if (__ldcg(P.feat_pos + (round & 1) * F + q) != INT_MAX && eq < e) e = eq, g = q;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const long long oe = __shfl_down_sync(0xffffffffu, e, off);
        const int og = __shfl_down_sync(0xffffffffu, g, off);
        if (og != INT_MAX && (g == INT_MAX || oe < e || (oe == e && og < g))) e = oe, g = og;
      }
      if (threadIdx.x == 0) s_be = e, s_bf = g == INT_MAX ? -1 : g;
    }
    if (threadIdx.x == 0) {
      const long long be = s_be;
      const int bf = s_bf;
      int bk = 0;
      double bt = 0.0;
      if (bf >= 0) {
        bk = __ldcg(P.feat_pos + (round & 1) * F + bf);
        bt = __ldcg(P.feat_thr + (round & 1) * F + bf);
      }
      long long miss = be;  // fixed-point weight of the misclassified samples
      if (bf < 0) {  // every feature constant: majority constant stump
        const double pol = 2 * tot_neg <= total ? 1.0 : -1.0;  // +1 iff sum(w y) >= 0
        s_feat = 0;
        s_thr = __longlong_as_double(0xfff0000000000000LL);
        s_pol = pol;
        miss = pol > 0 ? tot_neg : total - tot_neg;
        s_err = (double)miss / (double)total;
      } else {
        s_feat = bf;
        s_thr = bt;
        s_pol = (bk & 1) ? -1.0 : 1.0;
        s_err = (double)be / (double)total;
      }
      const double err = s_err;
      if (P.raw) {
        if (blockIdx.x == 0) {
          P.out_feat[0] = s_feat, P.out_thr[0] = s_thr, P.out_pol[0] = s_pol, P.out_alpha[0] = 1.0;
          P.out_err[0] = err;
        }
        s_stop = 3;
      } else if (err >= 0.5) {
        s_stop = 1;
      } else {
        const double a = 0.5 * log((1.0 - err) / (err > 1e-10 ? err : 1e-10));
        s_alpha = a;
        // the reweighted weights sum to e^-a (1 - err) + e^a err, err over the quantised weights
        // the split was searched on: known here, so no pass over the weights forms it
        const double eag = exp(-a), emi = exp(a);
        s_eag = eag, s_emi = emi;
        s_sum = (eag * (double)(total - miss) + emi * (double)miss) / (double)total;
        if (blockIdx.x == 0) {
          P.out_feat[count] = s_feat, P.out_thr[count] = s_thr, P.out_pol[count] = s_pol;
          P.out_alpha[count] = a, P.out_err[count] = err;
        }
        s_stop = err <= 0.0 ? 3 : 0;
      }
    }
    __syncthreads();
    if (s_stop == 1) break;
    ++count;
    if (s_stop == 3 || round + 1 == P.rounds) break;
    // ---- reweight this CTA's slice (the other CTAs gather it over DSMEM next round) ----------
    {
      const double thr = s_thr, pol = s_pol, e_agree = s_eag, e_miss = s_emi;
      const double *xcol = P.xt + (size_t)s_feat * n;
      for (int i = e_lo + (int)threadIdx.x; i < e_hi; i += blockDim.x) {
        const double pred = __ldg(xcol + i) > thr ? pol : -pol;
        wloc[i] = wloc[i] * inv_s * (((double)s_y[i - e_lo] * pred > 0.0) ? e_agree : e_miss);
      }
      ssum = s_sum;
      cluster.sync();
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) write_result(count, n, n_pos_all, P.out_count, P.out_intercept);
  cluster.sync();
}

}  // namespace brm
