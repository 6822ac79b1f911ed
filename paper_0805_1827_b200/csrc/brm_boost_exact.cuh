// brm_boost_exact.cuh -- the exact parallel cumsum of parity-mode AdaBoost
// (boosting.py:150-153), its self-test, and the per-feature column sort.
//
// Included by brm_boost.cu after the pairwise-sum helpers.  The production
// kernel (brm_boost_cluster.cuh) runs this scan split over a thread-block
// cluster; ex_tile below is the same algorithm on one CTA, kept as the unit
// the self-test (brm_selftest_math kind 10) checks against np.cumsum.
//
// Exact parallel cumsum.  numpy's cumsum is the sequential recurrence
// s_j = fl(s_{j-1} + v_j) (v_j >= 0 here).  While s stays inside one binade
// [2^e, 2^(e+1)), s is a multiple of ulp_e = 2^(e-52) and the rounded add is
// an integer add: s_j = s_{j-1} + r_j ulp_e with r_j = rint(v_j / ulp_e)
// (round-to-nearest-even of an exact power-of-two scaling), unless v_j / ulp_e
// sits exactly halfway (the even rule then depends on s_{j-1}).  So:
//   1. a block scan of the v's (fp64, any order) gives approximations S^_j
//      within (n + 64) ulps of the true prefixes;
//   2. element j is PLAIN when S^_{j-1} and S^_j lie in the same binade at
//      least 2 (n + 64) ulps from its edges (so the true s_{j-1}, s_j do too)
//      and v_j / ulp_e is not a tie; a plain element adds the integer r_j;
//   3. every other element (the first one, binade crossings, prefixes close to
//      a power of two, ties) is an EVENT: one thread per chain walks the
//      events in order, doing the real fp64 add at each from the exact value
//      before it (previous event + the integer prefix of the plain r's);
//   4. every position's value is the last event's value plus an integer
//      prefix times that segment's ulp -- the sequential chain's bits.
// A chain has one event per binade crossing (~20-40 per round) plus rare ties
// and near-edge prefixes, so the walk is short.  Positive and negative
// weights are two chains over the same sorted sequence (the other class adds
// an exact 0.0, which never changes a partial sum).
#pragma once

namespace brm {

constexpr int kExThreads = 512;          // threads per CTA
constexpr int kExQ = 20;                 // sorted positions per thread per tile
constexpr int kExTile = kExThreads * kExQ;
constexpr int kExEvents = 512;           // events per chain per tile (else the serial fallback)
constexpr unsigned kCodeNeg = 0x80000000u, kCodeBrk = 0x40000000u, kCodeId = 0x3fffffffu;

struct ExactParams {
  int n, F, rounds, raw;
  const double *xsorted;   // [F][n] feature values in sorted order (thresholds)
  const unsigned *code;    // [F][n] sample id | kCodeNeg (label -1) | kCodeBrk (distinct value after i)
  const double *xt;        // [F][n] feature columns in sample order (predictions)
  const double *y;         // [n] +-1
  const double *w0;        // [n] initial weights
  double *wn_g;            // [F][n] per-CTA weights when they do not fit in shared memory
  double *chain_g;         // [F][2][n] chain values per position (multi-tile fits)
  double *wsub;            // [F][n] scratch of the constant-stump fallback
  const int2 *leaves;
  int n_leaves;
  const int2 *children;
  const int *level_end;
  int n_levels, root;
  int wn_smem;             // 1: the weights live in shared memory
  int margin;              // certainty margin in ulps: 2 (n + 64)
  double *feat_err;        // [2][F] per round parity
  int *feat_pos;           // [2][F] 2 * position + (polarity == -1)
  int *out_feat;
  double *out_thr, *out_pol, *out_alpha, *out_err;
  int *out_count;
  double *out_intercept;
  const int *n_pos;
  unsigned long long *n_fallback;  // tiles that overflowed the event lists (diagnostic)
  long long *timing;               // optional per-phase clock64 totals of CTA 0 (BRM_BOOST_TIMING)
  int *n_events;                   // optional: events of CTA 0's chains, summed over rounds
};

__device__ __forceinline__ int ex_expo(double x) { return (int)((__double_as_longlong(x) >> 52) & 0x7ff); }

// ulp of a positive normal double (its binade's grid step)
__device__ __forceinline__ double ex_ulp(double x) {
  return __longlong_as_double((__double_as_longlong(x) & 0x7ff0000000000000LL) - (52LL << 52));
}

// S^ is far enough from its binade's edges that the true prefix shares its binade
__device__ __forceinline__ bool ex_certain(double x, long long margin) {
  const long long b = __double_as_longlong(x);
  const long long mant = b & 0x000fffffffffffffLL;
  return ((b >> 52) & 0x7ff) > 64 && mant >= margin && mant <= 0x000fffffffffffffLL - margin;
}

// Block-wide exclusive scan of one value per thread (warp shuffles + smem).
// The exclusive value is formed from sums of EARLIER elements only (never as
// inclusive - own value), so every fp64 intermediate is bounded by the
// exclusive prefix itself and its rounding error is relative to it.
template <typename T>
__device__ __forceinline__ T ex_scan(T v, T *s_warp, T &total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const T o = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x = x + o;
  }
  if (lane == 31) s_warp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    T t = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : T(0);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const T o = __shfl_up_sync(0xffffffffu, t, off);
      if (lane >= off) t = t + o;
    }
    if (lane < (int)(blockDim.x >> 5)) s_warp[lane] = t;
  }
  __syncthreads();
  const T before = wid > 0 ? s_warp[wid - 1] : T(0);
  total = s_warp[(blockDim.x >> 5) - 1];
  __syncthreads();
  const T in_warp = __shfl_up_sync(0xffffffffu, x, 1);
  return lane == 0 ? before : before + in_warp;
}

struct ExShared {
  long long ev_P[2][kExEvents];  // integer prefix (of plain r's) before each event
  double ev_v[2][kExEvents];     // the event's weight
  double ev_s[2][kExEvents];     // the chain value after the event (walker output)
  double carry[2];               // exact chain value before the current tile
  double s_d[2][kExThreads / 32];
  long long s_l[2][kExThreads / 32];
  int s_i[2][kExThreads / 32];
};

// v / ulp of the binade of a (exact power-of-two scaling)
__device__ __forceinline__ double ex_scaled(double v, double a) {
  return v * __longlong_as_double((long long)(2098 - ex_expo(a)) << 52);
}

// Split errors at sorted position i into the running best candidate
// (boosting.py:154-164: err+ = pos_cum + (tot_neg - neg_cum), err- = total - err+).
__device__ __forceinline__ void ex_split_at(int i, double pcv, double ncv, double tot_neg, double total, Cand &best) {
  const double ep = __dadd_rn(pcv, __dsub_rn(tot_neg, ncv));
  const double em = __dsub_rn(total, ep);
  const Cand ca{ep, 2 * i}, cb{em, 2 * i + 1};
  if (cand_less(ca, best)) best = ca;
  if (cand_less(cb, best)) best = cb;
}

// Both chains over sorted positions [t0, t0 + kExTile) of one feature.
// sh.carry: the exact chain values before the tile on entry, after it on exit.
// store: write every position's chain values to chain[i] / chain[n + i];
// otherwise (the whole sequence is this one tile) evaluate the splits here
// into `best`.  Returns false, leaving sh.carry alone, when an event list
// overflowed (the caller then runs ex_tile_serial).
__device__ __forceinline__ bool ex_tile(const ExactParams &P, const unsigned *code, const double *wn, int t0,
                                        ExShared &sh, double *chain, bool store, double total, Cand &best) {
  const int n = P.n;
  const double cin0 = sh.carry[0], cin1 = sh.carry[1];
  const int i0 = t0 + threadIdx.x * kExQ;
  const int q = max(0, min(kExQ, n - i0));
  double v[kExQ];
  unsigned neg_mask = 0, brk_mask = 0;
#pragma unroll
  for (int k = 0; k < kExQ; ++k) {
    v[k] = 0.0;
    if (k < q) {
      const unsigned c = __ldg(code + i0 + k);
      v[k] = wn[c & kCodeId];
      if (c & kCodeNeg) neg_mask |= 1u << k;
      if (c & kCodeBrk) brk_mask |= 1u << k;
    }
  }
  // 1. approximate prefixes
  double ls0 = 0.0, ls1 = 0.0;
#pragma unroll
  for (int k = 0; k < kExQ; ++k) {
    if ((neg_mask >> k) & 1u) ls1 += v[k];
    else ls0 += v[k];
  }
  double tot_d;
  const double as0 = ex_scan<double>(ls0, sh.s_d[0], tot_d) + cin0;
  const double as1 = ex_scan<double>(ls1, sh.s_d[1], tot_d) + cin1;
  // 2. plain elements and their integer increments (r recomputed below, not kept)
  const long long margin = P.margin;
  unsigned plain_mask = 0;
  long long rs0 = 0, rs1 = 0;
  int ne0 = 0, ne1 = 0;
  {
    double a0 = as0, a1 = as1;
#pragma unroll
    for (int k = 0; k < kExQ; ++k) {
      if (k < q) {
        const bool ng = (neg_mask >> k) & 1u;
        const double a = ng ? a1 : a0;
        const double b = a + v[k];
        bool plain = ex_certain(a, margin) && ex_certain(b, margin) && ex_expo(a) == ex_expo(b);
        long long r = 0;
        if (plain) {
          // < 2^53 because s stays in the binade
          const double t = ex_scaled(v[k], a);
          plain = (t - floor(t)) != 0.5;  // a tie's rounding depends on s: event
          r = __double2ll_rn(t);
        }
        if (plain) {
          plain_mask |= 1u << k;
          if (ng) rs1 += r;
          else rs0 += r;
        } else if (ng) {
          ++ne1;
        } else {
          ++ne0;
        }
        if (ng) a1 = b;
        else a0 = b;
      }
    }
  }
  long long Ptot0, Ptot1;
  int Etot0, Etot1;
  const long long P0 = ex_scan<long long>(rs0, sh.s_l[0], Ptot0);
  const long long P1 = ex_scan<long long>(rs1, sh.s_l[1], Ptot1);
  const int E0 = ex_scan<int>(ne0, sh.s_i[0], Etot0);
  const int E1 = ex_scan<int>(ne1, sh.s_i[1], Etot1);
  if (Etot0 > kExEvents || Etot1 > kExEvents) {
    if (threadIdx.x == 0 && P.n_fallback) atomicAdd(P.n_fallback, 1ull);
    return false;  // uniform across the CTA (scan totals)
  }
  // 3a. publish the events in order with the integer prefix before each
  {
    double a0 = as0, a1 = as1;
    long long p0 = P0, p1 = P1;
    int e0 = E0, e1 = E1;
#pragma unroll
    for (int k = 0; k < kExQ; ++k) {
      if (k < q) {
        const bool ng = (neg_mask >> k) & 1u;
        const double a = ng ? a1 : a0;
        if ((plain_mask >> k) & 1u) {
          const long long r = __double2ll_rn(ex_scaled(v[k], a));
          if (ng) p1 += r;
          else p0 += r;
        } else if (ng) {
          sh.ev_P[1][e1] = p1;
          sh.ev_v[1][e1++] = v[k];
        } else {
          sh.ev_P[0][e0] = p0;
          sh.ev_v[0][e0++] = v[k];
        }
        if (ng) a1 = a + v[k];
        else a0 = a + v[k];
      }
    }
  }
  __syncthreads();
  // 3b. walk the events: two threads, one per chain, the real fp64 add at each
  if ((threadIdx.x & 31) == 0 && threadIdx.x < 64) {
    const int c = threadIdx.x >> 5;
    const int ne = c ? Etot1 : Etot0;
    double s = c ? cin1 : cin0;
    long long pp = 0;
    for (int k = 0; k < ne; ++k) {
      const long long p = sh.ev_P[c][k];
      if (p != pp) s = __dadd_rn(s, __dmul_rn((double)(p - pp), ex_ulp(s)));
      s = __dadd_rn(s, sh.ev_v[c][k]);
      sh.ev_s[c][k] = s;
      pp = p;
    }
    const long long pt = c ? Ptot1 : Ptot0;
    if (pt != pp) s = __dadd_rn(s, __dmul_rn((double)(pt - pp), ex_ulp(s)));
    sh.carry[c] = s;  // chain value after the tile
    if (P.n_events && blockIdx.x == 0) atomicAdd(P.n_events + c, ne);
  }
  __syncthreads();
  // 4. every position: the last event at or before it plus an integer prefix
  const double tot_neg = sh.carry[1];  // final negative chain value when this is the only tile
  double bs0 = cin0, bs1 = cin1;
  long long bp0 = 0, bp1 = 0;
  if (E0 > 0) {
    bs0 = sh.ev_s[0][E0 - 1];
    bp0 = sh.ev_P[0][E0 - 1];
  }
  if (E1 > 0) {
    bs1 = sh.ev_s[1][E1 - 1];
    bp1 = sh.ev_P[1][E1 - 1];
  }
  long long p0 = P0, p1 = P1;
  int e0 = E0, e1 = E1;
  double cur0 = p0 != bp0 ? __dadd_rn(bs0, __dmul_rn((double)(p0 - bp0), ex_ulp(bs0))) : bs0;
  double cur1 = p1 != bp1 ? __dadd_rn(bs1, __dmul_rn((double)(p1 - bp1), ex_ulp(bs1))) : bs1;
#pragma unroll
  for (int k = 0; k < kExQ; ++k) {
    if (k < q) {
      const bool ng = (neg_mask >> k) & 1u;
      if ((plain_mask >> k) & 1u) {
        // the segment's binade is its base event's (or the tile carry's)
        if (ng) {
          p1 += __double2ll_rn(ex_scaled(v[k], bs1));
          cur1 = __dadd_rn(bs1, __dmul_rn((double)(p1 - bp1), ex_ulp(bs1)));
        } else {
          p0 += __double2ll_rn(ex_scaled(v[k], bs0));
          cur0 = __dadd_rn(bs0, __dmul_rn((double)(p0 - bp0), ex_ulp(bs0)));
        }
      } else if (ng) {
        cur1 = bs1 = sh.ev_s[1][e1];
        bp1 = p1;
        ++e1;
      } else {
        cur0 = bs0 = sh.ev_s[0][e0];
        bp0 = p0;
        ++e0;
      }
      const int i = i0 + k;
      if (store) {
        chain[i] = cur0;
        chain[n + i] = cur1;
      } else if (((brk_mask >> k) & 1u) && i < n - 1) {
        ex_split_at(i, cur0, cur1, tot_neg, total, best);
      }
    }
  }
  __syncthreads();  // event lists and carries are reused by the next tile
  return true;
}

// Serial walk of one tile (after an event-list overflow): thread 0 adds both
// chains in order into chain[i] / chain[n + i]; sh.carry before / after.
__device__ void ex_tile_serial(const ExactParams &P, const unsigned *code, const double *wn, int t0, ExShared &sh,
                               double *chain) {
  const int n = P.n;
  if (threadIdx.x == 0) {
    double s0 = sh.carry[0], s1 = sh.carry[1];
    for (int i = t0; i < min(t0 + kExTile, n); ++i) {
      const unsigned cd = code[i];
      if (cd & kCodeNeg) s1 = __dadd_rn(s1, wn[cd & kCodeId]);
      else s0 = __dadd_rn(s0, wn[cd & kCodeId]);
      chain[i] = s0;
      chain[n + i] = s1;
    }
    sh.carry[0] = s0;
    sh.carry[1] = s1;
  }
  __syncthreads();
}

// Self-test (brm_selftest_math kind 10): np.cumsum of a[0..n) (a >= 0) by the
// exact block scan, one chain, every tile through ex_tile / ex_tile_serial.
__global__ void __launch_bounds__(kExThreads, 1) exact_scan_selftest(const double *a, int n, unsigned *code,
                                                                     double *chain, double *out) {
  __shared__ ExShared sh;
  for (int i = threadIdx.x; i < n; i += blockDim.x) code[i] = (unsigned)i;
  if (threadIdx.x < 2) sh.carry[threadIdx.x] = 0.0;
  __syncthreads();
  ExactParams P{};
  P.n = n;
  P.margin = 2 * (n + 64);
  Cand best{0.0, 0};
  for (int t0 = 0; t0 < n; t0 += kExTile)
    if (!ex_tile(P, code, a, t0, sh, chain, true, 0.0, best)) ex_tile_serial(P, code, a, t0, sh, chain);
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = __ldcg(chain + i);
}

// ------------------------------------------------------------- sorting ----
// Stable per-column argsort (np.argsort(kind="stable"), boosting.py:143),
// once per fit, one CTA per feature: (key, sample id) pairs are unique, so
// any correct sort of them is the stable order.  Tiles of kSortTile pairs are
// bitonic-sorted in shared memory, then merged pairwise in global memory
// (merge path: each thread finds its output diagonal by binary search).
constexpr int kSortThreads = 1024;
constexpr int kSortTile = 2 * kSortThreads;

// order-preserving integer key of a double; -0.0 and +0.0 compare equal as in numpy
__device__ __forceinline__ unsigned long long sort_key(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(__dadd_rn(x, 0.0));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}

__device__ __forceinline__ bool kv_less(unsigned long long ka, unsigned ia, unsigned long long kb, unsigned ib) {
  return ka < kb || (ka == kb && ia < ib);
}

__global__ void __launch_bounds__(kSortThreads) sort_columns(const double *xt, int n, unsigned long long *k0,
                                                               unsigned *i0, unsigned long long *k1, unsigned *i1,
                                                               double *xsorted, int *order) {
  __shared__ unsigned long long s_k[kSortTile];
  __shared__ unsigned s_i[kSortTile];
  const int f = blockIdx.x;
  const double *col = xt + (size_t)f * n;
  unsigned long long *ka = k0 + (size_t)f * n, *kb = k1 + (size_t)f * n;
  unsigned *ia = i0 + (size_t)f * n, *ib = i1 + (size_t)f * n;
  for (int t0 = 0; t0 < n; t0 += kSortTile) {
    for (int j = threadIdx.x; j < kSortTile; j += blockDim.x) {
      const int i = t0 + j;
      s_k[j] = i < n ? sort_key(col[i]) : ~0ull;
      s_i[j] = i < n ? (unsigned)i : 0xffffffffu;
    }
    __syncthreads();
    for (int size = 2; size <= kSortTile; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        const int t = threadIdx.x;  // kSortTile / 2 compare-exchanges, one per thread
        const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
        const bool up = (lo & size) == 0;
        const unsigned long long kl = s_k[lo], kh = s_k[hi];
        const unsigned il = s_i[lo], ih = s_i[hi];
        if (kv_less(kh, ih, kl, il) == up) {
          s_k[lo] = kh;
          s_k[hi] = kl;
          s_i[lo] = ih;
          s_i[hi] = il;
        }
        __syncthreads();
      }
    }
    for (int j = threadIdx.x; j < kSortTile; j += blockDim.x) {
      const int i = t0 + j;
      if (i < n) {
        ka[i] = s_k[j];
        ia[i] = s_i[j];
      }
    }
    __syncthreads();
  }
  // merge passes: runs of R -> 2R
  constexpr int Q = 16;
  for (int R = kSortTile; R < n; R <<= 1) {
    for (int o0 = threadIdx.x * Q; o0 < n; o0 += blockDim.x * Q) {
      const int base = o0 / (2 * R) * (2 * R);
      const int a0 = base, la = min(R, n - base);
      const int b0 = base + la, lb = max(0, min(R, n - b0));
      const int d = o0 - base;
      int lo = max(0, d - lb), hi = min(d, la);
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (!kv_less(ka[b0 + d - 1 - mid], ia[b0 + d - 1 - mid], ka[a0 + mid], ia[a0 + mid])) lo = mid + 1;
        else hi = mid;
      }
      int x = lo, y = d - lo;
      const int end = min(o0 + Q, base + la + lb);
      for (int o = o0; o < end; ++o) {
        const bool take_a = y >= lb || (x < la && kv_less(ka[a0 + x], ia[a0 + x], ka[b0 + y], ia[b0 + y]));
        if (take_a) {
          kb[o] = ka[a0 + x];
          ib[o] = ia[a0 + x];
          ++x;
        } else {
          kb[o] = ka[b0 + y];
          ib[o] = ia[b0 + y];
          ++y;
        }
      }
    }
    __syncthreads();
    unsigned long long *tk = ka;
    ka = kb;
    kb = tk;
    unsigned *ti = ia;
    ia = ib;
    ib = ti;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const unsigned id = ia[i];
    order[(size_t)f * n + i] = (int)id;
    xsorted[(size_t)f * n + i] = col[id];
  }
}

// Per feature and sorted position: sample id | label -1 | distinct value follows.
__global__ void build_codes(const int *order, const double *y, const double *xsorted, int n, unsigned *code) {
  const int f = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int id = order[(size_t)f * n + i];
  const double *xf = xsorted + (size_t)f * n;
  unsigned c = (unsigned)id;
  if (!(y[id] > 0.0)) c |= kCodeNeg;
  if (i + 1 < n && __dsub_rn(xf[i + 1], xf[i]) > 0.0) c |= kCodeBrk;  // np.diff(xf) > 0 (boosting.py:145)
  code[(size_t)f * n + i] = c;
}

}  // namespace brm
