// brm_boost.cu -- AdaBoost decision stumps (boosting.py:126-206) and the
// quadratic boundary regression (boundary_iz.py:250-276) on the device.
//
// AdaBoost runs as ONE cooperative kernel for the whole ensemble: a CTA per
// feature.  Each column is sorted once per fit (stable radix sort, the
// reference re-sorts every round, boosting.py:143); per round
//   every CTA  : total = sum(w) in numpy's pairwise order (redundantly: no sync)
//   CTA f      : sequential prefix sums of positive / negative weights in the
//                sorted order (numpy cumsum order), then a parallel scan of
//                the split points for the interleaved first-hit argmin
//   grid sync  ; every CTA picks the same winner (lowest feature, then lowest
//                threshold, then +1 polarity at exact ties), forms alpha
//   all CTAs   : w *= exp(-alpha y pred) on a slice; grid sync; w /= sum(w)
//                (pairwise order); grid sync
// Products and sums are separately rounded fp64 like numpy's, so the split
// search reproduces the reference bit for bit on identical inputs; alpha and
// exp(+-alpha) come from CUDA's log/exp (<= 1 ulp from numpy's).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/bermuda_b200.h"
#include "brm_internal.h"
#include "brm_chain.cuh"
#include "brm_rng.cuh"

namespace cg = cooperative_groups;

namespace brm {

constexpr int kBoostThreads = 256;
constexpr int kTile = 4096;
constexpr int kPwBlock = 128;  // numpy PW_BLOCKSIZE

// numpy pairwise_sum leaf (n <= 128): 8 strided accumulators, fixed combine,
// then the tail added in order (n < 8: plain sequential from 0).
__device__ double pw_leaf(const double *a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

// numpy pairwise sum of a[0..n) by one thread (rare paths only).
__device__ double pw_serial(const double *a, int n) {
  struct Frame {
    int off, len, stage;
    double left;
  };
  Frame st[48];
  int sp = 0;
  double ret = 0.0;
  st[sp++] = Frame{0, n, 0, 0.0};
  while (sp > 0) {
    Frame &f = st[sp - 1];
    if (f.len <= kPwBlock) {
      ret = pw_leaf(a + f.off, f.len);
      --sp;
      continue;
    }
    int n2 = f.len / 2;
    n2 -= n2 % 8;
    if (f.stage == 0) {
      f.stage = 1;
      st[sp++] = Frame{f.off, n2, 0, 0.0};
    } else if (f.stage == 1) {
      f.left = ret;
      f.stage = 2;
      st[sp++] = Frame{f.off + n2, f.len - n2, 0, 0.0};
    } else {
      ret = __dadd_rn(f.left, ret);
      --sp;
    }
  }
  return ret;
}

// numpy's pairwise recursion over n elements as a tree: leaves in order,
// internal nodes grouped by height so a CTA combines a level at a time.
struct PwTree {
  std::vector<int2> leaves;    // (offset, length), left to right
  std::vector<int2> children;  // internal node L+j = children[j].x + children[j].y
  std::vector<int> level_end;  // internal nodes [level_end[h-1], level_end[h]) have height h+1
};

// Build the tree with explicit node ids: leaves 0..L-1, internal nodes L.. in
// level order.  Returns the root id.
static int pw_tree(int64_t n, PwTree &t) {
  struct Node {
    int left, right, height;
  };
  std::vector<Node> inner;
  std::function<int(int64_t, int64_t)> rec = [&](int64_t off, int64_t len) -> int {
    if (len <= kPwBlock) {
      t.leaves.push_back(make_int2((int)off, (int)len));
      return -(int)t.leaves.size();  // leaf k encoded as -(k+1)
    }
    int64_t n2 = len / 2;
    n2 -= n2 % 8;
    const int l = rec(off, n2);
    const int r = rec(off + n2, len - n2);
    auto h = [&](int id) { return id < 0 ? 0 : inner[id].height; };
    inner.push_back(Node{l, r, 1 + std::max(h(l), h(r))});
    return (int)inner.size() - 1;
  };
  const int root = rec(0, n);
  const int L = (int)t.leaves.size();
  if (root < 0) return 0;
  // order internal nodes by height
  std::vector<int> order(inner.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return inner[x].height < inner[y].height; });
  std::vector<int> newid(inner.size());
  for (size_t k = 0; k < order.size(); ++k) newid[order[k]] = L + (int)k;
  auto idof = [&](int id) { return id < 0 ? (-id - 1) : newid[id]; };
  int maxh = 0;
  for (size_t k = 0; k < order.size(); ++k) {
    const Node &nd = inner[order[k]];
    t.children.push_back(make_int2(idof(nd.left), idof(nd.right)));
    maxh = std::max(maxh, nd.height);
  }
  t.level_end.assign(maxh, 0);
  for (size_t k = 0; k < order.size(); ++k) t.level_end[inner[order[k]].height - 1] = (int)k + 1;
  return newid[root];
}

struct BoostParams {
  int n, F, rounds;
  const double *xs;        // [n][F]
  const double *xsorted;   // [F][n]
  const double *xt;        // [F][n] columns in sample order
  const double *y;         // [n] +-1
  double *w;               // [n] unnormalised weights of the current round
  double *wn;              // [F][n] per-CTA normalised copy (w / sum(w), numpy order)
  const int *pos_idx;      // [F][n] sample ids of the positives in sorted order (first n_pos[f])
  const int *neg_idx;      // [F][n] sample ids of the negatives in sorted order
  const int *cntpos;       // [F][n] positives among sorted positions 0..i
  const int2 *brk;         // [F][n] chain indices at split i (INT_MIN: no break after i)
  double *pcum, *ncum;     // [F][n] prefix sums of the positive / negative chains
  const int2 *leaves;
  int n_leaves;
  const int2 *children;
  const int *level_end;
  int n_levels, root;
  int tree_smem;           // 1: copy the tree tables into shared memory
  double *feat_err;        // [F]
  int *feat_pos;           // [F] 2*i + (pol == -1)
  double *wsub;            // [F][n] per-CTA scratch for the constant-stump sums
  double *leafsum;         // [L] pairwise leaf sums of w (written by the reweighting CTAs)
  int *out_feat;
  double *out_thr, *out_pol, *out_alpha, *out_err;
  int *out_count;
  double *out_intercept;
  const int *n_pos;        // positives in the training set (device)
  int raw;  // 1: one fit_stump search with the given weights, no boosting rules
  long long *timing;  // optional per-phase clock64 totals of CTA 0 (diagnostics)
};

// The recursion tree as the kernel reads it (shared-memory copy when it fits).
struct PwView {
  const int2 *leaves, *children;
  const int *level_end;
  int L, n_levels, root;
};

// numpy pairwise leaves [l_lo, l_hi) of a[0..n) into dst[l]: 8 lanes per
// leaf, lane j owns numpy's accumulator r[j] (elements j, j+8, ...); pair sums
// by shuffles are exact (IEEE addition commutes), the tail of len % 8 elements
// is added in order (values gathered by shuffles).  op(i, a[i]) maps each
// element to the value summed (loads only); sink(i, v) may then store it (the
// normalise / reweight passes).  Keeping the stores out of op lets all loads
// of a lane issue before the first store, which the compiler must otherwise
// order behind it (the pointers may alias).
struct PwNoSink {
  __device__ __forceinline__ void operator()(int, double) const {}
};

template <class Op, class Sink = PwNoSink>
__device__ __forceinline__ void pw_leaf_sums(const PwView &T, const double *a, int l_lo, int l_hi, double *dst,
                                             Op op, Sink sink = PwNoSink{}) {
  const int lane = threadIdx.x & 31, grp = lane >> 3, j = lane & 7;
  const int groups = (blockDim.x >> 5) * 4;
  for (int l0 = l_lo + (threadIdx.x >> 5) * 4; l0 < l_hi; l0 += groups) {
    const int l = l0 + grp;
    const bool ok = l < l_hi;
    const int2 lf = ok ? T.leaves[l] : make_int2(0, 0);
    const int off = lf.x, len = lf.y;
    const int main = len >= 8 ? len - (len % 8) : 0;
    // leaves hold <= 128 elements: all 16 loads of this lane are issued up front
    const int tail = len - main;  // < 8 elements added in order after the accumulators
    double col[kPwBlock / 8];
#pragma unroll
    for (int q = 0; q < kPwBlock / 8; ++q) col[q] = 8 * q < main ? a[off + 8 * q + j] : 0.0;
    double tv = j < tail ? a[off + main + j] : 0.0;
    // the 16 mapped values are independent: form them all before the
    // dependent adds so their loads / divisions overlap
    // op runs on every slot (masked slots read element `off` and map a zero):
    // branch-free, so the loads and dependency chains of all slots overlap
#pragma unroll
    for (int q = 0; q < kPwBlock / 8; ++q) col[q] = op(8 * q < main ? off + 8 * q + j : off, col[q]);
    tv = op(j < tail ? off + main + j : off, tv);
#pragma unroll
    for (int q = 0; q < kPwBlock / 8; ++q)
      if (8 * q < main) sink(off + 8 * q + j, col[q]);
    if (j < tail) sink(off + main + j, tv);
    double r = main ? col[0] : 0.0;
#pragma unroll
    for (int q = 1; q < kPwBlock / 8; ++q)
      if (8 * q < main) r = __dadd_rn(r, col[q]);
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
    double res = main ? r : 0.0;
#pragma unroll
    for (int t = 0; t < 7; ++t) {
      const double x = __shfl_sync(0xffffffffu, tv, (lane & ~7) + t);
      if (t < tail) res = __dadd_rn(res, x);
    }
    if (ok && j == 0) dst[l] = res;
  }
}

// Combine the leaf sums in s_node[0..L) up numpy's recursion tree; every
// thread gets the root.
__device__ __forceinline__ double pw_tree_sum(const PwView &T, double *s_node) {
  const int L = T.L;
  __syncthreads();
  int lo = 0;
  for (int h = 0; h < T.n_levels; ++h) {
    const int hi = T.level_end[h];
    for (int j = lo + threadIdx.x; j < hi; j += blockDim.x) {
      const int2 c = T.children[j];
      s_node[L + j] = __dadd_rn(s_node[c.x], s_node[c.y]);
    }
    lo = hi;
    __syncthreads();
  }
  const double r = s_node[T.root];
  __syncthreads();
  return r;
}

struct PwIdentity {
  __device__ __forceinline__ double operator()(int, double x) const { return x; }
};

// CTA-wide numpy-order sum of a[0..n); every thread gets the result.
// s_node holds L + I doubles.
__device__ double cta_pairwise(const PwView &T, const double *a, double *s_node) {
  pw_leaf_sums(T, a, 0, T.L, s_node, PwIdentity{});
  return pw_tree_sum(T, s_node);
}

// s[j] = w[idx[j]] for j < cnt (cnt <= kTile): all index loads of a thread
// are issued before the dependent value loads.
__device__ __forceinline__ void gather_tile(const double *__restrict__ w, const int *__restrict__ idx, int cnt,
                                            double *__restrict__ s) {
  constexpr int G = kTile / kBoostThreads;
  int id[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int j = threadIdx.x + g * kBoostThreads;
    id[g] = j < cnt ? __ldg(idx + j) : -1;
  }
  double v[G];
#pragma unroll
  for (int g = 0; g < G; ++g) v[g] = id[g] >= 0 ? w[id[g]] : 0.0;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int j = threadIdx.x + g * kBoostThreads;
    if (j < cnt) s[chain_pos<true>(j)] = v[g];  // warp_chain's padded layout
  }
}

// One class (boosting.py:185-187): a zero-round ensemble carrying the class
// sign; decided on the device so a fit needs no host round trip.
__device__ __forceinline__ bool one_class_exit(int raw, int n, int n_pos, int *out_count, double *out_intercept) {
  if (raw || (n_pos != 0 && n_pos != n)) return false;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *out_count = 0;
    *out_intercept = n_pos == n ? 1.0 : -1.0;
  }
  return true;
}

// No stump beat random guessing: the majority sign (boosting.py:202-205).
__device__ __forceinline__ void write_result(int count, int n, int n_pos, int *out_count, double *out_intercept) {
  *out_count = count;
  *out_intercept = count > 0 ? 0.0 : (2 * n_pos >= n ? 1.0 : -1.0);
}

struct Cand {
  double err;
  int key;  // 2*i + (minus polarity)
};

__device__ __forceinline__ bool cand_less(const Cand &a, const Cand &b) {
  return a.err < b.err || (a.err == b.err && a.key < b.key);
}

// Chain self-test (brm_selftest_math kinds 8 / 9): the prefix sums of a[0..n)
// by the one-thread sequential chain and by the warp's binade tiles.
__global__ void chain_selftest(int kind, const double *a, int64_t n, double *out) {
  double acc = 0.0;
  if (kind == 8) {
    if (threadIdx.x == 0) serial_chain<false>(a, out, 0, (int)n, acc);
  } else {
    warp_chain<false>(a, out, (int)n, acc);
  }
}

void *chain_selftest_kernel() { return (void *)&chain_selftest; }

__global__ void __launch_bounds__(kBoostThreads) boost_kernel(BoostParams P) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *s_node = reinterpret_cast<double *>(smem_raw);               // [L + I]
  double *s_in_p = s_node + 2 * P.n_leaves;
  constexpr int kTileP = chain_padded_len(kTile);  // padded tiles (chain_pos)
  double *s_in_n = s_in_p + kTileP;
  double *s_out_p = s_in_n + kTileP;
  double *s_out_n = s_out_p + kTileP;
  unsigned char *s_after = reinterpret_cast<unsigned char *>(s_out_n + kTileP);
  __shared__ Cand s_cand[kBoostThreads / 32];
  __shared__ int s_stop;
  __shared__ double s_alpha, s_thr, s_pol, s_err;
  __shared__ int s_feat;

  const int n = P.n, F = P.F;
  const int f = blockIdx.x;
  const int n_pos_all = *P.n_pos;
  if (one_class_exit(P.raw, n, n_pos_all, P.out_count, P.out_intercept)) return;
  // reweighting slices are whole pairwise leaves, so each CTA also publishes
  // the leaf sums of the new weights and sum(w) needs only the tree combine
  const int L = P.n_leaves;
  PwView T{P.leaves, P.children, P.level_end, L, P.n_levels, P.root};
  if (P.tree_smem) {  // tree tables after the tiles: leaves, children, level ends
    int2 *s_leaves = reinterpret_cast<int2 *>(s_after);
    int2 *s_children = s_leaves + L;
    int *s_level = reinterpret_cast<int *>(s_children + max(L - 1, 0));
    for (int i = threadIdx.x; i < L; i += blockDim.x) s_leaves[i] = P.leaves[i];
    for (int i = threadIdx.x; i < L - 1; i += blockDim.x) s_children[i] = P.children[i];
    for (int i = threadIdx.x; i < P.n_levels; i += blockDim.x) s_level[i] = P.level_end[i];
    T.leaves = s_leaves;
    T.children = s_children;
    T.level_end = s_level;
    __syncthreads();
  }
  const int l_lo = (int)((long long)blockIdx.x * L / gridDim.x), l_hi = (int)((long long)(blockIdx.x + 1) * L / gridDim.x);
  double *wn = P.wn + (size_t)f * n;
  int count = 0;
  // per-phase clock totals (diagnostics, BRM_BOOST_TIMING): thread 0 of CTA 0,
  // slot 7 the positive-chain thread; kept in registers, stored at the end
  const bool timed = P.timing && blockIdx.x == 0;
  long long t_mark = 0, tacc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#define BRM_TSLOT(k)                       \
  if (timed && threadIdx.x == 0) {         \
    const long long now_ = clock64();      \
    tacc[k] += now_ - t_mark;              \
    t_mark = now_;                         \
  }

  for (int round = 0; round < P.rounds; ++round) {
    if (timed && threadIdx.x == 0) t_mark = clock64();
    // ---- wn = w / w.sum() (numpy pairwise order), CTA-private copy, and
    // total = wn.sum() in the same pass ----------------------------------
    double total;
    if (round == 0) {
      pw_leaf_sums(T, P.w, 0, L, s_node, PwIdentity{}, [&](int i, double v) { wn[i] = v; });
      total = pw_tree_sum(T, s_node);
    } else {
      for (int l = threadIdx.x; l < L; l += blockDim.x) s_node[l] = __ldcg(P.leafsum + l);
      const double s = pw_tree_sum(T, s_node);
      if (timed && threadIdx.x == 0) tacc[9] += clock64() - t_mark;
      pw_leaf_sums(
          T, P.w, 0, L, s_node, [&](int, double x) { return div_nb(x, s); }, [&](int i, double v) { wn[i] = v; });
      if (timed && threadIdx.x == 0) tacc[10] += clock64() - t_mark;
      total = pw_tree_sum(T, s_node);
    }
    BRM_TSLOT(1);
    // ---- split search on feature f -------------------------------------
    if (f < F) {
      const int *pid = P.pos_idx + (size_t)f * n;
      const int *nid = P.neg_idx + (size_t)f * n;
      double *pc = P.pcum + (size_t)f * n;
      double *nc = P.ncum + (size_t)f * n;
      const int n_pos = n_pos_all, n_neg = n - n_pos_all;
      double pacc = 0.0, nacc = 0.0;  // np.cumsum(where(y>0, w, 0)): zeros never change a partial sum
      // tiles: all threads gather, the two highest warps run the two sequential
      // chains (the issue arbiter favours high warp ids), all threads write back
      const int wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
      for (int t0 = 0; t0 < max(n_pos, n_neg); t0 += kTile) {
        const int tp = max(0, min(kTile, n_pos - t0)), tn = max(0, min(kTile, n_neg - t0));
        gather_tile(wn, pid + t0, tp, s_in_p);
        gather_tile(wn, nid + t0, tn, s_in_n);
        __syncthreads();
        // one warp per chain: binade tiles (brm_chain.cuh), ~2x the sequential
        // fp64 add chain's 9 cycles per element
        if (wid == nwarp - 2) {
          const long long c0 = timed ? clock64() : 0;
          warp_chain<true, 32>(s_in_p, s_out_p, tp, pacc);
          if (timed) tacc[7] += clock64() - c0;
        } else if (wid == nwarp - 1) {
          warp_chain<true, 32>(s_in_n, s_out_n, tn, nacc);
        }
        __syncthreads();
        for (int j = threadIdx.x; j < tp; j += blockDim.x) pc[t0 + j] = s_out_p[chain_pos<true>(j)];
        for (int j = threadIdx.x; j < tn; j += blockDim.x) nc[t0 + j] = s_out_n[chain_pos<true>(j)];
      }
      __syncthreads();
    BRM_TSLOT(2);
      // split points: brk[i] = (positives up to i) - 1, (negatives up to i) - 1,
      // precomputed once per fit; x == INT_MIN marks "no distinct-value break"
      const int2 *brk = P.brk + (size_t)f * n;
      const double tot_neg = n_neg > 0 ? nc[n_neg - 1] : 0.0;
      Cand best{__longlong_as_double(0x7ff0000000000000LL), 0x7fffffff};
      constexpr int U = 16;
      for (int i0 = threadIdx.x; i0 < n - 1; i0 += U * blockDim.x) {
        int2 bi[U];
        double pcs[U], ncs[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = i0 + u * blockDim.x;
          bi[u] = i < n - 1 ? brk[i] : make_int2(INT_MIN, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          pcs[u] = bi[u].x >= 0 ? pc[bi[u].x] : 0.0;
          ncs[u] = bi[u].y >= 0 ? nc[bi[u].y] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (bi[u].x == INT_MIN) continue;
          const int i = i0 + u * blockDim.x;
          const double ep = __dadd_rn(pcs[u], __dsub_rn(tot_neg, ncs[u]));
          const double em = __dsub_rn(total, ep);
          const Cand ca{ep, 2 * i}, cb{em, 2 * i + 1};
          if (cand_less(ca, best)) best = ca;
          if (cand_less(cb, best)) best = cb;
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        Cand o;
        o.err = __shfl_down_sync(0xffffffffu, best.err, off);
        o.key = __shfl_down_sync(0xffffffffu, best.key, off);
        if (cand_less(o, best)) best = o;
      }
      if ((threadIdx.x & 31) == 0) s_cand[threadIdx.x >> 5] = best;
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int wi = 1; wi < (int)blockDim.x / 32; ++wi)
          if (cand_less(s_cand[wi], best)) best = s_cand[wi];
        P.feat_err[f] = best.err;
        P.feat_pos[f] = best.key;
      }
    }
    BRM_TSLOT(3);
    grid.sync();
    BRM_TSLOT(4);
    // ---- pick the winner (every CTA, same answer) ------------------------
    // first minimum over features in order: (err, feature) lexicographic
    double be = __longlong_as_double(0x7ff0000000000000LL);
    int bf = 0x7fffffff, bk = 0;
    if (threadIdx.x < 32) {
      for (int g = threadIdx.x; g < F; g += 32) {
        const int pos = __ldcg(P.feat_pos + g);
        const double e = __ldcg(P.feat_err + g);
        if (pos != 0x7fffffff && e < be) {
          be = e;
          bf = g;
          bk = pos;
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double oe = __shfl_down_sync(0xffffffffu, be, off);
        const int of = __shfl_down_sync(0xffffffffu, bf, off);
        const int ok = __shfl_down_sync(0xffffffffu, bk, off);
        if (oe < be || (oe == be && of < bf)) {
          be = oe;
          bf = of;
          bk = ok;
        }
      }
    }
    if (threadIdx.x == 0) {
      if (bf == 0x7fffffff) bf = -1;
      if (bf < 0) {
        s_stop = 2;  // every feature constant: resolved below by the whole CTA
        s_feat = 0;
        s_thr = __longlong_as_double(0xfff0000000000000LL);
      } else {
        const int i = bk >> 1;
        const double *xf = P.xsorted + (size_t)bf * n;
        s_feat = bf;
        s_thr = __dmul_rn(0.5, __dadd_rn(xf[i], xf[i + 1]));
        s_pol = (bk & 1) ? -1.0 : 1.0;
        s_err = be;
        s_stop = 0;
      }
    }
    __syncthreads();
    if (s_stop == 2) {
      // every feature constant (boosting.py:166-170): pol = +1 iff sum(w*y) >= 0,
      // err = sum(w[y != pol]), both in numpy's pairwise order
      double *ws = P.wsub + (size_t)blockIdx.x * n;
      for (int i = threadIdx.x; i < n; i += blockDim.x) ws[i] = __dmul_rn(wn[i], P.y[i]);
      __syncthreads();
      const double swy = cta_pairwise(T, ws, s_node);
      const double pol = swy >= 0.0 ? 1.0 : -1.0;
      if (threadIdx.x == 0) {
        int k = 0;
        for (int i = 0; i < n; ++i)
          if (P.y[i] != pol) ws[k++] = wn[i];
        s_pol = pol;
        s_err = pw_serial(ws, k);
        s_stop = 0;
      }
      __syncthreads();
    }
    // alpha = 0.5 * log((1 - err) / max(err, 1e-10)); stop rules of fit_ensemble
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
    BRM_TSLOT(5);
    // ---- reweight own slice: w = (w / sum) * exp(-alpha * y * pred) ------
    {
      const double a = s_alpha, thr = s_thr, pol = s_pol;
      const int feat = s_feat;
      const double e_agree = exp(-a), e_miss = exp(a);
      if (timed && threadIdx.x == 0) tacc[8] += clock64() - t_mark;
      pw_leaf_sums(
          T, wn, l_lo, l_hi, P.leafsum,
          [&](int i, double x) {
            const double pred = __ldg(P.xt + (size_t)feat * n + i) > thr ? pol : -pol;
            return __dmul_rn(x, (__ldg(P.y + i) * pred > 0.0) ? e_agree : e_miss);
          },
          [&](int i, double v) { P.w[i] = v; });
    }
    if (timed && threadIdx.x == 0) tacc[0] += clock64() - t_mark;
    grid.sync();
    BRM_TSLOT(6);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) write_result(count, n, n_pos_all, P.out_count, P.out_intercept);
  if (timed && threadIdx.x == 0)
    for (int k = 0; k < 12; ++k)
      if (k != 7) P.timing[k] = tacc[k];
  if (timed && threadIdx.x == blockDim.x - 64) P.timing[7] = tacc[7];
#undef BRM_TSLOT
}

// Per feature: ids of positives / negatives in sorted order and the running
// count of positives (once per fit; labels and order are fixed across rounds).
__global__ void __launch_bounds__(256) split_classes(const int *order, const double *y, const double *xsorted, int n,
                                                     int *pos_idx, int *neg_idx, int *cntpos, int2 *brk) {
  using Scan = cub::BlockScan<int, 256>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int s_carry;
  const int f = blockIdx.x;
  const int *ord = order + (size_t)f * n;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int t0 = 0; t0 < n; t0 += 256) {
    const int i = t0 + threadIdx.x;
    const int id = i < n ? ord[i] : 0;
    const int pos = (i < n && y[id] > 0.0) ? 1 : 0;
    int excl, tile_total;
    Scan(tmp).ExclusiveSum(pos, excl, tile_total);
    const int carry = s_carry;
    if (i < n) {
      const int before = carry + excl;  // positives strictly before position i
      cntpos[(size_t)f * n + i] = before + pos;
      if (pos) pos_idx[(size_t)f * n + before] = id;
      else neg_idx[(size_t)f * n + (i - before)] = id;
      const double *xf = xsorted + (size_t)f * n;
      const bool is_break = i + 1 < n && __dsub_rn(xf[i + 1], xf[i]) > 0.0;  // boosting.py:145
      const int np_ = before + pos, nn_ = i + 1 - np_;
      brk[(size_t)f * n + i] = is_break ? make_int2(np_ - 1, nn_ - 1) : make_int2(INT_MIN, 0);
    }
    __syncthreads();
    if (threadIdx.x == 0) s_carry = carry + tile_total;
    __syncthreads();
  }
}

// ---------------------------------------------------------- fast mode ----
// BRM_MODE_FAST AdaBoost: the same stump search and boosting rules, with the
// weights quantised to 62-bit fixed point for the split search.  Integer
// prefix sums are exact and associative, so every prefix is a parallel block
// scan (no sequential fp64 chain) and the result is identical for any
// scheduling; the fp64 weights are renormalised in a fixed tree order.
// Statistically equivalent to the reference, not bit-identical to numpy.
constexpr double kFix = 4611686018427387904.0;  // 2^62

struct FastBoostParams {
  int n, F, rounds, raw;
  const double *xs, *xsorted, *y;
  const int *order;
  double *ysorted;              // [F][n] labels in each feature's sorted order (filled by the kernel)
  double *wpart;                // [gridDim] per-slice sums of the new weights (fixed CTA order)
  double *w;                    // [n] fp64 weights (unnormalised between rounds)
  long long *feat_err;          // [F] best integer error of each feature
  int *feat_pos;                // [F]
  int *out_feat;
  double *out_thr, *out_pol, *out_alpha, *out_err;
  int *out_count;
  double *out_intercept;
  const int *n_pos;  // positives in the training set (device)
};

// Fixed-order CTA sum (thread-strided runs, shuffle tree, warps in order).
__device__ double cta_sum_fixed(const double *a, int n, double *s_red) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += a[i];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = acc;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < (int)blockDim.x / 32; ++w) t += s_red[w];
  __syncthreads();
  return t;
}

__device__ __forceinline__ long long fixw(double w, double inv_s) { return __double2ll_rn(w * inv_s * kFix); }

__global__ void __launch_bounds__(kBoostThreads) boost_fast_kernel(FastBoostParams P) {
  using Scan = cub::BlockScan<long long, kBoostThreads>;
  __shared__ typename Scan::TempStorage s_scan;
  __shared__ double s_red[kBoostThreads / 32];
  __shared__ long long s_carry_p, s_carry_n;
  __shared__ struct { long long err; int key; } s_cand[kBoostThreads / 32];
  __shared__ int s_stop, s_feat;
  __shared__ double s_thr, s_pol, s_alpha, s_err;
  cg::grid_group grid = cg::this_grid();
  const int n = P.n, F = P.F, f = blockIdx.x;
  const int slice = (n + gridDim.x - 1) / gridDim.x;
  const int w_lo = blockIdx.x * slice, w_hi = min(w_lo + slice, n);
  const int n_pos_all = *P.n_pos;
  if (one_class_exit(P.raw, n, n_pos_all, P.out_count, P.out_intercept)) return;
  int count = 0;
  const int *ord = P.order + (size_t)f * n;
  const double *xf = P.xsorted + (size_t)f * n;
  double *ysf = P.ysorted + (size_t)f * n;
  // labels in this feature's sorted order, once per fit: the split scan then
  // gathers only the weights
  for (int i = threadIdx.x; i < n; i += blockDim.x) ysf[i] = P.y[ord[i]];
  __syncthreads();
  for (int round = 0; round < P.rounds; ++round) {
    // sum of the weights: round 0 by every CTA, later rounds from the slice
    // sums the previous reweight published (same order in every CTA)
    double ssum;
    if (round == 0) {
      ssum = cta_sum_fixed(P.w, n, s_red);
    } else {
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int b = 0; b < (int)gridDim.x; ++b) t += __ldcg(P.wpart + b);
        s_red[0] = t;
      }
      __syncthreads();
      ssum = s_red[0];
      __syncthreads();
    }
    const double inv_s = 1.0 / ssum;
    if (threadIdx.x == 0) s_carry_p = s_carry_n = 0;
    __syncthreads();
    // split search: one block scan per tile of sorted positions.  With d_i =
    // (positives - negatives up to i), err+ = d_i + tot_neg and err- = tot_pos
    // - d_i, so the argmins need only min / max of d_i; the class totals are
    // the scan's final carries
    long long dmin = LLONG_MAX, dmax = LLONG_MIN;
    int kmin = INT_MAX, kmax = INT_MAX;
    constexpr int ITEMS = 8;  // consecutive sorted positions per thread per tile
    for (int t0 = 0; t0 < n; t0 += ITEMS * blockDim.x) {
      const int i0 = t0 + threadIdx.x * ITEMS;
      long long wp[ITEMS], wn_[ITEMS];
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        const int i = i0 + k;
        wp[k] = wn_[k] = 0;
        if (i < n) {
          const long long W = fixw(P.w[ord[i]], inv_s);
          if (ysf[i] > 0.0) wp[k] = W;
          else wn_[k] = W;
        }
      }
      long long lp = 0, ln = 0;
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) lp += wp[k], ln += wn_[k];
      long long ep_, en_, sp, sn;
      Scan(s_scan).ExclusiveSum(lp, ep_, sp);
      __syncthreads();
      Scan(s_scan).ExclusiveSum(ln, en_, sn);
      long long cp = s_carry_p + ep_, cn = s_carry_n + en_;
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        const int i = i0 + k;
        cp += wp[k];
        cn += wn_[k];
        if (i < n - 1 && __dsub_rn(xf[i + 1], xf[i]) > 0.0) {
          const long long dd = cp - cn;
          if (dd < dmin) dmin = dd, kmin = 2 * i;        // positions ascend: first hit keeps the lowest key
          if (dd > dmax) dmax = dd, kmax = 2 * i + 1;
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        s_carry_p += sp;
        s_carry_n += sn;
      }
      __syncthreads();
    }
    const long long tot_pos = s_carry_p, tot_neg = s_carry_n, total = tot_pos + tot_neg;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const long long o1 = __shfl_down_sync(0xffffffffu, dmin, off), o2 = __shfl_down_sync(0xffffffffu, dmax, off);
      const int k1 = __shfl_down_sync(0xffffffffu, kmin, off), k2 = __shfl_down_sync(0xffffffffu, kmax, off);
      if (o1 < dmin || (o1 == dmin && k1 < kmin)) dmin = o1, kmin = k1;
      if (o2 > dmax || (o2 == dmax && k2 < kmax)) dmax = o2, kmax = k2;
    }
    if ((threadIdx.x & 31) == 0) {
      // this warp's best of the two error lists (lowest key at equal error)
      long long best_err = LLONG_MAX;
      int best_key = INT_MAX;
      if (kmin != INT_MAX) best_err = dmin + tot_neg, best_key = kmin;
      if (kmax != INT_MAX) {
        const long long em = tot_pos - dmax;
        if (em < best_err || (em == best_err && kmax < best_key)) best_err = em, best_key = kmax;
      }
      s_cand[threadIdx.x >> 5] = {best_err, best_key};
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      long long best_err = s_cand[0].err;
      int best_key = s_cand[0].key;
      for (int w = 1; w < (int)blockDim.x / 32; ++w)
        if (s_cand[w].err < best_err || (s_cand[w].err == best_err && s_cand[w].key < best_key))
          best_err = s_cand[w].err, best_key = s_cand[w].key;
      P.feat_err[f] = best_err;
      P.feat_pos[f] = best_key;
    }
    grid.sync();
    if (threadIdx.x == 0) {
      long long be = LLONG_MAX;
      int bf = -1, bk = 0;
      for (int g = 0; g < F; ++g)
        if (P.feat_pos[g] != INT_MAX && P.feat_err[g] < be) be = P.feat_err[g], bf = g, bk = P.feat_pos[g];
      if (bf < 0) {  // every feature constant: majority constant stump
        const double pol = 2 * tot_neg <= total ? 1.0 : -1.0;  // +1 iff sum(w y) >= 0
        s_feat = 0;
        s_thr = __longlong_as_double(0xfff0000000000000LL);
        s_pol = pol;
        s_err = (double)(pol > 0 ? tot_neg : total - tot_neg) / (double)total;
      } else {
        const double *xb = P.xsorted + (size_t)bf * n;
        const int i = bk >> 1;
        s_feat = bf;
        s_thr = 0.5 * (xb[i] + xb[i + 1]);
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
    {
      const double a = s_alpha, thr = s_thr, pol = s_pol;
      const int feat = s_feat;
      const double e_agree = exp(-a), e_miss = exp(a);
      double part = 0.0;
      for (int i = w_lo + threadIdx.x; i < w_hi; i += blockDim.x) {
        const double pred = P.xs[(size_t)i * F + feat] > thr ? pol : -pol;
        const double wn = P.w[i] * inv_s * ((P.y[i] * pred > 0.0) ? e_agree : e_miss);
        P.w[i] = wn;
        part += wn;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) part += __shfl_down_sync(0xffffffffu, part, off);
      if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = part;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)blockDim.x / 32; ++w) t += s_red[w];
        P.wpart[blockIdx.x] = t;
      }
    }
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) write_result(count, n, n_pos_all, P.out_count, P.out_intercept);
}

__global__ void transpose_cols(const double *xs, int n, int F, double *xt, int *iota) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * F) return;
  const int r = (int)(i / F), c = (int)(i % F);
  xt[(size_t)c * n + r] = __dadd_rn(xs[i], 0.0);  // -0.0 -> +0.0: numpy sorts them as equal
  iota[(size_t)c * n + r] = r;  // per-column sample ids for the segmented sort
}

__global__ void labels_from_betas(const double *betas, int n, double *y, int *npos) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool pos = betas[i] > 0.0;
  y[i] = pos ? 1.0 : -1.0;
  if (pos) atomicAdd(npos, 1);
}

__global__ void fill_value(double *w, int n, double v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) w[i] = v;
}

// --------------------------------------------------------------- lstsq ----
// Householder QR with column pivoting in one CTA (fp64).  Returns rank.
constexpr int kLsMaxN = 4096, kLsMaxB = 64;

__global__ void lstsq_kernel(const double *design, const double *levels, int n, int nb, const int *cols, int ncols,
                             double *coeffs, int *rank_out) {
  extern __shared__ double sm[];
  double *A = sm;                       // [ncols][n] column-major
  double *b = A + (size_t)ncols * n;    // [n]
  __shared__ double s_norm[kLsMaxB];
  __shared__ int s_perm[kLsMaxB];
  __shared__ double s_tau, s_beta, s_r00;
  __shared__ int s_rank;
  for (int i = threadIdx.x; i < n * ncols; i += blockDim.x) {
    const int c = i / n, r = i % n;
    A[i] = design[(size_t)r * nb + cols[c]];
  }
  for (int r = threadIdx.x; r < n; r += blockDim.x) b[r] = levels[r];
  if (threadIdx.x < ncols) s_perm[threadIdx.x] = threadIdx.x;
  if (threadIdx.x == 0) s_rank = 0;
  __syncthreads();
  const int kmax = min(n, ncols);
  for (int k = 0; k < kmax; ++k) {
    // column norms of the trailing block, pick the largest
    for (int c = k + (threadIdx.x >> 5); c < ncols; c += blockDim.x >> 5) {
      double s = 0.0;
      for (int r = k + (threadIdx.x & 31); r < n; r += 32) s += A[(size_t)c * n + r] * A[(size_t)c * n + r];
      for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
      if ((threadIdx.x & 31) == 0) s_norm[c] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int best = k;
      for (int c = k + 1; c < ncols; ++c)
        if (s_norm[c] > s_norm[best]) best = c;
      s_beta = best;
    }
    __syncthreads();
    const int piv = (int)s_beta;
    if (piv != k) {
      for (int r = threadIdx.x; r < n; r += blockDim.x) {
        const double t = A[(size_t)k * n + r];
        A[(size_t)k * n + r] = A[(size_t)piv * n + r];
        A[(size_t)piv * n + r] = t;
      }
      if (threadIdx.x == 0) {
        const int t = s_perm[k];
        s_perm[k] = s_perm[piv];
        s_perm[piv] = t;
      }
    }
    __syncthreads();
    // Householder vector for column k
    if (threadIdx.x == 0) {
      double nrm = 0.0;
      for (int r = k; r < n; ++r) nrm += A[(size_t)k * n + r] * A[(size_t)k * n + r];
      nrm = sqrt(nrm);
      const double x0 = A[(size_t)k * n + k];
      const double alpha = x0 >= 0.0 ? -nrm : nrm;
      if (k == 0) s_r00 = fabs(alpha);
      const double tol = (double)max(n, ncols) * 2.220446049250313e-16 * s_r00;
      if (!(fabs(alpha) > tol) || nrm == 0.0) {
        s_tau = 0.0;
      } else {
        s_rank = k + 1;
        const double v0 = x0 - alpha;
        A[(size_t)k * n + k] = alpha;
        for (int r = k + 1; r < n; ++r) A[(size_t)k * n + r] /= v0;
        s_tau = -v0 / alpha;  // H = I - tau v v^T with v = [1, A[k+1..n)]
      }
    }
    __syncthreads();
    const double tau = s_tau;
    if (tau == 0.0) break;
    // apply H to trailing columns and b
    for (int c = k + 1 + (threadIdx.x >> 5); c <= ncols; c += blockDim.x >> 5) {
      double *col = c < ncols ? A + (size_t)c * n : b;
      double s = 0.0;
      for (int r = k + (threadIdx.x & 31); r < n; r += 32) s += (r == k ? 1.0 : A[(size_t)k * n + r]) * col[r];
      for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
      s = __shfl_sync(0xffffffffu, s, 0) * tau;
      for (int r = k + (threadIdx.x & 31); r < n; r += 32) col[r] -= s * (r == k ? 1.0 : A[(size_t)k * n + r]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int rk = s_rank;
    *rank_out = rk;
    double x[kLsMaxB];
    for (int i = rk - 1; i >= 0; --i) {
      double s = b[i];
      for (int j = i + 1; j < rk; ++j) s -= A[(size_t)j * n + i] * x[j];
      x[i] = s / A[(size_t)i * n + i];
    }
    for (int c = 0; c < nb; ++c) coeffs[c] = 0.0;
    for (int i = 0; i < rk; ++i) coeffs[cols[s_perm[i]]] = x[i];
  }
}

}  // namespace brm

using namespace brm;

namespace {
int bfail(int code, const std::string &msg) { return brm::set_error(code, "%s", msg.c_str()); }
bool is_dev(const void *p) {
  cudaPointerAttributes a;
  if (!p || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}
}  // namespace

#define BCU(call)                                                                        \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      rc = bfail(e_ == cudaErrorMemoryAllocation ? BRM_ENOMEM : BRM_ECUDA,               \
                 std::string(#call) + ": " + cudaGetErrorString(e_));                    \
      goto done;                                                                         \
    }                                                                                    \
  } while (0)

namespace {
// Stream-ordered scratch that frees itself.
struct Scratch {
  cudaStream_t s;
  std::vector<void *> ptrs;
  explicit Scratch(cudaStream_t st) : s(st) {}
  ~Scratch() {
    for (void *p : ptrs) cudaFreeAsync(p, s);
  }
  template <typename T>
  cudaError_t get(T **p, size_t count) {
    void *q = nullptr;
    cudaError_t e = cudaMallocAsync(&q, std::max<size_t>(count, 1) * sizeof(T), s);
    if (e == cudaSuccess) ptrs.push_back(q);
    *p = static_cast<T *>(q);
    return e;
  }
};
}  // namespace

extern "C" int brm_fit_ensemble(int32_t device, int32_t mode, int32_t flags, void *stream, const double *xs,
                                const double *betas, const double *weights, int64_t n64, int32_t F, int32_t rounds,
                                int32_t *out_feat, double *out_thr, double *out_pol, double *out_alpha,
                                double *out_err, int32_t *out_count, double *out_intercept) {
  const bool raw = flags & BRM_FIT_SINGLE_STUMP;
  const bool dev_out = flags & BRM_FIT_DEVICE_RESULT;
  if (!xs || !betas || !out_count || !out_intercept) return bfail(BRM_EINVAL, "NULL argument");
  if (dev_out && !(is_dev(out_feat) && is_dev(out_thr) && is_dev(out_pol) && is_dev(out_alpha) && is_dev(out_err) &&
                   is_dev(out_count) && is_dev(out_intercept)))
    return bfail(BRM_EINVAL, "BRM_FIT_DEVICE_RESULT needs device output pointers");
  if (rounds < 1) return bfail(BRM_EINVAL, "need at least one round, got " + std::to_string(rounds));
  if (n64 < 1 || n64 > (1 << 26)) return bfail(BRM_EINVAL, "training set size out of range");
  if (F < 1 || F > 148) return bfail(BRM_EINVAL, "feature count out of range");
  if (!out_feat || !out_thr || !out_pol || !out_alpha || !out_err) return bfail(BRM_EINVAL, "NULL stump outputs");
  const int n = (int)n64;
  if (raw) rounds = 1;
  int rc = BRM_OK;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  retain_pool(device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  {
    Scratch S(s);
    double *d_xs, *d_b, *d_xt, *d_xsorted, *d_y, *d_w, *d_wn, *d_pc, *d_nc, *d_err, *d_wsub, *d_thr, *d_pol,
        *d_alpha, *d_rerr;
    int *d_iota, *d_order, *d_pos, *d_npos, *d_feat, *d_count, *d_pid, *d_nid, *d_cnt, *d_lvl, *d_segoff;
    int2 *d_leaves, *d_children, *d_brk;
    void *d_tmp = nullptr;
    size_t tmp_bytes = 0;
    int npos = 0;
    PwTree tree;
    int root = 0;
    BCU(S.get(&d_xs, (size_t)n * F));
    BCU(cudaMemcpyAsync(d_xs, xs, sizeof(double) * (size_t)n * F, cudaMemcpyDefault, s));
    if (!is_dev(xs)) count_transfer(sizeof(double) * (size_t)n * F, 0);
    if (!is_dev(betas)) count_transfer(sizeof(double) * n, 0);
    BCU(S.get(&d_b, n));
    BCU(cudaMemcpyAsync(d_b, betas, sizeof(double) * n, cudaMemcpyDefault, s));
    BCU(S.get(&d_y, n));
    BCU(S.get(&d_npos, 1));
    BCU(cudaMemsetAsync(d_npos, 0, sizeof(int), s));
    {
      const int tok = prof_begin(PK_AUX, s);
      labels_from_betas<<<(n + 255) / 256, 256, 0, s>>>(d_b, n, d_y, d_npos);
      prof_end(tok, s);
    }
    if (!dev_out) {  // (device results: the kernel itself handles one class)
      BCU(cudaMemcpyAsync(&npos, d_npos, sizeof(int), cudaMemcpyDeviceToHost, s));
      BCU(cudaStreamSynchronize(s));
    }
    if (!dev_out && !raw && (npos == 0 || npos == n)) {
      // one class: zero-round ensemble carrying the class sign (boosting.py:185-187)
      *out_count = 0;
      *out_intercept = npos == n ? 1.0 : -1.0;
      goto done;
    }
    BCU(S.get(&d_xt, (size_t)n * F));
    BCU(S.get(&d_xsorted, (size_t)n * F));
    BCU(S.get(&d_iota, (size_t)n * F));
    BCU(S.get(&d_segoff, F + 1));
    BCU(S.get(&d_order, (size_t)n * F));
    {
      const int tok = prof_begin(PK_AUX, s);
      transpose_cols<<<(unsigned)(((int64_t)n * F + 255) / 256), 256, 0, s>>>(d_xs, n, F, d_xt, d_iota);
      prof_end(tok, s);
    }
    // stable LSD radix sort of each column: ties keep index order, as np.argsort(kind="stable")
    {
      // one segmented sort for all columns (segment f = column f)
      std::vector<int> off(F + 1);
      for (int f = 0; f <= F; ++f) off[f] = f * n;
      BCU(cudaMemcpyAsync(d_segoff, off.data(), sizeof(int) * (F + 1), cudaMemcpyHostToDevice, s));
      BCU(cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tmp_bytes, d_xt, d_xsorted, d_iota, d_order, n * F, F,
                                                   d_segoff, d_segoff + 1, 0, 64, s));
      BCU(S.get(reinterpret_cast<char **>(&d_tmp), tmp_bytes));
      BCU(cub::DeviceSegmentedRadixSort::SortPairs(d_tmp, tmp_bytes, d_xt, d_xsorted, d_iota, d_order, n * F, F,
                                                   d_segoff, d_segoff + 1, 0, 64, s));
    }
    BCU(S.get(&d_pid, (size_t)n * F));
    BCU(S.get(&d_nid, (size_t)n * F));
    BCU(S.get(&d_cnt, (size_t)n * F));
    BCU(S.get(&d_brk, (size_t)n * F));
    {
      const int tok = prof_begin(PK_AUX, s);
      split_classes<<<F, 256, 0, s>>>(d_order, d_y, d_xsorted, n, d_pid, d_nid, d_cnt, d_brk);
      prof_end(tok, s);
    }
    BCU(S.get(&d_w, n));
    if (weights) {
      BCU(cudaMemcpyAsync(d_w, weights, sizeof(double) * n, cudaMemcpyDefault, s));
    } else {
      const int tok = prof_begin(PK_AUX, s);
      fill_value<<<(n + 255) / 256, 256, 0, s>>>(d_w, n, 1.0 / n);
      prof_end(tok, s);
    }
    BCU(S.get(&d_wn, (size_t)n * F));
    BCU(S.get(&d_pc, (size_t)n * F));
    BCU(S.get(&d_nc, (size_t)n * F));
    BCU(S.get(&d_err, F));
    BCU(S.get(&d_pos, F));
    BCU(S.get(&d_wsub, (size_t)n * F));
    BCU(S.get(&d_feat, rounds));
    BCU(S.get(&d_thr, rounds));
    BCU(S.get(&d_pol, rounds));
    BCU(S.get(&d_alpha, rounds));
    BCU(S.get(&d_rerr, rounds));
    BCU(S.get(&d_count, 1));
    double *d_icept;
    BCU(S.get(&d_icept, 1));
    if (dev_out) {  // the kernel writes the caller's arrays
      d_feat = out_feat;
      d_thr = out_thr;
      d_pol = out_pol;
      d_alpha = out_alpha;
      d_rerr = out_err;
      d_count = out_count;
      d_icept = out_intercept;
    }
    root = pw_tree(n, tree);
    double *d_leafsum;
    BCU(S.get(&d_leafsum, tree.leaves.size()));
    BCU(S.get(&d_leaves, tree.leaves.size()));
    BCU(cudaMemcpyAsync(d_leaves, tree.leaves.data(), sizeof(int2) * tree.leaves.size(), cudaMemcpyHostToDevice, s));
    BCU(S.get(&d_children, tree.children.size()));
    if (!tree.children.empty())
      BCU(cudaMemcpyAsync(d_children, tree.children.data(), sizeof(int2) * tree.children.size(),
                          cudaMemcpyHostToDevice, s));
    BCU(S.get(&d_lvl, tree.level_end.size()));
    if (!tree.level_end.empty())
      BCU(cudaMemcpyAsync(d_lvl, tree.level_end.data(), sizeof(int) * tree.level_end.size(), cudaMemcpyHostToDevice,
                          s));
    {
      BoostParams P{};
      P.n = n;
      P.F = F;
      P.rounds = rounds;
      P.raw = raw ? 1 : 0;
      P.xs = d_xs;
      P.xsorted = d_xsorted;
      P.xt = d_xt;
      P.y = d_y;
      P.w = d_w;
      P.wn = d_wn;
      P.pos_idx = d_pid;
      P.neg_idx = d_nid;
      P.cntpos = d_cnt;
      P.brk = d_brk;
      P.pcum = d_pc;
      P.ncum = d_nc;
      P.leaves = d_leaves;
      P.n_leaves = (int)tree.leaves.size();
      P.children = d_children;
      P.level_end = d_lvl;
      P.n_levels = (int)tree.level_end.size();
      P.root = root;
      P.feat_err = d_err;
      P.feat_pos = d_pos;
      P.wsub = d_wsub;
      P.leafsum = d_leafsum;
      P.out_feat = d_feat;
      P.out_thr = d_thr;
      P.out_pol = d_pol;
      P.out_alpha = d_alpha;
      P.out_err = d_rerr;
      P.out_count = d_count;
      P.out_intercept = d_icept;
      P.n_pos = d_npos;
      long long *d_timing = nullptr;
      const bool timing = getenv("BRM_BOOST_TIMING") != nullptr;
      if (timing) {
        BCU(S.get(&d_timing, 12));
        BCU(cudaMemsetAsync(d_timing, 0, 12 * sizeof(long long), s));
      }
      P.timing = d_timing;
      int smem_max = 0;
      BCU(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
      const size_t smem_cap = (size_t)smem_max - 2048;  // static shared arrays of the kernel
      const size_t tree_bytes = sizeof(int2) * (tree.leaves.size() + tree.children.size()) +
                                sizeof(int) * tree.level_end.size();
      size_t smem = sizeof(double) * (2 * tree.leaves.size() + 4 * chain_padded_len(kTile));
      P.tree_smem = smem + tree_bytes <= smem_cap ? 1 : 0;
      if (P.tree_smem) smem += tree_bytes;
      void *boost_fn = (void *)boost_kernel;
      BCU(cudaFuncSetAttribute(boost_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      void *args[] = {&P};
      const int tok = prof_begin(PK_BOOST, s);
      if (mode == BRM_MODE_FAST) {
        FastBoostParams Q{};
        Q.n = n;
        Q.F = F;
        Q.rounds = rounds;
        Q.raw = raw ? 1 : 0;
        Q.xs = d_xs;
        Q.xsorted = d_xsorted;
        Q.y = d_y;
        Q.order = d_order;
        Q.w = d_w;
        BCU(S.get(&Q.ysorted, (size_t)F * n));
        BCU(S.get(&Q.wpart, F));
        long long *d_ferr = nullptr;
        BCU(S.get(&d_ferr, F));
        Q.feat_err = d_ferr;
        Q.feat_pos = d_pos;
        Q.out_feat = d_feat;
        Q.out_thr = d_thr;
        Q.out_pol = d_pol;
        Q.out_alpha = d_alpha;
        Q.out_err = d_rerr;
        Q.out_count = d_count;
        Q.out_intercept = d_icept;
        Q.n_pos = d_npos;
        void *qargs[] = {&Q};
        BCU(cudaLaunchCooperativeKernel((void *)boost_fast_kernel, dim3(F), dim3(kBoostThreads), qargs, 0, s));
      } else {
        BCU(cudaLaunchCooperativeKernel(boost_fn, dim3(F), dim3(kBoostThreads), args, smem, s));
      }
      prof_end(tok, s);
      if (timing) {
        long long h[12];
        BCU(cudaMemcpyAsync(h, d_timing, sizeof h, cudaMemcpyDeviceToHost, s));
        BCU(cudaStreamSynchronize(s));
        fprintf(stderr, "boost phases (kcycles, CTA 0): norm+total %.0f chains %.0f (positive chain alone %.0f) scan %.0f "
                "sync1 %.0f pick %.0f reweight+sync2 %.0f (reweight alone %.0f)\n",
                h[1] / 1e3, h[2] / 1e3, h[7] / 1e3, h[3] / 1e3, h[4] / 1e3, h[5] / 1e3, h[6] / 1e3, h[0] / 1e3);
        fprintf(stderr, "  sub-phases (kcycles): [8] %.0f [9] %.0f [10] %.0f [11] %.0f\n", h[8] / 1e3, h[9] / 1e3,
                h[10] / 1e3, h[11] / 1e3);
      }
    }
    BCU(cudaGetLastError());
    if (!dev_out) {
      int count = 0;
      double icept = 0.0;
      BCU(cudaMemcpyAsync(&count, d_count, sizeof(int), cudaMemcpyDeviceToHost, s));
      BCU(cudaMemcpyAsync(&icept, d_icept, sizeof(double), cudaMemcpyDeviceToHost, s));
      BCU(cudaStreamSynchronize(s));
      *out_count = count;
      *out_intercept = icept;
      if (count > 0) {
        BCU(cudaMemcpyAsync(out_feat, d_feat, sizeof(int) * count, cudaMemcpyDefault, s));
        BCU(cudaMemcpyAsync(out_thr, d_thr, sizeof(double) * count, cudaMemcpyDefault, s));
        BCU(cudaMemcpyAsync(out_pol, d_pol, sizeof(double) * count, cudaMemcpyDefault, s));
        BCU(cudaMemcpyAsync(out_alpha, d_alpha, sizeof(double) * count, cudaMemcpyDefault, s));
        BCU(cudaMemcpyAsync(out_err, d_rerr, sizeof(double) * count, cudaMemcpyDefault, s));
        count_transfer(0, (sizeof(int) + 4 * sizeof(double)) * count);
      }
    }
  }
done:
  if (!dev_out) cudaStreamSynchronize(s);
  if (prev >= 0) cudaSetDevice(prev);
  return rc;
}

extern "C" int brm_lstsq(int32_t device, void *stream, const double *design, const double *levels, int64_t n64,
                         int32_t nb, int32_t k, double *out_coeffs, int32_t *out_rank_deficient) {
  if (!design || !levels || !out_coeffs || !out_rank_deficient) return bfail(BRM_EINVAL, "NULL argument");
  if (nb < 1 || nb > kLsMaxB) return bfail(BRM_EINVAL, "basis size out of range");
  if (n64 < nb) return bfail(BRM_EINVAL, "need at least " + std::to_string(nb) + " probe points for the quadratic fit, got " + std::to_string(n64));
  if (n64 > kLsMaxN) return bfail(BRM_EINVAL, "too many probe points for the device fit");
  // the rank-deficient fallback keeps columns [1, z_a, z_a^2] of the quadratic basis
  // (packs.py:74-93), so the design must be that basis of k coordinates
  if (k < 0 || nb != 1 + k + k * (k + 1) / 2)
    return bfail(BRM_EINVAL, "basis size " + std::to_string(nb) + " is not the quadratic basis of " +
                                 std::to_string(k) + " coordinates");
  const int n = (int)n64;
  int rc = BRM_OK;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  retain_pool(device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // one device block: [coeffs nb][rank 1 (as int, in a double slot)][design n*nb][levels n][cols nb (int)],
  // so the full-rank case costs one allocation, one result copy and one sync
  unsigned char *blk = nullptr;
  std::vector<int> cols(nb);
  double hres[kLsMaxB + 1];  // coeffs, then the rank (an int) in the next slot
  int rank = 0;
  for (int c = 0; c < nb; ++c) cols[c] = c;
  const size_t smem_full = sizeof(double) * ((size_t)nb * n + n);
  const size_t off_rank = sizeof(double) * nb;
  const size_t off_design = off_rank + sizeof(double);
  const size_t off_levels = off_design + sizeof(double) * (size_t)n * nb;
  const size_t off_cols = off_levels + sizeof(double) * n;
  const size_t blk_bytes = off_cols + sizeof(int) * nb;
  double *d_coeffs, *d_design, *d_levels;
  int *d_rank, *d_cols;
  BCU(cudaMallocAsync(&blk, blk_bytes, s));
  d_coeffs = reinterpret_cast<double *>(blk);
  d_rank = reinterpret_cast<int *>(blk + off_rank);
  d_design = reinterpret_cast<double *>(blk + off_design);
  d_levels = reinterpret_cast<double *>(blk + off_levels);
  d_cols = reinterpret_cast<int *>(blk + off_cols);
  BCU(cudaMemcpyAsync(d_design, design, sizeof(double) * (size_t)n * nb, cudaMemcpyDefault, s));
  BCU(cudaMemcpyAsync(d_levels, levels, sizeof(double) * n, cudaMemcpyDefault, s));
  BCU(cudaMemcpyAsync(d_cols, cols.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, s));
  BCU(cudaFuncSetAttribute(lstsq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_full));
  {
    const int tok = prof_begin(PK_LSTSQ, s);
    lstsq_kernel<<<1, 256, smem_full, s>>>(d_design, d_levels, n, nb, d_cols, nb, d_coeffs, d_rank);
    prof_end(tok, s);
  }
  BCU(cudaGetLastError());
  BCU(cudaMemcpyAsync(hres, blk, off_rank + sizeof(int), cudaMemcpyDeviceToHost, s));
  BCU(cudaStreamSynchronize(s));
  std::memcpy(&rank, reinterpret_cast<unsigned char *>(hres) + off_rank, sizeof(int));
  *out_rank_deficient = rank < nb;
  if (rank < nb) {
    // keep [1, z_a, z_a^2], zero the cross terms (boundary_iz.py:264-275)
    std::vector<int> keep{0};
    for (int a = 1; a <= k; ++a) keep.push_back(a);
    int pos = 1 + k;
    for (int a = 0; a < k; ++a) {
      keep.push_back(pos);
      pos += k - a;
    }
    BCU(cudaMemcpyAsync(d_cols, keep.data(), sizeof(int) * keep.size(), cudaMemcpyHostToDevice, s));
    const int tok = prof_begin(PK_LSTSQ, s);
    lstsq_kernel<<<1, 256, sizeof(double) * (keep.size() * n + n), s>>>(d_design, d_levels, n, nb, d_cols,
                                                                        (int)keep.size(), d_coeffs, d_rank);
    prof_end(tok, s);
    BCU(cudaGetLastError());
    BCU(cudaMemcpyAsync(hres, blk, off_rank, cudaMemcpyDeviceToHost, s));
    BCU(cudaStreamSynchronize(s));
  }
  if (is_dev(out_coeffs)) {
    BCU(cudaMemcpyAsync(out_coeffs, d_coeffs, sizeof(double) * nb, cudaMemcpyDeviceToDevice, s));
  } else {
    std::memcpy(out_coeffs, hres, sizeof(double) * nb);
  }
done:
  if (blk) {
    cudaFreeAsync(blk, s);
    if (rc != BRM_OK) cudaStreamSynchronize(s);
  }
  if (prev >= 0) cudaSetDevice(prev);
  return rc;
}
