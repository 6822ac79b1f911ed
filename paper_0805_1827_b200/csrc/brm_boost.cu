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

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <cmath>
#include <string>
#include <mutex>
#include <vector>

#include "../../include/bermuda_b200.h"
#include "brm_internal.h"
#include "brm_rng.cuh"

namespace cg = cooperative_groups;

namespace brm {

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

// Self-test reference (brm_selftest_math kind 8): np.cumsum of a[0..n) by one
// thread, the sequential chain the exact scan (kind 10) must reproduce.
__global__ void chain_selftest(int kind, const double *a, int64_t n, double *out) {
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) out[i] = acc = __dadd_rn(acc, a[i]);
  }
}

void *chain_selftest_kernel() { return (void *)&chain_selftest; }

}  // namespace brm
#include "brm_boost_exact.cuh"
namespace brm {

void *exact_scan_selftest_kernel() { return (void *)&exact_scan_selftest; }

}  // namespace brm
#include "brm_boost_cluster.cuh"
namespace brm {

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
// Quadratic boundary regression (boundary_iz.py:250-276) on the device:
// Householder QR with column pivoting in one CTA per fit (fp64), the
// rank-deficient fallback to the cross-term-free basis inside the kernel.
// Fit g solves design[J x nb] (shared) against levels[g*J .. g*J+J) (their
// logs in log space), writes its coefficients to out[g*nb ..], its rank to
// rank_out[g], and -- for the device-resident I&Z date loop -- into the rule
// image: rows dst[g*row_stride + (0 .. rows-1)*nb] of the surface block.
__device__ __forceinline__ double ls_warp_sum(double s) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  return s;
}

// QR least squares over the design columns cols[0..ncols) of A (column-major,
// [ncols][n] in shared memory, overwritten) and b; returns the rank, x in x[].
__device__ int ls_solve(double *A, double *b, int n, int ncols, int *s_perm, double *s_norm, double *x,
                        double *s_scal) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (threadIdx.x < ncols) s_perm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  int rank = 0;
  double r00 = 0.0;
  const int kmax = min(n, ncols);
  for (int k = 0; k < kmax; ++k) {
    // column norms of the trailing block; the largest is the pivot
    for (int c = k + warp; c < ncols; c += nw) {
      double s = 0.0;
      for (int r = k + lane; r < n; r += 32) s += A[(size_t)c * n + r] * A[(size_t)c * n + r];
      s = ls_warp_sum(s);
      if (lane == 0) s_norm[c] = s;
    }
    __syncthreads();
    int piv = k;
    for (int c = k + 1; c < ncols; ++c)
      if (s_norm[c] > s_norm[piv]) piv = c;
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
    // Householder vector of column k (warp 0), then its scaling (all threads)
    if (warp == 0) {
      double s = 0.0;
      for (int r = k + lane; r < n; r += 32) s += A[(size_t)k * n + r] * A[(size_t)k * n + r];
      const double nrm = sqrt(ls_warp_sum(s));
      const double x0 = A[(size_t)k * n + k];
      const double alpha = x0 >= 0.0 ? -nrm : nrm;
      if (k == 0) r00 = fabs(alpha);
      const double tol = (double)max(n, ncols) * 2.220446049250313e-16 * (k == 0 ? fabs(alpha) : s_scal[2]);
      if (lane == 0) {
        if (k == 0) s_scal[2] = fabs(alpha);
        if (!(fabs(alpha) > tol) || nrm == 0.0) {
          s_scal[0] = 0.0;
        } else {
          s_scal[0] = -(x0 - alpha) / alpha;  // tau: H = I - tau v v^T, v = [1, A[k+1..n) / v0]
          s_scal[1] = x0 - alpha;             // v0
          A[(size_t)k * n + k] = alpha;
        }
      }
    }
    __syncthreads();
    const double tau = s_scal[0];
    if (tau == 0.0) break;
    rank = k + 1;
    const double v0 = s_scal[1];
    for (int r = k + 1 + threadIdx.x; r < n; r += blockDim.x) A[(size_t)k * n + r] /= v0;
    __syncthreads();
    // apply H to the trailing columns and b (a warp per column)
    for (int c = k + 1 + warp; c <= ncols; c += nw) {
      double *col = c < ncols ? A + (size_t)c * n : b;
      double s = 0.0;
      for (int r = k + lane; r < n; r += 32) s += (r == k ? 1.0 : A[(size_t)k * n + r]) * col[r];
      s = ls_warp_sum(s) * tau;
      for (int r = k + lane; r < n; r += 32) col[r] -= s * (r == k ? 1.0 : A[(size_t)k * n + r]);
    }
    __syncthreads();
  }
  (void)r00;
  if (threadIdx.x == 0) {
    double y[kLsMaxB];
    for (int i = rank - 1; i >= 0; --i) {
      double s = b[i];
      for (int j = i + 1; j < rank; ++j) s -= A[(size_t)j * n + i] * y[j];
      y[i] = s / A[(size_t)i * n + i];
    }
    for (int c = 0; c < ncols; ++c) x[c] = 0.0;
    for (int i = 0; i < rank; ++i) x[s_perm[i]] = y[i];
  }
  __syncthreads();
  return rank;
}

__global__ void __launch_bounds__(256) ls_fit_kernel(LsParams P) {
  extern __shared__ double sm[];
  const int n = P.J, nb = P.nb, g = blockIdx.x;
  double *A = sm;                      // [nb][n] column-major
  double *b = A + (size_t)nb * n;      // [n]
  __shared__ double s_norm[kLsMaxB], s_x[kLsMaxB], s_scal[4];
  __shared__ int s_perm[kLsMaxB], s_cols[kLsMaxB];
  const double *lv = P.levels + (size_t)g * n;
  for (int i = threadIdx.x; i < n * nb; i += blockDim.x) {
    const int c = i / n, r = i % n;
    A[i] = P.design[(size_t)r * nb + c];
  }
  for (int r = threadIdx.x; r < n; r += blockDim.x) b[r] = P.log_space ? log(lv[r]) : lv[r];
  __syncthreads();
  int rank = ls_solve(A, b, n, nb, s_perm, s_norm, s_x, s_scal);
  double coef[kLsMaxB];
  for (int c = 0; c < nb; ++c) coef[c] = s_x[c];
  const int rank_full = rank;
  if (rank < nb) {
    // keep [1, z_a, z_a^2], zero the cross terms (boundary_iz.py:264-275)
    if (threadIdx.x == 0) {
      int q = 0, pos = 1 + P.k;
      s_cols[q++] = 0;
      for (int a = 1; a <= P.k; ++a) s_cols[q++] = a;
      for (int a = 0; a < P.k; ++a) {
        s_cols[q++] = pos;
        pos += P.k - a;
      }
    }
    __syncthreads();
    const int nk = 1 + 2 * P.k;
    for (int i = threadIdx.x; i < n * nk; i += blockDim.x) {
      const int c = i / n, r = i % n;
      A[i] = P.design[(size_t)r * nb + s_cols[c]];
    }
    for (int r = threadIdx.x; r < n; r += blockDim.x) b[r] = P.log_space ? log(lv[r]) : lv[r];
    __syncthreads();
    ls_solve(A, b, n, nk, s_perm, s_norm, s_x, s_scal);
    for (int c = 0; c < nb; ++c) coef[c] = 0.0;
    for (int c = 0; c < nk; ++c) coef[s_cols[c]] = s_x[c];
  }
  if (threadIdx.x == 0) {
    if (P.out)
      for (int c = 0; c < nb; ++c) P.out[(size_t)g * nb + c] = coef[c];
    if (P.rank_out) P.rank_out[g] = rank_full;
    if (P.dst)
      for (int row = 0; row < P.dst_rows; ++row)
        for (int c = 0; c < nb; ++c) P.dst[(size_t)g * P.dst_fit_stride + (size_t)row * nb + c] = coef[c];
  }
}

size_t ls_fit_smem(int J, int nb) { return sizeof(double) * ((size_t)nb * J + J); }

int launch_ls_fit(const LsParams &P, int n_fits, cudaStream_t s) {
  const size_t smem = ls_fit_smem(P.J, P.nb);
  cudaError_t e = cudaFuncSetAttribute(ls_fit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return set_error(BRM_ECUDA, "ls_fit: %s", cudaGetErrorString(e));
  const int tok = prof_begin(PK_LSTSQ, s);
  ls_fit_kernel<<<n_fits, 256, smem, s>>>(P);
  prof_end(tok, s);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(BRM_ECUDA, "ls_fit launch: %s", cudaGetErrorString(e));
  return BRM_OK;
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

namespace {
// Column sorts enqueued ahead of their fit (brm_fit_presort): keyed by the
// feature matrix they sorted; brm_fit_ensemble on the same matrix takes the
// entry instead of transposing and sorting again.
struct Presort {
  int device;
  const double *xs;
  int n, F;
  double *xt, *xsorted;
  int *order;
  cudaEvent_t ready;
  const void *owner;  // the context whose brm_cmc_calc enqueued it (dropped with the context), or NULL
};
std::mutex g_ps_mu;
std::vector<Presort> g_ps;
constexpr size_t kPresortCap = 4;

void presort_release(const Presort &e, cudaStream_t s) {
  cudaFreeAsync(e.xt, s);
  cudaFreeAsync(e.xsorted, s);
  cudaFreeAsync(e.order, s);
  cudaEventDestroy(e.ready);
}

bool presort_take(int device, const double *xs, int n, int F, Presort *out) {
  std::lock_guard<std::mutex> lk(g_ps_mu);
  for (size_t i = 0; i < g_ps.size(); ++i)
    if (g_ps[i].device == device && g_ps[i].xs == xs && g_ps[i].n == n && g_ps[i].F == F) {
      *out = g_ps[i];
      g_ps.erase(g_ps.begin() + (long)i);
      return true;
    }
  return false;
}
}  // namespace

namespace brm {
int fit_presort(int32_t device, cudaStream_t s, const double *xs, int64_t n64, int32_t F, cudaEvent_t mid,
                const void *owner);
void fit_presort_drop(const void *owner, cudaStream_t s);
}
extern "C" int brm_fit_presort(int32_t device, void *stream, const double *xs, int64_t n64, int32_t F) {
  return brm::fit_presort(device, static_cast<cudaStream_t>(stream), xs, n64, F, nullptr, nullptr);
}

// Sorts a context enqueued and no fit took (an exception between brm_cmc_calc and the fit): dropped
// with the context, so that a later matrix at the same address never meets them.
void brm::fit_presort_drop(const void *owner, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_ps_mu);
  for (size_t i = 0; i < g_ps.size();) {
    if (g_ps[i].owner == owner) {
      presort_release(g_ps[i], s);
      g_ps.erase(g_ps.begin() + (long)i);
    } else {
      ++i;
    }
  }
}

// mid (optional): recorded between the transpose and the sort, so that a caller can hold its own
// next kernel until the sort is the next thing the side stream launches
int brm::fit_presort(int32_t device, cudaStream_t s, const double *xs, int64_t n64, int32_t F, cudaEvent_t mid,
                     const void *owner) {
  if (!xs || !is_dev(xs)) return bfail(BRM_EINVAL, "brm_fit_presort needs a device feature matrix");
  if (n64 < 1 || n64 > (int64_t)kCodeId || F < 1 || F > 148 || n64 * F > (int64_t)INT_MAX)
    return bfail(BRM_EINVAL, "training set size out of range");
  const int n = (int)n64;
  int rc = BRM_OK;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  retain_pool(device);
  Presort e{device, xs, n, F, nullptr, nullptr, nullptr, nullptr, owner};
  {
    Presort stale;
    while (presort_take(device, xs, n, F, &stale)) presort_release(stale, s);  // a sort of this matrix nobody used
    Scratch S(s);
    int *d_iota;
    unsigned long long *k0, *k1;
    unsigned *i0, *i1;
    BCU(cudaMallocAsync((void **)&e.xt, sizeof(double) * (size_t)n * F, s));
    BCU(cudaMallocAsync((void **)&e.xsorted, sizeof(double) * (size_t)n * F, s));
    BCU(cudaMallocAsync((void **)&e.order, sizeof(int) * (size_t)n * F, s));
    BCU(S.get(&d_iota, (size_t)n * F));
    BCU(S.get(&k0, (size_t)n * F));
    BCU(S.get(&k1, (size_t)n * F));
    BCU(S.get(&i0, (size_t)n * F));
    BCU(S.get(&i1, (size_t)n * F));
    {
      const int tok = prof_begin(PK_AUX, s);
      transpose_cols<<<(unsigned)(((int64_t)n * F + 255) / 256), 256, 0, s>>>(xs, n, F, e.xt, d_iota);
      prof_end(tok, s);
    }
    if (mid) BCU(cudaEventRecord(mid, s));
    {
      const int tok = prof_begin(PK_AUX, s);
      sort_columns<<<F, kSortThreads, 0, s>>>(e.xt, n, k0, i0, k1, i1, e.xsorted, e.order);
      prof_end(tok, s);
    }
    BCU(cudaGetLastError());
    BCU(cudaEventCreateWithFlags(&e.ready, cudaEventDisableTiming));
    BCU(cudaEventRecord(e.ready, s));
    {
      std::lock_guard<std::mutex> lk(g_ps_mu);
      while (g_ps.size() >= kPresortCap) {  // bounded: drop the oldest unused sort
        presort_release(g_ps.front(), s);
        g_ps.erase(g_ps.begin());
      }
      g_ps.push_back(e);
    }
    e = Presort{};
  }
done:
  if (rc != BRM_OK) {
    if (e.xt) cudaFreeAsync(e.xt, s);
    if (e.xsorted) cudaFreeAsync(e.xsorted, s);
    if (e.order) cudaFreeAsync(e.order, s);
    if (e.ready) cudaEventDestroy(e.ready);
  }
  if (prev >= 0) cudaSetDevice(prev);
  return rc;
}

extern "C" int brm_fit_ensemble(int32_t device, int32_t mode, int32_t flags, void *stream, const double *xs,
                                const double *betas, const double *weights, int64_t n64, int32_t F, int32_t rounds,
                                int32_t *out_feat, double *out_thr, double *out_pol, double *out_alpha,
                                double *out_err, int32_t *out_count, double *out_intercept, int32_t *out_n_pos) {
  const bool raw = flags & BRM_FIT_SINGLE_STUMP;
  const bool dev_out = flags & BRM_FIT_DEVICE_RESULT;
  if (!xs || !betas || !out_count || !out_intercept) return bfail(BRM_EINVAL, "NULL argument");
  if (dev_out && !(is_dev(out_feat) && is_dev(out_thr) && is_dev(out_pol) && is_dev(out_alpha) && is_dev(out_err) &&
                   is_dev(out_count) && is_dev(out_intercept) && (!out_n_pos || is_dev(out_n_pos))))
    return bfail(BRM_EINVAL, "BRM_FIT_DEVICE_RESULT needs device output pointers");
  if (rounds < 1) return bfail(BRM_EINVAL, "need at least one round, got " + std::to_string(rounds));
  if (n64 < 1 || n64 > (int64_t)kCodeId) return bfail(BRM_EINVAL, "training set size out of range");
  if (F < 1 || F > 148) return bfail(BRM_EINVAL, "feature count out of range");
  // every per-feature array is indexed [f * n + i] in 64-bit, but the kernels
  // take n as int and the fast kernel's scans are int: keep n * F in int range
  if (n64 * F > (int64_t)INT_MAX) return bfail(BRM_EINVAL, "training set too large (n * F > 2^31 - 1)");
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
    double *d_xs, *d_b, *d_xt, *d_xsorted, *d_y, *d_w, *d_err, *d_thr, *d_pol, *d_alpha, *d_rerr;
    int *d_iota, *d_order, *d_pos, *d_npos, *d_feat, *d_count;
    unsigned *d_code;
    int npos = 0;
    PwTree tree;
    int root = 0;
    Presort pre{};
    const bool presorted = presort_take(device, xs, n, F, &pre);
    if (presorted) {  // sorted ahead on another stream: take its arrays, freed in this call's stream order
      S.ptrs.push_back(pre.xt);
      S.ptrs.push_back(pre.xsorted);
      S.ptrs.push_back(pre.order);
      const cudaError_t we = cudaStreamWaitEvent(s, pre.ready, 0);
      cudaEventDestroy(pre.ready);
      BCU(we);
      d_xs = nullptr;
    } else {
      BCU(S.get(&d_xs, (size_t)n * F));
      BCU(cudaMemcpyAsync(d_xs, xs, sizeof(double) * (size_t)n * F, cudaMemcpyDefault, s));
    }
    if (!is_dev(xs)) count_transfer(sizeof(double) * (size_t)n * F, 0);
    if (!is_dev(betas)) count_transfer(sizeof(double) * n, 0);
    BCU(S.get(&d_b, n));
    BCU(cudaMemcpyAsync(d_b, betas, sizeof(double) * n, cudaMemcpyDefault, s));
    BCU(S.get(&d_y, n));
    if (out_n_pos && is_dev(out_n_pos)) {
      d_npos = out_n_pos;
    } else {
      BCU(S.get(&d_npos, 1));
    }
    BCU(cudaMemsetAsync(d_npos, 0, sizeof(int), s));
    {
      const int tok = prof_begin(PK_AUX, s);
      labels_from_betas<<<(n + 255) / 256, 256, 0, s>>>(d_b, n, d_y, d_npos);
      prof_end(tok, s);
    }
    if (!dev_out) {  // (device results: the kernel itself handles one class)
      BCU(cudaMemcpyAsync(&npos, d_npos, sizeof(int), cudaMemcpyDeviceToHost, s));
      BCU(cudaStreamSynchronize(s));
      if (out_n_pos && !is_dev(out_n_pos)) *out_n_pos = npos;
    }
    if (!dev_out && !raw && (npos == 0 || npos == n)) {
      // one class: zero-round ensemble carrying the class sign (boosting.py:185-187)
      *out_count = 0;
      *out_intercept = npos == n ? 1.0 : -1.0;
      goto done;
    }
    if (presorted) {
      d_xt = pre.xt;
      d_xsorted = pre.xsorted;
      d_order = pre.order;
    } else {
    BCU(S.get(&d_xt, (size_t)n * F));
    BCU(S.get(&d_xsorted, (size_t)n * F));
    BCU(S.get(&d_iota, (size_t)n * F));
    BCU(S.get(&d_order, (size_t)n * F));
    {
      const int tok = prof_begin(PK_AUX, s);
      transpose_cols<<<(unsigned)(((int64_t)n * F + 255) / 256), 256, 0, s>>>(d_xs, n, F, d_xt, d_iota);
      prof_end(tok, s);
    }
    {
      // stable argsort of every column (np.argsort(kind="stable")), own kernel
      unsigned long long *k0, *k1;
      unsigned *i0, *i1;
      BCU(S.get(&k0, (size_t)n * F));
      BCU(S.get(&k1, (size_t)n * F));
      BCU(S.get(&i0, (size_t)n * F));
      BCU(S.get(&i1, (size_t)n * F));
      const int tok = prof_begin(PK_AUX, s);
      sort_columns<<<F, kSortThreads, 0, s>>>(d_xt, n, k0, i0, k1, i1, d_xsorted, d_order);
      prof_end(tok, s);
    }
    }
    BCU(S.get(&d_w, n));
    if (weights) {
      BCU(cudaMemcpyAsync(d_w, weights, sizeof(double) * n, cudaMemcpyDefault, s));
    } else {
      const int tok = prof_begin(PK_AUX, s);
      fill_value<<<(n + 255) / 256, 256, 0, s>>>(d_w, n, 1.0 / n);
      prof_end(tok, s);
    }
    BCU(S.get(&d_err, 2 * F));
    BCU(S.get(&d_pos, 2 * F));
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
    {
      BCU(S.get(&d_code, (size_t)n * F));
      {
        const int tok = prof_begin(PK_AUX, s);
        build_codes<<<dim3((n + 255) / 256, F), 256, 0, s>>>(d_order, d_y, d_xsorted, n, d_code);
        prof_end(tok, s);
      }
      root = pw_tree(n, tree);
      int2 *d_leaves, *d_children;
      int *d_lvl;
      BCU(S.get(&d_leaves, tree.leaves.size()));
      BCU(cudaMemcpyAsync(d_leaves, tree.leaves.data(), sizeof(int2) * tree.leaves.size(), cudaMemcpyHostToDevice,
                          s));
      BCU(S.get(&d_children, std::max<size_t>(tree.children.size(), 1)));
      if (!tree.children.empty())
        BCU(cudaMemcpyAsync(d_children, tree.children.data(), sizeof(int2) * tree.children.size(),
                            cudaMemcpyHostToDevice, s));
      BCU(S.get(&d_lvl, std::max<size_t>(tree.level_end.size(), 1)));
      if (!tree.level_end.empty())
        BCU(cudaMemcpyAsync(d_lvl, tree.level_end.data(), sizeof(int) * tree.level_end.size(),
                            cudaMemcpyHostToDevice, s));
      CbParams P{};
      P.n = n;
      P.F = F;
      P.rounds = rounds;
      P.raw = raw ? 1 : 0;
      P.xsorted = d_xsorted;
      P.code = d_code;
      P.xt = d_xt;
      P.y = d_y;
      P.w0 = d_w;
      P.leaves = d_leaves;
      P.n_leaves = (int)tree.leaves.size();
      P.children = d_children;
      P.level_end = d_lvl;
      P.n_levels = (int)tree.level_end.size();
      P.root = root;
      P.margin = 2 * (n + 64);
      P.feat_err = d_err;
      P.feat_pos = d_pos;
      P.out_feat = d_feat;
      P.out_thr = d_thr;
      P.out_pol = d_pol;
      P.out_alpha = d_alpha;
      P.out_err = d_rerr;
      P.out_count = d_count;
      P.out_intercept = d_icept;
      P.n_pos = d_npos;
      const bool timing = getenv("BRM_BOOST_TIMING") != nullptr;
      long long *d_timing = nullptr;
      if (timing) {
        BCU(S.get(&d_timing, 16));
        BCU(cudaMemsetAsync(d_timing, 0, 16 * sizeof(long long), s));
        BCU(S.get(&P.n_fallback, 1));
        BCU(cudaMemsetAsync(P.n_fallback, 0, sizeof(unsigned long long), s));
        BCU(S.get(&P.n_events, 2));
        BCU(cudaMemsetAsync(P.n_events, 0, 2 * sizeof(int), s));
      }
      P.timing = d_timing;
      // cluster size: up to 8 CTAs per feature while every CTA of the
      // cooperative grid stays co-resident (one cluster per feature)
      int sms = 148;
      BCU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
      // fast mode with more features than SMs / 8: the two-CTAs-per-SM instance (wider clusters)
      const bool two_per_sm = mode == BRM_MODE_FAST && F * kCbMaxCluster > sms;
      const int slots = two_per_sm ? 2 * sms : sms;
      int cl = std::max(1, std::min(kCbMaxCluster, slots / F));
      // BRM_NCU_SAFE: one CTA per feature, no cluster launch attribute (Nsight
      // Compute cannot replay cooperative cluster launches); same results
      const bool ncu_safe = getenv("BRM_NCU_SAFE") != nullptr;
      if (ncu_safe) cl = 1;
      // BRM_BOOST_CL: cap the cluster size (A/B runs of the sync / work-per-thread trade)
      if (const char *e = getenv("BRM_BOOST_CL")) cl = std::max(1, std::min(cl, atoi(e)));
      const int L = (int)tree.leaves.size();
      // (slice_cap, pos_cap, dynamic shared memory) for cluster size c
      auto layout = [&](int c, int &slice_cap, int &pos_cap) {
        slice_cap = 0;
        for (int r = 0; r < c; ++r) {
          int lo, hi;
          cb_leaf_run(L, c, r, lo, hi);
          if (hi > lo) slice_cap = std::max(slice_cap, tree.leaves[hi - 1].x + tree.leaves[hi - 1].y - tree.leaves[lo].x);
        }
        slice_cap = std::max(slice_cap, 1);
        // positions per thread: spread one tile evenly when it fits, else full tiles
        const int qt = (int)std::min<int64_t>(kCbQ, ((int64_t)n + (int64_t)c * kCbThreads - 1) / ((int64_t)c * kCbThreads));
        const int ctile = c * qt * kCbThreads;
        pos_cap = (n + ctile - 1) / ctile * qt * kCbThreads;
        return cb_smem_bytes(L, (int)tree.children.size(), (int)tree.level_end.size(), slice_cap, pos_cap);
      };
      int smem_max = 0;
      BCU(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
      int slice_cap = 0, pos_cap = 0;
      size_t dyn = layout(cl, slice_cap, pos_cap);
      while (cl < kCbMaxCluster && cl * 2 <= slots / F && dyn + sizeof(CbShared) + 2048 > (size_t)smem_max)
        dyn = layout(++cl, slice_cap, pos_cap);  // (more CTAs -> smaller slices)
      if (dyn + sizeof(CbShared) + 2048 > (size_t)smem_max) {
        rc = bfail(BRM_EINVAL, "training set too large for the device AdaBoost's shared memory");
        goto done;
      }
      void *kfn = mode == BRM_MODE_FAST ? (two_per_sm ? (void *)boost_fast_cluster_kernel<2>
                                                      : (void *)boost_fast_cluster_kernel<1>)
                                        : (void *)boost_cluster_kernel;
      BCU(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
      cudaLaunchConfig_t lc{};
      cudaLaunchAttribute at[2];
      lc.blockDim = dim3(kCbThreads);
      lc.dynamicSmemBytes = dyn;
      lc.stream = s;
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
      at[1].id = cudaLaunchAttributeClusterDimension;
      at[1].val.clusterDim.y = 1;
      at[1].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 2;
      // every cluster must be resident at once (grid barrier)
      for (;; --cl) {
        dyn = layout(cl, slice_cap, pos_cap);
        BCU(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
        at[1].val.clusterDim.x = cl;
        lc.gridDim = dim3((unsigned)(F * cl));
        lc.dynamicSmemBytes = dyn;
        if (ncu_safe) {
          lc.numAttrs = 1;
          break;
        }
        if (max_active_clusters(kfn, lc, device) >= F || cl == 1) break;
      }
      P.cl = cl;
      P.qt = (int)std::min<int64_t>(kCbQ, ((int64_t)n + (int64_t)cl * kCbThreads - 1) / ((int64_t)cl * kCbThreads));
      P.slice_cap = slice_cap;
      P.pos_cap = pos_cap;
      double *d_fthr;
      BCU(S.get(&d_fthr, 2 * F));
      P.feat_thr = d_fthr;
      BCU(S.get(&P.feat_ierr, 2 * F));
      BCU(S.get(&P.chain_g, (size_t)2 * n * F));
      BCU(S.get(&P.wsub, (size_t)n * F * cl));
      {
        void *args[] = {&P};
        const int tok = prof_begin(PK_BOOST, s);
        // fast mode: the same cluster layout with fixed-point integer scans
        BCU(cudaLaunchKernelExC(&lc, kfn, args));
        prof_end(tok, s);
      }
      if (timing) {
        long long h[16];
        unsigned long long fb = 0;
        int ev[2];
        BCU(cudaMemcpyAsync(h, d_timing, sizeof(long long) * 16, cudaMemcpyDeviceToHost, s));
        BCU(cudaMemcpyAsync(&fb, P.n_fallback, sizeof fb, cudaMemcpyDeviceToHost, s));
        BCU(cudaMemcpyAsync(ev, P.n_events, sizeof ev, cudaMemcpyDeviceToHost, s));
        BCU(cudaStreamSynchronize(s));
        fprintf(stderr, "cluster boost (kcycles, cluster 0 CTA 0, %d rounds, %d x %d CTAs): chains %.0f "
                "split-merge %.0f grid-sync %.0f pick+alpha %.0f reweight %.0f setup %.0f; events %d + %d; "
                "fallback tiles %llu\n",
                rounds, F, cl, h[0] / 1e3, h[1] / 1e3, h[2] / 1e3, h[3] / 1e3, h[4] / 1e3, h[5] / 1e3, ev[0], ev[1],
                fb);
        fprintf(stderr, "  chain detail (kcycles): load+fpscan %.0f sync-d %.0f classify+scans %.0f sync-l %.0f "
                "push %.0f sync-e %.0f walk %.0f sync-w %.0f | reweight: pass1 %.0f tree1 %.0f\n",
                h[6] / 1e3, h[7] / 1e3, h[8] / 1e3, h[9] / 1e3, h[10] / 1e3, h[11] / 1e3, h[12] / 1e3, h[13] / 1e3,
                h[14] / 1e3, h[15] / 1e3);
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
  // one device block: [coeffs nb][rank (int, in a double slot)][design n*nb][levels n]
  unsigned char *blk = nullptr;
  double hres[kLsMaxB + 1];
  const size_t off_rank = sizeof(double) * nb;
  const size_t off_design = off_rank + sizeof(double);
  const size_t off_levels = off_design + sizeof(double) * (size_t)n * nb;
  const size_t blk_bytes = off_levels + sizeof(double) * n;
  LsParams P{};
  BCU(cudaMallocAsync(&blk, blk_bytes, s));
  BCU(cudaMemcpyAsync(blk + off_design, design, sizeof(double) * (size_t)n * nb, cudaMemcpyDefault, s));
  BCU(cudaMemcpyAsync(blk + off_levels, levels, sizeof(double) * n, cudaMemcpyDefault, s));
  P.design = reinterpret_cast<const double *>(blk + off_design);
  P.levels = reinterpret_cast<const double *>(blk + off_levels);
  P.J = n;
  P.nb = nb;
  P.k = k;
  P.out = reinterpret_cast<double *>(blk);
  P.rank_out = reinterpret_cast<int *>(blk + off_rank);
  if ((rc = launch_ls_fit(P, 1, s)) != BRM_OK) goto done;
  BCU(cudaMemcpyAsync(hres, blk, off_rank + sizeof(int), cudaMemcpyDeviceToHost, s));
  if (is_dev(out_coeffs)) BCU(cudaMemcpyAsync(out_coeffs, blk, sizeof(double) * nb, cudaMemcpyDeviceToDevice, s));
  BCU(cudaStreamSynchronize(s));
  {
    int rank = 0;
    std::memcpy(&rank, reinterpret_cast<unsigned char *>(hres) + off_rank, sizeof(int));
    *out_rank_deficient = rank < nb;
    if (!is_dev(out_coeffs)) std::memcpy(out_coeffs, hres, sizeof(double) * nb);
  }
done:
  if (blk) {
    cudaFreeAsync(blk, s);
    if (rc != BRM_OK) cudaStreamSynchronize(s);
  }
  if (prev >= 0) cudaSetDevice(prev);
  return rc;
}
