// brm_capi.cu -- extern "C" boundary (include/bermuda_b200.h).
//
// Host side of the engine: owns device images of the packs, stages host
// buffers, sizes grids to the SM count and launches the kernels on one
// stream.  No compute happens here besides argument checks and the
// 64-bit key hash of brm_derive_words.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cmath>
#include <map>
#include <tuple>
#include <limits>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/bermuda_b200.h"
#include "brm_internal.h"

using namespace brm;

namespace {
thread_local std::string g_err;
}

int brm::set_error(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

namespace {

#define fail brm::set_error

#define BRM_CUDA(call)                                                                           \
  do {                                                                                           \
    cudaError_t e_ = (call);                                                                     \
    if (e_ != cudaSuccess) {                                                                     \
      if (e_ == cudaErrorMemoryAllocation) return fail(BRM_ENOMEM, "%s: %s", #call, cudaGetErrorString(e_)); \
      return fail(BRM_ECUDA, "%s: %s", #call, cudaGetErrorString(e_));                           \
    }                                                                                            \
  } while (0)

#define BRM_TRY(expr)          \
  do {                         \
    int rc_ = (expr);          \
    if (rc_ != BRM_OK) return rc_; \
  } while (0)

struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

bool is_device_ptr(const void *p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// One argument buffer: the caller's device pointer, or a stream-ordered
// device copy of a host buffer (inputs) / a device buffer copied back to the
// host pointer by finish() (outputs).
struct Arg {
  void *host = nullptr;
  void *dev = nullptr;
  size_t bytes = 0;
  bool owned = false;
};

struct Call {
  cudaStream_t stream;
  std::vector<Arg> args;
  bool host_out = false;
  explicit Call(cudaStream_t s) : stream(s) {}
  ~Call() {
    for (auto &a : args)
      if (a.owned && a.dev) cudaFreeAsync(a.dev, stream);
  }
  template <typename T>
  int in(const T *p, size_t count, const T **out) {
    *out = nullptr;
    if (!p || count == 0) return BRM_OK;
    if (is_device_ptr(p)) {
      *out = p;
      return BRM_OK;
    }
    Arg a;
    a.bytes = count * sizeof(T);
    BRM_CUDA(cudaMallocAsync(&a.dev, a.bytes, stream));
    a.owned = true;
    args.push_back(a);
    BRM_CUDA(cudaMemcpyAsync(a.dev, p, a.bytes, cudaMemcpyHostToDevice, stream));
    count_transfer(a.bytes, 0);
    *out = static_cast<const T *>(a.dev);
    return BRM_OK;
  }
  template <typename T>
  int out(T *p, size_t count, T **dptr) {
    *dptr = nullptr;
    if (!p || count == 0) return BRM_OK;
    if (is_device_ptr(p)) {
      *dptr = p;
      return BRM_OK;
    }
    Arg a;
    a.host = p;
    a.bytes = count * sizeof(T);
    BRM_CUDA(cudaMallocAsync(&a.dev, a.bytes, stream));
    a.owned = true;
    args.push_back(a);
    host_out = true;
    *dptr = static_cast<T *>(a.dev);
    return BRM_OK;
  }
  template <typename T>
  int scratch(size_t count, T **dptr) {
    Arg a;
    a.bytes = std::max<size_t>(count, 1) * sizeof(T);
    BRM_CUDA(cudaMallocAsync(&a.dev, a.bytes, stream));
    a.owned = true;
    args.push_back(a);
    *dptr = static_cast<T *>(a.dev);
    return BRM_OK;
  }
  int finish() {
    BRM_CUDA(cudaGetLastError());
    for (auto &a : args)
      if (a.host) {
        BRM_CUDA(cudaMemcpyAsync(a.host, a.dev, a.bytes, cudaMemcpyDeviceToHost, stream));
        count_transfer(0, a.bytes);
      }
    if (host_out) BRM_CUDA(cudaStreamSynchronize(stream));
    return BRM_OK;
  }
};

struct DevInfo {
  int sms = 148;
  int max_smem = 227 * 1024;
};

DevInfo device_info(int dev) {
  DevInfo info;
  cudaDeviceGetAttribute(&info.sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&info.max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return info;
}

template <typename T>
int fetch(const T *src, size_t count, std::vector<T> &dst, const char *name) {
  dst.assign(count, T());
  if (count == 0) return BRM_OK;
  if (!src) return fail(BRM_EINVAL, "%s is NULL", name);
  // host arrays (the usual case: numpy packs) are copied on the host; a
  // cudaMemcpy per array is a driver round trip each
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, src) != cudaSuccess) cudaGetLastError();
  if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) {
    std::memcpy(dst.data(), src, count * sizeof(T));
    return BRM_OK;
  }
  BRM_CUDA(cudaMemcpy(dst.data(), src, count * sizeof(T), cudaMemcpyDefault));
  return BRM_OK;
}

int quad_basis_size(int k) { return 1 + k + k * (k + 1) / 2; }

}  // namespace

// cudaOccupancyMaxActiveClusters, cached per (kernel, cluster size, block,
// dynamic shared memory, device): the query costs tens of microseconds and
// the per-date probe / AdaBoost launches would repeat it.
int brm::max_active_clusters(const void *kernel, const cudaLaunchConfig_t &cfg, int device) {
  static std::mutex mu;
  static std::map<std::tuple<const void *, int, int, size_t, int>, int> cache;
  int csize = 1;
  for (unsigned i = 0; i < cfg.numAttrs; ++i)
    if (cfg.attrs[i].id == cudaLaunchAttributeClusterDimension) csize = (int)cfg.attrs[i].val.clusterDim.x;
  const auto key = std::make_tuple(kernel, csize, (int)cfg.blockDim.x, cfg.dynamicSmemBytes, device);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  int v = 0;
  if (cudaOccupancyMaxActiveClusters(&v, kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    v = 0;
  }
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = v;
  return v;
}

namespace {

}  // namespace

void brm::retain_pool(int dev) {
  static std::mutex mu;
  static bool done[64] = {};
  if (dev < 0 || dev >= 64) return;
  std::lock_guard<std::mutex> lk(mu);
  if (done[dev]) return;
  done[dev] = true;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    unsigned long long keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
}

namespace {

// Library stream of a device (created once, non-blocking, never destroyed).
cudaStream_t device_stream(int dev) {
  static std::mutex mu;
  static cudaStream_t streams[64] = {};
  if (dev < 0 || dev >= 64) return nullptr;
  retain_pool(dev);
  std::lock_guard<std::mutex> lk(mu);
  if (!streams[dev] && cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    streams[dev] = nullptr;
  }
  return streams[dev];
}

}  // namespace

struct brm_ctx {
  int device = 0;
  int mode = BRM_MODE_PARITY;
  ModelHdr hdr{};
  unsigned char *blob = nullptr;
  size_t blob_bytes = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t user_stream = nullptr;
  bool has_user_stream = false;
  DevInfo info;
  KernelTriple kern{};
  double *normals = nullptr;  // supplied-normals copy (device)
  cudaEvent_t ready = nullptr;  // image upload complete (waited on by every launch stream)
  cudaEvent_t retired = nullptr;  // scratch event: work of a stream the context stops using
  // brm_ctx_set_presort: brm_cmc_calc sorts the feature columns of the points it samples on a
  // side stream (high priority, beside the label walk), for the brm_fit_ensemble that follows
  bool presort = false;
  cudaStream_t side_stream = nullptr;
  cudaEvent_t side_event = nullptr, side_mid = nullptr;
  uint64_t nrm_base = 0, nrm_count = 0;
  int capacity = 0;  // > 0: slotted CMC image (brm_ctx_create_cmc)
  SlotDims slot{};
  cudaStream_t stream() const { return has_user_stream ? user_stream : own_stream; }
  bool fast() const { return mode == BRM_MODE_FAST; }
  const double *blob_dbl(int off) const { return reinterpret_cast<const double *>(blob) + off; }
};

namespace {

int smem_model(const brm_ctx *c) {
  return c->fast() ? model_smem_bytes<float>(c->hdr) : model_smem_bytes<double>(c->hdr);
}

// Opt in to `bytes` of dynamic shared memory and ask for the largest shared
// carve-out: the walkers' residency is a register / shared-memory trade, and
// the driver's default carve-out only fits the CTAs it predicts, which caps
// a 3-CTA-per-SM instance at 2.
int allow_smem(const void *kernel, int bytes) {
  BRM_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  BRM_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
  return BRM_OK;
}

int check_remaining(const brm_ctx *c, int m) {
  if (c->hdr.n_dates - m <= 0) return fail(BRM_EINVAL, "start date has no remaining exercise dates");
  if (m < 0) return fail(BRM_EINVAL, "negative start date %d", m);
  return BRM_OK;
}

// Launch walk_units over n_units x chunks and fold each unit.
struct WalkJob {
  int n_units = 0, per_unit = 0, chunk = 0;
  int64_t total_paths = 0;
  int m_start = 0;
  const double *starts = nullptr;
  int start_stride = 0;
  const uint64_t *keys = nullptr, *streams = nullptr;
  uint64_t seed = 0;
  int phase = 0, key_date = 0;
  int64_t item_base = 0;
  uint64_t draw_base = 0;
  double *path_out = nullptr;
  int32_t *stop_out = nullptr;
  int finish_mode = 0;
  const double *points = nullptr;
  double *out = nullptr;
};

int run_walk(brm_ctx *c, Call &call, const WalkJob &j) {
  if (j.n_units <= 0) return BRM_OK;
  WalkParams P{};
  P.hdr = c->hdr;
  P.blob = c->blob;
  P.n_units = j.n_units;
  P.per_unit = j.per_unit;
  P.chunk = std::max(1, std::min(j.chunk, kMaxChunk));
  P.chunks_per_unit = std::max(1, (j.per_unit + P.chunk - 1) / P.chunk);
  P.n_items = j.n_units * P.chunks_per_unit;
  P.total_paths = j.total_paths;
  P.m_start = j.m_start;
  P.n_steps = c->hdr.n_dates - j.m_start;
  P.starts = j.starts;
  P.start_stride = j.start_stride;
  P.keys = j.keys;
  P.streams = j.streams;
  P.seed = j.seed;
  P.phase = j.phase;
  P.key_date = j.key_date;
  P.item_base = j.item_base;
  P.draw_base = j.draw_base;
  P.normals = c->normals;
  P.nrm_base = c->nrm_base;
  P.nrm_count = c->nrm_count;
  P.path_out = j.path_out;
  P.stop_out = j.stop_out;
  P.steps = step_counter(PK_WALK);
  // the CMC instance assumes even draw indices at every step for even d (parity mode)
  const bool even_ok = c->fast() || c->hdr.d % 2 == 1 || (P.draw_base % 2 == 0);
  void *kwalk = c->kern.walk;
  P.vals_offset = smem_model(c);
  if (c->hdr.rule == BRM_RULE_CMC && !P.normals && even_ok) {
    // parity mode walks log-prices (brm_walk_log.cuh); BRM_WALK_LOG=0 keeps the price stepper (A/B runs)
    static const bool log_walk = !(std::getenv("BRM_WALK_LOG") && std::getenv("BRM_WALK_LOG")[0] == '0');
    // BRM_WALK_COLCONST=0 keeps the triangular product for a column-constant factor (A/B runs)
    static const bool no_colconst = std::getenv("BRM_WALK_COLCONST") && std::getenv("BRM_WALK_COLCONST")[0] == '0';
    const bool maxcall_unit = c->hdr.unit_diag && c->hdr.payoff == BRM_PAY_MAXCALL;
    if (maxcall_unit && !c->fast() && log_walk && c->kern.walk_cmc_log && c->hdr.n_dates <= 255) {
      kwalk = c->kern.walk_cmc_log;
      P.vals_offset = log_model_smem_bytes(c->hdr);  // search trees instead of the bucket tables
    } else if (maxcall_unit && c->kern.walk_cmc_unit) {
      kwalk = c->kern.walk_cmc_unit;
    } else if (c->fast() && c->hdr.chol_lower == 1 && c->hdr.chol_colconst && c->kern.walk_cmc_colconst &&
               !no_colconst) {
      kwalk = c->kern.walk_cmc_colconst;
    } else if (c->fast() && c->hdr.chol_lower == 1 && c->kern.walk_cmc_lower) {
      kwalk = c->kern.walk_cmc_lower;
    } else if (c->kern.walk_cmc) {
      kwalk = c->kern.walk_cmc;
    }
  }
  const int smem = P.vals_offset + 8 * P.chunk;
  if (smem > c->info.max_smem) return fail(BRM_EINVAL, "model image too large for shared memory (%d B)", smem);
  BRM_TRY(call.scratch<double>(2 * (size_t)P.n_items, &P.partials));
  BRM_TRY(call.scratch<int>(1, &P.next_item));
  BRM_CUDA(cudaMemsetAsync(P.next_item, 0, sizeof(int), call.stream));
  BRM_TRY(allow_smem(kwalk, smem));
  int per_sm = 0;
  BRM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kwalk, kWalkThreads, smem));
  if (per_sm < 1) return fail(BRM_EINVAL, "walker does not fit on an SM (smem %d B)", smem);
  const int grid = std::min(P.n_items, per_sm * c->info.sms);
  void *args[] = {&P};
  {
    const int tok_ = prof_begin(PK_WALK, call.stream);
    BRM_CUDA(cudaLaunchKernel(kwalk, dim3(grid), dim3(kWalkThreads), args, smem, call.stream));
    prof_end(tok_, call.stream);
  }
  FinishParams F{};
  F.partials = P.partials;
  F.n_units = j.n_units;
  F.chunks_per_unit = P.chunks_per_unit;
  F.per_unit = j.per_unit;
  F.mode = j.finish_mode;
  F.total_paths = j.total_paths;
  F.points = j.points;
  F.points_stride = j.start_stride;
  F.d = c->hdr.d;
  F.payoff = c->hdr.payoff;
  F.strike = c->hdr.strike;
  F.out = j.out;
  if (F.out) {
    void *fargs[] = {&F};
    {
    const int tok_ = prof_begin(PK_FINISH, call.stream);
    BRM_CUDA(cudaLaunchKernel(finish_kernel(), dim3((j.n_units + 127) / 128), dim3(128), fargs, 0, call.stream));
    prof_end(tok_, call.stream);
  }
  }
  return BRM_OK;
}

}  // namespace

extern "C" {

int brm_abi_version(void) { return BRM_ABI_VERSION; }

const char *brm_last_error(void) { return g_err.c_str(); }

int brm_device_count(int32_t *count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *count = 0;
    return fail(BRM_ENODEV, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  }
  *count = n;
  return BRM_OK;
}

}  // extern "C"

namespace {

// capacity > 0: a CMC image with a fixed slot of `capacity` stumps (and the
// matching step-table space) per date, every date empty; brm_ctx_set_ensemble
// then fills dates on the device.  capacity == 0: the image of `rl`.
int ctx_create_impl(const brm_market_desc *mk, const brm_rule_desc *rl, int32_t device, int32_t mode,
                    int32_t capacity, brm_ctx **out) {
  if (!mk || !rl || !out) return fail(BRM_EINVAL, "NULL argument");
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(BRM_ENODEV, "no CUDA device available");
  }
  if (device < 0 || device >= ndev) return fail(BRM_EINVAL, "device %d out of range (%d devices)", device, ndev);
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  if (major != 10) return fail(BRM_ENODEV, "device %d is sm_%d0, this build targets sm_100a", device, major);
  const int d = mk->d, nd = mk->n_dates;
  if (d < 1 || d > kMaxD) return fail(BRM_EINVAL, "d=%d outside 1..%d", d, kMaxD);
  if (nd < 1) return fail(BRM_EINVAL, "need at least one exercise date");
  if (mk->payoff_kind < 0 || mk->payoff_kind > 4) return fail(BRM_EINVAL, "unknown payoff kind %d", mk->payoff_kind);
  if ((mk->payoff_kind == BRM_PAY_PUT || mk->payoff_kind == BRM_PAY_CALL) && d != 1)
    return fail(BRM_EINVAL, "1-D payoff requires d=1, got d=%d", d);
  if (rl->kind < 0 || rl->kind > 3) return fail(BRM_EINVAL, "unknown rule kind %d", rl->kind);
  if (mode != BRM_MODE_PARITY && mode != BRM_MODE_FAST) return fail(BRM_EINVAL, "unknown mode %d", mode);

  DeviceScope scope(device);
  std::vector<double> mu, vol, chol, disc, s0, izc, izlo, izhi, icept, thr, pol, alpha;
  std::vector<int32_t> starts, counts, feat;
  BRM_TRY(fetch(mk->step_mu, d, mu, "step_mu"));
  BRM_TRY(fetch(mk->step_vol, d, vol, "step_vol"));
  BRM_TRY(fetch(mk->chol, (size_t)d * d, chol, "chol"));
  BRM_TRY(fetch(mk->disc_steps, nd + 1, disc, "disc_steps"));
  BRM_TRY(fetch(mk->s0, d, s0, "s0"));
  const int k = std::max(d - 1, 0);
  int nbasis = 1;
  if (rl->kind == BRM_RULE_IZ) {
    nbasis = rl->nbasis;
    if (nbasis != quad_basis_size(k)) return fail(BRM_EINVAL, "nbasis %d != %d for d=%d", nbasis, quad_basis_size(k), d);
    if (rl->iz_space == 1 && d < 2) return fail(BRM_EINVAL, "log-space surfaces need d>1");
    BRM_TRY(fetch(rl->iz_coeffs, (size_t)(nd + 1) * d * nbasis, izc, "iz_coeffs"));
    if (d > 1) {
      BRM_TRY(fetch(rl->iz_lo, k, izlo, "iz_lo"));
      BRM_TRY(fetch(rl->iz_hi, k, izhi, "iz_hi"));
    }
  }
  const int ns = rl->kind == BRM_RULE_CMC ? rl->n_stumps : 0;
  if (ns < 0) return fail(BRM_EINVAL, "negative stump count");
  if (rl->kind == BRM_RULE_CMC) {
    BRM_TRY(fetch(rl->cmc_starts, nd + 1, starts, "cmc_starts"));
    BRM_TRY(fetch(rl->cmc_counts, nd + 1, counts, "cmc_counts"));
    BRM_TRY(fetch(rl->cmc_intercept, nd + 1, icept, "cmc_intercept"));
    BRM_TRY(fetch(rl->cmc_feat, ns, feat, "cmc_feat"));
    BRM_TRY(fetch(rl->cmc_thr, ns, thr, "cmc_thr"));
    BRM_TRY(fetch(rl->cmc_pol, ns, pol, "cmc_pol"));
    BRM_TRY(fetch(rl->cmc_alpha, ns, alpha, "cmc_alpha"));
    const int nfeat = d > 1 ? d + 1 : 1;
    for (int m = 0; m <= nd; ++m)
      if (counts[m] < 0 || starts[m] < 0 || (counts[m] > 0 && starts[m] + counts[m] > ns))
        return fail(BRM_EINVAL, "stump range of date %d outside the stump arrays", m);
    for (int t = 0; t < ns; ++t)
      if (feat[t] < 0 || feat[t] >= nfeat) return fail(BRM_EINVAL, "stump %d feature %d outside 0..%d", t, feat[t], nfeat - 1);
  }

  ModelHdr h{};
  h.d = d;
  h.n_dates = nd;
  h.payoff = mk->payoff_kind;
  h.rule = rl->kind;
  h.call_like = rl->call_like ? 1 : 0;
  h.imm_date = rl->imm_date;
  h.nbasis = nbasis;
  h.iz_space = rl->kind == BRM_RULE_IZ ? rl->iz_space : 0;
  h.n_stumps = ns;
  h.strike = mk->strike;
  int lower = 1;
  for (int i = 0; i < d; ++i)
    for (int a = i + 1; a < d; ++a)
      if (chol[i * d + a] != 0.0) lower = 0;
  int diag = 1;
  for (int i = 0; i < d; ++i)
    for (int a = 0; a < d; ++a)
      if (a != i && chol[i * d + a] != 0.0) diag = 0;
  h.chol_lower = diag ? 2 : lower;
  h.unit_diag = diag;
  for (int i = 0; i < d; ++i)
    if (chol[i * d + i] != 1.0) h.unit_diag = 0;
  // column-constant below the diagonal in the fp32 image the fast walkers read
  // (the factor of an equicorrelated matrix): fast_step_colconst's prefix form
  h.chol_colconst = (lower && !diag && d > 2) ? 1 : 0;
  for (int a = 0; a + 2 < d && h.chol_colconst; ++a)
    for (int i = a + 2; i < d; ++i)
      if ((float)chol[i * d + a] != (float)chol[(a + 1) * d + a]) h.chol_colconst = 0;
  std::vector<double> dbl;
  auto put = [&](const std::vector<double> &v, size_t min_len) {
    int off = (int)dbl.size();
    dbl.insert(dbl.end(), v.begin(), v.end());
    if (v.size() < min_len) dbl.insert(dbl.end(), min_len - v.size(), 0.0);
    return off;
  };
  h.o_mu = put(mu, d);
  h.o_vol = put(vol, d);
  h.o_chol = put(chol, (size_t)d * d);
  h.o_disc = put(disc, nd + 1);
  h.o_s0 = put(s0, d);
  h.o_izc = put(izc, 1);
  h.o_izlo = put(izlo, std::max(k, 1));
  h.o_izhi = put(izhi, std::max(k, 1));
  if (icept.empty()) icept.assign(nd + 1, -1.0);
  h.o_icept = put(icept, nd + 1);
  std::vector<double> ap(ns);
  for (int t = 0; t < ns; ++t) ap[t] = alpha[t] * pol[t];  // the product the reference forms per vote
  // per (date, feature) step tables of the stump score (see cmc_stop in brm_model.cuh)
  const int nfeat = d > 1 ? d + 1 : 1;
  h.nfeat = nfeat;
  std::vector<double> tt, tv, bound(nd + 1, 0.0);
  std::vector<int32_t> toff((size_t)(nd + 1) * nfeat, 0), tcnt((size_t)(nd + 1) * nfeat, 0),
      voff((size_t)(nd + 1) * nfeat, 0);
  const SlotDims slot = slot_dims(capacity, nfeat);
  if (capacity > 0) {
    // slotted image: date m owns stumps [m R, m R + R), thresholds
    // [m TS, m TS + TS) and table values [m VS, m VS + VS); empty dates have
    // one zero-valued table entry per feature and the intercept -1
    const size_t R = (size_t)capacity;
    thr.assign((nd + 1) * R, 0.0);
    ap.assign((nd + 1) * R, 0.0);
    feat.assign((nd + 1) * R, 0);
    starts.assign(nd + 1, 0);
    counts.assign(nd + 1, 0);
    icept.assign(nd + 1, -1.0);
    for (int m = 0; m <= nd; ++m) starts[m] = (int32_t)(m * R);
    tt.assign((size_t)(nd + 1) * slot.ts, std::numeric_limits<double>::infinity());
    tv.assign((size_t)(nd + 1) * slot.vs, 0.0);
    for (int m = 0; m <= nd; ++m) {
      for (int f = 0; f < nfeat; ++f) {
        toff[(size_t)m * nfeat + f] = m * slot.ts;
        tcnt[(size_t)m * nfeat + f] = 1;
        voff[(size_t)m * nfeat + f] = m * slot.vs + f;
      }
      bound[m] = 4.0 * (double)(nfeat + 4) * std::ldexp(1.0, -53) + 1e-300;
    }
  }
  for (int m = 0; m <= nd && capacity == 0; ++m) {
    const int t0 = rl->kind == BRM_RULE_CMC ? starts[m] : 0, cnt = rl->kind == BRM_RULE_CMC ? counts[m] : 0;
    double absum = rl->kind == BRM_RULE_CMC ? std::fabs(icept[m]) : 0.0;
    for (int f = 0; f < nfeat; ++f) {
      std::vector<double> u;
      for (int t = t0; t < t0 + cnt; ++t)
        if (feat[t] == f) u.push_back(thr[t]);
      std::sort(u.begin(), u.end());
      u.erase(std::unique(u.begin(), u.end()), u.end());
      const size_t idx = (size_t)m * nfeat + f;
      // padded to P-1 entries (P = power of two > count) for a fixed-trip search
      int P = 1;
      while (P < (int)u.size() + 1) P <<= 1;
      toff[idx] = (int32_t)tt.size();
      tcnt[idx] = (int32_t)P;
      voff[idx] = (int32_t)tv.size();
      tt.insert(tt.end(), u.begin(), u.end());
      tt.insert(tt.end(), (size_t)(P - 1) - u.size(), std::numeric_limits<double>::infinity());
      // T[c] = votes when exactly c thresholds of f lie below x:
      //      = -sum(ap) + 2 * sum(ap of stumps with rank < c)   (long double, O(stumps))
      std::vector<long double> by_rank(u.size(), 0.0L);
      long double neg = 0.0L;
      for (int t = t0; t < t0 + cnt; ++t) {
        if (feat[t] != f) continue;
        by_rank[std::lower_bound(u.begin(), u.end(), thr[t]) - u.begin()] += (long double)ap[t];
        neg -= (long double)ap[t];
      }
      long double acc = neg;
      tv.push_back((double)acc);
      for (size_t r = 0; r < u.size(); ++r) {
        acc += 2.0L * by_rank[r];
        tv.push_back((double)acc);
      }
    }
    for (int t = t0; t < t0 + cnt; ++t) absum += std::fabs(ap[t]);
    bound[m] = 4.0 * (double)(cnt + nfeat + 4) * std::ldexp(absum, -53) + 1e-300;
  }
  h.o_bound = put(bound, nd + 1);
  // cold region (kernels read it from global memory): the stumps in stump
  // order for the exact fallback, and the step tables the CTAs index at start
  h.n_hot = (int)dbl.size();
  h.o_thr = put(thr, 1);
  h.o_ap = put(ap, 1);
  h.o_tt = put(tt, 1);
  h.o_tv = put(tv, 1);
  h.n_dbl = (int)dbl.size();
  // compact (threshold, table value) entries: u_f + 2 per (date, feature)
  h.n_tab = rl->kind == BRM_RULE_CMC ? (capacity > 0 ? (nd + 1) * capacity : ns) + 2 * (nd + 1) * nfeat + 3 : 0;
  std::vector<int32_t> ints;
  auto puti = [&](const std::vector<int32_t> &v, size_t min_len) {
    int off = (int)ints.size();
    ints.insert(ints.end(), v.begin(), v.end());
    if (v.size() < min_len) ints.insert(ints.end(), min_len - v.size(), 0);
    return off;
  };
  h.o_starts = puti(starts, nd + 1);
  h.o_counts = puti(counts, nd + 1);
  h.n_int_hot = (int)ints.size();  // feat and the table offsets stay in global memory
  h.o_feat = puti(feat, 1);
  h.o_toff = puti(toff, 1);
  h.o_tcnt = puti(tcnt, 1);
  h.o_voff = puti(voff, 1);
  h.n_int = (int)ints.size();

  brm_ctx *c = new brm_ctx();
  c->device = device;
  c->mode = mode;
  c->hdr = h;
  c->info = device_info(device);
  c->kern = kernels_for(d, mode == BRM_MODE_FAST);
  c->blob_bytes = 8 * dbl.size() + 4 * ints.size();
  count_transfer(c->blob_bytes, 0);
  // one non-blocking stream per device shared by its contexts; the image is a
  // stream-ordered allocation, so creating and dropping contexts never syncs the device
  c->own_stream = device_stream(device);
  cudaError_t e = c->own_stream ? cudaSuccess : cudaErrorUnknown;
  if (e == cudaSuccess) e = cudaMallocAsync(&c->blob, c->blob_bytes, c->own_stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(c->blob, dbl.data(), 8 * dbl.size(), cudaMemcpyHostToDevice, c->own_stream);
  if (e == cudaSuccess && !ints.empty())
    e = cudaMemcpyAsync(c->blob + 8 * dbl.size(), ints.data(), 4 * ints.size(), cudaMemcpyHostToDevice,
                        c->own_stream);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ready, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(c->ready, c->own_stream);
  if (e != cudaSuccess) {
    brm_ctx_destroy(c);
    return fail(e == cudaErrorMemoryAllocation ? BRM_ENOMEM : BRM_ECUDA, "context upload: %s", cudaGetErrorString(e));
  }
  if (h.n_tab > 65535) {
    brm_ctx_destroy(c);
    return fail(BRM_EINVAL, "too many stumps (%d step-table entries, at most 65535)", h.n_tab);
  }
  if (smem_model(c) + 8 * 64 > c->info.max_smem) {
    brm_ctx_destroy(c);
    return fail(BRM_EINVAL, "model image (%d B) exceeds shared memory", smem_model(c));
  }
  c->capacity = capacity;
  c->slot = slot;
  *out = c;
  return BRM_OK;
}

}  // namespace

extern "C" {

int brm_ctx_create(const brm_market_desc *mk, const brm_rule_desc *rl, int32_t device, int32_t mode,
                   brm_ctx **out) {
  return ctx_create_impl(mk, rl, device, mode, 0, out);
}

int brm_ctx_create_cmc(const brm_market_desc *mk, int32_t call_like, int32_t capacity, int32_t device, int32_t mode,
                       brm_ctx **out) {
  if (capacity < 1 || capacity > kMaxSlotStumps)
    return fail(BRM_EINVAL, "stump capacity %d outside 1..%d", capacity, kMaxSlotStumps);
  brm_rule_desc rl{};
  rl.kind = BRM_RULE_CMC;
  rl.call_like = call_like ? 1 : 0;
  rl.imm_date = -1;
  rl.nbasis = 1;
  rl.n_stumps = 0;
  // an empty rule: every date without an ensemble (starts / counts / intercepts
  // are rebuilt in slotted form, so these only have to pass validation)
  const int nd = mk ? mk->n_dates : 0;
  std::vector<int32_t> zeros(std::max(nd + 1, 1), 0);
  std::vector<double> icept(std::max(nd + 1, 1), -1.0);
  rl.cmc_starts = zeros.data();
  rl.cmc_counts = zeros.data();
  rl.cmc_intercept = icept.data();
  return ctx_create_impl(mk, &rl, device, mode, capacity, out);
}

int brm_ctx_set_ensemble(brm_ctx *c, int32_t date, const int32_t *feat, const double *thr, const double *pol,
                         const double *alpha, const int32_t *count, const double *intercept) {
  if (!c) return fail(BRM_EINVAL, "NULL context");
  if (c->capacity <= 0) return fail(BRM_EINVAL, "context was not created by brm_ctx_create_cmc");
  if (date < 1 || date >= c->hdr.n_dates)
    return fail(BRM_EINVAL, "ensemble date %d outside 1..%d", date, c->hdr.n_dates - 1);
  if (!feat || !thr || !pol || !alpha || !count || !intercept) return fail(BRM_EINVAL, "NULL argument");
  DeviceScope scope(c->device);
  const cudaStream_t s = c->stream();
  BRM_CUDA(cudaStreamWaitEvent(s, c->ready, 0));
  const int R = c->capacity;
  Call call(s);
  const int32_t *d_feat, *d_count;
  const double *d_thr, *d_pol, *d_alpha, *d_icept;
  BRM_TRY(call.in(feat, R, &d_feat));
  BRM_TRY(call.in(thr, R, &d_thr));
  BRM_TRY(call.in(pol, R, &d_pol));
  BRM_TRY(call.in(alpha, R, &d_alpha));
  BRM_TRY(call.in(count, 1, &d_count));
  BRM_TRY(call.in(intercept, 1, &d_icept));
  const int tok = prof_begin(PK_AUX, s);
  void *args[] = {(void *)&c->blob, (void *)&c->hdr, (void *)&date, (void *)&R, (void *)&c->slot,
                  (void *)&d_feat, (void *)&d_thr, (void *)&d_pol, (void *)&d_alpha, (void *)&d_count,
                  (void *)&d_icept};
  BRM_TRY(allow_smem(set_ensemble_kernel(), (int)set_ensemble_smem(R)));
  BRM_CUDA(cudaLaunchKernel(set_ensemble_kernel(), dim3(1), dim3(256), args, set_ensemble_smem(R), s));
  prof_end(tok, s);
  BRM_CUDA(cudaEventRecord(c->ready, s));  // later launches on any stream see the new date
  return call.finish();
}

namespace {
// Order the context's own stream after everything already enqueued on the
// stream it launched on last, so frees on the own stream never overtake a
// launch that reads the image.  A caller stream that no longer exists cannot
// take the event record: then wait for the whole device instead.
void retire_user_stream(brm_ctx *c) {
  if (!c->has_user_stream || c->user_stream == c->own_stream) return;
  if (!c->retired && cudaEventCreateWithFlags(&c->retired, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    cudaDeviceSynchronize();
    return;
  }
  if (cudaEventRecord(c->retired, c->user_stream) != cudaSuccess ||
      cudaStreamWaitEvent(c->own_stream, c->retired, 0) != cudaSuccess) {
    cudaGetLastError();
    cudaDeviceSynchronize();
  }
}
}  // namespace

int brm_iz_fit(brm_ctx *c, int32_t m, const double *design, int32_t J, int32_t nb, int32_t k_coords,
               const double *levels, int32_t n_fits, int32_t log_space, double *out_coeffs, int32_t *out_rank) {
  if (!c || !design || !levels) return fail(BRM_EINVAL, "NULL argument");
  if (c->hdr.rule != BRM_RULE_IZ) return fail(BRM_EINVAL, "context does not hold an I&Z boundary");
  if (m < 1 || m >= c->hdr.n_dates) return fail(BRM_EINVAL, "boundary date %d outside 1..%d", m, c->hdr.n_dates - 1);
  if (nb != c->hdr.nbasis) return fail(BRM_EINVAL, "basis size %d != the image's %d", nb, c->hdr.nbasis);
  if (k_coords < 0 || nb != quad_basis_size(k_coords) || nb > kLsMaxB)
    return fail(BRM_EINVAL, "basis size %d is not the quadratic basis of %d coordinates", nb, k_coords);
  if (J < nb) return fail(BRM_EINVAL, "need at least %d probe points for the quadratic fit, got %d", nb, J);
  if (J > kLsMaxN) return fail(BRM_EINVAL, "too many probe points for the device fit");
  const int d = c->hdr.d;
  const bool log_surface = c->hdr.iz_space == 1;
  if (log_surface ? n_fits != 1 : n_fits != d)
    return fail(BRM_EINVAL, "%d fits for a %s surface of d=%d", n_fits, log_surface ? "log-space" : "price", d);
  if (ls_fit_smem(J, nb) > (size_t)c->info.max_smem) return fail(BRM_EINVAL, "design too large for the device fit");
  DeviceScope scope(c->device);
  Call call(c->stream());
  BRM_CUDA(cudaStreamWaitEvent(call.stream, c->ready, 0));
  LsParams P{};
  BRM_TRY(call.in(design, (size_t)J * nb, &P.design));
  BRM_TRY(call.in(levels, (size_t)J * n_fits, &P.levels));
  BRM_TRY(call.out(out_coeffs, (size_t)n_fits * nb, &P.out));
  BRM_TRY(call.out(out_rank, (size_t)n_fits, &P.rank_out));
  P.J = J;
  P.nb = nb;
  P.k = k_coords;
  P.log_space = log_space ? 1 : 0;
  // the date's surface rows in the image: asset g's row, or (log space) every row
  P.dst = reinterpret_cast<double *>(c->blob) + c->hdr.o_izc + (size_t)m * d * nb;
  P.dst_fit_stride = nb;
  P.dst_rows = log_surface ? d : 1;
  BRM_TRY(launch_ls_fit(P, n_fits, call.stream));
  BRM_CUDA(cudaEventRecord(c->ready, call.stream));  // later launches on any stream see the new surface
  return call.finish();
}

int brm_ctx_destroy(brm_ctx *c) {
  if (!c) return BRM_OK;
  DeviceScope scope(c->device);
  // freed in stream order on the context's own (per-device, library-owned)
  // stream, after every launch that used the image on it or on the caller's
  // last stream
  retire_user_stream(c);
  const cudaStream_t s = c->own_stream;
  if (c->blob) cudaFreeAsync(c->blob, s);
  if (c->normals) cudaFreeAsync(c->normals, s);
  if (c->ready) cudaEventDestroy(c->ready);
  if (c->retired) cudaEventDestroy(c->retired);
  if (c->side_stream) fit_presort_drop(c, c->side_stream);
  if (c->side_event) cudaEventDestroy(c->side_event);
  if (c->side_mid) cudaEventDestroy(c->side_mid);
  if (c->side_stream) cudaStreamDestroy(c->side_stream);  // (its work completes first)
  cudaGetLastError();
  delete c;
  return BRM_OK;
}

int brm_ctx_set_stream(brm_ctx *c, void *s) {
  if (!c) return fail(BRM_EINVAL, "NULL context");
  DeviceScope scope(c->device);
  const cudaStream_t next = s ? static_cast<cudaStream_t>(s) : c->own_stream;
  if (next != c->stream()) {
    // work already enqueued on the previous stream is ordered before later
    // launches on the new one, and before the image is freed
    if (c->has_user_stream) retire_user_stream(c);
    if (next != c->own_stream) {
      if (!c->retired) BRM_CUDA(cudaEventCreateWithFlags(&c->retired, cudaEventDisableTiming));
      BRM_CUDA(cudaEventRecord(c->retired, c->own_stream));
      BRM_CUDA(cudaStreamWaitEvent(next, c->retired, 0));
    }
  }
  c->user_stream = static_cast<cudaStream_t>(s);
  c->has_user_stream = s != nullptr;
  return BRM_OK;
}

int brm_ctx_supply_normals(brm_ctx *c, const double *normals, uint64_t base, uint64_t count) {
  if (!c) return fail(BRM_EINVAL, "NULL context");
  DeviceScope scope(c->device);
  if (c->normals) cudaFreeAsync(c->normals, c->stream());
  c->normals = nullptr;
  c->nrm_base = c->nrm_count = 0;
  if (!normals || count == 0) return BRM_OK;
  BRM_CUDA(cudaMallocAsync(&c->normals, count * sizeof(double), c->stream()));
  BRM_CUDA(cudaMemcpyAsync(c->normals, normals, count * sizeof(double), cudaMemcpyDefault, c->stream()));
  BRM_CUDA(cudaStreamSynchronize(c->stream()));
  c->nrm_base = base;
  c->nrm_count = count;
  return BRM_OK;
}

int brm_derive_words(uint64_t seed, uint32_t phase, uint64_t item, uint64_t date, uint64_t *key64,
                     uint64_t *stream64) {
  if (!key64 || !stream64) return fail(BRM_EINVAL, "NULL output");
  derive_words(seed, phase, item, date, *key64, *stream64);
  return BRM_OK;
}

int brm_raw_uint64(int32_t device, uint64_t key64, uint64_t stream64, uint64_t start, int64_t count, uint64_t *out) {
  if (count < 0) return fail(BRM_EINVAL, "negative count");
  if (count == 0) return BRM_OK;
  DeviceScope scope(device);
  Call call(nullptr);
  uint64_t *o;
  BRM_TRY(call.out(out, count, &o));
  const int grid = (int)std::min<int64_t>((count + 255) / 256, 148 * 16);
  void *args[] = {&key64, &stream64, &start, &count, &o};
  {
    const int tok_ = prof_begin(PK_RNG, call.stream);
    BRM_CUDA(cudaLaunchKernel(fill_raw_kernel(), dim3(grid), dim3(256), args, 0, call.stream));
    prof_end(tok_, call.stream);
  }
  BRM_TRY(call.finish());
  BRM_CUDA(cudaStreamSynchronize(call.stream));
  return BRM_OK;
}

int brm_normals(int32_t device, uint64_t key64, uint64_t stream64, uint64_t start, int64_t count, double *out) {
  if (count < 0) return fail(BRM_EINVAL, "negative count");
  if (count == 0) return BRM_OK;
  DeviceScope scope(device);
  Call call(nullptr);
  double *o;
  BRM_TRY(call.out(out, count, &o));
  const int grid = (int)std::min<int64_t>((count + 255) / 256, 148 * 16);
  void *args[] = {&key64, &stream64, &start, &count, &o};
  {
    const int tok_ = prof_begin(PK_RNG, call.stream);
    BRM_CUDA(cudaLaunchKernel(fill_normals_kernel(), dim3(grid), dim3(256), args, 0, call.stream));
    prof_end(tok_, call.stream);
  }
  BRM_TRY(call.finish());
  BRM_CUDA(cudaStreamSynchronize(call.stream));
  return BRM_OK;
}

int brm_selftest_math(int32_t device, int32_t kind, const double *a, const double *b, int64_t n, double *out) {
  if (n <= 0) return BRM_OK;
  if (kind < 0 || kind > 10 || kind == 9) return fail(BRM_EINVAL, "unknown self-test %d", kind);
  if (kind == 10 && n > (1 << 30)) return fail(BRM_EINVAL, "exact-scan self-test too long");
  if (kind >= 8 && n > 2147483647LL) return fail(BRM_EINVAL, "chain self-test too long");
  DeviceScope scope(device);
  Call call(nullptr);
  const double *da, *db = nullptr;
  double *o;
  BRM_TRY(call.in(a, n, &da));
  if (kind == 2 || kind == 3) BRM_TRY(call.in(b, n, &db));
  BRM_TRY(call.out(out, n, &o));
  void *args[] = {&kind, &da, &db, &n, &o};
  if (kind == 10) {
    unsigned *code;
    double *chain;
    BRM_TRY(call.scratch(n, &code));
    BRM_TRY(call.scratch(2 * n, &chain));
    int ni = (int)n;
    void *eargs[] = {&da, &ni, &code, &chain, &o};
    BRM_CUDA(cudaLaunchKernel(exact_scan_selftest_kernel(), dim3(1), dim3(512), eargs, 0, call.stream));
  } else if (kind >= 8) {
    void *cargs[] = {&kind, &da, &n, &o};
    BRM_CUDA(cudaLaunchKernel(chain_selftest_kernel(), dim3(1), dim3(32), cargs, 0, call.stream));
  } else {
    BRM_CUDA(cudaLaunchKernel(math_selftest_kernel(), dim3((unsigned)((n + 255) / 256)), dim3(256), args, 0, call.stream));
  }
  return call.finish();
}

int brm_stopped_sums(brm_ctx *c, const double *start, int32_t m_start, int64_t n_paths, uint64_t key64,
                     uint64_t stream64, uint64_t draw_base, double *sum, double *sumsq) {
  if (!c || !sum || !sumsq) return fail(BRM_EINVAL, "NULL argument");
  BRM_TRY(check_remaining(c, m_start));
  if (n_paths < 0 || n_paths > (int64_t)1 << 30) return fail(BRM_EINVAL, "n_paths %lld out of range", (long long)n_paths);
  DeviceScope scope(c->device);
  Call call(c->stream());
  BRM_CUDA(cudaStreamWaitEvent(call.stream, c->ready, 0));
  const double *st;
  BRM_TRY(call.in(start, c->hdr.d, &st));
  if (!st) return fail(BRM_EINVAL, "start_values is NULL");
  double *res;
  BRM_TRY(call.scratch<double>(2, &res));
  if (n_paths == 0) {
    BRM_CUDA(cudaMemsetAsync(res, 0, 2 * sizeof(double), call.stream));
  } else {
    WalkJob j;
    j.n_units = 1;
    j.per_unit = (int)n_paths;
    j.total_paths = n_paths;
    j.chunk = 256;
    j.m_start = m_start;
    j.starts = st;
    j.key_date = 0;
    uint64_t keys[1] = {key64}, streams[1] = {stream64};
    const uint64_t *dk, *dsr;
    BRM_TRY(call.in(keys, 1, &dk));
    BRM_TRY(call.in(streams, 1, &dsr));
    j.keys = dk;
    j.streams = dsr;
    j.draw_base = draw_base;
    j.finish_mode = 0;
    j.out = res;
    BRM_TRY(run_walk(c, call, j));
  }
  double *o1, *o2;
  BRM_TRY(call.out(sum, 1, &o1));
  BRM_TRY(call.out(sumsq, 1, &o2));
  BRM_CUDA(cudaMemcpyAsync(o1, res, sizeof(double), cudaMemcpyDeviceToDevice, call.stream));
  BRM_CUDA(cudaMemcpyAsync(o2, res + 1, sizeof(double), cudaMemcpyDeviceToDevice, call.stream));
  return call.finish();
}

int brm_path_values(brm_ctx *c, const double *start, int32_t m_start, int64_t n_paths, uint64_t key64,
                    uint64_t stream64, uint64_t draw_base, double *values, int32_t *stop_dates) {
  if (!c) return fail(BRM_EINVAL, "NULL context");
  BRM_TRY(check_remaining(c, m_start));
  if (n_paths < 0 || n_paths > (int64_t)1 << 30) return fail(BRM_EINVAL, "n_paths out of range");
  if (n_paths == 0) return BRM_OK;
  DeviceScope scope(c->device);
  Call call(c->stream());
  BRM_CUDA(cudaStreamWaitEvent(call.stream, c->ready, 0));
  const double *st;
  BRM_TRY(call.in(start, c->hdr.d, &st));
  if (!st) return fail(BRM_EINVAL, "start_values is NULL");
  double *vo;
  int32_t *so;
  BRM_TRY(call.out(values, n_paths, &vo));
  BRM_TRY(call.out(stop_dates, n_paths, &so));
  uint64_t keys[1] = {key64}, streams[1] = {stream64};
  WalkJob j;
  BRM_TRY(call.in(keys, 1, &j.keys));
  BRM_TRY(call.in(streams, 1, &j.streams));
  j.n_units = 1;
  j.per_unit = (int)n_paths;
  j.total_paths = n_paths;
  j.chunk = 256;
  j.m_start = m_start;
  j.starts = st;
  j.draw_base = draw_base;
  j.path_out = vo;
  j.stop_out = so;
  BRM_TRY(run_walk(c, call, j));
  return call.finish();
}

int brm_decisions(brm_ctx *c, const double *states, int64_t n, int32_t m, int32_t *out) {
  if (!c) return fail(BRM_EINVAL, "NULL context");
  if (m < 1 || m > c->hdr.n_dates) return fail(BRM_EINVAL, "date %d outside 1..%d", m, c->hdr.n_dates);
  if (n <= 0) return BRM_OK;
  DeviceScope scope(c->device);
  Call call(c->stream());
  BRM_CUDA(cudaStreamWaitEvent(call.stream, c->ready, 0));
  DecisionParams P{};
  P.hdr = c->hdr;
  P.blob = c->blob;
  P.n = n;
  P.m = m;
  BRM_TRY(call.in(states, (size_t)n * c->hdr.d, &P.states));
  BRM_TRY(call.out(out, n, &P.out));
  const int smem = smem_model(c);
  BRM_TRY(allow_smem(c->kern.dec, smem));
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)c->info.sms * 4);
  void *args[] = {&P};
  {
    const int tok_ = prof_begin(PK_DEC, call.stream);
    BRM_CUDA(cudaLaunchKernel(c->kern.dec, dim3(grid), dim3(256), args, smem, call.stream));
    prof_end(tok_, call.stream);
  }
  return call.finish();
}

int brm_price_blocks(brm_ctx *c, int64_t n_paths, uint64_t seed, int64_t block_lo, int64_t block_hi,
                     double *out_stats) {
  if (!c || !out_stats) return fail(BRM_EINVAL, "NULL argument");
  if (n_paths < 1) return fail(BRM_EINVAL, "need at least one path, got %lld", (long long)n_paths);
  const int64_t n_blocks = (n_paths + kPathBlock - 1) / kPathBlock;
  if (block_lo < 0 || block_hi > n_blocks || block_lo > block_hi)
    return fail(BRM_EINVAL, "block range [%lld, %lld) outside 0..%lld", (long long)block_lo, (long long)block_hi,
                (long long)n_blocks);
  if (block_hi - block_lo > (1 << 24)) return fail(BRM_EINVAL, "too many blocks in one call");
  if (block_hi == block_lo) return BRM_OK;
  DeviceScope scope(c->device);
  Call call(c->stream());
  BRM_CUDA(cudaStreamWaitEvent(call.stream, c->ready, 0));
  double *o;
  BRM_TRY(call.out(out_stats, 3 * (size_t)(block_hi - block_lo), &o));
  WalkJob j;
  j.n_units = (int)(block_hi - block_lo);
  j.per_unit = kPathBlock;
  j.total_paths = n_paths - block_lo * kPathBlock;
  j.chunk = kPriceChunk;
  j.m_start = 0;
  j.starts = nullptr;
  j.seed = seed;
  j.phase = BRM_PHASE_PRICING;
  j.item_base = block_lo;
  j.key_date = 0;
  j.draw_base = 0;
  j.finish_mode = 1;
  j.out = o;
  BRM_TRY(run_walk(c, call, j));
  return call.finish();
}

int brm_cmc_labels(brm_ctx *c, const double *points, int64_t n, int32_t m, int32_t n_label, const uint64_t *keys,
                   const uint64_t *streams, uint64_t seed, int64_t item_lo, uint64_t draw_base, double *out_beta) {
  if (!c || !out_beta) return fail(BRM_EINVAL, "NULL argument");
  BRM_TRY(check_remaining(c, m));
  if (n_label < 1) return fail(BRM_EINVAL, "need at least one labeling path");
  if (n < 0 || n > (1 << 26)) return fail(BRM_EINVAL, "point count out of range");
  if (n == 0) return BRM_OK;
  DeviceScope scope(c->device);
  Call call(c->stream());
  BRM_CUDA(cudaStreamWaitEvent(call.stream, c->ready, 0));
  WalkJob j;
  BRM_TRY(call.in(points, (size_t)n * c->hdr.d, &j.starts));
  if (!j.starts) return fail(BRM_EINVAL, "points is NULL");
  if (keys) {
    BRM_TRY(call.in(keys, n, &j.keys));
    BRM_TRY(call.in(streams, n, &j.streams));
    if (!j.streams) return fail(BRM_EINVAL, "streams is NULL");
  }
  double *o;
  BRM_TRY(call.out(out_beta, n, &o));
  j.n_units = (int)n;
  j.per_unit = n_label;
  j.total_paths = n * (int64_t)n_label;
  j.chunk = std::min(n_label, kMaxChunk);
  j.m_start = m;
  j.start_stride = c->hdr.d;
  j.seed = seed;
  j.phase = BRM_PHASE_CMC_CALC;
  j.item_base = item_lo;
  j.key_date = m;
  j.draw_base = draw_base;
  j.finish_mode = 2;
  j.points = j.starts;
  j.out = o;
  BRM_TRY(run_walk(c, call, j));
  return call.finish();
}

int brm_sample_points(brm_ctx *c, int32_t mode, int32_t m, uint64_t seed, int64_t item_lo, int64_t n,
                      const double *bridge, double *out_points) {
  if (!c || !out_points) return fail(BRM_EINVAL, "NULL argument");
  if (m < 1 || m > c->hdr.n_dates) return fail(BRM_EINVAL, "date index %d outside 1..%d", m, c->hdr.n_dates);
  if (mode != 0 && mode != 1) return fail(BRM_EINVAL, "unknown sampler mode %d", mode);
  if (n <= 0) return BRM_OK;
  DeviceScope scope(c->device);
  Call call(c->stream());
  BRM_CUDA(cudaStreamWaitEvent(call.stream, c->ready, 0));
  SampleParams P{};
  P.mode = mode;
  P.m = m;
  P.d = c->hdr.d;
  P.n_dates = c->hdr.n_dates;
  P.seed = seed;
  P.item_lo = item_lo;
  P.n = n;
  P.s0 = c->blob_dbl(c->hdr.o_s0);
  P.chol = c->blob_dbl(c->hdr.o_chol);
  P.step_mu = c->blob_dbl(c->hdr.o_mu);
  P.step_vol = c->blob_dbl(c->hdr.o_vol);
  P.payoff = c->hdr.payoff;
  P.out_stride = c->hdr.d;
  if (mode == 0) {
    BRM_TRY(call.in(bridge, 4 * (size_t)c->hdr.d + 1, &P.bridge));
    if (!P.bridge) return fail(BRM_EINVAL, "bridge scalars are NULL");
  }
  BRM_TRY(call.out(out_points, (size_t)n * c->hdr.d, &P.out));
  void *args[] = {&P};
  {
    const int tok_ = prof_begin(PK_SAMPLE, call.stream);
    BRM_CUDA(cudaLaunchKernel(sample_kernel(), dim3((unsigned)((n + 127) / 128)), dim3(128), args, 0, call.stream));
    prof_end(tok_, call.stream);
  }
  return call.finish();
}

int brm_ctx_set_presort(brm_ctx *c, int32_t on) {
  if (!c) return fail(BRM_EINVAL, "NULL context");
  c->presort = on != 0;
  return BRM_OK;
}

int brm_cmc_calc(brm_ctx *c, int32_t sampler, int32_t m, uint64_t seed, int64_t item_lo, int64_t n,
                 int32_t n_label, const double *bridge, double *out_features, double *out_beta) {
  if (!c || !out_features || !out_beta) return fail(BRM_EINVAL, "NULL argument");
  BRM_TRY(check_remaining(c, m));
  if (m < 1) return fail(BRM_EINVAL, "date index %d outside 1..%d", m, c->hdr.n_dates);
  if (sampler != 0 && sampler != 1) return fail(BRM_EINVAL, "unknown sampler %d", sampler);
  if (n_label < 1) return fail(BRM_EINVAL, "need at least one labeling path");
  if (n < 0 || n > (1 << 26)) return fail(BRM_EINVAL, "point count out of range");
  if (n == 0) return BRM_OK;
  DeviceScope scope(c->device);
  Call call(c->stream());
  BRM_CUDA(cudaStreamWaitEvent(call.stream, c->ready, 0));
  const int d = c->hdr.d, F = d > 1 ? d + 1 : 1;
  SampleParams S{};
  S.mode = sampler;
  S.m = m;
  S.d = d;
  S.n_dates = c->hdr.n_dates;
  S.payoff = c->hdr.payoff;
  S.out_stride = F;
  S.seed = seed;
  S.item_lo = item_lo;
  S.n = n;
  S.s0 = c->blob_dbl(c->hdr.o_s0);
  S.chol = c->blob_dbl(c->hdr.o_chol);
  S.step_mu = c->blob_dbl(c->hdr.o_mu);
  S.step_vol = c->blob_dbl(c->hdr.o_vol);
  if (sampler == 0) {
    BRM_TRY(call.in(bridge, 4 * (size_t)d + 1, &S.bridge));
    if (!S.bridge) return fail(BRM_EINVAL, "bridge scalars are NULL");
  }
  BRM_TRY(call.out(out_features, (size_t)n * F, &S.out));
  double *o;
  BRM_TRY(call.out(out_beta, n, &o));
  void *sargs[] = {&S};
  {
    const int tok_ = prof_begin(PK_SAMPLE, call.stream);
    BRM_CUDA(cudaLaunchKernel(sample_kernel(), dim3((unsigned)((n + 127) / 128)), dim3(128), sargs, 0, call.stream));
    prof_end(tok_, call.stream);
  }
  if (c->presort && S.out == out_features) {
    // the features are final once the sampler is done: their column sort (AdaBoost's fixed cost)
    // runs on a few SMs beside the label walk instead of after it
    if (!c->side_stream) {
      int lo_p = 0, hi_p = 0;
      BRM_CUDA(cudaDeviceGetStreamPriorityRange(&lo_p, &hi_p));
      BRM_CUDA(cudaStreamCreateWithPriority(&c->side_stream, cudaStreamNonBlocking, hi_p));
      BRM_CUDA(cudaEventCreateWithFlags(&c->side_event, cudaEventDisableTiming));
    }
    BRM_CUDA(cudaEventRecord(c->side_event, call.stream));
    BRM_CUDA(cudaStreamWaitEvent(c->side_stream, c->side_event, 0));
    if (!c->side_mid) BRM_CUDA(cudaEventCreateWithFlags(&c->side_mid, cudaEventDisableTiming));
    BRM_TRY(fit_presort(c->device, c->side_stream, out_features, n, F, c->side_mid, c));
    // the walk starts once the sort is the side stream's next launch: the sort's few CTAs get
    // their SMs before the walker's persistent CTAs fill the device
    BRM_CUDA(cudaStreamWaitEvent(call.stream, c->side_mid, 0));
  }
  WalkJob j;
  j.n_units = (int)n;
  j.per_unit = n_label;
  j.total_paths = n * (int64_t)n_label;
  j.chunk = std::min(n_label, kMaxChunk);
  j.m_start = m;
  j.starts = S.out;
  j.start_stride = F;
  j.seed = seed;
  j.phase = BRM_PHASE_CMC_CALC;
  j.item_base = item_lo;
  j.key_date = m;
  // labels continue the point's stream after the sampler's draws
  j.draw_base = sampler == 0 ? 2 * (uint64_t)d : (uint64_t)m * d;
  j.finish_mode = 2;
  j.points = S.out;
  j.out = o;
  BRM_TRY(run_walk(c, call, j));
  return call.finish();
}

int brm_iz_solve(brm_ctx *c, int32_t solver, const double *seeds, const int32_t *assets, int64_t n, int32_t m,
                 int32_t n_inner, double eps, int32_t max_iter, int32_t avg_window, double lo, double hi, double tol,
                 const uint64_t *keys, const uint64_t *streams, uint64_t seed, int64_t item_lo, double *out_level,
                 int32_t *out_iterations, int32_t *out_converged) {
  if (!c || !out_level || !out_iterations || !out_converged) return fail(BRM_EINVAL, "NULL argument");
  BRM_TRY(check_remaining(c, m));
  if (solver != 0 && solver != 1) return fail(BRM_EINVAL, "unknown solver %d", solver);
  if (n_inner < 1) return fail(BRM_EINVAL, "need at least one inner path, got %d", n_inner);
  if (solver == 0 && !(eps > 0.0)) return fail(BRM_EINVAL, "epsilon must be positive, got %g", eps);
  if (solver == 0 && avg_window < 1) return fail(BRM_EINVAL, "avg_window must be >= 1");
  if (solver == 1 && !(lo < hi && tol > 0.0)) return fail(BRM_EINVAL, "bisection needs lo < hi and tol > 0");
  if (max_iter > 100000) return fail(BRM_EINVAL, "max_iter too large");
  if (n <= 0) return BRM_OK;
  if (n > (1 << 20)) return fail(BRM_EINVAL, "too many probes");
  DeviceScope scope(c->device);
  Call call(c->stream());
  BRM_CUDA(cudaStreamWaitEvent(call.stream, c->ready, 0));
  IzParams P{};
  P.hdr = c->hdr;
  P.blob = c->blob;
  P.n_probes = (int)n;
  P.m = m;
  P.n_steps = c->hdr.n_dates - m;
  P.n_inner = n_inner;
  P.solver = solver;
  P.eps = eps;
  P.max_iter = std::max(max_iter, 0);
  P.avg_window = avg_window;
  P.lo = lo;
  P.hi = hi;
  P.tol = tol;
  P.seed_stride = std::max(c->hdr.d - 1, 0);
  double dummy_seed = 0.0;
  if (P.seed_stride > 0) {
    BRM_TRY(call.in(seeds, (size_t)n * P.seed_stride, &P.seeds));
    if (!P.seeds) return fail(BRM_EINVAL, "seeds are NULL");
  } else {
    BRM_TRY(call.scratch<double>(1, const_cast<double **>(&P.seeds)));
    BRM_CUDA(cudaMemcpyAsync(const_cast<double *>(P.seeds), &dummy_seed, sizeof(double), cudaMemcpyHostToDevice,
                             call.stream));
  }
  BRM_TRY(call.in(assets, n, &P.assets));
  if (keys) {
    BRM_TRY(call.in(keys, n, &P.keys));
    BRM_TRY(call.in(streams, n, &P.streams));
    if (!P.streams) return fail(BRM_EINVAL, "streams is NULL");
  }
  P.seed = seed;
  P.item_base = item_lo;
  P.normals = c->normals;
  P.nrm_base = c->nrm_base;
  P.nrm_count = c->nrm_count;
  BRM_TRY(call.out(out_level, n, &P.out_level));
  BRM_TRY(call.out(out_iterations, n, &P.out_iter));
  BRM_TRY(call.out(out_converged, n, &P.out_conv));
  // cluster size: enough CTAs per probe to give each lane a path or two
  // cluster size: up to 8 CTAs per probe, fewer when the probes would not fit
  // in one wave (2 walker CTAs per SM) or when there are too few inner paths
  int csize = 8;
  while (csize > 1 && (int64_t)csize * kWalkThreads / 2 > n_inner) csize >>= 1;
  while (csize > 1 && n * csize > 2LL * c->info.sms) csize >>= 1;
  const int per_cta = iz_per_cta(n_inner, csize);
  if (per_cta > kIzMaxChunks * kIzFoldChunk)
    return fail(BRM_EINVAL, "%d inner paths per probe CTA exceed %d", per_cta, kIzMaxChunks * kIzFoldChunk);
  P.vals_offset = smem_model(c);
  P.steps = step_counter(PK_IZ);
  P.hist_offset = P.vals_offset + ((8 * per_cta + 15) & ~15);
  const int smem = P.hist_offset + 8 * (P.max_iter + 1);
  if (smem > c->info.max_smem) return fail(BRM_EINVAL, "probe solve needs %d B of shared memory", smem);
  void *kiz = (c->hdr.payoff == BRM_PAY_GEOPUT && !c->fast() && c->kern.iz_geo) ? c->kern.iz_geo : c->kern.iz;
  {
    // parity mode walks log-prices when the rule is the geometric put's log-space surface over
    // independent assets (brm_walk_log.cuh); BRM_WALK_LOG=0 keeps the price stepper (A/B runs)
    static const bool log_walk = !(std::getenv("BRM_WALK_LOG") && std::getenv("BRM_WALK_LOG")[0] == '0');
    if (log_walk && c->hdr.payoff == BRM_PAY_GEOPUT && !c->fast() && c->hdr.rule == BRM_RULE_IZ &&
        c->hdr.iz_space == 1 && c->hdr.unit_diag && !P.normals && c->kern.iz_geo_log)
      kiz = c->kern.iz_geo_log;
  }
  BRM_TRY(allow_smem(kiz, smem));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(n * csize));
  cfg.blockDim = dim3(kWalkThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = call.stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // Bisection tree: when the probes leave the GPU mostly idle (config 1: one
  // probe per date), evaluate the 2^L - 1 midpoints of L bisection levels at
  // once on as many clusters -- the same decisions and bits as L sequential
  // passes (common random numbers), L times fewer passes.
  P.tree_levels = 1;
  P.tree_passes = 0;
  P.tree_cont = nullptr;
  // (BRM_NCU_SAFE: Nsight Compute cannot replay cooperative cluster launches)
  if (solver == 1 && getenv("BRM_IZ_NO_TREE") == nullptr && getenv("BRM_NCU_SAFE") == nullptr) {
    const double span = (hi - lo) / tol;
    int levels = span > 1.0 ? (int)std::ceil(std::log2(span)) + 2 : 2;
    levels = std::min(levels, std::max(max_iter, 1));
    int L = 1;
    while (L < 6 && L < levels && n * (int64_t)((2 << L) - 1) * csize <= 2LL * c->info.sms) ++L;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    for (; L > 1; --L) {
      cfg.gridDim = dim3((unsigned)(n * ((1 << L) - 1) * csize));
      cfg.numAttrs = 2;
      if ((int64_t)max_active_clusters(kiz, cfg, c->device) >= n * ((1 << L) - 1)) break;
    }
    if (L > 1) {
      P.tree_levels = L;
      P.tree_passes = (levels + L - 1) / L;
      BRM_TRY(call.scratch((size_t)2 * n * ((1 << L) - 1), &P.tree_cont));
    } else {
      cfg.gridDim = dim3((unsigned)(n * csize));
      cfg.numAttrs = 1;
    }
  }
  // draw cache of the sequential bisection on the log-price walker: every pass walks the same
  // paths (common random numbers), so the first one records the increments and the rest replay
  // them from HBM (C2: 115 MB per date); BRM_IZ_NO_CACHE=1 re-simulates every pass (A/B runs)
  P.rec = nullptr;
  if (solver == 1 && P.tree_levels == 1 && kiz == c->kern.iz_geo_log && c->kern.iz_geo_log_rec && P.max_iter > 1 &&
      getenv("BRM_IZ_NO_CACHE") == nullptr) {
    const size_t cells = (size_t)n * P.n_steps * n_inner * 3;
    // a replay pass keeps the values of kIzReplayCand candidate levels per path in shared memory
    const int hist_rec = P.vals_offset + ((8 * kIzReplayCand * per_cta + 15) & ~15);
    const int smem_rec = hist_rec + 8 * (P.max_iter + 1);
    if (cells <= ((size_t)1 << 28) && smem_rec <= 88 * 1024) {  // <= 2 GB; two CTAs per SM with the static arrays
      if (call.scratch<double>(cells, &P.rec) == BRM_OK && P.rec) {
        kiz = c->kern.iz_geo_log_rec;  // same launch shape
        P.hist_offset = hist_rec;
        cfg.dynamicSmemBytes = smem_rec;
        BRM_TRY(allow_smem(kiz, smem_rec));
      } else {  // no room for the cache: every pass re-simulates
        P.rec = nullptr;
        cudaGetLastError();
      }
    }
  }
  void *args[] = {&P};
  {
    const int tok_ = prof_begin(PK_IZ, call.stream);
    BRM_CUDA(cudaLaunchKernelExC(&cfg, kiz, args));
    prof_end(tok_, call.stream);
  }
  return call.finish();
}

}  // extern "C"
