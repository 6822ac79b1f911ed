// brm_internal.h -- kernel parameter blocks shared by the kernels and the C ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "brm_model.cuh"

#include <algorithm>

namespace brm {

constexpr int kWalkThreads = 256;   // threads per walker CTA
constexpr int kPathBlock = 4096;    // pricer.py:32 PATH_BLOCK (stream convention)
constexpr int kPriceChunk = 2048;   // paths per pricing work item (2 per block: 8 paths per lane before the drain)
constexpr int kMaxChunk = 2048;     // largest chunk a walker CTA folds in smem
constexpr int kIzFoldChunk = 256;   // I&Z probes: paths per fixed-order fold chunk
constexpr int kIzMaxChunks = 64;    // fold chunks per probe CTA (16384 inner paths)
constexpr int kIzReplayLevels = 3;  // bisection levels a replay pass of the draw cache decides ...
constexpr int kIzReplayCand = (1 << kIzReplayLevels) - 1;  // ... from that many candidate levels

// Inner paths per CTA of an I&Z probe cluster: whole fold chunks, so the
// chunk boundaries (and the summation order) do not depend on the cluster size.
__host__ __device__ inline int iz_per_cta(int n_inner, int csize) {
  const int per = (n_inner + csize - 1) / csize;
  return (per + kIzFoldChunk - 1) / kIzFoldChunk * kIzFoldChunk;
}

struct WalkParams {
  ModelHdr hdr;
  const unsigned char *blob;
  int n_units, per_unit, chunk, chunks_per_unit, n_items;
  int64_t total_paths;
  int m_start, n_steps;
  const double *starts;  // [u * start_stride + i]; nullptr -> s0
  int start_stride;
  const uint64_t *keys, *streams;  // nullptr -> derive(seed, phase, item_base + u, key_date)
  uint64_t seed;
  int phase, key_date;
  int64_t item_base;
  uint64_t draw_base;
  const double *normals;
  uint64_t nrm_base, nrm_count;
  int vals_offset;  // byte offset of the per-path value buffer in dynamic smem
  double *partials;  // [n_items][2]
  unsigned long long *steps;  // executed path-steps counter (may be null)
  double *path_out;  // optional [n_units * per_unit]
  int32_t *stop_out;
  int *next_item;    // zeroed counter of claimed work items beyond the grid's first wave (null: static stride)
};

struct FinishParams {
  const double *partials;
  int n_units, chunks_per_unit, per_unit, mode;
  int64_t total_paths;
  const double *points;  // mode 2
  int points_stride;
  int d, payoff;
  double strike;
  double *out;
};

struct IzParams {
  ModelHdr hdr;
  const unsigned char *blob;
  int n_probes, m, n_steps, n_inner;
  int solver;
  double eps;
  int max_iter, avg_window;
  double lo, hi, tol;
  const double *seeds;
  int seed_stride;
  const int32_t *assets;
  const uint64_t *keys, *streams;
  uint64_t seed;
  int64_t item_base;
  const double *normals;
  uint64_t nrm_base, nrm_count;
  int vals_offset, hist_offset;
  unsigned long long *steps;
  double *out_level;
  int32_t *out_iter, *out_conv;
  // bisection tree (solver 1): tree_levels > 1 evaluates 2^L - 1 midpoints
  // per pass on as many clusters (cooperative launch), tree_passes passes
  int tree_levels, tree_passes;
  double *tree_cont;  // [2][n_probes][2^L - 1] node continuation values
  // bisection draw cache (log-price probe walker of the geometric put,
  // sequential bisection): the first pass records every path,
  // [n_probes][n_steps][n_inner][3] (brm_walk_log.cuh); the later passes replay
  double *rec;
};

struct DecisionParams {
  ModelHdr hdr;
  const unsigned char *blob;
  const double *states;
  int64_t n;
  int m;
  int32_t *out;
};

struct SampleParams {
  int mode, m, d, n_dates, payoff;
  int out_stride;  // d, or d+1 with the derived classifier feature in column d
  uint64_t seed;
  int64_t item_lo, n;
  const double *s0, *chol, *step_mu, *step_vol, *bridge;
  double *out;
};

struct KernelTriple {
  void *walk, *iz, *dec;
  void *iz_geo = nullptr;   // parity I&Z probes specialised for the geometric put (d > 1)
  void *walk_cmc = nullptr;       // walker specialised for CMC rules (d > 1)
  void *walk_cmc_unit = nullptr;  // ... max-call payoff, independent assets (unit diagonal factor)
  void *walk_cmc_lower = nullptr; // ... fast mode, lower-triangular factor
  void *walk_cmc_log = nullptr;   // ... walk_cmc_unit's case in parity mode on log-prices (brm_walk_log.cuh)
  void *iz_geo_log = nullptr;     // iz_geo on log-prices (log-space surface, independent assets; brm_walk_log.cuh)
  void *iz_geo_log_rec = nullptr; // ... with the bisection draw cache (first pass records, the others replay)
  void *walk_cmc_colconst = nullptr;  // walk_cmc_lower with a column-constant factor (equicorrelated assets)
};

// Kernel families for launch accounting (brm_prof.cu, BRM_PROF_* in the C ABI).
enum ProfKind { PK_WALK = 0, PK_IZ = 1, PK_BOOST = 2, PK_SAMPLE = 3, PK_FINISH = 4, PK_LSTSQ = 5, PK_RNG = 6,
                PK_DEC = 7, PK_AUX = 8, kProfKinds = 9 };
int prof_begin(int kind, cudaStream_t s);
void prof_end(int token, cudaStream_t s);
unsigned long long *step_counter(int kind);
void count_transfer(size_t h2d, size_t d2h);

KernelTriple kernels_for(int d, bool fast);
// brm_fit_presort with an event recorded between its transpose and its sort (brm_boost.cu)
int fit_presort(int32_t device, cudaStream_t s, const double *xs, int64_t n, int32_t F, cudaEvent_t mid,
                const void *owner);
void fit_presort_drop(const void *owner, cudaStream_t s);  // unused sorts of a context being destroyed
int set_error(int code, const char *fmt, ...);
void *finish_kernel();
void *sample_kernel();
void *fill_raw_kernel();
void *fill_normals_kernel();
void *math_selftest_kernel();
void *chain_selftest_kernel();
void *exact_scan_selftest_kernel();
// Slotted CMC images (brm_ctx_create_cmc): per date, `ts` threshold entries
// and `vs` table values.  Each feature's padded threshold list has at most
// 2 u_f entries (u_f distinct thresholds, padded to a power of two minus one)
// and u_f + 1 values, so ts = 2 R and vs = R + F bound any ensemble of at most
// R stumps on F features.
struct SlotDims {
  int ts, vs;
};
inline SlotDims slot_dims(int capacity, int nfeat) { return SlotDims{std::max(2 * capacity, 1), capacity + nfeat}; }
constexpr int kMaxSlotStumps = 1024;
void *set_ensemble_kernel();

// Device quadratic regression (brm_boost.cu): n_fits fits of design [J][nb]
// against levels [n_fits][J], coefficients optionally written into a rule image.
struct LsParams {
  const double *design;  // [J][nb] row-major
  const double *levels;  // [n_fits][J]
  int J, nb, k, log_space;
  double *out;           // [n_fits][nb] (may be null)
  int *rank_out;         // [n_fits] (may be null)
  double *dst;           // rule-image surface of the date (may be null)
  int dst_fit_stride;    // doubles between fits' first rows in dst
  int dst_rows;          // rows written per fit (nb doubles apart)
};
constexpr int kLsMaxN = 4096, kLsMaxB = 64;
int launch_ls_fit(const LsParams &P, int n_fits, cudaStream_t s);
size_t ls_fit_smem(int J, int nb);
size_t set_ensemble_smem(int capacity);

// Cached cudaOccupancyMaxActiveClusters for a launch configuration (brm_capi.cu).
int max_active_clusters(const void *kernel, const cudaLaunchConfig_t &cfg, int device);

// Keep freed stream-ordered allocations in the device's default pool across
// synchronisations (the pool's default release threshold of 0 hands them back
// to the driver at every sync, and the next call re-maps them).
void retain_pool(int dev);

}  // namespace brm
