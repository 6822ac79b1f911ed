// brm_chain.cuh -- numpy's sequential cumsum order, evaluated by a warp.
//
// AdaBoost's split search needs every prefix s_k = fl(s_{k-1} + w_k) of a
// chain of non-negative weights in the reference's order (np.cumsum,
// boosting.py:150-151): a dependent fp64 add per element when done one
// element at a time (~9 cycles each).  While the running sum stays inside
// one binade [2^E, 2^(E+1)) every prefix is an integer multiple of
// ulp_E = 2^(E-52), and adding w rounds w to that grid:
//     s_k = s_{k-1} + R_E(w_k) * ulp_E,  R_E(w) = round-to-nearest(w / ulp_E)
// as long as w / ulp_E is not an exact tie (whose rounding depends on the
// parity of s_{k-1}) and the sum stays below 2^(E+1).  So a warp converts a
// tile of 32 x kChainT weights to integers, prefix-sums them with integer
// adds (exact and associative), and writes s_k = M_k * ulp_E directly as the
// bit pattern of the double.  The first element that leaves the binade, is a
// tie, or is not below ulp_E * 2^52 (w comparable to s) is an event: its sum
// is formed by one fp64 add from the exact previous prefix, and the warp
// continues from there.  Every prefix is bit-identical to the sequential
// chain; events are rare once s is much larger than the weights (a handful
// of binade crossings and ~ln(n) ties per chain), and dense early stretches
// run element by element.
#pragma once
#include <cstdint>

namespace brm {

constexpr int kChainT = 16;  // elements per lane per tile

#ifdef BRM_CHAIN_STATS
__device__ long long g_chain_stats[6];  // tiles, events, seq elements, seq cycles, tile cycles
#define BRM_CHAIN_STAT(i, v) \
  if ((threadIdx.x & 31) == 0) g_chain_stats[i] += (v)
#else
#define BRM_CHAIN_STAT(i, v)
#endif

// Positive normal s = M * 2^(E - 1075), M in [2^52, 2^53) <-> bits (E - 1) << 52 | ... + M.
__device__ __forceinline__ double chain_value(int E, long long M) {
  return __longlong_as_double(((long long)(E - 1) << 52) + M);
}

// Storage position of chain element j: padded arrays insert one slot after
// every 16 elements, so the 16-element runs of consecutive lanes start in
// different shared-memory banks (2-way instead of 32-way conflicts).
template <bool PAD>
__device__ __forceinline__ int chain_pos(int j) {
  return PAD ? j + (j >> 4) : j;
}
__host__ __device__ constexpr int chain_padded_len(int n) { return n + (n >> 4) + 1; }

// One lane's sequential prefix over in[k0, k1) from s (used by lane 0 only).
template <bool PAD>
__device__ __forceinline__ double chain_seq(const double *__restrict__ in, double *__restrict__ out, int k0, int k1,
                                            double s) {
  for (int k = k0; k < k1; ++k) {
    s = __dadd_rn(s, in[chain_pos<PAD>(k)]);
    out[chain_pos<PAD>(k)] = s;
  }
  return s;
}

// out[k] = acc + in[0] + ... + in[k] in sequential fp64 order, k < cnt, for
// in[] >= 0 (finite); element k stored at chain_pos<PAD>(k).  Called by all
// 32 lanes of one warp; acc is updated in every lane.
template <bool PAD>
__device__ inline void warp_chain(const double *__restrict__ in, double *__restrict__ out, int cnt, double &acc) {
  const unsigned lane = threadIdx.x & 31;
  constexpr int TILE = 32 * kChainT;
  double s = acc;
  int k = 0;
  int seq = 0;  // elements to run one by one before trying tiles again
  while (k < cnt) {
    const long long sb = __double_as_longlong(s);
    const int Es = (int)((sb >> 52) & 0x7ff);
    if (seq > 0 || Es == 0 || s < 0.0) {
      // zero / subnormal start, or a dense run of events: lane 0 steps, then broadcast
      const int k1 = min(cnt, k + (seq > 0 ? seq : 1));
#ifdef BRM_CHAIN_STATS
      const long long c0 = clock64();
#endif
      if (lane == 0) s = chain_seq<PAD>(in, out, k, k1, s);
      s = __shfl_sync(0xffffffffu, s, 0);
      BRM_CHAIN_STAT(2, k1 - k);
#ifdef BRM_CHAIN_STATS
      BRM_CHAIN_STAT(3, clock64() - c0);
#endif
      k = k1;
      seq = 0;
      continue;
    }
#ifdef BRM_CHAIN_STATS
    const long long c0 = clock64();
#endif
    BRM_CHAIN_STAT(0, 1);
    const long long Ms = (sb & 0xFFFFFFFFFFFFFLL) | (1LL << 52);
    const int base = k + (int)lane * kChainT;
    long long pre[kChainT];
    unsigned flag = 0;  // bit i: element i is a tie or comparable to s (or past the end)
    long long run = 0;
    // branch-free, so the elements' integer chains interleave; values after
    // the first event are never used
#pragma unroll
    for (int i = 0; i < kChainT; ++i) {
      const int idx = base + i;
      const long long wb = __double_as_longlong(in[chain_pos<PAD>(idx < cnt ? idx : cnt - 1)]);
      const int ew = (int)(wb >> 52);  // w >= 0: no sign bit
      const long long mw = (wb & 0xFFFFFFFFFFFFFLL) | (ew ? (1LL << 52) : 0LL);
      const int d0 = Es - (ew ? ew : 1);
      const int dsh = min(max(d0, 1), 63);
      const long long rem = mw & ((1LL << dsh) - 1);
      const long long half = 1LL << (dsh - 1);
      run += (mw >> dsh) + (rem > half ? 1 : 0);
      pre[i] = run;
      flag |= (idx >= cnt || d0 <= 0 || rem == half) ? (1u << i) : 0u;
    }
    // exclusive scan of the lane totals
    long long incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if ((int)lane >= o) incl += y;
    }
    const long long excl = Ms + incl - run;  // M before this lane's first element
    // first event of the lane: flagged, or the prefix reaches 2^53 (monotone)
    int first = kChainT;
#pragma unroll
    for (int i = kChainT - 1; i >= 0; --i)
      if (((flag >> i) & 1u) || excl + pre[i] >= (1LL << 53)) first = i;
    const int jev = (int)__reduce_min_sync(0xffffffffu, (unsigned)(first < kChainT ? (int)lane * kChainT + first : TILE));
    // prefixes before the event are exact multiples of ulp_E
#pragma unroll
    for (int i = 0; i < kChainT; ++i)
      if ((int)lane * kChainT + i < jev) out[chain_pos<PAD>(base + i)] = chain_value(Es, excl + pre[i]);
    const int owner = jev / kChainT, at = jev - owner * kChainT;
    if (jev < TILE && k + jev < cnt) {
      // event element: one fp64 add from the exact previous prefix
      double sn = 0.0;
      if ((int)lane == owner) {
        long long Mp = excl;
#pragma unroll
        for (int i = 0; i < kChainT; ++i)
          if (i < at) Mp = excl + pre[i];
        sn = __dadd_rn(chain_value(Es, Mp), in[chain_pos<PAD>(k + jev)]);
        out[chain_pos<PAD>(k + jev)] = sn;
      }
      s = __shfl_sync(0xffffffffu, sn, owner);
      k += jev + 1;
      BRM_CHAIN_STAT(1, 1);
      if (jev < 2 * kChainT) seq = 32;  // events are dense here: step one by one for a while
    } else {
      // no event before the end of the tile / chain: continue from the last prefix
      const int last = min(TILE, cnt - k) - 1;
      const int lo = last / kChainT, li = last - lo * kChainT;
      long long Ml = 0;
#pragma unroll
      for (int i = 0; i < kChainT; ++i)
        if (i == li) Ml = excl + pre[i];
      Ml = __shfl_sync(0xffffffffu, Ml, lo);
      s = chain_value(Es, Ml);
      k += last + 1;
    }
#ifdef BRM_CHAIN_STATS
    BRM_CHAIN_STAT(4, clock64() - c0);
#endif
  }
  acc = s;
}

}  // namespace brm
