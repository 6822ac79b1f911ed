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
// tile of 32 x T weights to integers R_E(w) = rint(w / ulp_E) and
// prefix-sums them -- in fp64, where every integer below 2^53 and every
// power-of-two scaling is exact, so the sums are exact and associative --
// and writes s_k = M_k * ulp_E.  The first element that leaves the binade, is a
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

// Storage position of chain element j: padded arrays insert one slot after
// every 16 elements, so the 16-element runs of consecutive lanes start in
// different shared-memory banks (2-way instead of 32-way conflicts).
template <bool PAD>
__device__ __forceinline__ int chain_pos(int j) {
  return PAD ? j + (j >> 4) : j;
}
__host__ __device__ constexpr int chain_padded_len(int n) { return n + (n >> 4) + 1; }

// Sequential prefix sums out[k] = acc + in[k0] + ... + in[k] for k in
// [k0, k1), continuing acc (one thread; element k stored at chain_pos<PAD>(k)).
// Ping-pong over two register chunks: chunk A is summed while chunk B's
// shared-memory loads are in flight, then the reverse, so no load latency is
// exposed (tools/micro_cuda/chain.cu: 9.2 cycles/element vs 13.4 for the
// plain loop unrolled by 8).
template <bool PAD>
__device__ __forceinline__ void serial_chain(const double *__restrict__ in, double *__restrict__ out, int k0, int k1,
                                             double &acc) {
  constexpr int C = 16;                    // chunk = one padding period
  constexpr int SP = PAD ? C + 1 : C;      // storage stride of a chunk
  int k = k0;
  if (PAD) {  // align k to a chunk boundary
    const int ka = min(k1, (k0 + C - 1) & ~(C - 1));
    for (; k < ka; ++k) {
      acc = __dadd_rn(acc, in[chain_pos<PAD>(k)]);
      out[chain_pos<PAD>(k)] = acc;
    }
  }
  const double *ip = in + chain_pos<PAD>(k);
  double *op = out + chain_pos<PAD>(k);
  double a[C], b[C];
  if (k1 - k >= 2 * C) {
#pragma unroll
    for (int j = 0; j < C; ++j) a[j] = ip[j];
  }
  for (; k + 2 * C <= k1; k += 2 * C, ip += 2 * SP, op += 2 * SP) {
#pragma unroll
    for (int j = 0; j < C; ++j) b[j] = ip[SP + j];
#pragma unroll
    for (int j = 0; j < C; ++j) {
      acc = __dadd_rn(acc, a[j]);
      op[j] = acc;
    }
    const bool more = k + 4 * C <= k1;
#pragma unroll
    for (int j = 0; j < C; ++j) a[j] = more ? ip[2 * SP + j] : 0.0;
#pragma unroll
    for (int j = 0; j < C; ++j) {
      acc = __dadd_rn(acc, b[j]);
      op[SP + j] = acc;
    }
  }
  for (; k < k1; ++k) {
    acc = __dadd_rn(acc, in[chain_pos<PAD>(k)]);
    out[chain_pos<PAD>(k)] = acc;
  }
}

constexpr int kChainLead = 256;  // leading elements summed one by one (binade crossings are dense there)

// out[k] = acc + in[0] + ... + in[k] in sequential fp64 order, k < cnt, for
// in[] >= 0 (finite); element k stored at chain_pos<PAD>(k).  Called by all
// 32 lanes of one warp; acc is updated in every lane.
template <bool PAD, int T = kChainT>
__device__ inline void warp_chain(const double *__restrict__ in, double *__restrict__ out, int cnt, double &acc) {
  static_assert(T % 16 == 0, "lane runs are whole padding periods");
  const unsigned lane = threadIdx.x & 31;
  constexpr int TILE = 32 * T;
  double s = acc;
  int k = 0;
  int seq = kChainLead;  // elements to run one by one before trying tiles again
  while (k < cnt) {
    const long long sb = __double_as_longlong(s);
    const int Es = (int)((sb >> 52) & 0x7ff);
    if (seq > 0 || Es == 0 || s < 0.0) {
      // zero / subnormal start, or a dense run of events: lane 0 steps, then broadcast
      const int k1 = min(cnt, k + (seq > 0 ? seq : 1));
#ifdef BRM_CHAIN_STATS
      const long long c0 = clock64();
#endif
      if (lane == 0) serial_chain<PAD>(in, out, k, k1, s);
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
    // s = Ms * ulp with Ms an integer in [2^52, 2^53); x = w / ulp is exact
    // (power-of-two scaling), and every integer below 2^53 is a double, so
    // the tile's rounding and prefix sums run exactly in fp64
    if (Es < 53) {  // 1 / ulp not representable: step one by one
      seq = 32;
      continue;
    }
    if (PAD && (k & 15)) {  // tiles start on a padding period: step to the boundary
      seq = 16 - (k & 15);
      continue;
    }
    const double ulp = __longlong_as_double((long long)(Es - 52) << 52);     // 2^(Es - 1075)
    const double inv = __longlong_as_double((long long)(2098 - Es) << 52);   // 2^(1075 - Es)
    const double Ms = __dmul_rn(s, inv);
    const int base = k + (int)lane * T;
    const int nv = cnt - base;  // valid elements of this lane (may be <= 0 or >= T)
    // storage of element base + i: sb0 + off(i) (base is a multiple of 16 when PAD)
    const int sb0 = PAD ? chain_pos<PAD>(base) : base;
    auto off = [](int i) { return PAD ? i + (i >> 4) : i; };
    double pre[T];
    unsigned flag = 0;  // bit i: element i is a tie, not below s's binade (x >= 2^52), or past the end
#pragma unroll
    for (int i = 0; i < T; ++i) {
      const double x = __dmul_rn(i < nv ? in[sb0 + off(i)] : 0.0, inv);
      const double r = rint(x);
      pre[i] = r;
      flag |= (i >= nv || x >= 0x1p52 || fabs(__dsub_rn(x, r)) == 0.5) ? (1u << i) : 0u;
    }
    // in-lane inclusive prefix as two half chains (exact integers: any order)
    constexpr int H = T / 2;
#pragma unroll
    for (int i = 1; i < T; ++i)
      if (i != H) pre[i] = __dadd_rn(pre[i - 1], pre[i]);
#pragma unroll
    for (int i = H; i < T; ++i) pre[i] = __dadd_rn(pre[H - 1], pre[i]);
    const double run = pre[T - 1];
    // exclusive scan of the lane totals (exact integers until the first event)
    double incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, incl, o);
      if ((int)lane >= o) incl = __dadd_rn(incl, y);
    }
    // M before this lane's first element (the previous lane's inclusive sum;
    // no subtraction, so an overflowing element cannot poison its own lane)
    const double prev = __shfl_up_sync(0xffffffffu, incl, 1);
    const double excl = lane ? __dadd_rn(Ms, prev) : Ms;
    // first event of the lane: flagged, or the prefix reaches 2^53 (monotone,
    // so only a lane whose total crosses needs the per-element test)
    int first = flag ? __ffs(flag) - 1 : T;
    if (!(__dadd_rn(excl, run) < 0x1p53)) {
      const double lim = __dsub_rn(0x1p53, excl);  // exact: excl in [2^52, 2^53)
      int below = 0;
#pragma unroll
      for (int i = 0; i < T; ++i) below += pre[i] < lim ? 1 : 0;
      first = min(first, below);
    }
    const int jev = (int)__reduce_min_sync(0xffffffffu, (unsigned)(first < T ? (int)lane * T + first : TILE));
    // prefixes before the event are exact multiples of ulp
    const int mine = jev - (int)lane * T;
#pragma unroll
    for (int i = 0; i < T; ++i)
      if (i < mine) out[sb0 + off(i)] = __dmul_rn(__dadd_rn(excl, pre[i]), ulp);
    const int owner = jev / T, at = jev - owner * T;
    if (jev < TILE && k + jev < cnt) {
      // event element: one fp64 add from the exact previous prefix
      double sn = 0.0;
      if ((int)lane == owner) {
        double Mp = excl;
#pragma unroll
        for (int i = 0; i < T; ++i)
          if (i < at) Mp = __dadd_rn(excl, pre[i]);
        sn = __dadd_rn(__dmul_rn(Mp, ulp), in[sb0 + off(at)]);
        out[sb0 + off(at)] = sn;
      }
      s = __shfl_sync(0xffffffffu, sn, owner);
      k += jev + 1;
      BRM_CHAIN_STAT(1, 1);
      if (jev < 2 * T) seq = 32;  // events are dense here: step one by one for a while
    } else {
      // no event before the end of the tile / chain: continue from the last prefix
      const int last = min(TILE, cnt - k) - 1;
      const int lo = last / T, li = last - lo * T;
      double Ml = 0.0;
#pragma unroll
      for (int i = 0; i < T; ++i)
        if (i == li) Ml = __dadd_rn(excl, pre[i]);
      Ml = __shfl_sync(0xffffffffu, Ml, lo);
      s = __dmul_rn(Ml, ulp);
      k += last + 1;
    }
#ifdef BRM_CHAIN_STATS
    BRM_CHAIN_STAT(4, clock64() - c0);
#endif
  }
  acc = s;
}

}  // namespace brm
