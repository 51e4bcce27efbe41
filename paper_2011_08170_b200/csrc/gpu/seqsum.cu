// seqsum.cu — bit-exact parallel evaluation of SEQUENTIAL fp64 sums on sm_100a.
//
// The reference accumulates several quantities left to right in one fp64 chain: the objective
// sum_e c_e x_e (primal.cpp:226-230), the per-chunk partial sums of the dual objective
// (dual.cpp:96-109 through parallel.cpp's chunking) and mean_cost (graph.cpp:47-49). A chain of
// k dependent DADDs costs k x ~13.5 cycles on one thread (0.76 ms for the 100k objective). This
// file reproduces the chain's result exactly, in parallel:
//
//   Inside one binade [2^E, 2^(E+1)) the representable numbers are the multiples of
//   u = 2^(E-52). If acc is such a multiple and the exact sum acc + t stays inside the binade,
//   round-to-nearest-even gives fl(acc + t) = acc + RNE_u(t): the rounding of t to a multiple of
//   u no longer depends on acc (except for exact ties, t/u = k + 1/2, where "even" refers to the
//   result). So within a binade the sequential chain is an INTEGER prefix sum of
//   q_i = RNE_u(t_i)/u, which is associative.
//
// Algorithm (per segment of a uniform segmentation of the input; segment sums start from +0.0):
//   1. k_ss_approx   one warp per chunk of kChunk terms: any-order approximate chunk sum;
//   2. cub scan      approximate running value at every chunk start -> predicted binade/sign;
//   3. k_ss_desc     per chunk, in units of the predicted binade's ulp: Q = sum q_i and the min /
//                    max of the partial sums (magnitude direction); "bad" on ties, non-finite
//                    terms, terms >= 2^(E+1), or a zero / subnormal prediction;
//   4. k_ss_super    kSuper consecutive chunks with the same prediction combine associatively;
//   5. k_ss_walk     one CTA per segment walks the super-chunks in order with the EXACT running
//                    value (warp 0, 32 descriptors per round via a warp scan of their Q): a
//                    super-chunk (or, below it, a chunk) is applied in O(1) only if the
//                    exact value sits in the predicted binade with the predicted sign and every
//                    partial sum a + P_i stays in [2^52 + 1, 2^53 - 1] ulps (so every exact
//                    intermediate sum stays inside the binade); otherwise the chunk's terms are
//                    added one by one with __dadd_rn, exactly like the reference.
// Predictions only decide the fast/slow route, never the value: the result is the sequential
// chain's for every input. Mispredictions (binade crossings: ~log2(range) per segment; ties:
// ~2^-16 per term for random mantissas) cost one sequentially added chunk each.
#include <cub/cub.cuh>

#include "internal.cuh"

namespace f2mgpu {

namespace {

constexpr int kChunk = 64;   // terms per chunk (kLaneTerms per lane of the describing warp)
constexpr int kLaneTerms = kChunk / 32;
constexpr int kSuper = 32;   // chunks per super-chunk
constexpr int kWalkThreads = 256;
constexpr long long kTwo52 = 1LL << 52;
constexpr unsigned long long kMant = (1ull << 52) - 1;

enum : int { kBad = 1, kNeg = 2, kEmpty = 4 };

struct SumDesc {
  long long q;   // sum of q_i (ulps of the predicted binade, magnitude direction)
  long long mn;  // min over the chunk's partial sums (after each term)
  long long mx;  // max over the chunk's partial sums
  int be;        // predicted biased exponent of the running value
  int flags;
};

struct SegGeom {
  int64_t k, seg_len;
  int64_t cps;  // chunks per segment
  int64_t sps;  // super-chunks per segment
  __device__ __forceinline__ void chunk_range(int64_t c, int64_t& lo, int64_t& hi) const {
    const int64_t s = c / cps, i = c - s * cps;
    const int64_t seg_lo = s * seg_len, seg_hi = min64(seg_lo + seg_len, k);
    lo = min64(seg_lo + i * kChunk, seg_hi);
    hi = min64(lo + kChunk, seg_hi);
  }
};

__global__ void __launch_bounds__(256) k_ss_approx(SegGeom g, int64_t nchunks, const double* __restrict__ v,
                                                   double* __restrict__ approx) {
  const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= nchunks) return;
  int64_t lo, hi;
  g.chunk_range(c, lo, hi);
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < kLaneTerms; ++j) {
    const int64_t i = lo + lane + 32 * j;
    if (i < hi) s += v[i];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) approx[c] = s;
}

// q = RNE(|t| / u) in the magnitude direction of the running value (u = 2^(be - 1075));
// returns false for ties, non-finite t, or |t| >= 2^(E+1) (the step cannot stay in the binade)
__device__ __forceinline__ bool quantise(double t, int be, bool neg, long long& q) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(t);
  const int bt = (int)((bits >> 52) & 0x7ff);
  if (bt == 0x7ff) return false;
  const unsigned long long mt = (bits & kMant) | (bt ? (1ull << 52) : 0ull);
  const int shift = (bt ? bt : 1) - be;
  unsigned long long r;
  if (mt == 0) {
    r = 0;
  } else if (shift >= 1) {
    return false;
  } else if (shift == 0) {
    r = mt;
  } else {
    const int rs = -shift;
    if (rs >= 64) {
      r = 0;
    } else {
      r = mt >> rs;
      const unsigned long long rem = mt & ((1ull << rs) - 1), half = 1ull << (rs - 1);
      if (rem > half) ++r;
      else if (rem == half) return false;  // exact tie: depends on the running value's parity
    }
  }
  const bool tneg = (bits >> 63) != 0;
  q = (tneg == neg) ? (long long)r : -(long long)r;
  return true;
}

__global__ void __launch_bounds__(256) k_ss_desc(SegGeom g, int64_t nchunks, const double* __restrict__ v,
                                                 const double* __restrict__ pre, SumDesc* __restrict__ desc) {
  const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= nchunks) return;
  int64_t lo, hi;
  g.chunk_range(c, lo, hi);
  SumDesc d{0, 0, 0, 0, 0};
  if (lo >= hi) {
    if (lane == 0) {
      d.flags = kEmpty;
      desc[c] = d;
    }
    return;
  }
  const int64_t c0 = (c / g.cps) * g.cps;  // first chunk of the segment
  const double start = pre[c] - pre[c0];   // approximate running value before this chunk
  const unsigned long long sb = (unsigned long long)__double_as_longlong(start);
  const int be = (int)((sb >> 52) & 0x7ff);
  const bool neg = (sb >> 63) != 0;
  bool ok = be != 0 && be != 0x7ff;  // zero / subnormal / non-finite prediction: walk it
  // lane owns kLaneTerms consecutive terms (in order); local inclusive prefix, min / max
  long long p = 0, lmn = LLONG_MAX, lmx = LLONG_MIN;
#pragma unroll
  for (int j = 0; j < kLaneTerms; ++j) {
    const int64_t i = lo + kLaneTerms * lane + j;
    if (i < hi) {
      long long q = 0;
      ok = quantise(v[i], be, neg, q) && ok;
      p += q;
      lmn = min(lmn, p);
      lmx = max(lmx, p);
    }
  }
  // exclusive warp scan of the lane totals
  long long incl = p;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const long long excl = incl - p;
  if (lmn != LLONG_MAX) {
    lmn += excl;
    lmx += excl;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    lmn = min(lmn, __shfl_xor_sync(0xffffffffu, lmn, o));
    lmx = max(lmx, __shfl_xor_sync(0xffffffffu, lmx, o));
  }
  const bool all_ok = __all_sync(0xffffffffu, ok);
  if (lane == 31) {
    d.q = incl;
    d.mn = lmn;
    d.mx = lmx;
    d.be = be;
    // a valid chunk keeps every partial sum within 2^52 ulps of its start: larger cannot apply
    const bool small = lmn > -kTwo52 && lmx < kTwo52;
    d.flags = (all_ok && small ? 0 : kBad) | (neg ? kNeg : 0);
    desc[c] = d;
  }
}

// one warp per super-chunk, one lane per chunk (kSuper == 32): combine the non-empty chunks'
// descriptors in order (exclusive scan of Q shifts each chunk's min / max)
__global__ void __launch_bounds__(256) k_ss_super(int64_t nsup_total, int64_t cps, int64_t sps,
                                                  const SumDesc* __restrict__ desc, SumDesc* __restrict__ sdesc) {
  static_assert(kSuper == 32, "one lane per chunk");
  const int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= nsup_total) return;
  const int64_t s = t / sps, j = t - s * sps;
  const int64_t c = s * cps + j * kSuper + lane;
  const bool have = c < (s + 1) * cps;
  SumDesc d;
  if (have) d = desc[c];
  else d = SumDesc{0, 0, 0, 0, kEmpty};
  const bool empty = (d.flags & kEmpty) != 0;
  const unsigned ne = __ballot_sync(0xffffffffu, !empty);
  SumDesc r{0, 0, 0, -1, kEmpty};
  if (ne) {
    const int first = __ffs(ne) - 1;
    const int be0 = __shfl_sync(0xffffffffu, d.be, first);
    const int neg0 = __shfl_sync(0xffffffffu, d.flags & kNeg, first);
    const bool ok = empty || (!(d.flags & kBad) && d.be == be0 && (d.flags & kNeg) == neg0);
    const long long q = empty ? 0 : d.q;
    long long incl = q;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const long long excl = incl - q;
    long long mn = empty ? LLONG_MAX : excl + d.mn, mx = empty ? LLONG_MIN : excl + d.mx;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const long long total = __shfl_sync(0xffffffffu, incl, 31);
    if (__all_sync(0xffffffffu, ok)) r = SumDesc{total, mn, mx, be0, neg0};
    else r.flags = kBad;
  }
  if (lane == 0) sdesc[t] = r;
}

// Warp 0 advances the exact running value over descriptors D[i..cnt), 32 at a time: a
// descriptor applies in O(1) iff it is not bad, the running value is normal with the predicted
// binade and sign, and — given every earlier descriptor of the round applied (exclusive scan of
// their Q) — all of its partial sums stay inside [2^52 + 1, 2^53 - 1] ulps (then every exact
// intermediate sum is inside the binade and each add is acc + RNE_ulp(t)). Stops at the first
// descriptor that does not apply (returned in i, not applied) or at cnt. acc is warp-uniform.
__device__ __forceinline__ void warp_advance(const SumDesc* D, int cnt, int& i, double& acc) {
  const int lane = threadIdx.x & 31;
  while (i < cnt) {
    const int idx = i + lane;
    const bool have = idx < cnt;
    SumDesc d;
    if (have) d = D[idx];
    else d = SumDesc{0, 0, 0, 0, kEmpty};
    const unsigned long long bits = (unsigned long long)__double_as_longlong(acc);
    const int be = (int)((bits >> 52) & 0x7ff);
    const int sg = (int)(bits >> 63);
    const bool normal = be != 0 && be != 0x7ff;
    const long long a = (long long)((bits & kMant) | (1ull << 52));
    const bool empty = (d.flags & kEmpty) != 0;
    bool ok = empty || (!(d.flags & kBad) && normal && d.be == be && ((d.flags & kNeg) ? 1 : 0) == sg);
    const long long q = (ok && !empty) ? d.q : 0;
    long long incl = q;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const long long excl = incl - q;
    if (ok && !empty) ok = a + excl + d.mn >= kTwo52 + 1 && a + excl + d.mx <= 2 * kTwo52 - 1;
    const unsigned fail = __ballot_sync(0xffffffffu, have && !ok);
    const int f = fail ? __ffs(fail) - 1 : min(32, cnt - i);
    const long long add = f < 32 ? __shfl_sync(0xffffffffu, excl, f) : __shfl_sync(0xffffffffu, incl, 31);
    if (normal && add != 0) {
      const unsigned long long na = (unsigned long long)(a + add);
      acc = __longlong_as_double((long long)((bits & ~kMant) | (na & kMant)));
    }
    i += f;
    if (fail) return;
  }
}

__global__ void __launch_bounds__(kWalkThreads) k_ss_walk(SegGeom g, const double* __restrict__ v,
                                                          const SumDesc* __restrict__ desc,
                                                          const SumDesc* __restrict__ sdesc,
                                                          double* __restrict__ out) {
  __shared__ SumDesc s_sup[kWalkThreads];
  __shared__ SumDesc s_ch[kSuper];
  __shared__ double s_terms[kSuper * kChunk];  // every term of the super-chunk being descended
  __shared__ int s_idx;
  const int tid = threadIdx.x, lane = tid & 31;
  const bool walker = tid < 32;  // warp 0 holds the exact running value
  const int64_t seg = blockIdx.x;
  const int64_t sup0 = seg * g.sps, ch0 = seg * g.cps;
  const int64_t seg_lo = seg * g.seg_len;
  double acc = 0.0;
  for (int64_t sb = 0; sb < g.sps; sb += kWalkThreads) {
    const int nb = (int)min64(kWalkThreads, g.sps - sb);
    __syncthreads();
    if (tid < nb) s_sup[tid] = sdesc[sup0 + sb + tid];
    __syncthreads();
    int j = 0;
    for (;;) {
      if (walker) {
        warp_advance(s_sup, nb, j, acc);
        if (lane == 0) s_idx = j;
      }
      __syncthreads();
      j = s_idx;
      if (j >= nb) break;
      // descend into super-chunk sb + j: stage its chunk descriptors and all of its terms in one
      // round trip, then warp 0 walks the chunks, adding the terms of failing chunks in order
      const int64_t cfirst = ch0 + (sb + j) * kSuper;
      const int gc = (int)min64(kSuper, ch0 + g.cps - cfirst);
      const int64_t tlo = min64(seg_lo + (cfirst - ch0) * kChunk, g.k);
      const int64_t thi = min64(min64(tlo + (int64_t)gc * kChunk, seg_lo + g.seg_len), g.k);
      if (tid < gc) s_ch[tid] = desc[cfirst + tid];
      {  // all loads in flight at once: one memory round trip per descent
        constexpr int kPer = kSuper * kChunk / kWalkThreads;
        const int cnt = (int)(thi - tlo);
        double r[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          const int i = tid + u * kWalkThreads;
          r[u] = i < cnt ? __ldg(v + tlo + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) s_terms[tid + u * kWalkThreads] = r[u];
      }
      __syncthreads();
      if (walker) {
        int i = 0;
        for (;;) {
          warp_advance(s_ch, gc, i, acc);
          if (i >= gc) break;
          if (lane == 0) {
            const int lo = i * kChunk, hi = (int)min64((int64_t)lo + kChunk, thi - tlo);
            for (int t = lo; t < hi; ++t) acc = dadd(acc, s_terms[t]);
          }
          acc = __shfl_sync(0xffffffffu, acc, 0);
          ++i;
        }
      }
      ++j;
      __syncthreads();
    }
  }
  if (tid == 0) out[seg] = acc;
}

}  // namespace

void seq_sums_device(const double* v, int64_t k, int64_t seg_len, double* out, cudaStream_t s) {
  static_assert(kWalkThreads >= kSuper && (kSuper * kChunk) % kWalkThreads == 0, "walk CTA stages a super-chunk");
  if (k <= 0) return;
  if (seg_len <= 0 || seg_len > k) seg_len = k;
  const int64_t nseg = (k + seg_len - 1) / seg_len;
  SegGeom g;
  g.k = k;
  g.seg_len = seg_len;
  g.cps = (seg_len + kChunk - 1) / kChunk;
  g.sps = (g.cps + kSuper - 1) / kSuper;
  const int64_t nchunks = nseg * g.cps, nsup = nseg * g.sps;
  DBuf<double> approx(nchunks, s), pre(nchunks, s);
  DBuf<SumDesc> desc(nchunks, s), sdesc(nsup, s);
  k_ss_approx<<<grid_for(nchunks * 32, 256), 256, 0, s>>>(g, nchunks, v, approx.get());
  launched("ss_approx");
  size_t tmp = 0;
  F2M_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, approx.get(), pre.get(), nchunks, s));
  DBuf<char> tb(tmp, s);
  F2M_CUDA(cub::DeviceScan::ExclusiveSum(tb.get(), tmp, approx.get(), pre.get(), nchunks, s));
  launched("ss_scan");
  k_ss_desc<<<grid_for(nchunks * 32, 256), 256, 0, s>>>(g, nchunks, v, pre.get(), desc.get());
  launched("ss_desc");
  k_ss_super<<<grid_for(nsup * 32, 256), 256, 0, s>>>(nsup, g.cps, g.sps, desc.get(), sdesc.get());
  launched("ss_super");
  k_ss_walk<<<(unsigned)nseg, kWalkThreads, 0, s>>>(g, v, desc.get(), sdesc.get(), out);
  launched("ss_walk");
}

}  // namespace f2mgpu

// C ABI (include/f2m_gpu.h): exposed for the parity tests and for callers that need the
// reference's left-to-right fp64 accumulation of device data.
extern "C" int f2m_seq_sums(const double* d_v, int64_t k, int64_t seg_len, double* d_out, void* stream) {
  return f2mgpu::guard([&] {
    f2mgpu::seq_sums_device(d_v, k, seg_len, d_out, static_cast<cudaStream_t>(stream));
  });
}
