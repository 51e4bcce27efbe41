// Latency of one 16-slot row scan (the GDP sweep's per-node chain) on an idle SM, for two
// formulations of the top-3 bubble: A = fp64 DSETP + selects (k_gdp_sweep5), C = the doubles'
// order-preserving int64 keys compared with 64-bit integer compares. One warp, clock64.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false rowlat2.cu -o rowlat2
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void bubbleA(double (&s)[3], double v) {
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool lt = v < s[i];
    const double lo = lt ? v : s[i];
    v = lt ? s[i] : v;
    s[i] = lo;
  }
  s[2] = v < s[2] ? v : s[2];
}
__device__ __forceinline__ long long okey(double d) {
  const long long b = __double_as_longlong(d);
  return b ^ ((b >> 63) & 0x7fffffffffffffffLL);
}
__device__ __forceinline__ double ounkey(long long k) {
  return __longlong_as_double(k ^ ((k >> 63) & 0x7fffffffffffffffLL));
}
__device__ __forceinline__ void bubbleC(long long (&s)[3], long long v) {
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool lt = v < s[i];
    const long long lo = lt ? v : s[i];
    v = lt ? s[i] : v;
    s[i] = lo;
  }
  s[2] = v < s[2] ? v : s[2];
}

template <int V, int W>
__global__ void k(const double* gc, const uint16_t* gl, const double* glam, double* out, long long* cyc) {
  __shared__ double cst[32 * W];
  __shared__ uint16_t lid[32 * W];
  __shared__ double lam[1024];
  for (int i = threadIdx.x; i < 32 * W; i += blockDim.x) {
    cst[i] = gc[i];
    lid[i] = gl[i];
  }
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) lam[i] = glam[i];
  __syncthreads();
  const int lb = threadIdx.x;
  const double lv = lam[threadIdx.x];
  double acc = 0;
  long long best = 1LL << 60;
  for (int rep = 0; rep < 20; ++rep) {
    __syncwarp();
    const long long t0 = clock64();
    double r;
    if (V == 0) {
      double s[3] = {1e300, 1e300, 1e300};
#pragma unroll
      for (int j = 0; j < W; j += 8) {
        int li[8];
        double cs[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          li[u] = lid[lb + 32 * ((j + u + rep) % W)];
          cs[u] = cst[lb + 32 * ((j + u + rep) % W)];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) bubbleA(s, __dsub_rn(__dsub_rn(cs[u], lv), lam[li[u]]));
      }
      r = __dmul_rn(0.5, __dadd_rn(s[1], s[2]));
    } else {
      long long s[3] = {okey(1e300), okey(1e300), okey(1e300)};
#pragma unroll
      for (int j = 0; j < W; j += 8) {
        int li[8];
        double cs[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          li[u] = lid[lb + 32 * ((j + u + rep) % W)];
          cs[u] = cst[lb + 32 * ((j + u + rep) % W)];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) bubbleC(s, okey(__dsub_rn(__dsub_rn(cs[u], lv), lam[li[u]])));
      }
      r = __dmul_rn(0.5, __dadd_rn(ounkey(s[1]), ounkey(s[2])));
    }
    acc += r;
    const long long t1 = clock64();
    best = min(best, t1 - t0);
  }
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = best;
}

int main() {
  const int W = 16;
  double *c, *lam, *out;
  uint16_t* l;
  long long* cyc;
  cudaMallocManaged(&c, 32 * W * 8);
  cudaMallocManaged(&l, 32 * W * 2);
  cudaMallocManaged(&lam, 1024 * 8);
  cudaMallocManaged(&out, 1024 * 8);
  cudaMallocManaged(&cyc, 8);
  uint64_t x = 7;
  auto rnd = [&]() { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return x; };
  for (int i = 0; i < 32 * W; ++i) { c[i] = (rnd() % 100000) * 1e-3; l[i] = rnd() % 1024; }
  for (int i = 0; i < 1024; ++i) lam[i] = (rnd() % 100000) * 1e-4 - 3.0;
  for (int warps : {1, 4, 16}) {
    k<0, W><<<1, 32 * warps>>>(c, l, lam, out, cyc); cudaDeviceSynchronize();
    const long long a = cyc[0];
    const double ra = out[0];
    k<1, W><<<1, 32 * warps>>>(c, l, lam, out, cyc); cudaDeviceSynchronize();
    printf("warps %2d: %d-slot row: fp64 bubble %lld cycles | int64-key bubble %lld cycles (same result: %d)\n",
           warps, W, a, cyc[0], ra == out[0]);
  }
  return 0;
}
