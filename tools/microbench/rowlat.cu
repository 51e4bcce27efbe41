// Latency of one row scan (the GDP sweep's per-node work) on an otherwise idle SM: W slots of
// (cost - lv) - lam[lid] through the top-3 bubble, with 1 / 2 / 4 independent top lists per row.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false rowlat.cu -o rowlat
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void bubble(double (&s)[3], double v) {
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool lt = v < s[i];
    const double lo = lt ? v : s[i];
    v = lt ? s[i] : v;
    s[i] = lo;
  }
  s[2] = v < s[2] ? v : s[2];
}
__device__ __forceinline__ void merge(double (&s)[3], const double (&o)[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) s[i] = o[2 - i] < s[i] ? o[2 - i] : s[i];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j + 1 < 3 - i; ++j) {
      const bool sw = s[j + 1] < s[j];
      const double lo = sw ? s[j + 1] : s[j];
      s[j + 1] = sw ? s[j] : s[j + 1];
      s[j] = lo;
    }
}

template <int CH, int W>
__global__ void k(const double* gc, const uint16_t* gl, const double* glam, double* out, long long* cyc) {
  __shared__ double cst[32 * W * 4];
  __shared__ uint16_t lid[32 * W * 4];
  __shared__ double lam[1024];
  for (int i = threadIdx.x; i < 32 * W * 4; i += blockDim.x) {
    cst[i] = gc[i];
    lid[i] = gl[i];
  }
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) lam[i] = glam[i];
  __syncthreads();
  const int lb = threadIdx.x;  // SELL: slot j of this row at lb + 32*j (blockDim <= 128)
  const double lv = lam[threadIdx.x];
  double acc = 0;
  long long best = 1LL << 60;
  for (int rep = 0; rep < 20; ++rep) {
    __syncwarp();
    const long long t0 = clock64();
    double s[CH][3];
#pragma unroll
    for (int c = 0; c < CH; ++c) s[c][0] = s[c][1] = s[c][2] = 1e300;
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
      for (int u = 0; u < 8; ++u) bubble(s[u % CH], __dsub_rn(__dsub_rn(cs[u], lv), lam[li[u]]));
    }
    if (CH >= 2) merge(s[0], s[1]);
    if (CH == 4) {
      merge(s[2], s[3]);
      merge(s[0], s[2]);
    }
    acc += __dmul_rn(0.5, __dadd_rn(s[0][1], s[0][2]));
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
  cudaMallocManaged(&c, 32 * W * 4 * 8);
  cudaMallocManaged(&l, 32 * W * 4 * 2);
  cudaMallocManaged(&lam, 1024 * 8);
  cudaMallocManaged(&out, 1024 * 8);
  cudaMallocManaged(&cyc, 8);
  uint64_t x = 7;
  auto rnd = [&]() { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return x; };
  for (int i = 0; i < 32 * W * 4; ++i) { c[i] = (rnd() % 100000) * 1e-3; l[i] = rnd() % 1024; }
  for (int i = 0; i < 1024; ++i) lam[i] = (rnd() % 100000) * 1e-4;
  for (int warps : {1, 3, 4}) {
    k<1, W><<<1, 32 * warps>>>(c, l, lam, out, cyc); cudaDeviceSynchronize();
    const long long a = cyc[0];
    k<2, W><<<1, 32 * warps>>>(c, l, lam, out, cyc); cudaDeviceSynchronize();
    const long long b = cyc[0];
    k<4, W><<<1, 32 * warps>>>(c, l, lam, out, cyc); cudaDeviceSynchronize();
    printf("warps %d: row of %d slots: 1 chain %lld cycles | 2 chains %lld | 4 chains %lld\n", warps, W, a, b, cyc[0]);
  }
  return 0;
}
