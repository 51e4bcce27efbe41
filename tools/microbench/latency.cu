// Dependent-chain latencies on the target GPU (cycles): DADD, DSETP+FSEL select, int64 compare+select,
// LDS.64, and one top-3 bubble step. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 latency.cu
#include <cstdio>
#include <cstdint>
__global__ void k(double* out, long long* cyc, const double* in, int iters) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = in[i];
  __syncthreads();
  double a = in[threadIdx.x], b = in[threadIdx.x + 1];
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < iters; ++i) { a = __dadd_rn(a, b); a = __dadd_rn(a, -b); }
  long long t1 = clock64();
  double s0 = 1e300, s1 = 1e300, s2 = 1e300, v = a;
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {  // bubble of v through (s0,s1,s2); v depends on s2
    bool lt = v < s0; double lo = lt ? v : s0; double x = lt ? s0 : v; s0 = lo;
    lt = x < s1; lo = lt ? x : s1; x = lt ? s1 : x; s1 = lo;
    s2 = x < s2 ? x : s2;
    v = __dadd_rn(s2, -1e-3);
  }
  long long t2 = clock64();
  int idx = threadIdx.x & 1023;
#pragma unroll 1
  for (int i = 0; i < iters; ++i) { idx = (int)sm[idx]; }
  long long t3 = clock64();
  long long ka = __double_as_longlong(a), kb = __double_as_longlong(b);
#pragma unroll 1
  for (int i = 0; i < iters; ++i) { long long m = ka < kb ? ka : kb; kb = ka ^ m; ka = m + 1; }
  long long t4 = clock64();
  double c = a;
#pragma unroll 1
  for (int i = 0; i < iters; ++i) { bool lt = c < b; c = lt ? b : c; c = __dadd_rn(c, 1.0); }
  long long t5 = clock64();
  out[threadIdx.x] = a + s0 + s1 + s2 + idx + (double)ka + c;
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / (2 * iters); cyc[1] = (t2 - t1) / iters; cyc[2] = (t3 - t2) / iters;
    cyc[3] = (t4 - t3) / iters; cyc[4] = (t5 - t4) / iters;
  }
}
int main() {
  double *in, *out; long long* cyc;
  cudaMallocManaged(&in, 2048 * 8); cudaMallocManaged(&out, 2048 * 8); cudaMallocManaged(&cyc, 64);
  for (int i = 0; i < 2048; ++i) in[i] = (double)((i * 7) % 1024);
  for (int warps : {1, 8, 32}) {
    k<<<1, 32 * warps>>>(out, cyc, in, 4096);
    cudaDeviceSynchronize();
    printf("warps/SM=%2d  DADD %lld cyc | bubble step (3-level, + DADD) %lld | LDS.64 %lld | int64 min %lld | DSETP+sel+DADD %lld\n",
           warps, cyc[0], cyc[1], cyc[2], cyc[3], cyc[4]);
  }
  return 0;
}
