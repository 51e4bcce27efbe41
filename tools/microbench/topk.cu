// Throughput of the per-slot selection step of the GDP sweep (top-3 of (c - lv) - l over a row)
// on a full SM (148 CTAs x 1024 threads, rows in shared memory), for three formulations:
//   A  DSETP + selects bubble (k_gdp_sweep5 today)
//   B  fmin/fmax bubble (DMNMX if the ISA has it)
//   C  ordered-int64 keys: compare-exchange on integers
// Prints ns per slot-per-SM (lower is better) and the SASS opcode the compiler chose.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false topk.cu -o topk
#include <cstdint>
#include <cstdio>

constexpr int W = 16;        // slots per row
constexpr int ROWS = 4;      // rows per thread per iteration

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
__device__ __forceinline__ void bubbleB(double (&s)[3], double v) {
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double lo = fmin(v, s[i]);
    v = fmax(v, s[i]);
    s[i] = lo;
  }
  s[2] = fmin(v, s[2]);
}
__device__ __forceinline__ long long okey(double d) {
  const long long b = __double_as_longlong(d);
  return b ^ ((b >> 63) & 0x7fffffffffffffffLL);
}
__device__ __forceinline__ void bubbleC(long long (&s)[3], long long v) {
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const long long lo = min(v, s[i]);
    v = max(v, s[i]);
    s[i] = lo;
  }
  s[2] = min(v, s[2]);
}

// D: v < s decided by the sign of the exact-sign difference v - s (DADD + integer sign test
//    instead of DSETP); three independent compares against the old list, then selects.
__device__ __forceinline__ bool lt_sign(double v, double s) {
  return __double2hiint(__dsub_rn(v, s)) < 0;
}
__device__ __forceinline__ void insertD(double (&s)[3], double v) {
  const bool c0 = lt_sign(v, s[0]), c1 = lt_sign(v, s[1]), c2 = lt_sign(v, s[2]);
  s[2] = c1 ? s[1] : (c2 ? v : s[2]);
  s[1] = c0 ? s[0] : (c1 ? v : s[1]);
  s[0] = c0 ? v : s[0];
}
// E: the same three-compare insert with DSETP
__device__ __forceinline__ void insertE(double (&s)[3], double v) {
  const bool c0 = v < s[0], c1 = v < s[1], c2 = v < s[2];
  s[2] = c1 ? s[1] : (c2 ? v : s[2]);
  s[1] = c0 ? s[0] : (c1 ? v : s[1]);
  s[0] = c0 ? v : s[0];
}

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(const double* gcost, const uint16_t* glid, const double* glam,
                                             double* out, long long* cyc, int iters) {
  __shared__ double cst[1024 * 4];
  __shared__ uint16_t lid[1024 * 4];
  __shared__ double lam[1024];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) {
    cst[i] = gcost[i];
    lid[i] = glid[i];
  }
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) lam[i] = glam[i];
  __syncthreads();
  double acc = 0.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int r = 0; r < ROWS; ++r) {
      const int base = ((warp * ROWS + r) * 32 + lane) & 1023;  // row base in SELL-32 layout
      const double lv = lam[(base + it) & 1023];
      if (MODE == 2) {
        long long s[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX};
#pragma unroll
        for (int j = 0; j < W; ++j) {
          const int idx = (base + 32 * j) & 4095;
          bubbleC(s, okey(__dsub_rn(__dsub_rn(cst[idx], lv), lam[lid[idx]])));
        }
        const long long a = s[1], b = s[2];
        acc = __dadd_rn(acc, __dmul_rn(0.5, __dadd_rn(__longlong_as_double(a ^ ((a >> 63) & 0x7fffffffffffffffLL)),
                                                      __longlong_as_double(b ^ ((b >> 63) & 0x7fffffffffffffffLL)))));
      } else {
        double s[3] = {INFINITY, INFINITY, INFINITY};
#pragma unroll
        for (int j = 0; j < W; ++j) {
          const int idx = (base + 32 * j) & 4095;
          const double v = __dsub_rn(__dsub_rn(cst[idx], lv), lam[lid[idx]]);
          if (MODE == 0) bubbleA(s, v);
          else if (MODE == 1) bubbleB(s, v);
          else if (MODE == 3) insertD(s, v);
          else if (MODE == 4) insertE(s, v);
          else if (MODE == 5) { s[0] = __dadd_rn(s[0], v); s[1] = __dadd_rn(s[1], v); s[2] = __dadd_rn(s[2], v); }
          else { s[0] = (v < s[0]) ? s[1] : s[0]; s[1] = (v < s[1]) ? s[2] : s[1]; s[2] = (v < s[2]) ? s[0] : s[2]; }
        }
        acc = __dadd_rn(acc, __dmul_rn(0.5, __dadd_rn(s[1], s[2])));
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int G = 148;
  double *cost, *lamg, *out;
  uint16_t* lid;
  long long* cyc;
  cudaMallocManaged(&cost, 4096 * 8);
  cudaMallocManaged(&lamg, 2048 * 8);
  cudaMallocManaged(&lid, 4096 * 2);
  cudaMallocManaged(&out, (size_t)G * 1024 * 8);
  cudaMallocManaged(&cyc, G * 8);
  uint64_t x = 12345;
  auto rnd = [&]() { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return x; };
  for (int i = 0; i < 4096; ++i) { cost[i] = (rnd() % 100000) * 1e-3; lid[i] = rnd() % 1024; }
  for (int i = 0; i < 2048; ++i) lamg[i] = (rnd() % 100000) * 1e-4;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 200;
  const char* names[7] = {"A DSETP+select bubble", "B fmin/fmax bubble", "C ordered-int64 bubble",
                          "D sign-of-difference insert", "E DSETP 3-compare insert", "F 3 DADD only (ref)",
                          "G 3 DSETP+sel only (ref)"};
  for (int mode = 0; mode < 7; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<G, 1024>>>(cost, lid, lamg, out, cyc, iters);
      if (mode == 1) k<1><<<G, 1024>>>(cost, lid, lamg, out, cyc, iters);
      if (mode == 2) k<2><<<G, 1024>>>(cost, lid, lamg, out, cyc, iters);
      if (mode == 3) k<3><<<G, 1024>>>(cost, lid, lamg, out, cyc, iters);
      if (mode == 4) k<4><<<G, 1024>>>(cost, lid, lamg, out, cyc, iters);
      if (mode == 5) k<5><<<G, 1024>>>(cost, lid, lamg, out, cyc, iters);
      if (mode == 6) k<6><<<G, 1024>>>(cost, lid, lamg, out, cyc, iters);
      cudaDeviceSynchronize();
    }
    long long mx = 0;
    for (int i = 0; i < G; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
    const double slots_per_sm = 1024.0 * ROWS * W * iters;
    printf("%-26s %.3f cycles per slot per SM  (%.1f ps/slot/SM)  check %.6g\n", names[mode], mx / slots_per_sm,
           1e9 / clk * mx / slots_per_sm, out[0]);
  }
  return 0;
}
