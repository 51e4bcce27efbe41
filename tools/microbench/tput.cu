// Per-SM issue throughput of the instructions the GDP sweep is made of (1024 threads / SM,
// 8 independent chains per thread): DADD, DSETP(+FSEL), FSEL, IADD, SHFL, LDS.64 (coalesced and
// random), LDS.U16. Prints cycles per warp-instruction per SM (4 SMSPs: 0.25 = 1 per SMSP-clock).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tput.cu -o tput
#include <cstdint>
#include <cstdio>

template <int OP>
__global__ void __launch_bounds__(1024, 1) k(const double* in, double* out, long long* cyc, int iters) {
  __shared__ double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = in[i & 1023];
  __syncthreads();
  double x[8];
  int ix[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    x[c] = in[(threadIdx.x + c) & 1023];
    ix[c] = (threadIdx.x * 37 + c * 101) & 4095;
  }
  const double y = in[threadIdx.x & 7];
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (OP == 0) x[c] = __dadd_rn(x[c], y);                         // DADD
      if (OP == 1) x[c] = (x[c] < y) ? y : x[c];                        // DSETP + 2 FSEL
      if (OP == 2) ix[c] = ix[c] + (int)threadIdx.x;                    // IADD
      if (OP == 3) x[c] = __shfl_xor_sync(0xffffffffu, x[c], 1);        // 2 SHFL (64-bit)
      if (OP == 4) x[c] = sm[(threadIdx.x + c * 32 + it) & 4095] + 0.0; // LDS.64 coalesced (+DADD)
      if (OP == 5) { ix[c] = (int)sm[ix[c]]; }                          // LDS.64 random (+F2I)
      if (OP == 6) x[c] = __int_as_float((int)x[c] < 3 ? 1 : 2);        // misc int
    }
  }
  const long long t1 = clock64();
  double acc = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) acc += x[c] + ix[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  const int G = 148, iters = 1000;
  double *in, *out;
  long long* cyc;
  cudaMallocManaged(&in, 4096 * 8);
  cudaMallocManaged(&out, (size_t)G * 1024 * 8);
  cudaMallocManaged(&cyc, G * 8);
  for (int i = 0; i < 4096; ++i) in[i] = (double)((i * 2654435761u) % 4096);
  const char* names[7] = {"DADD", "DSETP+2FSEL", "IADD", "SHFL x2 (f64)", "LDS.64 coalesced +DADD",
                          "LDS.64 random", "I2F-ish int"};
  for (int op = 0; op < 6; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) {
        case 0: k<0><<<G, 1024>>>(in, out, cyc, iters); break;
        case 1: k<1><<<G, 1024>>>(in, out, cyc, iters); break;
        case 2: k<2><<<G, 1024>>>(in, out, cyc, iters); break;
        case 3: k<3><<<G, 1024>>>(in, out, cyc, iters); break;
        case 4: k<4><<<G, 1024>>>(in, out, cyc, iters); break;
        case 5: k<5><<<G, 1024>>>(in, out, cyc, iters); break;
      }
      cudaDeviceSynchronize();
    }
    long long mx = 0;
    for (int i = 0; i < G; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
    printf("%-24s %.3f cycles per warp-op per SM\n", names[op], (double)mx / (32.0 * 8 * iters));
  }
  return 0;
}
