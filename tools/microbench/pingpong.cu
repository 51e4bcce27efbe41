// Inter-SM signalling latency on the target GPU: CTA 0 ping-pongs with every other CTA in turn
// through global memory, three protocols:
//   LL   : one 8-byte word {payload32, tag32}, st.relaxed.gpu / ld.relaxed.gpu polling (no fences)
//   REL  : payload store + st.release.gpu flag; ld.acquire.gpu flag polling, then payload load
//   FENCE: payload store, fence.acq_rel.gpu, relaxed flag store; relaxed poll, fence, ld.cg payload
// Prints the round-trip time (clock64 cycles and ns) per partner SM, min / median / max over SMs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 pingpong.cu -o pingpong
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned long long ld_rlx64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rlx64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int ld_acq(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_rlx(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_rlx(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct Slot {  // one cache line per direction per protocol
  unsigned long long ll[16];
  int flag[32];
  double data[16];
};

__global__ void k_pingpong(Slot* s, int* turn, long long* out, int* smid_out, int reps, int proto) {
  const int c = blockIdx.x, G = gridDim.x;
  unsigned sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  if (threadIdx.x == 0) smid_out[c] = sm;
  if (threadIdx.x != 0) return;
  Slot* a2b = s + 2 * c;      // CTA 0 -> CTA c
  Slot* b2a = s + 2 * c + 1;  // CTA c -> CTA 0
  if (c == 0) {
    for (int j = 1; j < G; ++j) {
      Slot* x = s + 2 * j;
      Slot* y = s + 2 * j + 1;
      st_rlx(turn, j);
      long long t0 = 0;
      for (int r = 0; r < reps + 8; ++r) {
        if (r == 8) t0 = clock64();
        const unsigned tag = r + 1;
        if (proto == 0) {
          st_rlx64(&x->ll[0], ((unsigned long long)tag << 32) | (unsigned)(r * 3));
          while ((unsigned)(ld_rlx64(&y->ll[0]) >> 32) != tag) {
          }
        } else if (proto == 1) {
          x->data[0] = r;
          st_rel(&x->flag[0], tag);
          while (ld_acq(&y->flag[0]) != (int)tag) {
          }
          volatile double d = y->data[0];
          (void)d;
        } else {
          x->data[0] = r;
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          st_rlx(&x->flag[0], tag);
          while (ld_rlx(&y->flag[0]) != (int)tag) {
          }
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          volatile double d = __ldcg(&y->data[0]);
          (void)d;
        }
      }
      out[j] = (clock64() - t0) / reps;
    }
    st_rlx(turn, G);
  } else {
    while (ld_rlx(turn) != c) {
    }
    for (int r = 0; r < reps + 8; ++r) {
      const unsigned tag = r + 1;
      if (proto == 0) {
        while ((unsigned)(ld_rlx64(&a2b->ll[0]) >> 32) != tag) {
        }
        st_rlx64(&b2a->ll[0], ((unsigned long long)tag << 32) | 7u);
      } else if (proto == 1) {
        while (ld_acq(&a2b->flag[0]) != (int)tag) {
        }
        volatile double d = a2b->data[0];
        (void)d;
        b2a->data[0] = r;
        st_rel(&b2a->flag[0], tag);
      } else {
        while (ld_rlx(&a2b->flag[0]) != (int)tag) {
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        volatile double d = __ldcg(&a2b->data[0]);
        (void)d;
        b2a->data[0] = r;
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        st_rlx(&b2a->flag[0], tag);
      }
    }
  }
}

int main() {
  int dev = 0;
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, dev);
  const int G = p.multiProcessorCount;
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  Slot* s;
  int *turn, *smid;
  long long* out;
  cudaMalloc(&s, sizeof(Slot) * 2 * G);
  cudaMalloc(&turn, 4);
  cudaMalloc(&out, 8 * G);
  cudaMalloc(&smid, 4 * G);
  const char* names[3] = {"LL (8B tag+data, relaxed)", "REL (st.release / ld.acquire)", "FENCE (fence + relaxed flag)"};
  for (int proto = 0; proto < 3; ++proto) {
    cudaMemset(s, 0, sizeof(Slot) * 2 * G);
    cudaMemset(turn, 0, 4);
    cudaMemset(out, 0, 8 * G);
    const int reps = 200;
    void* args[] = {&s, &turn, &out, &smid, (void*)&reps, &proto};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_pingpong, dim3(G), dim3(32), args, 0, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    std::vector<long long> h(G);
    std::vector<int> sm(G);
    cudaMemcpy(h.data(), out, 8 * G, cudaMemcpyDeviceToHost);
    cudaMemcpy(sm.data(), smid, 4 * G, cudaMemcpyDeviceToHost);
    std::vector<long long> v(h.begin() + 1, h.end());
    std::sort(v.begin(), v.end());
    const double ns = 1e6 / clk_khz;
    printf("%-32s round trip cycles: min %lld  median %lld  max %lld  (~%.0f / %.0f / %.0f ns at %d MHz)\n", names[proto],
           v.front(), v[v.size() / 2], v.back(), v.front() * ns, v[v.size() / 2] * ns, v.back() * ns, clk_khz / 1000);
    if (proto == 0) {
      printf("  per partner (smid:cycles):");
      for (int j = 1; j < G; ++j) printf(" %d:%lld", sm[j], h[j]);
      printf("  [cta0 on sm %d]\n", sm[0]);
    }
  }
  return 0;
}
