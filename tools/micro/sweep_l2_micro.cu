// Micro benchmark (not product code): the slot sweep's load side alone
// (16-byte slots, due test + dead count, no per-instance min) with the slots
// in L1, in L2 (ld.global.cg) or in HBM (a 2 GiB array, a fresh region per
// rep), at U loads in flight per thread.  512 CTAs x 128 threads, 2500
// slots per CTA, like the C5 shard's tick sweep.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/m tools/micro/sweep_l2_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

struct alignas(16) Slot {
  double tp;
  float nx;
  int meta;
};

template <int CG>
__device__ __forceinline__ void ld(const Slot* p, double& tp, float& nx, int& m) {
  unsigned long long lo, hi;
  if (CG == 2) {
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.L2::cache_hint.v2.b64 {%0, %1}, [%2], %3;" : "=l"(lo), "=l"(hi) : "l"(p), "l"(pol));
  } else if (CG)
    asm volatile("ld.global.cg.v2.b64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(p));
  else
    asm volatile("ld.global.v2.b64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(p));
  tp = __longlong_as_double((long long)lo);
  nx = __int_as_float((int)(unsigned)hi);
  m = (int)(hi >> 32);
}

template <int U, int CG>
__global__ void __launch_bounds__(128, 4) sweep(const Slot* base, long long stride_rep, int n, int reps, long long* out,
                                                int* sink) {
  __shared__ int total, dead_all;
  long long cyc = 0;
  int acc = 0;
  for (int r = 0; r < reps; r++) {
    const Slot* s = base + stride_rep * r + (size_t)blockIdx.x * n;
    if (threadIdx.x == 0) total = dead_all = 0;
    __syncthreads();
    const long long t0 = clock64();
    double tp[U];
    float nx[U];
    int mt[U];
    int dead = 0;
    for (int b0 = 0; b0 < n; b0 += 128 * U) {
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int j = b0 + u * 128 + threadIdx.x;
        mt[u] = -1;
        if (j < n) ld<CG>(&s[j], tp[u], nx[u], mt[u]);
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        if (mt[u] < 0) continue;
        if (((mt[u] >> 7) & 7) > 0 && nx[u] < 102.0f) atomicAdd(&total, 1);
        if (tp[u] != tp[u]) dead++;
      }
    }
    if (dead) atomicAdd(&dead_all, dead);
    __syncthreads();
    cyc += clock64() - t0;
    acc += total + dead_all;
  }
  if (threadIdx.x == 0) {
    out[blockIdx.x] = cyc / reps;
    sink[blockIdx.x] = acc;
  }
}

int main() {
  const int nblk = 512, n = 2500, reps = 20;
  const size_t per_rep = (size_t)nblk * n;
  const size_t total = per_rep * 48; /* 2 GiB / 16 B ~ 48 reps of fresh data */
  Slot* d;
  long long* o;
  int* sink;
  cudaMalloc(&d, sizeof(Slot) * total);
  cudaMemset(d, 0, sizeof(Slot) * total);
  cudaMalloc(&o, 8 * nblk);
  cudaMalloc(&sink, 4 * nblk);
  long long h[512];
  auto run = [&](const char* name, auto kern, long long stride) {
    kern<<<nblk, 128>>>(d, stride, n, reps, o, sink);
    cudaDeviceSynchronize();
    cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0;
    for (int b = 0; b < nblk; b++) m += h[b];
    printf("%-22s %8.0f cycles/sweep\n", name, m / nblk);
  };
  run("L1 U=2", sweep<2, 0>, 0);
  run("L2 U=2", sweep<2, 1>, 0);
  run("L2 U=4", sweep<4, 1>, 0);
  run("L2 U=8", sweep<8, 1>, 0);
  run("L1/L2 evict_last U=2", sweep<2, 2>, 0);
  run("HBM evict_last U=2", sweep<2, 2>, (long long)per_rep * 2);
  run("HBM U=2", sweep<2, 1>, (long long)per_rep * 2);
  run("HBM U=4", sweep<4, 1>, (long long)per_rep * 2);
  run("HBM U=8", sweep<8, 1>, (long long)per_rep * 2);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
