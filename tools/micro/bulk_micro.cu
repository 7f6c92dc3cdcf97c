// Micro test of the bulk-staged slot sweep primitives (not product code):
// each CTA (128 threads) rewrites its slots with generic stores, then stages
// them into shared memory with cp.async.bulk + mbarrier (the same sequence as
// engine_core.h job_sweep under EC_BULK_SWEEP) and checks every staged value;
// also times the staged sweep against per-thread 16-byte loads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bulk_micro tools/micro/bulk_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

struct alignas(16) Slot {
  double tp;
  float nx;
  int meta;
};

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   saddr(dst)),
               "l"(__cvta_generic_to_global(src)), "r"(bytes), "r"(saddr(b))
               : "memory");
}
__device__ __forceinline__ void mwait(unsigned long long* b, unsigned par) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n}" ::"r"(saddr(b)),
      "r"(par)
      : "memory");
}

constexpr int NT = 128, CH = 256, NB = 7;

template <int MODE, bool WRITE>
__global__ void __launch_bounds__(NT, 4) kern(Slot* sl, int n, int reps, long long* cyc, int* bad) {
  __shared__ alignas(16) Slot stage[CH * NB];
  __shared__ unsigned long long smb[8];
  __shared__ unsigned long long acc;
  Slot* s = sl + (size_t)blockIdx.x * n;
  const int tid = threadIdx.x;
  long long tot = 0;
  int nbad = 0;
  for (int r = 0; r < reps; r++) {
    /* generic stores: slots, and garbage into the staging bytes */
    const int rw = WRITE ? r : 0; /* WRITE: fresh generic stores every rep; else only before rep 0 */
    if (WRITE || r == 0)
      for (int j = tid; j < n; j += NT) {
        s[j].tp = (double)(rw * 100000 + j);
        s[j].meta = rw * 7 + j;
      }
    for (int j = tid; j < CH * NB; j += NT) stage[j].meta = -12345;
    if (tid == 0) acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    unsigned long long sum = 0;
    if (MODE == 0) {
      asm volatile("fence.proxy.async;" ::: "memory");
      if (tid == 0) {
        for (int b = 0; b < NB; b++) mbar_init(&smb[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
      __syncthreads();
      for (int r0 = 0, round = 0; r0 < n; r0 += CH * NB, round++) {
        if (round > 0) {
          asm volatile("fence.proxy.async;" ::: "memory");
          __syncthreads();
        }
        if (tid == 0)
          for (int b = 0; b < NB; b++) {
            const int c0 = r0 + b * CH;
            if (c0 >= n) break;
            const unsigned bytes = (unsigned)((n - c0 < CH ? n - c0 : CH) * 16);
            expect_tx(&smb[b], bytes);
            bulk(&stage[b * CH], &s[c0], bytes, &smb[b]);
          }
        for (int b = 0; b < NB; b++) {
          const int c0 = r0 + b * CH;
          if (c0 >= n) break;
          const int cnt = n - c0 < CH ? n - c0 : CH;
          mwait(&smb[b], (unsigned)(round & 1));
          for (int j = tid; j < cnt; j += NT) {
            const Slot v = stage[b * CH + j];
            const int gj = c0 + j;
            if (v.tp != (double)(rw * 100000 + gj) || v.meta != rw * 7 + gj) nbad++;
            sum += (unsigned long long)v.meta;
          }
        }
      }
    } else {
      for (int j = tid; j < n; j += NT) {
        const Slot v = s[j];
        if (v.tp != (double)(rw * 100000 + j) || v.meta != rw * 7 + j) nbad++;
        sum += (unsigned long long)v.meta;
      }
    }
    atomicAdd(&acc, sum);
    __syncthreads();
    tot += clock64() - t0;
  }
  if (tid == 0) cyc[blockIdx.x] = tot / reps;
  if (nbad) atomicAdd(bad, nbad);
}

int main() {
  const int blocks = 512, n = 2500, reps = 20;
  Slot* sl;
  long long* cyc;
  int* bad;
  cudaMalloc(&sl, sizeof(Slot) * (size_t)blocks * n);
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  cudaMallocManaged(&bad, sizeof(int));
  long long h[512];
  for (int mode = 0; mode < 4; mode++) {
    *bad = 0;
    if (mode == 0) kern<0, true><<<blocks, NT>>>(sl, n, reps, cyc, bad);
    if (mode == 1) kern<1, true><<<blocks, NT>>>(sl, n, reps, cyc, bad);
    if (mode == 2) kern<0, false><<<blocks, NT>>>(sl, n, reps, cyc, bad);
    if (mode == 3) kern<1, false><<<blocks, NT>>>(sl, n, reps, cyc, bad);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < blocks; i++) m += h[i];
    const char* nm[4] = {"bulk after stores", "ld after stores", "bulk resident", "ld resident"};
    printf("mode %s: err=%s bad=%d mean cycles per sweep %.0f\n", nm[mode], cudaGetErrorString(e), *bad, m / blocks);
  }
  return 0;
}
