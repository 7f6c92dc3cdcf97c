// Microbenchmark of the agent-tick sweep in isolation (not product code):
// CTAs of 128 threads, each sweeping its own scenario's 16-byte alive slots
// (f64 throughput, f32 next time, meta) with a per-instance shared-memory
// min and due collection, like engine_core.h job_sweep.  Prints cycles per
// sweep for a few variants.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct alignas(16) Slot { double tp; float nx; int meta; };

__device__ __forceinline__ void ldslot(const Slot* p, double& tp, float& nx, int& m) {
  unsigned long long lo, hi;
  asm volatile("ld.global.v2.b64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(p));
  tp = __longlong_as_double((long long)lo); nx = __int_as_float((int)(unsigned)hi); m = (int)(hi >> 32);
}

__device__ unsigned long long g_tmin[512 * 16];

template <int U, int MODE>
__global__ void __launch_bounds__(128, 4) sweep(const Slot* sl, int n, int reps, double bound, long long* out, int* dueout) {
  unsigned long long* gt = g_tmin + blockIdx.x * 16;
  __shared__ unsigned long long tmin[16];
  __shared__ int total;
  __shared__ int due[256];
  __shared__ unsigned long long wmin[4][16];
  __shared__ unsigned fmin[16];
  const Slot* s = sl + (size_t)blockIdx.x * n;
  long long cyc = 0;
  for (int r = 0; r < reps; r++) {
    if (threadIdx.x < 16) { tmin[threadIdx.x] = 0x7ff0000000000000ull; fmin[threadIdx.x] = 0x7f800000u; }
    if (threadIdx.x < 64) wmin[threadIdx.x >> 4][threadIdx.x & 15] = 0x7ff0000000000000ull;
    if (MODE == 6 && threadIdx.x < 16) gt[threadIdx.x] = 0x7ff0000000000000ull;
    if (threadIdx.x == 0) total = 0;
    __syncthreads();
    long long t0 = clock64();
    double tp[U], tp2[U]; float nx[U], nx2[U]; int mt[U], mt2[U];
#pragma unroll
    for (int u = 0; u < U; u++) { int j = u * 128 + threadIdx.x; mt[u] = -1; if (j < n) ldslot(&s[j], tp[u], nx[u], mt[u]); }
    for (int base = 0; base < n; base += 128 * U) {
      const int nb = base + 128 * U;
#pragma unroll
      for (int u = 0; u < U; u++) { int j = nb + u * 128 + threadIdx.x; mt2[u] = -1; if (j < n) ldslot(&s[j], tp2[u], nx2[u], mt2[u]); }
#pragma unroll
      for (int u = 0; u < U; u++) {
        if (mt[u] < 0) continue;
        if (MODE == 7) { /* guards read for the whole round first (independent LDS), then the rare CAS */
        unsigned long long gv[U], bb[U];
        int ii[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
          ii[u] = mt[u] & 15;
          bb[u] = mt[u] >= 0 ? (unsigned long long)__double_as_longlong(tp[u]) : ~0ull;
          gv[u] = tmin[ii[u]];
        }
#pragma unroll
        for (int u = 0; u < U; u++)
          if (bb[u] < gv[u]) atomicMin(&tmin[ii[u]], bb[u]);
      }
      if (MODE == 3) { if (((mt[u] >> 7) & 7) > 0 && (double)nx[u] < bound) { int pos = atomicAdd(&total, 1); if (pos < 256) due[pos] = mt[u] >> 10; } continue; }
        if (((mt[u] >> 7) & 7) > 0 && (double)nx[u] < bound) {
          int pos = atomicAdd(&total, 1);
          if (pos < 256) due[pos] = mt[u] >> 10;
        }
        unsigned long long b = (unsigned long long)__double_as_longlong(tp[u]);
        int i = mt[u] & 15;
        if (MODE == 0) { if (b < tmin[i]) atomicMin(&tmin[i], b); }
        else if (MODE == 1) { if (b < tmin[i]) tmin[i] = b; }
        else if (MODE == 4) { /* per-warp private copies */
          unsigned long long* tw = wmin[threadIdx.x >> 5];
          if (b < tw[i]) atomicMin(&tw[i], b);
        } else if (MODE == 6) { /* fire-and-forget 64-bit min in L2 */
          asm volatile("red.relaxed.gpu.global.min.u64 [%0], %1;" ::"l"(gt + i), "l"(b) : "memory");
        } else if (MODE == 5) { /* f32 round-down key: native 32-bit min, 64-bit CAS only for candidates */
          const unsigned f = (unsigned)__float_as_int(__double2float_rd(tp[u]));
          if (f <= fmin[i]) {
            const unsigned old = atomicMin(&fmin[i], f);
            if (f <= old && b < tmin[i]) atomicMin(&tmin[i], b);
          }
        }
      }
      if (MODE == 7) { /* guards read for the whole round first (independent LDS), then the rare CAS */
        unsigned long long gv[U], bb[U];
        int ii[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
          ii[u] = mt[u] & 15;
          bb[u] = mt[u] >= 0 ? (unsigned long long)__double_as_longlong(tp[u]) : ~0ull;
          gv[u] = tmin[ii[u]];
        }
#pragma unroll
        for (int u = 0; u < U; u++)
          if (bb[u] < gv[u]) atomicMin(&tmin[ii[u]], bb[u]);
      }
      if (MODE == 3) { /* warp-aggregated: group lanes by instance, redux min on hi then lo */
#pragma unroll
        for (int u = 0; u < U; u++) {
          const bool ok = mt[u] >= 0;
          const unsigned long long b = ok ? (unsigned long long)__double_as_longlong(tp[u]) : ~0ull;
          const int i = ok ? (mt[u] & 15) : 16;
          const unsigned peers = __match_any_sync(0xffffffffu, i);
          const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
          const unsigned mh = __reduce_min_sync(peers, hi);
          const unsigned sub = __ballot_sync(0xffffffffu, hi == mh) & peers;
          unsigned ml = 0xffffffffu;
          if (hi == mh) ml = __reduce_min_sync(sub, lo);
          const int lead = __ffs(peers) - 1;
          if ((threadIdx.x & 31) == lead && ok) {
            const unsigned long long m = ((unsigned long long)mh << 32) | ml;
            if (m < tmin[i]) atomicMin(&tmin[i], m);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; u++) { mt[u] = mt2[u]; tp[u] = tp2[u]; nx[u] = nx2[u]; }
    }
    __syncthreads();
    if (MODE == 6 && threadIdx.x < 16) {
      unsigned long long v;
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(gt + threadIdx.x));
      tmin[threadIdx.x] = v;
    }
    __syncthreads();
    cyc += clock64() - t0;
  }
  if (threadIdx.x == 0) { out[blockIdx.x] = cyc / reps; dueout[blockIdx.x] = total + (int)(tmin[0] & 1); }
}

int main() {
  const int nblk = 512, n = 2700, reps = 200;
  Slot* h = new Slot[(size_t)nblk * n];
  unsigned x = 12345;
  for (size_t k = 0; k < (size_t)nblk * n; k++) {
    x = x * 1664525u + 1013904223u;
    h[k].tp = 5.0 + (x % 100000) * 0.001;
    h[k].nx = (float)(100.0 + (x >> 8) % 3000 * 0.5);
    int prio = (x >> 3) % 3;
    h[k].meta = ((x >> 5) % 16) | (prio << 7) | ((int)(k % n) << 10);
  }
  Slot* d; long long* o; int* du;
  cudaMalloc(&d, sizeof(Slot) * nblk * n); cudaMalloc(&o, 8 * nblk); cudaMalloc(&du, 4 * nblk);
  cudaMemcpy(d, h, sizeof(Slot) * nblk * n, cudaMemcpyHostToDevice);
  long long* ho = new long long[nblk];
  auto run = [&](const char* name, auto kern) {
    kern<<<nblk, 128>>>(d, n, reps, 102.0, o, du);
    cudaDeviceSynchronize();
    cudaMemcpy(ho, o, 8 * nblk, cudaMemcpyDeviceToHost);
    double m = 0; for (int b = 0; b < nblk; b++) m += ho[b]; m /= nblk;
    printf("%-28s %8.0f cycles/sweep (%d slots, %d CTAs)\n", name, m, n, nblk);
  };
  run("U=2 atomic", sweep<2, 0>); run("U=2 racy", sweep<2, 1>); run("U=2 no-min", sweep<2, 2>);
run("U=2 per-warp copies", sweep<2, 4>); run("U=2 f32 key", sweep<2, 5>);
  run("U=2 batched guards", sweep<2, 7>); run("U=4 batched guards", sweep<4, 7>); run("U=8 batched guards", sweep<8, 7>); run("U=4 no-min", sweep<4, 2>);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
