/*
 * unit_ops.cu — batched policy/model kernels and per-scenario statistics.
 *
 *   asb_select_level_batch  select_frequency_level   controller.py:81-86
 *   asb_service_time_batch  service_time             instance.py:184-204
 *   asb_assign_batch        assign_agent / route_least_loaded  router.py:75-94,142-151
 *   asb_reassign_batch      maybe_reassign           router.py:97-128
 *   asb_scenario_stats      SystemMetrics            engine.py:632-655, metrics.py:49-69
 *   asb_reduce_stats        cross-scenario stats vector (allreduced over ranks)
 *
 * All element-wise kernels are grid-stride with 128-bit friendly SoA inputs;
 * the router kernels give one warp per usage vector (lexicographic argmin by
 * warp shuffle).  Stats: one CTA per scenario, nearest-rank P5 by an 8-pass
 * radix select over the IEEE bit patterns of the non-negative throughputs.
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/agentsim_b200.h"

#define FULLMASK 0xffffffffu

namespace {

inline int grid_for(int64_t n, int threads) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t b = (n + threads - 1) / threads;
  int64_t cap = (int64_t)sms * 8;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

__global__ void select_level_kernel(const double* __restrict__ usage, const double* __restrict__ capacity,
                                    const int32_t* __restrict__ num_levels, const double* __restrict__ alpha,
                                    int32_t* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    /* usage and capacity are floats in the reference's signature */
    double ac = alpha[i] * capacity[i];
    int L = num_levels[i];
    double u = usage[i];
    out[i] = u >= ac ? L : (int)floor(u / ac * (double)(L - 1)) + 1;
  }
}

__global__ void service_time_kernel(const int32_t* __restrict__ prefill, const int32_t* __restrict__ decode,
                                    const double* __restrict__ pr, const double* __restrict__ dr,
                                    const int32_t* __restrict__ concurrent, const int32_t* __restrict__ thrashing,
                                    double interference, double thrash_factor, double* __restrict__ out,
                                    int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double base = (double)prefill[i] / pr[i] + (double)decode[i] / dr[i];
    int extra = concurrent[i] - 1 > 0 ? concurrent[i] - 1 : 0;
    double factor = 1.0 + interference * (double)extra;
    if (thrashing[i]) factor *= thrash_factor;
    out[i] = base * factor;
  }
}

/* warp argmin of (usage, id) over ids 1..m with an optional candidate mask */
__device__ __forceinline__ void warp_argmin(double& bu, int& bi) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ou = __shfl_xor_sync(FULLMASK, bu, o);
    int oi = __shfl_xor_sync(FULLMASK, bi, o);
    bool take = oi > 0 && (bi == 0 || ou < bu || (ou == bu && oi < bi));
    if (take) {
      bu = ou;
      bi = oi;
    }
  }
}

__global__ void assign_kernel(const double* __restrict__ usages, const int32_t* __restrict__ m, int max_m,
                              int64_t capacity, double theta, int policy, int32_t* __restrict__ out, int64_t n) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    const int mr = m[r];
    const double* u = usages + r * max_m;
    const double threshold = theta * (double)capacity;
    double bu = 0;
    int bi = 0;
    int light = 0x7fffffff;
    for (int i = lane; i < mr; i += 32) {
      double v = u[i];
      if (policy == ASB_POLICY_CONTEXT_AWARE && v < threshold && i + 1 < light) light = i + 1;
      if (bi == 0 || v < bu) {
        bu = v;
        bi = i + 1;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) light = min(light, __shfl_xor_sync(FULLMASK, light, o));
    warp_argmin(bu, bi);
    if (lane == 0) out[r] = (policy == ASB_POLICY_CONTEXT_AWARE && light != 0x7fffffff) ? light : bi;
  }
}

__global__ void reassign_kernel(const double* __restrict__ usages, const int32_t* __restrict__ m, int max_m,
                                const int32_t* __restrict__ current, int32_t* __restrict__ counters, int interval,
                                double ratio, int include_idle, int reset_only, int32_t* __restrict__ out,
                                int64_t n) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    const int mr = m[r];
    const int cur = current[r];
    const double* u = usages + r * max_m;
    int counter = counters[r] + 1;
    int target = 0;
    if (counter >= interval) {
      double bu = 0;
      int bi = 0;
      for (int i = lane; i < mr; i += 32) {
        double v = u[i];
        if (!include_idle && !(v > 0 || i + 1 == cur)) continue;
        if (bi == 0 || v < bu) {
          bu = v;
          bi = i + 1;
        }
      }
      warp_argmin(bu, bi);
      if (bi && bi != cur && u[cur - 1] >= ratio * u[bi - 1]) target = bi;
      if (target || !reset_only) counter = 0;
    }
    if (lane == 0) {
      counters[r] = counter;
      out[r] = target;
    }
  }
}

/* K0 stand-alone: segmented min of decode_total/llm_time over agents with
 * llm_time > 0 (running_throughput/min_throughput, controller.py:89-103) */
__global__ void min_tp_init_kernel(unsigned long long* bits, int n_seg) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_seg; i += gridDim.x * blockDim.x)
    bits[i] = 0x7ff0000000000000ull;
}
__global__ void min_tp_kernel(const int64_t* __restrict__ dec, const double* __restrict__ llm,
                              const int32_t* __restrict__ seg, int64_t n, unsigned long long* bits) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double l = llm[i];
    if (!(l > 0.0)) continue;
    double tp = (double)dec[i] / l;
    atomicMin(&bits[seg[i]], (unsigned long long)__double_as_longlong(tp));
  }
}
__global__ void min_tp_final_kernel(const unsigned long long* bits, double* out, int n_seg) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_seg; i += gridDim.x * blockDim.x)
    out[i] = bits[i] == 0x7ff0000000000000ull ? __longlong_as_double(0x7ff8000000000000ll)
                                               : __longlong_as_double((long long)bits[i]);
}

/* Python >= 3.12 builtin sum() over floats (int start 0, Neumaier
 * compensation), as _build_result sums instance energy / thrash time
 * (engine.py:632-633). */
__device__ double py_sum(const double* x, int n) {
  if (n == 0) return 0.0;
  double f = 0.0 + x[0], c = 0.0;
  for (int i = 1; i < n; i++) {
    double t = f + x[i];
    if (fabs(f) >= fabs(x[i]))
      c += (f - t) + x[i];
    else
      c += (x[i] - t) + f;
    f = t;
  }
  if (c != 0.0 && isfinite(c)) f += c;
  return f;
}

/* one CTA per scenario */
__global__ void stats_kernel(const AsbScenario* __restrict__ scen, int n_scen, AsbOutputs out,
                             AsbStats* __restrict__ stats) {
  const int s = blockIdx.x;
  if (s >= n_scen) return;
  const AsbScenario& sc = scen[s];
  const int64_t a0 = out.agent_off[s], a1 = out.agent_off[s + 1];
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ unsigned int hist[256];
  __shared__ unsigned long long s_prefix;
  __shared__ long long s_n, s_met, s_rank;
  __shared__ long long red_n[32], red_m[32];
  /* count completed-with-throughput agents and SLO hits (metrics.py:49-58) */
  long long n = 0, met = 0;
  for (int64_t a = a0 + tid; a < a1; a += nt) {
    if (out.phase[a] != ASB_PHASE_DONE || !(out.llm_time[a] > 0.0)) continue;
    double tp = (double)out.decode_total[a] / out.llm_time[a];
    n++;
    if (tp >= sc.slo_target) met++;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    n += __shfl_xor_sync(FULLMASK, n, o);
    met += __shfl_xor_sync(FULLMASK, met, o);
  }
  if ((tid & 31) == 0) {
    red_n[tid >> 5] = n;
    red_m[tid >> 5] = met;
  }
  __syncthreads();
  if (tid == 0) {
    long long tn = 0, tm = 0;
    for (int w = 0; w < (nt + 31) / 32; w++) {
      tn += red_n[w];
      tm += red_m[w];
    }
    s_n = tn;
    s_met = tm;
    s_prefix = 0;
    /* nearest rank: ceil(0.05 * n), metrics.py:61-69 */
    s_rank = tn ? (long long)ceil(0.05 * (double)tn) : 0;
  }
  __syncthreads();
  const long long total = s_n;
  double p5 = __longlong_as_double(0x7ff8000000000000ll);
  if (total > 0) {
    /* radix select of the s_rank-th smallest bit pattern, 8 bits per pass */
    long long k = s_rank; /* 1-based */
    unsigned long long prefix = 0;
    for (int pass = 7; pass >= 0; pass--) {
      for (int b = tid; b < 256; b += nt) hist[b] = 0;
      __syncthreads();
      const int shift = pass * 8;
      const unsigned long long hmask = pass == 7 ? 0ull : (~0ull << (shift + 8));
      for (int64_t a = a0 + tid; a < a1; a += nt) {
        if (out.phase[a] != ASB_PHASE_DONE || !(out.llm_time[a] > 0.0)) continue;
        unsigned long long b = (unsigned long long)__double_as_longlong((double)out.decode_total[a] / out.llm_time[a]);
        if ((b & hmask) != prefix) continue;
        atomicAdd(&hist[(b >> shift) & 255], 1u);
      }
      __syncthreads();
      if (tid == 0) {
        long long run = 0;
        int digit = 0;
        for (; digit < 256; digit++) {
          if (run + hist[digit] >= k) break;
          run += hist[digit];
        }
        k -= run;
        s_rank = k;
        s_prefix = prefix | ((unsigned long long)digit << shift);
      }
      __syncthreads();
      prefix = s_prefix;
      k = s_rank;
    }
    p5 = __longlong_as_double((long long)prefix);
  }
  if (tid == 0) {
    AsbStats st;
    const int64_t i0 = out.inst_off[s];
    const double e = py_sum(out.energy + i0, sc.n_instances);
    const double th = py_sum(out.thrash_time + i0, sc.n_instances);
    const double T = sc.sim_duration;
    st.slo_met = s_met;
    st.n_completed_with_tp = total;
    st.slo_attainment = total ? (double)s_met / (double)total : __longlong_as_double(0x7ff8000000000000ll);
    st.p5_throughput = p5;
    st.job_throughput = (double)out.counters[(int64_t)s * ASB_NCOUNTERS + ASB_CTR_COMPLETED] / T;
    st.average_power = e / T;
    st.energy = e;
    st.thrash_fraction = th / (T * (double)sc.n_instances);
    stats[s] = st;
  }
}

/* deterministic fixed-order fold of per-scenario rows into ASB_NRED doubles */
__global__ void reduce_stats_kernel(const AsbStats* __restrict__ stats, const int64_t* __restrict__ counters,
                                    int n_scen, double* __restrict__ red) {
  __shared__ double part[ASB_NRED][256];
  const int tid = threadIdx.x;
  double acc[ASB_NRED];
  for (int j = 0; j < ASB_NRED; j++) acc[j] = 0.0;
  for (int s = tid; s < n_scen; s += blockDim.x) {
    const int64_t* c = counters + (int64_t)s * ASB_NCOUNTERS;
    acc[ASB_RED_ENERGY] += stats[s].energy;
    acc[ASB_RED_THRASH_FRAC] += stats[s].thrash_fraction;
    acc[ASB_RED_COMPLETED] += (double)c[ASB_CTR_COMPLETED];
    acc[ASB_RED_SLO_MET] += (double)stats[s].slo_met;
    acc[ASB_RED_TICKS] += (double)c[ASB_CTR_TICKS];
    acc[ASB_RED_THRASH_FLIPS] += (double)c[ASB_CTR_THRASH_FLIPS];
    acc[ASB_RED_MIGRATIONS] += (double)c[ASB_CTR_MIGRATIONS];
    acc[ASB_RED_TURNS] += (double)c[ASB_CTR_TURNS];
  }
  for (int j = 0; j < ASB_NRED; j++) part[j][tid] = acc[j];
  __syncthreads();
  if (tid < ASB_NRED) {
    double t = 0.0;
    for (int i = 0; i < (int)blockDim.x; i++) t += part[tid][i];
    red[tid] = t;
  }
}

/* regime_classify (metrics.py:72-109), one warp per scenario, a lane per
 * instance (groups of 32 instances).  Rows are read in chunks of 32 (one
 * coalesced row per lane) and broadcast lane by lane; each lane follows its
 * instance's points.  Pass 0 counts every instance's spans, pass 1 writes
 * them at the exclusive-scan offsets and sums the thrashing durations. */
struct RegimeLane {
  bool has_prev, has_span;
  double prev_t, prev_u;
  double s0, s1;
  int flag;
  long long n;    /* spans emitted so far */
  double f, c;    /* Python float sum() of thrashing durations (Neumaier) */
  bool sum_started;
};

__device__ void regime_emit(RegimeLane& L, AsbRegimeSpan* out, int iid) {
  if (!L.has_span) return;
  if (out) {
    AsbRegimeSpan sp;
    sp.start = L.s0;
    sp.end = L.s1;
    sp.instance_id = iid;
    sp.thrashing = L.flag;
    out[L.n] = sp;
  }
  if (L.flag) {
    const double x = L.s1 - L.s0;
    if (!L.sum_started) {
      L.f = 0.0 + x;
      L.c = 0.0;
      L.sum_started = true;
    } else {
      const double t = L.f + x;
      if (fabs(L.f) >= fabs(x))
        L.c += (L.f - t) + x;
      else
        L.c += (x - t) + L.f;
      L.f = t;
    }
  }
  L.n++;
}

/* add(start, end, flag) of the reference: skip empty spans, merge with the
 * previous span when it has the same flag and ends where this one starts */
__device__ void regime_add(RegimeLane& L, AsbRegimeSpan* out, int iid, double a, double b, int flag) {
  if (b <= a) return;
  if (L.has_span && L.flag == flag && L.s1 == a) {
    L.s1 = b;
    return;
  }
  regime_emit(L, out, iid);
  L.has_span = true;
  L.s0 = a;
  L.s1 = b;
  L.flag = flag;
}

__global__ void regime_kernel(const AsbTimeseriesRow* __restrict__ rows, const int64_t* __restrict__ ts_off,
                              const int64_t* __restrict__ ts_count, int n_scen, const int32_t* __restrict__ n_inst,
                              const double* __restrict__ capacity, const double* __restrict__ window,
                              const int64_t* __restrict__ span_off, AsbRegimeSpan* __restrict__ spans,
                              int64_t* __restrict__ span_count, double* __restrict__ frac, int32_t* __restrict__ status) {
  const int s = blockIdx.x;
  if (s >= n_scen) return;
  const int lane = threadIdx.x;
  const AsbTimeseriesRow* R = rows + ts_off[s];
  const long long nr = ts_count[s];
  const int M = n_inst[s];
  const double cap = capacity[s], W = window[s];
  const long long room = span_off[s + 1] - span_off[s];
  long long base = 0;   /* spans of the instances before this group */
  double total = 0.0;   /* thrash_total, instances in id order */
  int bad = 0;
  for (int g0 = 0; g0 < M; g0 += 32) {
    const int iid = g0 + lane + 1;
    long long my_off = 0;
    for (int pass = 0; pass < 2; pass++) {
      RegimeLane L;
      L.has_prev = L.has_span = L.sum_started = false;
      L.n = 0;
      L.f = L.c = 0.0;
      AsbRegimeSpan* out = pass == 1 && iid <= M ? spans + span_off[s] + base + my_off : nullptr;
      for (long long r0 = 0; r0 < nr; r0 += 32) {
        const long long r = r0 + lane;
        double t = 0.0, u = 0.0;
        int id = 0;
        if (r < nr) {
          t = R[r].time;
          u = (double)R[r].context_usage;
          id = R[r].instance_id;
        }
        const int k_end = (int)(nr - r0 < 32 ? nr - r0 : 32);
        for (int k = 0; k < k_end; k++) {
          const int idk = __shfl_sync(FULLMASK, id, k);
          const double tk = __shfl_sync(FULLMASK, t, k);
          const double uk = __shfl_sync(FULLMASK, u, k);
          if (idk != iid) continue;
          if (L.has_prev) {
            const double a = L.prev_t < W ? L.prev_t : W, b = tk < W ? tk : W;
            regime_add(L, out, iid, a, b, L.prev_u > cap ? 1 : 0);
          }
          L.has_prev = true;
          L.prev_t = tk;
          L.prev_u = uk;
        }
      }
      if (iid <= M && L.has_prev && L.prev_t < W) regime_add(L, out, iid, L.prev_t, W, L.prev_u > cap ? 1 : 0);
      if (iid <= M) regime_emit(L, out, iid);
      if (pass == 0) {
        /* exclusive scan of the group's span counts */
        long long c = iid <= M ? L.n : 0, inc = c;
        for (int o = 1; o < 32; o <<= 1) {
          const long long v = __shfl_up_sync(FULLMASK, inc, o);
          if (lane >= o) inc += v;
        }
        my_off = inc - c;
        if (base + __shfl_sync(FULLMASK, inc, 31) > room) bad = -1;
        bad = __shfl_sync(FULLMASK, bad, 0);
        if (bad) break;
      } else {
        /* sum() of an instance with no thrashing span is int 0 */
        double inst_sum = 0.0;
        if (L.sum_started) inst_sum = (L.c != 0.0 && isfinite(L.c)) ? L.f + L.c : L.f;
        for (int k = 0; k < 32 && g0 + k < M; k++) total += __shfl_sync(FULLMASK, inst_sum, k);
        base += __shfl_sync(FULLMASK, my_off + (iid <= M ? L.n : 0), 31);
      }
    }
    if (bad) break;
  }
  /* coverage of the window start (metrics.py:88-91): every instance
   * 1..M has points and its first is at t <= 0 (the engine writes a forced
   * row per instance at t = 0, engine.py:576-579) */
  if (!bad) {
    for (int g0 = 0; g0 < M; g0 += 32) {
      const int iid = g0 + lane + 1;
      double first = __longlong_as_double(0x7ff0000000000000ll);
      bool found = false;
      for (long long r0 = 0; r0 < nr && iid <= M && !found; r0 += 1) {
        if (R[r0].instance_id == iid) {
          first = R[r0].time;
          found = true;
        }
      }
      const unsigned m = __ballot_sync(FULLMASK, iid <= M && (!found || first > 0.0));
      if (m && !bad) bad = g0 + __ffs(m);
    }
  }
  if (lane == 0) {
    status[s] = bad;
    span_count[s] = bad ? 0 : base;
    frac[s] = total / (W * (double)M);
  }
}

}  // namespace

extern "C" {

int asb_select_level_batch(const double* usage, const double* capacity, const int32_t* num_levels,
                           const double* alpha, int32_t* level_out, int64_t n, void* stream) {
  if (n < 0) return ASB_ERR_ARG;
  if (n == 0) return ASB_OK;
  select_level_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(usage, capacity, num_levels, alpha,
                                                                           level_out, n);
  return cudaGetLastError() == cudaSuccess ? ASB_OK : ASB_ERR_LAUNCH;
}

int asb_service_time_batch(const int32_t* prefill, const int32_t* decode, const double* prefill_rate,
                           const double* decode_rate, const int32_t* concurrent, const int32_t* thrashing,
                           double interference, double thrash_factor, double* out, int64_t n, void* stream) {
  if (n < 0) return ASB_ERR_ARG;
  if (n == 0) return ASB_OK;
  service_time_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
      prefill, decode, prefill_rate, decode_rate, concurrent, thrashing, interference, thrash_factor, out, n);
  return cudaGetLastError() == cudaSuccess ? ASB_OK : ASB_ERR_LAUNCH;
}

int asb_assign_batch(const double* usages, const int32_t* m, int32_t max_m, int64_t capacity,
                     double consolidation_threshold, int32_t policy, int32_t* target_out, int64_t n,
                     void* stream) {
  if (n < 0 || max_m < 1) return ASB_ERR_ARG;
  if (policy != ASB_POLICY_CONTEXT_AWARE && policy != ASB_POLICY_LEAST_LOADED) return ASB_ERR_ARG;
  if (n == 0) return ASB_OK;
  assign_kernel<<<grid_for(n * 32, 256), 256, 0, (cudaStream_t)stream>>>(
      usages, m, max_m, capacity, consolidation_threshold, policy, target_out, n);
  return cudaGetLastError() == cudaSuccess ? ASB_OK : ASB_ERR_LAUNCH;
}

int asb_reassign_batch(const double* usages, const int32_t* m, int32_t max_m, const int32_t* current,
                       int32_t* counters, int32_t reassign_interval, double imbalance_ratio, int32_t include_idle,
                       int32_t reset_only, int32_t* target_out, int64_t n, void* stream) {
  if (n < 0 || max_m < 1) return ASB_ERR_ARG;
  if (n == 0) return ASB_OK;
  reassign_kernel<<<grid_for(n * 32, 256), 256, 0, (cudaStream_t)stream>>>(
      usages, m, max_m, current, counters, reassign_interval, imbalance_ratio, include_idle, reset_only,
      target_out, n);
  return cudaGetLastError() == cudaSuccess ? ASB_OK : ASB_ERR_LAUNCH;
}

int asb_min_throughput_batch(const int64_t* decode_total, const double* llm_time, const int32_t* segment,
                             int64_t n, int32_t n_seg, double* scratch_bits, double* min_out, void* stream) {
  if (n < 0 || n_seg < 1) return ASB_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* bits = (unsigned long long*)scratch_bits;
  min_tp_init_kernel<<<grid_for(n_seg, 256), 256, 0, st>>>(bits, n_seg);
  if (n > 0) min_tp_kernel<<<grid_for(n, 256), 256, 0, st>>>(decode_total, llm_time, segment, n, bits);
  min_tp_final_kernel<<<grid_for(n_seg, 256), 256, 0, st>>>(bits, min_out, n_seg);
  return cudaGetLastError() == cudaSuccess ? ASB_OK : ASB_ERR_LAUNCH;
}

int asb_scenario_stats(const AsbScenario* d_scen, int32_t n_scen, AsbOutputs out, AsbStats* d_stats,
                       void* d_workspace, size_t workspace_bytes, void* stream) {
  (void)d_workspace;
  (void)workspace_bytes;
  if (n_scen < 0) return ASB_ERR_ARG;
  if (n_scen == 0) return ASB_OK;
  stats_kernel<<<n_scen, 256, 0, (cudaStream_t)stream>>>(d_scen, n_scen, out, d_stats);
  return cudaGetLastError() == cudaSuccess ? ASB_OK : ASB_ERR_LAUNCH;
}

int asb_reduce_stats(const AsbStats* d_stats, const int64_t* d_counters, int32_t n_scen, double* d_red,
                     void* stream) {
  if (n_scen < 0) return ASB_ERR_ARG;
  reduce_stats_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(d_stats, d_counters, n_scen, d_red);
  return cudaGetLastError() == cudaSuccess ? ASB_OK : ASB_ERR_LAUNCH;
}

int asb_regime_classify(const AsbTimeseriesRow* rows, const int64_t* ts_off, const int64_t* ts_count,
                        int32_t n_scen, const int32_t* n_instances, const double* capacity, const double* window,
                        const int64_t* span_off, AsbRegimeSpan* spans, int64_t* span_count,
                        double* thrash_fraction, int32_t* status, void* stream) {
  if (n_scen < 0) return ASB_ERR_ARG;
  if (n_scen == 0) return ASB_OK;
  if (!rows || !ts_off || !ts_count || !n_instances || !capacity || !window || !span_off || !spans ||
      !span_count || !thrash_fraction || !status)
    return ASB_ERR_ARG;
  regime_kernel<<<n_scen, 32, 0, (cudaStream_t)stream>>>(rows, ts_off, ts_count, n_scen, n_instances, capacity,
                                                          window, span_off, spans, span_count, thrash_fraction,
                                                          status);
  return cudaGetLastError() == cudaSuccess ? ASB_OK : ASB_ERR_LAUNCH;
}

int asb_struct_sizes(int64_t* out4) {  /* NOLINT */
  out4[0] = (int64_t)sizeof(AsbScenario);
  out4[1] = (int64_t)sizeof(AsbTracePool);
  out4[2] = (int64_t)sizeof(AsbTablePool);
  out4[3] = (int64_t)sizeof(AsbOutputs);
  out4[4] = (int64_t)sizeof(AsbDecision);
  out4[5] = (int64_t)sizeof(AsbStats);
  out4[6] = (int64_t)sizeof(AsbTimeseriesRow);
  out4[7] = (int64_t)sizeof(AsbRegimeSpan);
  return 8;
}

}  // extern "C"
