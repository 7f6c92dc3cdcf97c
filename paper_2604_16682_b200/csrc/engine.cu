/*
 * engine.cu — sm_100a kernels behind the C ABI (include/agentsim_b200.h).
 *
 *   asb_engine_kernel : persistent, one warp per scenario, dynamic scenario
 *                       queue (heavy-tailed scenario costs), per-warp engine
 *                       state in shared memory; the engine itself is
 *                       engine_core.h instantiated with the warp team below.
 *   asb_ring_offsets  : device prefix sum of per-scenario FIFO/log sizes.
 *
 * Build: nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -O3
 * (--fmad=false: the reference is Python, which never fuses multiply-add).
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/agentsim_b200.h"

#define FULLMASK 0xffffffffu
#define EC_DEV __device__ __forceinline__
#ifndef ASB_COLD_MASK
#define ASB_COLD_MASK 7 /* 1 jobs, 2 serial handlers, 4 phases: out of line */
#endif
#define EC_COLD __device__ __noinline__
#if ASB_COLD_MASK & 1
#define EC_COLD1 __device__ __noinline__
#else
#define EC_COLD1 __device__ __forceinline__
#endif
#if ASB_COLD_MASK & 2
#define EC_COLD2 __device__ __noinline__
#else
#define EC_COLD2 __device__ __forceinline__
#endif
#if ASB_COLD_MASK & 4
#define EC_COLD3 __device__ __noinline__
#else
#define EC_COLD3 __device__ __forceinline__
#endif
#define EC_COLD4 __device__ __noinline__
#define EC_LANE ((int)(threadIdx.x & 31))
#ifndef ASB_NO_PREFETCH
#ifdef ASB_PREFETCH_L1 /* experiment: the due agents' lines into the SM's L1 instead of L2 */
#define EC_PREFETCH_L2(p) asm volatile("prefetch.global.L1 [%0];" ::"l"(p))
#else
#define EC_PREFETCH_L2(p) asm volatile("prefetch.global.L2 [%0];" ::"l"(p))
#endif
#endif
#define EC_TSIZE 32
#define EC_NAN __longlong_as_double(0x7ff8000000000000ll)
#define EC_INF __longlong_as_double(0x7ff0000000000000ll)
#define EC_INF_BITS 0x7ff0000000000000ull

EC_DEV void t_sync() { __syncwarp(); }
EC_DEV unsigned t_ballot(bool p) { return __ballot_sync(FULLMASK, p); }
EC_DEV unsigned t_lt_mask() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
EC_DEV int ec_popc(unsigned m) { return __popc(m); }
EC_DEV int ec_ffs(unsigned m) { return __ffs(m); } /* 1-based lowest set bit, 0 if none */
EC_DEV unsigned t_match_any_i(int v) { return __match_any_sync(FULLMASK, v); } /* lanes holding the same v */
EC_DEV unsigned t_redux_min_u32(unsigned v) { return __reduce_min_sync(FULLMASK, v); }
EC_DEV long long t_bcast_ll(long long v, int src) { return __shfl_sync(FULLMASK, v, src); }
/* warp collectives used at many call sites: out of line and rolled to keep
 * the hot code small (the co-resident teams of an SM share the I-cache) */
#ifndef ASB_INLINE_COLLECTIVES
#define EC_COLL __device__ __noinline__
#define EC_COLL_UNROLL _Pragma("unroll 1")
#else
#define EC_COLL EC_DEV
#define EC_COLL_UNROLL _Pragma("unroll")
#endif
EC_COLL long long t_scan_add_ll(long long v) {
EC_COLL_UNROLL
  for (int o = 1; o < 32; o <<= 1) {
    long long n = __shfl_up_sync(FULLMASK, v, o);
    if (EC_LANE >= o) v += n;
  }
  return v;
}
EC_DEV int t_scan_add_i(int v) {
EC_COLL_UNROLL
  for (int o = 1; o < 32; o <<= 1) {
    int n = __shfl_up_sync(FULLMASK, v, o);
    if (EC_LANE >= o) v += n;
  }
  return v;
}
EC_DEV int t_shfl_i(int v, int src) { return __shfl_sync(FULLMASK, v, src); }
EC_DEV int t_redux_add_i(int v) { return (int)__reduce_add_sync(FULLMASK, (unsigned)v); }
EC_COLL long long t_sum_ll(long long v) {
EC_COLL_UNROLL
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o);
  return v;
}
EC_DEV unsigned long long t_shfl_xor_ull(unsigned long long v, int o) { return __shfl_xor_sync(FULLMASK, v, o); }
EC_DEV long long t_shfl_xor_ll(long long v, int o) { return __shfl_xor_sync(FULLMASK, v, o); }
EC_DEV int t_shfl_xor_i(int v, int o) { return __shfl_xor_sync(FULLMASK, v, o); }
EC_DEV long long t_shfl_up_ll(long long v, int o) { return __shfl_up_sync(FULLMASK, v, o); }
EC_DEV int t_shfl_up_i(int v, int o) { return __shfl_up_sync(FULLMASK, v, o); }
EC_DEV void t_atomic_min_ull(unsigned long long* p, unsigned long long v) { atomicMin(p, v); }
EC_DEV int t_atomic_add_i(int* p, int v) { return atomicAdd(p, v); }
EC_DEV bool ec_isnan(double x) { return isnan(x); }
EC_DEV double ec_floor(double x) { return floor(x); }
EC_DEV unsigned long long ec_bits(double x) { return (unsigned long long)__double_as_longlong(x); }
EC_DEV double ec_from_bits(unsigned long long b) { return __longlong_as_double((long long)b); }
EC_DEV long long ec_clock() { return clock64(); }
#ifdef ASB_PROFILE_PLACEMENT
EC_DEV long long ec_smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
EC_DEV long long ec_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return (long long)t;
}
#endif
EC_DEV float ec_f32_down(double x) { return __double2float_rd(x); } /* rounded toward -inf: <= x */
#define EC_INF_F32 __int_as_float(0x7f800000)
/* a team is NT consecutive threads (NT a power of two): one team per CTA */
#define EC_TID_OF(nt) ((int)(threadIdx.x & ((nt) - 1)))
/* named CTA barriers for the fork-join team.  Each warp reconverges first
 * (__syncwarp): a warp that reaches a CTA barrier with some lanes still
 * inside the job would let the barrier complete early.  (Constant ids: a
 * computed id makes ptxas reserve all 16 barriers.) */
/* a single-warp team is its own team: a warp barrier is enough */
EC_DEV void ec_fork_begin(int nt) {
  __syncwarp();
  if (nt > 32) asm volatile("bar.sync 1, %0;" ::"r"(nt) : "memory");
}
EC_DEV void ec_fork_end(int nt) {
  __syncwarp();
  if (nt > 32) asm volatile("bar.sync 2, %0;" ::"r"(nt) : "memory");
}
EC_DEV void ec_team_barrier(int nt) {
  __syncwarp();
  if (nt > 32) asm volatile("bar.sync 3, %0;" ::"r"(nt) : "memory");
}
EC_DEV int t_atomic_min_i(int* p, int v) { return atomicMin(p, v); }
EC_COLL unsigned long long t_warp_min_ull(unsigned long long v) {
EC_COLL_UNROLL
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long x = __shfl_xor_sync(FULLMASK, v, o);
    v = x < v ? x : v;
  }
  return v;
}
/* warp min of (time bits, prio) keys */
EC_COLL void t_warp_min_key(unsigned long long& t, unsigned& p) {
EC_COLL_UNROLL
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long xt = __shfl_xor_sync(FULLMASK, t, o);
    unsigned xp = __shfl_xor_sync(FULLMASK, p, o);
    if (xt < t || (xt == t && xp < p)) {
      t = xt;
      p = xp;
    }
  }
}

#ifdef ASB_DEBUG_TRACE
__device__ long long* volatile g_asb_dbg;
#define EC_DBG(slot, value)                                                 \
  do {                                                                      \
    long long* d_ = g_asb_dbg;                                              \
    if (d_ && blockIdx.x == 0 && (threadIdx.x & 31) == 0) {                 \
      ((volatile long long*)d_)[(slot)] = (long long)(value);               \
      ((volatile long long*)d_)[32 + (slot)] += 1;                          \
      ((volatile long long*)d_)[63] = (long long)(slot) | ((long long)threadIdx.x << 32); \
      __threadfence_system();                                               \
    }                                                                       \
  } while (0)
#endif

#ifndef ASB_NO_L2_HINTS
/* the alive-slot arrays are re-read by every epoch's sweep: keep them in L2
 * (and, with ASB_L1_KEEP, in L1) */
#ifndef ASB_L1_KEEP
#define ASB_L1_KEEP ""
#endif
EC_DEV unsigned long long l2_keep() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
EC_DEV int ldk_i32(const int* p) {
  int v;
  asm volatile("ld.global" ASB_L1_KEEP ".L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(l2_keep()));
  return v;
}
EC_DEV void stk_f64(double* p, double v) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(l2_keep()) : "memory");
}
EC_DEV void stk_i32(int* p, int v) {
  asm volatile("st.global.L2::cache_hint.s32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(l2_keep()) : "memory");
}
/* a whole 16-byte alive slot in one vector load */
template <class S>
EC_DEV void ldk_slot(const S* p, double& tp, float& nx, int& meta) {
  unsigned long long lo, hi;
  asm volatile("ld.global" ASB_L1_KEEP ".L2::cache_hint.v2.b64 {%0, %1}, [%2], %3;"
               : "=l"(lo), "=l"(hi) : "l"(p), "l"(l2_keep()));
  tp = __longlong_as_double((long long)lo);
  nx = __int_as_float((int)(unsigned)hi);
  meta = (int)(unsigned)(hi >> 32);
}
/* the slot's (nx, meta) half in one 8-byte store */
template <class S>
EC_DEV void stk_ev(S* p, float nx, int meta) {
  const unsigned long long v = (unsigned long long)(unsigned)__float_as_int(nx) | ((unsigned long long)(unsigned)meta << 32);
  asm volatile("st.global.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(&p->nx), "l"(v), "l"(l2_keep()) : "memory");
}
#define EC_LDK_I32(p) ldk_i32(p)
#define EC_STK_F64(p, v) stk_f64((p), (v))
#define EC_STK_I32(p, v) stk_i32((p), (v))
#define EC_LDK_SLOT(p, tp_, nx_, mt_) ldk_slot((p), (tp_), (nx_), (mt_))
#define EC_STK_EV(p, nx_, mt_) stk_ev((p), (nx_), (mt_))
#define EC_SLOT_ACCESSORS /* the cache-hinted accessors above replace engine_core.h's defaults */
#endif

#include "engine_core.h"

namespace {

struct Workspace {
  asb::AgentHot* hot;
  asb::Slot* sl;
  double *notbefore, *pissue, *arr_t;
  int* dstamp;
  int *ring, *log;
  long long* ring_off;
  int* work;
};

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

/* carve the workspace; returns bytes used (ptrs filled when base != nullptr) */
size_t carve(unsigned char* base, int32_t n_scen, int64_t total_agents, int64_t total_ring, Workspace* w) {
  size_t off = 0;
  auto take = [&](size_t bytes) -> unsigned char* {
    unsigned char* p = base ? base + off : nullptr;
    off += align_up(bytes > 0 ? bytes : 1);
    return p;
  };
  size_t na = (size_t)(total_agents > 0 ? total_agents : 1);
  Workspace t;
  t.hot = (asb::AgentHot*)take(na * sizeof(asb::AgentHot));
  t.arr_t = (double*)take(na * 8);
  t.sl = (asb::Slot*)take(na * sizeof(asb::Slot));
  t.notbefore = (double*)take(na * 8);
  t.pissue = (double*)take(na * 8);
  t.dstamp = (int*)take(na * 4);
  t.ring = (int*)take((size_t)(total_ring > 0 ? total_ring : 1) * 4);
  t.log = (int*)take((size_t)(total_ring > 0 ? total_ring : 1) * 4);
  t.ring_off = (long long*)take((size_t)(n_scen + 1) * 8);
  t.work = (int*)take(64);
  if (w) *w = t;
  return off;
}

__global__ void ring_offsets_kernel(const AsbScenario* scen, int n_scen, const int64_t* trace_agent_off,
                                    long long* ring_off, int* work) {
  /* single block: chunked exclusive scan of n_instances * n_agents */
  __shared__ long long part[1024];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (n_scen + nt - 1) / nt;
  const int s0 = tid * per, s1 = min(n_scen, s0 + per);
  long long sum = 0;
  for (int s = s0; s < s1; s++) {
    const AsbScenario& sc = scen[s];
    sum += (long long)sc.n_instances * (trace_agent_off[sc.trace_id + 1] - trace_agent_off[sc.trace_id]);
  }
  part[tid] = sum;
  __syncthreads();
  if (tid == 0) {
    long long run = 0;
    for (int i = 0; i < nt; i++) {
      long long v = part[i];
      part[i] = run;
      run += v;
    }
    ring_off[n_scen] = run;
    *work = 0;
  }
  __syncthreads();
  long long run = part[tid];
  for (int s = s0; s < s1; s++) {
    ring_off[s] = run;
    const AsbScenario& sc = scen[s];
    run += (long long)sc.n_instances * (trace_agent_off[sc.trace_id + 1] - trace_agent_off[sc.trace_id]);
  }
}

template <int MAXM, int RCAP, int DCAP, int ACAP, int NT, int LMAX>
/* min blocks per SM: 4-warp teams 4 per SM; single-warp teams 16 per SM,
 * i.e. <= 128 registers, so that 14 of them fit next to their shared memory
 * (C3's 2,048 scenarios in one wave of 148 x 14) */
#ifndef EC_QUAD_MINB
#define EC_QUAD_MINB 4 /* 4-warp teams per SM the register budget is cut for */
#endif
__global__ void __launch_bounds__(NT, NT <= 32 ? 16 : (NT <= 64 ? 8 : (NT <= 128 ? EC_QUAD_MINB : 1)))
    asb_engine_kernel(const AsbScenario* __restrict__ scen, int n_scen, AsbTracePool tp, AsbTablePool tb,
                      AsbOutputs out, Workspace ws) {
  /* one CTA = one scenario team: warp 0 runs the engine, warps 1.. are
   * helpers joining the slot sweeps, speculation, rank sort and apply */
  using W = asb::WS<MAXM, RCAP, DCAP, ACAP, NT, LMAX>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  W* w = reinterpret_cast<W*>(smem_raw);
  if (threadIdx.x >= 32) {
    asb::helper_loop(w);
    return;
  }
  for (;;) {
    int s = 0;
    if (EC_LANE == 0) s = atomicAdd(ws.work, 1);
    s = __shfl_sync(FULLMASK, s, 0);
    if (s >= n_scen) break;
    /* scenario parameters and frequency table into shared memory */
    {
      const int* src = reinterpret_cast<const int*>(&scen[s]);
      int* dst = reinterpret_cast<int*>(&w->sc);
      for (int j = EC_LANE; j < (int)(sizeof(AsbScenario) / 4); j += 32) dst[j] = src[j];
    }
    __syncwarp();
    const AsbScenario& sc = w->sc;
    {
      const long long t0 = tb.table_off[sc.table_id];
      for (int l = EC_LANE; l < sc.n_levels; l += 32) {
        w->pr[l] = tb.prefill_rate[t0 + l];
        w->dr[l] = tb.decode_rate[t0 + l];
        w->act[l] = tb.active_power[t0 + l];
        w->idle[l] = tb.idle_power[t0 + l];
      }
    }
    asb::GP g;
    const long long a0 = tp.trace_agent_off[sc.trace_id];
    const int A = (int)(tp.trace_agent_off[sc.trace_id + 1] - a0);
    const long long oa = out.agent_off[s], oi = out.inst_off[s];
    g.arrival = tp.arrival + a0;
    g.aturn = reinterpret_cast<const long long*>(tp.agent_turn_off) + a0;
    g.prefill = tp.prefill;
    g.decode = tp.decode;
    g.tool = tp.tool;
    g.arr_order = tp.arrival_order + a0;
    g.arr_t = ws.arr_t + oa;
    g.turn_base = tp.trace_turn_off[sc.trace_id];
    g.H = ws.hot + oa;
    g.ctime = out.completion_time + oa;
    g.notbefore = ws.notbefore + oa;
    g.pissue = ws.pissue + oa;
    g.rank = out.arrival_rank + oa;
    g.o_llm = out.llm_time + oa;
    g.o_dec = reinterpret_cast<long long*>(out.decode_total) + oa;
    g.o_maxctx = reinterpret_cast<long long*>(out.max_context) + oa;
    g.o_ctx = reinterpret_cast<long long*>(out.context) + oa;
    g.o_steps = out.turns_completed + oa;
    g.o_inst = out.final_instance + oa;
    g.o_mig = out.migrations + oa;
    g.o_phase = out.phase + oa;
    g.sl = ws.sl + oa;
    g.dstamp = ws.dstamp + oa;
    g.ring = ws.ring + ws.ring_off[s];
    g.log = ws.log + ws.ring_off[s];
    g.turn_issue = out.turn_issue ? out.turn_issue + out.turn_off[s] : nullptr;
    g.turn_done = out.turn_done ? out.turn_done + out.turn_off[s] : nullptr;
    g.dec_rows = out.decisions ? out.decisions + out.dec_off[s] : nullptr;
    g.o_energy = out.energy + oi;
    g.o_thr = out.thrash_time + oi;
    g.o_usage = reinterpret_cast<long long*>(out.final_usage) + oi;
    g.o_pending = out.final_pending + oi;
    g.o_level = out.final_level + oi;
    g.o_ctr = reinterpret_cast<long long*>(out.counters) + (long long)s * ASB_NCOUNTERS;
    const bool ts_on = out.timeseries && out.ts_off && out.ts_off[s + 1] > out.ts_off[s];
    g.ts_rows = ts_on ? out.timeseries + out.ts_off[s] : nullptr;
    g.ts_cap = ts_on ? out.ts_off[s + 1] - out.ts_off[s] : 0;
    g.ts_count = out.ts_count ? reinterpret_cast<long long*>(out.ts_count) + s : nullptr;
    g.A = A;
    g.M = sc.n_instances;
    g.L = sc.n_levels;
    if (EC_LANE == 0) w->gp = g;
    __syncwarp();
    if (ts_on) /* smem copy of GP: no local-memory frame */
      asb::run_scenario<W, RCAP, DCAP, ACAP, true>(w, w->gp);
    else
      asb::run_scenario<W, RCAP, DCAP, ACAP, false>(w, w->gp);
    __syncwarp();
  }
  if (EC_LANE == 0) w->job = asb::JOB_EXIT;
  __syncwarp();
  ec_fork_begin(NT);
}

template <int MAXM, int RCAP, int DCAP, int ACAP, int NT, int LMAX = 16>
int launch_engine(const AsbScenario* d_scen, int n_scen, const AsbTracePool& tp, const AsbTablePool& tb,
                  const AsbOutputs& out, const Workspace& ws, cudaStream_t st) {
  using W = asb::WS<MAXM, RCAP, DCAP, ACAP, NT, LMAX>;
  static_assert(RCAP >= DCAP + ACAP, "record buffer must hold every first record");
  static_assert(NT % 32 == 0 && NT >= 32 && (NT & (NT - 1)) == 0, "team = a power-of-two number of whole warps");
  /* 4 teams per SM need <= ~54 KB of shared memory each (228 KB per SM) */
  static_assert(NT > 128 || W::MX > 16 || sizeof(W) <= 54 * 1024, "small-team workspace must allow 4 CTAs per SM");
  const size_t smem = (sizeof(W) + 15) / 16 * 16;
  auto kern = asb_engine_kernel<MAXM, RCAP, DCAP, ACAP, NT, LMAX>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return ASB_ERR_LAUNCH;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem) != cudaSuccess || per_sm < 1)
    return ASB_ERR_LAUNCH;
  if (const char* cap_env = getenv("ASB_TEAMS_PER_SM")) { /* experiment: fewer co-resident teams */
    const int c = atoi(cap_env);
    if (c >= 1 && c < per_sm) per_sm = c;
  }
  if (getenv("ASB_DEBUG_LAUNCH"))
    fprintf(stderr, "asb launch: team %d, smem %zu B, %d blocks/SM, %d SMs\n", NT, smem, per_sm, sms);
  long long want = n_scen;
  long long cap = (long long)sms * per_sm;
  int blocks = (int)(want < cap ? want : cap);
  if (blocks < 1) blocks = 1;
  kern<<<blocks, NT, smem, st>>>(d_scen, n_scen, tp, tb, out, ws);
  return cudaGetLastError() == cudaSuccess ? ASB_OK : ASB_ERR_LAUNCH;
}

}  // namespace

extern "C" {

int asb_abi_version(void) { return ASB_ABI_VERSION; }

#ifdef ASB_DEBUG_TRACE
/* debug builds only: host-mapped long long[64] progress markers (block 0) */
int asb_debug_trace(void* host_mapped) {
  return cudaMemcpyToSymbol(g_asb_dbg, &host_mapped, sizeof(void*)) == cudaSuccess ? 0 : -2;
}
#endif

size_t asb_workspace_bytes(int32_t n_scen, int64_t total_agents, int64_t total_ring_slots) {
  return carve(nullptr, n_scen, total_agents, total_ring_slots, nullptr);
}

int asb_run_scenarios(const AsbScenario* d_scen, int32_t n_scen, int32_t max_instances, AsbTracePool traces,
                      AsbTablePool tables, AsbOutputs out, int64_t total_agents, int64_t total_ring_slots,
                      void* d_workspace, size_t workspace_bytes, void* stream) {
  const bool fixed_m = max_instances < 0; /* -m: every scenario has exactly m instances */
  if (fixed_m) max_instances = -max_instances;
  if (n_scen < 0 || max_instances < 1 || max_instances > ASB_MAX_INSTANCES) return ASB_ERR_ARG;
  if (tables.max_levels < 0 || tables.max_levels > ASB_MAX_LEVELS) return ASB_ERR_ARG;
  if (out.timeseries && (!out.ts_off || !out.ts_count)) return ASB_ERR_ARG; /* rows need their offsets and counts */
  if (n_scen == 0) return ASB_OK;
  size_t need = carve(nullptr, n_scen, total_agents, total_ring_slots, nullptr);
  if (!d_workspace || workspace_bytes < need) return ASB_ERR_WORKSPACE;
  Workspace ws;
  carve((unsigned char*)d_workspace, n_scen, total_agents, total_ring_slots, &ws);
  cudaStream_t st = (cudaStream_t)stream;
  if (const char* pl = getenv("ASB_L2_PERSIST_MB")) { /* experiment: L2 set-aside for evict_last lines */
    size_t want = (size_t)atol(pl) << 20;
    int dev0 = 0, mx = 0;
    cudaGetDevice(&dev0);
    cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, dev0);
    if (want > (size_t)mx) want = (size_t)mx;
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
  }
  ring_offsets_kernel<<<1, 1024, 0, st>>>(d_scen, n_scen, traces.trace_agent_off, ws.ring_off, ws.work);
  if (cudaGetLastError() != cudaSuccess) return ASB_ERR_LAUNCH;
  /* team shape by scenario size (ASB_TEAM=solo|quad|big overrides, for tests):
   *  - few large scenarios (each gets an SM of its own anyway): a 16-warp
   *    team with 5x larger optimistic batches;
   *  - small scenarios (< 2k agents on average): a single warp, no fork-join
   *    barriers, 40-record batches (their per-epoch work is a few events),
   *    ~15 KB of shared memory so ~14 teams fit per SM;
   *  - otherwise 4-warp teams, 4 per SM. */
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t per = n_scen > 0 ? total_agents / n_scen : 0;
  bool big = n_scen <= sms && per >= 8192;
  bool solo = !big && per < 2048;
  if (const char* force = getenv("ASB_TEAM")) {
    big = !strcmp(force, "big");
    solo = !strcmp(force, "solo");
  }
  /* more than 64 instances or more than 16 DVFS levels: the wide kernel
   * (128 instance slots, 64 levels; ~2 teams per SM, correctness first) */
  if (max_instances > 64 || tables.max_levels > 16)
    return launch_engine<128, 192, 128, 64, 128, ASB_MAX_LEVELS>(d_scen, n_scen, traces, tables, out, ws, st);
#ifndef ASB_BIG_RC /* the 16-warp team's batch buffers: 768 records (153 KB of shared
                      memory, the 164 KB carveout: L1 92 KB instead of 60 KB); C4 442 -> 438 ms
                      against 1,024 (188 KB); 896 measured 442 ms */
#define ASB_BIG_RC 768
#define ASB_BIG_DC 576
#endif
  if (big) {
    /* every scenario with exactly 64 instances (the thrashing regime C4): the
     * count is a compile-time constant, as for the 16-instance sweep */
    if (fixed_m && max_instances == 64 && !getenv("ASB_NO_FIXED_M"))
      return launch_engine<-64, ASB_BIG_RC, ASB_BIG_DC, 128, 512>(d_scen, n_scen, traces, tables, out, ws, st);
    return launch_engine<64, ASB_BIG_RC, ASB_BIG_DC, 128, 512>(d_scen, n_scen, traces, tables, out, ws, st);
  }
  /* single-instance scenarios (the DVFS sweep): a kernel whose instance
   * count is the constant 1, with the per-instance machinery folded away */
#ifndef ASB_SOLO1_RC
#define ASB_SOLO1_RC 64 /* 64-record batches: fewer window splits, still 14 teams per SM (15.5 KB) */
#endif
  if (max_instances == 1 && solo)
    return launch_engine<1, ASB_SOLO1_RC, ASB_SOLO1_RC / 2, ASB_SOLO1_RC / 2, 32>(d_scen, n_scen, traces, tables, out, ws, st);
  if (max_instances <= 16) {
    if (solo) return launch_engine<16, 40, 20, 20, 32>(d_scen, n_scen, traces, tables, out, ws, st);
    /* every scenario with exactly 16 instances (the Monte-Carlo sweep): the
     * count is a compile-time constant */
#ifdef ASB_EXP_C5_NT /* experiment: another team shape for the 16-instance sweep */
    if (fixed_m && max_instances == 16)
      return launch_engine<-16, ASB_EXP_C5_RC, ASB_EXP_C5_DC, ASB_EXP_C5_RC - ASB_EXP_C5_DC, ASB_EXP_C5_NT>(d_scen, n_scen, traces, tables, out, ws, st);
#endif
    /* 176-record batches with 116 due agents: 48.2 KB of shared memory, so
     * four teams fit the 196 KB carveout and L1 keeps 60 KB instead of 28 KB
     * (192 / 128: 52.2 KB, the 228 KB carveout); whole C5 job 1005 -> 980 ms */
    if (fixed_m && max_instances == 16 && !getenv("ASB_NO_FIXED_M")) return launch_engine<-16, 176, 116, 60, 128>(d_scen, n_scen, traces, tables, out, ws, st);
    return launch_engine<16, 176, 116, 60, 128>(d_scen, n_scen, traces, tables, out, ws, st);
  }
  if (solo) return launch_engine<64, 40, 20, 20, 32>(d_scen, n_scen, traces, tables, out, ws, st);
  return launch_engine<64, 192, 128, 64, 128>(d_scen, n_scen, traces, tables, out, ws, st);
}

}  // extern "C"
