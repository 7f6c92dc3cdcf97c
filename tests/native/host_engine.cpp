/*
 * host_engine.cpp — TEST HARNESS ONLY.  Compiles the GPU engine's batching
 * logic (paper_2604_16682_b200/csrc/engine_core.h) with a 1-lane "team" so
 * the optimistic epoch batches, the commit walk and the serial coupling
 * handlers can be differential-tested against the serial oracle on CPU in
 * the `-m "not gpu"` suite.  Nothing in the package loads this library; the
 * product path is the sm_100a build of the same header (engine.cu).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/agentsim_b200.h"

#define EC_DEV static inline
#define EC_LANE 0
#define EC_TSIZE 1
#define EC_NAN (__builtin_nan(""))
#define EC_INF (__builtin_inf())
#define EC_INF_BITS 0x7ff0000000000000ull

static inline void t_sync() {}
static inline unsigned t_ballot(bool p) { return p ? 1u : 0u; }
static inline unsigned t_lt_mask() { return 0u; }
static inline int ec_popc(unsigned m) { return __builtin_popcount(m); }
static inline int ec_ffs(unsigned m) { return __builtin_ffs((int)m); }
static inline unsigned t_match_any_i(int) { return 1u; }
static inline unsigned t_redux_min_u32(unsigned v) { return v; }
static inline long long t_bcast_ll(long long v, int) { return v; }
static inline long long t_scan_add_ll(long long v) { return v; }
static inline int t_scan_add_i(int v) { return v; }
static inline int t_shfl_i(int v, int) { return v; }
static inline int t_redux_add_i(int v) { return v; }
static inline long long t_sum_ll(long long v) { return v; }
static inline unsigned long long t_shfl_xor_ull(unsigned long long v, int) { return v; }
static inline long long t_shfl_xor_ll(long long v, int) { return v; }
static inline int t_shfl_xor_i(int v, int) { return v; }
static inline long long t_shfl_up_ll(long long v, int) { return v; }
static inline int t_shfl_up_i(int v, int) { return v; }
static inline void t_atomic_min_ull(unsigned long long* p, unsigned long long v) { if (v < *p) *p = v; }
static inline int t_atomic_add_i(int* p, int v) { int o = *p; *p += v; return o; }
static inline bool ec_isnan(double x) { return x != x; }
static inline double ec_floor(double x) { return floor(x); }
static inline unsigned long long ec_bits(double x) { unsigned long long b; memcpy(&b, &x, 8); return b; }
static inline double ec_from_bits(unsigned long long b) { double x; memcpy(&x, &b, 8); return x; }
static inline long long ec_clock() { return 0; }
/* round toward -inf to f32 (<= x), as __double2float_rd */
static inline float ec_f32_down(double x) {
  float f = (float)x;
  if ((double)f > x) f = nextafterf(f, -__builtin_inff());
  return f;
}
#define EC_INF_F32 (__builtin_inff())
#define EC_TID_OF(nt) 0
static inline void ec_fork_begin(int) {}
static inline void ec_fork_end(int) {}
static inline void ec_team_barrier(int) {}
static inline int t_atomic_min_i(int* p, int v) { int o = *p; if (v < o) *p = v; return o; }
static inline unsigned long long t_warp_min_ull(unsigned long long v) { return v; }
static inline void t_warp_min_key(unsigned long long&, unsigned&) {}

/* the small-window serial loop (single-warp GPU teams) on demand */
static int host_serial_due = 0;
#define EC_SERIAL_DUE_ON(W) (host_serial_due != 0)
#define EC_SERIAL_DUE_MAX 8 /* off in the GPU build (measured slower); an exact alternative here */

#include "../../paper_2604_16682_b200/csrc/engine_core.h"

/* small buffers on purpose: exercises the overflow / horizon / bisection paths */
template <int RCAP, int DCAP, int ACAP>
static int run_all(const AsbScenario* scen, int32_t n_scen, const AsbTracePool* tp, const AsbTablePool* tb,
                   const AsbOutputs* out) {
  using W = asb::WS<64, RCAP, DCAP, ACAP, 1>;
  W* w = (W*)calloc(1, sizeof(W));
  int err = 0;
  for (int s = 0; s < n_scen; s++) {
    const AsbScenario& sc = scen[s];
    w->sc = sc;
    long long t0 = tb->table_off[sc.table_id];
    for (int l = 0; l < sc.n_levels; l++) {
      w->pr[l] = tb->prefill_rate[t0 + l];
      w->dr[l] = tb->decode_rate[t0 + l];
      w->act[l] = tb->active_power[t0 + l];
      w->idle[l] = tb->idle_power[t0 + l];
    }
    const long long a0 = tp->trace_agent_off[sc.trace_id];
    const int A = (int)(tp->trace_agent_off[sc.trace_id + 1] - a0);
    const long long oa = out->agent_off[s], oi = out->inst_off[s];
    size_t na = (size_t)(A > 0 ? A : 1);
    asb::GP g;
    double* f64 = (double*)calloc(na * 10, 8);
    asb::AgentHot* hot = (asb::AgentHot*)aligned_alloc(128, na * sizeof(asb::AgentHot));
    long long* i64 = (long long*)calloc(na * 2, 8);
    asb::Slot* sl = (asb::Slot*)aligned_alloc(16, na * sizeof(asb::Slot));
    int* i32 = (int*)calloc(na * 7, 4);
    int* rl = (int*)calloc(na * (size_t)sc.n_instances * 2, 4);
    g.arrival = tp->arrival + a0;
    g.aturn = (const long long*)tp->agent_turn_off + a0;
    g.prefill = tp->prefill;
    g.decode = tp->decode;
    g.tool = tp->tool;
    g.arr_order = tp->arrival_order + a0;
    g.turn_base = tp->trace_turn_off[sc.trace_id];
    g.H = hot;
    g.ctime = out->completion_time + oa;
    g.arr_t = f64 + 9 * na;
    g.notbefore = f64 + 6 * na;
    g.pissue = f64 + 7 * na;
    g.rank = out->arrival_rank + oa;
    g.o_llm = out->llm_time + oa;
    g.o_dec = (long long*)out->decode_total + oa;
    g.o_maxctx = (long long*)out->max_context + oa;
    g.o_ctx = (long long*)out->context + oa;
    g.o_steps = out->turns_completed + oa;
    g.o_inst = out->final_instance + oa;
    g.o_mig = out->migrations + oa;
    g.o_phase = out->phase + oa;
    g.dstamp = i32 + 6 * na;
    g.sl = sl;
    g.ring = rl;
    g.log = rl + na * (size_t)sc.n_instances;
    g.turn_issue = out->turn_issue ? out->turn_issue + out->turn_off[s] : nullptr;
    g.turn_done = out->turn_done ? out->turn_done + out->turn_off[s] : nullptr;
    g.dec_rows = out->decisions ? out->decisions + out->dec_off[s] : nullptr;
    g.o_energy = out->energy + oi;
    g.o_thr = out->thrash_time + oi;
    g.o_usage = (long long*)out->final_usage + oi;
    g.o_pending = out->final_pending + oi;
    g.o_level = out->final_level + oi;
    g.o_ctr = (long long*)out->counters + (long long)s * ASB_NCOUNTERS;
    const bool ts_on = out->timeseries && out->ts_off && out->ts_off[s + 1] > out->ts_off[s];
    g.ts_rows = ts_on ? out->timeseries + out->ts_off[s] : nullptr;
    g.ts_cap = ts_on ? out->ts_off[s + 1] - out->ts_off[s] : 0;
    g.ts_count = out->ts_count ? (long long*)out->ts_count + s : nullptr;
    g.A = A;
    g.M = sc.n_instances;
    g.L = sc.n_levels;
    w->gp = g;
    if (ts_on)
      asb::run_scenario<W, RCAP, DCAP, ACAP, true>(w, g);
    else
      asb::run_scenario<W, RCAP, DCAP, ACAP, false>(w, g);
    err |= (int)g.o_ctr[ASB_CTR_STATUS];
    free(f64);
    free(hot);
    free(i64);
    free(sl);
    free(i32);
    free(rl);
  }
  free(w);
  return err;
}

extern "C" int host_engine_run(const AsbScenario* scen, int32_t n_scen, const AsbTracePool* tp,
                               const AsbTablePool* tb, const AsbOutputs* out, int32_t small_buffers) {
  /* bit 0: small buffers; bit 1: the small-window serial loop */
  host_serial_due = (small_buffers & 2) != 0;
  if (small_buffers & 1) return run_all<16, 8, 4>(scen, n_scen, tp, tb, out);
  return run_all<256, 128, 64>(scen, n_scen, tp, tb, out);
}
