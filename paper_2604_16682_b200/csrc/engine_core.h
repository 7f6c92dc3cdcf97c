/*
 * engine_core.h — the batched, epoch-synchronous scenario engine.
 *
 * One TEAM (a warp on the GPU) runs one scenario = one reference
 * `run_simulation` (/root/reference/pkg/src/agentsim/engine.py:576-604).
 * The reference pops one event at a time from a global heap; this engine
 * reproduces exactly the same event order and arithmetic, but processes the
 * events between two control epochs as an optimistic batch:
 *
 *   1. epoch event (engine.py:436-488): the agent-tick sweep computes every
 *      instance's min running throughput over its ongoing ∪ pending agents
 *      (controller.py:96-103) in one coalesced pass over the alive slots;
 *      level select / SLO boost / power run lane-per-instance; β/γ admission
 *      is a prefix scan over the pending FIFO; push sequence numbers of the
 *      epoch's re-timings and admissions are an exclusive scan over
 *      instances (the reference pushes them instance-major);
 *   2. due collection: agents whose next event falls before the next epoch;
 *   3. speculation (lane per agent): each agent's own event chain
 *      (complete → tool gap → next turn → …, engine.py:374-401, 509-568)
 *      inside the window, assuming the instance's thrash flag and level stay
 *      as they are — the only instance state an agent's timing reads;
 *   4. sort the records by (time, priority); exact ties are ordered by the
 *      reference's push sequence number (engine.py:300-301);
 *   5. commit walk: the serial state machine decomposes by instance, so each
 *      lane replays its instances' records (usage, running count, thrash
 *      flag, power, running log) and the first coupling event is found by a
 *      min-reduction — a completion that flips the thrash flag, a
 *      reassignment check that migrates (evaluated on usage snapshots), or
 *      any start/complete under interference.  That event is then executed
 *      serially with the exact handler semantics and speculation restarts;
 *   6. apply (lane per agent): committed chain prefixes are written back.
 *
 * The file is compiled twice: by nvcc for sm_100a with the warp team
 * (engine.cu), and by g++ with a 1-lane team (tests/native/host_engine.cpp)
 * purely as a test harness for the batching logic on CPU.  The host build is
 * never loaded by the package.
 *
 * Arithmetic follows the reference operation by operation in IEEE binary64
 * (no FMA contraction: built with --fmad=false / -ffp-contract=off).
 */
#ifndef ASB_ENGINE_CORE_H
#define ASB_ENGINE_CORE_H

#include "../../include/agentsim_b200.h"

/* ---- team primitives: provided by the includer ----------------------------
 *   EC_DEV, EC_LANE, EC_TSIZE, t_sync(), t_ballot(p), t_lt_mask(), ec_popc,
 *   t_bcast_ll, t_scan_add_ll, t_sum_ll, t_shfl_xor_{ull,ll,i}, t_match_any_i,
 *   t_atomic_min_ull, t_atomic_add_i, ec_isnan, ec_floor, ec_bits,
 *   ec_from_bits, ec_clock, EC_NAN, EC_INF, EC_INF_BITS
 */

/* EC_COLD: large phase functions, kept out of line so the hot loops stay
 * inside the instruction cache (includer may override) */
#ifndef EC_COLD
#define EC_COLD EC_DEV
#endif
#ifndef EC_COLD1
#define EC_COLD1 EC_COLD /* fork-join job bodies */
#endif
#ifndef EC_COLD2
#define EC_COLD2 EC_COLD /* serial handlers */
#endif
#ifndef EC_COLD3
#define EC_COLD3 EC_COLD /* epoch / batch phases */
#endif
#ifndef EC_COLD4
#define EC_COLD4 EC_COLD /* shared helpers called from many sites */
#endif

/* EC_LANE0 { ... }: a lane-0 section of the main warp's serial code.  Lanes
 * of a warp are independently scheduled, so every lane must have read the
 * shared state it needs before lane 0 starts mutating it: the section opens
 * with a warp barrier (and every section is followed by one, so the other
 * lanes read lane 0's results only after it finished). */
#define EC_LANE0 if ((t_sync(), EC_LANE == 0))

/* EC_DBG(slot, value): progress markers for hang debugging (GPU debug build
 * -DASB_DEBUG_TRACE writes them to host-mapped memory); no-op otherwise */
#ifndef EC_DBG
#define EC_DBG(slot, value) \
  do {                      \
  } while (0)
#endif

/* EC_LDK_* / EC_STK_*: loads / stores of the alive slots that every
 * epoch's sweep reads, marked to stay in L2 (evict_last) on the GPU */
#ifndef EC_SLOT_ACCESSORS
#define EC_LDK_I32(p) (*(p))
#define EC_STK_F64(p, v) (*(p) = (v))
#define EC_STK_I32(p, v) (*(p) = (v))
/* one 16-byte alive slot: (tp, nx, meta) */
#define EC_LDK_SLOT(p, tp_, nx_, mt_) ((tp_) = (p)->tp, (nx_) = (p)->nx, (mt_) = (p)->meta)
/* the slot's (nx, meta) half in one 8-byte store */
#define EC_STK_EV(p, nx_, mt_) ((p)->nx = (nx_), (p)->meta = (mt_))
#endif

#ifndef EC_DEPCAP
#define EC_DEPCAP 16 /* arrivals + reassignment checks per parallel walk (small teams) */
#endif
#ifndef EC_TEAMSORT_MIN_NT
#define EC_TEAMSORT_MIN_NT 512 /* teams of at least this many threads build the sort's horizon cut and
                                  per-instance lists with the whole team (smaller: warp 0; experiment knob) */
#endif
#ifndef EC_CCAP
#define EC_CCAP 0 /* cached due-agent cursors per batch; 0 = all DCAP (experiment knob: 64 or 48 on
                     the 16-instance kernels reach the 164 KB carveout, whole C5 job within 0.4%) */
#endif
/* loops over instances: kept rolled, the trip count is small and the
 * co-resident teams share a 32 KB instruction cache */
#ifndef EC_BITONIC_MIN
#define EC_BITONIC_MIN 256 /* the 16-warp team bitonic-sorts batches of more records than this */
#endif
#ifndef EC_PREFETCH_L2
#define EC_PREFETCH_L2(p) ((void)(p))
#endif
#ifndef EC_ILOOP
#define EC_ILOOP _Pragma("unroll 1")
#endif
#ifndef EC_SWEEP_UNROLL
#define EC_SWEEP_UNROLL 2 /* independent loads in flight per lane in the slot sweeps (small: I-cache) */
#endif
#ifndef EC_SWEEP_UNROLL_QUAD
#define EC_SWEEP_UNROLL_QUAD EC_SWEEP_UNROLL /* the same for the 4-warp team */
#endif

namespace asb {

enum { EV_EPOCH = 0, EV_COMPLETE = 1, EV_TOOL = 2, EV_ISSUE = 3, EV_ARRIVAL = 4 };
enum { F_LAST = 1, F_CHECK = 2, F_COMMITTED = 4, F_EMPTY = 8 };
enum { STOP_NONE = 0, STOP_COUPLING = 1, STOP_HORIZON = 2, STOP_LOGFULL = 3 };
enum { BATCH_DONE = 0, BATCH_MORE = 1, BATCH_SERIAL = 2 };

/* one speculative event record (engine.py handler invocation) */
struct Rec {
  double t;
  long long seq;       /* own push sequence number (-1 until known) */
  long long push_seq;  /* seq of the event this one pushes */
  long long aux64;     /* COMPLETE: context after growth; start: start rank */
  int agent;
  short prio;          /* EV_* kind == tie-break priority */
  short flags;
  int delta;           /* COMPLETE: prefill+decode */
  int dd;              /* COMPLETE: decode tokens */
  double nt;           /* time of the event this one pushes (tool gap end / turn done) */
  int child;           /* next record of the same agent chain, -1 none */
  int logpos;          /* start: position in the instance running log */
  int inst;
};

/* one alive slot, what every epoch's agent-tick sweep reads (16 bytes, one
 * vector load): the running throughput (+inf = None, NaN = finished), the
 * next event time rounded DOWN to f32 (a conservative due test: the exact
 * time is H[a].next_t, re-checked by the speculation, so a slot whose f32
 * time is in the window but whose exact time is not becomes an empty
 * candidate), and meta = instance | next-event kind << 7 | agent << 10, so
 * that collecting a due slot needs no second (dependent) load for its agent */
struct alignas(16) Slot {
  double tp;
  float nx;
  int meta;
};
static_assert(sizeof(Slot) == 16, "one 16-byte vector load per slot");
#define EC_SLOT_MAX_AGENTS (1 << 21) /* agent ids in meta bits 10..30 (packing.py checks) */
EC_DEV int slot_meta(int inst, int prio, int a) { return inst | (prio << 7) | (a << 10); }
EC_DEV int sm_inst(int m) { return m & 0x7f; }
EC_DEV int sm_prio(int m) { return (m >> 7) & 7; }
EC_DEV int sm_agent(int m) { return m >> 10; }

struct SortE {
  unsigned long long tb; /* time bits (times are >= 0, so bits order like values) */
  unsigned int prio;
  unsigned int idx;
};

/* hot per-agent state (AgentRuntimeState instance.py:148-160 + _Agent /
 * _RunningTurn engine.py:210-231), one 128-byte record per agent so that an
 * event touches one cache line instead of a sector in each of ~20 arrays */
struct alignas(16) AgentHot {
  double next_t, llm, issue, anchor, rem, done;
  long long ctx, dec, maxctx, next_seq, start_rank;
  int steps, inst, sa, logpos, phase, next_prio, slot, mig, pad0, pad1;
};
static_assert(sizeof(AgentHot) == 128, "one 128-byte line per agent");

/* one agent's event cursor (agent state in registers) */
struct Cur {
  int a, inst, phase, prio, steps, n_turns, sa;
  int slot; /* the agent's alive slot (fixed between the speculation and the apply) */
  double t, llm, issue, anchor, rem, done;
  long long ctx, dec, maxctx, turn0;
  /* turn records of the current and the next turn, prefetched with the
   * agent's state (one memory round trip for a complete -> issue chain) */
  int pf_p0, pf_d0, pf_p1, pf_d1;
  double pf_tool0;
  int pf_step;
};

/* per-instance engine state: InstanceState (instance.py:163-181) + _Instance (engine.py:234-247) */
struct Inst {
  long long usage;
  double watts, t_pow, energy, thr_since, thr_time;
  int level, running, thr, thr_flag;
  int key_valid, key_level, key_thr, key_run;
  int fifo_head, fifo_len, log_len, pad_;
};

/* pointers for one scenario (row bases applied) */
struct GP {
  /* trace */
  const double* arrival;
  const long long* aturn;  /* [A+1] global turn offsets */
  const int* prefill;
  const int* decode;
  const double* tool;
  const int* arr_order;
  double* arr_t; /* [A] arrival times in arrival order (filled at scenario init) */
  long long turn_base;
  /* agent state (SoA, by agent) */
  AgentHot* H;        /* hot per-agent state, one 128-byte record per agent */
  double *ctime, *notbefore, *pissue;
  int *rank, *dstamp;
  /* outputs written from H when the scenario finishes */
  double* o_llm;
  long long *o_dec, *o_maxctx, *o_ctx;
  int *o_steps, *o_inst, *o_mig, *o_phase;
  /* alive slots: the agent-tick / due sweeps read only these, coalesced */
  Slot* sl;        /* (throughput, next event time, instance | kind | agent) per slot */
  int* ring;       /* [M*A] pending FIFOs */
  int* log;        /* [M*A] running logs (insertion order of inst.running) */
  /* outputs */
  double *turn_issue, *turn_done;
  AsbDecision* dec_rows;
  double *o_energy, *o_thr;
  long long* o_usage;
  int *o_pending, *o_level;
  long long* o_ctr;
  /* timeseries rows (NULL: off; then the scenario runs the exact serial loop) */
  AsbTimeseriesRow* ts_rows;
  long long ts_cap;
  long long* ts_count;
  int A, M, L;
};

/* the scenario pointers a team job's loop reads, copied out of the shared
 * GP once: read through the GP reference they are reloaded after every
 * shared-memory store the loop makes (the compiler cannot rule out that the
 * store changed them).  Passed by value to the inline cursor helpers. */
struct GV {
  AgentHot* H;
  Slot* sl;
  const long long* aturn;
  const int* prefill;
  const int* decode;
  const double* tool;
  double* ctime;
  double *turn_issue, *turn_done;
  long long turn_base;
  int *ring, *log, *dstamp, *rank;
  double *pissue, *notbefore;
  int A;
};
EC_DEV GV gview(const GP& g) {
  GV v;
  v.H = g.H;
  v.sl = g.sl;
  v.aturn = g.aturn;
  v.prefill = g.prefill;
  v.decode = g.decode;
  v.tool = g.tool;
  v.ctime = g.ctime;
  v.turn_issue = g.turn_issue;
  v.turn_done = g.turn_done;
  v.turn_base = g.turn_base;
  v.ring = g.ring;
  v.log = g.log;
  v.dstamp = g.dstamp;
  v.rank = g.rank;
  v.pissue = g.pissue;
  v.notbefore = g.notbefore;
  v.A = g.A;
  return v;
}

/* GV for the multi-warp teams; the single-warp teams keep reading through
 * the shared GP (the view's registers cost them more than the reloads) */
template <bool VIEW>
struct GPick {
  using T = GV;
};
template <>
struct GPick<false> {
  using T = const GP&;
};
template <bool VIEW>
struct GTag {};
EC_DEV GV gpick(const GP& g, GTag<true>) { return gview(g); }
EC_DEV const GP& gpick(const GP& g, GTag<false>) { return g; }
#define EC_GVIEW(W_, gp_) typename GPick<(W_::NT > 32)>::T g = gpick(gp_, GTag<(W_::NT > 32)>())

enum { JOB_EXIT = 0, JOB_INIT = 1, JOB_SWEEP = 2, JOB_SPEC = 3, JOB_SORT = 4, JOB_APPLY = 5, JOB_ADMIT = 6,
       JOB_EPOCH = 7, JOB_FINISH = 8, JOB_DEPS = 9 };

template <int MAXM, int RCAP, int DCAP, int ACAP, int NTHR, int LMAX = 16>
struct WS {
  static constexpr int NT = NTHR;          /* threads of the team (main warp + helpers) */
  static constexpr int NW = (NTHR + 31) / 32;
  static constexpr int RC = RCAP, DC = DCAP, AC = ACAP;
  /* instance capacity of the kernel; a negative MAXM: every scenario of
   * the launch has exactly -MAXM instances (a compile-time count) */
  static constexpr int MX = MAXM < 0 ? -MAXM : MAXM;
  static constexpr bool FIXM = MAXM < 0;
  /* large-batch teams: more dependent records per walk, and the apply
   * reloads agent state instead of caching it in shared memory */
  static constexpr int DEP = RCAP >= 512 ? 64 : EC_DEPCAP;
  static constexpr bool CC = RCAP < 512;
  /* cached cursors: the first CCN due agents of a batch (the rest reload) */
  static constexpr int CCN = CC ? (EC_CCAP > 0 && EC_CCAP < DCAP ? EC_CCAP : DCAP) : 1;
  /* the 16-warp team's sort: horizon cut and per-instance lists by the
   * whole team (the smaller teams keep the shorter warp-0 code) */
  static constexpr bool BIGSORT = NTHR >= EC_TEAMSORT_MIN_NT;
  /* the bitonic network's ping-pong buffers (the key buffer and the sorted
   * view) hold the next power of two of RCAP */
  static constexpr int SK = NTHR >= 512 ? (RCAP <= 256 ? 256 : RCAP <= 512 ? 512 : RCAP <= 1024 ? 1024 : 2048) : RCAP;
  AsbScenario sc;
  GP gp;                                   /* shared with the helper warps */
  /* fork-join job state */
  int job;
  int j_tick, j_collect, j_incl, j_token;
  double j_bound;
  int j_dead, j_total, j_cut, j_tie_unknown, j_order_err;
  unsigned long long j_hz_t[NW];
  unsigned j_hz_p[NW];
  /* scratch reused phase by phase: the sort's keys, then the walk's scans */
  union {
    alignas(16) unsigned long long skey[2 * SK]; /* 16-byte sort keys (GPU counting sort / bitonic) */
    struct {
      unsigned long long kt[RCAP]; /* generic (1-lane) rank sort */
      long long ks[RCAP];
      unsigned char kp[RCAP];
    };
    struct {
      /* scan walk: per entry of the per-instance lists (ilist order) the
       * usage, running count and log length after it, and the power-change flag */
      long long wu[RCAP];
      int wr[RCAP], wl[RCAP];
    };
    /* rank sort, after the keys: per 32-record chunk of the sorted order and
     * per instance, its record count, then the count in earlier chunks */
    unsigned short kcc[(RCAP + 31) / 32][MX];
  };
  unsigned char depflag[RCAP];
  short ki[RCAP], kir[RCAP], krank[RCAP], ilist[RCAP]; /* per-instance record lists */
  int icnt[MX], ioff[MX + 1];
  double now, bound;
  long long seq, start_ctr;
  long long ctr[ASB_NCOUNTERS];
  unsigned long long hz_t;
  int hz_p;
  long long hz_s;
  int n_alive, rr_next, arr_ptr, arr_rank, status, incl;
  int n_rec, n_due, n_arr, stop_kind, stop_rec, flag, tmp_i, n_dep;
  int due_ready, n_cand, cand_token, n_empty, cand_collect;
  int stamp_ctr; /* last due-list stamp handed out (dstamp de-duplication) */
  double pr[LMAX], dr[LMAX], act[LMAX], idle[LMAX]; /* the scenario's frequency table (levels 1..L) */
  Inst in[MX];
  unsigned long long tmin[MX];
  /* epoch scratch (per instance) */
  long long ep_uobs[MX], ep_seq[MX];
  double ep_mintp[MX];
  int ep_level[MX], ep_boost[MX], ep_nadm[MX], ep_head[MX], ep_retime[MX], ep_def[MX], ep_thr0[MX];
  int ep_nstart[MX];
  long long ep_rank[MX];
  int ep_list[MX];
  int n_eplist;
  double ep_gcap;
  int due[DCAP];
  Cur ccache[CCN]; /* due agents' state loaded by the speculation, reused by the apply */
  Rec rec[RCAP];
  SortE srt[SK];
  /* sorted structure-of-arrays view of the records for the commit walk */
  double sw_t[RCAP];
  long long sw_du[RCAP];
  int sw_idx[RCAP];
  short sw_inst[RCAP];
  unsigned char sw_prio[RCAP], sw_flags[RCAP];
  int dep_pos[DEP];
  int dep_target[DEP]; /* routed instance of each dependent arrival; -1: a migrating check (JOB_DEPS) */
  int j_stop;          /* JOB_DEPS: records at or after this position are not committed */
  long long snap[DEP][MX];
  long long carry_u;
  int carry_r, carry_l;
  unsigned wmask[(RCAP + 31) / 32]; /* power-change entries of the scan walk, one bit per ilist entry */
  Rec stop_r;
  long long prof[6];
  long long prof_t;
  /* timeseries: rows written, next sample index, each instance's last row */
  long long ts_n, ts_k;
  long long ts_last[MX];
};

/* the scenario's instance count; a compile-time constant in the
 * single-instance kernels (MAXM = 1) and the fixed-count kernels (MAXM < 0),
 * so that their per-instance loops, scans and argmins fold away */
template <class W>
EC_DEV int ec_nm(const W* w) {
  return (W::FIXM || W::MX == 1) ? W::MX : w->sc.n_instances;
}

/* optional sub-step timing of one team job: thread 0's cycles per step in
 * prof[0..5], for JOB_SORT (-DASB_PROFILE -DASB_PROFILE_SORT, EC_QPROF) or
 * the speculation (-DASB_PROFILE -DASB_PROFILE_SPEC, EC_PPROF) */
#define EC_STEPPROF_T0_ long long qprof_t_ = ec_clock()
#define EC_STEPPROF_(w, k)                           \
  do {                                               \
    if (tid == 0) {                                  \
      const long long qn_ = ec_clock();              \
      (w)->prof[k] += qn_ - qprof_t_;                \
      qprof_t_ = qn_;                                \
    }                                                \
  } while (0)
#define EC_STEPPROF_NONE_ \
  do {                    \
  } while (0)
#if defined(ASB_PROFILE_SORT)
#define EC_QPROF_T0() EC_STEPPROF_T0_
#define EC_QPROF(w, k) EC_STEPPROF_(w, k)
#else
#define EC_QPROF_T0() EC_STEPPROF_NONE_
#define EC_QPROF(w, k) EC_STEPPROF_NONE_
#endif
#if defined(ASB_PROFILE_APPLY)
#define EC_APROF_T0() EC_STEPPROF_T0_
#define EC_APROF(w, k) EC_STEPPROF_(w, k)
#else
#define EC_APROF_T0() EC_STEPPROF_NONE_
#define EC_APROF(w, k) EC_STEPPROF_NONE_
#endif
#if defined(ASB_PROFILE_EPOCH)
#define EC_EPROF_T0() EC_STEPPROF_T0_
#define EC_EPROF(w, k) EC_STEPPROF_(w, k)
#else
#define EC_EPROF_T0() EC_STEPPROF_NONE_
#define EC_EPROF(w, k) EC_STEPPROF_NONE_
#endif
#if defined(ASB_PROFILE_SPEC)
#define EC_PPROF_T0() EC_STEPPROF_T0_
#define EC_PPROF(w, k) EC_STEPPROF_(w, k)
#else
#define EC_PPROF_T0() EC_STEPPROF_NONE_
#define EC_PPROF(w, k) EC_STEPPROF_NONE_
#endif

/* optional phase timing (built with -DASB_PROFILE): cycles per engine phase
 * accumulated by lane 0 and reported in counters[10..15];
 * -DASB_PROFILE -DASB_PROFILE_WALK times the commit-walk steps instead */
#if defined(ASB_PROFILE_SWEEP)
#define EC_SPROF_T0(w) long long sprof_t0_ = ec_clock()
#define EC_SPROF_ADD(w, k)                                      \
  do {                                                          \
    if (EC_LANE == 0) (w)->prof[k] += ec_clock() - sprof_t0_;   \
  } while (0)
#define EC_SPROF_CNT(w, k)               \
  do {                                   \
    if (EC_LANE == 0) (w)->prof[k] += 1; \
  } while (0)
#else
#define EC_SPROF_T0(w) \
  do {                 \
  } while (0)
#define EC_SPROF_ADD(w, k) \
  do {                     \
  } while (0)
#define EC_SPROF_CNT(w, k) \
  do {                     \
  } while (0)
#endif

#if defined(ASB_PROFILE) && defined(ASB_PROFILE_WALK)
#define EC_WPROF_START(w) \
  do {                    \
    if (EC_LANE == 0) (w)->prof_t = ec_clock(); \
  } while (0)
#define EC_WPROF(w, k)                    \
  do {                                    \
    if (EC_LANE == 0) {                   \
      long long now_ = ec_clock();        \
      (w)->prof[k] += now_ - (w)->prof_t; \
      (w)->prof_t = now_;                 \
    }                                     \
  } while (0)
#define EC_PROF_START(w) \
  do {                   \
  } while (0)
#define EC_PROF(w, k) \
  do {                \
  } while (0)
#elif defined(ASB_PROFILE) && !defined(ASB_PROFILE_SWEEP) && !defined(ASB_PROFILE_SORT) && !defined(ASB_PROFILE_SPEC) && !defined(ASB_PROFILE_EPOCH) && !defined(ASB_PROFILE_APPLY)
#define EC_WPROF_START(w) \
  do {                    \
  } while (0)
#define EC_WPROF(w, k) \
  do {                 \
  } while (0)
#define EC_PROF_START(w)                            \
  do {                                              \
    if (EC_LANE == 0) (w)->prof_t = ec_clock();     \
  } while (0)
#define EC_PROF(w, k)                     \
  do {                                    \
    if (EC_LANE == 0) {                   \
      long long now_ = ec_clock();        \
      (w)->prof[k] += now_ - (w)->prof_t; \
      (w)->prof_t = now_;                 \
    }                                     \
  } while (0)
#else
#define EC_PROF_START(w) \
  do {                   \
  } while (0)
#define EC_PROF(w, k) \
  do {                \
  } while (0)
#define EC_WPROF_START(w) \
  do {                    \
  } while (0)
#define EC_WPROF(w, k) \
  do {                 \
  } while (0)
#endif

/* ----------------------------------------------------------------------------
 * small helpers
 * -------------------------------------------------------------------------- */

EC_DEV int ring_idx(int head, int j, int A) {
  int x = head + j; /* head < A, j < A */
  return x >= A ? x - A : x;
}

EC_DEV bool key_less(unsigned long long ta, unsigned pa, unsigned long long tb, unsigned pb) {
  return ta < tb || (ta == tb && pa < pb);
}

/* horizon key: records are committed only while (t, prio, seq) < (hz_t, hz_p, hz_s) */
EC_DEV bool below_horizon(unsigned long long tb, unsigned pr, long long seq, unsigned long long ht, unsigned hp,
                          long long hs) {
  if (tb != ht) return tb < ht;
  if (pr != hp) return pr < hp;
  return seq < hs;
}

/* next-event bookkeeping: per-agent copy + the alive-slot copy the sweeps read */
template <class G>
EC_DEV void set_event(const G& g, int a, int inst, int prio, double t, long long seq) {
  g.H[a].next_t = t;
  g.H[a].next_prio = prio;
  g.H[a].next_seq = seq;
  const int j = g.H[a].slot;
  EC_STK_EV(&g.sl[j], ec_f32_down(t), slot_meta(inst, prio, a));
}

template <class G>
EC_DEV void clear_event(const G& g, int a, int inst) {
  g.H[a].next_prio = 0;
  EC_STK_EV(&g.sl[g.H[a].slot], EC_INF_F32, slot_meta(inst, 0, a));
}

template <class G>
EC_DEV void set_tp(const G& g, int a, double tp) { EC_STK_F64(&g.sl[g.H[a].slot].tp, tp); }

/* the same three with the alive slot already known (no dependent load of
 * H[a].slot): the apply has it from the speculation's record load */
template <class G>
EC_DEV void set_event_at(const G& g, int a, int j, int inst, int prio, double t, long long seq) {
  g.H[a].next_t = t;
  g.H[a].next_prio = prio;
  g.H[a].next_seq = seq;
  EC_STK_EV(&g.sl[j], ec_f32_down(t), slot_meta(inst, prio, a));
}
template <class G>
EC_DEV void clear_event_at(const G& g, int a, int j, int inst) {
  g.H[a].next_prio = 0;
  EC_STK_EV(&g.sl[j], EC_INF_F32, slot_meta(inst, 0, a));
}
template <class G>
EC_DEV void set_tp_at(const G& g, int j, double tp) { EC_STK_F64(&g.sl[j].tp, tp); }

/* a fresh slot j for agent a: pending on instance `inst`, no throughput yet */
template <class G>
EC_DEV void init_slot(const G& g, int j, int inst, int a) {
  EC_STK_F64(&g.sl[j].tp, EC_INF);
  EC_STK_EV(&g.sl[j], 0.0f, slot_meta(inst, 0, a));
}

template <class W>
EC_COLD4 double svc_time(const W* w, const GP& g, long long turn, int level, int concurrent, int thr) {
  /* service_time, instance.py:184-204 */
  double base = (double)g.prefill[turn] / w->pr[level - 1] + (double)g.decode[turn] / w->dr[level - 1];
  int extra = concurrent - 1 > 0 ? concurrent - 1 : 0;
  double factor = 1.0 + w->sc.interference * (double)extra;
  if (thr) factor *= w->sc.thrash_factor;
  return base * factor;
}

template <class W>
EC_COLD4 void update_power(W* w, int i, double now) {
  /* _update_power, engine.py:321-327 (one lane) */
  Inst& in = w->in[i - 1];
  double wt = in.running > 0 ? w->act[in.level - 1] : w->idle[in.level - 1];
  if (wt != in.watts) {
    in.energy += in.watts * (now - in.t_pow);
    in.t_pow = now;
    in.watts = wt;
  }
}

template <class W>
EC_DEV void sync_thrash(W* w, int i, double now) {
  /* _sync_thrash, engine.py:329-336 (one lane) */
  Inst& in = w->in[i - 1];
  if (in.thr != in.thr_flag) {
    if (in.thr_flag)
      in.thr_time += now - in.thr_since;
    else
      in.thr_since = now;
    in.thr_flag = in.thr;
  }
}

/* _mark_row, engine.py:403-429 (one lane): a row when the instance's key
 * (usage, level, watts, pending, running, thrashing) differs from its last
 * row's, or always when forced (samples, start and end of the run) */
template <class W>
EC_COLD4 void mark_row(W* w, const GP& g, int i, double now, bool force) {
  const Inst& in = w->in[i - 1];
  const long long last = w->ts_last[i - 1];
  if (!force && last >= 0) {
    const AsbTimeseriesRow& p = g.ts_rows[last];
    if (p.context_usage == in.usage && p.level_index == in.level && p.power_watts == in.watts &&
        p.pending_depth == in.fifo_len && p.running_requests == in.running && p.thrashing == in.thr)
      return;
  }
  if (w->ts_n >= g.ts_cap) {
    w->status = ASB_SIMERR_OVERFLOW;
    return;
  }
  AsbTimeseriesRow& r = g.ts_rows[w->ts_n];
  r.time = now;
  r.power_watts = in.watts;
  r.context_usage = in.usage;
  r.instance_id = i;
  r.level_index = in.level;
  r.pending_depth = in.fifo_len;
  r.running_requests = in.running;
  r.thrashing = in.thr;
  r.pad_ = 0;
  w->ts_last[i - 1] = w->ts_n++;
}

/* the handler's row (engine.py:488, 507, 535, 549, 560, 568), lane 0 */
template <class W>
EC_DEV void ts_mark(W* w, const GP& g, int i) {
  if (g.ts_rows) mark_row(w, g, i, w->now, false);
}

/* _on_sample (engine.py:570-572): flush every sample event k*interval that
 * precedes `limit` (samples have the lowest priority: a sample at t runs
 * after every event at t), lane 0 */
template <class W>
EC_COLD4 void ts_samples(W* w, const GP& g, double limit) {
  const double iv = w->sc.record_interval, T = w->sc.sim_duration;
  for (;;) {
    const double st = (double)w->ts_k * iv;
    if (!(st < limit && st < T) || w->status) break;
    for (int i = 1; i <= ec_nm(w); i++) mark_row(w, g, i, st, true);
    w->ts_k++;
  }
}

/* lexicographic argmin over (usage, id), router.py:91,123,150; cand_mode:
 * 0 all instances, 1 reassignment candidates (usage > 0 or current) */
template <class W>
EC_COLD4 int argmin_usage(const W* w, int cand_mode, int current) {
  int best = 0;
  long long bu = 0;
  for (int i = 1; i <= ec_nm(w); i++) {
    long long u = w->in[i - 1].usage;
    if (cand_mode == 1 && !(u > 0 || i == current)) continue;
    if (!best || u < bu) {
      best = i;
      bu = u;
    }
  }
  return best;
}

/* argmin_usage by the whole warp: a lane per instance, one 32-bit REDUX of
 * usage << 7 | id; *ok = false (result unused) when a usage does not fit */
template <class W>
EC_COLD4 int argmin_usage_team(const W* w, int cand_mode, int current, bool* ok) {
  const int M = ec_nm(w);
  unsigned key = 0xffffffffu;
  bool wide = false;
  EC_ILOOP /* per-instance loop: rolled (instruction cache) */
  for (int i = EC_LANE + 1; i <= M; i += EC_TSIZE) {
    const long long u = w->in[i - 1].usage;
    if (cand_mode == 1 && !(u > 0 || i == current)) continue;
    wide |= u < 0 || u >= (1ll << 25);
    const unsigned kk = ((unsigned)u << 7) | (unsigned)(i - 1);
    key = kk < key ? kk : key;
  }
  *ok = !t_ballot(wide);
  const unsigned mn = t_redux_min_u32(key);
  return mn == 0xffffffffu ? 0 : (int)(mn & 127u) + 1;
}

/* maybe_reassign decision once the counter reached the interval (router.py:110-128) */
template <class W>
EC_COLD4 int reassign_target(const W* w, int current) {
  int best = argmin_usage(w, w->sc.include_idle ? 0 : 1, current);
  if (best && best != current &&
      (double)w->in[current - 1].usage >= w->sc.imbalance_ratio * (double)w->in[best - 1].usage)
    return best;
  return 0;
}

/* arrival routing, engine.py:496-503 / router.py:75-94,131-151 (lane 0) */
template <class W>
EC_COLD4 int route_arrival(W* w) {
  const AsbScenario& sc = w->sc;
  if (sc.policy == ASB_POLICY_ROUND_ROBIN) {
    int t = (w->rr_next % ec_nm(w)) + 1;
    w->rr_next++;
    return t;
  }
  if (sc.policy == ASB_POLICY_LEAST_LOADED) return argmin_usage(w, 0, 0);
  double threshold = sc.consolidation_threshold * (double)sc.capacity;
  for (int i = 1; i <= ec_nm(w); i++)
    if ((double)w->in[i - 1].usage < threshold) return i;
  return argmin_usage(w, 0, 0);
}

/* _on_arrival bookkeeping after routing (engine.py:490-507), lane 0 */
template <class W>
EC_COLD4 void commit_arrival(W* w, const GP& g, int a, int target, int order_pos) {
  Inst& dst = w->in[target - 1];
  g.ring[(long long)(target - 1) * g.A + ring_idx(dst.fifo_head, dst.fifo_len, g.A)] = a;
  dst.fifo_len++;
  g.H[a].inst = target;
  g.H[a].sa = 0;
  g.H[a].phase = ASB_PHASE_PENDING;
  g.H[a].next_prio = 0;
  const int j = w->n_alive++;
  g.H[a].slot = j;
  init_slot(g, j, target, a);
  g.rank[a] = w->arr_rank++;
  w->arr_ptr = order_pos + 1;
  w->ctr[ASB_CTR_ARRIVED]++;
}

/* add agents whose next event changed during the epoch (re-timed or just
 * admitted) to the due candidates, once each (team; `cand` per lane) */
template <class W, int DCAP, class G>
EC_DEV void add_candidate_at(W* w, const G& g, int a, bool cand, int stamp, double t) {
  /* add_candidates with the agent's dedup stamp and next event time known */
  const bool add = cand && a >= 0 && stamp != w->cand_token && (w->incl ? t <= w->bound : t < w->bound);
  if (add) {
    const int pos = t_atomic_add_i(&w->n_cand, 1);
    if (pos < DCAP) w->due[pos] = a;
    g.dstamp[a] = w->cand_token;
  }
}

template <class W, int DCAP, class G>
EC_DEV void add_candidates(W* w, const G& g, int a, bool cand) {
  bool add = false;
  if (cand && a >= 0 && g.dstamp[a] != w->cand_token) {
    const double t = g.H[a].next_t;
    add = w->incl ? t <= w->bound : t < w->bound;
  }
  if (add) {
    const int pos = t_atomic_add_i(&w->n_cand, 1);
    if (pos < DCAP) w->due[pos] = a;
    g.dstamp[a] = w->cand_token;
  }
}

/* ----------------------------------------------------------------------------
 * running log: insertion-ordered `inst.running` (engine.py:239, 398, 517)
 * -------------------------------------------------------------------------- */

/* Iterate instance i's running log in insertion order; live entries are
 * compacted to the front; if `retime`, each live turn is re-timed
 * (engine.py:355-372) with push sequence numbers seq0, seq0+1, ...  Returns
 * the number of live entries (== running turns).  (team) */
template <class W, int DCAP = 0>
EC_COLD2 int log_pass(W* w, const GP& gp, int i, int retime, long long seq0, double now, bool collect = false,
                    bool count = true) {
  EC_GVIEW(W, gp);
  Inst& in = w->in[i - 1];
  const int len = in.log_len;
  int* lg = g.log + (long long)(i - 1) * g.A;
  const int level = in.level, running = in.running, thr = in.thr;
  int out = 0;
  EC_DBG(9, len);
  for (int base = 0; base < len; base += EC_TSIZE) {
    EC_DBG(10, base);
    int p = base + EC_LANE;
    int a = -1;
    bool live = false;
    if (p < len) {
      a = lg[p];
      live = g.H[a].phase == ASB_PHASE_RUNNING && g.H[a].inst == i && g.H[a].logpos == p;
    }
    unsigned m = t_ballot(live);
    int pos = out + ec_popc(m & t_lt_mask());
    t_sync(); /* every lane has read its entry before any entry is rewritten */
    if (live) {
      if (retime) {
        double anchor = g.H[a].anchor, done = g.H[a].done, rem = g.H[a].rem;
        double segment = done - anchor;
        if (segment > 0) {
          double fraction_done = (now - anchor) / segment;
          double x = 1.0 - fraction_done;
          rem *= (x > 0.0 ? x : 0.0);
        }
        long long turn = g.aturn[a] + g.H[a].steps;
        double full = svc_time(w, gp, turn, level, running, thr);
        done = now + rem * full;
        g.H[a].anchor = now;
        g.H[a].rem = rem;
        g.H[a].done = done;
        set_event(g, a, i, EV_COMPLETE, done, seq0 + pos);
      }
      g.H[a].logpos = pos;
      lg[pos] = a;
    }
    out += ec_popc(m);
    t_sync();
    if (DCAP > 0 && collect) add_candidates<W, DCAP>(w, g, live ? a : -1, retime && live);
  }
  EC_LANE0 {
    in.log_len = out;
    if (retime && count) w->ctr[ASB_CTR_RETIMES] += out;
  }
  t_sync();
  return out;
}

/* _conditions_changed, engine.py:344-372 (team, serial context: uses w->seq) */
template <class W>
EC_COLD2 void cond_changed(W* w, const GP& g, int i) {
  EC_LANE0 {
    Inst& in = w->in[i - 1];
    int kr = w->sc.interference > 0 ? in.running : 0;
    int changed = !(in.key_valid && in.key_level == in.level && in.key_thr == in.thr && in.key_run == kr);
    if (changed) {
      in.key_valid = 1;
      in.key_level = in.level;
      in.key_thr = in.thr;
      in.key_run = kr;
    }
    w->flag = changed && in.log_len > 0;
  }
  t_sync();
  if (w->flag) {
    /* re-timed turns that now fall inside the window become due candidates
     * when a coupling follow-up keeps the batch's due list (cand_collect) */
    int cnt = log_pass<W, W::DC>(w, g, i, 1, w->seq, w->now, w->cand_collect != 0);
    EC_LANE0 w->seq += cnt;
    t_sync();
  }
}

/* append agent a to instance i's running log (one lane); returns position */
template <class W>
EC_DEV int log_append(W* w, const GP& g, int i, int a) {
  Inst& in = w->in[i - 1];
  int p = in.log_len++;
  g.log[(long long)(i - 1) * g.A + p] = a;
  return p;
}

/* ----------------------------------------------------------------------------
 * serial handlers (exact reference semantics on committed state) — team
 * -------------------------------------------------------------------------- */

template <class W>
EC_DEV void count_flip(W* w, int i, double now) {
  Inst& in = w->in[i - 1];
  if (in.thr != in.thr_flag) w->ctr[ASB_CTR_THRASH_FLIPS]++;
  sync_thrash(w, i, now);
}

/* _start_turn, engine.py:374-401 */
template <class W>
EC_COLD2 void start_turn_serial(W* w, const GP& g, int i, int a, double issue) {
  EC_LANE0 w->in[i - 1].running += 1;
  t_sync();
  cond_changed(w, g, i);
  const bool full = w->in[i - 1].log_len >= g.A;
  t_sync(); /* every lane has read log_len before lane 0 appends */
  if (full) log_pass(w, g, i, 0, 0, w->now);
  EC_LANE0 {
    Inst& in = w->in[i - 1];
    double now = w->now;
    long long turn = g.aturn[a] + g.H[a].steps;
    double dur = svc_time(w, g, turn, in.level, in.running, in.thr);
    g.H[a].issue = issue;
    g.H[a].anchor = now;
    g.H[a].rem = 1.0;
    g.H[a].done = now + dur;
    g.H[a].phase = ASB_PHASE_RUNNING;
    set_event(g, a, i, EV_COMPLETE, now + dur, w->seq++);
    g.H[a].start_rank = w->start_ctr++;
    g.H[a].logpos = log_append(w, g, i, a);
    update_power(w, i, now);
  }
  t_sync();
}

/* _on_complete, engine.py:509-535 */
template <class W>
EC_COLD2 void complete_serial(W* w, const GP& gp, int a) {
  EC_GVIEW(W, gp);
  int i = g.H[a].inst;
  EC_LANE0 {
    Inst& in = w->in[i - 1];
    double now = w->now;
    in.running -= 1;
    double llm = now - g.H[a].issue;
    long long turn = g.aturn[a] + g.H[a].steps;
    int p = g.prefill[turn], d = g.decode[turn];
    long long ctx = g.H[a].ctx + p + d;
    int steps = g.H[a].steps + 1;
    long long dec = g.H[a].dec + d;
    double lt = g.H[a].llm + llm;
    g.H[a].ctx = ctx;
    g.H[a].steps = steps;
    g.H[a].dec = dec;
    g.H[a].llm = lt;
    if (ctx > g.H[a].maxctx) g.H[a].maxctx = ctx;
    in.usage += p + d;
    w->ctr[ASB_CTR_TURNS]++;
    w->ctr[ASB_CTR_EVENTS]++;
    if (g.turn_issue) {
      long long lt_idx = turn - g.turn_base;
      g.turn_issue[lt_idx] = g.H[a].issue;
      g.turn_done[lt_idx] = now;
    }
    int n_turns = (int)(g.aturn[a + 1] - g.aturn[a]);
    if (steps == n_turns) {
      in.usage -= ctx;
      g.H[a].phase = ASB_PHASE_DONE;
      g.ctime[a] = now;
      set_tp(g, a, EC_NAN);
      clear_event(g, a, i);
      w->ctr[ASB_CTR_COMPLETED]++;
    } else {
      g.H[a].phase = ASB_PHASE_TOOL;
      set_tp(g, a, (double)dec / lt);
      set_event(g, a, i, EV_TOOL, now + g.tool[turn], w->seq++);
    }
    in.thr = in.usage > w->sc.capacity;
    count_flip(w, i, now);
  }
  t_sync();
  cond_changed(w, gp, i);
  EC_LANE0 {
    update_power(w, i, w->now);
    ts_mark(w, gp, i);
  }
  t_sync();
}

/* _on_tool, engine.py:537-561 */
template <class W>
EC_COLD2 void tool_serial(W* w, const GP& gp, int a) {
  EC_GVIEW(W, gp);
  int source = g.H[a].inst;
  /* the reassignment check's argmin over the instances by the whole warp
   * (many instances: a serial loop on lane 0 would dominate the event) */
  int team_target = 0;
  bool team_ok = false;
  if (W::MX > 1 && w->sc.policy == ASB_POLICY_CONTEXT_AWARE && g.H[a].sa + 1 >= w->sc.reassign_interval) {
    const int best = argmin_usage_team(w, w->sc.include_idle ? 0 : 1, source, &team_ok);
    team_target = best && best != source &&
                          (double)w->in[source - 1].usage >= w->sc.imbalance_ratio * (double)w->in[best - 1].usage
                      ? best
                      : 0;
  }
  t_sync(); /* every lane has read the source before lane 0 migrates the agent */
  EC_LANE0 {
    int target = 0;
    w->ctr[ASB_CTR_EVENTS]++;
    if (w->sc.policy == ASB_POLICY_CONTEXT_AWARE) {
      int sa = g.H[a].sa + 1;
      if (sa >= w->sc.reassign_interval) {
        target = team_ok ? team_target : reassign_target(w, source);
        if (target || !w->sc.reset_only_on_reassign) sa = 0;
      }
      g.H[a].sa = sa;
    }
    w->flag = target;
    if (target) {
      double now = w->now;
      Inst& src = w->in[source - 1];
      Inst& dst = w->in[target - 1];
      g.H[a].mig += 1;
      w->ctr[ASB_CTR_MIGRATIONS]++;
      /* migrate_context, router.py:154-176 */
      src.usage -= g.H[a].ctx;
      src.thr = src.usage > w->sc.capacity;
      g.ring[(long long)(target - 1) * g.A + ring_idx(dst.fifo_head, dst.fifo_len, g.A)] = a;
      dst.fifo_len++;
      g.H[a].inst = target;
      g.H[a].phase = ASB_PHASE_PENDING;
      g.pissue[a] = now;
      g.notbefore[a] = now + w->sc.migration_delay;
      clear_event(g, a, target);
      count_flip(w, source, now);
    }
  }
  t_sync();
  if (!w->flag) {
    start_turn_serial(w, gp, source, a, w->now);
    EC_LANE0 ts_mark(w, gp, source);
    t_sync();
    return;
  }
  cond_changed(w, gp, source);
  EC_LANE0 {
    update_power(w, source, w->now);
    ts_mark(w, gp, source);
    ts_mark(w, gp, g.H[a].inst); /* the target, engine.py:560-561 */
  }
  t_sync();
}

template <class W>
EC_COLD2 void exec_serial(W* w, const GP& g, const Rec& r) {
  EC_DBG(7, r.prio * 1000000 + r.agent);
  EC_LANE0 w->now = r.t;
  t_sync();
  if (r.prio == EV_COMPLETE) {
    complete_serial(w, g, r.agent);
  } else if (r.prio == EV_TOOL) {
    tool_serial(w, g, r.agent);
  } else {
    EC_LANE0 w->ctr[ASB_CTR_EVENTS]++;
    t_sync();
    const int i = g.H[r.agent].inst;
    start_turn_serial(w, g, i, r.agent, g.H[r.agent].issue);
    EC_LANE0 ts_mark(w, g, i); /* _on_delayed_start, engine.py:563-568 */
    t_sync();
  }
}

/* ----------------------------------------------------------------------------
 * speculation cursor: one agent's own event chain (lane-local)
 * -------------------------------------------------------------------------- */


template <class G>
EC_DEV void cur_load(const G& g, Cur& c, int a, long long* next_seq = nullptr, bool with_turns = true) {
  const AgentHot h = g.H[a]; /* one line, 128-bit loads */
  if (next_seq) *next_seq = h.next_seq;
  c.a = a;
  c.inst = h.inst;
  c.phase = h.phase;
  c.slot = h.slot;
  c.prio = h.next_prio;
  c.t = h.next_t;
  c.steps = h.steps;
  c.turn0 = g.aturn[a];
  c.n_turns = (int)(g.aturn[a + 1] - c.turn0);
  c.sa = h.sa;
  c.llm = h.llm;
  c.issue = h.issue;
  c.anchor = h.anchor;
  c.rem = h.rem;
  c.done = h.done;
  c.ctx = h.ctx;
  c.dec = h.dec;
  c.maxctx = h.maxctx;
  if (!with_turns) { /* the apply replays records: no turn data needed */
    c.pf_step = -2;
    return;
  }
  /* the turn data the next two events read (complete: turn k; issue: k or k+1) */
  const long long k = c.turn0 + c.steps;
  const bool ok0 = c.steps < c.n_turns, ok1 = c.steps + 1 < c.n_turns;
  c.pf_step = c.steps;
  c.pf_p0 = ok0 ? g.prefill[k] : 0;
  c.pf_d0 = ok0 ? g.decode[k] : 0;
  c.pf_tool0 = ok0 ? g.tool[k] : 0.0;
  c.pf_p1 = ok1 ? g.prefill[k + 1] : 0;
  c.pf_d1 = ok1 ? g.decode[k + 1] : 0;
}

/* prefill / decode tokens of the cursor's current turn (prefetched when possible) */
template <class G>
EC_DEV void cur_turn_pd(const G& g, const Cur& c, int& p, int& d) {
  if (c.steps == c.pf_step) {
    p = c.pf_p0;
    d = c.pf_d0;
  } else if (c.steps == c.pf_step + 1) {
    p = c.pf_p1;
    d = c.pf_d1;
  } else {
    const long long turn = c.turn0 + c.steps;
    p = g.prefill[turn];
    d = g.decode[turn];
  }
}

/* service_time (instance.py:184-204) from the token counts */
template <class W>
EC_COLD4 double svc_time_pd(const W* w, int p, int d, int level, int concurrent, int thr) {
  double base = (double)p / w->pr[level - 1] + (double)d / w->dr[level - 1];
  int extra = concurrent - 1 > 0 ? concurrent - 1 : 0;
  double factor = 1.0 + w->sc.interference * (double)extra;
  if (thr) factor *= w->sc.thrash_factor;
  return base * factor;
}

/* Advance the cursor over its next event, filling record r.  Mirrors the
 * agent-local part of _on_complete / _on_tool / _on_delayed_start. Returns
 * false on an event-order violation (child scheduled at or before parent). */
template <class W, class G>
EC_DEV bool cur_step(const W* w, const G& g, Cur& c, Rec& r, bool apply) {
  r.t = c.t;
  r.prio = (short)c.prio;
  r.agent = c.a;
  r.inst = c.inst;
  r.flags = 0;
  r.child = -1;
  if (c.prio == EV_COMPLETE) {
    long long turn = c.turn0 + c.steps;
    int p, d;
    cur_turn_pd(g, c, p, d);
    const double tool = c.steps == c.pf_step ? c.pf_tool0 : g.tool[turn];
    double llm = c.t - c.issue;
    if (apply && g.turn_issue) {
      g.turn_issue[turn - g.turn_base] = c.issue;
      g.turn_done[turn - g.turn_base] = c.t;
    }
    c.ctx += p + d;
    c.steps += 1;
    c.dec += d;
    c.llm += llm;
    if (c.ctx > c.maxctx) c.maxctx = c.ctx;
    r.delta = p + d;
    r.dd = d;
    r.aux64 = c.ctx;
    if (c.steps == c.n_turns) {
      r.flags |= F_LAST;
      c.phase = ASB_PHASE_DONE;
      c.prio = 0;
      r.nt = c.t;
    } else {
      c.phase = ASB_PHASE_TOOL;
      c.prio = EV_TOOL;
      c.t = c.t + tool;
      r.nt = c.t;
    }
    return true;
  }
  /* EV_TOOL (issue = now) or EV_ISSUE (issue carried in c.issue) */
  if (c.prio == EV_TOOL) {
    c.issue = c.t;
    if (w->sc.policy == ASB_POLICY_CONTEXT_AWARE) {
      c.sa += 1;
      if (c.sa >= w->sc.reassign_interval) {
        r.flags |= F_CHECK;
        if (!w->sc.reset_only_on_reassign) c.sa = 0;
      }
    }
  }
  const Inst& in = w->in[c.inst - 1];
  int p, d;
  cur_turn_pd(g, c, p, d);
  double dur = svc_time_pd(w, p, d, in.level, in.running, in.thr);
  double t0 = c.t;
  c.anchor = t0;
  c.rem = 1.0;
  c.done = t0 + dur;
  c.phase = ASB_PHASE_RUNNING;
  c.prio = EV_COMPLETE;
  c.t = c.done;
  r.nt = c.t;
  return c.t > t0;
}

/* Re-apply a committed record to the cursor from the record alone (no trace
 * reads): the write-back half of cur_step. */
template <class W, class G>
EC_DEV void cur_apply(const W* w, const G& g, Cur& c, const Rec& r) {
  if (r.prio == EV_COMPLETE) {
    if (g.turn_issue) {
      const long long turn = c.turn0 + c.steps;
      g.turn_issue[turn - g.turn_base] = c.issue;
      g.turn_done[turn - g.turn_base] = r.t;
    }
    const double llm = r.t - c.issue;
    c.ctx += r.delta;
    c.steps += 1;
    c.dec += r.dd;
    c.llm += llm;
    if (c.ctx > c.maxctx) c.maxctx = c.ctx;
    if (r.flags & F_LAST) {
      c.phase = ASB_PHASE_DONE;
      c.prio = 0;
      c.t = r.t;
    } else {
      c.phase = ASB_PHASE_TOOL;
      c.prio = EV_TOOL;
      c.t = r.nt;
    }
    return;
  }
  if (r.prio == EV_TOOL) {
    c.issue = r.t;
    if (w->sc.policy == ASB_POLICY_CONTEXT_AWARE) {
      c.sa += 1;
      if (c.sa >= w->sc.reassign_interval && !w->sc.reset_only_on_reassign) c.sa = 0;
    }
  }
  c.anchor = r.t;
  c.rem = 1.0;
  c.done = r.nt;
  c.phase = ASB_PHASE_RUNNING;
  c.prio = EV_COMPLETE;
  c.t = r.nt;
}

/* ----------------------------------------------------------------------------
 * epoch event
 * -------------------------------------------------------------------------- */

/* ----------------------------------------------------------------------------
 * fork-join over the team's helper warps
 * -------------------------------------------------------------------------- */
template <class W>
EC_DEV void do_job(W* w, int job, int tid, int nthr);

/* main warp: release the helper warps on `job`, take part as threads
 * [0, 32), and join.  Helpers run helper_loop().  (1-lane host build: the
 * job simply runs on the single lane.) */
template <class W>
EC_DEV void fork_job(W* w, int job) {
  EC_LANE0 w->job = job;
  t_sync();
  ec_fork_begin(W::NT);
  do_job(w, job, EC_TID_OF(W::NT), W::NT);
  ec_fork_end(W::NT);
}

template <class W>
EC_DEV void helper_loop(W* w) {
  for (;;) {
    ec_fork_begin(W::NT);
    const int job = w->job;
    if (job == JOB_EXIT) break;
    do_job(w, job, EC_TID_OF(W::NT), W::NT);
    ec_fork_end(W::NT);
  }
}

/* JOB_SWEEP (thread-level, all warps): one pass over the alive slots.
 * j_tick: per-instance min running throughput (per-thread partials, then a
 * warp reduction into wpart) and the finished-slot count; j_collect: agents
 * whose next event falls before j_bound become due candidates (stamped
 * j_token). */
template <class W>
EC_COLD1 void job_sweep(W* w, const GP& g, int tid, int nthr) {
  constexpr int U = W::NT == 128 ? EC_SWEEP_UNROLL_QUAD : EC_SWEEP_UNROLL;
  const bool tick = w->j_tick, collect = w->j_collect != 0, count_only = w->j_collect == 2;
  const double bound = w->j_bound;
  /* the slots hold next-event times rounded down to f32: comparing them
   * with the bound is a conservative due test (see Slot) */
  const int incl = w->j_incl, token = w->j_token;
  const int n = w->n_alive;
  int dead = 0, counted = 0;
  /* the scenario's pointers in registers: read through the shared GP they
   * would be reloaded after every shared-memory store of the loop */
  const Slot* const sl = g.sl;
  int* const dstamp = g.dstamp;
  const AgentHot* const hot = g.H;
  const long long* const aturn = g.aturn;
#if defined(ASB_PROFILE_SWEEP)
  const long long js_t0 = ec_clock();
#endif
  /* software-pipelined: the next chunk's 16-byte slot loads are in flight
   * while this chunk is folded */
  double tp[U], tp2[U];
  float nx[U], nx2[U];
  int mt[U], mt2[U];
#pragma unroll
  for (int u = 0; u < U; u++) {
    const int j = u * nthr + tid;
    mt[u] = -1;
    if (j < n) EC_LDK_SLOT(&sl[j], tp[u], nx[u], mt[u]);
  }
  for (int base = 0; base < n; base += nthr * U) {
    const int nb = base + nthr * U;
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int j = nb + u * nthr + tid;
      mt2[u] = -1;
      if (j < n) EC_LDK_SLOT(&sl[j], tp2[u], nx2[u], mt2[u]);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (mt[u] < 0) continue;
      if (collect && sm_prio(mt[u]) > 0 && (incl ? (double)nx[u] <= bound : (double)nx[u] < bound)) {
        if (count_only) {
          counted++;
        } else {
          const int a = sm_agent(mt[u]);
          const int pos = t_atomic_add_i(&w->j_total, 1);
          if (pos < W::DC) w->due[pos] = a;
          dstamp[a] = token;
          /* the speculation reads this agent's record and turn offsets after
           * the epoch: start bringing them into L2 now (not on the 16-warp
           * team, whose sweeps collect hundreds: C4 +4% with it) */
          if (W::NT < 512) {
            EC_PREFETCH_L2(&hot[a]);
            EC_PREFETCH_L2(&aturn[a]);
          }
        }
      }
      if (!tick) continue;
      /* throughputs are >= 0, so the f64 bit patterns order like the values;
       * +inf = None (no LLM time yet) never lowers the min; the positive
       * quiet NaN marks a finished agent (not in process) */
      const unsigned long long b = ec_bits(tp[u]);
      if (b > EC_INF_BITS)
        dead++;
      else if (b < w->tmin[sm_inst(mt[u]) - 1])
        t_atomic_min_ull(&w->tmin[sm_inst(mt[u]) - 1], b);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      mt[u] = mt2[u];
      tp[u] = tp2[u];
      nx[u] = nx2[u];
    }
  }
  if (tick && dead) t_atomic_add_i(&w->j_dead, dead);
  if (counted) t_atomic_add_i(&w->j_total, counted);
#if defined(ASB_PROFILE_SWEEP)
  /* a helper's (thread 32's) time inside the tick sweeps: load rounds + fold */
  if (tid == 32 && tick) w->prof[2] += ec_clock() - js_t0;
#endif
}

/* agent-tick sweep (main warp): fork the slot sweep, fold the partial
 * minima into tmin (controller.py:89-103, engine.py:437-454), count the
 * ticks, and compact finished agents out lazily. */
template <class W>
EC_COLD3 void tick_sweep(W* w, const GP& g, bool collect, double bound, int incl, int) {
  const int M = ec_nm(w);
  const int n = w->n_alive;
  const int token = w->stamp_ctr + 1; /* a fresh stamp per due list */
  EC_LANE0 {
    w->stamp_ctr = token;
    w->j_tick = 1;
    w->j_collect = collect;
    w->j_bound = bound;
    w->j_incl = incl;
    w->j_token = token;
    w->j_dead = 0;
    w->j_total = 0;
  }
  EC_ILOOP /* per-instance loop: rolled (instruction cache) */
  for (int i = EC_LANE; i < M; i += EC_TSIZE) w->tmin[i] = EC_INF_BITS; /* the sweep's smem atomics fold into it */
  EC_SPROF_T0(w);
  fork_job(w, JOB_SWEEP);
  EC_SPROF_ADD(w, 0);
  const int dead_all = w->j_dead;
  EC_LANE0 {
    w->ctr[ASB_CTR_TICKS] += n - dead_all;
    w->n_cand = collect ? w->j_total : 0;
    w->cand_token = token;
  }
  if (dead_all * 4 > n && dead_all > 0) {
    /* order-free compaction of the slots (in place: write index <= read index) */
    int out = 0;
    for (int base = 0; base < n; base += EC_TSIZE) {
      int j = base + EC_LANE;
      bool live = false;
      int a = -1, mt = 0;
      double tp = 0.0;
      float nx = 0.0f;
      if (j < n) {
        EC_LDK_SLOT(&g.sl[j], tp, nx, mt);
        live = !ec_isnan(tp);
        a = sm_agent(mt);
      }
      unsigned m = t_ballot(live);
      t_sync();
      if (live) {
        const int o = out + ec_popc(m & t_lt_mask());
        EC_STK_F64(&g.sl[o].tp, tp);
        EC_STK_EV(&g.sl[o], nx, mt);
        g.H[a].slot = o;
      }
      out += ec_popc(m);
      t_sync();
    }
    EC_LANE0 w->n_alive = out;
  }
  t_sync();
}

/* β/γ FIFO admission as a prefix scan (controller.py:112-130); returns count (team) */
template <class W>
EC_COLD3 int admission(W* w, const GP& gp, int i, double gcap, int* n_start = nullptr) {
  EC_GVIEW(W, gp);
  Inst& in = w->in[i - 1];
  const int len = in.fifo_len, head = in.fifo_head;
  const int* ring = g.ring + (long long)(i - 1) * g.A;
  const double now = w->now;
  long long usage = in.usage;
  int n_adm = 0, n_st = 0;
  if (!((double)usage < gcap)) {
    /* the head cannot be admitted (controller.py:121): nothing changes */
    if (n_start) *n_start = 0;
    return 0;
  }
  for (int base = 0; base < len; base += EC_TSIZE) {
    int j = base + EC_LANE;
    bool valid = j < len;
    int a = valid ? ring[ring_idx(head, j, g.A)] : -1;
    long long c = valid ? g.H[a].ctx : 0;
    const double nb = valid ? g.notbefore[a] : 0.0;
    /* prefix sums of the pending contexts: 32-bit when every one is below
     * 2^26 (32 of them cannot overflow), else 64-bit */
    long long incl;
    if (!t_ballot(c >= (1ll << 26)))
      incl = t_scan_add_i((int)c);
    else
      incl = t_scan_add_ll(c);
    long long excl = incl - c;
    bool ok = valid && (double)(usage + excl) < gcap;
    unsigned m = t_ballot(ok);
    n_st += ec_popc(t_ballot(ok && !(now < nb)));
    int cnt = ec_popc(m);
    if (cnt) usage += t_bcast_ll(incl, cnt - 1);
    n_adm += cnt;
    if (cnt < EC_TSIZE) break;
  }
  if (n_start) *n_start = n_st;
  t_sync();
  EC_LANE0 {
    in.usage = usage;
    in.fifo_head = ring_idx(head, n_adm, g.A);
    in.fifo_len = len - n_adm;
    in.thr = usage > w->sc.capacity;
  }
  t_sync();
  return n_adm;
}

/* level select + SLO boost for instance i at the epoch (controller.py:81-86,147-163) */
template <class W>
EC_COLD4 int choose_level(const W* w, int i, int* boosted) {
  const AsbScenario& sc = w->sc;
  const int L = sc.n_levels;
  const long long usage = w->in[i - 1].usage;
  int level;
  if (sc.variant == ASB_VARIANT_OFF)
    level = L;
  else if (sc.variant == ASB_VARIANT_FIXED)
    level = sc.fixed_level;
  else {
    double ac = sc.alpha * (double)sc.capacity;
    if ((double)usage >= ac)
      level = L;
    else
      level = (int)ec_floor((double)usage / ac * (double)(L - 1)) + 1;
  }
  *boosted = 0;
  const bool has_tp = w->tmin[i - 1] != EC_INF_BITS;
  if (sc.variant == ASB_VARIANT_CONTEXT_AWARE && sc.boost_enabled && has_tp &&
      ec_from_bits(w->tmin[i - 1]) < sc.slo_target) {
    level = L;
    *boosted = 1;
  }
  return level;
}

/* start the admitted agents' turns of instance i (engine.py:458-473), no
 * interference: durations are independent, pushes numbered from seq0 (team) */
template <class W, int DCAP>
EC_COLD3 void start_admitted(W* w, const GP& gp, int i, int head0, int n_adm, long long seq0, long long rank0,
                           bool collect) {
  EC_GVIEW(W, gp);
  Inst& in = w->in[i - 1];
  if (in.log_len + n_adm > g.A) log_pass(w, gp, i, 0, 0, w->now);
  const int log0 = in.log_len, lvl = in.level, thr = in.thr;
  const double now = w->now;
  int started = 0;
  for (int base = 0; base < n_adm; base += EC_TSIZE) {
    int j = base + EC_LANE;
    bool valid = j < n_adm;
    int a = valid ? g.ring[(long long)(i - 1) * g.A + ring_idx(head0, j, g.A)] : -1;
    bool start = false;
    double issue = 0.0, nb = 0.0, t_next = 0.0;
    int slot = 0, steps = 0, stamp = 0;
    long long turn0 = 0;
    if (valid) {
      /* everything this agent's start reads, in one round of independent
       * loads after the FIFO entry (no dependent reload of H[a] fields) */
      double pi = g.pissue[a];
      nb = g.notbefore[a];
      slot = g.H[a].slot;
      steps = g.H[a].steps;
      turn0 = g.aturn[a];
      if (collect) stamp = g.dstamp[a];
      issue = ec_isnan(pi) ? now : pi;
      g.pissue[a] = EC_NAN;
      start = !(now < nb);
    }
    unsigned m = t_ballot(start);
    int sidx = started + ec_popc(m & t_lt_mask());
    if (valid) {
      g.H[a].issue = issue;
      if (!start) {
        g.H[a].phase = ASB_PHASE_WAITING_START;
        t_next = nb;
        set_event_at(g, a, slot, i, EV_ISSUE, nb, seq0 + j);
      } else {
        double dur = svc_time(w, gp, turn0 + steps, lvl, 0, thr);
        t_next = now + dur;
        g.H[a].anchor = now;
        g.H[a].rem = 1.0;
        g.H[a].done = t_next;
        g.H[a].phase = ASB_PHASE_RUNNING;
        set_event_at(g, a, slot, i, EV_COMPLETE, t_next, seq0 + j);
        g.H[a].start_rank = rank0 + sidx;
        g.H[a].logpos = log0 + sidx;
        g.log[(long long)(i - 1) * g.A + log0 + sidx] = a;
      }
    }
    started += ec_popc(m);
    if (collect) add_candidate_at<W, DCAP>(w, g, a, valid, stamp, t_next);
  }
  t_sync();
  EC_LANE0 {
    in.running += started;
    in.log_len += started;
  }
  t_sync();
}

template <class W>
EC_COLD4 void write_decision(W* w, const GP& g, long long k, int i) {
  if (!g.dec_rows) return;
  const Inst& in = w->in[i - 1];
  AsbDecision& d = g.dec_rows[k * ec_nm(w) + (i - 1)];
  d.time = w->now;
  d.min_throughput = w->tmin[i - 1] != EC_INF_BITS ? ec_from_bits(w->tmin[i - 1]) : EC_NAN;
  d.usage_observed = w->ep_uobs[i - 1];
  d.instance_id = i;
  d.frequency_level = w->ep_level[i - 1];
  d.admitted_count = w->ep_nadm[i - 1];
  d.pending_depth = in.fifo_len;
  d.boosted = w->ep_boost[i - 1];
  d.deferred = w->ep_def[i - 1];
}

/* exact serial epoch (interference mode: every start re-times its instance) */
template <class W>
EC_COLD2 void epoch_serial(W* w, const GP& g, long long k) {
  EC_DBG(8, k);
  const AsbScenario& sc = w->sc;
  const int M = ec_nm(w);
  for (int i = 1; i <= M; i++) {
    Inst& in = w->in[i - 1];
    EC_LANE0 {
      int boosted;
      w->ep_uobs[i - 1] = in.usage;
      in.level = w->ep_level[i - 1] = choose_level(w, i, &boosted);
      w->ep_boost[i - 1] = boosted;
    }
    t_sync();
    cond_changed(w, g, i);
    EC_LANE0 update_power(w, i, w->now);
    t_sync();
    double gamma = 1.0, beta = 1.0;
    if (sc.variant == ASB_VARIANT_CONTEXT_AWARE && sc.thrash_avoidance) {
      gamma = sc.gamma;
      beta = sc.beta;
    }
    const int head0 = in.fifo_head;
    const int n_adm = admission(w, g, i, gamma * (double)sc.capacity);
    EC_LANE0 {
      w->ep_nadm[i - 1] = n_adm;
      w->ep_def[i - 1] = (double)in.usage > beta * (double)sc.capacity;
      count_flip(w, i, w->now);
    }
    t_sync();
    cond_changed(w, g, i);
    for (int j = 0; j < n_adm; j++) {
      int a = g.ring[(long long)(i - 1) * g.A + ring_idx(head0, j, g.A)];
      double issue = ec_isnan(g.pissue[a]) ? w->now : g.pissue[a];
      const bool wait = w->now < g.notbefore[a];
      t_sync();
      EC_LANE0 g.pissue[a] = EC_NAN;
      if (wait) {
        EC_LANE0 {
          g.H[a].phase = ASB_PHASE_WAITING_START;
          g.H[a].issue = issue;
          set_event(g, a, i, EV_ISSUE, g.notbefore[a], w->seq++);
        }
        t_sync();
      } else {
        start_turn_serial(w, g, i, a, issue);
      }
    }
    EC_LANE0 {
      update_power(w, i, w->now);
      write_decision(w, g, k, i);
      ts_mark(w, g, i);
    }
    t_sync();
  }
}

/* _on_epoch, engine.py:436-488 + control_epoch, controller.py:133-186 (team).
 * Instances are independent within an epoch except for the instance-major
 * order of their pushes, which an exclusive scan reproduces. */
template <class W, int DCAP>
EC_COLD3 void epoch_event(W* w, const GP& g, long long k) {
  const AsbScenario& sc = w->sc;
  const int M = ec_nm(w);
  const bool collect = sc.interference == 0 && !g.ts_rows;
  EC_PROF_START(w);
  tick_sweep(w, g, collect, w->bound, w->incl, 0);
  EC_PROF(w, 0);
  if (!collect) {
    epoch_serial(w, g, k);
    EC_LANE0 w->due_ready = 0;
    t_sync();
    EC_PROF(w, 1);
    return;
  }
  const double now = w->now;
  const int tid = EC_LANE; /* sub-step profile: lane 0 of the main warp */
  (void)tid;
  EC_EPROF_T0();
  /* (a) lane per instance: observe, level, boost, level-hook power */
  EC_ILOOP /* per-instance loop: rolled (instruction cache) */
  for (int i = EC_LANE + 1; i <= M; i += EC_TSIZE) {
    Inst& in = w->in[i - 1];
    int boosted;
    w->ep_uobs[i - 1] = in.usage;
    in.level = w->ep_level[i - 1] = choose_level(w, i, &boosted);
    w->ep_boost[i - 1] = boosted;
    w->ep_head[i - 1] = in.fifo_head;
    w->ep_nadm[i - 1] = 0;
    w->ep_thr0[i - 1] = in.thr;
    update_power(w, i, now);
  }
  t_sync();
  /* (b) β/γ admission where agents are pending — instances in parallel, one
   * warp each (JOB_ADMIT) */
  const bool ca = sc.variant == ASB_VARIANT_CONTEXT_AWARE && sc.thrash_avoidance;
  const double bcap = (ca ? sc.beta : 1.0) * (double)sc.capacity;
  {
    int cnt = 0;
    EC_ILOOP /* per-instance loop: rolled (instruction cache) */
    for (int r0 = 0; r0 < M; r0 += EC_TSIZE) {
      const int i = r0 + EC_LANE + 1;
      /* pending agents and room below gamma * cap (else admission_pass admits nothing) */
      const bool pend = i <= M && w->in[i - 1].fifo_len > 0 &&
                        (double)w->in[i - 1].usage < (ca ? sc.gamma : 1.0) * (double)sc.capacity;
      if (i <= M) w->ep_nstart[i - 1] = 0;
      const unsigned m = t_ballot(pend);
      if (pend) w->ep_list[cnt + ec_popc(m & t_lt_mask())] = i;
      cnt += ec_popc(m);
    }
    EC_LANE0 {
      w->n_eplist = cnt;
      w->ep_gcap = (ca ? sc.gamma : 1.0) * (double)sc.capacity;
    }
    t_sync();
    EC_EPROF(w, 0); /* (a) and the pending scan */
    if (cnt) {
      EC_SPROF_CNT(w, 5);
      fork_job(w, JOB_ADMIT);
    }
    EC_EPROF(w, 1); /* (b) the admission job */
  }
  /* (c) lane per instance: deferral, thrash sync, rate key, push counts;
   * exclusive scans over instances -> each instance's first push seq and
   * first start rank (the reference pushes / starts instance-major) */
  long long seq_base = w->seq, rank_base = w->start_ctr;
  int flips = 0;
  int extra_retimes = 0, all_retimes = 0; /* per epoch: at most the running agents */
  int nwork = 0;
  constexpr bool single = W::MX == 1; /* one instance: lane 0 holds everything, no scans */
  EC_ILOOP /* per-instance loop: rolled (instruction cache) */
  for (int r0 = 0; r0 < M; r0 += EC_TSIZE) {
    const int i = r0 + EC_LANE + 1;
    int pushes = 0, starts = 0; /* per instance and epoch: at most its agents */
    bool flip = false, work = false;
    if (i <= M) {
      Inst& in = w->in[i - 1];
      w->ep_def[i - 1] = (double)in.usage > bcap;
      flip = in.thr != in.thr_flag;
      sync_thrash(w, i, now);
      /* the reference re-times twice: after the level hook (key (level,
       * thr before admission)) and after admission (thrash flip).  Both at
       * `now`: the second leaves rem unchanged, so one pass with the final
       * key gives the same times; the re-time counter counts both. */
      const int thr0 = w->ep_thr0[i - 1];
      const int changed1 = !(in.key_valid && in.key_level == in.level && in.key_thr == thr0);
      const int changed2 = in.thr != thr0;
      in.key_valid = 1;
      in.key_level = in.level;
      in.key_thr = in.thr;
      in.key_run = 0;
      const int rt = (changed1 || changed2) && in.running > 0 ? in.running : 0;
      w->ep_retime[i - 1] = rt;
      extra_retimes += (changed1 && changed2) ? rt : 0;
      all_retimes += rt;
      pushes = rt + w->ep_nadm[i - 1];
      starts = w->ep_nstart[i - 1];
      work = pushes > 0;
    }
    if (single) { /* lane 0 is instance 1 and the only lane whose values are used */
      flips += flip ? 1 : 0;
      if (i <= M) {
        w->ep_seq[0] = seq_base;
        w->ep_rank[0] = rank_base;
      }
      seq_base += pushes;
      rank_base += starts;
      if (work) w->ep_list[0] = 1;
      nwork += ec_popc(t_ballot(work)); /* warp-uniform: the fork below is taken by the whole warp */
      continue;
    }
    flips += ec_popc(t_ballot(flip));
    const int incl = t_scan_add_i(pushes);
    const int incs = t_scan_add_i(starts);
    if (i <= M) {
      w->ep_seq[i - 1] = seq_base + incl - pushes;
      w->ep_rank[i - 1] = rank_base + incs - starts;
    }
    seq_base += t_shfl_i(incl, EC_TSIZE - 1);
    rank_base += t_shfl_i(incs, EC_TSIZE - 1);
    const unsigned m = t_ballot(work);
    if (work) w->ep_list[nwork + ec_popc(m & t_lt_mask())] = i;
    nwork += ec_popc(m);
  }
  if (!single) {
    extra_retimes = t_redux_add_i(extra_retimes);
    all_retimes = t_redux_add_i(all_retimes);
  }
  t_sync();
  EC_LANE0 {
    w->seq = seq_base;
    w->start_ctr = rank_base;
    w->ctr[ASB_CTR_THRASH_FLIPS] += flips;
    w->ctr[ASB_CTR_RETIMES] += all_retimes + extra_retimes;
    w->n_eplist = nwork;
  }
  t_sync();
  /* (d)+(e) re-time in-flight turns where the rate key changed, then start
   * the admitted turns — instances in parallel, one warp each (JOB_EPOCH) */
  EC_EPROF(w, 2); /* (c) deferral, thrash sync, keys, push scans */
  if (nwork) {
    fork_job(w, JOB_EPOCH);
  }
  EC_EPROF(w, 3); /* (d)+(e) the re-time / start job */
  /* (f) lane per instance: final power, decision rows */
  EC_ILOOP /* per-instance loop: rolled (instruction cache) */
  for (int i = EC_LANE + 1; i <= M; i += EC_TSIZE) {
    update_power(w, i, now);
    write_decision(w, g, k, i);
  }
  EC_LANE0 w->due_ready = w->n_cand <= DCAP;
  t_sync();
  EC_EPROF(w, 4); /* (f) final power, decision rows */
  EC_PROF(w, 1);
}

/* ----------------------------------------------------------------------------
 * optimistic batch
 * -------------------------------------------------------------------------- */

/* count alive agents whose next event is due before `bound`: the whole
 * team sweeps in count-only mode (main warp; forks the sweep) */
template <class W>
EC_COLD3 int count_due(W* w, const GP& g, double bound, int incl) {
  (void)g;
  EC_LANE0 {
    w->j_tick = 0;
    w->j_collect = 2;
    w->j_bound = bound;
    w->j_incl = incl;
    w->j_total = 0;
  }
  fork_job(w, JOB_SWEEP);
  return w->j_total;
}

/* collect due agents into w->due (up to DCAP); returns the total due count
 * (> DCAP means the list is incomplete).  (main warp; forks the sweep) */
template <class W, int DCAP>
EC_DEV int collect_due(W* w, const GP& g, double bound, int incl) {
  EC_LANE0 {
    w->j_tick = 0;
    w->j_collect = 1;
    w->j_bound = bound;
    w->j_incl = incl;
    /* a fresh stamp per due list: candidates added later (re-timed turns)
     * are de-duplicated against this list only */
    w->cand_token = ++w->stamp_ctr;
    w->j_token = w->cand_token;
    w->j_total = 0;
  }
  fork_job(w, JOB_SWEEP);
  return w->j_total;
}

/* Serial commit walk (lane 0): the reference's handlers in (time, prio, seq)
 * order, stopping before the first coupling event.  Used for interference
 * mode and for tie groups whose push order is only known during the walk. */
template <class W>
EC_COLD2 void walk_serial(W* w, const GP& g, const int n) {
  EC_LANE0 {
    const AsbScenario& sc = w->sc;
    int stop = STOP_NONE, stop_idx = -1;
    int p = 0;
    while (p < n && stop == STOP_NONE) {
      const unsigned long long tb = w->srt[p].tb;
      const unsigned pr = w->srt[p].prio;
      if (!key_less(tb, pr, w->hz_t, (unsigned)w->hz_p) && !(tb == w->hz_t && pr == (unsigned)w->hz_p)) {
        stop = STOP_HORIZON;
        break;
      }
      int q = p + 1;
      while (q < n && w->srt[q].tb == tb && w->srt[q].prio == pr) q++;
      if (q - p > 1) {
        /* tie group: order by push sequence (every parent is already walked) */
        for (int x = p + 1; x < q; x++) {
          SortE e = w->srt[x];
          long long sq = w->rec[e.idx].seq;
          int y = x - 1;
          while (y >= p && w->rec[w->srt[y].idx].seq > sq) {
            w->srt[y + 1] = w->srt[y];
            y--;
          }
          w->srt[y + 1] = e;
        }
      }
      for (int x = p; x < q; x++) {
        const int ri = (int)w->srt[x].idx;
        Rec& r = w->rec[ri];
        if (!below_horizon(tb, pr, r.seq, w->hz_t, (unsigned)w->hz_p, w->hz_s)) {
          stop = STOP_HORIZON;
          break;
        }
        const double t = r.t;
        if (r.prio == EV_COMPLETE) {
          Inst& in = w->in[r.inst - 1];
          long long nu = in.usage + r.delta - ((r.flags & F_LAST) ? r.aux64 : 0);
          int flip = (nu > sc.capacity ? 1 : 0) != in.thr;
          if (flip || sc.interference > 0) {
            stop = STOP_COUPLING;
            stop_idx = ri;
            break;
          }
          in.running -= 1;
          in.usage = nu;
          w->ctr[ASB_CTR_TURNS]++;
          w->ctr[ASB_CTR_EVENTS]++;
          if (r.flags & F_LAST) {
            w->ctr[ASB_CTR_COMPLETED]++;
          } else {
            r.push_seq = w->seq++;
            if (r.child >= 0) w->rec[r.child].seq = r.push_seq;
          }
          update_power(w, r.inst, t);
        } else if (r.prio == EV_ARRIVAL) {
          commit_arrival(w, g, r.agent, route_arrival(w), (int)r.seq);
        } else {
          /* EV_TOOL (maybe a reassignment check) or EV_ISSUE, then _start_turn */
          if (((r.flags & F_CHECK) && reassign_target(w, r.inst)) || sc.interference > 0) {
            stop = STOP_COUPLING;
            stop_idx = ri;
            break;
          }
          Inst& in = w->in[r.inst - 1];
          if (in.log_len >= g.A) {
            stop = STOP_LOGFULL;
            stop_idx = ri;
            break;
          }
          in.running += 1;
          r.push_seq = w->seq++;
          if (r.child >= 0) w->rec[r.child].seq = r.push_seq;
          r.aux64 = w->start_ctr++;
          r.logpos = log_append(w, g, r.inst, r.agent);
          w->ctr[ASB_CTR_EVENTS]++;
          update_power(w, r.inst, t);
        }
        r.flags |= F_COMMITTED;
      }
      p = q;
    }
    /* something was dropped (buffer overflow): the window is not exhausted */
    if (stop == STOP_NONE && w->hz_t != EC_INF_BITS) stop = STOP_HORIZON;
    w->stop_kind = stop;
    w->stop_rec = stop_idx;
    if (stop_idx >= 0) w->stop_r = w->rec[stop_idx];
  }
  t_sync();
}

/* usage snapshots for many instances (M > team width): lane per instance,
 * merging its sorted record list with the sorted dependent positions */
template <class W>
EC_COLD4 void snapshots_merge(W* w, int n_dep, int stop_p) {
  const int M = ec_nm(w);
  EC_ILOOP /* per-instance loop: rolled (instruction cache) */
  for (int i = EC_LANE + 1; i <= M; i += EC_TSIZE) {
    const int e1 = w->ioff[i];
    int e = w->ioff[i - 1];
    long long u = w->in[i - 1].usage;
    for (int k = 0; k < n_dep; k++) {
      const int dp = w->dep_pos[k];
      if (dp >= stop_p) break;
      while (e < e1 && w->ilist[e] < dp) {
        u = w->wu[e];
        e++;
      }
      w->snap[k][i - 1] = u;
    }
  }
}

/* lane-serial argmin of (usage, id) over snapshot k (router.py:91,123,150):
 * cand_mode 0 = all instances, 1 = reassignment candidates; 0 = none */
template <class W>
EC_DEV int snap_argmin_lane(const W* w, int k, bool all, int cur, long long* bu_out) {
  const int M = ec_nm(w);
  long long bu = 0;
  int bi = 0;
  for (int i = 1; i <= M; i++) {
    const long long u = w->snap[k][i - 1];
    if (!(all || u > 0 || i == cur)) continue;
    if (!bi || u < bu) {
      bu = u;
      bi = i;
    }
  }
  *bu_out = bu;
  return bi;
}

/* reassignment checks of the dependent records before stop_p, one lane per
 * check (each reads only its own usage snapshot): the position of the
 * first that migrates (maybe_reassign, router.py:110-128), or stop_p */
template <class W>
EC_COLD4 int checks_parallel(const W* w, int n_dep, int stop_p) {
  const AsbScenario& sc = w->sc;
  const bool all = sc.include_idle;
  int first = stop_p;
  for (int k = EC_LANE; k < n_dep; k += EC_TSIZE) {
    const int p = w->dep_pos[k];
    if (p >= stop_p || w->sw_prio[p] != EV_TOOL) continue;
    const int cur = w->sw_inst[p];
    long long bu = 0;
    const int bi = snap_argmin_lane(w, k, all, cur, &bu);
    if (bi && bi != cur && (double)w->snap[k][cur - 1] >= sc.imbalance_ratio * (double)bu && p < first) first = p;
  }
  return (int)t_redux_min_u32((unsigned)first);
}

/* arrival routing of the dependent records before stop_p, one lane per
 * arrival (router.py:75-94,131-151 on its usage snapshot) into
 * w->dep_target[k]; round-robin takes rr_next + its rank among the batch's
 * arrivals */
template <class W>
EC_COLD4 void route_parallel(W* w, int n_dep, int stop_p) {
  const AsbScenario& sc = w->sc;
  const int M = ec_nm(w);
  const double threshold = sc.consolidation_threshold * (double)sc.capacity;
  int before = 0; /* arrivals ahead of this lane's chunk */
  for (int base = 0; base < n_dep; base += EC_TSIZE) {
    const int k = base + EC_LANE;
    const int p = k < n_dep ? w->dep_pos[k] : 0x7fffffff;
    const bool arr = p < stop_p && w->sw_prio[p] == EV_ARRIVAL;
    const unsigned m = t_ballot(arr);
    if (arr) {
      int target;
      if (sc.policy == ASB_POLICY_ROUND_ROBIN) {
        target = (int)(((long long)w->rr_next + before + ec_popc(m & t_lt_mask())) % M) + 1;
      } else {
        int light = 0;
        if (sc.policy == ASB_POLICY_CONTEXT_AWARE)
          for (int i = 1; i <= M && !light; i++)
            if ((double)w->snap[k][i - 1] < threshold) light = i;
        long long bu = 0;
        target = light ? light : snap_argmin_lane(w, k, true, 0, &bu);
      }
      w->dep_target[k] = target;
    }
    before += ec_popc(m);
  }
  t_sync();
}

/* snap_argmin for M > 32: each lane folds its instances into one 32-bit
 * key (usage << IDB | id, IDB = 6 bits of instance id, 7 for the 128-wide
 * kernel), one warp reduction; -1 when a usage does not fit the key */
template <class W>
EC_COLD4 int snap_argmin_wide(const W* w, int k, bool all, int cur, long long* bu_out) {
  constexpr int IDB = W::MX > 64 ? 7 : 6;
  const int M = ec_nm(w);
  unsigned key = 0xffffffffu;
  bool wide = false;
  EC_ILOOP /* per-instance loop: rolled (instruction cache) */
  for (int i = EC_LANE + 1; i <= M; i += EC_TSIZE) {
    const long long u = w->snap[k][i - 1];
    if (!(all || u > 0 || i == cur)) continue;
    wide |= u < 0 || u >= (1ll << (32 - IDB));
    const unsigned kk = ((unsigned)u << IDB) | (unsigned)(i - 1);
    key = kk < key ? kk : key;
  }
  if (t_ballot(wide)) return -1;
  const unsigned mn = t_redux_min_u32(key);
  if (mn == 0xffffffffu) return 0;
  *bu_out = (long long)(mn >> IDB);
  return (int)(mn & ((1u << IDB) - 1u)) + 1;
}

/* Team argmin of (usage, id) over the usage snapshot k (router.py:91,123,150):
 * cand_mode 0 = all instances, 1 = reassignment candidates (usage > 0 or the
 * current instance, unless include_idle).  Returns the 1-based id (0 none)
 * and its usage in *bu.  Fast path: one warp reduction of a 32-bit
 * (usage << 6 | id) key when every instance has a lane and usages fit. */
template <class W>
EC_DEV int snap_argmin(const W* w, int k, int cand_mode, int cur, long long* bu_out) {
  const int M = ec_nm(w);
  const bool all = cand_mode == 0 || w->sc.include_idle;
  if (M <= EC_TSIZE) {
    const int i = EC_LANE + 1;
    const long long u = i <= M ? w->snap[k][i - 1] : 0;
    const bool cand = i <= M && (all || u > 0 || i == cur);
    if (!t_ballot(cand && (u < 0 || u >= (1ll << 26)))) {
      const unsigned key = cand ? ((unsigned)u << 6) | (unsigned)(i - 1) : 0xffffffffu;
      const unsigned mn = t_redux_min_u32(key);
      if (mn == 0xffffffffu) return 0;
      *bu_out = (long long)(mn >> 6);
      return (int)(mn & 63u) + 1;
    }
  } else {
    const int r = snap_argmin_wide(w, k, all, cur, bu_out);
    if (r >= 0) return r;
  }
  long long bu = 0;
  int bi = 0;
  EC_ILOOP /* per-instance loop: rolled (instruction cache) */
  for (int i = EC_LANE + 1; i <= M; i += EC_TSIZE) {
    const long long u = w->snap[k][i - 1];
    if (!all && !(u > 0 || i == cur)) continue;
    if (!bi || u < bu) {
      bu = u;
      bi = i;
    }
  }
  EC_ILOOP
  for (int o = EC_TSIZE / 2; o > 0; o >>= 1) {
    const long long ou = t_shfl_xor_ll(bu, o);
    const int oi = t_shfl_xor_i(bi, o);
    if (oi && (!bi || ou < bu || (ou == bu && oi < bi))) {
      bu = ou;
      bi = oi;
    }
  }
  *bu_out = bu;
  return bi;
}

/* JOB_DEPS (team, M > 32): the dependent records' usage snapshots, one
 * binary search per (record, instance) pair across all threads; then one
 * warp per record: the reassignment check (dep_target[k] = -1 when it
 * migrates, maybe_reassign router.py:110-128) or the arrival's routing
 * (router.py:75-94,131-151; round-robin is left to the in-order commit) */
template <class W>
EC_COLD1 void job_deps(W* w, const GP& g, int tid, int nthr) {
  (void)g;
  const AsbScenario& sc = w->sc;
  const int M = ec_nm(w), n_dep = w->n_dep, stop_p = w->j_stop;
  for (int x = tid; x < n_dep * M; x += nthr) {
    const int k = x / M, i = x - k * M + 1;
    const int dp = w->dep_pos[k];
    if (dp >= stop_p) continue;
    int lo = w->ioff[i - 1], hi = w->ioff[i]; /* first entry with position >= dp */
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (w->ilist[mid] < dp)
        lo = mid + 1;
      else
        hi = mid;
    }
    w->snap[k][i - 1] = lo > w->ioff[i - 1] ? w->wu[lo - 1] : w->in[i - 1].usage;
  }
  ec_team_barrier(W::NT);
  const double threshold = sc.consolidation_threshold * (double)sc.capacity;
  for (int k = tid >> 5; k < n_dep; k += nthr >> 5) {
    const int p = w->dep_pos[k];
    if (p >= stop_p) continue;
    const int pr = w->sw_prio[p];
    long long bu = 0;
    if (pr == EV_TOOL) {
      const int cur = w->sw_inst[p];
      const int bi = snap_argmin(w, k, 1, cur, &bu);
      const bool mig = bi && bi != cur && (double)w->snap[k][cur - 1] >= sc.imbalance_ratio * (double)bu;
      if (EC_LANE == 0) w->dep_target[k] = mig ? -1 : 0;
    } else if (pr == EV_ARRIVAL && sc.policy != ASB_POLICY_ROUND_ROBIN) {
      int light = 0;
      if (sc.policy == ASB_POLICY_CONTEXT_AWARE)
        EC_ILOOP /* per-instance loop: rolled (instruction cache) */
        for (int base = 0; base < M && !light; base += 32) {
          const int i = base + EC_LANE + 1;
          const unsigned m = t_ballot(i <= M && (double)w->snap[k][i - 1] < threshold);
          if (m) light = base + ec_ffs(m);
        }
      const int target = light ? light : snap_argmin(w, k, 0, 0, &bu);
      if (EC_LANE == 0) w->dep_target[k] = target;
    }
  }
}

/* M > 32: reassignment checks and arrival routing one lane per record
 * (1) or one warp reduction per record, in order (0) */
#ifndef EC_WIDE_LANE_PAR
#define EC_WIDE_LANE_PAR 1
#endif
/* multi-warp teams with <= 32 instances: snapshots, checks and arrival
 * routing as the same team job (a warp per dependent record) instead of one
 * warp reduction per record in order on the main warp */
#ifndef EC_TEAM_DEPS_SMALL
#define EC_TEAM_DEPS_SMALL 1
#endif

/* Parallel commit walk (team).  The serial walk's state machine decomposes
 * by instance: usage, running count, thrash flag, power and the running log
 * of instance i change only at records on i.  Each lane owns instances and
 * replays their records in walk order (finding the first thrash flip / log
 * overflow), usage snapshots are taken at the records that read all
 * instances (arrivals, reassignment checks), and push sequence numbers /
 * start ranks are warp prefix scans.  Returns false (caller falls back to
 * walk_serial) under interference or when a tie group contains a record
 * whose push order is only known during the walk. */
template <class W, int RCAP>
EC_COLD3 bool walk_parallel(W* w, const GP& g, const int n) {
  const AsbScenario& sc = w->sc;
  if (sc.interference > 0) return false;
  const int M = ec_nm(w);
  EC_WPROF_START(w);
  /* ---- step 0: the rank sort already ordered exact ties by push seq; an
   * unknown seq inside a tie needs the serial walk */
  if (w->j_tie_unknown) return false;
  int cut = w->j_cut < n ? w->j_cut : n;
  int ndep = 0;
  for (int base = 0; base < n; base += EC_TSIZE) {
    const int p = base + EC_LANE;
    const bool dep = p < n && w->depflag[p];
    unsigned m = t_ballot(dep);
    int k = ndep + ec_popc(m & t_lt_mask());
    if (dep) {
      if (k < W::DEP)
        w->dep_pos[k] = p;
      else if (k == W::DEP && p < cut)
        cut = p; /* snapshot table full: stop before it */
    }
    ndep += ec_popc(m);
  }
  cut = (int)t_redux_min_u32((unsigned)cut); /* cut >= 0 */
  EC_LANE0 w->n_dep = ndep < W::DEP ? ndep : W::DEP;
  t_sync();
  EC_WPROF(w, 0);
  /* ---- step 1: per-instance prefix scans over the instances' record
   * lists (ilist, grouped by instance, in walk order): usage, running count
   * and running-log length after each record, the first thrash flip /
   * log overflow, and the power-change points.  Segmented inclusive scans
   * (segments = instances) across the team; values by record, in shared
   * memory, for the snapshot and write-back lookups below. */
  const long long cap = sc.capacity;
  const int n_list = w->ioff[M];
  int first = cut, first_lf = cut;
  for (int base = 0; base < n_list; base += EC_TSIZE) {
    const int e = base + EC_LANE;
    const bool valid = e < n_list;
    const int p = valid ? w->ilist[e] : 0x7fffffff;
    const int i = valid ? (int)w->sw_inst[p] : 1; /* instance of entry e */
    const int s0 = w->ioff[i - 1];     /* first entry of its segment */
    const bool live = valid && p < cut;
    const int pr = live ? w->sw_prio[p] : 0;
    const bool comp = pr == EV_COMPLETE, start = pr == EV_TOOL || pr == EV_ISSUE;
    long long vu = comp ? w->sw_du[p] : 0;
    int vr = comp ? -1 : (start ? 1 : 0), vl = start ? 1 : 0;
    EC_ILOOP
    for (int o = 1; o < EC_TSIZE; o <<= 1) {
      const long long nu = t_shfl_up_ll(vu, o);
      const int nr = t_shfl_up_i(vr, o), nl = t_shfl_up_i(vl, o);
      if (EC_LANE >= o && e - o >= s0) {
        vu += nu;
        vr += nr;
        vl += nl;
      }
    }
    if (base > 0 && s0 < base) { /* segment continues from the previous chunk */
      vu += w->carry_u;
      vr += w->carry_r;
      vl += w->carry_l;
    }
    const Inst& in = w->in[i - 1];
    const long long U = in.usage + vu;
    const int R = in.running + vr, Lg = in.log_len + vl;
    const int Rprev = R - (comp ? -1 : (start ? 1 : 0));
    const bool chg = valid && ((R > 0) != (Rprev > 0) || e == s0); /* a segment's first entry always checks */
    if (valid) {
      w->wu[e] = U;
      w->wr[e] = R;
      w->wl[e] = Lg;
    }
    {
      const unsigned cm = t_ballot(chg);
      if (EC_TSIZE == 32) {
        if (EC_LANE == 0) w->wmask[base >> 5] = cm;
      } else if (EC_LANE == 0) { /* 1-lane host build: one bit per entry */
        unsigned& m = w->wmask[e >> 5];
        if ((e & 31) == 0) m = 0;
        if (chg) m |= 1u << (e & 31);
      }
    }
    if (live && comp && (U > cap ? 1 : 0) != in.thr && p < first) first = p;
    if (live && start && Lg - 1 >= g.A && p < first_lf) first_lf = p;
    t_sync();
    if (EC_LANE == EC_TSIZE - 1) {
      w->carry_u = vu;
      w->carry_r = vr;
      w->carry_l = vl;
    }
    t_sync();
  }
  first = (int)t_redux_min_u32((unsigned)first);
  first_lf = (int)t_redux_min_u32((unsigned)first_lf);
  EC_WPROF(w, 1);
  /* ---- step 2: reassignment checks in order (team argmin on the snapshot) */
  int stop_p = first < first_lf ? first : first_lf;
  int stop_kind = stop_p == cut ? STOP_NONE : (first <= first_lf ? STOP_COUPLING : STOP_LOGFULL);
  const int n_dep = w->n_dep;
  /* usage snapshots: instance i's usage just before dependent record k =
   * its usage after its last record ahead of dep_pos[k].  Few instances:
   * one binary search per (record, instance) pair across the lanes; many
   * instances (M > 32): lane per instance, merging its sorted record list
   * with the sorted dependent positions */
  /* a single instance (compile-time): every arrival routes to it and no
   * reassignment can migrate (the argmin is the current instance,
   * router.py:110-128), so no snapshots or checks are needed */
  constexpr bool single = W::MX == 1;
  const bool team_deps = !single && W::NW > 1 && n_dep > 0 && (M > EC_TSIZE ? W::MX > 32 : EC_TEAM_DEPS_SMALL);
  if (single) {
  } else if (team_deps) {
    /* many instances, helper warps: snapshots, checks and routing as a team job */
    EC_LANE0 w->j_stop = stop_p;
    t_sync();
    fork_job(w, JOB_DEPS);
    int mig = stop_p;
    for (int k = EC_LANE; k < n_dep; k += EC_TSIZE) {
      const int p = w->dep_pos[k];
      if (p < stop_p && w->sw_prio[p] == EV_TOOL && w->dep_target[k] < 0 && p < mig) mig = p;
    }
    mig = (int)t_redux_min_u32((unsigned)mig);
    if (mig < stop_p) {
      stop_p = mig;
      stop_kind = STOP_COUPLING;
    }
  } else if (M <= EC_TSIZE) {
    for (int x = EC_LANE; x < n_dep * M; x += EC_TSIZE) {
      const int k = x / M, i = x - k * M + 1;
      const int dp = w->dep_pos[k];
      if (dp >= stop_p) continue;
      int lo = w->ioff[i - 1], hi = w->ioff[i]; /* first entry with position >= dp */
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (w->ilist[mid] < dp)
          lo = mid + 1;
        else
          hi = mid;
      }
      w->snap[k][i - 1] = lo > w->ioff[i - 1] ? w->wu[lo - 1] : w->in[i - 1].usage;
    }
  } else {
    snapshots_merge(w, n_dep, stop_p);
  }
  t_sync();
  if (single || team_deps) {
    /* nothing to check / done by JOB_DEPS */
  } else if (EC_WIDE_LANE_PAR && M > EC_TSIZE) {
    /* many instances: one lane per check */
    if (n_dep > 0) {
      const int mig = checks_parallel(w, n_dep, stop_p);
      if (mig < stop_p) {
        stop_p = mig;
        stop_kind = STOP_COUPLING;
      }
    }
  } else {
    /* few instances: one warp reduction per check, in order */
    for (int k = 0; k < n_dep; k++) {
      const int p = w->dep_pos[k];
      if (p >= stop_p) break;
      if (w->sw_prio[p] != EV_TOOL) continue;
      const int cur = w->sw_inst[p];
      long long bu = 0;
      const int bi = snap_argmin(w, k, 1, cur, &bu);
      if (bi && bi != cur && (double)w->snap[k][cur - 1] >= sc.imbalance_ratio * (double)bu) {
        stop_p = p;
        stop_kind = STOP_COUPLING;
        break;
      }
    }
  }
  EC_WPROF(w, 2);
  /* ---- step 3: write back the committed prefix: running-log entries of
   * the starts (parallel), then per instance the state after its last
   * record ahead of stop_p and the power integration over its change
   * points in order (lane per instance; engine.py:321-327) */
  for (int e = EC_LANE; e < n_list; e += EC_TSIZE) {
    const int p = w->ilist[e];
    if (p >= stop_p) continue;
    const int pr = w->sw_prio[p];
    if (pr != EV_TOOL && pr != EV_ISSUE) continue;
    const int i = w->sw_inst[p];
    Rec& r = w->rec[w->sw_idx[p]];
    r.logpos = w->wl[e] - 1;
    g.log[(long long)(i - 1) * g.A + r.logpos] = r.agent;
  }
  EC_ILOOP /* per-instance loop: rolled (instruction cache) */
  for (int i = EC_LANE + 1; i <= M; i += EC_TSIZE) {
    Inst& in = w->in[i - 1];
    const int e0 = w->ioff[i - 1];
    int lo = e0, hi = w->ioff[i]; /* entries [e0, lo) lie before stop_p */
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (w->ilist[mid] < stop_p)
        lo = mid + 1;
      else
        hi = mid;
    }
    const int last = lo - 1;
    const double act = w->act[in.level - 1], idle = w->idle[in.level - 1];
    double watts = in.watts, t_pow = in.t_pow, energy = in.energy;
    /* power changes only where the running count crosses zero: visit those
     * entries (bitmask), in order */
    for (int e = e0; e <= last;) {
      const unsigned m = w->wmask[e >> 5] >> (e & 31);
      if (!m) {
        e = (e | 31) + 1;
        continue;
      }
      e += ec_ffs(m) - 1;
      if (e > last) break;
      const double wt = w->wr[e] > 0 ? act : idle;
      if (wt != watts) {
        const double t = w->sw_t[w->ilist[e]];
        energy += watts * (t - t_pow);
        t_pow = t;
        watts = wt;
      }
      e++;
    }
    if (last >= e0) {
      in.usage = w->wu[last];
      in.running = w->wr[last];
      in.log_len = w->wl[last];
      in.watts = watts;
      in.t_pow = t_pow;
      in.energy = energy;
    }
  }
  t_sync();
  EC_WPROF(w, 3);
  /* ---- step 4: push sequence numbers, start ranks, counters (prefix scans) */
  const long long seq0 = w->seq, rank0 = w->start_ctr;
  int pushes = 0, starts = 0, turns = 0, completed = 0;
  for (int base = 0; base < stop_p; base += EC_TSIZE) {
    const int p = base + EC_LANE;
    bool push = false, start = false, comp = false, last = false;
    if (p < stop_p) {
      const int pr = w->sw_prio[p];
      start = pr == EV_TOOL || pr == EV_ISSUE;
      comp = pr == EV_COMPLETE;
      last = comp && (w->sw_flags[p] & F_LAST);
      push = start || (comp && !last);
    }
    unsigned mp = t_ballot(push), ms = t_ballot(start);
    turns += ec_popc(t_ballot(comp));
    completed += ec_popc(t_ballot(last));
    if (p < stop_p) {
      Rec& r = w->rec[w->sw_idx[p]];
      if (push) {
        r.push_seq = seq0 + pushes + ec_popc(mp & t_lt_mask());
        if (r.child >= 0) w->rec[r.child].seq = r.push_seq;
      }
      if (start) r.aux64 = rank0 + starts + ec_popc(ms & t_lt_mask());
      r.flags |= F_COMMITTED;
    }
    pushes += ec_popc(mp);
    starts += ec_popc(ms);
  }
  t_sync();
  EC_WPROF(w, 4);
  /* ---- step 5: arrivals in order (routing on the usage snapshot) */
  if (team_deps || single) {
    /* many instances, routed by JOB_DEPS: commit the arrivals a lane each
     * (_on_arrival bookkeeping, engine.py:490-507, as commit_arrival does
     * it one by one): arrival rank, alive slot and arrival_rank from the
     * lane's rank among the batch's arrivals, FIFO position from the earlier
     * arrivals to the same instance */
    int done = 0;
    for (int base = 0; base < n_dep; base += EC_TSIZE) {
      const int k = base + EC_LANE;
      const int p = k < n_dep ? w->dep_pos[k] : 0x7fffffff;
      const bool arr = p < stop_p && w->sw_prio[p] == EV_ARRIVAL;
      const unsigned m = t_ballot(arr);
      if (!m) continue;
      const int rank = done + ec_popc(m & t_lt_mask());
      int target = 0, a = -1, order_pos = 0;
      if (arr) {
        const Rec& r = w->rec[w->sw_idx[p]];
        a = r.agent;
        order_pos = (int)r.seq;
        target = single ? 1
                 : sc.policy == ASB_POLICY_ROUND_ROBIN ? (int)(((long long)w->rr_next + rank) % M) + 1
                                                       : w->dep_target[k];
      }
      const unsigned peers = t_match_any_i(arr ? target : 0) & m;
      const int same_before = ec_popc(peers & t_lt_mask());
      if (arr) {
        const Inst& dst = w->in[target - 1];
        g.ring[(long long)(target - 1) * g.A + ring_idx(dst.fifo_head, dst.fifo_len + same_before, g.A)] = a;
        g.H[a].inst = target;
        g.H[a].sa = 0;
        g.H[a].phase = ASB_PHASE_PENDING;
        g.H[a].next_prio = 0;
        const int j = w->n_alive + rank;
        g.H[a].slot = j;
        init_slot(g, j, target, a);
        g.rank[a] = w->arr_rank + rank;
      }
      t_sync(); /* every lane has read fifo_len before the groups advance it */
      if (arr && (peers >> EC_LANE) == 1u) w->in[target - 1].fifo_len += ec_popc(peers); /* last lane of its group */
      if (arr && (m >> EC_LANE) == 1u) w->arr_ptr = order_pos + 1; /* the chunk's last arrival */
      done += ec_popc(m);
      t_sync();
    }
    EC_LANE0 {
      w->n_alive += done;
      w->arr_rank += done;
      if (sc.policy == ASB_POLICY_ROUND_ROBIN) w->rr_next += done;
      w->ctr[ASB_CTR_ARRIVED] += done;
    }
    t_sync();
  } else if (EC_WIDE_LANE_PAR && n_dep > 0 && M > EC_TSIZE) {
    /* many instances: route every arrival in parallel (a lane per arrival),
     * commit in order */
    route_parallel(w, n_dep, stop_p);
    EC_LANE0 {
      for (int k = 0; k < n_dep; k++) {
        const int p = w->dep_pos[k];
        if (p >= stop_p) break;
        if (w->sw_prio[p] != EV_ARRIVAL) continue;
        const Rec& r = w->rec[w->sw_idx[p]];
        int target = w->dep_target[k];
        if (sc.policy == ASB_POLICY_ROUND_ROBIN) {
          target = (w->rr_next % M) + 1;
          w->rr_next++;
        }
        commit_arrival(w, g, r.agent, target, (int)r.seq);
      }
    }
    t_sync();
  } else {
    for (int k = 0; k < n_dep; k++) {
      const int p = w->dep_pos[k];
      if (p >= stop_p) break;
      if (w->sw_prio[p] != EV_ARRIVAL) continue;
      int target;
      if (sc.policy == ASB_POLICY_ROUND_ROBIN) {
        target = (w->rr_next % M) + 1;
      } else {
        /* context_aware: lowest id below theta * cap, else argmin (router.py:85-90) */
        int light = 0;
        if (sc.policy == ASB_POLICY_CONTEXT_AWARE) {
          const double threshold = sc.consolidation_threshold * (double)sc.capacity;
          EC_ILOOP /* per-instance loop: rolled (instruction cache) */
          for (int base = 0; base < M && !light; base += EC_TSIZE) {
            const int i = base + EC_LANE + 1;
            const unsigned m = t_ballot(i <= M && (double)w->snap[k][i - 1] < threshold);
            if (m) light = base + ec_ffs(m);
          }
        }
        long long bu = 0;
        target = light ? light : snap_argmin(w, k, 0, 0, &bu);
      }
      EC_LANE0 {
        const Rec& r = w->rec[w->sw_idx[p]];
        if (sc.policy == ASB_POLICY_ROUND_ROBIN) w->rr_next++;
        commit_arrival(w, g, r.agent, target, (int)r.seq);
      }
      t_sync();
    }
  }
  EC_LANE0 {
    w->seq += pushes;
    w->start_ctr += starts;
    w->ctr[ASB_CTR_TURNS] += turns;
    w->ctr[ASB_CTR_COMPLETED] += completed;
    w->ctr[ASB_CTR_EVENTS] += turns + starts;
    int stop = stop_kind;
    if (stop == STOP_NONE && (cut < n || w->hz_t != EC_INF_BITS)) stop = STOP_HORIZON;
    const int stop_idx = (stop == STOP_COUPLING || stop == STOP_LOGFULL) ? w->sw_idx[stop_p] : -1;
    w->stop_kind = stop;
    w->stop_rec = stop_idx;
    if (stop_idx >= 0) w->stop_r = w->rec[stop_idx];
  }
  t_sync();
  EC_WPROF(w, 5);
  return true;
}

/* JOB_SPEC (thread-level): each thread runs its due agents' own event
 * chains inside the window; continuation records are allocated atomically;
 * the smallest dropped key becomes the batch horizon. */
template <class W>
EC_COLD1 void job_spec(W* w, const GP& gp, int tid, int nthr) {
  const GV g = gview(gp);
  const double bound = w->j_bound;
  const int incl = w->j_incl;
  const int nd = w->n_due;
  const int nr0 = w->n_rec;
  unsigned long long my_t = EC_INF_BITS;
  unsigned my_p = 0;
  int order_err = 0;
  EC_PPROF_T0();
  for (int d = tid; d < nd; d += nthr) {
    Cur c;
    long long seq0;
    cur_load(g, c, w->due[d], &seq0);
    if (W::CC && d < W::CCN) w->ccache[d] = c;
    EC_PPROF(w, 1); /* the record and turn loads */
    Rec* r = &w->rec[d];
    r->seq = seq0;
    if (!(c.prio > 0 && (incl ? c.t <= bound : c.t < bound))) {
      /* a candidate whose event moved out of the window (re-timed) */
      r->flags = F_EMPTY;
      r->child = -1;
      r->prio = 0;
      r->agent = c.a;
      t_atomic_add_i(&w->n_empty, 1);
      continue;
    }
    if (!cur_step(w, g, c, *r, false)) order_err = 1;
    EC_PPROF(w, 2); /* the first event */
    while (c.prio > 0 && (incl ? c.t <= bound : c.t < bound)) {
      const int slot = t_atomic_add_i(&w->tmp_i, 1) + nr0;
      if (slot >= W::RC) {
        /* dropped continuation: its seq is unknown, so nothing at its
         * (time, prio) may commit in this batch */
        const unsigned long long tb = ec_bits(c.t);
        if (key_less(tb, (unsigned)c.prio, my_t, my_p)) {
          my_t = tb;
          my_p = (unsigned)c.prio;
        }
        break;
      }
      r->child = slot;
      r = &w->rec[slot];
      r->seq = -1;
      if (!cur_step(w, g, c, *r, false)) order_err = 1;
    }
  }
  EC_PPROF(w, 3); /* the chain's continuations */
  if (order_err) w->j_order_err = 1;
  /* the warp's smallest dropped key; almost always none (no drops) */
  if (t_ballot(my_t != EC_INF_BITS)) t_warp_min_key(my_t, my_p);
  if ((tid & 31) == 0) {
    w->j_hz_t[tid >> 5] = my_t;
    w->j_hz_p[tid >> 5] = my_p;
  }
  EC_PPROF(w, 4); /* the warp's horizon key */
}

/* JOB_SORT (thread-level): rank sort of the records by (time, prio, seq) —
 * seq only breaks exact (time, prio) ties, and an unknown seq in a tie sends
 * the walk to the serial fallback — writing the sorted SoA view, the
 * dependent-record flags and the horizon cut. */
/* the sorted-record outputs shared by both sort implementations: the
 * sorted SoA view at rank `rank` of record j */
template <class W>
EC_DEV void sort_emit(W* w, int j, int rank, unsigned long long tj, unsigned pj) {
  const Rec& r = w->rec[j];
  SortE& e = w->srt[rank];
  e.tb = tj;
  e.prio = pj;
  e.idx = (unsigned)j;
  w->sw_t[rank] = r.t;
  w->sw_idx[rank] = j;
  w->sw_prio[rank] = (unsigned char)pj;
  w->sw_flags[rank] = (unsigned char)r.flags;
  w->sw_inst[rank] = (short)(pj == EV_ARRIVAL ? 0 : r.inst);
  w->sw_du[rank] = pj == EV_COMPLETE ? (long long)r.delta - ((r.flags & F_LAST) ? r.aux64 : 0) : 0;
  w->depflag[rank] = pj == EV_ARRIVAL || (pj == EV_TOOL && (r.flags & F_CHECK));
}

#if EC_TSIZE == 32
/* 128-bit sort key of record j: (time bits, prio, seq, index); empty
 * records sort last.  seq -1 (unknown) sorts first inside its (t, prio)
 * tie; such ties are flagged and resolved by the serial walk. */
struct SKey {
  unsigned long long k1, k2;
};
template <class W>
EC_DEV SKey skey_of(const W* w, int j, int n_all) {
  SKey k;
  if (j >= n_all) {
    k.k1 = ~0ull;
    k.k2 = ~0ull;
    return k;
  }
  const Rec& r = w->rec[j];
  if (r.flags & F_EMPTY) {
    k.k1 = ~0ull;
    k.k2 = 0xff00000000000000ull | (unsigned long long)j;
    return k;
  }
  /* record index in the low 11 bits (RCAP <= 2048), push seq + 1 above it
   * (< 2^45), the priority on top */
  static_assert(W::RC <= 2048, "sort key holds an 11-bit record index");
  k.k1 = ec_bits(r.t);
  k.k2 = ((unsigned long long)(unsigned)r.prio << 56) | ((unsigned long long)(r.seq + 1) << 11) |
         (unsigned long long)j;
  return k;
}

/* JOB_SORT, GPU team: counting rank.  The 16-byte keys of all records are
 * staged in shared memory; each thread ranks its records by one broadcast
 * 128-bit load + a branch-free compare per record (independent iterations,
 * so a lone warp keeps several loads in flight).  Keys are unique (the
 * record index is the last component), so ranks are a permutation. */
template <class W>
EC_COLD1 void job_sort(W* w, const GP& g, int tid, int nthr) {
  (void)g;
  const int n_all = w->n_rec;
  const int M = ec_nm(w);
  const int lane = tid & 31, wid = tid >> 5;
  EC_QPROF_T0();
  ulonglong2* key = reinterpret_cast<ulonglong2*>(w->skey);
  auto emit = [&](int j, int rank, unsigned long long tj) {
    const Rec& rr = w->rec[j];
    const bool empty = rr.flags & F_EMPTY;
    const unsigned pj = empty ? 0xffu : (unsigned)rr.prio;
    sort_emit(w, j, rank, empty ? ~0ull : tj, pj);
    w->ki[rank] = (short)(empty || pj == EV_ARRIVAL ? 0 : rr.inst); /* by rank */
    if (!W::BIGSORT && !empty && !below_horizon(tj, pj, rr.seq, w->hz_t, (unsigned)w->hz_p, w->hz_s))
      t_atomic_min_i(&w->j_cut, rank);
  };
  if (W::NT == 512 && n_all > EC_BITONIC_MIN) {
    /* the 16-warp team's batches of more than 256 records: a bitonic sort
     * of the keys (the record index sits in the low 11 bits of the second
     * half), O(n log^2 n) steps instead of the counting rank's O(n^2)
     * compares (C4: 527 -> 511 ms) */
    static_assert(W::NT < 512 || W::SK >= 1024, "the bitonic buffers hold N = 1024 keys");
    int N = 1024;
    while (N / 2 >= n_all) N >>= 1;
    /* the network runs in registers: thread tid holds elements tid and
     * tid + NT (N = 1024); exchanges between elements of one warp (j <= 16)
     * are shuffles, between warps a shared-memory round (ping-pong between
     * the key buffer and the not-yet-written sorted view: one barrier per
     * cross-warp step, 10-14 instead of one per step, 45-55) */
    constexpr int NT = 512; /* the branch is taken by the 512-thread team only */
    ulonglong2 v[2];
    for (int e = 0; e < 2; e++) {
      const int i = tid + e * NT;
      if (i < N) {
        const SKey k = skey_of(w, i, n_all); /* i >= n_all: (~0, ~0), sorts last */
        v[e] = make_ulonglong2(k.k1, k.k2);
      }
    }
    EC_QPROF(w, 0);
    ulonglong2* bufs[2] = {key, reinterpret_cast<ulonglong2*>(w->srt)};
    static_assert(sizeof(SortE) == sizeof(ulonglong2), "the sorted view doubles as a key buffer");
    int flip = 0;
    auto keep = [](ulonglong2& me, const ulonglong2& o, bool take_min) {
      const bool o_less = o.x < me.x || (o.x == me.x && o.y < me.y);
      if (take_min == o_less) me = o;
    };
    for (int k = 2; k <= N; k <<= 1) {
      for (int jj = k >> 1; jj > 0; jj >>= 1) {
        if (jj >= NT) { /* k = N = 1024, j = 512: the thread's own two elements */
          const ulonglong2 a0 = v[0], a1 = v[1];
          keep(v[0], a1, true); /* element tid < tid + 512, ascending (k = N) */
          keep(v[1], a0, false);
        } else if (jj >= 32) {
          ulonglong2* buf = bufs[flip];
          flip ^= 1;
          for (int e = 0; e < 2; e++) {
            const int i = tid + e * NT;
            if (i < N) buf[i] = v[e];
          }
          ec_team_barrier(NT);
          for (int e = 0; e < 2; e++) {
            const int i = tid + e * NT;
            if (i < N) {
              const int pj = i ^ jj;
              keep(v[e], buf[pj], (i < pj) == ((i & k) == 0));
            }
          }
        } else {
          for (int e = 0; e < 2; e++) {
            const int i = tid + e * NT;
            if (e * NT < N) { /* warp-uniform */
              ulonglong2 o;
              o.x = __shfl_xor_sync(0xffffffffu, v[e].x, jj);
              o.y = __shfl_xor_sync(0xffffffffu, v[e].y, jj);
              keep(v[e], o, (i < (i ^ jj)) == ((i & k) == 0));
            }
          }
        }
      }
    }
    ec_team_barrier(NT); /* every cross-warp read is done before the final store */
    for (int e = 0; e < 2; e++) {
      const int i = tid + e * NT;
      if (i < N) key[i] = v[e];
    }
    ec_team_barrier(NT);
    EC_QPROF(w, 1);
    for (int p = tid; p < n_all; p += nthr) {
      const ulonglong2 kp = key[p];
      emit((int)(kp.y & 0x7ffull), p, kp.x);
    }
    EC_QPROF(w, 2);
  } else {
  for (int j = tid; j < n_all; j += nthr) {
    const SKey k = skey_of(w, j, n_all);
    key[j] = make_ulonglong2(k.k1, k.k2);
  }
  ec_team_barrier(W::NT);
  EC_QPROF(w, 0);
  for (int j = tid; j < n_all; j += nthr) {
    const ulonglong2 me = key[j];
    int rank = 0;
    int q = 0;
#pragma unroll 1
    for (; q + 4 <= n_all; q += 4) {
      const ulonglong2 o0 = key[q], o1 = key[q + 1], o2 = key[q + 2], o3 = key[q + 3];
      rank += (o0.x < me.x) | ((o0.x == me.x) & (o0.y < me.y));
      rank += (o1.x < me.x) | ((o1.x == me.x) & (o1.y < me.y));
      rank += (o2.x < me.x) | ((o2.x == me.x) & (o2.y < me.y));
      rank += (o3.x < me.x) | ((o3.x == me.x) & (o3.y < me.y));
    }
    for (; q < n_all; q++) {
      const ulonglong2 o = key[q];
      rank += (o.x < me.x) | ((o.x == me.x) & (o.y < me.y));
    }
    emit(j, rank, me.x);
  }
  EC_QPROF(w, 2);
  }
  ec_team_barrier(W::NT);
  EC_QPROF(w, 3);
  /* exact (time, prio) ties with an unknown push seq need the serial walk;
   * the horizon cut: records at or beyond the horizon key form a suffix of
   * the non-empty sorted records (the key orders like (time, prio, seq)),
   * whose first position is the cut (one writer, no atomics) */
  int tie_unknown = 0;
  if (!W::BIGSORT) {
    for (int p = tid + 1; p < n_all; p += nthr) {
      if (w->sw_prio[p] == 0xff) continue;
      if (w->srt[p].tb == w->srt[p - 1].tb && w->sw_prio[p] == w->sw_prio[p - 1] &&
          (w->rec[w->sw_idx[p]].seq < 0 || w->rec[w->sw_idx[p - 1]].seq < 0))
        tie_unknown = 1;
    }
    if (tie_unknown) w->j_tie_unknown = 1;
    EC_QPROF(w, 4);
    /* per-instance lists of sorted positions, in rank order (warp 0) */
    if (wid == 0) {
      EC_ILOOP /* per-instance loop: rolled (instruction cache) */
      for (int i = lane; i < M; i += 32) w->icnt[i] = 0;
      __syncwarp();
      for (int base = 0; base < n_all; base += 32) {
        const int p = base + lane;
        const int ij = p < n_all ? w->ki[p] : 0;
        const unsigned peers = __match_any_sync(0xffffffffu, ij);
        const int before = __popc(peers & t_lt_mask());
        if (ij) w->krank[p] = (short)(w->icnt[ij - 1] + before); /* position in instance ij's list */
        __syncwarp();
        if (ij && before == 0) w->icnt[ij - 1] += __popc(peers);
        __syncwarp();
      }
      int run = 0;
      EC_ILOOP /* per-instance loop: rolled (instruction cache) */
      for (int base = 0; base < M; base += 32) {
        const int i = base + lane;
        const int c = i < M ? w->icnt[i] : 0; /* record counts: 32-bit scans */
        const int inc = t_scan_add_i(c);
        if (i < M) w->ioff[i] = run + inc - c;
        run += t_shfl_i(inc, 31);
      }
      if (lane == 0) w->ioff[M] = (int)run;
      __syncwarp();
      for (int p = lane; p < n_all; p += 32) {
        const int ij = w->ki[p];
        if (ij) w->ilist[w->ioff[ij - 1] + w->krank[p]] = (short)p;
      }
    }
    EC_QPROF(w, 5);
    return;
  }
  const unsigned long long hzt = w->hz_t;
  const unsigned hzp = (unsigned)w->hz_p;
  const long long hzs = w->hz_s;
  for (int p = tid; p < n_all; p += nthr) {
    const unsigned pp = w->sw_prio[p];
    if (pp == 0xff) continue;
    const unsigned long long tb = w->srt[p].tb;
    const long long sq = w->rec[w->sw_idx[p]].seq;
    if (p > 0) {
      const unsigned long long tb1 = w->srt[p - 1].tb;
      const unsigned pp1 = w->sw_prio[p - 1];
      const long long sq1 = w->rec[w->sw_idx[p - 1]].seq;
      if (tb == tb1 && pp == pp1 && (sq < 0 || sq1 < 0)) tie_unknown = 1;
      if (!below_horizon(tb, pp, sq, hzt, hzp, hzs) && below_horizon(tb1, pp1, sq1, hzt, hzp, hzs)) w->j_cut = p;
    } else if (!below_horizon(tb, pp, sq, hzt, hzp, hzs)) {
      w->j_cut = 0;
    }
  }
  if (tie_unknown) w->j_tie_unknown = 1;
  EC_QPROF(w, 4);
  /* per-instance lists of sorted positions, in rank order, by the whole
   * team: each warp counts its 32-record chunks per instance (match_any),
   * warp 0 turns the chunk counts into offsets, then every record is placed */
  const int nch = (n_all + 31) >> 5;
  for (int c = wid; c < nch; c += W::NW) {
    EC_ILOOP /* per-instance loop: rolled (instruction cache) */
    for (int i = lane; i < M; i += 32) w->kcc[c][i] = 0;
    __syncwarp();
    const int p = (c << 5) + lane;
    const int ij = p < n_all ? w->ki[p] : 0;
    const unsigned peers = __match_any_sync(0xffffffffu, ij);
    const int before = __popc(peers & t_lt_mask());
    if (ij) w->krank[p] = (short)before; /* position among the chunk's records on ij */
    if (ij && before == 0) w->kcc[c][ij - 1] = (unsigned short)__popc(peers);
  }
  ec_team_barrier(W::NT);
  if (wid == 0) {
    int run = 0;
    EC_ILOOP /* per-instance loop: rolled (instruction cache) */
    for (int base = 0; base < M; base += 32) {
      const int i = base + lane;
      int cnt = 0;
      if (i < M)
        for (int c = 0; c < nch; c++) {
          const int t = w->kcc[c][i];
          w->kcc[c][i] = (unsigned short)cnt;
          cnt += t;
        }
      const int inc = t_scan_add_i(cnt);
      if (i < M) w->ioff[i] = run + inc - cnt;
      run += t_shfl_i(inc, 31);
    }
    if (lane == 0) w->ioff[M] = (int)run;
  }
  ec_team_barrier(W::NT);
  for (int p = tid; p < n_all; p += nthr) {
    const int ij = w->ki[p];
    if (ij) w->ilist[w->ioff[ij - 1] + w->kcc[p >> 5][ij - 1] + w->krank[p]] = (short)p;
  }
  EC_QPROF(w, 5);
}
#else
/* JOB_SORT, generic team (the 1-lane host harness): O(n^2) rank sort */
template <class W>
EC_COLD1 void job_sort(W* w, const GP& g, int tid, int nthr) {
  const int n_all = w->n_rec;
  const int M = ec_nm(w);
  EC_ILOOP /* per-instance loop: rolled (instruction cache) */
  for (int i = tid; i < M; i += nthr) w->icnt[i] = 0;
  for (int j = tid; j < n_all; j += nthr) {
    const Rec& r = w->rec[j];
    const bool empty = r.flags & F_EMPTY;
    w->kt[j] = empty ? ~0ull : ec_bits(r.t);
    w->kp[j] = empty ? 0xff : (unsigned char)r.prio;
    w->ks[j] = r.seq;
    w->ki[j] = (short)(empty || r.prio == EV_ARRIVAL ? 0 : r.inst);
  }
  ec_team_barrier(W::NT);
  int tie_unknown = 0;
  for (int j = tid; j < n_all; j += nthr) {
    if (w->kp[j] == 0xff) continue;
    const unsigned long long tj = w->kt[j];
    const unsigned pj = w->kp[j];
    const long long sj = w->ks[j];
    const int ij = w->ki[j];
    int rank = 0, irank = 0;
    for (int q = 0; q < n_all; q++) {
      const unsigned long long tq = w->kt[q];
      const unsigned pq = w->kp[q];
      bool less = false;
      if (tq < tj || (tq == tj && pq < pj)) {
        less = true;
      } else if (tq == tj && pq == pj && q != j) {
        const long long sq = w->ks[q];
        if (sq < 0 || sj < 0) tie_unknown = 1;
        less = sq < sj || (sq == sj && q < j);
      }
      if (less) {
        rank++;
        if (w->ki[q] == ij) irank++;
      }
    }
    w->krank[j] = (short)rank;
    w->kir[j] = (short)irank;
    if (ij) t_atomic_add_i(&w->icnt[ij - 1], 1);
    const Rec& r = w->rec[j];
    SortE& e = w->srt[rank];
    e.tb = tj;
    e.prio = pj;
    e.idx = (unsigned)j;
    w->sw_t[rank] = r.t;
    w->sw_idx[rank] = j;
    w->sw_prio[rank] = (unsigned char)pj;
    w->sw_flags[rank] = (unsigned char)r.flags;
    w->sw_inst[rank] = (short)(pj == EV_ARRIVAL ? 0 : r.inst);
    w->sw_du[rank] = pj == EV_COMPLETE ? (long long)r.delta - ((r.flags & F_LAST) ? r.aux64 : 0) : 0;
    w->depflag[rank] = pj == EV_ARRIVAL || (pj == EV_TOOL && (r.flags & F_CHECK));
    if (!below_horizon(tj, pj, sj, w->hz_t, (unsigned)w->hz_p, w->hz_s)) t_atomic_min_i(&w->j_cut, rank);
  }
  if (tie_unknown) w->j_tie_unknown = 1;
  ec_team_barrier(W::NT);
  if (tid < EC_TSIZE) { /* warp 0: exclusive scan of the per-instance record counts */
    long long run = 0;
    EC_ILOOP /* per-instance loop: rolled (instruction cache) */
    for (int base = 0; base < M; base += EC_TSIZE) {
      const int i = base + EC_LANE;
      const long long c = i < M ? w->icnt[i] : 0;
      const long long inc = t_scan_add_ll(c);
      if (i < M) w->ioff[i] = (int)(run + inc - c);
      run += t_bcast_ll(inc, EC_TSIZE - 1);
    }
    EC_LANE0 w->ioff[M] = (int)run;
  }
  ec_team_barrier(W::NT);
  for (int j = tid; j < n_all; j += nthr) {
    const int ij = w->ki[j];
    if (ij && w->kp[j] != 0xff) w->ilist[w->ioff[ij - 1] + w->kir[j]] = w->krank[j];
  }
}
#endif

/* JOB_APPLY (thread-level): write back every due agent's committed chain
 * prefix (records carry everything, no trace reads) and its alive slot. */
template <class W>
EC_COLD1 void job_apply(W* w, const GP& gp, int tid, int nthr) {
  const GV g = gview(gp);
  const int nd = w->n_due;
  EC_APROF_T0();
  for (int d = tid; d < nd; d += nthr) {
    if (!(w->rec[d].flags & F_COMMITTED)) continue;
    Cur c; /* unchanged since the speculation loaded it */
    if (W::CC && d < W::CCN)
      c = w->ccache[d];
    else
      cur_load(g, c, w->due[d], nullptr, false);
    EC_APROF(w, 0); /* the cursor */
    int ri = d;
    long long nseq = -1, srank = -1;
    int lpos = -1;
    while (ri >= 0 && (w->rec[ri].flags & F_COMMITTED)) {
      const Rec& r = w->rec[ri];
      cur_apply(w, g, c, r);
      nseq = r.push_seq;
      if (r.prio != EV_COMPLETE) {
        srank = r.aux64;
        lpos = r.logpos;
      }
      ri = r.child;
    }
    EC_APROF(w, 1); /* the committed records */
    const int a = c.a;
    g.H[a].ctx = c.ctx;
    g.H[a].dec = c.dec;
    g.H[a].maxctx = c.maxctx;
    g.H[a].llm = c.llm;
    g.H[a].steps = c.steps;
    g.H[a].sa = c.sa;
    g.H[a].phase = c.phase;
    g.H[a].issue = c.issue;
    g.H[a].anchor = c.anchor;
    g.H[a].rem = c.rem;
    g.H[a].done = c.done;
    if (c.prio > 0)
      set_event_at(g, a, c.slot, c.inst, c.prio, c.t, nseq);
    else
      clear_event_at(g, a, c.slot, c.inst);
    if (srank >= 0) {
      g.H[a].start_rank = srank;
      g.H[a].logpos = lpos;
    }
    if (c.phase == ASB_PHASE_DONE) {
      set_tp_at(g, c.slot, EC_NAN);
      g.ctime[a] = c.t;
    } else if (c.llm > 0.0) {
      set_tp_at(g, c.slot, (double)c.dec / c.llm);
    }
    EC_APROF(w, 2); /* the write-back */
  }
  EC_APROF(w, 3); /* the loop's exit */
}

/* JOB_INIT (thread-level): per-agent state of a fresh scenario (engine.py:251-276) */
template <class W>
EC_COLD1 void job_init(W* w, const GP& g, int tid, int nthr) {
  const int A = g.A;
  for (int p = tid; p < A; p += nthr) g.arr_t[p] = g.arrival[g.arr_order[p]];
  AgentHot h0;
  h0.next_t = h0.llm = h0.issue = h0.anchor = h0.rem = h0.done = 0.0;
  h0.ctx = h0.dec = h0.maxctx = h0.next_seq = 0;
  h0.start_rank = -1;
  h0.steps = h0.inst = h0.sa = h0.mig = h0.next_prio = h0.pad0 = h0.pad1 = 0;
  h0.logpos = h0.slot = -1;
  h0.phase = ASB_PHASE_ARRIVING;
  for (int a = tid; a < A; a += nthr) {
    g.H[a] = h0;
    g.ctime[a] = EC_NAN;
    g.notbefore[a] = 0.0;
    g.pissue[a] = EC_NAN;
    g.rank[a] = -1;
    g.dstamp[a] = 0;
  }
  if (g.turn_issue) {
    const long long nt = g.aturn[A] - g.aturn[0];
    const long long t0 = g.aturn[0] - g.turn_base;
    for (long long t = tid; t < nt; t += nthr) {
      g.turn_issue[t0 + t] = EC_NAN;
      g.turn_done[t0 + t] = EC_NAN;
    }
  }
}

/* JOB_FINISH (thread-level): AgentResult fields from the hot records */
template <class W>
EC_COLD1 void job_finish(W* w, const GP& g, int tid, int nthr) {
  (void)w;
  for (int a = tid; a < g.A; a += nthr) {
    const AgentHot h = g.H[a];
    g.o_llm[a] = h.llm;
    g.o_dec[a] = h.dec;
    g.o_maxctx[a] = h.maxctx;
    g.o_ctx[a] = h.ctx;
    g.o_steps[a] = h.steps;
    g.o_inst[a] = h.inst;
    g.o_mig[a] = h.mig;
    g.o_phase[a] = h.phase;
  }
}

/* JOB_ADMIT (warp per instance): β/γ admission of the listed instances */
template <class W>
EC_COLD1 void job_admit(W* w, const GP& g, int tid, int nthr) {
  const int warp = tid / EC_TSIZE, nwarps = nthr >= EC_TSIZE ? nthr / EC_TSIZE : 1;
  for (int k = warp; k < w->n_eplist; k += nwarps) {
    const int i = w->ep_list[k];
    int n_start = 0;
    const int n_adm = admission(w, g, i, w->ep_gcap, &n_start);
    EC_LANE0 {
      w->ep_nadm[i - 1] = n_adm;
      w->ep_nstart[i - 1] = n_start;
    }
  }
}

/* JOB_EPOCH (warp per instance): re-time and start admitted turns of the
 * listed instances with their precomputed push seq / start rank bases */
template <class W>
EC_COLD1 void job_epoch(W* w, const GP& g, int tid, int nthr) {
  const int warp = tid / EC_TSIZE, nwarps = nthr >= EC_TSIZE ? nthr / EC_TSIZE : 1;
  const double now = w->now;
  for (int k = warp; k < w->n_eplist; k += nwarps) {
    const int i = w->ep_list[k];
    const int rt = w->ep_retime[i - 1];
    if (rt) log_pass<W, W::DC>(w, g, i, 1, w->ep_seq[i - 1], now, true, false);
    const int n_adm = w->ep_nadm[i - 1];
    if (n_adm)
      start_admitted<W, W::DC>(w, g, i, w->ep_head[i - 1], n_adm, w->ep_seq[i - 1] + rt, w->ep_rank[i - 1], true);
  }
}

template <class W>
EC_DEV void do_job(W* w, int job, int tid, int nthr) {
  const GP& g = w->gp;
  switch (job) {
    case JOB_INIT: job_init(w, g, tid, nthr); break;
    case JOB_SWEEP: job_sweep(w, g, tid, nthr); break;
    case JOB_SPEC: job_spec(w, g, tid, nthr); break;
    case JOB_SORT: job_sort(w, g, tid, nthr); break;
    case JOB_APPLY: job_apply(w, g, tid, nthr); break;
    case JOB_ADMIT: job_admit(w, g, tid, nthr); break;
    case JOB_EPOCH: job_epoch(w, g, tid, nthr); break;
    case JOB_FINISH: job_finish(w, g, tid, nthr); break;
    case JOB_DEPS:
      if (W::NW > 1 && (W::MX > 32 || EC_TEAM_DEPS_SMALL)) job_deps(w, g, tid, nthr);
      break;
    default: break;
  }
}

/* one optimistic batch inside the current window (main warp, forks jobs) */
template <class W, int RCAP, int DCAP, int ACAP>
EC_COLD3 int batch(W* w, const GP& g, double win_end) {
  /* ---- 1. due collection (shrink the window if too many agents are due) */
  EC_PROF_START(w);
  double bound = win_end;
  int incl = w->incl;
  int nd;
  EC_SPROF_T0(w);
  if (w->due_ready) {
    nd = w->n_cand; /* gathered by the tick sweep + epoch (may include agents no longer due) */
    t_sync();
    EC_LANE0 w->due_ready = 0;
  } else {
    nd = collect_due<W, DCAP>(w, g, bound, incl);
    EC_SPROF_ADD(w, 1);
  }
  if (nd > DCAP) {
    EC_SPROF_CNT(w, 3);
    /* bisection: largest exclusive bound lo with count(lo) <= DCAP */
    double lo = w->now, hi = bound;
    int clo = 0;
    for (int it = 0; it < 128; it++) {
      double mid = lo + (hi - lo) * 0.5;
      if (!(mid > lo && mid < hi)) break;
      int c = count_due(w, g, mid, 0);
      if (c > DCAP) {
        hi = mid;
      } else {
        lo = mid;
        clo = c;
        if (c * 2 >= DCAP) break;
      }
    }
    if (clo == 0) return BATCH_SERIAL; /* a same-timestamp burst larger than DCAP */
    bound = lo;
    incl = 0;
    nd = collect_due<W, DCAP>(w, g, bound, incl);
  }
  EC_SPROF_ADD(w, 4);
  t_sync();
  EC_PROF(w, 0);
  EC_LANE0 {
    w->n_due = nd;
    w->hz_t = EC_INF_BITS;
    w->hz_p = 0;
    w->hz_s = 0;
  }
  t_sync();
  EC_PROF(w, 2);
  /* ---- 2. arrivals in the window (sorted by (time, trace index)): the
   * window is a prefix of the sorted arrival times, read warp-parallel */
  {
    int n_arr = 0;
    const int p0 = w->arr_ptr;
    const double T = w->sc.sim_duration;
    const int nd = w->n_due;
    for (;;) {
      const int p = p0 + n_arr + EC_LANE;
      const double t = p < g.A ? g.arr_t[p] : EC_INF;
      const bool in = p < g.A && t < T && (incl ? t <= bound : t < bound);
      const int k = ec_popc(t_ballot(in)); /* in-window lanes form a prefix */
      const int room = ACAP - n_arr;
      const int take = k < room ? k : room;
      if (EC_LANE < take) {
        Rec& r = w->rec[nd + n_arr + EC_LANE];
        r.t = t;
        r.prio = EV_ARRIVAL;
        r.agent = g.arr_order[p];
        r.seq = p; /* arrivals tie-break by trace order (engine.py:315-317) */
        r.flags = 0;
        r.child = -1;
        r.inst = 0;
      }
      if (k > room && EC_LANE == room) {
        /* the first arrival that does not fit bounds the batch */
        const unsigned long long tb = ec_bits(t);
        if (below_horizon(tb, EV_ARRIVAL, p, w->hz_t, (unsigned)w->hz_p, w->hz_s)) {
          w->hz_t = tb;
          w->hz_p = EV_ARRIVAL;
          w->hz_s = p;
        }
      }
      n_arr += take;
      if (k < EC_TSIZE || take < k) break;
    }
    EC_LANE0 {
      w->n_arr = n_arr;
      w->n_rec = nd + n_arr;
      w->tmp_i = 0;
      w->n_empty = 0;
      w->j_bound = bound;
      w->j_incl = incl;
      w->j_order_err = 0;
    }
  }
  /* ---- 3. speculation */
  EC_DBG(2, w->n_rec);
  fork_job(w, JOB_SPEC);
  EC_DBG(3, w->tmp_i);
  {
    unsigned long long k = EC_INF_BITS;
    unsigned kp = 0;
    for (int q = 0; q < W::NW; q++)
      if (key_less(w->j_hz_t[q], w->j_hz_p[q], k, kp)) {
        k = w->j_hz_t[q];
        kp = w->j_hz_p[q];
      }
    t_sync();
    EC_LANE0 {
      if (below_horizon(k, kp, -1, w->hz_t, (unsigned)w->hz_p, w->hz_s)) {
        w->hz_t = k;
        w->hz_p = (int)kp;
        w->hz_s = -1;
      }
      const int nr0 = w->n_rec;
      const int extra = w->tmp_i;
      w->n_rec = nr0 + (extra < RCAP - nr0 ? extra : RCAP - nr0);
      if (w->j_order_err) w->status = ASB_SIMERR_ORDER;
      w->j_cut = 0x7fffffff;
      w->j_tie_unknown = 0;
    }
    t_sync();
  }
  /* ---- 4. rank sort + sorted SoA view */
  EC_PROF(w, 2);
#if defined(ASB_PROFILE) && !defined(ASB_PROFILE_WALK) && !defined(ASB_PROFILE_SWEEP) && !defined(ASB_PROFILE_SORT) && !defined(ASB_PROFILE_SPEC) && !defined(ASB_PROFILE_EPOCH) && !defined(ASB_PROFILE_APPLY)
  EC_LANE0 w->ctr[ASB_CTR_RETIMES] += w->n_rec; /* profile builds: sum of batch sizes */
  t_sync();
#endif
  fork_job(w, JOB_SORT);
  EC_DBG(4, w->n_rec);
  const int n = w->n_rec - w->n_empty; /* empty records rank last and are never walked */
  EC_PROF(w, 3);
  /* ---- 5. commit walk: parallel segmented scans, serial fallback */
  if (!walk_parallel<W, RCAP>(w, g, n)) walk_serial(w, g, n);
  EC_DBG(5, w->stop_kind);
  EC_PROF(w, 4);
  /* ---- 6. apply committed chain prefixes */
  {
    const int tid = EC_LANE; /* sub-step profile: lane 0 of the main warp */
    (void)tid;
    EC_APROF_T0();
    fork_job(w, JOB_APPLY);
    EC_APROF(w, 4); /* the apply fork-join, as the main warp sees it */
  }
  EC_DBG(6, w->ctr[ASB_CTR_BATCHES]);
  EC_LANE0 w->ctr[ASB_CTR_BATCHES]++;
  /* ---- 7. coupling / overflow follow-ups */
  const int stop = w->stop_kind;
  /* the rest of the (unshrunk) window keeps this batch's due list: every
   * agent with an event left in the window is one of them, or is re-timed
   * by the coupling event's handler (collected as it happens) */
  const bool keep = (bound == win_end && incl == w->incl) && w->n_due <= DCAP;
  if (stop == STOP_COUPLING) {
    EC_LANE0 {
      w->n_cand = w->n_due;
      w->cand_collect = keep;
    }
    t_sync();
    {
      const int tid = EC_LANE;
      (void)tid;
      EC_APROF_T0();
      exec_serial(w, g, w->stop_r); /* smem record: no local-memory copy */
      EC_APROF(w, 5); /* the coupling event, serially */
    }
    EC_LANE0 {
      w->cand_collect = 0;
      w->due_ready = keep && w->n_cand <= DCAP;
    }
    t_sync();
    EC_PROF(w, 5);
    return BATCH_MORE;
  }
  EC_PROF(w, 5);
  if (stop == STOP_LOGFULL || stop == STOP_HORIZON) {
    if (stop == STOP_LOGFULL) log_pass(w, g, w->stop_r.inst, 0, 0, w->now);
    EC_LANE0 {
      w->n_cand = w->n_due;
      w->due_ready = keep;
    }
    t_sync();
    return BATCH_MORE;
  }
  if (bound != win_end || incl != w->incl) {
    /* the shrunk window is fully committed: continue from its end */
    EC_LANE0 w->now = bound;
    t_sync();
    return BATCH_MORE;
  }
  return BATCH_DONE;
}

/* exact single-event fallback: process the minimum pending event serially
 * (the timeseries loop, and a burst of identical timestamps larger than the
 * batch buffers) */
template <class W>
EC_COLD2 bool serial_step(W* w, const GP& g, double win_end) {
  EC_DBG(11, w->n_alive);
  unsigned long long bt = EC_INF_BITS;
  unsigned bp = 0xffffffffu;
  long long bs = 0x7fffffffffffffffll;
  int ba = -1;
  for (int j = EC_LANE; j < w->n_alive; j += EC_TSIZE) {
    const int mt = g.sl[j].meta;
    const int pr = sm_prio(mt);
    if (pr <= 0) continue;
    const int a = sm_agent(mt);
    unsigned long long tb = ec_bits(g.H[a].next_t); /* the exact time (the slot's is rounded down) */
    long long s = g.H[a].next_seq;
    if (key_less(tb, (unsigned)pr, bt, bp) || (tb == bt && (unsigned)pr == bp && s < bs)) {
      bt = tb;
      bp = (unsigned)pr;
      bs = s;
      ba = a;
    }
  }
  for (int off = EC_TSIZE / 2; off > 0; off >>= 1) {
    unsigned long long ot = t_shfl_xor_ull(bt, off);
    unsigned op = (unsigned)t_shfl_xor_i((int)bp, off);
    long long os = t_shfl_xor_ll(bs, off);
    int oa = t_shfl_xor_i(ba, off);
    if (key_less(ot, op, bt, bp) || (ot == bt && op == bp && os < bs)) {
      bt = ot;
      bp = op;
      bs = os;
      ba = oa;
    }
  }
  /* the next arrival competes at priority 4 */
  int arr = -1;
  if (w->arr_ptr < g.A) {
    int a = g.arr_order[w->arr_ptr];
    double t = g.arrival[a];
    if (t < w->sc.sim_duration && key_less(ec_bits(t), EV_ARRIVAL, bt, bp)) arr = a;
  }
  t_sync(); /* every lane has read arr_ptr before lane 0 commits an arrival */
  if (arr < 0 && ba < 0) return false;
  double t = arr >= 0 ? g.arrival[arr] : ec_from_bits(bt);
  if (!(w->incl ? t <= win_end : t < win_end)) return false;
  if (g.ts_rows) {
    EC_LANE0 ts_samples(w, g, t);
    t_sync();
  }
  if (arr >= 0) {
    EC_LANE0 {
      w->now = t;
      const int target = route_arrival(w);
      commit_arrival(w, g, arr, target, w->arr_ptr);
      ts_mark(w, g, target);
    }
    t_sync();
    return true;
  }
  Rec r;
  r.t = t;
  r.prio = (short)bp;
  r.agent = ba;
  r.inst = g.H[ba].inst;
  exec_serial(w, g, r);
  return true;
}

/* Single-warp teams, windows with a handful of due agents (C3 averages 2.7
 * records per batch): the exact serial event loop over the window's due
 * list instead of speculate / sort / walk / apply.  The list holds every
 * agent with an event left in the window (the tick sweep and the epoch
 * collected them; agents the handlers re-time are appended as it runs,
 * cand_collect), so the next event is the minimum over the list and the
 * next arrival — serial_step's argmin without its sweep over every alive
 * slot.  A list that outgrows DCAP hands the rest of the window back to the
 * batches (due_ready = 0: they re-collect from the slots).
 * Measured slower on C3 and therefore OFF (EC_SERIAL_DUE_MAX = 0; an
 * experiment knob, exact either way — tests/test_host_engine.py runs it):
 * 342 ms with lists of <= 8, 328 ms with <= 20, 414 ms with <= 3, against
 * 310 ms for the batches.  One serial handler costs more than a whole
 * batch's share per record, and mixing both paths doubles the hot code. */
#ifndef EC_SERIAL_DUE_MAX
#define EC_SERIAL_DUE_MAX 0
#endif
#ifndef EC_SERIAL_DUE_ON /* which teams take the serial path (the 1-lane host harness switches it at run time) */
#define EC_SERIAL_DUE_ON(W) (W::NT == 32)
#endif
template <class W, int DCAP>
EC_COLD3 int serial_due(W* w, const GP& g, double win_end) {
  EC_LANE0 w->cand_collect = 1;
  t_sync();
  int rc = BATCH_DONE;
  for (;;) {
    const int nd = w->n_cand;
    if (nd > DCAP) {
      rc = BATCH_MORE;
      break;
    }
    unsigned long long bt = EC_INF_BITS;
    unsigned bp = 0xffffffffu;
    long long bs = 0x7fffffffffffffffll;
    int ba = -1;
    for (int j = EC_LANE; j < nd; j += EC_TSIZE) {
      const int a = w->due[j];
      const int pr = g.H[a].next_prio;
      if (pr <= 0) continue; /* a candidate no longer due */
      const unsigned long long tb = ec_bits(g.H[a].next_t);
      const long long s = g.H[a].next_seq;
      if (key_less(tb, (unsigned)pr, bt, bp) || (tb == bt && (unsigned)pr == bp && s < bs)) {
        bt = tb;
        bp = (unsigned)pr;
        bs = s;
        ba = a;
      }
    }
    for (int off = EC_TSIZE / 2; off > 0; off >>= 1) {
      unsigned long long ot = t_shfl_xor_ull(bt, off);
      unsigned op = (unsigned)t_shfl_xor_i((int)bp, off);
      long long os = t_shfl_xor_ll(bs, off);
      int oa = t_shfl_xor_i(ba, off);
      if (key_less(ot, op, bt, bp) || (ot == bt && op == bp && os < bs)) {
        bt = ot;
        bp = op;
        bs = os;
        ba = oa;
      }
    }
    /* the next arrival competes at priority 4 (as in serial_step) */
    int arr = -1;
    if (w->arr_ptr < g.A) {
      const int a = g.arr_order[w->arr_ptr];
      const double t = g.arrival[a];
      if (t < w->sc.sim_duration && key_less(ec_bits(t), EV_ARRIVAL, bt, bp)) arr = a;
    }
    t_sync(); /* every lane has read arr_ptr and the list before lane 0 commits */
    if (arr < 0 && ba < 0) break;
    const double t = arr >= 0 ? g.arrival[arr] : ec_from_bits(bt);
    if (!(w->incl ? t <= win_end : t < win_end)) break;
    if (arr >= 0) {
      EC_LANE0 {
        w->now = t;
        const int target = route_arrival(w);
        commit_arrival(w, g, arr, target, w->arr_ptr);
      }
      t_sync();
      continue;
    }
    Rec r;
    r.t = t;
    r.prio = (short)bp;
    r.agent = ba;
    r.inst = g.H[ba].inst;
    exec_serial(w, g, r);
  }
  EC_LANE0 {
    w->cand_collect = 0;
    w->due_ready = 0;
  }
  t_sync();
  return rc;
}

/* TS: the scenario writes timeseries rows (g.ts_rows) and runs the exact
 * serial loop; a separate instantiation keeps the batched engine's code
 * unchanged */
template <class W, int RCAP, int DCAP, int ACAP, bool TS>
EC_DEV void run_scenario(W* w, const GP& g) {
  const AsbScenario& sc = w->sc;
  const int M = ec_nm(w), L = sc.n_levels;
#ifdef ASB_PROFILE_PLACEMENT
  EC_LANE0 w->prof_t = ec_globaltimer();
#endif
  /* ---- init (engine.py:251-276) */
  fork_job(w, JOB_INIT);
  EC_ILOOP /* per-instance loop: rolled (instruction cache) */
  for (int i = EC_LANE; i < M; i += EC_TSIZE) {
    Inst& in = w->in[i];
    in.usage = 0;
    in.watts = w->idle[L - 1];
    in.t_pow = in.energy = in.thr_since = in.thr_time = 0.0;
    in.level = L;
    in.running = in.thr = in.thr_flag = 0;
    in.key_valid = in.key_level = in.key_thr = in.key_run = 0;
    in.fifo_head = in.fifo_len = in.log_len = 0;
  }
  EC_LANE0 {
    w->now = 0.0;
    w->seq = 0;
    w->start_ctr = 0;
    for (int c = 0; c < ASB_NCOUNTERS; c++) w->ctr[c] = 0;
    w->n_alive = w->rr_next = w->arr_ptr = w->arr_rank = w->status = 0;
    w->due_ready = w->n_cand = w->cand_token = w->n_empty = w->cand_collect = 0;
    w->stamp_ctr = 0;
    for (int c = 0; c < 6; c++) w->prof[c] = 0;
    if (TS) {
      w->ts_n = 0;
      w->ts_k = 1;
      for (int i = 0; i < M; i++) w->ts_last[i] = -1;
      /* run(), engine.py:576-579: a forced row per instance before any event */
      if (g.ts_rows)
        for (int i = 1; i <= M; i++) mark_row(w, g, i, 0.0, true);
    }
  }
  t_sync();
  const long long K = sc.n_epochs;
  const double E = sc.epoch_length, T = sc.sim_duration;
  for (long long k = 0; k < K && w->status == 0; k++) {
    const bool last = k + 1 == K;
    const double win_end = last ? T : (double)(k + 1) * E;
    EC_LANE0 {
      w->now = (double)k * E;
      w->incl = last ? 1 : 0;
      w->bound = win_end;
    }
    t_sync();
    EC_DBG(0, k);
    epoch_event<W, DCAP>(w, g, k);
    EC_DBG(1, k);
    /* watchdog: every batch commits or executes at least one event, so a
     * window never needs more batches than live events + arrivals (+ the
     * window-shrink restarts); exceeding a generous bound is a bug */
    long long guard = 64 + 4 * (long long)(g.A + w->n_alive) + 8 * (long long)g.A;
    for (;;) {
      if (w->status) break;
      if (--guard < 0) {
        EC_LANE0 {
          w->status = ASB_SIMERR_LIVELOCK;
          w->ctr[10] = k;
          w->ctr[11] = w->stop_kind;
          w->ctr[12] = w->n_rec;
          w->ctr[13] = (long long)ec_bits(w->now);
          w->ctr[14] = w->n_due;
          w->ctr[15] = w->ctr[ASB_CTR_EVENTS];
        }
        t_sync();
        break;
      }
      if (TS) {
        /* timeseries: the exact serial loop, one event at a time (each step
         * executes an event, so the watchdog does not apply) */
        guard++;
        if (!serial_step(w, g, win_end)) {
          EC_LANE0 if (g.ts_rows) ts_samples(w, g, win_end);
          t_sync();
          break;
        }
        continue;
      }
      int rc;
      if (EC_SERIAL_DUE_ON(W) && EC_SERIAL_DUE_MAX > 0 && w->due_ready && w->n_cand <= EC_SERIAL_DUE_MAX)
        rc = serial_due<W, DCAP>(w, g, win_end);
      else
        rc = batch<W, RCAP, DCAP, ACAP>(w, g, win_end);
      if (rc == BATCH_MORE) continue;
      if (rc == BATCH_DONE) break;
      /* a same-timestamp burst larger than the due buffer: one exact step */
      if (!serial_step(w, g, win_end)) break;
    }
  }
  /* ---- final accounting (engine.py:595-603) and outputs */
  EC_ILOOP /* per-instance loop: rolled (instruction cache) */
  for (int i = EC_LANE; i < M; i += EC_TSIZE) {
    Inst& in = w->in[i];
    in.energy += in.watts * (T - in.t_pow);
    in.t_pow = T;
    if (in.thr_flag) {
      in.thr_time += T - in.thr_since;
      in.thr_since = T;
    }
    g.o_energy[i] = in.energy;
    g.o_thr[i] = in.thr_time;
    g.o_usage[i] = in.usage;
    g.o_pending[i] = in.fifo_len;
    g.o_level[i] = in.level;
  }
  if (TS) {
    t_sync();
    EC_LANE0 {
      /* engine.py:595-603: a forced row per instance at the end */
      if (g.ts_rows)
        for (int i = 1; i <= M; i++) mark_row(w, g, i, T, true);
      if (g.ts_count) *g.ts_count = w->ts_n;
    }
    t_sync();
  }
  fork_job(w, JOB_FINISH);
  EC_LANE0 {
    w->ctr[ASB_CTR_STATUS] = w->status;
#ifdef ASB_PROFILE
    for (int c = 0; c < 6; c++) w->ctr[10 + c] = w->prof[c];
#endif
#ifdef ASB_PROFILE_PLACEMENT
    /* experiment: where and when the scenario ran (SM id, global ns) */
    w->ctr[10] = ec_smid();
    w->ctr[11] = w->prof_t;
    w->ctr[12] = ec_globaltimer();
#endif
    for (int c = 0; c < ASB_NCOUNTERS; c++) g.o_ctr[c] = w->ctr[c];
  }
  t_sync();
}

}  // namespace asb

#endif
