/*
 * agentsim_b200.h — C ABI of the B200-native batched scenario engine.
 *
 * This is the drop-in boundary for the reference's hot path: one call runs
 * many independent agentic-serving scenarios (each one a full
 * `run_simulation`, /root/reference/pkg/src/agentsim/engine.py:752-754) on
 * the GPU.  The reference has no FFI of its own (it is pure Python); the
 * Python mirror in `paper_2604_16682_b200/` binds these symbols with ctypes
 * exactly as a maintainer would bind them from `agentsim`.
 *
 * Conventions
 *  - plain pointers and sizes only; every pointer inside the pool/output
 *    structs is a DEVICE pointer for the `asb_*` GPU entry points;
 *  - caller owns all memory (no allocation inside), including the workspace
 *    sized by `asb_workspace_bytes`;
 *  - calls are stream-ordered on `stream` (a cudaStream_t, NULL = legacy);
 *  - return value: 0 ok, <0 launch/argument error (see asb_status_t);
 *    invariant violations that the reference raises as SimulationError
 *    (engine.py, instance.py:209-227, router.py:160-174) are reported per
 *    scenario in counters[ASB_CTR_STATUS] and raised by the host mirror.
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src/agentsim):
 *   asb_run_scenarios       run_simulation                 engine.py:752-754
 *                           (_Simulation.run               engine.py:576-604)
 *   asb_select_level_batch  select_frequency_level         controller.py:81-86
 *   asb_service_time_batch  service_time                   instance.py:184-204
 *   asb_assign_batch        assign_agent / route_least_loaded router.py:75-94, 142-151
 *   asb_reassign_batch      maybe_reassign                 router.py:97-128
 *   asb_min_throughput_batch min_throughput / running_throughput controller.py:89-103
 *   asb_scenario_stats      SystemMetrics in _build_result engine.py:632-655,
 *                           slo_attainment / percentile_throughput metrics.py:49-69
 *   asb_regime_classify     regime_classify over SimulationResult.usage_series()
 *                           metrics.py:72-109, engine.py:176-182
 */
#ifndef AGENTSIM_B200_H
#define AGENTSIM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ASB_ABI_VERSION 1
/* engine limits: instance ids fit 7 bits of an alive slot's meta word;
 * frequency tables are staged in shared memory per scenario */
#define ASB_MAX_INSTANCES 127
#define ASB_MAX_LEVELS 64

typedef enum {
  ASB_OK = 0,
  ASB_ERR_ARG = -1,
  ASB_ERR_LAUNCH = -2,
  ASB_ERR_WORKSPACE = -3,
} asb_status_t;

/* controller variants, controller.py:26 */
enum { ASB_VARIANT_CONTEXT_AWARE = 0, ASB_VARIANT_OFF = 1, ASB_VARIANT_FIXED = 2 };
/* router policies, router.py:21 */
enum { ASB_POLICY_CONTEXT_AWARE = 0, ASB_POLICY_ROUND_ROBIN = 1, ASB_POLICY_LEAST_LOADED = 2 };
/* agent phases, engine.py:226 + AgentResult.final_phase engine.py:131 */
enum {
  ASB_PHASE_ARRIVING = 0,
  ASB_PHASE_PENDING = 1,
  ASB_PHASE_RUNNING = 2,
  ASB_PHASE_TOOL = 3,
  ASB_PHASE_WAITING_START = 4,
  ASB_PHASE_DONE = 5
};

/* per-scenario counters (int64) */
enum {
  ASB_CTR_TICKS = 0,        /* agent-ticks: running_throughput evaluations, controller.py:89-103 */
  ASB_CTR_ARRIVED = 1,      /* SimulationResult.arrived */
  ASB_CTR_COMPLETED = 2,    /* SimulationResult.completed */
  ASB_CTR_TURNS = 3,        /* completed turns (sum of turns_completed) */
  ASB_CTR_EVENTS = 4,       /* live events processed (stale completions excluded) */
  ASB_CTR_MIGRATIONS = 5,   /* executed reassignments */
  ASB_CTR_THRASH_FLIPS = 6, /* thrash-flag transitions, engine.py:329-336 */
  ASB_CTR_RETIMES = 7,      /* re-timed in-flight turns, engine.py:355-372 */
  ASB_CTR_STATUS = 8,       /* 0 ok; otherwise ASB_SIMERR_* */
  ASB_CTR_BATCHES = 9,      /* engine-internal: commit batches (GPU) / 0 (oracle) */
  ASB_NCOUNTERS = 16
};

enum {
  ASB_SIMERR_NONE = 0,
  ASB_SIMERR_INVARIANT = 1, /* state-machine misuse (SimulationError) */
  ASB_SIMERR_OVERFLOW = 2,  /* a bounded engine buffer overflowed */
  ASB_SIMERR_ORDER = 3,     /* an event was scheduled before its parent */
  ASB_SIMERR_LIVELOCK = 4   /* engine watchdog: a window made no progress */
};

/* One scenario = one SimConfig (engine.py:57-88) bound to a trace. 8-byte aligned. */
typedef struct AsbScenario {
  int32_t trace_id;              /* index into the trace pool */
  int32_t table_id;              /* index into the frequency-table pool */
  int32_t n_instances;           /* SimConfig.instance_count */
  int32_t n_levels;              /* FrequencyTable.num_levels */
  int64_t capacity;              /* InstanceConfig.capacity_tokens */
  double thrash_factor;          /* InstanceConfig.thrash_latency_factor */
  double interference;           /* InstanceConfig.interference_coeff */
  /* controller, controller.py:29-66 */
  int32_t variant;
  int32_t fixed_level;           /* 1-based level for variant fixed (host resolves index_of_mhz) */
  int32_t boost_enabled;
  int32_t thrash_avoidance;
  double alpha, beta, gamma, slo_target, epoch_length;
  /* router, router.py:24-59 */
  int32_t policy;
  int32_t reassign_interval;
  int32_t include_idle;
  int32_t reset_only_on_reassign;
  double consolidation_threshold;
  double imbalance_ratio;
  double migration_delay;
  /* sim */
  double sim_duration;
  int64_t n_epochs;              /* #{k : k*epoch_length < sim_duration}, engine.py:306-309 */
  double record_interval;        /* SimConfig.record_interval: sample events at k*interval, engine.py:310-313 */
} AsbScenario;

/* Trace pool: CSR of AgentTrace/TurnRecord (workload.py:83-116), shared by scenarios. */
typedef struct AsbTracePool {
  int32_t n_traces;
  int32_t pad_;
  const int64_t* trace_agent_off;  /* [n_traces+1] -> agent rows */
  const int64_t* trace_turn_off;   /* [n_traces+1] -> turn rows (first turn of the trace) */
  const double* arrival;           /* [n_agents] AgentTrace.arrival_time */
  const int64_t* agent_turn_off;   /* [n_agents+1] global turn offsets */
  const int32_t* prefill;          /* [n_turns] TurnRecord.prefill_tokens */
  const int32_t* decode;           /* [n_turns] TurnRecord.decode_tokens */
  const double* tool;              /* [n_turns] TurnRecord.tool_time */
  const int32_t* arrival_order;    /* [n_agents] per trace: local agent ids sorted by (arrival, index) */
} AsbTracePool;

/* Frequency tables (instance.py:24-112), 1-based level l at table_off[t] + l - 1. */
typedef struct AsbTablePool {
  int32_t n_tables;
  int32_t max_levels;              /* host-side: the largest level count in the pool, 0 = at most 16 */
  const int64_t* table_off;        /* [n_tables+1] */
  const double* mhz;
  const double* prefill_rate;
  const double* decode_rate;
  const double* active_power;
  const double* idle_power;
} AsbTablePool;

/* DecisionRow, engine.py:104-114.  min_throughput = NaN encodes None. */
typedef struct AsbDecision {
  double time;
  double min_throughput;
  int64_t usage_observed;
  int32_t instance_id;
  int32_t frequency_level;
  int32_t admitted_count;
  int32_t pending_depth;
  int32_t boosted;
  int32_t deferred;
} AsbDecision;

/* TimeseriesRow, engine.py:91-101, as _mark_row writes it (engine.py:403-429).
 * level_mhz is not stored: it is table.level(level_index).nominal_mhz. */
typedef struct AsbTimeseriesRow {
  double time;
  double power_watts;
  int64_t context_usage;
  int32_t instance_id;
  int32_t level_index;           /* 1-based */
  int32_t pending_depth;
  int32_t running_requests;
  int32_t thrashing;
  int32_t pad_;
} AsbTimeseriesRow;

/* Outputs.  Agent rows are in TRACE order (local agent index); arrival_rank
 * gives the reference's result order (engine.py:609, dict insertion order),
 * -1 for agents that never arrived inside the window. */
typedef struct AsbOutputs {
  const int64_t* agent_off;        /* [n_scen+1] agent row offset per scenario */
  const int64_t* inst_off;         /* [n_scen+1] instance row offset per scenario */
  /* per agent */
  double* completion_time;         /* NaN = None */
  double* llm_time;                /* AgentRuntimeState.llm_time_total */
  int64_t* decode_total;
  int64_t* max_context;
  int64_t* context;
  int32_t* turns_completed;
  int32_t* final_instance;         /* 1-based; 0 = None */
  int32_t* migrations;
  int32_t* phase;
  int32_t* arrival_rank;
  /* per instance */
  double* energy;                  /* instance_energy */
  double* thrash_time;             /* instance_thrash_time */
  int64_t* final_usage;
  int32_t* final_pending;
  int32_t* final_level;
  int32_t pad_;
  /* per scenario */
  int64_t* counters;               /* [n_scen * ASB_NCOUNTERS] */
  /* optional (NULL to skip): decision log, [dec_off[s], dec_off[s+1]) = n_epochs * n_instances rows */
  const int64_t* dec_off;
  AsbDecision* decisions;
  /* optional (NULL to skip): per-turn log at turn_off[s] + (turn - trace_turn_off[trace]) */
  const int64_t* turn_off;
  double* turn_issue;              /* NaN when the turn did not complete */
  double* turn_done;
  /* optional (NULL to skip): timeseries rows in the reference's emission
   * order, capacity [ts_off[s], ts_off[s+1]) per scenario, the number written
   * in ts_count[s].  A scenario with rows enabled runs the engine's exact
   * serial event loop (one event at a time, sample events included) instead
   * of the optimistic batches: same results, far slower; meant for single
   * runs that need the series.  A capacity of
   *   n_instances * (2 + n_samples + n_epochs) + n_agents + n_turns
   *     + 3 * (n_turns - n_agents)
   * can never overflow: forced rows per instance (engine.py:488, 572, 579,
   * 603), one per arrival and completion (507, 535), two per tool event
   * (source and migration target, 549, 560-561) and one per delayed start,
   * which only follows a migration (568).
   * timeseries != NULL requires ts_off and ts_count (else ASB_ERR_ARG). */
  const int64_t* ts_off;
  AsbTimeseriesRow* timeseries;
  int64_t* ts_count;
} AsbOutputs;

/* per-scenario system metrics (SystemMetrics, metrics.py:37-46). NaN encodes None. */
typedef struct AsbStats {
  double slo_attainment;
  double p5_throughput;
  double job_throughput;
  double average_power;
  double energy;
  double thrash_fraction;
  int64_t slo_met;
  int64_t n_completed_with_tp;
} AsbStats;

/* ---------------- GPU entry points (device pointers) ---------------- */

int asb_abi_version(void);

/* bytes of device workspace needed for a batch of n_scen scenarios covering
 * `total_agents` agent rows (sum over scenarios of their trace's agent count,
 * == out.agent_off[n_scen]) and `total_ring_slots` = sum over scenarios of
 * n_instances * agent count (pending FIFOs and running logs). */
size_t asb_workspace_bytes(int32_t n_scen, int64_t total_agents, int64_t total_ring_slots);

/* Run all scenarios to completion (one CTA team per scenario, persistent grid).
 * d_scen: device array of n_scen AsbScenario; max_instances = max
 * n_instances over the batch (<= 64), or -m when every scenario of the batch
 * has exactly m instances (the launcher then picks a kernel whose instance
 * count is a compile-time constant). */
int asb_run_scenarios(const AsbScenario* d_scen, int32_t n_scen, int32_t max_instances,
                      AsbTracePool traces, AsbTablePool tables, AsbOutputs out,
                      int64_t total_agents, int64_t total_ring_slots, void* d_workspace,
                      size_t workspace_bytes, void* stream);

/* device-side SystemMetrics per scenario (engine.py:632-655). */
int asb_scenario_stats(const AsbScenario* d_scen, int32_t n_scen, AsbOutputs out,
                       AsbStats* d_stats, void* d_workspace, size_t workspace_bytes,
                       void* stream);

/* Batched unit ops (SPEC acceptance criteria 1-2 grids; K3/K4 of SURVEY §2). */
int asb_select_level_batch(const double* usage, const double* capacity,
                           const int32_t* num_levels, const double* alpha, int32_t* level_out,
                           int64_t n, void* stream);
int asb_service_time_batch(const int32_t* prefill, const int32_t* decode,
                           const double* prefill_rate, const double* decode_rate,
                           const int32_t* concurrent, const int32_t* thrashing,
                           double interference, double thrash_factor, double* out, int64_t n,
                           void* stream);
/* usages: [n, max_m] row-major (tokens as double, exact below 2^53); m[r]
 * instances in row r (ids 1..m).  policy: CONTEXT_AWARE or LEAST_LOADED. */
int asb_assign_batch(const double* usages, const int32_t* m, int32_t max_m, int64_t capacity,
                     double consolidation_threshold, int32_t policy, int32_t* target_out,
                     int64_t n, void* stream);
/* counters in/out; target_out 0 = None. */
int asb_reassign_batch(const double* usages, const int32_t* m, int32_t max_m,
                       const int32_t* current, int32_t* counters, int32_t reassign_interval,
                       double imbalance_ratio, int32_t include_idle, int32_t reset_only,
                       int32_t* target_out, int64_t n, void* stream);

/* K0 stand-alone: min running throughput per segment (NaN = None);
 * scratch_bits: n_seg doubles of device scratch.  controller.py:89-103 */
int asb_min_throughput_batch(const int64_t* decode_total, const double* llm_time,
                             const int32_t* segment, int64_t n, int32_t n_seg,
                             double* scratch_bits, double* min_out, void* stream);

/* Stats vector allreduced across ranks; filled from counters/stats. */
enum {
  ASB_RED_ENERGY = 0,
  ASB_RED_THRASH_FRAC = 1,  /* sum of per-scenario thrash fractions */
  ASB_RED_COMPLETED = 2,
  ASB_RED_SLO_MET = 3,
  ASB_RED_TICKS = 4,
  ASB_RED_THRASH_FLIPS = 5,
  ASB_RED_MIGRATIONS = 6,
  ASB_RED_TURNS = 7,
  ASB_NRED = 8
};
/* fold per-scenario counters + stats into one double[ASB_NRED] vector on device */
int asb_reduce_stats(const AsbStats* d_stats, const int64_t* d_counters, int32_t n_scen,
                     double* d_red, void* stream);

/* One span of regime_classify's per-instance segments (metrics.py:72-109). */
typedef struct AsbRegimeSpan {
  double start;
  double end;
  int32_t instance_id;
  int32_t thrashing; /* usage > capacity over [start, end) */
} AsbRegimeSpan;

/* regime_classify(usage_series, capacity, window) on the device, per scenario,
 * over the timeseries rows asb_run_scenarios wrote (AsbOutputs.timeseries /
 * ts_off / ts_count): each instance's usage points (row.time,
 * float(row.context_usage)) in row order, split into merged non-thrashing /
 * thrashing spans clipped to the window (spans grouped by instance id
 * 1..n_instances, in time order), and the thrashing share of the total
 * instance-time (thrash sums restate Python's float sum()).  Span buffer of
 * scenario s: [span_off[s], span_off[s+1]), needing at least ts_count[s] +
 * n_instances[s] entries.  status[s]: 0, or the first instance id whose
 * series does not cover the window start (the reference's SimulationError),
 * or -1 when the span buffer is too small.  window must be > 0 (the host
 * raises ConfigurationError first). */
int asb_regime_classify(const AsbTimeseriesRow* rows, const int64_t* ts_off, const int64_t* ts_count,
                        int32_t n_scen, const int32_t* n_instances, const double* capacity,
                        const double* window, const int64_t* span_off, AsbRegimeSpan* spans,
                        int64_t* span_count, double* thrash_fraction, int32_t* status, void* stream);

/* ABI self-check: writes sizeof of AsbScenario, AsbTracePool, AsbTablePool,
 * AsbOutputs, AsbDecision, AsbStats, AsbTimeseriesRow, AsbRegimeSpan into
 * out[0..7]; returns 8. */
int asb_struct_sizes(int64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* AGENTSIM_B200_H */
