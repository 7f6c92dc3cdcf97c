/*
 * des_oracle.c — TEST INFRASTRUCTURE ONLY (the checker and the CPU baseline).
 *
 * A serial, single-threaded-per-scenario C restatement of the reference's
 * discrete-event engine (/root/reference/pkg/src/agentsim/engine.py) and the
 * policy/instance functions it calls (controller.py, router.py,
 * instance.py).  It keeps the reference's global event heap with
 * (time, priority, seq) ordering and lazy deletion of superseded
 * completions, so it reproduces the reference's push order, tie breaks and
 * IEEE-754 double arithmetic operation for operation (compiled with
 * -ffp-contract=off; Python never fuses multiply-add).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may load this
 * library.  The product path (paper_2604_16682_b200) never does.
 *
 * Parity pin: tests/test_oracle_golden.py checks this oracle against golden
 * vectors produced by the reference itself (tests/golden/make_golden.py).
 *
 * Deliberate, result-preserving restatements (each argued in DESIGN.md):
 *  - `sample` events (engine.py:570-572) only emit timeseries rows; they are
 *    scheduled only when the caller asks for rows (AsbOutputs.timeseries).
 *    They never change state, and their priority (5) is the lowest, so they
 *    do not change the order of the other events.
 *  - `min_throughput` of every instance is evaluated once at the start of
 *    the epoch event over the alive list: epoch processing of instance j
 *    never changes the in-process set or throughputs of instance i != j
 *    (engine.py:436-488), and the strict `<` min is order independent
 *    (controller.py:96-103).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/agentsim_b200.h"

#ifdef _OPENMP
#include <omp.h>
#endif

/* event kinds and tie-break priorities, engine.py:48-54 */
enum { EV_EPOCH = 0, EV_COMPLETE = 1, EV_TOOL = 2, EV_ISSUE = 3, EV_ARRIVAL = 4, EV_SAMPLE = 5 };

typedef struct {
  double t;
  int64_t seq;
  int32_t prio;
  int32_t agent; /* agent id, arrival: trace-local index */
  int64_t version;
  double issue; /* delayed_start payload */
} Ev;

typedef struct {
  Ev* a;
  int64_t n, cap;
} Heap;

static int ev_less(const Ev* x, const Ev* y) {
  if (x->t != y->t) return x->t < y->t;
  if (x->prio != y->prio) return x->prio < y->prio;
  return x->seq < y->seq;
}

static int heap_push(Heap* h, Ev e) {
  if (h->n == h->cap) {
    int64_t nc = h->cap ? h->cap * 2 : 1024;
    Ev* na = (Ev*)realloc(h->a, (size_t)nc * sizeof(Ev));
    if (!na) return -1;
    h->a = na;
    h->cap = nc;
  }
  int64_t i = h->n++;
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (!ev_less(&e, &h->a[p])) break;
    h->a[i] = h->a[p];
    i = p;
  }
  h->a[i] = e;
  return 0;
}

static Ev heap_pop(Heap* h) {
  Ev top = h->a[0];
  Ev last = h->a[--h->n];
  int64_t i = 0;
  for (;;) {
    int64_t l = 2 * i + 1;
    if (l >= h->n) break;
    int64_t c = l;
    if (l + 1 < h->n && ev_less(&h->a[l + 1], &h->a[l])) c = l + 1;
    if (!ev_less(&h->a[c], &last)) break;
    h->a[i] = h->a[c];
    i = c;
  }
  if (h->n > 0) h->a[i] = last;
  return top;
}

typedef struct {
  int64_t ctx, dec_tot, max_ctx;
  double llm_t;
  int32_t steps, s_a, inst, phase, migrations, n_turns;
  double completion_time, not_before, pending_issue;
  int32_t has_pending_issue;
  /* running turn (engine.py:210-219) */
  int32_t running, turn_idx;
  double issue_t, anchor, rem, done;
  int64_t version;
  int32_t run_prev, run_next; /* insertion-ordered running dict */
  int32_t fifo_next;          /* pending deque */
  int32_t alive_pos;
  int64_t turn0;              /* global turn offset */
} Agent;

typedef struct {
  int32_t level, running, thrashing;
  int64_t usage;
  int32_t fifo_head, fifo_tail, fifo_len;
  int32_t run_head, run_tail;
  double watts, t_pow, energy;
  int32_t thr_flag;
  double thr_since, thr_time;
  int32_t key_valid, key_level, key_thr, key_run;
  /* last timeseries row key, engine.py:405-414 */
  int32_t row_valid, row_level, row_pending, row_running, row_thr;
  int64_t row_usage;
  double row_watts;
} Inst;

typedef struct {
  const AsbScenario* sc;
  const AsbTracePool* tp;
  const AsbTablePool* tb;
  int64_t tbl0;   /* table offset */
  int64_t a0;     /* first global agent row of the trace */
  int32_t A, M;
  Agent* ag;
  Inst* in;       /* 1-based */
  int32_t* alive;
  int32_t n_alive;
  Heap heap;
  int64_t seq, versions;
  double now;
  int32_t rr_next;
  int64_t ctr[ASB_NCOUNTERS];
  int32_t status;
  /* epoch scratch */
  double* min_tp;
  int32_t* has_tp;
  int64_t* cnt;
  int32_t* admitted;
  /* outputs */
  const AsbOutputs* out;
  int64_t oa0, oi0;
  AsbDecision* dec;
  double *turn_issue, *turn_done;
  int32_t arrival_rank;
  int32_t* rank;
  AsbTimeseriesRow* ts; /* NULL: no rows */
  int64_t ts_cap, ts_n;
} Sim;

static inline double lvl_pr(const Sim* s, int l) { return s->tb->prefill_rate[s->tbl0 + l - 1]; }
static inline double lvl_dr(const Sim* s, int l) { return s->tb->decode_rate[s->tbl0 + l - 1]; }
static inline double lvl_act(const Sim* s, int l) { return s->tb->active_power[s->tbl0 + l - 1]; }
static inline double lvl_idle(const Sim* s, int l) { return s->tb->idle_power[s->tbl0 + l - 1]; }

static void push(Sim* s, double t, int prio, int agent, int64_t version, double issue) {
  Ev e;
  e.t = t;
  e.prio = prio;
  e.seq = s->seq++;
  e.agent = agent;
  e.version = version;
  e.issue = issue;
  if (heap_push(&s->heap, e)) s->status = ASB_SIMERR_OVERFLOW;
}

/* service_time, instance.py:184-204 */
static double service_time(const Sim* s, int64_t turn, int level, int concurrent, int thrashing) {
  double base = (double)s->tp->prefill[turn] / lvl_pr(s, level) +
                (double)s->tp->decode[turn] / lvl_dr(s, level);
  int extra = concurrent - 1 > 0 ? concurrent - 1 : 0;
  double factor = 1.0 + s->sc->interference * (double)extra;
  if (thrashing) factor *= s->sc->thrash_factor;
  return base * factor;
}

/* InstanceState.refresh_thrashing, instance.py:180-181 */
static inline void refresh_thrashing(Sim* s, Inst* in) { in->thrashing = in->usage > s->sc->capacity; }

/* _update_power, engine.py:321-327 */
static void update_power(Sim* s, Inst* in) {
  double w = in->running > 0 ? lvl_act(s, in->level) : lvl_idle(s, in->level);
  if (w != in->watts) {
    in->energy += in->watts * (s->now - in->t_pow);
    in->t_pow = s->now;
    in->watts = w;
  }
}

/* _sync_thrash, engine.py:329-336 */
static void sync_thrash(Sim* s, Inst* in) {
  int flag = in->thrashing;
  if (flag != in->thr_flag) {
    if (in->thr_flag)
      in->thr_time += s->now - in->thr_since;
    else
      in->thr_since = s->now;
    in->thr_flag = flag;
    s->ctr[ASB_CTR_THRASH_FLIPS]++;
  }
}

/* _mark_row, engine.py:403-429: a row when the instance's observable key
 * changed since its last row (or always, when forced) */
static void mark_row(Sim* s, int i, int force) {
  if (!s->ts) return;
  Inst* in = &s->in[i];
  if (!force && in->row_valid && in->row_usage == in->usage && in->row_level == in->level &&
      in->row_watts == in->watts && in->row_pending == in->fifo_len && in->row_running == in->running &&
      in->row_thr == in->thrashing)
    return;
  in->row_valid = 1;
  in->row_usage = in->usage;
  in->row_level = in->level;
  in->row_watts = in->watts;
  in->row_pending = in->fifo_len;
  in->row_running = in->running;
  in->row_thr = in->thrashing;
  if (s->ts_n >= s->ts_cap) {
    s->status = ASB_SIMERR_OVERFLOW;
    return;
  }
  AsbTimeseriesRow* r = &s->ts[s->ts_n++];
  r->time = s->now;
  r->power_watts = in->watts;
  r->context_usage = in->usage;
  r->instance_id = i;
  r->level_index = in->level;
  r->pending_depth = in->fifo_len;
  r->running_requests = in->running;
  r->thrashing = in->thrashing;
  r->pad_ = 0;
}

/* _conditions_changed, engine.py:344-372 */
static void conditions_changed(Sim* s, Inst* in) {
  int kl = in->level, kt = in->thrashing, kr = s->sc->interference > 0 ? in->running : 0;
  if (in->key_valid && kl == in->key_level && kt == in->key_thr && kr == in->key_run) return;
  in->key_valid = 1;
  in->key_level = kl;
  in->key_thr = kt;
  in->key_run = kr;
  for (int32_t a = in->run_head; a >= 0; a = s->ag[a].run_next) {
    Agent* g = &s->ag[a];
    double segment = g->done - g->anchor;
    if (segment > 0) {
      double fraction_done = (s->now - g->anchor) / segment;
      double x = 1.0 - fraction_done;
      g->rem *= (x > 0.0 ? x : 0.0);
    }
    double full = service_time(s, g->turn0 + g->turn_idx, in->level, in->running, in->thrashing);
    g->anchor = s->now;
    g->done = s->now + g->rem * full;
    g->version = s->versions++;
    push(s, g->done, EV_COMPLETE, a, g->version, 0.0);
    s->ctr[ASB_CTR_RETIMES]++;
  }
}

static void run_append(Sim* s, Inst* in, int32_t a) {
  Agent* g = &s->ag[a];
  g->run_prev = in->run_tail;
  g->run_next = -1;
  if (in->run_tail >= 0)
    s->ag[in->run_tail].run_next = a;
  else
    in->run_head = a;
  in->run_tail = a;
  g->running = 1;
}

static void run_remove(Sim* s, Inst* in, int32_t a) {
  Agent* g = &s->ag[a];
  if (g->run_prev >= 0)
    s->ag[g->run_prev].run_next = g->run_next;
  else
    in->run_head = g->run_next;
  if (g->run_next >= 0)
    s->ag[g->run_next].run_prev = g->run_prev;
  else
    in->run_tail = g->run_prev;
  g->running = 0;
}

static void fifo_append(Inst* in, Sim* s, int32_t a) {
  s->ag[a].fifo_next = -1;
  if (in->fifo_tail >= 0)
    s->ag[in->fifo_tail].fifo_next = a;
  else
    in->fifo_head = a;
  in->fifo_tail = a;
  in->fifo_len++;
}

static int32_t fifo_pop(Inst* in, Sim* s) {
  int32_t a = in->fifo_head;
  in->fifo_head = s->ag[a].fifo_next;
  if (in->fifo_head < 0) in->fifo_tail = -1;
  in->fifo_len--;
  s->ag[a].fifo_next = -1;
  return a;
}

/* _start_turn, engine.py:374-401 */
static void start_turn(Sim* s, Inst* in, int32_t a, double issue) {
  Agent* g = &s->ag[a];
  int idx = g->steps;
  in->running += 1;
  conditions_changed(s, in);
  double dur = service_time(s, g->turn0 + idx, in->level, in->running, in->thrashing);
  g->turn_idx = idx;
  g->issue_t = issue;
  g->anchor = s->now;
  g->rem = 1.0;
  g->done = s->now + dur;
  g->version = s->versions++;
  run_append(s, in, a);
  g->phase = ASB_PHASE_RUNNING;
  push(s, g->done, EV_COMPLETE, a, g->version, 0.0);
  update_power(s, in);
}

static void alive_add(Sim* s, int32_t a) {
  s->ag[a].alive_pos = s->n_alive;
  s->alive[s->n_alive++] = a;
}

static void alive_remove(Sim* s, int32_t a) {
  int32_t p = s->ag[a].alive_pos;
  int32_t last = s->alive[--s->n_alive];
  s->alive[p] = last;
  s->ag[last].alive_pos = p;
  s->ag[a].alive_pos = -1;
}

/* select_frequency_level, controller.py:81-86 */
static int select_level(int64_t usage, int64_t capacity, int L, double alpha) {
  double ac = alpha * (double)capacity;
  if ((double)usage >= ac) return L;
  return (int)floor((double)usage / ac * (double)(L - 1)) + 1;
}

/* _on_epoch + control_epoch, engine.py:436-488, controller.py:133-186 */
static void on_epoch(Sim* s, int64_t k) {
  const AsbScenario* sc = s->sc;
  int M = s->M, L = sc->n_levels;
  for (int i = 1; i <= M; i++) {
    s->has_tp[i] = 0;
    s->cnt[i] = 0;
  }
  /* min_throughput over ongoing ∪ pending of every instance (the agent-ticks) */
  for (int32_t j = 0; j < s->n_alive; j++) {
    const Agent* g = &s->ag[s->alive[j]];
    int i = g->inst;
    s->cnt[i]++;
    if (g->llm_t > 0.0) {
      double tp = (double)g->dec_tot / g->llm_t;
      if (!s->has_tp[i] || tp < s->min_tp[i]) {
        s->min_tp[i] = tp;
        s->has_tp[i] = 1;
      }
    }
  }
  for (int i = 1; i <= M; i++) {
    Inst* in = &s->in[i];
    s->ctr[ASB_CTR_TICKS] += s->cnt[i];
    int64_t usage = in->usage;
    int level;
    if (sc->variant == ASB_VARIANT_OFF)
      level = L;
    else if (sc->variant == ASB_VARIANT_FIXED)
      level = sc->fixed_level;
    else
      level = select_level(usage, sc->capacity, L, sc->alpha);
    int boosted = 0;
    if (sc->variant == ASB_VARIANT_CONTEXT_AWARE && sc->boost_enabled && s->has_tp[i] &&
        s->min_tp[i] < sc->slo_target) {
      level = L;
      boosted = 1;
    }
    in->level = level;
    conditions_changed(s, in);
    update_power(s, in);
    double gamma, beta;
    if (sc->variant == ASB_VARIANT_CONTEXT_AWARE && sc->thrash_avoidance) {
      gamma = sc->gamma;
      beta = sc->beta;
    } else {
      gamma = 1.0;
      beta = 1.0;
    }
    int n_adm = 0;
    double gcap = gamma * (double)sc->capacity;
    while (in->fifo_len > 0 && (double)in->usage < gcap) {
      int32_t a = fifo_pop(in, s);
      in->usage += s->ag[a].ctx;
      s->ag[a].inst = i;
      refresh_thrashing(s, in);
      s->admitted[n_adm++] = a;
    }
    int deferred = (double)in->usage > beta * (double)sc->capacity;
    sync_thrash(s, in);
    conditions_changed(s, in);
    for (int j = 0; j < n_adm; j++) {
      int32_t a = s->admitted[j];
      Agent* g = &s->ag[a];
      double issue = g->has_pending_issue ? g->pending_issue : s->now;
      g->has_pending_issue = 0;
      if (s->now < g->not_before) {
        g->phase = ASB_PHASE_WAITING_START;
        push(s, g->not_before, EV_ISSUE, a, 0, issue);
      } else {
        start_turn(s, in, a, issue);
      }
    }
    update_power(s, in);
    if (s->dec) {
      AsbDecision* d = &s->dec[k * M + (i - 1)];
      d->time = s->now;
      d->min_throughput = s->has_tp[i] ? s->min_tp[i] : NAN;
      d->usage_observed = usage;
      d->instance_id = i;
      d->frequency_level = level;
      d->admitted_count = n_adm;
      d->pending_depth = in->fifo_len;
      d->boosted = boosted;
      d->deferred = deferred;
    }
    mark_row(s, i, 0);
  }
}

/* argmin over (usage, id), router.py:91, 123, 150 */
static int argmin_usage(const Sim* s) {
  int best = 1;
  for (int i = 2; i <= s->M; i++)
    if (s->in[i].usage < s->in[best].usage) best = i;
  return best;
}

/* _on_arrival, engine.py:490-507 with router.py:75-94, 131-151 */
static void on_arrival(Sim* s, int32_t a) {
  const AsbScenario* sc = s->sc;
  Agent* g = &s->ag[a];
  s->ctr[ASB_CTR_ARRIVED]++;
  s->rank[a] = s->arrival_rank++;
  int target;
  if (sc->policy == ASB_POLICY_ROUND_ROBIN) {
    target = (s->rr_next % s->M) + 1;
    s->rr_next++;
  } else if (sc->policy == ASB_POLICY_LEAST_LOADED) {
    target = argmin_usage(s);
  } else {
    double threshold = sc->consolidation_threshold * (double)sc->capacity;
    target = 0;
    for (int i = 1; i <= s->M; i++)
      if ((double)s->in[i].usage < threshold) {
        target = i;
        break;
      }
    if (!target) target = argmin_usage(s);
  }
  g->inst = target;
  g->s_a = 0;
  fifo_append(&s->in[target], s, a);
  g->phase = ASB_PHASE_PENDING;
  alive_add(s, a);
  mark_row(s, target, 0);
}

/* _on_complete, engine.py:509-535 */
static void on_complete(Sim* s, int32_t a, int64_t version) {
  Agent* g = &s->ag[a];
  if (!g->running || g->version != version) return; /* superseded by a re-timing */
  s->ctr[ASB_CTR_EVENTS]++;
  Inst* in = &s->in[g->inst];
  run_remove(s, in, a);
  in->running -= 1;
  double llm = s->now - g->issue_t;
  int64_t turn = g->turn0 + g->turn_idx;
  int64_t delta = (int64_t)s->tp->prefill[turn] + (int64_t)s->tp->decode[turn];
  /* grow_context, instance.py:233-241 */
  g->ctx += delta;
  g->steps += 1;
  g->dec_tot += s->tp->decode[turn];
  g->llm_t += llm;
  if (g->ctx > g->max_ctx) g->max_ctx = g->ctx;
  in->usage += delta;
  s->ctr[ASB_CTR_TURNS]++;
  if (s->turn_issue) {
    s->turn_issue[g->turn0 - s->tp->trace_turn_off[s->sc->trace_id] + g->turn_idx] = g->issue_t;
    s->turn_done[g->turn0 - s->tp->trace_turn_off[s->sc->trace_id] + g->turn_idx] = s->now;
  }
  if (g->steps == g->n_turns) {
    in->usage -= g->ctx; /* complete_agent, instance.py:223-230 */
    g->phase = ASB_PHASE_DONE;
    g->completion_time = s->now;
    s->ctr[ASB_CTR_COMPLETED]++;
    alive_remove(s, a);
  } else {
    g->phase = ASB_PHASE_TOOL;
    push(s, s->now + s->tp->tool[turn], EV_TOOL, a, 0, 0.0);
  }
  refresh_thrashing(s, in);
  sync_thrash(s, in);
  conditions_changed(s, in);
  update_power(s, in);
  mark_row(s, g->inst, 0);
}

/* _on_tool, engine.py:537-561 with maybe_reassign router.py:97-128 */
static void on_tool(Sim* s, int32_t a) {
  const AsbScenario* sc = s->sc;
  Agent* g = &s->ag[a];
  s->ctr[ASB_CTR_EVENTS]++;
  int source = g->inst;
  int target = 0;
  if (sc->policy == ASB_POLICY_CONTEXT_AWARE) {
    g->s_a += 1;
    if (g->s_a >= sc->reassign_interval) {
      int best = 0;
      for (int i = 1; i <= s->M; i++) {
        if (!sc->include_idle && !(s->in[i].usage > 0 || i == source)) continue;
        if (!best || s->in[i].usage < s->in[best].usage) best = i;
      }
      if (best && best != source &&
          (double)s->in[source].usage >= sc->imbalance_ratio * (double)s->in[best].usage)
        target = best;
      if (target)
        g->s_a = 0;
      else if (!sc->reset_only_on_reassign)
        g->s_a = 0;
    }
  }
  Inst* src = &s->in[source];
  if (!target) {
    start_turn(s, src, a, s->now);
    mark_row(s, source, 0);
    return;
  }
  Inst* dst = &s->in[target];
  g->migrations += 1;
  s->ctr[ASB_CTR_MIGRATIONS]++;
  /* migrate_context, router.py:154-176 (agent is ongoing on the source) */
  src->usage -= g->ctx;
  refresh_thrashing(s, src);
  fifo_append(dst, s, a);
  g->inst = target;
  g->phase = ASB_PHASE_PENDING;
  g->pending_issue = s->now;
  g->has_pending_issue = 1;
  g->not_before = s->now + sc->migration_delay;
  sync_thrash(s, src);
  conditions_changed(s, src);
  update_power(s, src);
  mark_row(s, source, 0);
  mark_row(s, target, 0);
}

static void on_issue(Sim* s, int32_t a, double issue) {
  s->ctr[ASB_CTR_EVENTS]++;
  start_turn(s, &s->in[s->ag[a].inst], a, issue);
  mark_row(s, s->ag[a].inst, 0);
}

static int run_one(const AsbScenario* sc, const AsbTracePool* tp, const AsbTablePool* tb,
                   const AsbOutputs* out, int32_t sidx) {
  Sim S;
  memset(&S, 0, sizeof(S));
  Sim* s = &S;
  s->sc = sc;
  s->tp = tp;
  s->tb = tb;
  s->out = out;
  s->tbl0 = tb->table_off[sc->table_id];
  s->a0 = tp->trace_agent_off[sc->trace_id];
  s->A = (int32_t)(tp->trace_agent_off[sc->trace_id + 1] - s->a0);
  s->M = sc->n_instances;
  int A = s->A, M = s->M, L = sc->n_levels;
  s->ag = (Agent*)calloc((size_t)(A > 0 ? A : 1), sizeof(Agent));
  s->in = (Inst*)calloc((size_t)M + 1, sizeof(Inst));
  s->alive = (int32_t*)malloc(sizeof(int32_t) * (size_t)(A > 0 ? A : 1));
  s->min_tp = (double*)malloc(sizeof(double) * (size_t)(M + 1));
  s->has_tp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(M + 1));
  s->cnt = (int64_t*)malloc(sizeof(int64_t) * (size_t)(M + 1));
  s->admitted = (int32_t*)malloc(sizeof(int32_t) * (size_t)(A > 0 ? A : 1));
  s->rank = (int32_t*)malloc(sizeof(int32_t) * (size_t)(A > 0 ? A : 1));
  s->oa0 = out->agent_off[sidx];
  s->oi0 = out->inst_off[sidx];
  s->dec = out->decisions ? out->decisions + out->dec_off[sidx] : NULL;
  if (out->turn_issue) {
    s->turn_issue = out->turn_issue + out->turn_off[sidx];
    s->turn_done = out->turn_done + out->turn_off[sidx];
    int64_t nt = tp->trace_turn_off[sc->trace_id + 1] - tp->trace_turn_off[sc->trace_id];
    for (int64_t t = 0; t < nt; t++) s->turn_issue[t] = s->turn_done[t] = NAN;
  }
  if (out->timeseries && out->ts_off && out->ts_count) {
    s->ts = out->timeseries + out->ts_off[sidx];
    s->ts_cap = out->ts_off[sidx + 1] - out->ts_off[sidx];
  }
  for (int a = 0; a < A; a++) {
    Agent* g = &s->ag[a];
    g->turn0 = tp->agent_turn_off[s->a0 + a];
    g->n_turns = (int32_t)(tp->agent_turn_off[s->a0 + a + 1] - g->turn0);
    g->run_prev = g->run_next = g->fifo_next = g->alive_pos = -1;
    g->completion_time = NAN;
    g->phase = ASB_PHASE_ARRIVING;
    s->rank[a] = -1;
  }
  for (int i = 1; i <= M; i++) {
    Inst* in = &s->in[i];
    in->level = L;
    in->fifo_head = in->fifo_tail = -1;
    in->run_head = in->run_tail = -1;
    in->watts = lvl_idle(s, L);
  }
  /* _schedule_initial, engine.py:303-317 (samples only with rows, see header) */
  double T = sc->sim_duration, E = sc->epoch_length;
  for (int64_t k = 0; k < sc->n_epochs; k++) push(s, (double)k * E, EV_EPOCH, (int32_t)k, 0, 0.0);
  if (s->ts)
    for (int64_t k = 1; (double)k * sc->record_interval < T; k++)
      push(s, (double)k * sc->record_interval, EV_SAMPLE, 0, 0, 0.0);
  for (int a = 0; a < A; a++) {
    double arr = tp->arrival[s->a0 + a];
    if (arr < T) push(s, arr, EV_ARRIVAL, a, 0, 0.0);
  }
  /* run(), engine.py:576-579: a forced row per instance at t = 0 */
  for (int i = 1; i <= M; i++) mark_row(s, i, 1);
  /* hot loop, engine.py:589-594 */
  while (s->heap.n > 0 && s->status == 0) {
    Ev e = heap_pop(&s->heap);
    if (e.t > T) break;
    s->now = e.t;
    switch (e.prio) {
      case EV_EPOCH: on_epoch(s, e.agent); break;
      case EV_COMPLETE: on_complete(s, e.agent, e.version); break;
      case EV_TOOL: on_tool(s, e.agent); break;
      case EV_ISSUE: on_issue(s, e.agent, e.issue); break;
      case EV_ARRIVAL: on_arrival(s, e.agent); break;
      case EV_SAMPLE: /* _on_sample, engine.py:570-572 */
        for (int i = 1; i <= M; i++) mark_row(s, i, 1);
        break;
    }
  }
  /* final accounting, engine.py:595-603 */
  s->now = T;
  for (int i = 1; i <= M; i++) {
    Inst* in = &s->in[i];
    in->energy += in->watts * (T - in->t_pow);
    in->t_pow = T;
    if (in->thr_flag) {
      in->thr_time += T - in->thr_since;
      in->thr_since = T;
    }
    mark_row(s, i, 1);
  }
  if (s->ts) out->ts_count[sidx] = s->ts_n;
  /* outputs */
  for (int a = 0; a < A; a++) {
    const Agent* g = &s->ag[a];
    int64_t o = s->oa0 + a;
    out->completion_time[o] = g->completion_time;
    out->llm_time[o] = g->llm_t;
    out->decode_total[o] = g->dec_tot;
    out->max_context[o] = g->max_ctx;
    out->context[o] = g->ctx;
    out->turns_completed[o] = g->steps;
    out->final_instance[o] = g->inst;
    out->migrations[o] = g->migrations;
    out->phase[o] = g->phase;
    out->arrival_rank[o] = s->rank[a];
  }
  for (int i = 1; i <= M; i++) {
    const Inst* in = &s->in[i];
    int64_t o = s->oi0 + i - 1;
    out->energy[o] = in->energy;
    out->thrash_time[o] = in->thr_time;
    out->final_usage[o] = in->usage;
    out->final_pending[o] = in->fifo_len;
    out->final_level[o] = in->level;
  }
  s->ctr[ASB_CTR_STATUS] = s->status;
  for (int c = 0; c < ASB_NCOUNTERS; c++) out->counters[(int64_t)sidx * ASB_NCOUNTERS + c] = s->ctr[c];
  free(s->ag);
  free(s->in);
  free(s->alive);
  free(s->min_tp);
  free(s->has_tp);
  free(s->cnt);
  free(s->admitted);
  free(s->rank);
  free(s->heap.a);
  return s->status;
}

/* Run scenarios [first, first+count) with `threads` OpenMP threads (<=0: all). */
int oracle_run_scenarios(const AsbScenario* scen, int32_t n_scen, const AsbTracePool* traces,
                         const AsbTablePool* tables, const AsbOutputs* out, int32_t threads) {
  int err = 0;
#ifdef _OPENMP
  if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads) reduction(| : err)
#endif
  for (int32_t i = 0; i < n_scen; i++) err |= run_one(&scen[i], traces, tables, out, i);
  (void)threads;
  return err;
}

/* Python >= 3.12 builtin sum() over floats: int start 0, then Neumaier
 * compensated summation (Objects/bltinmodule.c); _build_result uses it for
 * total energy / thrash time (engine.py:632-633). */
static double py_sum(const double* x, int n) {
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

/* SystemMetrics of one scenario from the outputs (engine.py:632-655, metrics.py:49-69). */
static int cmp_double(const void* x, const void* y) {
  double a = *(const double*)x, b = *(const double*)y;
  return (a > b) - (a < b);
}

int oracle_scenario_stats(const AsbScenario* scen, int32_t n_scen, const AsbOutputs* out,
                          AsbStats* stats) {
  for (int32_t s = 0; s < n_scen; s++) {
    const AsbScenario* sc = &scen[s];
    int64_t a0 = out->agent_off[s], a1 = out->agent_off[s + 1];
    int64_t i0 = out->inst_off[s];
    double* tps = (double*)malloc(sizeof(double) * (size_t)(a1 - a0 + 1));
    int64_t n = 0, met = 0;
    for (int64_t a = a0; a < a1; a++) {
      if (out->phase[a] != ASB_PHASE_DONE || !(out->llm_time[a] > 0.0)) continue;
      double tp = (double)out->decode_total[a] / out->llm_time[a];
      tps[n++] = tp;
      if (tp >= sc->slo_target) met++;
    }
    AsbStats* st = &stats[s];
    st->slo_met = met;
    st->n_completed_with_tp = n;
    st->slo_attainment = n ? (double)met / (double)n : NAN;
    if (n) {
      qsort(tps, (size_t)n, sizeof(double), cmp_double);
      int64_t rank = (int64_t)ceil(0.05 * (double)n);
      st->p5_throughput = tps[rank - 1];
    } else {
      st->p5_throughput = NAN;
    }
    double e = py_sum(out->energy + i0, sc->n_instances);
    double th = py_sum(out->thrash_time + i0, sc->n_instances);
    double T = sc->sim_duration;
    st->job_throughput = (double)out->counters[(int64_t)s * ASB_NCOUNTERS + ASB_CTR_COMPLETED] / T;
    st->average_power = e / T;
    st->energy = e;
    st->thrash_fraction = th / (T * (double)sc->n_instances);
    free(tps);
  }
  return 0;
}
