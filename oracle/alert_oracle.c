/*
 * alert_oracle.c — FP64 CPU restatement of the alertsim hot path.
 * TEST INFRASTRUCTURE (checker + timed CPU baseline), never a product path.
 *
 * Every function cites the reference function it restates (paths relative to
 * /root/reference/pkg/src/alertsim/).  Arithmetic is written in the
 * reference's left-to-right order; build with -ffp-contract=off and
 * -fno-builtin so erf/pow are the glibc calls CPython makes.
 */
#include "alert_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------- */
/* small helpers mirroring Python builtins                                  */

static double py_max(double a, double b) { return (b > a) ? b : a; } /* max(a, b) */
static double py_min(double a, double b) { return (b < a) ? b : a; } /* min(a, b) */

/* float ** y goes through libm pow() in CPython (floatobject.c float_pow);
 * the volatile pointer keeps the compiler from rewriting pow(x, 2.0) as x*x. */
static double (*volatile libm_pow)(double, double) = pow;
static double (*volatile libm_erf)(double) = erf;

typedef struct Space {
  const AlertSpaceDesc* d;
  int32_t* stage_off; /* [n_dnns] first stage row of each dnn */
  int n_cand;
} Space;

static int space_open(const AlertSpaceDesc* d, Space* s) {
  s->d = d;
  s->stage_off = (int32_t*)malloc(sizeof(int32_t) * (size_t)(d->n_dnns > 0 ? d->n_dnns : 1));
  if (!s->stage_off) return -1;
  int off = 0, n = 0;
  for (int i = 0; i < d->n_dnns; ++i) {
    s->stage_off[i] = off;
    off += d->dnn_n_stages[i];
    n += d->n_powers * (d->dnn_kind[i] == ALERT_KIND_TRADITIONAL ? 1 : d->dnn_n_stages[i]);
  }
  s->n_cand = n;
  return 0;
}
static void space_close(Space* s) { free(s->stage_off); }

static double t_prof_of(const Space* s, int dnn, int stage0, int power) {
  return s->d->stage_t_prof[(size_t)(s->stage_off[dnn] + stage0) * s->d->n_powers + power];
}
static double acc_of(const Space* s, int dnn, int stage0) {
  return s->d->stage_accuracy[s->stage_off[dnn] + stage0];
}

int oracle_num_candidates(const AlertSpaceDesc* sp) {
  Space s;
  if (space_open(sp, &s)) return -1;
  int n = s.n_cand;
  space_close(&s);
  return n;
}

/* policies.py:59-67 _configs enumeration order */
int oracle_candidate(const AlertSpaceDesc* d, int c, int32_t* dnn, int32_t* power, int32_t* stage) {
  int k = 0;
  for (int i = 0; i < d->n_dnns; ++i)
    for (int j = 0; j < d->n_powers; ++j) {
      int nt = d->dnn_kind[i] == ALERT_KIND_TRADITIONAL ? 1 : d->dnn_n_stages[i];
      if (c < k + nt) {
        *dnn = i;
        *power = j;
        *stage = d->dnn_kind[i] == ALERT_KIND_TRADITIONAL ? 0 : (c - k) + 1;
        return 0;
      }
      k += nt;
    }
  return -1;
}

/* ---------------------------------------------------------------------- */
/* predictor.py                                                             */

static const double SQRT2 = 1.4142135623730951; /* math.sqrt(2.0), predictor.py:21 */

/* predictor.py:25-27 */
double oracle_normal_cdf(double x) { return 0.5 * (1.0 + libm_erf(x / SQRT2)); }

static double est_sigma(const OracleEst* e) { return libm_pow(e->sigma2, 0.5); } /* estimator.py:42-44 */

/* predictor.py:56-65 (via latency_distribution :48-53) */
double oracle_deadline_probability(const OracleEst* est, double t_prof, double t_goal) {
  double mean = est->mu * t_prof;
  double sigma = est_sigma(est) * t_prof;
  if (sigma == 0.0) return mean <= t_goal ? 1.0 : 0.0;
  return oracle_normal_cdf((t_goal - mean) / sigma);
}

/* predictor.py:68-70 */
static double accuracy_blend(double pr, double q_on_time, double q_fail) {
  return pr * q_on_time + (1.0 - pr) * q_fail;
}

static double anytime_acc(const Space* s, const OracleEst* est, int dnn, int power, int target,
                          double t_goal) {
  /* predictor.py:100-108: prs for stages 1..target, prs[target] = 0, telescoping sum */
  double prs[ALERT_MAX_STAGES + 1];
  for (int k = 0; k < target; ++k)
    prs[k] = oracle_deadline_probability(est, t_prof_of(s, dnn, k, power), t_goal);
  prs[target] = 0.0;
  double acc = (1.0 - prs[0]) * s->d->dnn_q_fail[dnn];
  for (int k = 0; k < target; ++k) acc += acc_of(s, dnn, k) * (prs[k] - prs[k + 1]);
  return acc;
}

double oracle_expected_accuracy_anytime(const AlertSpaceDesc* sp, const OracleEst* est, int dnn,
                                        int power, int target, double t_goal) {
  Space s;
  if (space_open(sp, &s)) return NAN;
  double a = anytime_acc(&s, est, dnn, power, target, t_goal);
  space_close(&s);
  return a;
}

/* predictor.py:111-126 */
double oracle_energy_mean(const OracleEst* est, const OracleIdle* idle, double p, double t_prof,
                          double goal) {
  double lat = est->mu * t_prof;
  return p * lat + idle->phi * p * py_max(0.0, goal - lat);
}

/* predictor.py:129-144 (z_q = normal_quantile(pr_th), computed by the caller) */
double oracle_energy_percentile(const OracleEst* est, const OracleIdle* idle, double p, double t_prof,
                                double goal, double z_q) {
  double lat = (est->mu + z_q * est_sigma(est)) * t_prof;
  double idl = py_max(0.0, goal - py_min(lat, goal));
  return p * lat + idle->phi * p * idl;
}

static int predict_all_s(const Space* s, const OracleEst* est, const OracleIdle* idle,
                         const AlertSpec* spec, double goal, AlertPrediction* out) {
  const AlertSpaceDesc* d = s->d;
  int n = 0;
  for (int i = 0; i < d->n_dnns; ++i) {
    int trad = d->dnn_kind[i] == ALERT_KIND_TRADITIONAL;
    int nt = trad ? 1 : d->dnn_n_stages[i];
    for (int j = 0; j < d->n_powers; ++j) {
      double pw = d->power_cap[j];
      for (int tk = 0; tk < nt; ++tk) {
        int target = trad ? 0 : tk + 1;
        int st = trad ? 0 : target - 1;
        double t = t_prof_of(s, i, st, j);
        AlertPrediction* p = &out[n++];
        p->latency_mean = est->mu * t;
        p->latency_sigma = est_sigma(est) * t;
        p->pr_deadline = oracle_deadline_probability(est, t, goal);
        p->expected_accuracy = trad ? accuracy_blend(p->pr_deadline, acc_of(s, i, 0), d->dnn_q_fail[i])
                                    : anytime_acc(s, est, i, j, target, goal);
        p->energy = spec->has_pr ? oracle_energy_percentile(est, idle, pw, t, goal, spec->z_q)
                                 : oracle_energy_mean(est, idle, pw, t, goal);
        p->dnn_index = i;
        p->power_index = j;
        p->target_stage = target;
        p->_pad = 0;
      }
    }
  }
  return n;
}

/* predictor.py:147-197 */
int oracle_predict_all(const AlertSpaceDesc* sp, const OracleEst* est, const OracleIdle* idle,
                       const AlertSpec* spec, double goal, AlertPrediction* out) {
  Space s;
  if (space_open(sp, &s)) return -1;
  int n = predict_all_s(&s, est, idle, spec, goal, out);
  space_close(&s);
  return n;
}

/* ---------------------------------------------------------------------- */
/* selector.py                                                              */

/* selector.py:73-84 */
static int feasible(const AlertPrediction* p, const AlertSpec* spec, int use_e, int use_a, int use_pr) {
  if (use_pr && spec->has_pr && p->pr_deadline < spec->pr_threshold) return 0;
  if (spec->mode == ALERT_MODE_MAX_ACCURACY) return !use_e || p->energy <= spec->e_goal;
  return !use_a || p->expected_accuracy >= spec->q_goal;
}

/* selector.py:87-91 rank key as a lexicographic comparison: a < b ? */
static int rank_less(const AlertPrediction* a, const AlertPrediction* b, int mode) {
  double a0, a1, b0, b1;
  if (mode == ALERT_MODE_MAX_ACCURACY) {
    a0 = -a->expected_accuracy; a1 = a->energy; b0 = -b->expected_accuracy; b1 = b->energy;
  } else {
    a0 = a->energy; a1 = -a->expected_accuracy; b0 = b->energy; b1 = -b->expected_accuracy;
  }
  if (a0 != b0) return a0 < b0;
  if (a1 != b1) return a1 < b1;
  if (a->power_index != b->power_index) return a->power_index < b->power_index;
  if (a->dnn_index != b->dnn_index) return a->dnn_index < b->dnn_index;
  return a->target_stage < b->target_stage;
}

static const int LEVELS[3][3] = {{1, 1, 1}, {0, 1, 1}, {0, 0, 0}}; /* selector.py:94-99 */

static int kind_ok(const Space* s, const AlertPrediction* p, int kinds_mask) {
  return (kinds_mask >> s->d->dnn_kind[p->dnn_index]) & 1;
}

static double rel_dist(double a, double b) {
  double den = fabs(b) > 1e-300 ? fabs(b) : 1e-300;
  return fabs(a - b) / den;
}

static int select_s(const Space* s, const AlertPrediction* preds, int n, const AlertSpec* spec,
                    int kinds_mask, int32_t* level, double* gap, double* boundary) {
  /* selector.py:102-131 */
  if (boundary) {
    double b = INFINITY;
    for (int c = 0; c < n; ++c) {
      if (!kind_ok(s, &preds[c], kinds_mask)) continue;
      if (spec->mode == ALERT_MODE_MAX_ACCURACY)
        b = py_min(b, rel_dist(preds[c].energy, spec->e_goal));
      else
        b = py_min(b, rel_dist(preds[c].expected_accuracy, spec->q_goal));
      if (spec->has_pr) b = py_min(b, rel_dist(preds[c].pr_deadline, spec->pr_threshold));
    }
    *boundary = b;
  }
  for (int L = 0; L < 3; ++L) {
    int mode = L == ALERT_LEVEL_DROPPED_ACCURACY ? ALERT_MODE_MAX_ACCURACY : spec->mode;
    int best = -1, second = -1;
    for (int c = 0; c < n; ++c) {
      if (!kind_ok(s, &preds[c], kinds_mask)) continue;
      if (!feasible(&preds[c], spec, LEVELS[L][0], LEVELS[L][1], LEVELS[L][2])) continue;
      if (best < 0 || rank_less(&preds[c], &preds[best], mode)) {
        second = best;
        best = c;
      } else if (second < 0 || rank_less(&preds[c], &preds[second], mode)) {
        second = c;
      }
    }
    if (best >= 0) {
      *level = L;
      if (gap) {
        if (second < 0) {
          *gap = INFINITY;
        } else if (mode == ALERT_MODE_MAX_ACCURACY) {
          *gap = rel_dist(preds[second].expected_accuracy, preds[best].expected_accuracy);
        } else {
          *gap = rel_dist(preds[second].energy, preds[best].energy);
        }
      }
      return best;
    }
  }
  return -1;
}

int oracle_select(const AlertSpaceDesc* sp, const AlertPrediction* preds, int n, const AlertSpec* spec,
                  int kinds_mask, int32_t* level, double* gap, double* boundary) {
  Space s;
  if (space_open(sp, &s)) return -1;
  int r = select_s(&s, preds, n, spec, kinds_mask, level, gap, boundary);
  space_close(&s);
  return r;
}

/* selector.py:134-182 — pairwise "better" written out independently */
int oracle_brute_force_select(const AlertSpaceDesc* sp, const AlertPrediction* preds, int n,
                              const AlertSpec* spec, int kinds_mask, int32_t* level) {
  Space s;
  if (space_open(sp, &s)) return -1;
  int result = -1;
  for (int L = 0; L < 3 && result < 0; ++L) {
    int mode = L == 2 ? ALERT_MODE_MAX_ACCURACY : spec->mode;
    int best = -1;
    for (int c = 0; c < n; ++c) {
      const AlertPrediction* a = &preds[c];
      if (!kind_ok(&s, a, kinds_mask)) continue;
      if (!feasible(a, spec, LEVELS[L][0], LEVELS[L][1], LEVELS[L][2])) continue;
      if (best < 0) { best = c; continue; }
      const AlertPrediction* b = &preds[best];
      int better;
      if (mode == ALERT_MODE_MAX_ACCURACY && a->expected_accuracy != b->expected_accuracy)
        better = a->expected_accuracy > b->expected_accuracy;
      else if (mode == ALERT_MODE_MAX_ACCURACY && a->energy != b->energy)
        better = a->energy < b->energy;
      else if (mode != ALERT_MODE_MAX_ACCURACY && a->energy != b->energy)
        better = a->energy < b->energy;
      else if (mode != ALERT_MODE_MAX_ACCURACY && a->expected_accuracy != b->expected_accuracy)
        better = a->expected_accuracy > b->expected_accuracy;
      else if (a->power_index != b->power_index)
        better = a->power_index < b->power_index;
      else if (a->dnn_index != b->dnn_index)
        better = a->dnn_index < b->dnn_index;
      else
        better = a->target_stage < b->target_stage;
      if (better) best = c;
    }
    if (best >= 0) { result = best; *level = L; }
  }
  space_close(&s);
  return result;
}

/* selector.py:48-70 with floor_min = 0.001 */
double oracle_adjust_goal(const AlertSpec* spec, int has_group, double budget, int32_t count) {
  double goal;
  if (!has_group) {
    goal = spec->t_goal - spec->overhead_budget;
  } else {
    double share = budget / (double)count;
    goal = share - spec->overhead_budget;
  }
  return py_max(goal, 0.001);
}

/* ---------------------------------------------------------------------- */
/* estimator.py                                                             */

/* estimator.py:47-56 */
void oracle_slowdown_init(const AlertFilterConfig* cfg, OracleEst* e) {
  e->mu = cfg->mu0;
  e->sigma2 = cfg->sigma2_0;
  e->k_gain = cfg->k0;
  e->q_noise = cfg->q0;
  e->innov = 0.0;
}

/* estimator.py:59-84 */
int oracle_slowdown_update(const AlertFilterConfig* cfg, OracleEst* e, double obs, double t_prof) {
  if (obs <= 0 || t_prof <= 0) return -1;
  double q = py_max(cfg->q0, cfg->alpha * e->q_noise +
                                 (1.0 - cfg->alpha) * libm_pow(e->k_gain * e->innov, 2.0));
  double prior = (1.0 - e->k_gain) * e->sigma2 + q;
  double k = prior / (prior + cfg->r);
  double y = obs / t_prof - e->mu;
  double mu = e->mu + k * y;
  double sigma2 = cfg->sigma2_uses_current_gain ? (1.0 - k) * e->sigma2 + q
                                                : (1.0 - e->k_gain) * e->sigma2 + q;
  e->mu = mu;
  e->sigma2 = sigma2;
  e->k_gain = k;
  e->q_noise = q;
  e->innov = y;
  return 0;
}

/* estimator.py:110-127 */
int oracle_idle_update(const AlertFilterConfig* cfg, OracleIdle* st, double measured, double cap) {
  if (measured <= 0 || cap <= 0) return -1;
  double ratio = py_min(1.0, measured / cap);
  double w = (st->m_var + cfg->s) / (st->m_var + cfg->s + cfg->v);
  double m = (1.0 - w) * (st->m_var + cfg->s);
  st->phi = st->phi + w * (ratio - st->phi);
  st->m_var = m;
  return 0;
}

/* ---------------------------------------------------------------------- */
/* simulator.py                                                             */

typedef struct Exec { double latency, fb_latency, fb_t_prof; int completed; } Exec;

/* simulator.py:249-280 */
static Exec execute_decision(const Space* s, double sd, int dnn, int power, int target, double goal) {
  Exec o;
  if (s->d->dnn_kind[dnn] == ALERT_KIND_TRADITIONAL) {
    double t = t_prof_of(s, dnn, 0, power);
    double lat = sd * t;
    o.latency = lat;
    o.completed = lat <= goal ? 1 : 0;
    o.fb_latency = lat;
    o.fb_t_prof = t;
    return o;
  }
  int tg = target ? target : s->d->dnn_n_stages[dnn];
  double stop = py_min(sd * t_prof_of(s, dnn, tg - 1, power), goal);
  int completed = 0;
  for (int k = 0; k < tg; ++k)
    if (sd * t_prof_of(s, dnn, k, power) <= stop) completed = k + 1;
  o.latency = stop;
  o.completed = completed;
  if (completed) {
    double t = t_prof_of(s, dnn, completed - 1, power);
    o.fb_latency = sd * t;
    o.fb_t_prof = t;
  } else {
    o.fb_latency = stop;
    o.fb_t_prof = t_prof_of(s, dnn, 0, power);
  }
  return o;
}

typedef struct Meas { double latency, delivered, energy; int met, vl, va, ve; } Meas;

/* simulator.py:329-382 (overhead = spec.overhead_budget) */
static Meas measure(const Space* s, const AlertSpec* spec, int dnn, int power, const Exec* o,
                    double idle_true, double period) {
  Meas m;
  double cap = s->d->power_cap[power];
  m.latency = o->latency + spec->overhead_budget;
  m.delivered = o->completed >= 1 ? acc_of(s, dnn, o->completed - 1) : s->d->dnn_q_fail[dnn];
  m.met = o->completed >= 1 && m.latency <= period;
  m.energy = cap * py_min(m.latency, period) + idle_true * py_max(0.0, period - m.latency);
  m.vl = !m.met;
  m.va = spec->mode == ALERT_MODE_MIN_ENERGY && m.delivered < spec->q_goal;
  m.ve = spec->mode == ALERT_MODE_MAX_ACCURACY && m.energy > spec->e_goal;
  return m;
}

/* policies.py:111-126 _exact_eval */
typedef struct Exact { double delivered, energy, latency; int met; } Exact;
static Exact exact_eval(const Space* s, const AlertSpec* spec, double sd, double idle_true, int i,
                        int j, int target, double goal) {
  Exec o = execute_decision(s, sd, i, j, target, goal);
  Exact x;
  x.latency = o.latency + spec->overhead_budget;
  double period = goal + spec->overhead_budget;
  x.delivered = o.completed >= 1 ? acc_of(s, i, o.completed - 1) : s->d->dnn_q_fail[i];
  x.met = o.completed >= 1 && x.latency <= period;
  double cap = s->d->power_cap[j];
  x.energy = cap * py_min(x.latency, period) + idle_true * py_max(0.0, period - x.latency);
  return x;
}

/* policies.py:142-146 _rank: a < b ? */
static int orank_less(int mode, const Exact* a, int ja, int ia, int ta, const Exact* b, int jb, int ib,
                      int tb) {
  double a0, a1, b0, b1;
  if (mode == ALERT_MODE_MAX_ACCURACY) {
    a0 = -a->delivered; a1 = a->energy; b0 = -b->delivered; b1 = b->energy;
  } else {
    a0 = a->energy; a1 = -a->delivered; b0 = b->energy; b1 = -b->delivered;
  }
  if (a0 != b0) return a0 < b0;
  if (a1 != b1) return a1 < b1;
  if (ja != jb) return ja < jb;
  if (ia != ib) return ia < ib;
  return ta < tb;
}

static int oracle_decide_s(const Space* s, const AlertSpec* spec, double sd, double idle_true,
                           double goal, int32_t* level, double* gap) {
  /* policies.py:160-205 */
  const AlertSpaceDesc* d = s->d;
  for (int L = 0; L < 3; ++L) {
    int use_energy = L == 0, use_acc = L < 2;
    int mode = L == 2 ? ALERT_MODE_MAX_ACCURACY : spec->mode;
    int best = -1, second = -1, c = 0;
    Exact bx = {0}, sx = {0};
    int bi = 0, bj = 0, bt = 0, si = 0, sj = 0, st = 0;
    for (int i = 0; i < d->n_dnns; ++i) {
      int trad = d->dnn_kind[i] == ALERT_KIND_TRADITIONAL;
      int nt = trad ? 1 : d->dnn_n_stages[i];
      for (int j = 0; j < d->n_powers; ++j)
        for (int tk = 0; tk < nt; ++tk, ++c) {
          int target = trad ? 0 : tk + 1;
          Exact x = exact_eval(s, spec, sd, idle_true, i, j, target, goal);
          if (L != 2 && !x.met) continue;
          if (spec->mode == ALERT_MODE_MAX_ACCURACY) {
            if (use_energy && x.energy > spec->e_goal) continue;
          } else if (use_acc && x.delivered < spec->q_goal) {
            continue;
          }
          if (best < 0 || orank_less(mode, &x, j, i, target, &bx, bj, bi, bt)) {
            second = best; sx = bx; si = bi; sj = bj; st = bt;
            best = c; bx = x; bi = i; bj = j; bt = target;
          } else if (second < 0 || orank_less(mode, &x, j, i, target, &sx, sj, si, st)) {
            second = c; sx = x; si = i; sj = j; st = target;
          }
        }
    }
    if (best >= 0) {
      *level = L;
      if (gap) {
        if (second < 0) *gap = INFINITY;
        else if (mode == ALERT_MODE_MAX_ACCURACY) *gap = rel_dist(sx.delivered, bx.delivered);
        else *gap = rel_dist(sx.energy, bx.energy);
      }
      return best;
    }
  }
  return -1;
}

int oracle_oracle_decide(const AlertSpaceDesc* sp, const AlertSpec* spec, double sd, double idle,
                         double goal, int32_t* level, double* gap) {
  Space s;
  if (space_open(sp, &s)) return -1;
  int r = oracle_decide_s(&s, spec, sd, idle, goal, level, gap);
  space_close(&s);
  return r;
}

/* CPython 3.12 sum() over floats: Neumaier compensated summation
 * (Python/bltinmodule.c builtin_sum_impl); the result is s + c when c is
 * nonzero and finite.  The reference's means (simulator.py:428-458) are sums
 * of this kind divided by the count. */
static void neumaier(double* s, double* c, double x) {
  double t = *s + x;
  if (fabs(*s) >= fabs(x))
    *c += (*s - t) + x;
  else
    *c += (x - t) + *s;
  *s = t;
}

/* index of (dnn i, power j, target) in the candidate enumeration
 * (policies.py:59-67 _configs order) */
static int cand_index(const Space* s, int i, int j, int target) {
  const AlertSpaceDesc* d = s->d;
  int c = 0;
  for (int k = 0; k < i; ++k)
    c += d->n_powers * (d->dnn_kind[k] == ALERT_KIND_TRADITIONAL ? 1 : d->dnn_n_stages[k]);
  if (d->dnn_kind[i] == ALERT_KIND_TRADITIONAL) return c + j;
  return c + j * d->dnn_n_stages[i] + (target - 1);
}

/* OracleStaticPolicy.begin (policies.py:221-265): best fixed candidate over
 * the realized trace; tot_energy / tot_acc are plain running sums. */
/* returns cand | eligible << 16 (AlertState.policy_aux layout) */
static int oracle_static_choice(const Space* s, const AlertSpec* spec, int64_t n, const double* sd,
                                const double* idle) {
  const AlertSpaceDesc* d = s->d;
  double t_goal = spec->t_goal - spec->overhead_budget;
  int best = -1, bel = 0, bi = 0, bj = 0, bt = 0;
  double bo = 0.0, bv = 0.0;
  int c = 0;
  for (int i = 0; i < d->n_dnns; ++i) {
    int trad = d->dnn_kind[i] == ALERT_KIND_TRADITIONAL;
    int nt = trad ? 1 : d->dnn_n_stages[i];
    for (int j = 0; j < d->n_powers; ++j)
      for (int tk = 0; tk < nt; ++tk, ++c) {
        int target = trad ? 0 : tk + 1;
        int64_t lv = 0, av = 0, ev = 0;
        double te = 0.0, ta = 0.0;
        for (int64_t k = 0; k < n; ++k) {
          Exact x = exact_eval(s, spec, sd[k], idle[k], i, j, target, t_goal);
          lv += !x.met;
          if (spec->mode == ALERT_MODE_MIN_ENERGY) av += x.delivered < spec->q_goal;
          else ev += x.energy > spec->e_goal;
          te += x.energy;
          ta += x.delivered;
        }
        double mean_obj = spec->mode == ALERT_MODE_MIN_ENERGY ? te / (double)n : -ta / (double)n;
        int64_t mx = lv > av ? lv : av;
        if (ev > mx) mx = ev;
        int eligible = (double)mx <= 0.10 * (double)n;
        double tv = (double)(lv + av + ev);
        /* key = (0, mean_obj, total_viol, j, i, t) if eligible else (1, total_viol, mean_obj, j, i, t) */
        double k1 = eligible ? mean_obj : tv, k2 = eligible ? tv : mean_obj;
        int less;
        if (best < 0) less = 1;
        else if (!eligible != !bel) less = eligible;
        else if (k1 != bo) less = k1 < bo;
        else if (k2 != bv) less = k2 < bv;
        else if (j != bj) less = j < bj;
        else if (i != bi) less = i < bi;
        else less = target < bt;
        if (less) {
          best = c; bel = eligible; bo = k1; bv = k2; bi = i; bj = j; bt = target;
        }
      }
  }
  return best < 0 ? best : best | (bel << 16);
}

/* SysOnlyPolicy.decide (policies.py:298-313): cheapest cap predicted on time
 * (*found = some cap is, policies.py:305-310) */
static int sys_only_power(const Space* s, const OracleEst* est, const OracleIdle* idl, int dnn, int stage0,
                          double goal, int* found) {
  const AlertSpaceDesc* d = s->d;
  int bj = -1;
  double be = 0.0;
  for (int j = 0; j < d->n_powers; ++j) {
    double t = t_prof_of(s, dnn, stage0, j);
    if (est->mu * t > goal) continue;
    double e = oracle_energy_mean(est, idl, d->power_cap[j], t, goal);
    if (bj < 0 || e < be) { be = e; bj = j; }
  }
  if (found) *found = bj >= 0;
  return bj < 0 ? d->n_powers - 1 : bj;
}

/* AppOnlyPolicy.decide (policies.py:350-356): best expected-accuracy stage
 * (its expected accuracy in *best_acc) */
static int app_only_stage(const Space* s, const OracleEst* est, int dnn, int power, double goal,
                          double* best_acc) {
  int best = 1;
  double ba = -1.0;
  for (int k = 1; k <= s->d->dnn_n_stages[dnn]; ++k) {
    double acc = anytime_acc(s, est, dnn, power, k, goal);
    if (acc > ba) { best = k; ba = acc; }
  }
  if (best_acc) *best_acc = ba;
  return best;
}

static int kinds_for(int policy) {
  if (policy == ALERT_POLICY_ALERT_ANY) return 1 << ALERT_KIND_ANYTIME;
  if (policy == ALERT_POLICY_ALERT_TRAD) return 1 << ALERT_KIND_TRADITIONAL;
  return 3;
}

/* simulator.py:461-507 over an injected environment */
static int run_s(const Space* s, const AlertSpec* specs, const int32_t* spec_index, const AlertFilterConfig* cfg,
                 int policy, int64_t n_steps, const double* sd, const double* idle, const int32_t* phase,
                 const int32_t* forced, OracleRecord* rec, double* agg, double* state, int state_in,
                 AlertPrediction* preds) {
  const AlertSpec* spec = spec_index ? &specs[spec_index[0]] : specs; /* spec at begin() */
  const AlertSpaceDesc* d = s->d;
  int kinds = kinds_for(policy);
  /* AlertPolicy.begin, policies.py:86-95 */
  int any = 0;
  for (int i = 0; i < d->n_dnns; ++i) any |= (kinds >> d->dnn_kind[i]) & 1;
  if (!any) return ALERT_ERR_NO_CANDIDATE;
  const int baseline = policy >= ALERT_POLICY_ORACLE_STATIC;
  if ((policy == ALERT_POLICY_SYS_ONLY && d->sys_dnn < 0) ||
      ((policy == ALERT_POLICY_APP_ONLY || policy == ALERT_POLICY_NO_COORD) && d->app_dnn < 0))
    return ALERT_ERR_NO_CANDIDATE;
  int32_t aux = -1;  /* oracle-static: candidate; no-coord: stage | power << 8 */
  OracleEst est;
  OracleIdle idl;
  double budget = 0.0;
  int32_t count = 0;
  if (state && state_in) {
    est.mu = state[0]; est.sigma2 = state[1]; est.k_gain = state[2]; est.q_noise = state[3];
    est.innov = state[4]; idl.phi = state[5]; idl.m_var = state[6];
    budget = state[7]; count = (int32_t)state[8];
    aux = (int32_t)state[9];
  } else {
    oracle_slowdown_init(cfg, &est);
    idl.phi = py_min(1.0, d->p_idle_prof / d->power_cap[d->n_powers - 1]);
    idl.m_var = cfg->m0;
  }
  if (aux < 0 && policy == ALERT_POLICY_ORACLE_STATIC) aux = oracle_static_choice(s, spec, n_steps, sd, idle);
  if (aux < 0 && policy == ALERT_POLICY_NO_COORD)
    aux = d->dnn_n_stages[d->app_dnn] | ((d->n_powers - 1) << 8); /* policies.py:385-386 */
  for (int64_t n = 0; n < n_steps; ++n) {
    const int32_t spec_k = spec_index ? spec_index[n] : 0;
    spec = &specs[spec_k]; /* policy.spec swapped (goal changes) */
    int has_group = spec->group_size > 0;
    if (has_group && count == 0) { /* simulator.py:473-478 */
      budget = (double)spec->group_size * spec->t_goal;
      count = spec->group_size;
    }
    double goal = oracle_adjust_goal(spec, has_group, budget, count);
    double period = goal + spec->overhead_budget;
    int32_t level = 0;
    double gap = INFINITY, boundary = INFINITY;
    int cand;
    int or_cand = -1;
    int32_t or_level = 0;
    int feasible = 1;
    /* ConfigDecision.prediction of the decision (latency mean / sigma, pr, accuracy, energy) */
    double pv[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (policy == ALERT_POLICY_ORACLE) {
      cand = oracle_decide_s(s, spec, sd[n], idle[n], goal, &level, &gap);
      feasible = level == 0;
      if (cand >= 0) { /* _exact_pred, policies.py:201-205 */
        int32_t oi, oj, ot;
        oracle_candidate(d, cand, &oi, &oj, &ot);
        Exact x = exact_eval(s, spec, sd[n], idle[n], oi, oj, ot, goal);
        pv[0] = x.latency; pv[2] = x.met ? 1.0 : 0.0; pv[3] = x.delivered; pv[4] = x.energy;
      }
    } else if (policy == ALERT_POLICY_ORACLE_STATIC) {
      cand = aux & 0xFFFF; /* OracleStaticPolicy.decide, policies.py:268-269 */
      feasible = (aux >> 16) != 0;
      pv[2] = feasible ? 1.0 : 0.0; /* _exact_pred(i, j, t, eligible, 0, 0, 0), policies.py:266-271 */
    } else if (policy == ALERT_POLICY_SYS_ONLY) {
      int pj = sys_only_power(s, &est, &idl, d->sys_dnn, 0, goal, &feasible);
      cand = cand_index(s, d->sys_dnn, pj, 0);
      double t = t_prof_of(s, d->sys_dnn, 0, pj); /* policies.py:314-320 */
      pv[0] = est.mu * t; pv[1] = est_sigma(&est) * t; pv[2] = feasible ? 1.0 : 0.0;
      pv[3] = acc_of(s, d->sys_dnn, 0); pv[4] = oracle_energy_mean(&est, &idl, d->power_cap[pj], t, goal);
    } else if (policy == ALERT_POLICY_APP_ONLY) {
      int pj = d->n_powers - 1;
      double ba;
      int st = app_only_stage(s, &est, d->app_dnn, pj, goal, &ba);
      cand = cand_index(s, d->app_dnn, pj, st);
      double t = t_prof_of(s, d->app_dnn, st - 1, pj); /* policies.py:357-368 */
      pv[0] = est.mu * t; pv[1] = est_sigma(&est) * t; pv[3] = ba;
    } else if (policy == ALERT_POLICY_NO_COORD) {
      /* NoCoordPolicy.decide (policies.py:392-428): the stage for the old
       * power, the power for the old stage, both from the same feedback (the
       * two estimators receive identical updates, so one is kept) */
      int st_old = aux & 0xff, pj_old = aux >> 8;
      double ba;
      int st = app_only_stage(s, &est, d->app_dnn, pj_old, goal, &ba);
      int pj = sys_only_power(s, &est, &idl, d->app_dnn, st_old - 1, goal, NULL);
      aux = st | (pj << 8);
      cand = cand_index(s, d->app_dnn, pj, st);
      double t = t_prof_of(s, d->app_dnn, st - 1, pj); /* policies.py:417-428 */
      pv[0] = est.mu * t; pv[1] = est_sigma(&est) * t; pv[3] = ba;
    } else {
      int np = predict_all_s(s, &est, &idl, spec, goal, preds);
      cand = select_s(s, preds, np, spec, kinds, &level, &gap, &boundary);
      feasible = level == 0;
      if (cand >= 0) {
        const AlertPrediction* p = &preds[cand];
        pv[0] = p->latency_mean; pv[1] = p->latency_sigma; pv[2] = p->pr_deadline;
        pv[3] = p->expected_accuracy; pv[4] = p->energy;
      }
      if (policy == ALERT_POLICY_ALERT_WITH_ORACLE)
        or_cand = oracle_decide_s(s, spec, sd[n], idle[n], goal, &or_level, NULL);
    }
    if (cand < 0) return ALERT_ERR_NO_CANDIDATE;
    int exec_c = (forced && forced[n] >= 0) ? forced[n] : cand;
    int32_t di, pj, tg;
    oracle_candidate(d, exec_c, &di, &pj, &tg);
    Exec o = execute_decision(s, sd[n], di, pj, tg, goal);
    Meas m = measure(s, spec, di, pj, &o, idle[n], period);
    /* AlertPolicy.observe, policies.py:105-108 (oracle: no-op, :207-208);
     * sys-only / no-coord :315-318 / :430-439; app-only slow-down only :359-360 */
    if (policy != ALERT_POLICY_ORACLE && policy != ALERT_POLICY_ORACLE_STATIC) {
      if (oracle_slowdown_update(cfg, &est, o.fb_latency, o.fb_t_prof)) return ALERT_ERR_INVALID_TRACE;
      if (policy != ALERT_POLICY_APP_ONLY && oracle_idle_update(cfg, &idl, idle[n], d->power_cap[pj]))
        return ALERT_ERR_INVALID_TRACE;
    }
    if (has_group) { /* simulator.py:501-503 */
      budget -= m.latency;
      count -= 1;
    }
    int ph = phase ? phase[n] : 0;
    if (rec) {
      OracleRecord* r = &rec[n];
      memset(r, 0, sizeof(*r));
      r->cand = exec_c; r->dnn = di; r->power = pj; r->stage = tg;
      r->level = level; r->completed = o.completed; r->met = m.met; r->phase = ph;
      r->viol_lat = m.vl; r->viol_acc = m.va; r->viol_energy = m.ve; r->or_cand = or_cand;
      r->feasible = feasible; r->spec_index = spec_k;
      r->pred_latency_mean = pv[0]; r->pred_latency_sigma = pv[1]; r->pred_pr = pv[2];
      r->pred_accuracy = pv[3]; r->pred_energy = pv[4];
      r->plan_goal = goal; r->period = period; r->latency = m.latency; r->accuracy = m.delivered;
      r->energy = m.energy; r->fb_latency = o.fb_latency; r->fb_t_prof = o.fb_t_prof; r->s = sd[n];
      r->mu = est.mu; r->sigma2 = est.sigma2; r->k_gain = est.k_gain; r->q_noise = est.q_noise;
      r->innov = est.innov; r->phi = idl.phi; r->m_var = idl.m_var;
      r->gap = gap; r->boundary = boundary;
    }
    if (agg) {
      agg[ALERT_AGG_N] += 1.0;
      neumaier(&agg[ALERT_AGG_ENERGY], &agg[ALERT_AGG_ENERGY_C], m.energy);
      neumaier(&agg[ALERT_AGG_ACC], &agg[ALERT_AGG_ACC_C], m.delivered);
      agg[ALERT_AGG_VIOL_LAT] += m.vl;
      agg[ALERT_AGG_VIOL_ACC] += m.va;
      agg[ALERT_AGG_VIOL_ENERGY] += m.ve;
      agg[ALERT_AGG_LEVEL0 + level] += 1.0;
      if (ph >= 0 && ph < ALERT_MAX_PHASES) {
        double* pa = agg + ALERT_AGG_PHASE_BASE + ALERT_AGG_PHASE_STRIDE * ph;
        pa[0] += 1.0;
        neumaier(&pa[1], &pa[2], m.energy);
        neumaier(&pa[3], &pa[4], m.delivered);
        pa[5] += m.vl; pa[6] += m.va; pa[7] += m.ve;
      }
      if (policy == ALERT_POLICY_ALERT_WITH_ORACLE) {
        int32_t oi, oj, ot;
        oracle_candidate(d, or_cand, &oi, &oj, &ot);
        Exec oo = execute_decision(s, sd[n], oi, oj, ot, goal);
        Meas om = measure(s, spec, oi, oj, &oo, idle[n], period);
        neumaier(&agg[ALERT_AGG_OR_ENERGY], &agg[ALERT_AGG_OR_ENERGY_C], om.energy);
        neumaier(&agg[ALERT_AGG_OR_ACC], &agg[ALERT_AGG_OR_ACC_C], om.delivered);
        agg[ALERT_AGG_OR_VIOL_LAT] += om.vl;
        agg[ALERT_AGG_OR_VIOL_ACC] += om.va;
        agg[ALERT_AGG_OR_VIOL_ENERGY] += om.ve;
        agg[ALERT_AGG_OR_SAME] += (or_cand == exec_c);
      }
    }
  }
  if (state) {
    state[0] = est.mu; state[1] = est.sigma2; state[2] = est.k_gain; state[3] = est.q_noise;
    state[4] = est.innov; state[5] = idl.phi; state[6] = idl.m_var;
    state[7] = budget; state[8] = (double)count;
    state[9] = (double)aux;
  }
  (void)baseline;
  return 0;
}

int oracle_run_goals(const AlertSpaceDesc* sp, const AlertSpec* specs, int32_t n_specs,
                     const int32_t* spec_index, const AlertFilterConfig* cfg, int policy, int64_t n_steps,
                     const double* sd, const double* idle, const int32_t* phase, const int32_t* forced,
                     OracleRecord* rec, double* agg, double* state, int state_in) {
  if (!specs || n_specs < 1) return ALERT_ERR_INVALID_ARGUMENT;
  if (spec_index)
    for (int64_t n = 0; n < n_steps; ++n)
      if (spec_index[n] < 0 || spec_index[n] >= n_specs) return ALERT_ERR_INVALID_ARGUMENT;
  Space s;
  if (space_open(sp, &s)) return ALERT_ERR_INVALID_ARGUMENT;
  AlertPrediction* preds = (AlertPrediction*)malloc(sizeof(AlertPrediction) * (size_t)(s.n_cand + 1));
  int r = preds ? run_s(&s, specs, spec_index, cfg, policy, n_steps, sd, idle, phase, forced, rec, agg, state,
                        state_in, preds)
                : ALERT_ERR_INVALID_ARGUMENT;
  free(preds);
  space_close(&s);
  return r;
}

int oracle_run(const AlertSpaceDesc* sp, const AlertSpec* spec, const AlertFilterConfig* cfg,
               int policy, int64_t n_steps, const double* sd, const double* idle,
               const int32_t* phase, const int32_t* forced, OracleRecord* rec, double* agg,
               double* state, int state_in) {
  return oracle_run_goals(sp, spec, 1, NULL, cfg, policy, n_steps, sd, idle, phase, forced, rec, agg, state,
                          state_in);
}

/* ---------------------------------------------------------------------- */
/* batched runner (CPU baseline / large parity checks)                      */

typedef struct BatchJob {
  const AlertSpaceDesc* sp;
  const AlertSpec* specs;
  int32_t n_specs;
  const int32_t* stream_spec;
  const AlertFilterConfig* cfg;
  int policy;
  const AlertTrace* tr;
  int64_t n_streams, step_begin, step_end;
  double* agg;
  double* state;
  int64_t next;
  pthread_mutex_t mu;
  int status;
} BatchJob;

static void* batch_worker(void* arg) {
  BatchJob* J = (BatchJob*)arg;
  Space s;
  if (space_open(J->sp, &s)) return NULL;
  int64_t len = J->step_end - J->step_begin;
  double* sd = (double*)malloc(sizeof(double) * (size_t)(len > 0 ? len : 1));
  double* idle = (double*)malloc(sizeof(double) * (size_t)(len > 0 ? len : 1));
  int32_t* ph = (int32_t*)malloc(sizeof(int32_t) * (size_t)(len > 0 ? len : 1));
  int32_t* gi = (int32_t*)malloc(sizeof(int32_t) * (size_t)(len > 0 ? len : 1));
  AlertPrediction* preds = (AlertPrediction*)malloc(sizeof(AlertPrediction) * (size_t)(s.n_cand + 1));
  for (;;) {
    pthread_mutex_lock(&J->mu);
    int64_t k = J->next++;
    pthread_mutex_unlock(&J->mu);
    if (k >= J->n_streams) break;
    const AlertTrace* t = J->tr;
    int64_t row = t->stream_row ? t->stream_row[k] : k;
    for (int64_t n = 0; n < len; ++n) {
      int64_t step = J->step_begin + n;
      int64_t off = row * t->row_stride + (step - t->step_offset) * t->step_stride;
      sd[n] = t->slowdown_dtype == ALERT_DTYPE_F64 ? ((const double*)t->slowdown)[off]
                                                   : (double)((const float*)t->slowdown)[off];
      int seg = 0;
      while (seg + 1 < t->n_segments[row] && step >= t->seg_end[row * t->max_segments + seg]) ++seg;
      idle[n] = t->seg_idle[row * t->max_segments + seg];
      ph[n] = t->seg_phase[row * t->max_segments + seg];
    }
    int32_t si = J->stream_spec ? J->stream_spec[k] : (int32_t)(k % J->n_specs);
    const int ng = t->n_goal_segments ? t->n_goal_segments[row] : 0;
    for (int64_t n = 0; n < len; ++n) { /* goal changes: the row's spec segments */
      int64_t step = J->step_begin + n;
      int g = 0;
      while (g + 1 < ng && step >= t->goal_seg_end[row * t->max_goal_segments + g]) ++g;
      gi[n] = ng ? t->goal_seg_spec[row * t->max_goal_segments + g] : si;
    }
    double* st = J->state ? J->state + ORACLE_STATE_FIELDS * k : NULL;
    int r = run_s(&s, J->specs, gi, J->cfg, J->policy, len, sd, idle, ph, NULL, NULL,
                  J->agg + (size_t)ALERT_AGG_FIELDS * k, st, J->step_begin > 0, preds);
    if (r) J->status = r;
  }
  free(sd); free(idle); free(ph); free(gi); free(preds);
  space_close(&s);
  return NULL;
}

int oracle_run_batch(const AlertSpaceDesc* sp, const AlertSpec* specs, int32_t n_specs,
                     const int32_t* stream_spec, const AlertFilterConfig* cfg, int policy,
                     const AlertTrace* trace, int64_t n_streams, int64_t step_begin, int64_t step_end,
                     double* agg, double* state, int n_threads) {
  if (!sp || !specs || n_specs < 1 || !cfg || !trace || !agg || n_threads < 1) return ALERT_ERR_INVALID_ARGUMENT;
  BatchJob J = {sp, specs, n_specs, stream_spec, cfg, policy, trace, n_streams, step_begin, step_end,
                agg, state, 0, PTHREAD_MUTEX_INITIALIZER, 0};
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
  for (int t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, batch_worker, &J);
  for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
  free(th);
  return J.status;
}
