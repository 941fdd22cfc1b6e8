/*
 * alert_oracle.h — CPU restatement of the reference (alertsim) hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the timed CPU baseline — never as a product path.
 *
 * Plain FP64 C with the reference's operation order, compiled with
 * -ffp-contract=off and without builtin pow/erf so every libm call is the same
 * glibc call CPython makes (math.erf -> erf, float ** -> pow).  Pinned against
 * golden vectors produced by the reference itself (tests/golden/).
 */
#ifndef ALERT_ORACLE_H
#define ALERT_ORACLE_H

#include <stdint.h>
#include "../include/alert_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct OracleEst {   /* SlowdownEstimate, estimator.py:33-40 */
  double mu, sigma2, k_gain, q_noise, innov;
} OracleEst;

typedef struct OracleIdle {  /* IdlePowerEstimate, estimator.py:94-98 */
  double phi, m_var;
} OracleIdle;

#define ORACLE_STATE_FIELDS 10

/* One StepRecord (simulator.py:311-326) plus the policy state after observe
 * and near-tie diagnostics (top-2 relative gap of the primary objective at the
 * chosen fallback level; minimum relative constraint-boundary distance). */
typedef struct OracleRecord {
  int32_t cand, dnn, power, stage;      /* stage 0 = None                    */
  int32_t level, completed, met, phase;
  int32_t viol_lat, viol_acc, viol_energy, or_cand;
  int32_t feasible, spec_index;         /* ConfigDecision.feasible; spec in force (goal changes) */
  double plan_goal, period, latency, accuracy, energy, fb_latency, fb_t_prof, s;
  double mu, sigma2, k_gain, q_noise, innov, phi, m_var;
  double gap, boundary;
  /* ConfigDecision.prediction: latency_mean, latency_sigma, pr_deadline,
   * expected_accuracy, energy (predictor.py:36-45) */
  double pred_latency_mean, pred_latency_sigma, pred_pr, pred_accuracy, pred_energy;
} OracleRecord;

int oracle_num_candidates(const AlertSpaceDesc* sp);
int oracle_candidate(const AlertSpaceDesc* sp, int c, int32_t* dnn, int32_t* power, int32_t* stage);

/* predictor.py:25-33, 48-65 */
double oracle_normal_cdf(double x);
double oracle_deadline_probability(const OracleEst* est, double t_prof, double t_goal);
/* predictor.py:83-108 (reference O(S^2) form) */
double oracle_expected_accuracy_anytime(const AlertSpaceDesc* sp, const OracleEst* est, int dnn,
                                        int power, int target, double t_goal);
/* predictor.py:111-144 */
double oracle_energy_mean(const OracleEst* est, const OracleIdle* idle, double p, double t_prof, double goal);
double oracle_energy_percentile(const OracleEst* est, const OracleIdle* idle, double p, double t_prof,
                                double goal, double z_q);
/* predictor.py:147-197; returns number of predictions written */
int oracle_predict_all(const AlertSpaceDesc* sp, const OracleEst* est, const OracleIdle* idle,
                       const AlertSpec* spec, double goal, AlertPrediction* out);
/* selector.py:102-131 and 134-182.  kinds_mask bit k admits ALERT_KIND k
 * (policies.py:99-102).  Returns the index into preds (or -1), level in *level. */
int oracle_select(const AlertSpaceDesc* sp, const AlertPrediction* preds, int n, const AlertSpec* spec,
                  int kinds_mask, int32_t* level, double* gap, double* boundary);
int oracle_brute_force_select(const AlertSpaceDesc* sp, const AlertPrediction* preds, int n,
                              const AlertSpec* spec, int kinds_mask, int32_t* level);
/* estimator.py:47-127 */
void oracle_slowdown_init(const AlertFilterConfig* cfg, OracleEst* est);
int oracle_slowdown_update(const AlertFilterConfig* cfg, OracleEst* est, double obs, double t_prof);
int oracle_idle_update(const AlertFilterConfig* cfg, OracleIdle* idle, double measured, double cap);
/* selector.py:48-70 (floor 0.001) */
double oracle_adjust_goal(const AlertSpec* spec, int has_group, double budget, int32_t count);
/* policies.py:160-205: candidate index chosen by the clairvoyant oracle */
int oracle_oracle_decide(const AlertSpaceDesc* sp, const AlertSpec* spec, double s, double idle,
                         double goal, int32_t* level, double* gap);

/* simulator.run (simulator.py:461-507) over injected per-step arrays
 * (s, idle power, phase id) for one stream.  policy = ALERT_POLICY_*.
 * forced[n] >= 0 executes that candidate instead (teacher forcing).
 * rec (nullable) gets n_steps records; agg (nullable) ALERT_AGG_FIELDS sums;
 * state (nullable, in/out, ORACLE_STATE_FIELDS doubles: mu sigma2 k q y phi m
 * budget count aux; aux = AlertState.policy_aux of the comparison schemes) —
 * when state_in is nonzero the run resumes from it instead of begin(). */
int oracle_run(const AlertSpaceDesc* sp, const AlertSpec* spec, const AlertFilterConfig* cfg,
               int policy, int64_t n_steps, const double* s, const double* idle,
               const int32_t* phase, const int32_t* forced, OracleRecord* rec, double* agg,
               double* state, int state_in);
/* oracle_run with goal changes: step n runs under specs[spec_index[n]]
 * (spec_index NULL: specs[0] throughout) — the reference's run loop with
 * policy.spec swapped before each decide and each input measured against the
 * spec in force (SURVEY.md §7 hard part 8; simulator.py:473-497). */
int oracle_run_goals(const AlertSpaceDesc* sp, const AlertSpec* specs, int32_t n_specs,
                     const int32_t* spec_index, const AlertFilterConfig* cfg, int policy, int64_t n_steps,
                     const double* s, const double* idle, const int32_t* phase, const int32_t* forced,
                     OracleRecord* rec, double* agg, double* state, int state_in);

/* Batched runs over a HOST AlertTrace (same layout as the device one) with
 * n_threads POSIX threads, one stream at a time per thread.  agg:
 * [n_streams][ALERT_AGG_FIELDS]; state: [n_streams][ORACLE_STATE_FIELDS] (nullable). */
int oracle_run_batch(const AlertSpaceDesc* sp, const AlertSpec* specs, int32_t n_specs,
                     const int32_t* stream_spec, const AlertFilterConfig* cfg, int policy,
                     const AlertTrace* trace, int64_t n_streams, int64_t step_begin, int64_t step_end,
                     double* agg, double* state, int n_threads);

#ifdef __cplusplus
}
#endif
#endif
