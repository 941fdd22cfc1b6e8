/*
 * alert_b200.h — C ABI of the B200-native ALERT scheduling step.
 *
 * The reference (alertsim, pure Python) has no FFI; every entry point below
 * replaces one Python call on the hot path and says which (path:line relative
 * to the reference root /root/reference):
 *
 *   alert_run            simulator.run                pkg/src/alertsim/simulator.py:461-507
 *                        with AlertPolicy / OraclePolicy pkg/src/alertsim/policies.py:70-108,149-208
 *   alert_decide         AlertPolicy.decide           pkg/src/alertsim/policies.py:97-103
 *                        (= predict_all + kinds filter + select, predictor.py:147, selector.py:102)
 *   alert_predict        predict_all                  pkg/src/alertsim/predictor.py:147-197
 *   alert_observe        AlertPolicy.observe          pkg/src/alertsim/policies.py:105-108
 *                        (= slowdown_update estimator.py:59-84, idle_power_update estimator.py:110-127)
 *   alert_oracle_decide  OraclePolicy.decide          pkg/src/alertsim/policies.py:160-205
 *   alert_reduce         _summarize (aggregate part)  pkg/src/alertsim/simulator.py:428-458
 *
 * Conventions
 *   - Plain C types only.  Pointers inside AlertTrace / AlertState / AlertOutputs /
 *     spec arrays are DEVICE pointers owned by the caller; the library never frees
 *     or allocates caller-visible memory.  AlertSpaceDesc holds HOST pointers and is
 *     copied into a device-resident AlertTable by alert_table_create.
 *   - Every call is asynchronous on the caller's cudaStream_t (passed as void*).
 *   - Return value: ALERT_OK (0) or a negative AlertStatus; alert_strerror() names
 *     it and alert_last_error() gives the detailed message of the last failure on
 *     the calling thread.  The library never aborts the process.
 *   - Arithmetic: per-candidate scan in FP32 with an FP64 re-rank of every
 *     near-tie / constraint-boundary candidate; filter state, execution and
 *     accounting in FP64 with the reference's operation order.
 */
#ifndef ALERT_B200_H
#define ALERT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ALERT_ABI_VERSION 4  /* 2: comparison-scheme policies, AlertSpaceDesc.sys_dnn/app_dnn, AlertState.policy_aux, AlertOutputs.fb_*, alert_xi_stats
                               3: goal schedules (AlertTrace.goal_*), AlertOutputs.plan_goal/phi, decision bit 30
                                  (feasible), alert_baseline_decide / alert_static_choice (per-step comparison schemes)
                               4: ALERT_FLAG_FRESH (state initialised / aggregates zeroed inside alert_run) */

/* ---- status codes ------------------------------------------------------ */
typedef enum AlertStatus {
  ALERT_OK = 0,
  ALERT_ERR_INVALID_ARGUMENT = -1, /* bad pointer / size / enum                */
  ALERT_ERR_INVALID_SPACE = -2,    /* model.validate() would report problems  */
  ALERT_ERR_INVALID_SPEC = -3,     /* ConstraintSpec.__post_init__ would raise */
  ALERT_ERR_INVALID_TRACE = -4,    /* TraceError-class problem                */
  ALERT_ERR_CUDA = -5,             /* CUDA runtime error                       */
  ALERT_ERR_UNSUPPORTED = -6,      /* size outside the compiled limits         */
  ALERT_ERR_NO_CANDIDATE = -7      /* kinds filter leaves nothing (policies.py:92-95) */
} AlertStatus;

/* ---- enums ------------------------------------------------------------- */
enum { ALERT_KIND_TRADITIONAL = 0, ALERT_KIND_ANYTIME = 1 };      /* model.py:17-19 */
enum { ALERT_MODE_MIN_ENERGY = 0, ALERT_MODE_MAX_ACCURACY = 1 };  /* model.py:22-24 */
enum { ALERT_LEVEL_NONE = 0, ALERT_LEVEL_DROPPED_ENERGY = 1,
       ALERT_LEVEL_DROPPED_ACCURACY = 2 };                         /* selector.py:20-23 */
enum {                                                            /* policies.py:457-490 */
  ALERT_POLICY_ALERT = 0,       /* "alert"                                    */
  ALERT_POLICY_ALERT_ANY = 1,   /* "alert-any"  (anytime DNNs only)           */
  ALERT_POLICY_ALERT_TRAD = 2,  /* "alert-trad" (traditional DNNs only)       */
  ALERT_POLICY_ORACLE = 3,      /* "oracle" (clairvoyant per-input optimum)   */
  ALERT_POLICY_ALERT_WITH_ORACLE = 4, /* ALERT executed, oracle evaluated alongside
                                        on the same step (config 5 fused path) */
  /* comparison schemes (policies.py:211-454) */
  ALERT_POLICY_ORACLE_STATIC = 5, /* "oracle-static": best fixed candidate over the whole trace */
  ALERT_POLICY_SYS_ONLY = 6,      /* "sys-only": fastest traditional DNN, power cap adapted    */
  ALERT_POLICY_APP_ONLY = 7,      /* "app-only": one anytime DNN at max power, stage adapted   */
  ALERT_POLICY_NO_COORD = 8       /* "no-coord": stage and power controllers uncoordinated     */
};
enum { ALERT_DTYPE_F32 = 0, ALERT_DTYPE_F64 = 1 };

/* Run flags */
#define ALERT_FLAG_FP64_ALL 0x1u   /* skip the FP32 scan: every candidate in FP64 (debug / proof) */
#define ALERT_FLAG_NO_REFINE 0x2u  /* FP32 decision only (measures the refinement cost; not reference-exact) */
#define ALERT_FLAG_NO_FAST 0x4u    /* disable the min-energy fast scan (full FP32 scan every step; A/B and tests) */
#define ALERT_FLAG_FAST_ROWS 0x8u  /* fast scan in row mode even for small tables (tests) */
#define ALERT_FLAG_ANY_WINDOW 0x10u /* anytime cells by the two-pass window instead of column skips (A/B, tests) */
#define ALERT_FLAG_NO_ORACLE_FAST 0x40u /* oracle: full scan only (no certified min-energy fast scan; A/B, tests) */
#define ALERT_FLAG_FRESH 0x20u     /* the step range starts the runs: the filter state is initialised in the
                                    * launch (state arrays written, not read: no alert_state_init needed) and
                                    * the aggregate blocks are written from zero (not accumulated: no memset) */

/* Compiled limits */
#define ALERT_MAX_STAGES 8         /* stages per anytime DNN                   */
#define ALERT_MAX_PHASES 8         /* phase ids per trace for per-phase sums   */
#define ALERT_MAX_CANDIDATES 6144   /* 32 B/candidate of shared memory per block */

/* ---- candidate table (host description) -------------------------------- */
/* Flattened model.ConfigSpace (model.py:55-63).  Stages are stored dnn-major;
 * stage_t_prof is [total_stages][n_powers] (Stage.t_prof, model.py:36-40). */
typedef struct AlertSpaceDesc {
  int32_t n_dnns;
  int32_t n_powers;
  const int32_t* dnn_kind;       /* [n_dnns] ALERT_KIND_*                      */
  const int32_t* dnn_n_stages;   /* [n_dnns] 1 for traditional, >=2 anytime    */
  const double* dnn_q_fail;      /* [n_dnns] DnnProfile.q_fail                 */
  const double* stage_accuracy;  /* [total_stages]                             */
  const double* stage_t_prof;    /* [total_stages][n_powers] seconds           */
  const double* power_cap;       /* [n_powers] PowerSetting.cap_watts          */
  double p_idle_prof;            /* ConfigSpace.p_idle_prof                    */
  /* DNNs of the comparison schemes, chosen by the host from the DnnProfile ids
   * (the ABI carries no ids): sys-only = fastest_dnn(space, last power,
   * TRADITIONAL) (policies.py:292, model.py:166-176); app-only / no-coord =
   * _pick_anytime (policies.py:324-329).  -1 = no such DNN. */
  int32_t sys_dnn;
  int32_t app_dnn;
} AlertSpaceDesc;

/* Filter constants: KalmanConfig (estimator.py:18-30) + IdleFilterConfig (:87-91). */
typedef struct AlertFilterConfig {
  double k0, r, q0, alpha, mu0, sigma2_0;
  int32_t sigma2_uses_current_gain;
  int32_t _pad;
  double m0, s, v;
} AlertFilterConfig;

/* model.ConstraintSpec (model.py:66-97) plus the trace's group_size
 * (simulator.py:103).  64 bytes, 8-byte aligned. */
typedef struct AlertSpec {
  int32_t mode;           /* ALERT_MODE_*                                      */
  int32_t has_pr;         /* 1 when pr_threshold is not None                   */
  int32_t group_size;     /* 0 = no shared-deadline groups                     */
  int32_t _pad;
  double t_goal;          /* seconds                                           */
  double e_goal;          /* joules (max-accuracy mode)                        */
  double q_goal;          /* accuracy (min-energy mode)                        */
  double pr_threshold;    /* in (0,1) when has_pr                              */
  double z_q;             /* NormalDist().inv_cdf(pr_threshold), predictor.py:30-33,
                             computed on the host (bit-identical to the reference) */
  double overhead_budget; /* seconds                                           */
} AlertSpec;

/* ---- opaque handles ---------------------------------------------------- */
typedef struct AlertContext AlertContext;
typedef struct AlertTable AlertTable;

/* ---- trace, state, outputs (DEVICE pointers) --------------------------- */
/* A realized environment (simulator.TrueEnvironment, simulator.py:212-218)
 * for n_rows traces.  Streams map to rows through stream_row (NULL: row =
 * stream), so many scenarios can share one trace.  Each row is cut into
 * segments of constant (phase id, idle power) — what realize() produces
 * (simulator.py:221-235). */
typedef struct AlertTrace {
  const void* slowdown;       /* true slow-down s per (row, step)              */
  int32_t slowdown_dtype;     /* ALERT_DTYPE_F32 | ALERT_DTYPE_F64             */
  int32_t n_rows;
  int64_t n_steps;            /* steps available per row                       */
  int64_t row_stride;         /* elements between rows  (time-major: 1)        */
  int64_t step_stride;        /* elements between steps (time-major: n_rows)   */
  int64_t step_offset;        /* first step held by `slowdown` (chunked streaming:
                                 element (row, n) is at (n - step_offset) * step_stride
                                 + row * row_stride); 0 for a whole trace        */
  int32_t max_segments;       /* per-row capacity of the segment arrays        */
  int32_t _pad;
  const int32_t* n_segments;  /* [n_rows]                                      */
  const int32_t* seg_end;     /* [n_rows][max_segments] exclusive end step     */
  const int32_t* seg_phase;   /* [n_rows][max_segments] phase id (< ALERT_MAX_PHASES) */
  const double* seg_idle;     /* [n_rows][max_segments] idle_power_true, W     */
  const int32_t* stream_row;  /* [n_streams] or NULL                           */
  /* Goal changes (optional, NULL = none): per row, segments of constant
   * constraint spec.  Step n of row r runs under specs[goal_seg_spec[r][g]]
   * for the segment g with goal_seg_end[r][g-1] <= n < goal_seg_end[r][g]
   * (the last segment is open-ended); rows with n_goal_segments[r] == 0 use
   * the stream's spec (stream_spec).  The reference keeps one spec per run;
   * a change is mirrored there by swapping policy.spec before decide and
   * measuring against the new spec (SURVEY.md §7 hard part 8; policies.py:97-103,
   * simulator.py:473-497).  A shared-deadline group that is open when the spec
   * changes keeps its remaining budget; a new group takes the current spec's
   * group_size and t_goal.  oracle-static chooses with the spec in force at
   * the first step of the call (OracleStaticPolicy.begin, policies.py:221-227). */
  int32_t max_goal_segments;  /* per-row capacity of the goal arrays           */
  int32_t _pad2;
  const int32_t* n_goal_segments; /* [n_rows]                                  */
  const int32_t* goal_seg_end;    /* [n_rows][max_goal_segments] exclusive end  */
  const int32_t* goal_seg_spec;   /* [n_rows][max_goal_segments] index into specs */
} AlertTrace;

/* Per-stream policy state, FP64 SoA, read at step_begin and written back at
 * step_end so runs can be chunked over steps and resumed bit-identically.
 * mu..innov = SlowdownEstimate (estimator.py:33-40); phi, m_var =
 * IdlePowerEstimate (:94-98); group_* = GroupState (selector.py:36-41). */
typedef struct AlertState {
  double* mu;
  double* sigma2;
  double* k_gain;
  double* q_noise;
  double* innov;
  double* phi;
  double* m_var;
  double* group_budget;
  int32_t* group_count;
  /* per-stream state of the comparison schemes (NULL allowed for the others):
   * oracle-static = chosen candidate, no-coord = stage | power << 8;
   * -1 = not begun (the run performs begin()) */
  int32_t* policy_aux;
} AlertState;

/* Per-stream FP64 aggregate block (in/out, accumulated in step order).  The
 * reference's means are CPython 3.12 sum() results, i.e. Neumaier-compensated
 * sums (bltinmodule.c builtin_sum_impl); every float sum therefore carries its
 * compensation term *_C and the mean is (S + C) / N (C added only when nonzero
 * and finite).  Integer counts are exact.  Field offsets: */
enum {
  ALERT_AGG_N = 0, ALERT_AGG_ENERGY = 1, ALERT_AGG_ENERGY_C = 2, ALERT_AGG_ACC = 3,
  ALERT_AGG_ACC_C = 4, ALERT_AGG_VIOL_LAT = 5, ALERT_AGG_VIOL_ACC = 6, ALERT_AGG_VIOL_ENERGY = 7,
  ALERT_AGG_LEVEL0 = 8, ALERT_AGG_LEVEL1 = 9, ALERT_AGG_LEVEL2 = 10,
  ALERT_AGG_REFINED = 11,     /* steps whose decision needed the FP64 re-rank  */
  ALERT_AGG_OR_ENERGY = 12,   /* ALERT_POLICY_ALERT_WITH_ORACLE: oracle sums   */
  ALERT_AGG_OR_ENERGY_C = 13, ALERT_AGG_OR_ACC = 14, ALERT_AGG_OR_ACC_C = 15,
  ALERT_AGG_OR_VIOL_LAT = 16, ALERT_AGG_OR_VIOL_ACC = 17, ALERT_AGG_OR_VIOL_ENERGY = 18,
  ALERT_AGG_OR_SAME = 19,     /* steps where both chose the same candidate     */
  ALERT_AGG_FULL_SCAN = 20,   /* min-energy steps the fast scan could not certify (full scan ran) */
  ALERT_AGG_PHASE_BASE = 24,  /* + 8*phase + {n, e, e_c, acc, acc_c, vl, va, ve} */
  ALERT_AGG_PHASE_STRIDE = 8,
  ALERT_AGG_FIELDS = 88
};

/* Per-step record fields (all optional).  Layout [step][stream] through the
 * strides (time-major: stream_stride 1, step_stride n_streams) so a warp's
 * stores coalesce.  `decision` packs:
 *   bits  0..15 candidate index (reference enumeration order, policies.py:59-67)
 *   bits 16..17 fallback level        bit 18 deadline_met
 *   bits 19..21 violations (latency, accuracy, energy)
 *   bits 22..25 completed_stage        bit 26 FP64 re-rank used
 *   bits 27..29 phase id (low 3 bits)
 *   bit  30     ConfigDecision.feasible (selector.py:126: level NONE; sys-only:
 *               some cap predicted on time, policies.py:305-310; oracle-static:
 *               the choice is eligible, policies.py:257-271; app-only / no-coord: 1) */
typedef struct AlertOutputs {
  uint32_t* decision;
  void* energy;         /* StepRecord.energy                 */
  void* accuracy;       /* StepRecord.delivered_accuracy     */
  void* latency;        /* StepRecord.observed_latency       */
  void* mu;             /* slow-down mean after observe      */
  void* sigma2;         /* slow-down variance after observe  */
  uint32_t* oracle_decision; /* ALERT_POLICY_ALERT_WITH_ORACLE only */
  int32_t record_dtype; /* ALERT_DTYPE_F32 (default) or ALERT_DTYPE_F64 for the five value arrays */
  int32_t _pad;
  int64_t stream_stride;
  int64_t step_stride;
  double* agg;          /* [n_streams][ALERT_AGG_FIELDS] or NULL */
  const int32_t* forced; /* [step][stream] candidate to execute (teacher
                            forcing) or -1; NULL = free running.  Same strides. */
  double* fb_latency;   /* StepRecord.fb_latency (FP64, same strides) or NULL */
  double* fb_t_prof;    /* StepRecord.fb_t_prof  (FP64, same strides) or NULL */
  double* plan_goal;    /* adjusted per-input goal the decision was made for
                           (simulator.py:479-483; StepRecord.period = plan_goal +
                           overhead_budget) (FP64, same strides) or NULL */
  double* phi;          /* idle-power ratio estimate after observe (FP64) or NULL;
                           with mu / sigma2 it is the state the next decide uses */
} AlertOutputs;

/* One prediction (predictor.Prediction, predictor.py:36-45), FP64. */
typedef struct AlertPrediction {
  double latency_mean, latency_sigma, pr_deadline, expected_accuracy, energy;
  int32_t dnn_index, power_index, target_stage, _pad;
} AlertPrediction;

/* ---- API --------------------------------------------------------------- */
int alert_abi_version(void);
const char* alert_strerror(int status);
const char* alert_last_error(void);

int alert_create(AlertContext** out, int device);
int alert_destroy(AlertContext* ctx);

/* Validates like model.validate (model.py:100-163) and uploads. */
int alert_table_create(AlertContext* ctx, const AlertSpaceDesc* space, AlertTable** out);
int alert_table_destroy(AlertTable* table);
int alert_table_num_candidates(const AlertTable* table);
/* Candidate c -> (dnn, power, target stage; 0 = None), reference order. */
int alert_table_candidate(const AlertTable* table, int c, int32_t* dnn, int32_t* power, int32_t* stage);

/* Initial state (slowdown_init estimator.py:47-56; phi0 policies.py:90;
 * idle_power_init estimator.py:101-107; empty group). */
int alert_state_init(AlertContext* ctx, const AlertTable* table, const AlertFilterConfig* cfg,
                     AlertState state, int64_t n_streams, void* cuda_stream);

/* Fused closed loop for streams [stream_begin, stream_end) over steps
 * [step_begin, step_end): goal adjust -> decide -> execute -> measure ->
 * observe, per step, state in registers.  Specs are a device array indexed
 * by stream_spec[stream] (NULL: stream % n_specs). */
int alert_run(AlertContext* ctx, const AlertTable* table, const AlertFilterConfig* cfg,
              const AlertSpec* specs, int32_t n_specs, const int32_t* stream_spec,
              const AlertTrace* trace, AlertState state, const AlertOutputs* out,
              int32_t policy, uint32_t flags,
              int64_t stream_begin, int64_t stream_end,
              int64_t step_begin, int64_t step_end, void* cuda_stream);

/* One decide for each of n streams given their state and plan goal
 * (plan_goal[n], FP64).  decision[n] packed as in AlertOutputs (bits 0..17, 26). */
int alert_decide(AlertContext* ctx, const AlertTable* table, const AlertSpec* specs,
                 int32_t n_specs, const int32_t* stream_spec, AlertState state,
                 const double* plan_goal, int32_t policy, uint32_t flags,
                 uint32_t* decision, int64_t n, void* cuda_stream);

/* predict_all for each of n streams: out[n][n_candidates] (unfiltered). */
int alert_predict(AlertContext* ctx, const AlertTable* table, const AlertSpec* specs,
                  int32_t n_specs, const int32_t* stream_spec, AlertState state,
                  const double* plan_goal, AlertPrediction* out, int64_t n, void* cuda_stream);

/* observe for each of n streams: fb pair, true idle power, chosen power index. */
int alert_observe(AlertContext* ctx, const AlertTable* table, const AlertFilterConfig* cfg,
                  AlertState state, const double* fb_latency, const double* fb_t_prof,
                  const double* idle_power_true, const int32_t* power_index, int64_t n,
                  void* cuda_stream);

/* OraclePolicy.decide for n (stream, step) items: true slow-down s[n] (FP64),
 * true idle power idle[n], plan goal[n].  exact (nullable): the chosen
 * config's _exact_pred (policies.py:172-205: measured latency incl. overhead,
 * sigma 0, pr 1/0 = deadline met, delivered accuracy, energy). */
int alert_oracle_decide(AlertContext* ctx, const AlertTable* table, const AlertSpec* specs,
                        int32_t n_specs, const int32_t* stream_spec, const double* s,
                        const double* idle, const double* plan_goal, uint32_t flags,
                        uint32_t* decision, AlertPrediction* exact, int64_t n, void* cuda_stream);

/* Comparison schemes step by step (policies.py:211-454).
 * alert_static_choice = OracleStaticPolicy.begin (policies.py:221-265) for
 * streams [stream_begin, stream_end) over steps [step_begin, step_end) of the
 * trace: writes AlertState.policy_aux = candidate | eligible << 16.
 * alert_baseline_decide = SysOnly / AppOnly / NoCoord / OracleStatic.decide
 * (policies.py:298-313, 350-368, 392-428, 268-269) for n streams from their
 * state and plan goal; no-coord updates policy_aux (its controllers' memory).
 * Decisions packed as in AlertOutputs (bits 0..17, 30).  The filters are
 * updated with alert_observe. */
int alert_static_choice(AlertContext* ctx, const AlertTable* table, const AlertSpec* specs, int32_t n_specs,
                        const int32_t* stream_spec, const AlertTrace* trace, AlertState state,
                        int64_t stream_begin, int64_t stream_end, int64_t step_begin, int64_t step_end,
                        void* cuda_stream);
int alert_baseline_decide(AlertContext* ctx, const AlertTable* table, const AlertSpec* specs, int32_t n_specs,
                          const int32_t* stream_spec, AlertState state, const double* plan_goal,
                          int32_t policy, uint32_t* decision, int64_t n, void* cuda_stream);

/* Deterministic fixed-order sum of agg[n_streams][ALERT_AGG_FIELDS] into
 * out[ALERT_AGG_FIELDS] (device), pairwise tree in stream order. */
int alert_reduce(AlertContext* ctx, const double* agg, int64_t n_streams, double* out,
                 void* cuda_stream);

/* Launch geometry used by alert_run: lanes per stream (1..32) and threads per
 * block; 0 = library default.  Returns the values in effect. */
int alert_set_launch(AlertContext* ctx, int lanes_per_stream, int threads_per_block);
int alert_get_launch(AlertContext* ctx, int* lanes_per_stream, int* threads_per_block);

/* Number of alert_* kernels launched through this context (instrumentation). */
int64_t alert_launch_count(AlertContext* ctx);

/* Measured FP32 issue peak (FFMA lane-ops/s) of a device: the denominator of
 * the FP32 roofline (instrumentation, not part of the scheduling path). */
int alert_probe_fp32_peak(int device, double* slots_per_s);

/* On-device trace realization: one stream per
 * thread, Philox4x32-10 (curand) keyed by (seed, stream_offset + stream), the
 * reference's per-phase recipe (simulator.py:221-235: draw from the phase's
 * distribution, multiply by N(1, input_noise_sd) when > 0, floor at 0.01).
 * The VALUES differ from numpy's PCG64 streams (distributional parity only);
 * decisions are checked against the CPU oracle on the exported arrays.
 * out: time-major [sum(length)][n_streams] with row stride n_streams, FP32
 * (dtype ALERT_DTYPE_F32) or FP64. */
enum { ALERT_DIST_CONSTANT = 0, ALERT_DIST_GAUSSIAN = 1, ALERT_DIST_LOGNORMAL = 2, ALERT_DIST_UNIFORM = 3 };
typedef struct AlertPhaseDesc {
  int64_t length;
  int32_t dist;          /* ALERT_DIST_* */
  int32_t _pad;
  double a, b;           /* Constant: value; Gaussian: mean, sd; LogNormal: mu_log, sd_log; Uniform: lo, hi */
  double input_noise_sd;
} AlertPhaseDesc;
int alert_realize(AlertContext* ctx, const AlertPhaseDesc* phases, int32_t n_phases, uint64_t seed,
                  int64_t stream_offset, int64_t n_streams, void* out, int32_t dtype, void* cuda_stream);

/* xi_diagnostics_from_values (simulator.py:521-543): xi = num / den (den may be
 * NULL: xi = num), n >= 1 values, DEVICE buffers.  counts[bins] / edges[bins+1]
 * follow numpy.histogram(xi, bins) bit for bit (min/max edges, linspace,
 * numpy's index correction); mean_sd[2] = numpy.mean / numpy.std with numpy's
 * pairwise summation order.  (The reference needs >= 30 values; the caller
 * checks, as the reference raises ValueError.) */
int alert_xi_stats(AlertContext* ctx, const double* num, const double* den, int64_t n, int32_t bins,
                   int64_t* counts, double* edges, double* mean_sd, void* cuda_stream);

/* The scan's FP32 normal CDF: out[i] = Phi(sqrt(2) * x[i]) for device arrays
 * (instrumentation: lets tests bound its error against FP64). */
int alert_probe_phi32(const float* x, float* out, int64_t n, void* cuda_stream);
/* erfc(x) with relative accuracy (max-accuracy tail ordering), instrumentation. */
int alert_probe_erfc_rel(const float* x, float* out, int64_t n, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* ALERT_B200_H */
