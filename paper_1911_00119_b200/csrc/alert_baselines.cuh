// alert_baselines.cuh — the reference's comparison schemes on the GPU
// (policies.py:211-454): oracle-static, sys-only, app-only,
// no-coord.  All FP64 with the reference's operation order; one thread per
// stream for the closed loop (each scheme scans <= n_powers or <= n_stages
// candidates per step), one block per stream for oracle-static's begin().
#pragma once
#include "alert_kernels.cuh"

namespace alert {

struct BaseParams {
  DevTable T;
  AlertFilterConfig cfg;
  const SpecDev* specs;
  int n_specs;
  const int32_t* stream_spec;
  AlertTrace tr;
  AlertState st;
  AlertOutputs out;
  int policy;
  long long stream_begin, stream_end, step_begin, step_end;
};

__device__ __forceinline__ double base_s(const AlertTrace& tr, long long row, long long n) {
  return s_of_raw(tr, load_s_raw(tr, row, n));
}

// predict_energy_mean (predictor.py:111-126), reference order
__device__ __forceinline__ double energy_mean64(double mu, double phi, double p, double t, double goal) {
  const double lat = xmul(mu, t);
  return xadd(xmul(p, lat), xmul(xmul(phi, p), py_max(0.0, xsub(goal, lat))));
}

// SysOnlyPolicy.decide (policies.py:298-313) / NoCoord's system side
// (:409-419): cheapest cap whose predicted mean latency meets the goal; none
// -> the last (fastest) power.  cell_at(j) = the cell whose t_prof is used.
template <class F>
__device__ __forceinline__ int cheapest_power(const DevTable& T, const Cell64* C, const Filter& f, double goal,
                                              F cell_at, bool* feasible = nullptr) {
  int bj = -1;
  double be = 0.0;
  for (int j = 0; j < T.n_powers; ++j) {
    const Cell64& c = C[cell_at(j)];
    if (xmul(f.mu, c.t) > goal) continue;
    const double e = energy_mean64(f.mu, f.phi, c.cap, c.t, goal);
    if (bj < 0 || e < be) {
      be = e;
      bj = j;
    }
  }
  if (feasible) *feasible = bj >= 0;  // policies.py:305-310
  return bj < 0 ? T.n_powers - 1 : bj;
}

// AppOnlyPolicy.decide (policies.py:350-356) / NoCoord's application side
// (:399-405): the stage with the best expected_accuracy_anytime
// (predictor.py:83-108) at one power; the per-stage deadline probabilities
// are shared by every target (the reference recomputes identical values).
__device__ __forceinline__ int best_stage(const Cell64* C, int first, int S, const Filter& f, double goal) {
  const double sig = sqrt(f.sigma2);  // estimator.py:42-44 (pow(x, 0.5); ulp-level difference documented)
  double prs[ALERT_MAX_STAGES + 1];
  for (int m = 0; m < S; ++m) prs[m] = phi64(goal, f.mu, sig, C[first + m].t);
  const double qf = C[first].qf;
  int best = 1;
  double ba = -1.0;
  for (int k = 1; k <= S; ++k) {
    double acc = xmul(xsub(1.0, prs[0]), qf);
    for (int m = 0; m < k; ++m) {
      const double nxt = m + 1 < k ? prs[m + 1] : 0.0;
      acc = xadd(acc, xmul(C[first + m].a, xsub(prs[m], nxt)));
    }
    if (acc > ba) {
      best = k;
      ba = acc;
    }
  }
  return best;
}

// OracleStaticPolicy.begin (policies.py:221-265) for one stream per block:
// every candidate evaluated exactly over every input of the call's step range
// (plain running sums in step order, as the reference), then the
// lexicographic key (eligible first; objective, violations, power, dnn,
// stage).  Writes the chosen CANDIDATE index to policy_aux.
__global__ void static_choice_kernel(const BaseParams P) {
  const long long stream = P.stream_begin + blockIdx.x;
  if (stream >= P.stream_end || P.st.policy_aux[stream] >= 0) return;
  const DevTable& T = P.T;
  const AlertTrace& tr = P.tr;
  const long long row = tr.stream_row ? tr.stream_row[stream] : stream;
  // begin() sees the spec in force at the call's first step (goal changes)
  const int ng = tr.n_goal_segments ? tr.n_goal_segments[row] : 0;
  const int si = ng ? tr.goal_seg_spec[row * (long long)tr.max_goal_segments +
                                       goal_seek(tr, row * (long long)tr.max_goal_segments, ng, 0, P.step_begin)]
                    : (P.stream_spec ? P.stream_spec[stream] : (int)(stream % P.n_specs));
  const SpecDev sp = P.specs[si];
  const double goal = xsub(sp.t_goal, sp.oh);  // policies.py:227 (no 1 ms floor)
  const double period = xadd(goal, sp.oh);
  const long long n_in = P.step_end - P.step_begin;
  // per-thread best: (eligible, k1, k2, tie key, cell)
  int b_el = 0, b_cell = -1;
  double b_k1 = 0.0, b_k2 = 0.0;
  uint32_t b_tk = 0xFFFFFFFFu;
  const int nseg = tr.n_segments[row];
  const long long seg0 = row * tr.max_segments;
  for (int c = threadIdx.x; c < T.n_cells; c += blockDim.x) {
    int lv = 0, av = 0, ev = 0;
    double te = 0.0, ta = 0.0;
    int seg = 0;
    while (seg + 1 < nseg && P.step_begin >= tr.seg_end[seg0 + seg]) ++seg;
    int cur_end = seg + 1 < nseg ? tr.seg_end[seg0 + seg] : 0x7fffffff;
    double idle = tr.seg_idle[seg0 + seg];
    for (long long n = P.step_begin; n < P.step_end; ++n) {
      if (n >= cur_end) {
        while (seg + 1 < nseg && n >= tr.seg_end[seg0 + seg]) ++seg;
        cur_end = seg + 1 < nseg ? tr.seg_end[seg0 + seg] : 0x7fffffff;
        idle = tr.seg_idle[seg0 + seg];
      }
      const Outcome o = execute_measure(T.cellB, T.c64, &sp, c, base_s(tr, row, n), goal, period, idle);
      lv += o.vl;
      av += o.va;
      ev += o.ve;
      te = xadd(te, o.energy);
      ta = xadd(ta, o.delivered);
    }
    const double mean_obj = sp.mode == ALERT_MODE_MIN_ENERGY ? xdiv(te, (double)n_in) : -xdiv(ta, (double)n_in);
    const int mx = max(lv, max(av, ev));
    const int el = (double)mx <= xmul(0.10, (double)n_in);
    const double tv = (double)(lv + av + ev);
    const double k1 = el ? mean_obj : tv, k2 = el ? tv : mean_obj;
    const uint32_t tk = __float_as_uint(T.cellB[c].y);  // power << 20 | dnn << 8 | stage
    bool less;
    if (b_cell < 0) less = true;
    else if (el != b_el) less = el;
    else if (k1 != b_k1) less = k1 < b_k1;
    else if (k2 != b_k2) less = k2 < b_k2;
    else less = tk < b_tk;
    if (less) {
      b_el = el; b_k1 = k1; b_k2 = k2; b_tk = tk; b_cell = c;
    }
  }
  // block argmin (fixed tree, full key: unique winner)
  __shared__ double s_k1[256], s_k2[256];
  __shared__ int s_el[256], s_cell[256];
  __shared__ uint32_t s_tk[256];
  s_k1[threadIdx.x] = b_k1; s_k2[threadIdx.x] = b_k2; s_el[threadIdx.x] = b_el;
  s_cell[threadIdx.x] = b_cell; s_tk[threadIdx.x] = b_tk;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const int o = threadIdx.x + w;
      bool take = false;
      if (s_cell[o] >= 0) {
        if (s_cell[threadIdx.x] < 0) take = true;
        else if (s_el[o] != s_el[threadIdx.x]) take = s_el[o];
        else if (s_k1[o] != s_k1[threadIdx.x]) take = s_k1[o] < s_k1[threadIdx.x];
        else if (s_k2[o] != s_k2[threadIdx.x]) take = s_k2[o] < s_k2[threadIdx.x];
        else take = s_tk[o] < s_tk[threadIdx.x];
      }
      if (take) {
        s_k1[threadIdx.x] = s_k1[o]; s_k2[threadIdx.x] = s_k2[o]; s_el[threadIdx.x] = s_el[o];
        s_cell[threadIdx.x] = s_cell[o]; s_tk[threadIdx.x] = s_tk[o];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) P.st.policy_aux[stream] = cell_cand(T.cellB[s_cell[0]]) | (s_el[0] << 16);
}

// The closed loop of a comparison scheme (simulator.run, simulator.py:461-507),
// one thread per stream, FP64 throughout.
template <int POL>
__global__ void __launch_bounds__(128) baseline_kernel(const BaseParams P) {
  const long long stream = P.stream_begin + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (stream >= P.stream_end) return;
  const DevTable& T = P.T;
  const Cell64* C = T.c64;
  const AlertTrace& tr = P.tr;
  const long long row = tr.stream_row ? tr.stream_row[stream] : stream;
  const int ng = tr.n_goal_segments ? tr.n_goal_segments[row] : 0;  // goal changes
  const long long gseg0 = row * (long long)tr.max_goal_segments;
  int gseg = ng ? goal_seek(tr, gseg0, ng, 0, P.step_begin) : 0;
  int gend = ng ? goal_end(tr, gseg0, ng, gseg) : 0x7fffffff;
  SpecDev sp = P.specs[ng ? tr.goal_seg_spec[gseg0 + gseg]
                          : (P.stream_spec ? P.stream_spec[stream] : (int)(stream % P.n_specs))];
  Filter f;
  f.mu = P.st.mu[stream];
  f.sigma2 = P.st.sigma2[stream];
  f.k_gain = P.st.k_gain[stream];
  f.q_noise = P.st.q_noise[stream];
  f.innov = P.st.innov[stream];
  f.phi = P.st.phi[stream];
  f.m_var = P.st.m_var[stream];
  bool k_valid = false;
  int ik = -1;  // idle-filter gain table unused here (division path)
  double budget = P.st.group_budget[stream];
  int count = P.st.group_count[stream];
  int aux = P.st.policy_aux ? P.st.policy_aux[stream] : -1;
  const int Pw = T.n_powers;
  if (POL == ALERT_POLICY_NO_COORD && aux < 0) aux = T.app_stages | ((Pw - 1) << 8);  // policies.py:385-386
  const int static_cell = POL == ALERT_POLICY_ORACLE_STATIC ? T.cell_of_cand[aux & 0xFFFF] : -1;
  const bool static_ok = POL == ALERT_POLICY_ORACLE_STATIC && (aux >> 16) != 0;  // eligible

  const int nseg = tr.n_segments[row];
  const long long seg0 = row * tr.max_segments;
  int seg = 0;
  while (seg + 1 < nseg && P.step_begin >= tr.seg_end[seg0 + seg]) ++seg;
  int cur_end = seg + 1 < nseg ? tr.seg_end[seg0 + seg] : 0x7fffffff;
  int phase = tr.seg_phase[seg0 + seg];
  double idle = tr.seg_idle[seg0 + seg];

  double* agg = P.out.agg ? P.out.agg + stream * ALERT_AGG_FIELDS : nullptr;
  TileAgg G{};
  if (agg) {
    G.e = agg[ALERT_AGG_ENERGY]; G.ec = agg[ALERT_AGG_ENERGY_C];
    G.a = agg[ALERT_AGG_ACC]; G.ac = agg[ALERT_AGG_ACC_C];
    open_segment(G, agg, phase, false);
  }
  for (long long n = P.step_begin; n < P.step_end; ++n) {
    if (n >= cur_end) {
      if (agg) flush_segment(G, agg, phase, false);
      while (seg + 1 < nseg && n >= tr.seg_end[seg0 + seg]) ++seg;
      cur_end = seg + 1 < nseg ? tr.seg_end[seg0 + seg] : 0x7fffffff;
      phase = tr.seg_phase[seg0 + seg];
      idle = tr.seg_idle[seg0 + seg];
      if (agg) open_segment(G, agg, phase, false);
    }
    if (n >= gend) {  // goal change (policy.spec swapped)
      gseg = goal_seek(tr, gseg0, ng, gseg, n);
      gend = goal_end(tr, gseg0, ng, gseg);
      sp = P.specs[tr.goal_seg_spec[gseg0 + gseg]];
    }
    double goal, period;  // adjust_goal (selector.py:48-70), simulator.py:473-483
    if (sp.group_size > 0) {
      if (count == 0) {
        budget = xmul((double)sp.group_size, sp.t_goal);
        count = sp.group_size;
      }
      goal = py_max(xsub(xdiv(budget, (double)count), sp.oh), 0.001);
      period = xadd(goal, sp.oh);
    } else {
      goal = sp.goal0;
      period = sp.period0;
    }
    int cell;
    bool feasible = true;
    if (POL == ALERT_POLICY_ORACLE_STATIC) {
      cell = static_cell;
      feasible = static_ok;
    } else if (POL == ALERT_POLICY_SYS_ONLY) {
      cell = T.sys_cells[cheapest_power(T, C, f, goal, [&](int j) { return T.sys_cells[j]; }, &feasible)];
    } else if (POL == ALERT_POLICY_APP_ONLY) {
      cell = T.app_first[Pw - 1] + best_stage(C, T.app_first[Pw - 1], T.app_stages, f, goal) - 1;
    } else {  // no-coord: stage for the old power, power for the old stage
      const int st_old = aux & 0xff, pj_old = aux >> 8;
      const int st = best_stage(C, T.app_first[pj_old], T.app_stages, f, goal);
      const int pj = cheapest_power(T, C, f, goal, [&](int j) { return T.app_first[j] + st_old - 1; });
      aux = st | (pj << 8);
      cell = T.app_first[pj] + st - 1;
    }
    int exec_cell = cell;
    if (P.out.forced) {
      const int fc = P.out.forced[stream * P.out.stream_stride + n * P.out.step_stride];
      if (fc >= 0) exec_cell = T.cell_of_cand[fc];
    }
    const Outcome o = execute_measure(T.cellB, C, &sp, exec_cell, base_s(tr, row, n), goal, period, idle);
    if (POL != ALERT_POLICY_ORACLE_STATIC) {  // observe: policies.py:315-318, :359-360, :430-439
      slowdown_update(P.cfg, f, o.fb_latency, o.fb_t_prof, k_valid);
      if (POL != ALERT_POLICY_APP_ONLY)
        idle_update(P.cfg, f, py_min(1.0, xdiv(idle, C[exec_cell].cap)), ik, -1, nullptr, nullptr);
    }
    if (sp.group_size > 0) {
      budget = xsub(budget, o.latency);
      count -= 1;
    }
    const AlertOutputs& out = P.out;
    if (out.fb_latency) {
      const long long oidx = stream * out.stream_stride + n * out.step_stride;
      out.fb_latency[oidx] = o.fb_latency;
      out.fb_t_prof[oidx] = o.fb_t_prof;
      if (out.plan_goal) out.plan_goal[oidx] = goal;
      if (out.phi) out.phi[oidx] = f.phi;
    }
    if (out.decision) {
      const long long oidx = stream * out.stream_stride + n * out.step_stride;
      out.decision[oidx] = pack_decision(cell_cand(T.cellB[cell]), 0, o, false, phase, feasible);
      if (out.record_dtype == ALERT_DTYPE_F64) {
        if (out.energy) static_cast<double*>(out.energy)[oidx] = o.energy;
        if (out.accuracy) static_cast<double*>(out.accuracy)[oidx] = o.delivered;
        if (out.latency) static_cast<double*>(out.latency)[oidx] = o.latency;
        if (out.mu) static_cast<double*>(out.mu)[oidx] = f.mu;
        if (out.sigma2) static_cast<double*>(out.sigma2)[oidx] = f.sigma2;
      } else {
        if (out.energy) static_cast<float*>(out.energy)[oidx] = (float)o.energy;
        if (out.accuracy) static_cast<float*>(out.accuracy)[oidx] = (float)o.delivered;
        if (out.latency) static_cast<float*>(out.latency)[oidx] = (float)o.latency;
        if (out.mu) static_cast<float*>(out.mu)[oidx] = (float)f.mu;
        if (out.sigma2) static_cast<float*>(out.sigma2)[oidx] = (float)f.sigma2;
      }
    }
    if (agg) {
      neumaier(G.e, G.ec, o.energy);
      neumaier(G.a, G.ac, o.delivered);
      neumaier(G.pe, G.pec, o.energy);
      neumaier(G.pa, G.pac, o.delivered);
      G.dn += 1;
      G.dvl += o.vl; G.dva += o.va; G.dve += o.ve;
    }
  }
  P.st.mu[stream] = f.mu;
  P.st.sigma2[stream] = f.sigma2;
  P.st.k_gain[stream] = f.k_gain;
  P.st.q_noise[stream] = f.q_noise;
  P.st.innov[stream] = f.innov;
  P.st.phi[stream] = f.phi;
  P.st.m_var[stream] = f.m_var;
  P.st.group_budget[stream] = budget;
  P.st.group_count[stream] = count;
  if (P.st.policy_aux) P.st.policy_aux[stream] = aux;
  if (agg) {
    flush_segment(G, agg, phase, false);
    const double steps = (double)(P.step_end - P.step_begin);
    agg[ALERT_AGG_N] += steps;
    agg[ALERT_AGG_ENERGY] = G.e; agg[ALERT_AGG_ENERGY_C] = G.ec;
    agg[ALERT_AGG_ACC] = G.a; agg[ALERT_AGG_ACC_C] = G.ac;
    agg[ALERT_AGG_LEVEL0] += steps;  // the comparison schemes never fall back (level NONE)
  }
}

// SysOnly / AppOnly / NoCoord / OracleStatic .decide for n streams (one
// thread each) from their filter state and plan goal: the same device
// functions as the fused loop.  No-coord writes its new (stage, power) memory.
__global__ void baseline_decide_kernel(const DevTable T, const SpecDev* specs, int n_specs, const int32_t* stream_spec,
                                       AlertState st, const double* plan_goal, int policy, uint32_t* decision,
                                       long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  (void)specs; (void)n_specs; (void)stream_spec;  // the schemes read only the plan goal (policies.py:298-428)
  const Cell64* C = T.c64;
  Filter f;
  f.mu = st.mu[i];
  f.sigma2 = st.sigma2[i];
  f.phi = st.phi[i];
  const double goal = plan_goal[i];
  const int Pw = T.n_powers;
  int cell;
  bool feasible = true;
  if (policy == ALERT_POLICY_ORACLE_STATIC) {
    const int aux = st.policy_aux[i];
    cell = T.cell_of_cand[aux & 0xFFFF];
    feasible = (aux >> 16) != 0;
  } else if (policy == ALERT_POLICY_SYS_ONLY) {
    cell = T.sys_cells[cheapest_power(T, C, f, goal, [&](int j) { return T.sys_cells[j]; }, &feasible)];
  } else if (policy == ALERT_POLICY_APP_ONLY) {
    cell = T.app_first[Pw - 1] + best_stage(C, T.app_first[Pw - 1], T.app_stages, f, goal) - 1;
  } else {
    int aux = st.policy_aux[i];
    if (aux < 0) aux = T.app_stages | ((Pw - 1) << 8);  // policies.py:385-386
    const int st_old = aux & 0xff, pj_old = aux >> 8;
    const int stg = best_stage(C, T.app_first[pj_old], T.app_stages, f, goal);
    const int pj = cheapest_power(T, C, f, goal, [&](int j) { return T.app_first[j] + st_old - 1; });
    st.policy_aux[i] = stg | (pj << 8);
    cell = T.app_first[pj] + stg - 1;
  }
  decision[i] = (uint32_t)cell_cand(T.cellB[cell]) | ((uint32_t)feasible << 30);
}

}  // namespace alert
