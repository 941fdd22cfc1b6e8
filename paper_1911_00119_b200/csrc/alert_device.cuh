// alert_device.cuh — device side of the B200 ALERT scheduling step.
//
// One "tile" of W lanes (W = 1..32, a cooperative-groups partition of a warp)
// owns one stream.  Per step the tile
//   1. adjusts the goal                 selector.py:48-70, simulator.py:473-483
//   2. scans every candidate in FP32    predictor.py:147-197 + selector.py:102-131
//      (Phi via erff on the FMA/MUFU pipes, running top-2 per fallback level,
//      constraint-boundary uncertainty), lanes striding over candidates,
//      then merges lanes with shuffles;
//   3. re-ranks in FP64 — with the reference's exact formulas and operation
//      order — only when the FP32 top-2 gap or a constraint margin is inside
//      the FP32 error bound (near-tie), so decisions equal the FP64 reference;
//   4. executes / measures / observes in FP64   simulator.py:249-382,
//      estimator.py:59-127, keeping the filter state in registers.
//
// Candidates are stored as "cells" (one per (dnn, power, target stage)); the
// table is reordered so traditional cells come first (flat loop) and anytime
// DNNs follow as columns of consecutive stages (the telescoping expected
// accuracy, predictor.py:100-108, becomes a running FMA along the column).
#pragma once

#include <cooperative_groups.h>
#include <cstdint>
#include <math_constants.h>

#include "../../include/alert_b200.h"

namespace alert {

namespace cg = cooperative_groups;

constexpr float kInfF = __builtin_huge_valf();
constexpr double kInf = __builtin_huge_val();
constexpr float kEps = 1.1920929e-07f;  // 2^-23
constexpr double kSqrt2 = 1.4142135623730951;  // math.sqrt(2.0), predictor.py:21

// --------------------------------------------------------------------------
// device table
struct DevTable {
  int n_cells;      // == number of candidates
  int n_trad;       // cells [0, n_trad) are traditional, one per (dnn, power)
  int n_any_cols;   // anytime columns (dnn, power) after the traditional cells
  int n_powers;
  const float4* cellA;    // {1/t, cap*t, d = a_k - a_{k-1} (a_0 = q_fail), q_fail}   FP32 scan
  const float4* cellB;    // {t, tie-key, candidate | stage << 16, rank(acc) | rank(q_fail) << 16}
  const int2* any_cols;   // {first cell, number of stages}
  const struct Cell64* c64;  // FP64 cell data (exact path), AoS
  const int* cell_of_cand;
  const double* power_cap64;  // [n_powers] caps by power index
  double phi0;            // min(1, p_idle_prof / max cap), policies.py:90
  int any_mono;           // every anytime column's t_prof is non-decreasing per stage
  // comparison schemes (alert_baselines.cuh): cells of the sys-only DNN per
  // power, first cell of the app-only / no-coord DNN's column per power
  // max-accuracy fast scan (fast_max_accuracy): units = traditional cells and
  // anytime columns sorted by their accuracy upper bound, descending
  const int2* units;      // {first cell, n cells | anytime << 16}
  const float* unit_lb;   // lower bound of any key of the unit: 2 - bound - 1e-5
  int n_units;
  // units flattened per cell (tables of <= 64 cells, else n_seq = 0), one
  // sequence per DNN-kinds filter (kinds 1, 2, 3 at offsets 0, n_seq, 2 n_seq):
  // cellA rows (.w = q_fail at a unit start, 0 after) and {unit lb, dead-group
  // multiplier, chain carry, k | cell << 8 | (skip to) - 1 << 16 | (chain out
  // to) - 1 << 24} (fast_max_accuracy_flat)
  const float4* useqA;
  const float4* useqM;
  int n_seq;       // the longest sequence (shared-memory slots)
  int n_seqk[4];   // length per kinds (index 1..3)
  const float4* trad_rows;  // min-energy row mode: {dnn bits, min cap * t, max 1/t, 0}, min cap * t ascending
  const float4* or_rows;    // oracle max-accuracy: {first cell bits, accuracy rank bits, min t, 0}, rank ascending
  float cap_min;            // smallest cap (FP32)

  const int* sys_cells;   // [n_powers] or null
  const int* app_first;   // [n_powers] or null
  int app_stages;
  float cap_max;          // largest cap (FP32 error bound of the oracle scan)
};

// FP64 data of one cell for the exact path: profiled latency of the cell's
// stage at its power, stage accuracy, q_fail of its DNN, cap of its power.
struct Cell64 {
  double t, a, qf, cap;
};

// Device form of one AlertSpec, built on the host: the FP64 fields of the
// reference spec, the per-stream constants of the step loop (goal and period
// without groups, selector.py:48-70 / simulator.py:479-483, computed with the
// reference's operations), and FP32 copies for the scan.
struct SpecDev {
  double t_goal, e_goal, q_goal, pr_th, zq, oh, goal0, period0;
  float q_f, e_f, th_f, zq_f;
  int mode, has_pr, group_size;
  int rank_q;  // delivered >= q_goal  <=>  accuracy rank < rank_q (oracle scan)
};

// cellB field accessors
__device__ __forceinline__ int cell_cand(const float4& B) { return __float_as_uint(B.z) & 0xFFFF; }
__device__ __forceinline__ int cell_stage(const float4& B) { return __float_as_uint(B.z) >> 16; }
__device__ __forceinline__ int cell_rank_a(const float4& B) { return __float_as_uint(B.w) & 0xFFFF; }
__device__ __forceinline__ int cell_rank_qf(const float4& B) { return __float_as_uint(B.w) >> 16; }

// Exact FP64 helpers: no FMA contraction, Python's min/max semantics.
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xdiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double py_max(double a, double b) { return (b > a) ? b : a; }
__device__ __forceinline__ double py_min(double a, double b) { return (b < a) ? b : a; }

// Neumaier step exactly as CPython 3.12 sum() (bltinmodule.c): its
// correction (s - t) + x or (x - t) + s is the EXACT rounding error of s + x
// (Fast2Sum on the larger operand), which TwoSum yields without the compare
// and selects — bit-identical, shorter dependency chain.
__device__ __forceinline__ void neumaier(double& s, double& c, double x) {
  const double t = xadd(s, x);
  const double bp = xsub(t, s);
  const double ap = xsub(t, bp);
  c = xadd(c, xadd(xsub(s, ap), xsub(x, bp)));
  s = t;
}

// Standard normal CDF in FP32 from x = z / sqrt(2): Phi = 1 - erfc(a)/2 for
// x >= 0 else erfc(a)/2, a = |x>, one branch-free formula (phi32_x below):
// FFMA + RCP + 4 FFMA (immediate coefficients) + FMUL + FFMA + EX2 + 2 FMUL +
// FADD/FSEL.  Absolute error bound used by the near-tie logic (checked on the
// GPU against FP64, tests/test_gpu_parity.py::test_phi32_error_bound):
#define ALERT_PHI32_ERR_EPS 4.0f  // in units of 2^-23
// Shared-memory padding (rows of the FP32 cell table and column descriptors)
// that lets look-ahead loads run past the end without clamping: 2 chunks of 4
// cells at the widest tile (32 lanes).
#define ALERT_SMEM_PAD 256
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// Abramowitz & Stegun 7.1.26: erfc(a) = t (a1 + t(a2 + t(a3 + t(a4 + t a5)))) e^{-a^2},
// t = 1/(1 + p a), |error| <= 1.5e-7 absolute — absolute accuracy is all the
// scan needs (probabilities enter accuracies and thresholds additively).
__device__ __forceinline__ float phi32_x(float x) {
  const float a = fabsf(x);
  const float t = rcp_approx(fmaf(0.3275911f, a, 1.0f));
  float p = fmaf(t, 1.061405429f, -1.453152027f);
  p = fmaf(t, p, 1.421413741f);
  p = fmaf(t, p, -0.284496736f);
  p = fmaf(t, p, 0.254829592f);
  const float al = a * 1.44269504088896341f;
  const float e = ex2_approx(fmaf(-al, a, -1.0f));  // e^{-a^2} / 2
  const float h = (p * t) * e;                      // erfc(a) / 2
  // Phi = 1/2 + sign(x) (1/2 - h): copysign is one LOP3, the rest FMA-pipe work
  const float half_sgn = __uint_as_float((__float_as_uint(x) & 0x80000000u) | 0x3f000000u);
  return fmaf(half_sgn, fmaf(-2.0f, h, 1.0f), 0.5f);
}

// deadline_probability, exact reference arithmetic (predictor.py:48-65).
__device__ __forceinline__ double phi64(double goal, double mu, double sig, double t) {
  double mean = xmul(mu, t);
  double sd = xmul(sig, t);
  if (sd == 0.0) return mean <= goal ? 1.0 : 0.0;
  double x = xdiv(xsub(goal, mean), sd);
  return xmul(0.5, xadd(1.0, erf(xdiv(x, kSqrt2))));
}

// --------------------------------------------------------------------------
// per-step context shared by the lanes of a tile
struct StepCtx {
  // FP64 state (exact path)
  double mu, sig, phi, goal, zq;
  const SpecDev* spec;
  const Cell64* c64;  // FP64 cell data (shared memory when it fits)
  // FP32 scan inputs: x = (goal/t - mu) * inv_sig_s  (= z / sqrt 2),
  //                   E = (cap t) * max(mu_e, phig / t + ompmu)
  float goal_f, mu_f, inv_sig_s, mu_e, ompmu, phig, sig_f;
  // FP32 error bounds
  float d_pr, d_acc, d_erel;
  // thresholds with margins
  float q_hi, q_lo, th_hi, th_lo, e_hi, e_lo;
  bool fp64_all;
  unsigned sv;   // shared-space address of the tile's per-cell FP32 objectives
  bool has_sv;   // stored objectives enabled
  // min-energy fast scan (fast_min_energy): per-step feasibility thresholds
  // of the traditional DNNs, tile-shared, element d at tT[d * tS]
  bool fast;
  const float* tT;
  int tS;
  const float4* sF;  // traditional cells {1/t, cap t, byte offset of the DNN's threshold in tT, 0}
  const float* zrow; // row mode (large tables): the spec's z' per traditional DNN in trad_rows order (global, L1)
  const unsigned* wst;  // per 32-cell window of anytime cells: column-start bits (shared)
  bool any_window;      // ALERT_FLAG_ANY_WINDOW: two-pass window for anytime cells (A/B)
  const int2* su;       // max-accuracy fast scan: units / key lower bounds staged in shared memory
  const float* slb;
  const float4* sqA;    // the kinds' T.useqA / T.useqM sequence staged in shared memory (or null)
  const float4* sqM;
  int n_seq;            // its length
  float hs, hm;      // T_d = fma(z'_d, hs, hm)
  float Tpr;     // same for the pr_threshold z-bound (anytime cells)
};

__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Per-step scan context.  Only FP32 work here: the FP64 sigma (sqrt) is
// computed lazily by ensure_fp64() when the re-rank needs exact values.
__device__ __forceinline__ void make_ctx(StepCtx& x, const SpecDev* sp, const Cell64* c64, double mu,
                                         double sigma2, double phi, double goal, bool fp64_all) {
  x.spec = sp;
  x.c64 = c64;
  x.sv = 0;
  x.has_sv = false;
  x.fast = false;
  x.tT = nullptr;
  x.tS = 0;
  x.sF = nullptr;
  x.zrow = nullptr;
  x.wst = nullptr;
  x.su = nullptr;
  x.slb = nullptr;
  x.sqA = nullptr;
  x.sqM = nullptr;
  x.n_seq = 0;
  x.any_window = false;
  x.hs = x.hm = 0.f;
  x.Tpr = -kInfF;
  x.mu = mu;
  x.sig = sigma2;  // holds sigma2 until ensure_fp64()
  x.phi = phi;
  x.goal = goal;
  x.zq = sp->zq;
  x.goal_f = (float)goal;
  x.mu_f = (float)mu;
  const float s2f = (float)sigma2;
  const float inv_sig = rsqrt_approx(s2f);  // MUFU.RSQ, rel. error <= 2 ulp
  x.inv_sig_s = inv_sig * 0.70710678118654752f;
  const float sig_f = s2f * inv_sig;
  x.sig_f = sig_f;
  x.mu_e = sp->has_pr ? fmaf(sp->zq_f, sig_f, x.mu_f) : x.mu_f;  // predictor.py:140
  const float phi_f = (float)phi;
  x.ompmu = (1.0f - phi_f) * x.mu_e;
  x.phig = phi_f * x.goal_f;
  const float r = fabsf(x.mu_f) * inv_sig;
  // |dPhi| <= eps*(1.0 + 0.6*mu/sigma) from the rounding of z (incl. the
  // approximate rsqrt), plus the Phi32 evaluation error, times 2 for safety.
  x.d_pr = 2.0f * kEps * (1.0f + 0.6f * r + ALERT_PHI32_ERR_EPS);
  x.d_acc = x.d_pr + 8.0f * kEps;
  x.d_erel = 12.0f * kEps;
  x.fp64_all = fp64_all || !(s2f > 0.0f) || !isfinite(inv_sig) || !isfinite(x.d_pr) ||
               !(fabsf(x.mu_e) < 1e30f) || !(x.mu_e >= 0.0f);
  x.q_hi = sp->q_f + x.d_acc;
  x.q_lo = sp->q_f - x.d_acc;
  x.th_hi = sp->th_f + x.d_pr;
  x.th_lo = sp->th_f - x.d_pr;
  x.e_hi = sp->e_f * (1.0f - x.d_erel);  // sure: E <= e_hi
  x.e_lo = sp->e_f * (1.0f + x.d_erel);  // possible: E <= e_lo
}

// sigma = sigma2 ** 0.5 (estimator.py:42-44) for the exact FP64 path.
__device__ __forceinline__ void ensure_fp64(StepCtx& x) { x.sig = sqrt(x.sig); }

// --------------------------------------------------------------------------
// FP32 running top-2 per fallback level
struct Tracker {
  float b1, b2, un;
  int i1;
  __device__ __forceinline__ void init() { b1 = b2 = un = kInfF; i1 = -1; }
  __device__ __forceinline__ void push(float v, bool sure, bool unc, int c) {
    float vs = sure ? v : kInfF;
    b2 = fminf(b2, fmaxf(b1, vs));
    if (vs < b1) i1 = c;
    b1 = fminf(b1, vs);
    un = fminf(un, unc ? v : kInfF);
  }
  template <class Tile>
  __device__ __forceinline__ void merge(const Tile& tile) {
#pragma unroll
    for (int m = 1; m < Tile::num_threads(); m <<= 1) {
      float ob1 = tile.shfl_xor(b1, m), ob2 = tile.shfl_xor(b2, m), oun = tile.shfl_xor(un, m);
      int oi = tile.shfl_xor(i1, m);
      b2 = fminf(fminf(b2, ob2), fmaxf(b1, ob1));
      if (ob1 < b1 || (ob1 == b1 && (unsigned)oi < (unsigned)i1)) i1 = oi;
      b1 = fminf(b1, ob1);
      un = fminf(un, oun);
    }
  }
};

// FP64 lexicographic key (selector.py:87-91 / policies.py:142-146)
struct Key64 {
  double p0, p1;
  uint32_t tk;
  int cell;
  __device__ __forceinline__ void init() { p0 = p1 = kInf; tk = 0xFFFFFFFFu; cell = -1; }
  __device__ __forceinline__ bool less(const Key64& o) const {
    if (p0 != o.p0) return p0 < o.p0;
    if (p1 != o.p1) return p1 < o.p1;
    return tk < o.tk;
  }
  template <class Tile>
  __device__ __forceinline__ void merge(const Tile& tile) {
#pragma unroll
    for (int m = 1; m < Tile::num_threads(); m <<= 1) {
      Key64 o;
      o.p0 = tile.shfl_xor(p0, m);
      o.p1 = tile.shfl_xor(p1, m);
      o.tk = tile.shfl_xor(tk, m);
      o.cell = tile.shfl_xor(cell, m);
      if (o.cell >= 0 && (cell < 0 || o.less(*this))) *this = o;
    }
  }
};

// --------------------------------------------------------------------------
// FP64 exact prediction of one cell (predict_all, predictor.py:147-197)
struct Pred64 {
  double pr, acc, energy;
};

__device__ __forceinline__ Pred64 eval64(const DevTable& T, const StepCtx& x, int c) {
  Pred64 r;
  const int stage = cell_stage(T.cellB[c]);  // 0 = traditional
  const Cell64* C = x.c64;
  double t = C[c].t;
  double qf = C[c].qf;
  r.pr = phi64(x.goal, x.mu, x.sig, t);
  if (stage == 0) {
    r.acc = xadd(xmul(r.pr, C[c].a), xmul(xsub(1.0, r.pr), qf));  // accuracy_blend
  } else {
    // expected_accuracy_anytime (predictor.py:100-108), reference order,
    // streaming prs[m], prs[m+1] instead of materialising the list
    int first = c - (stage - 1);
    double p_cur = stage == 1 ? r.pr : phi64(x.goal, x.mu, x.sig, C[first].t);
    double acc = xmul(xsub(1.0, p_cur), qf);
    for (int m = 0; m < stage; ++m) {
      double p_next = (m + 1 == stage) ? 0.0
                      : (m + 2 == stage) ? r.pr
                                         : phi64(x.goal, x.mu, x.sig, C[first + m + 1].t);
      acc = xadd(acc, xmul(C[first + m].a, xsub(p_cur, p_next)));
      p_cur = p_next;
    }
    r.acc = acc;
  }
  double p = C[c].cap;
  if (x.spec->has_pr) {  // predict_energy_percentile, predictor.py:129-144
    double lat = xmul(xadd(x.mu, xmul(x.zq, x.sig)), t);
    double idle = py_max(0.0, xsub(x.goal, py_min(lat, x.goal)));
    r.energy = xadd(xmul(p, lat), xmul(xmul(x.phi, p), idle));
  } else {  // predict_energy_mean, predictor.py:111-126
    double lat = xmul(x.mu, t);
    r.energy = xadd(xmul(p, lat), xmul(xmul(x.phi, p), py_max(0.0, xsub(x.goal, lat))));
  }
  return r;
}

// feasibility at a fallback level (selector.py:73-84, _LEVELS :94-99)
__device__ __forceinline__ bool feasible64(const StepCtx& x, const Pred64& p, int level) {
  const SpecDev* s = x.spec;
  if (level < 2 && s->has_pr && p.pr < s->pr_th) return false;
  if (s->mode == ALERT_MODE_MAX_ACCURACY) return level != 0 || p.energy <= s->e_goal;
  return level == 2 || p.acc >= s->q_goal;
}

__device__ __forceinline__ Key64 key64(const StepCtx& x, const Pred64& p, int level, uint32_t tk, int c) {
  Key64 k;
  bool acc_mode = level == 2 || x.spec->mode == ALERT_MODE_MAX_ACCURACY;
  k.p0 = acc_mode ? -p.acc : p.energy;
  k.p1 = acc_mode ? p.energy : -p.acc;
  k.tk = tk;
  k.cell = c;
  return k;
}

// --------------------------------------------------------------------------
// The decision: FP32 scan, FP64 re-rank of near-ties.
struct Decision {
  int cell;
  int level;
  bool refined;
  bool full = false;  // the min-energy fast scan ran but could not certify
};

// Level-l objective in FP32: min-energy L0 -> E (relative bound), otherwise -acc.
template <int MODE>
__device__ __forceinline__ bool energy_objective(int level) {
  return MODE == ALERT_MODE_MIN_ENERGY && level == 0;
}

// Which fallback levels a pass tracks: the FP32 scan tracks the constrained
// levels (0, and 1 for max-accuracy); level 2 (no constraints, max accuracy)
// is scanned only when those are empty (rare), saving its tracker per cell.
enum { TRACK_CONSTRAINED = 0, TRACK_L2 = 1 };

template <int MODE, bool HAS_PR>
struct AlertScan {
  Tracker t[3];
  // refine-pass state
  int level;
  float cut;
  bool all;
  Key64 best;

  // FP32 classification of a cell at a level: sure / possible, objective value
  __device__ __forceinline__ void classify(const StepCtx& x, int lvl, float pr, float acc, float E,
                                           bool& sure, bool& poss, float& v) const {
    bool pr_s = !HAS_PR || lvl == 2 || pr >= x.th_hi;
    bool pr_p = !HAS_PR || lvl == 2 || pr >= x.th_lo;
    if (MODE == ALERT_MODE_MIN_ENERGY) {
      if (lvl == 2) { sure = true; poss = true; }
      else { sure = pr_s && acc >= x.q_hi; poss = pr_p && acc >= x.q_lo; }
    } else {
      if (lvl == 0) { sure = pr_s && E <= x.e_hi; poss = pr_p && E <= x.e_lo; }
      else { sure = pr_s; poss = pr_p; }
    }
    v = energy_objective<MODE>(lvl) ? E : -acc;
  }

  template <int TRACK>
  __device__ __forceinline__ void scan_cell(const StepCtx& x, int c, float pr, float acc, float E) {
    if (TRACK == TRACK_L2) {
      t[2].push(-acc, true, false, c);
      return;
    }
    bool s, p;
    float v;
    classify(x, 0, pr, acc, E, s, p, v);
    t[0].push(v, s, p && !s, c);
    bool p1 = false;
    if (MODE == ALERT_MODE_MAX_ACCURACY) {
      classify(x, 1, pr, acc, E, s, p1, v);
      t[1].push(v, s, p1 && !s, c);
    }
    // keep the level-0 objective (min-energy: E; max-accuracy: -acc, the same
    // for every level) with the "possible" bits of levels 0/1 in its two low
    // mantissa bits, for the re-rank pass
    // only the refine-heavy variant (max-accuracy with pr_threshold) stores
    if (MODE == ALERT_MODE_MAX_ACCURACY && HAS_PR && x.has_sv)
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(x.sv + 4u * c),
                   "r"((__float_as_uint(v) & ~3u) | (unsigned)p | ((unsigned)p1 << 1)));
  }

  __device__ __forceinline__ void refine_cell(const DevTable& T, const StepCtx& x, int c, float pr,
                                              float acc, float E, uint32_t tk) {
    bool relevant = all;
    if (!relevant) {
      bool s, p;
      float v;
      classify(x, level, pr, acc, E, s, p, v);
      relevant = p && v <= cut;
    }
    if (!relevant) return;
    Pred64 q = eval64(T, x, c);
    if (!feasible64(x, q, level)) return;
    Key64 k = key64(x, q, level, tk, c);
    if (best.cell < 0 || k.less(best)) best = k;
  }
};

template <int MODE>
__device__ __forceinline__ float cutoff(const StepCtx& x, int level, float b1) {
  if (!(b1 < kInfF)) return kInfF;
  if (energy_objective<MODE>(level)) return b1 + fabsf(b1) * (4.0f * x.d_erel) + 1e-30f;
  return b1 + 2.0f * x.d_acc;
}

// FP32 prediction of one cell: pr, expected accuracy (running along an
// anytime column: acc_k = acc_{k-1} + Phi_k * (a_k - a_{k-1})), energy.
__device__ __forceinline__ void predict32(const StepCtx& x, const float4& A, float base, float& pr,
                                          float& acc, float& E) {
  pr = phi32_x(fmaf(x.goal_f, A.x, -x.mu_f) * x.inv_sig_s);
  acc = fmaf(pr, A.z, base);
  E = A.y * fmaxf(x.mu_e, fmaf(x.phig, A.x, x.ompmu));
}

// One pass over the cells (PASS 0 = FP32 scan, 1 = refine at scan.level).
template <int PASS, int TRACK, int MODE, bool HAS_PR, class Tile>
__device__ __forceinline__ void cell_pass(const DevTable& T, const float4* __restrict__ sA,
                                          const float4* __restrict__ sB, const int2* __restrict__ sCol,
                                          const Tile& tile, const StepCtx& x, int kinds,
                                          AlertScan<MODE, HAS_PR>& S) {
  const int W = Tile::num_threads();
  const int lane = tile.thread_rank();
  const bool skip32 = PASS == 1 && S.all;
  // Traditional cells, U per chunk.  Two register sets (a, b) ping-pong so the
  // rows of the next chunk are loaded while the current one is evaluated,
  // without register copies; the shared table is padded by ALERT_SMEM_PAD rows
  // so look-ahead loads need no clamping.  Full double chunks first, then the
  // remainder one cell at a time.
  // One lane per stream (W = 1) with every kind admitted: ALL cells in one
  // flat loop; an anytime stage continues the running accuracy of the previous
  // cell (A.w < 0 marks "carry"), so columns need no inner loop.
  const bool flat = W == 1 && kinds == 3;
  const int n = flat ? T.n_cells : T.n_trad;
  if ((kinds & 1) && n > 0) {
    constexpr int U = 4;
    float carry = 0.f;
    auto cell = [&](const float4& A, int c) {
      float pr = 0.f, acc = 0.f, E = 0.f;
      const float base = A.w >= 0.0f ? A.w : carry;
      if (!skip32) predict32(x, A, base, pr, acc, E);
      carry = acc;
      if (PASS == 0) S.template scan_cell<TRACK>(x, c, pr, acc, E);
      else S.refine_cell(T, x, c, pr, acc, E, __float_as_uint(sB[c].y));
    };
    int c0 = lane;
    float4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = sA[c0 + u * W];
    for (; c0 + (2 * U - 1) * W < n; c0 += 2 * U * W) {
#pragma unroll
      for (int u = 0; u < U; ++u) b[u] = sA[c0 + (U + u) * W];
#pragma unroll
      for (int u = 0; u < U; ++u) cell(a[u], c0 + u * W);
#pragma unroll
      for (int u = 0; u < U; ++u) a[u] = sA[c0 + (2 * U + u) * W];
#pragma unroll
      for (int u = 0; u < U; ++u) cell(b[u], c0 + (U + u) * W);
    }
    // tail (< 2U cells): a[] already holds the next U rows
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c0 + u * W < n) cell(a[u], c0 + u * W);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c0 + (U + u) * W < n) cell(sA[c0 + (U + u) * W], c0 + (U + u) * W);
  }
  // Anytime columns: consecutive stages; the next stage row and the next
  // column descriptor are prefetched one step ahead.
  const int ncol = T.n_any_cols;
  if (!flat && (kinds & 2) && lane < ncol) {
    int2 cd = sCol[lane];
    for (int col = lane; col < ncol; col += W) {
      const int2 cd_next = sCol[col + W];  // sCol is padded too
      float4 A = sA[cd.x];
      float acc = A.w;
      for (int k = 0; k < cd.y; ++k) {
        const int c = cd.x + k;
        const float4 A_next = sA[c + 1];  // padded table: always in bounds
        float pr = 0.f, E = 0.f;
        if (!skip32) predict32(x, A, acc, pr, acc, E);
        if (PASS == 0) S.template scan_cell<TRACK>(x, c, pr, acc, E);
        else S.refine_cell(T, x, c, pr, acc, E, __float_as_uint(sB[c].y));
        A = A_next;
      }
      cd = cd_next;
    }
  }
}

// --------------------------------------------------------------------------
// Min-energy fast scan (level 0 of selector.py:102-131 in MINIMIZE_ENERGY).
//
// The level-0 objective is the energy, which needs no Phi.  Feasibility of a
// traditional cell, acc = Pr a + (1 - Pr) q_fail >= q_goal (and Pr >= pr_th),
// is a z-threshold per (spec, DNN): z >= Zlo_d (zlo_kernel, FP64, widened by
// the reference's rounding).  Per step, Zlo_d becomes an additive threshold
// T_d = H (mu + Zlo_d sigma - slack) so that, per cell, ONE sign-exact FFMA
//   pen = T_d - H goal / t
// is <= 0 for every cell the reference can find feasible; pen is folded into
// the energy's max (FMNMX3), so an excluded cell just gets a huge key.
// Anytime stages keep the running Phi-based expected accuracy (predict32) and
// are penalised from it the same way.  Keys are the energy with the cell's
// index within its row / column in the 6 low mantissa bits; a running top-2
// of keys (P1, P2) plus the row id of P1 is all the per-cell state.
//
// The decision is CERTIFIED only if P1's cell is surely feasible (FP32 check
// with the same margins as the full scan) and P2 exceeds P1 by more than the
// FP32 energy error and the key truncation: then every other feasible cell
// has a strictly larger FP64 energy and P1 is the reference's choice.
// Otherwise (near-ties, boundary cells, empty level 0) the full scan runs.
constexpr float kPenH = 1099511627776.0f;  // 2^40: sign-exact scaling of the penalty


__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// key = energy bits with the low 3 mantissa bits replaced by idx < 8: one
// LOP3 (select by the immediate mask; idx in a register)
__device__ __forceinline__ float pack_key(float e, unsigned idx) {
  unsigned r;
  asm("lop3.b32 %0, %1, 0xfffffff8, %2, 0xE2;" : "=r"(r) : "r"(__float_as_uint(e)), "r"(idx));
  return __uint_as_float(r);
}

struct Top2 {
  float p1, p2;
  int blk;
  __device__ __forceinline__ void push(float k) {
    p2 = fminf(p2, fmaxf(p1, k));
    p1 = fminf(p1, k);
  }
  __device__ __forceinline__ void push2(float a, float b) {
    const float lo = fminf(a, b), hi = fmaxf(a, b);
    p2 = fmin3(fmaxf(p1, lo), p2, hi);
    p1 = fminf(p1, lo);
  }
  // eight keys: their top 2 by a tournament (independent of the running
  // pair), then one merge — the loop-carried chain is 3 operations, not 10
  __device__ __forceinline__ void push8(const float (&k)[8]) {
    float lo[4], hi[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      lo[j] = fminf(k[2 * j], k[2 * j + 1]);
      hi[j] = fmaxf(k[2 * j], k[2 * j + 1]);
    }
    const float a1 = fminf(lo[0], lo[1]), a2 = fmin3(fmaxf(lo[0], lo[1]), hi[0], hi[1]);
    const float b1 = fminf(lo[2], lo[3]), b2 = fmin3(fmaxf(lo[2], lo[3]), hi[2], hi[3]);
    const float m1 = fminf(a1, b1), m2 = fmin3(fmaxf(a1, b1), a2, b2);
    p2 = fmin3(fmaxf(p1, m1), p2, m2);
    p1 = fminf(p1, m1);
  }
  template <class Tile>
  __device__ __forceinline__ void merge(const Tile& tile) {
#pragma unroll
    for (int m = 1; m < Tile::num_threads(); m <<= 1) {
      const float o1 = tile.shfl_xor(p1, m), o2 = tile.shfl_xor(p2, m);
      const int ob = tile.shfl_xor(blk, m);
      p2 = fmin3(p2, o2, fmaxf(p1, o1));
      if (o1 < p1 || (o1 == p1 && ob < blk)) blk = ob;
      p1 = fminf(p1, o1);
    }
  }
};

// Per-step thresholds T_d = H (z'_d sigma + mu') (and the pr_threshold
// bound for anytime cells): one FFMA per DNN.  z' = z - 20 eps |z| (zlo_kernel)
// and mu' = mu - 20 eps |mu| absorb the FP32 rounding of mu, sigma (rsqrt),
// goal, 1/t, the threshold FFMA and of z itself: for every cell
// the reference can find feasible, H goal / t >= T_d holds in FP32.
template <class Tile>
__device__ __forceinline__ void fast_prep(StepCtx& x, const Tile& tile, const float* zt, float* tT, int tS,
                                          int n_tdnn, float zpr, const float* zrow) {
  x.hs = x.sig_f * kPenH;
  x.hm = fmaf(-20.0f * kEps, fabsf(x.mu_f), x.mu_f) * kPenH;
  x.Tpr = fmaf(zpr, x.hs, x.hm);
  if (zrow) {  // row mode: thresholds computed per DNN inside the scan
    x.zrow = zrow;
    return;
  }
  // flat mode: the scan forms T_d = fma(z'_d, hs, hm) per cell from the
  // tile's z' copy (one FFMA; no per-step table, no store -> load dependency)
  (void)tT;
  (void)n_tdnn;
  x.tT = zt;
  x.tS = tS;
}

// FP32 sureness of one cell at min-energy level 0 (the full scan's margins).
__device__ __forceinline__ bool fast_sure(const DevTable& T, const float4* sA, const float4* sB, const StepCtx& x,
                                          int c, bool has_pr) {
  const int stage = cell_stage(sB[c]);
  const int first = stage == 0 ? c : c - (stage - 1);
  float acc = sA[first].w, pr = 0.f;
  for (int k = first; k <= c; ++k) {
    const float4 A = sA[k];
    pr = phi32_x(fmaf(x.goal_f, A.x, -x.mu_f) * x.inv_sig_s);
    acc = fmaf(pr, A.z, acc);
  }
  return acc >= x.q_hi && (!has_pr || pr >= x.th_hi);
}

template <bool HAS_PR, class Tile>
__device__ __forceinline__ bool fast_min_energy(const DevTable& T, const float4* __restrict__ sA,
                                                const float4* __restrict__ sB, const int2* __restrict__ sCol,
                                                const Tile& tile, const StepCtx& x, int kinds, Decision& d) {
  const int W = Tile::num_threads();
  const int lane = tile.thread_rank();
  const float mgH = -x.goal_f * kPenH;
  Top2 t{kInfF, kInfF, -1};
  // Traditional cells: flat loop, 8 cells in flight per lane; the key index
  // is the position u = (c / W) & 7 of the cell in its lane's chunk (staged in
  // sF[c].w), the chunk's first cell is recorded when P1 improves.  Each
  // cell's DNN threshold is read through the byte offset staged in sF[c].z.  Anytime columns: key index = stage,
  // recorded cell = the column's first stage.
  if ((kinds & 1) && x.zrow) {
    // row mode (large tables): DNN-major, lanes split the powers of a row in
    // chunks of 8 (masked at the row end); T_d from the spec's z' (L1), the
    // next DNN's z' in flight while the current row is scanned
    // Rows go by their smallest cap * t (m_r), ascending.  Every key of a
    // row is >= cap t max(mu_e, phig / t + ompmu) >= max(mu_e m_r, phig
    // cap_min + ompmu m_r) (phig, ompmu >= 0; the penalty only raises a key),
    // a bound increasing with m_r: once it (scaled by 1 - 4e-6 for the FP32
    // rounding and the packed key's truncation) reaches the lane's P2, no
    // cell of this or any later row can enter (P1, P2) and the scan stops.
    const int P = T.n_powers;
    const int n_tdnn = T.n_trad / P;
    const float mu_es = x.mu_e * (1.0f - 4e-6f);
    const bool lin = x.ompmu >= 0.0f && x.phig >= 0.0f;  // else the mu_e bound alone
    const float om_s = lin ? x.ompmu * (1.0f - 4e-6f) : 0.0f;
    const float ph_s = lin ? x.phig * T.cap_min * (1.0f - 4e-6f) : 0.0f;
    float4 rw = n_tdnn > 0 ? __ldg(T.trad_rows) : make_float4(0.f, 0.f, 0.f, 0.f);
    float zn = n_tdnn > 0 ? __ldg(x.zrow) : 0.f;  // z' in row order: independent of rw
    for (int r = 0; r < n_tdnn; ++r) {
      if (fmaxf(rw.y * mu_es, fmaf(om_s, rw.y, ph_s)) >= t.p2) break;
      const int dn = __float_as_int(rw.x);
      const float Td = fmaf(zn, x.hs, x.hm);
      // a row whose fastest cell already carries the deadline / accuracy
      // penalty (fma monotone in 1/t: so does every cell) is surely
      // infeasible at level 0 throughout: it can neither be a certified P1
      // nor undercut one, so it is not scanned
      const bool dead = fmaf(mgH, rw.z, Td) > 0.0f;
      if (r + 1 < n_tdnn) {
        rw = __ldg(T.trad_rows + r + 1);
        zn = __ldg(x.zrow + r + 1);
      }
      if (dead) continue;
      const float4* row = sA + dn * P;  // padded table: reads past the row are masked
      for (int p0 = lane; p0 < P; p0 += 8 * W) {
        const float s1 = t.p1;
        float k[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const float4 A = row[p0 + u * W];
          const float kk = pack_key(A.y * fmax3(x.mu_e, fmaf(x.phig, A.x, x.ompmu), fmaf(mgH, A.x, Td)), u);
          k[u] = p0 + u * W < P ? kk : kInfF;
        }
        t.push8(k);
        if (t.p1 != s1) t.blk = dn * P + p0;
      }
    }
  } else if (kinds & 1) {
    const float* zt = x.tT;  // the tile's z' per traditional cell, element c at zt[c * tS]
    const int tS = x.tS;
    const float4* sF = x.sF;
    auto key_of = [&](const float4& F, int c) {  // F.w = the cell's position in its chunk
      const float Td = fmaf(zt[c * tS], x.hs, x.hm);
      return pack_key(F.y * fmax3(x.mu_e, fmaf(x.phig, F.x, x.ompmu), fmaf(mgH, F.x, Td)), __float_as_uint(F.w));
    };
    const int n = T.n_trad;
    int c = lane;
    for (; c + 7 * W < n; c += 8 * W) {
      const float s1 = t.p1;
      float k[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) k[u] = key_of(sF[c + u * W], c + u * W);
      t.push8(k);
      if (t.p1 != s1) t.blk = c;
    }
    // remainder (< 8 cells) in quarter-chunks: positions 0-3 then 4-7 of the
    // last 8-group (keys carry the staged position, blk the group start)
    const int c8 = c;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (c < n) {
        const float s1 = t.p1;
        float k[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          // padded tables: reads past the end are masked (the z' index clamped)
          const float kk = key_of(sF[c + u * W], min(c + u * W, n - 1));
          k[u] = c + u * W < n ? kk : kInfF;
        }
        t.push2(k[0], k[1]);
        t.push2(k[2], k[3]);
        if (t.p1 != s1) t.blk = c8;
        c += 4 * W;
      }
    }
  }
  if (kinds & 2) {
    // Anytime columns after the traditional cells, with an exact skip: a
    // stage whose energy-only key is already >= P2 cannot change (P1, P2)
    // (the penalty only raises a key).  When every column's profiled latency
    // is non-decreasing with the stage (T.any_mono: the exact energy is then
    // non-decreasing, the FP32 keys within 4e-6 relative), a column whose
    // stage-0 key clears P2 by that margin on every lane of the warp is
    // skipped whole; in the others the Phi chain runs up to the last
    // stage some lane still needs.  Energies of later stages are rarely
    // competitive, so this is usually stage 0 of a few columns or nothing.
    const float qloH = x.q_lo * kPenH;
    const unsigned am = __activemask();
    const int rounds = (T.n_any_cols + W - 1) / W;
    auto ekey = [&](const float4& A, unsigned k) {
      return pack_key(A.y * fmaxf(x.mu_e, fmaf(x.phig, A.x, x.ompmu)), k);
    };
    auto eval = [&](const float4& A, float& acc, unsigned k) {
      const float pr = phi32_x(fmaf(x.goal_f, A.x, -x.mu_f) * x.inv_sig_s);
      acc = fmaf(pr, A.z, acc);
      float pen = fmaf(-kPenH, acc, qloH);
      if (HAS_PR) pen = fmaxf(pen, fmaf(mgH, A.x, x.Tpr));
      t.push(pack_key(A.y * fmax3(x.mu_e, fmaf(x.phig, A.x, x.ompmu), pen), k));
    };
    if (W == 1 && T.any_mono && !x.any_window) {
      // One lane per stream, stage latencies non-decreasing: a column whose
      // stage-0 energy-only key clears P2 (with the 4e-6 monotonicity margin)
      // is skipped whole, and a column stops at its first such stage — per
      // lane, no warp vote; usually no Phi at all (profiles/).
      const float sc = 1.0f - 4e-6f;
      const float mu_es = x.mu_e * sc, phigs = x.phig * sc, ompmus = x.ompmu * sc;
      for (int col = 0; col < T.n_any_cols; ++col) {
        const int2 cd = sCol[col];
        const float4 A0 = sA[cd.x];
        if (!(A0.y * fmaxf(mu_es, fmaf(phigs, A0.x, ompmus)) < t.p2)) continue;
        float acc = A0.w;
        for (int k = 0; k < cd.y; ++k) {
          const float4 A = k == 0 ? A0 : sA[cd.x + k];
          if (k > 0 && !(A.y * fmaxf(mu_es, fmaf(phigs, A.x, ompmus)) < t.p2)) break;
          const float before = t.p1;
          eval(A, acc, (unsigned)k);
          if (t.p1 != before) t.blk = cd.x;
        }
      }
    } else if (W == 1) {
      // One lane per stream: windows of 32 anytime cells.  Pass 1 (all cells,
      // independent): energy-only keys -> cells some lane of the warp needs
      // (key < P2); extended down to their column start (the Phi chain needs
      // the earlier stages).  Pass 2: the Phi chain over those cells only.
      // energy-only keys scaled by (1 - 4e-6): below P2 whenever the packed
      // key could be (truncation <= 7 ulp, FP32 rounding of the scaling)
      const float sc = 1.0f - 4e-6f;
      const float mu_es = x.mu_e * sc, phigs = x.phig * sc, ompmus = x.ompmu * sc;
      for (int c0 = T.n_trad; c0 < T.n_cells; c0 += 32) {
        const int nw = min(32, T.n_cells - c0);
        unsigned m = 0;
        for (int ub = 0; ub < nw; ub += 8) {
          unsigned b = 0;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 A = sA[c0 + ub + u];  // padded table; bits past the end are cleared below
            if (A.y * fmaxf(mu_es, fmaf(phigs, A.x, ompmus)) < t.p2) b |= 1u << u;
          }
          m |= b << ub;
        }
        if (nw < 32) m &= (1u << nw) - 1u;
        m = __reduce_or_sync(am, m);
        if (!m) continue;
        const unsigned st = x.wst[(c0 - T.n_trad) >> 5];  // column starts in this window
        // fill each needed cell down to its column start (the Phi chain needs
        // the earlier stages); a handful of iterations, warp-uniform
        unsigned need = 0;
        for (unsigned mm = m; mm;) {
          const int hb = 31 - __clz(mm);
          const unsigned below = hb == 31 ? ~0u : (2u << hb) - 1u;
          const unsigned sb = st & below;
          const int s0 = sb ? 31 - __clz(sb) : 0;
          need |= below & ~((1u << s0) - 1u);
          mm &= (1u << s0) - 1u;
        }
        // a window may start inside a column: its carry is rebuilt from the start
        float acc = 0.f;
        if (!(st & 1u) && (need & 1u)) {
          int cs = c0;
          while (sA[cs].w < 0.0f) --cs;
          acc = sA[cs].w;
          for (int c = cs; c < c0; ++c) {
            const float4 A = sA[c];
            acc = fmaf(phi32_x(fmaf(x.goal_f, A.x, -x.mu_f) * x.inv_sig_s), A.z, acc);
          }
        }
        while (need) {
          const int u = __ffs(need) - 1;
          need &= need - 1;
          const float4 A = sA[c0 + u];
          if (A.w >= 0.0f) acc = A.w;
          const float before = t.p1;
          eval(A, acc, (unsigned)(u & 7));
          if (t.p1 != before) t.blk = c0 + (u & ~7);
        }
      }
    } else
    for (int j0 = 0; j0 < rounds; j0 += 32) {
      const int jn = min(rounds, j0 + 32);
      unsigned m;
      if (T.any_mono) {
        m = 0;
#pragma unroll 4
        for (int j = j0; j < jn; ++j) {
          const int col = lane + j * W;
          // later stages: exact energy non-decreasing, FP32 keys within 4e-6 relative
          if (col < T.n_any_cols && ekey(sA[sCol[col].x], 0u) * (1.0f - 4e-6f) < t.p2) m |= 1u << (j - j0);
        }
        m = __reduce_or_sync(am, m);
      } else {
        m = jn - j0 == 32 ? ~0u : (1u << (jn - j0)) - 1u;
      }
      while (m) {
        const int j = j0 + __ffs(m) - 1;
        m &= m - 1;
        const int col = lane + j * W;
        const int2 cd = col < T.n_any_cols ? sCol[col] : make_int2(0, 0);
        int need = -1;
#pragma unroll
        for (int k = 0; k < ALERT_MAX_STAGES; ++k)
          if (k < cd.y && ekey(sA[cd.x + k], (unsigned)k) < t.p2) need = k;
        const int K = __reduce_max_sync(am, need);
        const float s1 = t.p1;
        float acc = sA[cd.x].w;
        for (int k = 0; k <= K && k < cd.y; ++k) eval(sA[cd.x + k], acc, (unsigned)k);
        if (t.p1 != s1) t.blk = cd.x;
      }
    }
  }
  t.merge(tile);
  if (!(t.p1 < kInfF) || t.blk < 0) return false;
  const float cut = t.p1 + t.p1 * (4.0f * x.d_erel + 3.1e-5f);  // 2^-15 >> truncation of both keys
  if (!(t.p2 > cut)) return false;
  const int idx = (int)(__float_as_uint(t.p1) & 7u);
  const int c = t.blk < T.n_trad ? t.blk + idx * W : t.blk + idx;
  if (!fast_sure(T, sA, sB, x, c, HAS_PR)) return false;
  d.cell = c;
  d.level = 0;
  d.refined = false;
  return true;
}

// --------------------------------------------------------------------------
// Max-accuracy fast scan (level 0 of selector.py:102-131 in MAXIMIZE_ACCURACY:
// Pr >= pr_th and E <= e_goal, objective (-acc, E, power, dnn, stage)).
//
// Units (traditional cells and anytime columns) are visited in descending
// order of their accuracy upper bound (max of q_fail and the stage
// accuracies: expected accuracy is a convex combination of them); keys are
// 2 - acc with the L0 constraints folded in as sign-exact penalties (pr via
// the z-bound T_pr, energy via E - e_lo), so the warp stops as soon as no
// remaining unit can reach the current second-best key P2.
//
// Certified when P1's cell is surely feasible and either
//  (b) P2 exceeds P1 by more than the FP32 accuracy error, or
//  (c) every key within that margin belongs to a cell whose deadline
//      probability is EXACTLY 1 in FP64 (z >= 8.6: erfc below 2^-53, so
//      0.5 (1 + erf) rounds to 1 and the expected accuracy equals the stage
//      accuracy bit for bit) of P1's accuracy class: the reference then ranks
//      them by energy, resolved here in FP32 unless the energies are within
//      their error bound.
// Otherwise the full scan runs.
constexpr float kExactOneX = 6.0811183f;  // z = 8.6 in units of z / sqrt 2

// erfc(x) for 0 <= x < ~9 with RELATIVE accuracy (Chebyshev-fitted
// exponent form, fractional error < 1.2e-7 in exact arithmetic; FP32
// evaluation adds a few ulp of the exponent): t = 1/(1 + x/2),
// erfc = t exp(-x^2 + P(t)).  ~14 instructions vs erfcf's ~50.
__device__ __forceinline__ float erfc_rel(float x) {
  const float t = rcp_approx(fmaf(0.5f, x, 1.0f));
  float p = fmaf(t, 0.17087277f, -0.82215223f);
  p = fmaf(t, p, 1.48851587f);
  p = fmaf(t, p, -1.13520398f);
  p = fmaf(t, p, 0.27886807f);
  p = fmaf(t, p, -0.18628806f);
  p = fmaf(t, p, 0.09678418f);
  p = fmaf(t, p, 0.37409196f);
  p = fmaf(t, p, 1.00002368f);
  p = fmaf(t, p, -1.26551223f);
  return t * ex2_approx(fmaf(-x, x, p) * 1.44269504088896341f);
}

template <bool HAS_PR, class Tile>
__device__ __forceinline__ bool fast_max_accuracy(const DevTable& T, const float4* __restrict__ sA,
                                                  const float4* __restrict__ sB, const Tile& tile,
                                                  const StepCtx& x, int kinds, Decision& d) {
  const int W = Tile::num_threads();
  const int lane = tile.thread_rank();
  const float mgH = -x.goal_f * kPenH;
  const float elH = -x.e_lo * kPenH;
  const int n_units = T.n_units;
  // units / key lower bounds: staged in shared memory for tables up to 1,024
  // units, else read through L1 (read-only path)
  const bool staged = x.su != nullptr;
  auto unit_at = [&](int u) { return staged ? x.su[u] : __ldg(T.units + u); };
  auto lb_at = [&](int u) { return staged ? x.slb[u] : __ldg(T.unit_lb + u); };
  // key of one cell, its energy and exact-one flag (running accuracy carried)
  auto cell_key = [&](const float4& A, float& acc, bool& one, unsigned k, float& E) {
    const float xz = fmaf(x.goal_f, A.x, -x.mu_f) * x.inv_sig_s;
    acc = fmaf(phi32_x(xz), A.z, acc);
    one = one && xz >= kExactOneX;
    E = A.y * fmaxf(x.mu_e, fmaf(x.phig, A.x, x.ompmu));
    float pen = fmaf(E, kPenH, elH);
    if (HAS_PR) pen = fmaxf(pen, fmaf(mgH, A.x, x.Tpr));
    return pack_key(fmaxf(2.0f - acc, pen), k);
  };
  Top2 t{kInfF, kInfF, -1};
  // pass 1: units in bound order; a lane stops at its first unit whose key
  // lower bound reaches its running P2 (sorted: no later unit can matter).
  // With the per-tile store (x.has_sv) every key is kept for the near-tie
  // pass, which then re-derives only the tails of the few tied cells.
  const bool store = W == 1 && x.has_sv;
  int u_end = lane;
  // the next unit and its bound are loaded one iteration ahead (their
  // latency hides behind the current unit)
  float lb_n = lane < n_units ? lb_at(lane) : kInfF;
  int2 un_n = lane < n_units ? unit_at(lane) : make_int2(0, 0);
  for (int u = lane; u < n_units; u += W) {
    const float lb = lb_n;
    const int2 un = un_n;
    if (u + W < n_units) {
      lb_n = lb_at(u + W);
      un_n = unit_at(u + W);
    }
    if (lb >= t.p2) break;
    u_end = u + W;
    if (!((kinds >> ((un.y >> 16) ? 1 : 0)) & 1)) continue;
    const int n = un.y & 0xFFFF;
    float acc = sA[un.x].w;
    bool one = true;
    for (int k = 0; k < n; ++k) {
      const float4 A = sA[un.x + k];
      // constraints first (no Phi): a cell that is surely infeasible at L0
      // cannot enter (P1, P2); with non-decreasing stage latencies every
      // later stage of the column is infeasible too (Pr falls, E grows —
      // the energy test then uses a 2 d_erel margin to absorb FP64 rounding)
      const float E0 = A.y * fmaxf(x.mu_e, fmaf(x.phig, A.x, x.ompmu));
      const float pp = HAS_PR ? fmaf(mgH, A.x, x.Tpr) : -kInfF;
      if (fmaxf(fmaf(E0, kPenH, elH), pp) > 0.0f) {
        if (store) asm volatile("st.shared.f32 [%0], %1;" ::"r"(x.sv + 4u * (un.x + k)), "f"(kInfF));
        const bool later_out = pp > 0.0f || E0 > x.e_lo * (1.0f + x.d_erel);
        if (T.any_mono && later_out) {
          for (int k2 = k + 1; k2 < n && store; ++k2)
            asm volatile("st.shared.f32 [%0], %1;" ::"r"(x.sv + 4u * (un.x + k2)), "f"(kInfF));
          break;
        }
        acc = fmaf(phi32_x(fmaf(x.goal_f, A.x, -x.mu_f) * x.inv_sig_s), A.z, acc);  // carry only
        one = false;
        continue;
      }
      float E;
      const float before = t.p1;
      const float key = cell_key(A, acc, one, (unsigned)k, E);
      if (store) asm volatile("st.shared.f32 [%0], %1;" ::"r"(x.sv + 4u * (un.x + k)), "f"(key));
      t.push(key);
      if (t.p1 != before) t.blk = un.x;
    }
  }
  t.merge(tile);
  if (!(t.p1 < 2.0f) || t.blk < 0) return false;  // P1 must be a possible cell (no penalty)
  const int c1 = t.blk + (int)(__float_as_uint(t.p1) & 7u);
  if (c1 >= T.n_cells) return false;
  // sureness of a cell at level 0: energy and deadline probability
  auto sure = [&](int c) {
    const float4 A = sA[c];
    const float E = A.y * fmaxf(x.mu_e, fmaf(x.phig, A.x, x.ompmu));
    if (!(E <= x.e_hi)) return false;
    if (!HAS_PR) return true;
    return phi32_x(fmaf(x.goal_f, A.x, -x.mu_f) * x.inv_sig_s) >= x.th_hi;
  };
  const float cut = t.p1 + 2.0f * x.d_acc + 4e-6f;  // + truncation of both keys
  if (t.p2 > cut) {  // (b) strict accuracy winner (keys distinct: blk is P1's unit)
    if (!sure(c1)) return false;
    d.cell = c1;
    d.level = 0;
    d.refined = false;
    return true;
  }
  {
    // (c') near-ties within P1's class (same DNN and
    // target stage) are ordered by the deadline-miss tail T = sum_m h_m d_m
    // (acc = a_k - T exactly; h_m = erfc(x_m) / 2, relatively accurate via
    // erfcf, 0 when x_m >= kExactOneX where FP64 rounds Pr to exactly 1):
    // the smaller tail wins unless the intervals T (1 -+ r) (r from the FP32
    // error of x_m) come within mrg (FP64 blend rounding and the 2^-53
    // quantisation of Pr); equal zero tails tie exactly and go by energy.
    const uint32_t ccls = __float_as_uint(sB[c1].y) & 0xFFFFFu;  // dnn << 8 | stage
    // FP64 accuracy of a k-stage chain: ~2k + 2 roundings of <= 2^-53 plus the
    // 2^-53 quantisation of each Pr (and erf's ulp): 1e-15 (2 + 2k) bounds the
    // difference of two such accuracies with room to spare
    const float mrg = 1e-15f * (2.0f + 2.0f * (float)max(1u, ccls & 0xFFu));
    bool ok1 = true;
    float ze1 = kInfF, ze2 = kInfF, bh = kInfF, bl = kInfF, lo2 = kInfF, nzlo = kInfF;
    int zc = -1, bc = -1;
    for (int u = lane; u < n_units; u += W) {
      if (lb_at(u) > cut) break;
      const int2 un = unit_at(u);
      if (!((kinds >> ((un.y >> 16) ? 1 : 0)) & 1)) continue;
      int n = un.y & 0xFFFF;
      if (store && u < u_end) {  // keys kept by pass 1: the chain only up to the last key <= cut
        int last = -1;
        for (int k = 0; k < n; ++k) {
          float kk;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(kk) : "r"(x.sv + 4u * (un.x + k)));
          if (kk <= cut) last = k;
        }
        if (last < 0) continue;
        n = last + 1;
      }
      float acc = sA[un.x].w, tail = 0.f, r = 0.f;
      bool one = true, bad = false;
      for (int k = 0; k < n; ++k) {
        const float4 A = sA[un.x + k];
        float E;
        const float xz = fmaf(x.goal_f, A.x, -x.mu_f) * x.inv_sig_s;
        const float key = cell_key(A, acc, one, (unsigned)k, E);
        if (!(xz >= kExactOneX)) {
          bad |= !(xz >= 0.0f) || !(A.z >= 0.0f);
          tail = fmaf(0.5f * erfc_rel(xz), A.z, tail);
          // relative error: FP32 x (propagated by d ln erfc / dx ~ 2x + 2),
          // the fit (1.2e-7) and the FP32 exponent (<= 40 ulp of 1 at x ~ 6)
          const float dx = 4.0f * kEps * (fmaf(x.goal_f, A.x, fabsf(x.mu_f)) * x.inv_sig_s + fabsf(xz));
          r = fmaxf(r, fmaf(2.0f * xz + 2.0f, dx, 1e-4f));
        }
        if (key > cut) continue;
        const int c = un.x + k;
        if (bad || (__float_as_uint(sB[c].y) & 0xFFFFFu) != ccls) ok1 = false;
        if (tail == 0.0f) {  // exact acc = a_k: energy decides among these
          ze2 = fminf(ze2, fmaxf(ze1, E));
          if (E < ze1) zc = c;
          ze1 = fminf(ze1, E);
        } else {
          const float hi = tail * (1.0f + r), lo = tail * (1.0f - r);
          nzlo = fminf(nzlo, lo);
          if (hi < bh) {
            lo2 = fminf(lo2, bl);
            bh = hi; bl = lo; bc = c;
          } else {
            lo2 = fminf(lo2, lo);
          }
        }
      }
    }
    // tile-wide merge: every lane ok; zero-tail energies (top-2 + cell);
    // nonzero tails: best by upper bound, the smallest lower bound of the rest
#pragma unroll
    for (int m = 1; m < W; m <<= 1) {
      ok1 = tile.shfl_xor((int)ok1, m) && ok1;
      const float o1 = tile.shfl_xor(ze1, m), o2 = tile.shfl_xor(ze2, m);
      const int oz = tile.shfl_xor(zc, m);
      ze2 = fmin3(ze2, o2, fmaxf(ze1, o1));
      if (o1 < ze1 || (o1 == ze1 && oz >= 0 && (zc < 0 || oz < zc))) zc = oz;
      ze1 = fminf(ze1, o1);
      const float obh = tile.shfl_xor(bh, m), obl = tile.shfl_xor(bl, m), olo2 = tile.shfl_xor(lo2, m);
      const int obc = tile.shfl_xor(bc, m);
      nzlo = fminf(nzlo, tile.shfl_xor(nzlo, m));
      lo2 = fminf(lo2, olo2);
      if (obh < bh || (obh == bh && obc >= 0 && (bc < 0 || obc < bc))) {
        lo2 = fminf(lo2, bl);
        bh = obh; bl = obl; bc = obc;
      } else {
        lo2 = fminf(lo2, obl);
      }
    }
    int w;
    if (!ok1) return false;
    if (zc >= 0) {  // zero tails win; nonzero ones must be strictly worse
      if (!(nzlo > mrg) || !(ze2 > ze1 + ze1 * (4.0f * x.d_erel) + 1e-30f)) return false;
      w = zc;
    } else {
      if (bc < 0 || !(lo2 > bh + mrg)) return false;
      w = bc;
    }
    if (!sure(w)) return false;
    d.cell = w;
    d.level = 0;
    d.refined = false;
    return true;
  }
}

// W = 1, up to 64 cells (the preset-sized tables): the same certified scan
// with the bound-ordered units flattened to one loop over their cells
// (T.useq, one sequence per DNN-kinds filter, so excluded units are simply
// absent), so every lane issues the same cell body each iteration instead of
// a divergent chain loop nested in a unit loop; a unit whose first cell fails
// the deadline-probability bound skips the rest of its DNN's group (units
// sorted by latency).  Pass 1 runs on until the next cell's unit bound
// exceeds both the running P2 and the running tie cut, and marks (64-bit mask
// over sequence positions) every key within the running cut: the final cut is
// never larger, so the near-tie pass (c') re-derives only the marked cells.
// The per-cell body is laid out for the FMA pipe: the sequence metadata
// {unit lb, dead-group multiplier, chain carry, k | cell << 8 | skip target
// << 16 | chain-out target << 24} needs no bit-field decoding on the key
// path, the running accuracy restarts by an FMA with the carry, and the
// P1 / P2 sentinels (2.5 > any feasible key 2 - acc) need no clamp.
template <bool HAS_PR>
__device__ __forceinline__ bool fast_max_accuracy_flat(const DevTable& T, const float4* __restrict__ sA,
                                                       const float4* __restrict__ sB, const StepCtx& x,
                                                       int kinds, Decision& d) {
  const float mgH = -x.goal_f * kPenH;
  const float elH = -x.e_lo * kPenH;
  const float elim = x.e_lo * (1.0f + x.d_erel);  // chain-out energy test (2 d_erel margin)
  const int n_seq = x.n_seq;
  // 32-bit shared addresses (no generic-to-shared conversion per cell)
  const unsigned aqa = (unsigned)__cvta_generic_to_shared(x.sqA);
  const unsigned aqm = (unsigned)__cvta_generic_to_shared(x.sqM);
  const unsigned aA = (unsigned)__cvta_generic_to_shared(sA);
  auto f4 = [](unsigned a) {
    float4 v;
    asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
  };
  auto meta_w = [&](int i) {
    unsigned v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(aqm + 16u * i + 12u));
    return v;
  };
  auto shl = [](unsigned v, unsigned s) {  // PTX shl clamps s >= 32 to 0 bits left
    unsigned r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(v), "r"(s));
    return r;
  };
  auto cell_at = [&](int c) { return f4(aA + 16u * c); };
  auto energy = [&](const float4& A) { return A.y * fmaxf(x.mu_e, fmaf(x.phig, A.x, x.ompmu)); };
  auto penalty = [&](const float4& A, float E) {
    const float pp = HAS_PR ? fmaf(mgH, A.x, x.Tpr) : -kInfF;
    return fmaxf(fmaf(E, kPenH, elH), pp);
  };
  const float dcut = 2.0f * x.d_acc + 4e-6f;  // tie cut above P1: + truncation of both keys
  float p1 = 2.5f, p2 = 2.5f, pd = 2.5f + dcut;
  int bi = -1;
  unsigned mlo = 0u, mhi = 0u;
  float acc = 0.0f;
  // per cell: the order-independent part (deadline penalty, Phi, energy),
  // then the running accuracy, the key, the top 2 and the marks in order.
  // (Two cells in flight per iteration measured 5% slower on c3: more
  // registers, and the jumps drop the second cell.)
  auto part = [&](const float4& A, float& pp, float& ph, float& E, float& pen) {
    pp = HAS_PR ? fmaf(mgH, A.x, x.Tpr) : -kInfF;
    ph = phi32_x(fmaf(x.goal_f, A.x, -x.mu_f) * x.inv_sig_s);
    E = energy(A);
    pen = fmaxf(fmaf(E, kPenH, elH), pp);
  };
  // the order-dependent part; returns the next index - 1 (i = no jump)
  auto take = [&](int i, const float4& A, const float4& M, float pp, float ph, float E, float pen) {
    const unsigned w = __float_as_uint(M.w);
    const bool skip = pp * M.y > 0.0f;  // unit start of a group the deadline bound kills
    acc = fmaf(acc, M.z, A.w);          // chain carry (0 at a unit start: restart at q_fail)
    acc = fmaf(ph, A.z, acc);
    // surely infeasible at L0 (see fast_max_accuracy): no key; with monotone
    // stage latencies the rest of the chain is out too (host: target = next
    // cell when latencies are not monotone)
    const bool out = skip || pen > 0.0f;
    int nxt = i;
    if (out && (pp > 0.0f || E > elim)) nxt = (int)(w >> 24);
    if (skip) nxt = (int)((w >> 16) & 0xFFu);
    const float key = out ? kInfF : pack_key(fmaxf(2.0f - acc, pen), w);
    if (key < p1) bi = i;
    // a new P1 more than the tie cut below the old one: every earlier key is
    // >= the old P1 > key + dcut >= the final cut, so their marks could only
    // fail the near-tie pass's key check after a chain re-derivation (c3 +3%)
    if (key + dcut < p1) mlo = mhi = 0u;
    p2 = fminf(p2, fmaxf(p1, key));
    p1 = fminf(p1, key);
    pd = p1 + dcut;
    if (key <= pd) {
      mlo |= shl(1u, (unsigned)i);
      mhi |= shl(1u, (unsigned)(i - 32));
    }
    return nxt;
  };
  for (int i = 0; i < n_seq; ++i) {
    const float4 A = f4(aqa + 16u * i);
    const float4 M = f4(aqm + 16u * i);
    // stop once no later unit (nor the rest of this one) can be P1, P2 or tied with P1
    if (M.x >= p2 && M.x > pd) break;
    float pp, ph, E, pen;
    part(A, pp, ph, E, pen);
    i = take(i, A, M, pp, ph, E, pen);
  }
  if (!(p1 < 2.0f) || bi < 0) return false;  // P1 must be a possible cell (no penalty)
  const int c1 = (int)((meta_w(bi) >> 8) & 0xFFu);
  if (c1 >= T.n_cells) return false;
  unsigned long long marks = ((unsigned long long)mhi << 32) | mlo;
  Top2 t{p1, p2, bi};
  auto sure = [&](int c) {
    const float4 A = cell_at(c);
    if (!(energy(A) <= x.e_hi)) return false;
    if (!HAS_PR) return true;
    return phi32_x(fmaf(x.goal_f, A.x, -x.mu_f) * x.inv_sig_s) >= x.th_hi;
  };
  const float cut = t.p1 + dcut;
  int w = c1;
  if (!(t.p2 > cut)) {
    // (c') near-ties within P1's class ordered by the deadline-miss tail, as
    // in fast_max_accuracy: marked cells re-derived with their chain's tail
    const uint32_t ccls = __float_as_uint(sB[c1].y) & 0xFFFFFu;
    const float mrg = 1e-15f * (2.0f + 2.0f * (float)max(1u, ccls & 0xFFu));
    bool ok1 = true;
    float ze1 = kInfF, ze2 = kInfF, bh = kInfF, bl = kInfF, lo2 = kInfF, nzlo = kInfF;
    int zc = -1, bc = -1;
    while (marks) {
      const int i = __ffsll((long long)marks) - 1;
      marks &= marks - 1;
      const float4 Mi = f4(aqm + 16u * i);
      if (Mi.x > cut) continue;  // every key of the cell's unit is >= its bound: outside the final cut
      const unsigned mw = __float_as_uint(Mi.w);
      const int k = (int)(mw & 7u), c = (int)((mw >> 8) & 0xFFu);
      float a = 0.f, tail = 0.f, r = 0.f;
      bool bad = false;
      float4 A;
      for (int m = c - k; m <= c; ++m) {  // the chain up to this cell, as pass 1 carried it
        A = cell_at(m);
        if (m == c - k) a = A.w;
        const float xz = fmaf(x.goal_f, A.x, -x.mu_f) * x.inv_sig_s;
        a = fmaf(phi32_x(xz), A.z, a);
        if (!(xz >= kExactOneX)) {
          bad |= !(xz >= 0.0f) || !(A.z >= 0.0f);
          tail = fmaf(0.5f * erfc_rel(xz), A.z, tail);
          const float dx = 4.0f * kEps * (fmaf(x.goal_f, A.x, fabsf(x.mu_f)) * x.inv_sig_s + fabsf(xz));
          r = fmaxf(r, fmaf(2.0f * xz + 2.0f, dx, 1e-4f));
        }
      }
      const float E = energy(A);
      if (pack_key(fmaxf(2.0f - a, penalty(A, E)), (unsigned)k) > cut) continue;
      if (bad || (__float_as_uint(sB[c].y) & 0xFFFFFu) != ccls) ok1 = false;
      if (tail == 0.0f) {  // exact acc = a_k: energy decides among these
        ze2 = fminf(ze2, fmaxf(ze1, E));
        if (E < ze1) zc = c;
        ze1 = fminf(ze1, E);
      } else {
        const float hi = tail * (1.0f + r), lo = tail * (1.0f - r);
        nzlo = fminf(nzlo, lo);
        if (hi < bh) {
          lo2 = fminf(lo2, bl);
          bh = hi;
          bl = lo;
          bc = c;
        } else {
          lo2 = fminf(lo2, lo);
        }
      }
    }
    if (!ok1) return false;
    if (zc >= 0) {  // zero tails win; nonzero ones must be strictly worse
      if (!(nzlo > mrg) || !(ze2 > ze1 + ze1 * (4.0f * x.d_erel) + 1e-30f)) return false;
      w = zc;
    } else {
      if (bc < 0 || !(lo2 > bh + mrg)) return false;
      w = bc;
    }
  }
  if (!sure(w)) return false;
  d.cell = w;
  d.level = 0;
  d.refined = false;
  return true;
}

// Re-rank pass from the stored FP32 objectives (no re-scan): the same
// cell-to-lane assignment as cell_pass, so each lane reads what it wrote.
template <int MODE, bool HAS_PR, class Tile>
__device__ __forceinline__ void refine_stored(const DevTable& T, const float4* __restrict__ sB,
                                              const int2* __restrict__ sCol, const Tile& tile, const StepCtx& x,
                                              int kinds, AlertScan<MODE, HAS_PR>& S) {
  const int W = Tile::num_threads();
  const int lane = tile.thread_rank();
  const int L = S.level;
  // packing perturbs the stored value by <= 3 ulp: widen the cut accordingly
  const float cut = S.cut + fabsf(S.cut) * 4.8e-7f + 1e-30f;
  auto check = [&](int c) {
    unsigned u;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(u) : "r"(x.sv + 4u * c));
    const bool poss = L == 2 || ((u >> L) & 1u);
    if (!S.all && !(poss && __uint_as_float(u) <= cut)) return;
    Pred64 q = eval64(T, x, c);
    if (!feasible64(x, q, L)) return;
    Key64 k = key64(x, q, L, __float_as_uint(sB[c].y), c);
    if (S.best.cell < 0 || k.less(S.best)) S.best = k;
  };
  if (kinds & 1)
    for (int c = lane; c < T.n_trad; c += W) check(c);
  if (kinds & 2)
    for (int col = lane; col < T.n_any_cols; col += W) {
      const int2 cd = sCol[col];
      for (int k = 0; k < cd.y; ++k) check(cd.x + k);
    }
}

// AlertPolicy.decide (policies.py:97-103) for the tile's stream: the full
// FP32 scan + FP64 re-rank.
template <int MODE, bool HAS_PR, class Tile>
__device__ __forceinline__ Decision alert_decide_full(const DevTable& T, const float4* sA, const float4* sB,
                                                      const int2* sCol, const Tile& tile, StepCtx& x, int kinds,
                                                      bool no_refine) {
  AlertScan<MODE, HAS_PR> S;
#pragma unroll
  for (int l = 0; l < 3; ++l) S.t[l].init();
  // fallback levels that can be distinct (selector.py:94-99): min-energy L1 == L0;
  // max-accuracy without pr_threshold: L1 admits everything, L2 unreachable.
  constexpr int NL = (MODE == ALERT_MODE_MIN_ENERGY) ? 2 : (HAS_PR ? 3 : 2);
  Decision d{-1, 0, false};
  int start = 0;
  if (!x.fp64_all) {
    cell_pass<0, TRACK_CONSTRAINED>(T, sA, sB, sCol, tile, x, kinds, S);
    S.t[0].merge(tile);
    if (MODE == ALERT_MODE_MAX_ACCURACY) S.t[1].merge(tile);
    // level 2 is needed only if every constrained level is empty (uniform per tile)
    const bool need_l2 = !(S.t[0].b1 < kInfF) && !(S.t[0].un < kInfF) &&
                         (MODE == ALERT_MODE_MIN_ENERGY || (HAS_PR && !(S.t[1].b1 < kInfF) && !(S.t[1].un < kInfF)));
    if ((MODE == ALERT_MODE_MIN_ENERGY || HAS_PR) && need_l2) {
      cell_pass<0, TRACK_L2>(T, sA, sB, sCol, tile, x, kinds, S);
      S.t[2].merge(tile);
    }
    start = -1;
    bool done = false;
#pragma unroll
    for (int li = 0; li < NL; ++li) {
      const int L = (li == 1 && MODE == ALERT_MODE_MIN_ENERGY) ? 2 : li;
      const Tracker& tr = S.t[L];
      if (!done) {
        float cut = cutoff<MODE>(x, L, tr.b1);
        if (tr.un < kInfF && (!(tr.b1 < kInfF) || tr.un <= cut)) {
          start = li;
          done = true;
        } else if (tr.b1 < kInfF) {
          if (tr.b2 <= cut) start = li;
          else { d.cell = tr.i1; d.level = L; }
          done = true;
        }
      }
    }
    if (start < 0) return d;
    if (no_refine) {  // FP32-only decision (measurement mode, not reference-exact)
#pragma unroll
      for (int li = 0; li < NL; ++li) {
        const int L = (li == 1 && MODE == ALERT_MODE_MIN_ENERGY) ? 2 : li;
        if (li >= start && d.cell < 0 && S.t[L].b1 < kInfF) { d.cell = S.t[L].i1; d.level = L; }
      }
      if (d.cell >= 0) return d;
    }
  }
  // FP64 re-rank, level by level from the first uncertain one.  A level-2
  // tracker that was never scanned keeps b1 = inf: every candidate is relevant.
  ensure_fp64(x);
#pragma unroll
  for (int li = 0; li < NL; ++li) {
    const int L = (li == 1 && MODE == ALERT_MODE_MIN_ENERGY) ? 2 : li;
    if (li >= start && d.cell < 0) {
      S.level = L;
      S.all = x.fp64_all || (L == 2 && !(S.t[2].b1 < kInfF));  // level 2 never scanned: all relevant
      S.cut = S.all ? kInfF : cutoff<MODE>(x, L, S.t[L].b1);
      S.best.init();
      // stored objectives cover levels 0/1 and, for max-accuracy, level 2
      // (same objective); min-energy level 2 (-acc) needs the re-scan
      if (MODE == ALERT_MODE_MAX_ACCURACY && HAS_PR && x.has_sv && !x.fp64_all)
        refine_stored(T, sB, sCol, tile, x, kinds, S);
      else
        cell_pass<1, TRACK_CONSTRAINED>(T, sA, sB, sCol, tile, x, kinds, S);
      S.best.merge(tile);
      if (S.best.cell >= 0) {
        d.cell = S.best.cell;
        d.level = L;
        d.refined = true;
      }
    }
  }
  return d;
}

// Mode sets compiled into a kernel: every mode, or min-energy only (smaller
// code and register footprint when every spec of a launch minimises energy).
enum { MS_ALL = 0, MS_MIN_ENERGY = 1, MS_MAX_ACCURACY = 2 };

// The full scan as an out-of-line call: in the min-energy kernel it runs only
// when the fast scan cannot certify (rare), so its registers are saved around
// the call instead of being reserved (or spilled) across the whole step loop.
template <int MODE, bool HAS_PR, class Tile>
__device__ __noinline__ Decision alert_decide_full_call(const DevTable& T, const float4* sA, const float4* sB,
                                                        const int2* sCol, Tile tile, StepCtx x, int kinds,
                                                        bool no_refine) {
  return alert_decide_full<MODE, HAS_PR>(T, sA, sB, sCol, tile, x, kinds, no_refine);
}

template <int MODE, bool HAS_PR, bool OUTLINE, class Tile>
__device__ __forceinline__ Decision alert_decide_t(const DevTable& T, const float4* sA, const float4* sB,
                                                   const int2* sCol, const Tile& tile, StepCtx& x, int kinds,
                                                   bool no_refine) {
  bool tried = false;
  // the fast scans vote across the converged lanes (__activemask); the
  // explicit __syncwarp re-converges them before the (divergent) fallback
  if (MODE == ALERT_MODE_MIN_ENERGY && x.fast && !x.fp64_all) {
    const unsigned am = __activemask();
    Decision d{-1, 0, false};
    const bool ok = fast_min_energy<HAS_PR>(T, sA, sB, sCol, tile, x, kinds, d);
    __syncwarp(am);
    if (ok) return d;
    tried = true;
  }
  if (MODE == ALERT_MODE_MAX_ACCURACY && x.fast && !x.fp64_all && T.units) {
    const unsigned am = __activemask();
    Decision d{-1, 0, false};
    const bool ok = (Tile::num_threads() == 1 && x.sqA)
                        ? fast_max_accuracy_flat<HAS_PR>(T, sA, sB, x, kinds, d)
                        : fast_max_accuracy<HAS_PR>(T, sA, sB, tile, x, kinds, d);
    __syncwarp(am);
    if (ok) return d;
    tried = true;
  }
  Decision d = OUTLINE ? alert_decide_full_call<MODE, HAS_PR>(T, sA, sB, sCol, tile, x, kinds, no_refine)
                       : alert_decide_full<MODE, HAS_PR>(T, sA, sB, sCol, tile, x, kinds, no_refine);
  d.full = tried;
  return d;
}

template <int MS = MS_ALL, class Tile>
__device__ __forceinline__ Decision alert_decide(const DevTable& T, const float4* sA, const float4* sB,
                                                 const int2* sCol, const Tile& tile, StepCtx& x,
                                                 int kinds, bool no_refine) {
#ifndef ALERT_OUTLINE_FULL
#define ALERT_OUTLINE_FULL 0
#endif
  constexpr bool OUT = ALERT_OUTLINE_FULL && MS == MS_MIN_ENERGY;
  if (MS == MS_MIN_ENERGY || (MS == MS_ALL && x.spec->mode == ALERT_MODE_MIN_ENERGY)) {
    if (x.spec->has_pr)
      return alert_decide_t<ALERT_MODE_MIN_ENERGY, true, OUT>(T, sA, sB, sCol, tile, x, kinds, no_refine);
    return alert_decide_t<ALERT_MODE_MIN_ENERGY, false, OUT>(T, sA, sB, sCol, tile, x, kinds, no_refine);
  }
  if (x.spec->has_pr)
    return alert_decide_t<ALERT_MODE_MAX_ACCURACY, true, false>(T, sA, sB, sCol, tile, x, kinds, no_refine);
  return alert_decide_t<ALERT_MODE_MAX_ACCURACY, false, false>(T, sA, sB, sCol, tile, x, kinds, no_refine);
}

// --------------------------------------------------------------------------
// execute_decision + measure (simulator.py:249-280, 329-382), FP64
struct Outcome {
  double latency;    // StepRecord.observed_latency (incl. overhead tax)
  double delivered;  // delivered accuracy
  double energy;
  double fb_latency, fb_t_prof;
  int completed;
  bool met, vl, va, ve;
};

__device__ __forceinline__ Outcome execute_measure(const float4* sB, const Cell64* C, const SpecDev* sp, int c,
                                                   double s, double goal, double period, double idle) {
  Outcome o;
  const int stage = cell_stage(sB[c]);
  const int first = stage == 0 ? c : c - (stage - 1);
  double lat;
  if (stage == 0) {
    double t = C[c].t;
    lat = xmul(s, t);
    o.completed = lat <= goal ? 1 : 0;
    o.fb_latency = lat;
    o.fb_t_prof = t;
  } else {
    double stop = py_min(xmul(s, C[c].t), goal);
    int completed = 0;
    for (int m = 0; m < stage; ++m)
      if (xmul(s, C[first + m].t) <= stop) completed = m + 1;
    o.completed = completed;
    lat = stop;
    if (completed) {
      double t = C[first + completed - 1].t;
      o.fb_latency = xmul(s, t);
      o.fb_t_prof = t;
    } else {
      o.fb_latency = stop;
      o.fb_t_prof = C[first].t;
    }
  }
  const double cap = C[c].cap;
  o.latency = xadd(lat, sp->oh);
  o.delivered = o.completed >= 1 ? C[first + o.completed - 1].a : C[c].qf;
  o.met = o.completed >= 1 && o.latency <= period;
  o.energy = xadd(xmul(cap, py_min(o.latency, period)), xmul(idle, py_max(0.0, xsub(period, o.latency))));
  o.vl = !o.met;
  o.va = sp->mode == ALERT_MODE_MIN_ENERGY && o.delivered < sp->q_goal;
  o.ve = sp->mode == ALERT_MODE_MAX_ACCURACY && o.energy > sp->e_goal;
  return o;
}

// --------------------------------------------------------------------------
// filters (estimator.py:59-84, 110-127), FP64 in registers
struct Filter {
  double mu, sigma2, k_gain, q_noise, innov, phi, m_var;
};

// k_valid: the previous update of this launch left k_gain = prior/(prior + r)
// and sigma2 = prior (reference gain convention), so an unchanged prior (the
// filter's fixed point whenever Q sits at its floor) reuses k_gain exactly
// instead of dividing again.
__device__ __forceinline__ void slowdown_update(const AlertFilterConfig& cfg, Filter& f, double obs, double t_prof,
                                                bool& k_valid) {
  double ky = xmul(f.k_gain, f.innov);
  double q = py_max(cfg.q0, xadd(xmul(cfg.alpha, f.q_noise), xmul(xsub(1.0, cfg.alpha), xmul(ky, ky))));
  double prior = xadd(xmul(xsub(1.0, f.k_gain), f.sigma2), q);
  double k = (k_valid && prior == f.sigma2) ? f.k_gain : xdiv(prior, xadd(prior, cfg.r));
  double y = xsub(xdiv(obs, t_prof), f.mu);
  double mu = xadd(f.mu, xmul(k, y));
  double s2 = cfg.sigma2_uses_current_gain ? xadd(xmul(xsub(1.0, k), f.sigma2), q) : prior;
  f.mu = mu;
  f.sigma2 = s2;
  f.k_gain = k;
  f.q_noise = q;
  f.innov = y;
  k_valid = !cfg.sigma2_uses_current_gain;
}

// ratio = min(1, measured / cap) is supplied by the caller (per-segment
// table).  The gain W depends only on M, whose sequence from m0 is the same
// for every stream: position ik in the host-computed table (ik < 0: divide).
__device__ __forceinline__ void idle_update(const AlertFilterConfig& cfg, Filter& f, double ratio, int& ik,
                                            int fix, const double* tw, const double* tm) {
  double w;
  if (ik >= 0) {
    w = tw[ik];
    if (ik < fix) ++ik;
    f.m_var = tm[ik];
  } else {
    double ms = xadd(f.m_var, cfg.s);
    w = xdiv(ms, xadd(ms, cfg.v));
    f.m_var = xmul(xsub(1.0, w), ms);
  }
  f.phi = xadd(f.phi, xmul(w, xsub(ratio, f.phi)));
}

// --------------------------------------------------------------------------
// OraclePolicy.decide (policies.py:160-205): exact per-cell outcome under the
// true slow-down, three fallback levels at once, FP64.
template <class Tile>
__device__ Decision oracle_decide_exact(const DevTable& T, const float4* sB, const Cell64* C, const int2* sCol,
                                  const Tile& tile, const SpecDev* sp, double s,
                                  double idle, double goal) {
  const int W = Tile::num_threads();
  const int lane = tile.thread_rank();
  const double oh = sp->oh;
  const double period = xadd(goal, oh);
  const bool maxacc = sp->mode == ALERT_MODE_MAX_ACCURACY;
  Key64 best[3];
  best[0].init(); best[1].init(); best[2].init();
  auto consider = [&](int c, int completed, double lat_raw, double delivered) {
    double cap = C[c].cap;
    double L = xadd(lat_raw, oh);
    bool met = completed >= 1 && L <= period;
    double E = xadd(xmul(cap, py_min(L, period)), xmul(idle, py_max(0.0, xsub(period, L))));
    uint32_t tk = __float_as_uint(sB[c].y);
#pragma unroll
    for (int lvl = 0; lvl < 3; ++lvl) {
      if (lvl != 2 && !met) continue;
      if (maxacc) {
        if (lvl == 0 && E > sp->e_goal) continue;
      } else if (lvl < 2 && delivered < sp->q_goal) {
        continue;
      }
      bool acc_obj = lvl == 2 || maxacc;
      Key64 k;
      k.p0 = acc_obj ? -delivered : E;
      k.p1 = acc_obj ? E : -delivered;
      k.tk = tk;
      k.cell = c;
      if (best[lvl].cell < 0 || k.less(best[lvl])) best[lvl] = k;
    }
  };
  for (int c = lane; c < T.n_trad; c += W) {
    double lat = xmul(s, C[c].t);
    bool done = lat <= goal;
    consider(c, done ? 1 : 0, lat, done ? C[c].a : C[c].qf);
  }
  for (int col = lane; col < T.n_any_cols; col += W) {
    int2 cd = sCol[col];
    int K = 0;
    double deliv = C[cd.x].qf;
    for (int k = 0; k < cd.y; ++k) {
      int c = cd.x + k;
      double st = xmul(s, C[c].t);
      if (st <= goal) { K = k + 1; deliv = C[c].a; }
      consider(c, K, py_min(st, goal), deliv);
    }
  }
  Decision d{-1, 0, true};
#pragma unroll
  for (int lvl = 0; lvl < 3; ++lvl) {
    best[lvl].merge(tile);
    if (d.cell < 0 && best[lvl].cell >= 0) { d.cell = best[lvl].cell; d.level = lvl; }
  }
  return d;
}


// --------------------------------------------------------------------------
// OraclePolicy.decide with an FP32 scan (policies.py:160-205).  Per cell, in
// FP32: completion under the true slow-down (x = s t vs the goal, with an
// uncertainty band: "poison" when x is within a few ulp of the goal), the
// delivered-accuracy CLASS (exact integer rank of the table value, see
// alert_table_create) and the energy.  Max-delivered-accuracy levels use a
// lexicographic (rank, energy) tracker, so exact accuracy ties between powers
// of one DNN are resolved in FP32; min-energy levels use the energy tracker.
// Anything not provably decided (energy within the FP32 bound, poisoned
// completions) is re-ranked exactly in FP64 (execute_measure + the reference
// keys).  ALERT_FLAG_FP64_ALL uses oracle_decide_exact throughout.
struct LexTracker {
  int r1, i1, un;   // best rank (sure), its cell, lowest possible rank among uncertain
  float e1, e2;     // best / second-best energy inside class r1
  __device__ __forceinline__ void init() { r1 = un = 0x7fffffff; i1 = -1; e1 = e2 = kInfF; }
  __device__ __forceinline__ void push(int r, float e, bool sure, bool unc, int r_unc, int c) {
    const bool lt = sure && r < r1, eq = sure && r == r1;
    const bool nb = lt || (eq && e < e1);
    e2 = lt ? kInfF : (eq ? fminf(e2, fmaxf(e1, e)) : e2);
    e1 = lt ? e : (eq ? fminf(e1, e) : e1);
    i1 = nb ? c : i1;
    r1 = lt ? r : r1;
    un = unc ? min(un, r_unc) : un;
  }
  template <class Tile>
  __device__ __forceinline__ void merge(const Tile& tile) {
#pragma unroll
    for (int m = 1; m < Tile::num_threads(); m <<= 1) {
      const int or1 = tile.shfl_xor(r1, m), oi1 = tile.shfl_xor(i1, m), oun = tile.shfl_xor(un, m);
      const float oe1 = tile.shfl_xor(e1, m), oe2 = tile.shfl_xor(e2, m);
      if (or1 < r1) {
        r1 = or1; i1 = oi1; e1 = oe1; e2 = oe2;
      } else if (or1 == r1) {
        e2 = fminf(fminf(e2, oe2), fmaxf(e1, oe1));
        if (oe1 < e1 || (oe1 == e1 && (unsigned)oi1 < (unsigned)i1)) { e1 = oe1; i1 = oi1; }
      }
      un = min(un, oun);
    }
  }
};

struct OrCtx {
  double s, goal, period, idle;   // exact inputs
  float sf, goal_f, glo, ghi, oh, P, idle_f, idleP, dE, e_lo, e_hi;
  int rank_q;
};

__device__ __forceinline__ void make_or_ctx(OrCtx& o, const DevTable& T, const SpecDev* sp, double s, double idle,
                                            double goal) {
  o.s = s; o.goal = goal; o.idle = idle; o.period = xadd(goal, sp->oh);
  o.sf = (float)s;
  o.goal_f = (float)goal;
  o.glo = o.goal_f * (1.0f - 8.0f * kEps);
  o.ghi = o.goal_f * (1.0f + 8.0f * kEps);
  o.oh = (float)sp->oh;
  o.P = (float)o.period;
  o.idle_f = (float)idle;
  o.idleP = o.idle_f * o.P;
  o.dE = 8.0f * kEps * (T.cap_max + o.idle_f) * o.P;
  o.e_lo = sp->e_f - o.dE;
  o.e_hi = sp->e_f + o.dE;
  o.rank_q = sp->rank_q;
}

// Running per-column state of the FP32 oracle evaluation.
struct OrRun {
  bool done;    // some stage of the column completed
  bool poison;  // a completion test so far was inside the uncertainty band
  int rank;     // class of the delivered accuracy
};

// FP32 outcome of one cell (updates the running column state).
__device__ __forceinline__ void or_cell(const OrCtx& o, const float4& A, const float4& B, OrRun& run, float& E,
                                        int& rank, bool& met, bool& poison) {
  const float x = o.sf * B.x;
  const bool done = x <= o.goal_f;
  const bool band = x >= o.glo && x <= o.ghi;
  if (A.w >= 0.0f) {  // traditional cell or first stage of a column
    run.done = false;
    run.poison = false;
    run.rank = cell_rank_qf(B);
  }
  run.poison |= band;
  if (done) {
    run.done = true;
    run.rank = cell_rank_a(B);
  }
  met = run.done;
  rank = run.rank;
  poison = run.poison;
  const float L = (cell_stage(B) == 0 ? x : fminf(x, o.goal_f)) + o.oh;
  const float cap = A.y * A.x;  // (cap t) * (1/t)
  E = fmaf(cap - o.idle_f, fminf(L, o.P), o.idleP);
}

template <int MAXACC>
struct OracleScan {
  Tracker te;       // min-energy level 0 (energy objective)
  LexTracker lx[3]; // rank-objective levels
  // refine state
  int level;
  float ecut;
  int rcut;
  bool all;
  Key64 best;

  // classification at a level: sure / possible and the lowest possible rank
  __device__ __forceinline__ void classify(const OrCtx& o, int L, float E, int rank, bool met, bool poison,
                                           bool& sure, bool& unc, int& r_unc) const {
    r_unc = poison ? 0 : rank;
    if (L == 2) { sure = !poison; unc = poison; return; }
    if (MAXACC) {
      if (L == 0) {
        sure = !poison && met && E <= o.e_lo;
        unc = (poison && E <= o.e_hi) || (!poison && met && E > o.e_lo && E <= o.e_hi);
      } else {
        sure = !poison && met;
        unc = poison;
      }
    } else {  // min-energy levels 0/1: met and delivered >= q_goal
      sure = !poison && met && rank < o.rank_q;
      unc = poison;
    }
  }

  template <int TRACK>
  __device__ __forceinline__ void scan_cell(const OrCtx& o, int c, float E, int rank, bool met, bool poison) {
    bool sure, unc;
    int ru;
    if (TRACK == TRACK_L2) {
      classify(o, 2, E, rank, met, poison, sure, unc, ru);
      lx[2].push(rank, E, sure, unc, ru, c);
      return;
    }
    classify(o, 0, E, rank, met, poison, sure, unc, ru);
    if (MAXACC) {
      lx[0].push(rank, E, sure, unc, ru, c);
      classify(o, 1, E, rank, met, poison, sure, unc, ru);
      lx[1].push(rank, E, sure, unc, ru, c);
    } else {
      te.push(E, sure, unc, c);
    }
  }

  __device__ __forceinline__ void refine_cell(const float4* sB, const Cell64* C, const SpecDev* sp, const OrCtx& o,
                                              int c, float E, int rank, bool met, bool poison) {
    if (!all) {
      bool sure, unc;
      int ru;
      classify(o, level, E, rank, met, poison, sure, unc, ru);
      if (!(sure || unc)) return;
      const bool energy_level = !MAXACC && level != 2;
      if (energy_level ? !(E <= ecut) : (ru > rcut)) return;
    }
    const Outcome x = execute_measure(sB, C, sp, c, o.s, o.goal, o.period, o.idle);
    // _exact_eval + the level filters of policies.py:171-186
    if (level != 2 && !x.met) return;
    if (MAXACC) {
      if (level == 0 && x.energy > sp->e_goal) return;
    } else if (level < 2 && x.delivered < sp->q_goal) {
      return;
    }
    const bool acc_obj = level == 2 || MAXACC;
    Key64 k;
    k.p0 = acc_obj ? -x.delivered : x.energy;
    k.p1 = acc_obj ? x.energy : -x.delivered;
    k.tk = __float_as_uint(sB[c].y);
    k.cell = c;
    if (best.cell < 0 || k.less(best)) best = k;
  }
};

// Traversal shared by the oracle scan / refine passes (flat at W = 1).
template <int PASS, int TRACK, int MAXACC, class Tile>
__device__ __forceinline__ void oracle_pass(const DevTable& T, const float4* __restrict__ sA,
                                            const float4* __restrict__ sB, const int2* __restrict__ sCol,
                                            const Cell64* C, const SpecDev* sp, const Tile& tile, const OrCtx& o,
                                            OracleScan<MAXACC>& S) {
  const int W = Tile::num_threads();
  const int lane = tile.thread_rank();
  auto visit = [&](int c, OrRun& run) {
    float E;
    int rank;
    bool met, poison;
    or_cell(o, sA[c], sB[c], run, E, rank, met, poison);
    if (PASS == 0) S.template scan_cell<TRACK>(o, c, E, rank, met, poison);
    else S.refine_cell(sB, C, sp, o, c, E, rank, met, poison);
  };
  if (W == 1) {
    OrRun run{false, false, 0};
#pragma unroll 4
    for (int c = 0; c < T.n_cells; ++c) visit(c, run);
    return;
  }
  for (int c = lane; c < T.n_trad; c += W) {
    OrRun run{false, false, 0};
    visit(c, run);
  }
  for (int col = lane; col < T.n_any_cols; col += W) {
    const int2 cd = sCol[col];
    OrRun run{false, false, 0};
    for (int k = 0; k < cd.y; ++k) visit(cd.x + k, run);
  }
}

template <int MAXACC, class Tile>
__device__ Decision oracle_decide_t(const DevTable& T, const float4* sA, const float4* sB, const Cell64* C,
                                    const int2* sCol, const Tile& tile, const SpecDev* sp, const OrCtx& o) {
  OracleScan<MAXACC> S;
  S.te.init();
  S.lx[0].init(); S.lx[1].init(); S.lx[2].init();
  oracle_pass<0, TRACK_CONSTRAINED>(T, sA, sB, sCol, C, sp, tile, o, S);
  if (MAXACC) {
    S.lx[0].merge(tile);
    S.lx[1].merge(tile);
  } else {
    S.te.merge(tile);
  }
  const bool empty01 = MAXACC ? (S.lx[0].r1 == 0x7fffffff && S.lx[0].un == 0x7fffffff &&
                                 S.lx[1].r1 == 0x7fffffff && S.lx[1].un == 0x7fffffff)
                              : (!(S.te.b1 < kInfF) && !(S.te.un < kInfF));
  if (empty01) {
    oracle_pass<0, TRACK_L2>(T, sA, sB, sCol, C, sp, tile, o, S);
    S.lx[2].merge(tile);
  }
  constexpr int NL = MAXACC ? 3 : 2;
  Decision d{-1, 0, false};
  int start = -1;
  bool done = false;
#pragma unroll
  for (int li = 0; li < NL; ++li) {
    const int L = (!MAXACC && li == 1) ? 2 : li;
    if (done) continue;
    if (!MAXACC && L == 0) {
      const Tracker& tr = S.te;
      const float cut = tr.b1 + 2.0f * o.dE;
      if (tr.un < kInfF && (!(tr.b1 < kInfF) || tr.un <= cut)) { start = li; done = true; }
      else if (tr.b1 < kInfF) {
        if (tr.b2 <= cut) start = li;
        else { d.cell = tr.i1; d.level = L; }
        done = true;
      }
    } else {
      const LexTracker& lt = S.lx[L];
      if (lt.r1 == 0x7fffffff && lt.un == 0x7fffffff) continue;  // empty level
      if (lt.r1 != 0x7fffffff && lt.un > lt.r1 && lt.e2 > lt.e1 + 2.0f * o.dE) {
        d.cell = lt.i1;
        d.level = L;
      } else {
        start = li;
      }
      done = true;
    }
  }
  if (start < 0) return d;
#pragma unroll
  for (int li = 0; li < NL; ++li) {
    const int L = (!MAXACC && li == 1) ? 2 : li;
    if (li >= start && d.cell < 0) {
      S.level = L;
      const bool e_level = !MAXACC && L == 0;
      const bool scanned = e_level ? (S.te.b1 < kInfF) : (S.lx[L].r1 != 0x7fffffff);
      S.all = !scanned && !(e_level ? (S.te.un < kInfF) : (S.lx[L].un != 0x7fffffff));
      S.ecut = e_level && scanned ? S.te.b1 + 2.0f * o.dE : kInfF;
      S.rcut = (!e_level && scanned) ? S.lx[L].r1 : 0x7fffffff;
      S.best.init();
      oracle_pass<1, TRACK_CONSTRAINED>(T, sA, sB, sCol, C, sp, tile, o, S);
      S.best.merge(tile);
      if (S.best.cell >= 0) {
        d.cell = S.best.cell;
        d.level = L;
        d.refined = true;
      }
    }
  }
  return d;
}

// OraclePolicy.decide, min-energy level 0 (policies.py:160-205) as a
// certified fast scan.  Level 0 needs the input to complete (s t <= goal) and
// the delivered accuracy >= q_goal; a traditional cell that completes delivers
// its DNN's accuracy, so a DNN row whose accuracy class fails q_goal can never
// be feasible and is skipped as a whole (uniform over the tile).  Per cell of
// the remaining rows: energy E (as or_cell) and a sign-exact deadline penalty
// H (s t - goal (1 + 8 eps)) > 0 for cells that surely miss; the key is their
// max, so possible cells (surely or maybe completing) compete on energy.
// Anytime columns run the column logic of or_cell (possible = sure or
// uncertain at level 0).  Certified when P1 surely completes and every other
// possible cell is more than the FP32 energy bound 2 dE above it (the full
// scan's margin); otherwise oracle_decide_t decides.
template <class Tile>
__device__ __forceinline__ bool oracle_fast_min_energy(const DevTable& T, const float4* __restrict__ sA,
                                                       const float4* __restrict__ sB, const int2* __restrict__ sCol,
                                                       const Tile& tile, const OrCtx& o, Decision& d) {
  const int W = Tile::num_threads();
  const int lane = tile.thread_rank();
  const int P = T.n_powers;
  const int n_rows = P > 0 ? T.n_trad / P : 0;
  const float mgH = -o.ghi * kPenH;
  float p1 = kInfF, p2 = kInfF;
  int bi = -1;
  auto push = [&](float key, int c) {
    if (key < p1) bi = c;
    p2 = fminf(p2, fmaxf(p1, key));
    p1 = fminf(p1, key);
  };
  for (int r = 0; r < n_rows; ++r) {
    const int c0 = r * P;
    if (cell_rank_a(sB[c0]) >= o.rank_q) continue;  // the DNN's accuracy fails q_goal: no cell can be feasible
    for (int j = lane; j < P; j += W) {
      const int c = c0 + j;
      const float4 A = sA[c];
      const float x = o.sf * sB[c].x;
      const float cap = A.y * A.x;  // (cap t) * (1/t), as or_cell
      const float E = fmaf(cap - o.idle_f, fminf(x + o.oh, o.P), o.idleP);
      push(pack_key(fmaxf(E, fmaf(x, kPenH, mgH)), (unsigned)c & 7u), c);
    }
  }
  for (int col = lane; col < T.n_any_cols; col += W) {
    const int2 cd = sCol[col];
    OrRun run{false, false, 0};
    for (int k = 0; k < cd.y; ++k) {
      float E;
      int rank;
      bool met, poison;
      or_cell(o, sA[cd.x + k], sB[cd.x + k], run, E, rank, met, poison);
      const bool possible = poison || (met && rank < o.rank_q);
      push(possible ? pack_key(E, (unsigned)(cd.x + k) & 7u) : kInfF, cd.x + k);
    }
  }
#pragma unroll
  for (int m = 1; m < W; m <<= 1) {
    const float o1 = tile.shfl_xor(p1, m), o2 = tile.shfl_xor(p2, m);
    const int ob = tile.shfl_xor(bi, m);
    p2 = fmin3(p2, o2, fmaxf(p1, o1));
    if (o1 < p1 || (o1 == p1 && (unsigned)ob < (unsigned)bi)) bi = ob;
    p1 = fminf(p1, o1);
  }
  // margin: the FP32 energy bound of both keys (2 dE) and their 3-bit packing (< 8 ulp each)
  if (!(p1 < kInfF) || bi < 0 || !(p2 * (1.0f - 16.0f * kEps) > p1 + 2.0f * o.dE)) return false;
  // P1 must surely complete (and, anytime, surely deliver >= q_goal)
  if (bi < T.n_trad) {
    if (!(o.sf * sB[bi].x < o.glo)) return false;
  } else {
    const int st = cell_stage(sB[bi]);
    OrRun run{false, false, 0};
    float E;
    int rank;
    bool met = false, poison = true;
    for (int c = bi - (st - 1); c <= bi; ++c) or_cell(o, sA[c], sB[c], run, E, rank, met, poison);
    if (poison || !met || rank >= o.rank_q) return false;
  }
  d.cell = bi;
  d.level = 0;
  d.refined = false;
  return true;
}

// OraclePolicy.decide, max-accuracy level 0 (policies.py:160-205: complete
// and E <= e_goal, then the highest delivered accuracy, then the lowest
// energy) with the full scan's classification and certificate, visiting
// only the DNN rows that can matter.  Anytime columns first (their delivered
// class varies per stage), then the traditional rows best accuracy class
// first (T.or_rows): a completing traditional cell delivers its DNN's
// accuracy, so once the tile holds a surely feasible cell of class r1, rows
// of a worse class can neither beat r1 nor make it uncertain (a maybe-
// completing cell of such a row still delivers a worse class or fails level
// 0) and the scan stops; a row whose fastest cell surely misses the deadline
// is skipped.  Certified as in oracle_decide_t (no uncertain cell of class
// <= r1, the best energy of class r1 clear of the next by 2 dE); otherwise the
// full scan decides.
template <class Tile>
__device__ __forceinline__ bool oracle_fast_max_accuracy(const DevTable& T, const float4* __restrict__ sA,
                                                         const float4* __restrict__ sB,
                                                         const int2* __restrict__ sCol, const Tile& tile,
                                                         const OrCtx& o, Decision& d) {
  const int W = Tile::num_threads();
  const int lane = tile.thread_rank();
  const int P = T.n_powers;
  const int n_rows = P > 0 ? T.n_trad / P : 0;
  LexTracker lx;
  lx.init();
  for (int col = lane; col < T.n_any_cols; col += W) {
    const int2 cd = sCol[col];
    OrRun run{false, false, 0};
    for (int k = 0; k < cd.y; ++k) {
      float E;
      int rank;
      bool met, poison;
      or_cell(o, sA[cd.x + k], sB[cd.x + k], run, E, rank, met, poison);
      const bool sure = !poison && met && E <= o.e_lo;
      const bool unc = (poison && E <= o.e_hi) || (!poison && met && E > o.e_lo && E <= o.e_hi);
      lx.push(rank, E, sure, unc, poison ? 0 : rank, cd.x + k);
    }
  }
  for (int r = 0; r < n_rows; ++r) {
    const float4 R = __ldg(T.or_rows + r);
    const int rank = __float_as_int(R.y);
    if (tile.any(lx.r1 < rank)) break;             // a better class is surely feasible: no later row matters
    if (!(o.sf * R.z <= o.ghi)) continue;          // even the fastest cell surely misses the deadline
    const int c0 = __float_as_int(R.x);
    for (int j = lane; j < P; j += W) {
      const int c = c0 + j;
      const float4 A = sA[c];
      const float x = o.sf * sB[c].x;
      const float cap = A.y * A.x;  // as or_cell
      const float E = fmaf(cap - o.idle_f, fminf(x + o.oh, o.P), o.idleP);
      const bool band = x >= o.glo && x <= o.ghi;
      const bool done = x <= o.goal_f;
      const bool sure = !band && done && E <= o.e_lo;
      const bool unc = (band && E <= o.e_hi) || (!band && done && E > o.e_lo && E <= o.e_hi);
      lx.push(rank, E, sure, unc, rank, c);  // a maybe-completing traditional cell can only deliver its DNN's class
    }
  }
  lx.merge(tile);
  if (lx.r1 == 0x7fffffff || !(lx.un > lx.r1) || !(lx.e2 > lx.e1 + 2.0f * o.dE)) return false;
  d.cell = lx.i1;
  d.level = 0;
  d.refined = false;
  return true;
}

template <class Tile>
__device__ __forceinline__ Decision oracle_decide(const DevTable& T, const float4* sA, const float4* sB,
                                                  const Cell64* C, const int2* sCol, const Tile& tile,
                                                  const SpecDev* sp, double s, double idle, double goal,
                                                  bool fp64_all, bool fast_off = false) {
  if (fp64_all) return oracle_decide_exact(T, sB, C, sCol, tile, sp, s, idle, goal);
  OrCtx o;
  make_or_ctx(o, T, sp, s, idle, goal);
  if (!(o.P > 0.0f) || !isfinite(o.dE)) return oracle_decide_exact(T, sB, C, sCol, tile, sp, s, idle, goal);
  if (sp->mode == ALERT_MODE_MAX_ACCURACY) {
    if (!fast_off && T.or_rows) {
      const unsigned am = __activemask();
      Decision d{-1, 0, false};
      const bool ok = oracle_fast_max_accuracy(T, sA, sB, sCol, tile, o, d);
      __syncwarp(am);
      if (ok) return d;
    }
    return oracle_decide_t<1>(T, sA, sB, C, sCol, tile, sp, o);
  }
  if (!fast_off) {
    const unsigned am = __activemask();
    Decision d{-1, 0, false};
    const bool ok = oracle_fast_min_energy(T, sA, sB, sCol, tile, o, d);
    __syncwarp(am);
    if (ok) return d;
  }
  return oracle_decide_t<0>(T, sA, sB, C, sCol, tile, sp, o);
}

__device__ __forceinline__ uint32_t pack_decision(int cand, int level, const Outcome& o, bool refined, int phase,
                                                  bool feasible) {
  return (uint32_t)cand | ((uint32_t)level << 16) | ((uint32_t)o.met << 18) | ((uint32_t)o.vl << 19) |
         ((uint32_t)o.va << 20) | ((uint32_t)o.ve << 21) | ((uint32_t)(o.completed & 0xF) << 22) |
         ((uint32_t)refined << 26) | ((uint32_t)(phase & 0x7) << 27) | ((uint32_t)feasible << 30);
}

}  // namespace alert
