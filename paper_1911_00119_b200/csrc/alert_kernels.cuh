// alert_kernels.cuh — kernel templates of the fused scheduling loop and the
// per-step decide / oracle kernels; instantiated per lane width W in
// alert_inst_w*.cu (compiled in parallel) and dispatched from alert_capi.cu.
#pragma once
#include <cuda_runtime.h>

#include "alert_device.cuh"

namespace alert {

struct RunParams {
  DevTable T;
  AlertFilterConfig cfg;
  const AlertSpec* specs;
  int n_specs;
  const int32_t* stream_spec;
  AlertTrace tr;
  AlertState st;
  AlertOutputs out;
  int policy;
  unsigned flags;
  int kinds;
  long long stream_begin, stream_end, step_begin, step_end;
};

__device__ __forceinline__ void load_table_smem(const DevTable& T, float4* sA, float4* sB, int2* sCol) {
  for (int i = threadIdx.x; i < T.n_cells; i += blockDim.x) {
    sA[i] = T.cellA[i];
    sB[i] = T.cellB[i];
  }
  for (int i = threadIdx.x; i < T.n_any_cols; i += blockDim.x) sCol[i] = T.any_cols[i];
  __syncthreads();
}

__device__ __forceinline__ double load_s(const AlertTrace& tr, long long row, long long n) {
  const long long off = row * tr.row_stride + (n - tr.step_offset) * tr.step_stride;
  if (tr.slowdown_dtype == ALERT_DTYPE_F64) return __ldg(reinterpret_cast<const double*>(tr.slowdown) + off);
  return (double)__ldg(reinterpret_cast<const float*>(tr.slowdown) + off);
}

// Per-tile FP64 accumulators, kept in shared memory: they are touched once
// per step (not per candidate), so they need not occupy registers.
struct TileAgg {
  double e, ec, a, ac;          // Neumaier sums of energy / delivered accuracy
  double pn, pe, pec, pa, pac;  // current phase: count, sums
  double pvl, pva, pve;         // current phase violation counts
  double oe, oec, oa, oac;      // oracle-alongside sums
};

enum { PF_ALERT = 0, PF_ORACLE = 1, PF_BOTH = 2 };  // policy families

__device__ __forceinline__ void load_phase(TileAgg& g, const double* agg, int phase) {
  const double* p = agg + ALERT_AGG_PHASE_BASE + ALERT_AGG_PHASE_STRIDE * phase;
  g.pn = p[0]; g.pe = p[1]; g.pec = p[2]; g.pa = p[3]; g.pac = p[4]; g.pvl = p[5]; g.pva = p[6]; g.pve = p[7];
}
__device__ __forceinline__ void store_phase(const TileAgg& g, double* agg, int phase) {
  double* p = agg + ALERT_AGG_PHASE_BASE + ALERT_AGG_PHASE_STRIDE * phase;
  p[0] = g.pn; p[1] = g.pe; p[2] = g.pec; p[3] = g.pa; p[4] = g.pac; p[5] = g.pvl; p[6] = g.pva; p[7] = g.pve;
}

// The fused closed loop (simulator.run, simulator.py:461-507): one tile of W
// lanes per stream, filter state in registers for the whole step range.
template <int W, int PF>
__global__ void __launch_bounds__(256, 2) run_kernel(const RunParams P) {
  extern __shared__ float4 smem[];
  const DevTable& T = P.T;
  float4* sA = smem;
  float4* sB = smem + T.n_cells;
  int2* sCol = reinterpret_cast<int2*>(sB + T.n_cells);
  TileAgg* sAgg = reinterpret_cast<TileAgg*>(sCol + T.n_any_cols + 1);
  load_table_smem(T, sA, sB, sCol);

  auto tile = cg::tiled_partition<W>(cg::this_thread_block());
  const long long stream = P.stream_begin + ((long long)blockIdx.x * blockDim.x + threadIdx.x) / W;
  if (stream >= P.stream_end) return;
  const bool writer = tile.thread_rank() == 0;
  TileAgg& G = sAgg[threadIdx.x / W];

  const int si = P.stream_spec ? P.stream_spec[stream] : (int)(stream % P.n_specs);
  const AlertSpec* spec = P.specs + si;
  const AlertTrace& tr = P.tr;
  const long long row = tr.stream_row ? tr.stream_row[stream] : stream;

  Filter f;
  f.mu = P.st.mu[stream];
  f.sigma2 = P.st.sigma2[stream];
  f.k_gain = P.st.k_gain[stream];
  f.q_noise = P.st.q_noise[stream];
  f.innov = P.st.innov[stream];
  f.phi = P.st.phi[stream];
  f.m_var = P.st.m_var[stream];
  double budget = P.st.group_budget[stream];
  int count = P.st.group_count[stream];
  const int group_size = spec->group_size;

  // segment (phase) tracking
  const int nseg = tr.n_segments[row];
  const int32_t* seg_end = tr.seg_end + row * tr.max_segments;
  const int32_t* seg_phase = tr.seg_phase + row * tr.max_segments;
  const double* seg_idle = tr.seg_idle + row * tr.max_segments;
  int seg = 0;
  while (seg + 1 < nseg && P.step_begin >= seg_end[seg]) ++seg;
  int cur_end = seg_end[seg];
  int phase = seg_phase[seg];
  double idle = seg_idle[seg];

  double* agg = P.out.agg ? P.out.agg + stream * ALERT_AGG_FIELDS : nullptr;
  int cVL = 0, cVA = 0, cVE = 0, cL1 = 0, cL2 = 0, cRef = 0;
  int oVL = 0, oVA = 0, oVE = 0, oSame = 0;
  if (writer) {
    G = TileAgg{};
    if (agg) {
      G.e = agg[ALERT_AGG_ENERGY]; G.ec = agg[ALERT_AGG_ENERGY_C];
      G.a = agg[ALERT_AGG_ACC]; G.ac = agg[ALERT_AGG_ACC_C];
      if (PF == PF_BOTH) {
        G.oe = agg[ALERT_AGG_OR_ENERGY]; G.oec = agg[ALERT_AGG_OR_ENERGY_C];
        G.oa = agg[ALERT_AGG_OR_ACC]; G.oac = agg[ALERT_AGG_OR_ACC_C];
      }
      if (phase >= 0 && phase < ALERT_MAX_PHASES) load_phase(G, agg, phase);
    }
  }

  const int kinds = P.kinds;
  const bool fp64_all = P.flags & ALERT_FLAG_FP64_ALL;
  const bool no_refine = P.flags & ALERT_FLAG_NO_REFINE;
  const int* forced = P.out.forced;

  double s_next = load_s(tr, row, P.step_begin);
  for (long long n = P.step_begin; n < P.step_end; ++n) {
    const double s = s_next;
    if (n + 1 < P.step_end) s_next = load_s(tr, row, n + 1);
    while (seg + 1 < nseg && n >= cur_end) {
      if (agg && writer && phase >= 0 && phase < ALERT_MAX_PHASES) store_phase(G, agg, phase);
      ++seg;
      cur_end = seg_end[seg];
      phase = seg_phase[seg];
      idle = seg_idle[seg];
      if (writer) {
        if (agg && phase >= 0 && phase < ALERT_MAX_PHASES) load_phase(G, agg, phase);
        else G.pn = G.pe = G.pec = G.pa = G.pac = G.pvl = G.pva = G.pve = 0.0;
      }
    }
    // adjust_goal (selector.py:48-70) with group budgets (simulator.py:473-483)
    const double oh = spec->overhead_budget;
    double goal;
    if (group_size > 0) {
      if (count == 0) {
        budget = xmul((double)group_size, spec->t_goal);
        count = group_size;
      }
      goal = xsub(xdiv(budget, (double)count), oh);
    } else {
      goal = xsub(spec->t_goal, oh);
    }
    goal = py_max(goal, 0.001);
    const double period = xadd(goal, oh);

    Decision d;
    if (PF == PF_ORACLE) {
      d = oracle_decide(T, tile, spec, s, idle, goal);
      d.refined = false;
    } else {
      StepCtx x;
      make_ctx(x, spec, f.mu, f.sigma2, f.phi, goal, fp64_all);
      d = alert_decide(T, sA, sB, sCol, tile, x, kinds, no_refine);
    }
    int exec_cell = d.cell;
    const long long oidx = stream * P.out.stream_stride + n * P.out.step_stride;
    if (forced) {
      int fc = forced[oidx];
      if (fc >= 0) exec_cell = T.cell_of_cand[fc];
    }
    const Outcome o = execute_measure(T, spec, exec_cell, s, goal, period, idle);
    if (PF != PF_ORACLE) {  // AlertPolicy.observe, policies.py:105-108
      slowdown_update(P.cfg, f, o.fb_latency, o.fb_t_prof);
      idle_update(P.cfg, f, idle, T.cap64[exec_cell]);
    }
    if (group_size > 0) {  // simulator.py:501-503
      budget = xsub(budget, o.latency);
      count -= 1;
    }
    cVL += o.vl; cVA += o.va; cVE += o.ve;
    cL1 += d.level == 1; cL2 += d.level == 2;
    cRef += d.refined;
    if (writer) {
      const AlertOutputs& out = P.out;
      if (out.decision) out.decision[oidx] = pack_decision(__float_as_int(sB[d.cell].z), d.level, o, d.refined, phase);
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
      // aggregates in step order (CPython 3.12 sum() semantics)
      neumaier(G.e, G.ec, o.energy);
      neumaier(G.a, G.ac, o.delivered);
      G.pn += 1.0;
      neumaier(G.pe, G.pec, o.energy);
      neumaier(G.pa, G.pac, o.delivered);
      G.pvl += o.vl; G.pva += o.va; G.pve += o.ve;
    }
    if (PF == PF_BOTH) {  // OraclePolicy alongside on the same step
      Decision od = oracle_decide(T, tile, spec, s, idle, goal);
      const Outcome oo = execute_measure(T, spec, od.cell, s, goal, period, idle);
      oVL += oo.vl; oVA += oo.va; oVE += oo.ve;
      oSame += od.cell == exec_cell;
      if (writer) {
        neumaier(G.oe, G.oec, oo.energy);
        neumaier(G.oa, G.oac, oo.delivered);
        if (P.out.oracle_decision)
          P.out.oracle_decision[oidx] = pack_decision(__float_as_int(sB[od.cell].z), od.level, oo, false, phase);
      }
    }
  }
  if (!writer) return;
  P.st.mu[stream] = f.mu;
  P.st.sigma2[stream] = f.sigma2;
  P.st.k_gain[stream] = f.k_gain;
  P.st.q_noise[stream] = f.q_noise;
  P.st.innov[stream] = f.innov;
  P.st.phi[stream] = f.phi;
  P.st.m_var[stream] = f.m_var;
  P.st.group_budget[stream] = budget;
  P.st.group_count[stream] = count;
  if (agg) {
    if (phase >= 0 && phase < ALERT_MAX_PHASES) store_phase(G, agg, phase);
    const double steps = (double)(P.step_end - P.step_begin);
    agg[ALERT_AGG_N] += steps;
    agg[ALERT_AGG_ENERGY] = G.e; agg[ALERT_AGG_ENERGY_C] = G.ec;
    agg[ALERT_AGG_ACC] = G.a; agg[ALERT_AGG_ACC_C] = G.ac;
    agg[ALERT_AGG_VIOL_LAT] += (double)cVL;
    agg[ALERT_AGG_VIOL_ACC] += (double)cVA;
    agg[ALERT_AGG_VIOL_ENERGY] += (double)cVE;
    agg[ALERT_AGG_LEVEL0] += steps - (double)cL1 - (double)cL2;
    agg[ALERT_AGG_LEVEL1] += (double)cL1;
    agg[ALERT_AGG_LEVEL2] += (double)cL2;
    agg[ALERT_AGG_REFINED] += (double)cRef;
    if (PF == PF_BOTH) {
      agg[ALERT_AGG_OR_ENERGY] = G.oe; agg[ALERT_AGG_OR_ENERGY_C] = G.oec;
      agg[ALERT_AGG_OR_ACC] = G.oa; agg[ALERT_AGG_OR_ACC_C] = G.oac;
      agg[ALERT_AGG_OR_VIOL_LAT] += (double)oVL;
      agg[ALERT_AGG_OR_VIOL_ACC] += (double)oVA;
      agg[ALERT_AGG_OR_VIOL_ENERGY] += (double)oVE;
      agg[ALERT_AGG_OR_SAME] += (double)oSame;
    }
  }
}

struct StepParams {
  DevTable T;
  AlertFilterConfig cfg;
  const AlertSpec* specs;
  int n_specs;
  const int32_t* stream_spec;
  AlertState st;
  const double* goal;
  int policy;
  unsigned flags;
  int kinds;
  long long n;
};

// AlertPolicy.decide for n streams (one tile each).
template <int W>
__global__ void __launch_bounds__(256) decide_kernel(const StepParams P, uint32_t* decision) {
  extern __shared__ float4 smem[];
  const DevTable& T = P.T;
  float4* sA = smem;
  float4* sB = smem + T.n_cells;
  int2* sCol = reinterpret_cast<int2*>(sB + T.n_cells);
  load_table_smem(T, sA, sB, sCol);
  auto tile = cg::tiled_partition<W>(cg::this_thread_block());
  const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / W;
  if (i >= P.n) return;
  const int si = P.stream_spec ? P.stream_spec[i] : (int)(i % P.n_specs);
  const AlertSpec spec = P.specs[si];
  StepCtx x;
  make_ctx(x, &spec, P.st.mu[i], P.st.sigma2[i], P.st.phi[i], P.goal[i], P.flags & ALERT_FLAG_FP64_ALL);
  Decision d = alert_decide(T, sA, sB, sCol, tile, x, P.kinds, P.flags & ALERT_FLAG_NO_REFINE);
  if (tile.thread_rank() == 0)
    decision[i] = (uint32_t)__float_as_int(sB[d.cell].z) | ((uint32_t)d.level << 16) | ((uint32_t)d.refined << 26);
}

template <int W>
__global__ void oracle_decide_kernel(const DevTable T, const AlertSpec* specs, int n_specs, const int32_t* stream_spec,
                                     const double* s, const double* idle, const double* goal, uint32_t* decision,
                                     long long n) {
  auto tile = cg::tiled_partition<W>(cg::this_thread_block());
  const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / W;
  if (i >= n) return;
  const int si = stream_spec ? stream_spec[i] : (int)(i % n_specs);
  const AlertSpec spec = specs[si];
  Decision d = oracle_decide(T, tile, &spec, s[i], idle[i], goal[i]);
  if (tile.thread_rank() == 0) decision[i] = (uint32_t)__float_as_int(T.cellB[d.cell].z) | ((uint32_t)d.level << 16);
}


// launchers (defined per W in alert_inst_w*.cu)
template <int W>
cudaError_t launch_run(int pf, const RunParams& P, int tpb, size_t smem, cudaStream_t st);
template <int W>
cudaError_t launch_decide(const StepParams& P, uint32_t* out, int tpb, size_t smem, cudaStream_t st);
template <int W>
cudaError_t launch_oracle(const DevTable& T, const AlertSpec* specs, int n_specs, const int32_t* stream_spec,
                          const double* s, const double* idle, const double* goal, uint32_t* decision,
                          long long n, int tpb, cudaStream_t st);

template <class K>
inline cudaError_t set_smem(K kern, size_t smem) {
  if (smem > 48 * 1024) return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return cudaSuccess;
}

#define ALERT_INSTANTIATE(W)                                                                          \
  template <>                                                                                         \
  cudaError_t launch_run<W>(int pf, const RunParams& P, int tpb, size_t smem, cudaStream_t st) {      \
    long long blocks = ((P.stream_end - P.stream_begin) * W + tpb - 1) / tpb;                        \
    cudaError_t e;                                                                                    \
    if (pf == PF_ORACLE) {                                                                            \
      if ((e = set_smem(run_kernel<W, PF_ORACLE>, smem))) return e;                                   \
      run_kernel<W, PF_ORACLE><<<(unsigned)blocks, tpb, smem, st>>>(P);                               \
    } else if (pf == PF_BOTH) {                                                                       \
      if ((e = set_smem(run_kernel<W, PF_BOTH>, smem))) return e;                                     \
      run_kernel<W, PF_BOTH><<<(unsigned)blocks, tpb, smem, st>>>(P);                                 \
    } else {                                                                                          \
      if ((e = set_smem(run_kernel<W, PF_ALERT>, smem))) return e;                                    \
      run_kernel<W, PF_ALERT><<<(unsigned)blocks, tpb, smem, st>>>(P);                                \
    }                                                                                                 \
    return cudaGetLastError();                                                                        \
  }                                                                                                   \
  template <>                                                                                         \
  cudaError_t launch_decide<W>(const StepParams& P, uint32_t* out, int tpb, size_t smem, cudaStream_t st) { \
    cudaError_t e;                                                                                    \
    if ((e = set_smem(decide_kernel<W>, smem))) return e;                                             \
    long long blocks = (P.n * W + tpb - 1) / tpb;                                                     \
    decide_kernel<W><<<(unsigned)blocks, tpb, smem, st>>>(P, out);                                    \
    return cudaGetLastError();                                                                        \
  }                                                                                                   \
  template <>                                                                                         \
  cudaError_t launch_oracle<W>(const DevTable& T, const AlertSpec* specs, int n_specs,                \
                               const int32_t* stream_spec, const double* s, const double* idle,       \
                               const double* goal, uint32_t* decision, long long n, int tpb,         \
                               cudaStream_t st) {                                                     \
    long long blocks = (n * W + tpb - 1) / tpb;                                                       \
    oracle_decide_kernel<W><<<(unsigned)blocks, tpb, 0, st>>>(T, specs, n_specs, stream_spec, s, idle, goal, \
                                                             decision, n);                           \
    return cudaGetLastError();                                                                        \
  }

}  // namespace alert
