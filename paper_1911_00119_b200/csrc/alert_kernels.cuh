// alert_kernels.cuh — kernel templates of the fused scheduling loop and the
// per-step decide / oracle kernels; instantiated per lane width W in
// alert_inst_w*.cu (compiled in parallel) and dispatched from alert_capi.cu.
#pragma once
#include <cuda_runtime.h>

#include "alert_device.cuh"

namespace alert {

constexpr int kIdleTab = 96;       // entries of the idle-filter gain table
constexpr int kSpecSmemMax = 64;   // specs staged in shared memory up to this count
constexpr int kC64SmemMax = 1024;  // FP64 cell rows staged in shared memory up to this count
constexpr int kRatioSmemMax = 64;  // powers of the per-segment idle-ratio table

struct RunParams {
  DevTable T;
  AlertFilterConfig cfg;
  const SpecDev* specs;
  int n_specs;
  const int32_t* stream_spec;
  AlertTrace tr;
  AlertState st;
  AlertOutputs out;
  int policy;
  unsigned flags;
  int kinds;
  int c64_smem, ratio_smem, sv_smem;  // staging decisions (host computed)
  long long stream_begin, stream_end, step_begin, step_end;
  // Idle-filter gains (estimator.py:123-125) do not depend on the data: the
  // sequence M_k (state after k updates from m0) and W_k reaches an exact FP64
  // fixed point at k = idle_fix; M/W are precomputed on the host with the
  // reference's operations.  idle_fix < 0: table unused (division path).
  int idle_fix;
  double idle_w[kIdleTab];
  double idle_m[kIdleTab];
};

// Shared-memory layout of run_kernel (host and device compute it identically).
struct SmemLayout {
  size_t B, col, spec, c64, ratio, agg, sv, slot, total;
  __host__ __device__ static size_t up16(size_t x) { return (x + 15) & ~size_t(15); }
  // pad = look-ahead rows past the end of the cell / column tables for a tile
  // width W: 2 chunks of 4 cells (see cell_pass), so 8 W + 8.
  __host__ __device__ static int pad_rows(int W) { return 8 * W + 8; }
  __host__ __device__ SmemLayout(int n_cells, int n_cols, int n_spec, int n_c64, int n_tiles, int n_ratio,
                                 size_t agg_bytes, int n_sv, int W) {
    B = sizeof(float4) * (size_t)(n_cells + pad_rows(W));
    col = B + sizeof(float4) * (size_t)n_cells;
    spec = up16(col + sizeof(int2) * (size_t)(n_cols + pad_rows(W)));
    c64 = up16(spec + sizeof(SpecDev) * (size_t)n_spec);
    ratio = up16(c64 + sizeof(Cell64) * (size_t)n_c64);
    agg = up16(ratio + sizeof(double) * (size_t)n_tiles * (size_t)n_ratio);
    sv = up16(agg + agg_bytes * (size_t)n_tiles);
    slot = up16(sv + sizeof(float) * (size_t)n_tiles * (size_t)n_sv);
    total = up16(slot + 16 * (size_t)n_tiles * (size_t)W);  // two 8-byte trace slots per thread
  }
};

__device__ __forceinline__ void load_table_smem(const DevTable& T, float4* sA, float4* sB, int2* sCol) {
  for (int i = threadIdx.x; i < T.n_cells; i += blockDim.x) {
    sA[i] = T.cellA[i];
    sB[i] = T.cellB[i];
  }
  for (int i = threadIdx.x; i < T.n_any_cols; i += blockDim.x) sCol[i] = T.any_cols[i];
}

// The trace value is prefetched one step ahead as RAW bits and converted only
// when consumed, so the load latency overlaps a whole step of scan work.
__device__ __forceinline__ unsigned long long load_s_raw(const AlertTrace& tr, long long row, long long n) {
  const long long off = row * tr.row_stride + (n - tr.step_offset) * tr.step_stride;
  if (tr.slowdown_dtype == ALERT_DTYPE_F64)
    return __ldg(reinterpret_cast<const unsigned long long*>(tr.slowdown) + off);
  return __ldg(reinterpret_cast<const unsigned int*>(tr.slowdown) + off);
}
__device__ __forceinline__ double s_of_raw(const AlertTrace& tr, unsigned long long raw) {
  return tr.slowdown_dtype == ALERT_DTYPE_F64 ? __longlong_as_double((long long)raw)
                                              : (double)__uint_as_float((unsigned int)raw);
}

__device__ __forceinline__ void prefetch_s(unsigned dst, const char* src, bool f64) {
  if (f64)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\ncp.async.commit_group;\n" ::"r"(dst), "l"(src)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\ncp.async.commit_group;\n" ::"r"(dst), "l"(src)
                 : "memory");
}

// Per-tile accumulators in shared memory (touched once per step by the tile's
// writer lane, never per candidate).  Float sums are Neumaier pairs (CPython
// 3.12 sum()); counts are int deltas since the current segment started.
struct TileAgg {
  double e, ec, a, ac;      // overall energy / delivered accuracy
  double pe, pec, pa, pac;  // current phase (loaded / stored at segment changes)
  double oe, oec, oa, oac;  // oracle alongside
  int dn, dvl, dva, dve;    // current segment counts
  int l1, l2, ref, osame;   // launch totals
  int ovl, ova, ove, pad;
};

enum { PF_ALERT = 0, PF_ORACLE = 1, PF_BOTH = 2 };  // policy families

// Close the current segment: per-phase slot (phase ids < ALERT_MAX_PHASES) and
// overall violation counts.
__device__ __forceinline__ void flush_segment(TileAgg& g, double* agg, int phase) {
  if (phase >= 0 && phase < ALERT_MAX_PHASES) {
    double* p = agg + ALERT_AGG_PHASE_BASE + ALERT_AGG_PHASE_STRIDE * phase;
    p[0] += (double)g.dn;
    p[1] = g.pe; p[2] = g.pec; p[3] = g.pa; p[4] = g.pac;
    p[5] += (double)g.dvl; p[6] += (double)g.dva; p[7] += (double)g.dve;
  }
  agg[ALERT_AGG_VIOL_LAT] += (double)g.dvl;
  agg[ALERT_AGG_VIOL_ACC] += (double)g.dva;
  agg[ALERT_AGG_VIOL_ENERGY] += (double)g.dve;
  g.dn = g.dvl = g.dva = g.dve = 0;
}
__device__ __forceinline__ void open_segment(TileAgg& g, const double* agg, int phase) {
  if (phase >= 0 && phase < ALERT_MAX_PHASES) {
    const double* p = agg + ALERT_AGG_PHASE_BASE + ALERT_AGG_PHASE_STRIDE * phase;
    g.pe = p[1]; g.pec = p[2]; g.pa = p[3]; g.pac = p[4];
  } else {
    g.pe = g.pec = g.pa = g.pac = 0.0;
  }
}

// min(1, idle / cap) for every power of the current segment (estimator.py:123),
// lanes of the tile split the powers.
template <class Tile>
__device__ __forceinline__ void fill_ratios(const DevTable& T, const Tile& tile, double* r, double idle) {
  for (int j = tile.thread_rank(); j < T.n_powers; j += Tile::num_threads())
    r[j] = py_min(1.0, xdiv(idle, T.power_cap64[j]));
  tile.sync();
}

// The fused closed loop (simulator.run, simulator.py:461-507): one tile of W
// lanes per stream, filter state in registers for the whole step range.
template <int W, int PF>
__global__ void __launch_bounds__(256, 2) run_kernel(const RunParams P) {
  extern __shared__ float4 smem[];
  const DevTable& T = P.T;
  const int n_tiles = blockDim.x / W;
  const SmemLayout L(T.n_cells, T.n_any_cols, n_tiles, P.c64_smem ? T.n_cells : 0, n_tiles,
                     P.ratio_smem ? T.n_powers : 0, sizeof(TileAgg), P.sv_smem ? T.n_cells : 0, W);
  char* base = reinterpret_cast<char*>(smem);
  float4* sA = smem;
  float4* sB = reinterpret_cast<float4*>(base + L.B);
  int2* sCol = reinterpret_cast<int2*>(base + L.col);
  SpecDev* sSpec = reinterpret_cast<SpecDev*>(base + L.spec);
  Cell64* sC64 = reinterpret_cast<Cell64*>(base + L.c64);
  double* sRatio = reinterpret_cast<double*>(base + L.ratio);
  TileAgg* sAgg = reinterpret_cast<TileAgg*>(base + L.agg);
  float* sV = reinterpret_cast<float*>(base + L.sv);
  load_table_smem(T, sA, sB, sCol);
  if (P.c64_smem)
    for (int i = threadIdx.x; i < T.n_cells; i += blockDim.x) sC64[i] = T.c64[i];
  __syncthreads();
  const Cell64* C64 = P.c64_smem ? sC64 : T.c64;

  auto tile = cg::tiled_partition<W>(cg::this_thread_block());
  const long long stream = P.stream_begin + ((long long)blockIdx.x * blockDim.x + threadIdx.x) / W;
  if (stream >= P.stream_end) return;
  const bool writer = tile.thread_rank() == 0;
  TileAgg& G = sAgg[threadIdx.x / W];
  double* ratio_tab = P.ratio_smem ? sRatio + (size_t)(threadIdx.x / W) * T.n_powers : nullptr;
  const unsigned sv_tile = (unsigned)__cvta_generic_to_shared(sV + (size_t)(threadIdx.x / W) * T.n_cells);

  const int si = P.stream_spec ? P.stream_spec[stream] : (int)(stream % P.n_specs);
  // the stream's spec, copied once into the tile's shared slot (all per-step
  // spec reads are then shared-memory loads)
  SpecDev* spec = sSpec + threadIdx.x / W;
  {
    const float4* src = reinterpret_cast<const float4*>(P.specs + si);
    float4* dst = reinterpret_cast<float4*>(spec);
    for (int k = tile.thread_rank(); k < (int)(sizeof(SpecDev) / 16); k += W) dst[k] = src[k];
    tile.sync();
  }
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
  bool k_valid = false;  // k_gain == sigma2 / (sigma2 + r) holds after one update here
  int ik = -1;           // position in the idle-filter gain table
  if (P.idle_fix >= 0)
    for (int k = 0; k <= P.idle_fix; ++k)
      if (P.idle_m[k] == f.m_var) { ik = k; break; }
  double budget = P.st.group_budget[stream];
  int count = P.st.group_count[stream];
  const int group_size = spec->group_size;

  // segment (phase) tracking
  const int nseg = tr.n_segments[row];
  const long long seg0 = row * tr.max_segments;  // segment arrays are re-read only at segment changes
  int seg = 0;
  while (seg + 1 < nseg && P.step_begin >= tr.seg_end[seg0 + seg]) ++seg;
  int cur_end = tr.seg_end[seg0 + seg];
  int phase = tr.seg_phase[seg0 + seg];
  double idle = tr.seg_idle[seg0 + seg];
  if (ratio_tab) fill_ratios(T, tile, ratio_tab, idle);

  double* agg = P.out.agg ? P.out.agg + stream * ALERT_AGG_FIELDS : nullptr;
  if (writer && agg) {
    G = TileAgg{};
    G.e = agg[ALERT_AGG_ENERGY]; G.ec = agg[ALERT_AGG_ENERGY_C];
    G.a = agg[ALERT_AGG_ACC]; G.ac = agg[ALERT_AGG_ACC_C];
    if (PF == PF_BOTH) {
      G.oe = agg[ALERT_AGG_OR_ENERGY]; G.oec = agg[ALERT_AGG_OR_ENERGY_C];
      G.oa = agg[ALERT_AGG_OR_ACC]; G.oac = agg[ALERT_AGG_OR_ACC_C];
    }
    open_segment(G, agg, phase);
  }

  const int kinds = P.kinds;
  const bool fp64_all = P.flags & ALERT_FLAG_FP64_ALL;
  const bool no_refine = P.flags & ALERT_FLAG_NO_REFINE;
  const int* forced = P.out.forced;

  // Trace prefetch: the next step's slow-down is copied global -> shared with
  // cp.async (LDGSTS) into one of two per-thread slots, so no register is held
  // across the step and the load latency hides behind a whole step of work.
  unsigned long long* slot = reinterpret_cast<unsigned long long*>(base + L.slot) + 2 * threadIdx.x;
  const unsigned slot_sa = (unsigned)__cvta_generic_to_shared(slot);
  const bool f64 = tr.slowdown_dtype == ALERT_DTYPE_F64;
  const int esz = f64 ? 8 : 4;
  const char* sptr = static_cast<const char*>(tr.slowdown) +
                     (row * tr.row_stride + (P.step_begin - tr.step_offset) * tr.step_stride) * esz;
  const long long sinc = tr.step_stride * esz;
  prefetch_s(slot_sa, sptr, f64);
  const int nsteps = (int)(P.step_end - P.step_begin);
  for (int i = 0; i < nsteps; ++i) {
    const long long n = P.step_begin + i;
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    const unsigned long long s_raw = slot[i & 1];
    if (i + 1 < nsteps) {
      sptr += sinc;
      prefetch_s(slot_sa + 8u * ((i + 1) & 1), sptr, f64);
    }
    if (n >= cur_end && seg + 1 < nseg) {
      if (agg && writer) flush_segment(G, agg, phase);
      while (seg + 1 < nseg && n >= cur_end) {
        ++seg;
        cur_end = tr.seg_end[seg0 + seg];
      }
      phase = tr.seg_phase[seg0 + seg];
      idle = tr.seg_idle[seg0 + seg];
      if (ratio_tab) fill_ratios(T, tile, ratio_tab, idle);
      if (agg && writer) open_segment(G, agg, phase);
    }
    // adjust_goal (selector.py:48-70) with group budgets (simulator.py:473-483)
    double goal, period;
    if (group_size > 0) {
      if (count == 0) {
        budget = xmul((double)group_size, spec->t_goal);
        count = group_size;
      }
      goal = py_max(xsub(xdiv(budget, (double)count), spec->oh), 0.001);
      period = xadd(goal, spec->oh);
    } else {
      goal = spec->goal0;
      period = spec->period0;
    }

    Decision d;
    double s;  // true slow-down of this input: consumed only after the decision
    if (PF == PF_ORACLE) {
      s = s_of_raw(tr, s_raw);
      d = oracle_decide(T, sA, sB, C64, sCol, tile, spec, s, idle, goal, fp64_all);
    } else {
      StepCtx x;
      make_ctx(x, spec, C64, f.mu, f.sigma2, f.phi, goal, fp64_all);
      x.sv = sv_tile;
      x.has_sv = P.sv_smem;
      d = alert_decide(T, sA, sB, sCol, tile, x, kinds, no_refine);
      s = s_of_raw(tr, s_raw);
    }
    int exec_cell = d.cell;
    if (forced) {
      const int fc = forced[stream * P.out.stream_stride + n * P.out.step_stride];
      if (fc >= 0) exec_cell = T.cell_of_cand[fc];
    }
    const Outcome o = execute_measure(sB, C64, spec, exec_cell, s, goal, period, idle);
    if (PF != PF_ORACLE) {  // AlertPolicy.observe, policies.py:105-108
      slowdown_update(P.cfg, f, o.fb_latency, o.fb_t_prof, k_valid);
      const int pw = __float_as_uint(sB[exec_cell].y) >> 20;  // power index from the tie key
      const double ratio = ratio_tab ? ratio_tab[pw] : py_min(1.0, xdiv(idle, C64[exec_cell].cap));
      idle_update(P.cfg, f, ratio, ik, P.idle_fix, P.idle_w, P.idle_m);
    }
    if (group_size > 0) {  // simulator.py:501-503
      budget = xsub(budget, o.latency);
      count -= 1;
    }
    const AlertOutputs& out = P.out;
    if (writer && out.decision) {
      const long long oidx = stream * out.stream_stride + n * out.step_stride;
      out.decision[oidx] = pack_decision(cell_cand(sB[d.cell]), d.level, o, d.refined, phase);
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
    if (writer && agg) {  // aggregates in step order (CPython 3.12 sum() semantics)
      neumaier(G.e, G.ec, o.energy);
      neumaier(G.a, G.ac, o.delivered);
      neumaier(G.pe, G.pec, o.energy);
      neumaier(G.pa, G.pac, o.delivered);
      G.dn += 1;
      G.dvl += o.vl; G.dva += o.va; G.dve += o.ve;
      G.l1 += d.level == 1; G.l2 += d.level == 2;
      G.ref += d.refined;
    }
    if (PF == PF_BOTH) {  // OraclePolicy alongside on the same step
      Decision od = oracle_decide(T, sA, sB, C64, sCol, tile, spec, s, idle, goal, fp64_all);
      const Outcome oo = execute_measure(sB, C64, spec, od.cell, s, goal, period, idle);
      if (writer && agg) {
        neumaier(G.oe, G.oec, oo.energy);
        neumaier(G.oa, G.oac, oo.delivered);
        G.ovl += oo.vl; G.ova += oo.va; G.ove += oo.ve;
        G.osame += od.cell == exec_cell;
      }
      if (writer && out.oracle_decision)
        out.oracle_decision[stream * out.stream_stride + n * out.step_stride] =
            pack_decision(cell_cand(sB[od.cell]), od.level, oo, false, phase);
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
    flush_segment(G, agg, phase);
    const double steps = (double)(P.step_end - P.step_begin);
    agg[ALERT_AGG_N] += steps;
    agg[ALERT_AGG_ENERGY] = G.e; agg[ALERT_AGG_ENERGY_C] = G.ec;
    agg[ALERT_AGG_ACC] = G.a; agg[ALERT_AGG_ACC_C] = G.ac;
    agg[ALERT_AGG_LEVEL0] += steps - (double)G.l1 - (double)G.l2;
    agg[ALERT_AGG_LEVEL1] += (double)G.l1;
    agg[ALERT_AGG_LEVEL2] += (double)G.l2;
    agg[ALERT_AGG_REFINED] += (double)G.ref;
    if (PF == PF_BOTH) {
      agg[ALERT_AGG_OR_ENERGY] = G.oe; agg[ALERT_AGG_OR_ENERGY_C] = G.oec;
      agg[ALERT_AGG_OR_ACC] = G.oa; agg[ALERT_AGG_OR_ACC_C] = G.oac;
      agg[ALERT_AGG_OR_VIOL_LAT] += (double)G.ovl;
      agg[ALERT_AGG_OR_VIOL_ACC] += (double)G.ova;
      agg[ALERT_AGG_OR_VIOL_ENERGY] += (double)G.ove;
      agg[ALERT_AGG_OR_SAME] += (double)G.osame;
    }
  }
}

struct StepParams {
  DevTable T;
  AlertFilterConfig cfg;
  const SpecDev* specs;
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
  const SmemLayout L(T.n_cells, T.n_any_cols, 0, 0, 0, 0, 0, 0, W);
  char* base = reinterpret_cast<char*>(smem);
  float4* sA = smem;
  float4* sB = reinterpret_cast<float4*>(base + L.B);
  int2* sCol = reinterpret_cast<int2*>(base + L.col);
  load_table_smem(T, sA, sB, sCol);
  __syncthreads();
  auto tile = cg::tiled_partition<W>(cg::this_thread_block());
  const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / W;
  if (i >= P.n) return;
  const int si = P.stream_spec ? P.stream_spec[i] : (int)(i % P.n_specs);
  const SpecDev* spec = P.specs + si;
  StepCtx x;
  make_ctx(x, spec, T.c64, P.st.mu[i], P.st.sigma2[i], P.st.phi[i], P.goal[i], P.flags & ALERT_FLAG_FP64_ALL);
  Decision d = alert_decide(T, sA, sB, sCol, tile, x, P.kinds, P.flags & ALERT_FLAG_NO_REFINE);
  if (tile.thread_rank() == 0)
    decision[i] = (uint32_t)cell_cand(sB[d.cell]) | ((uint32_t)d.level << 16) | ((uint32_t)d.refined << 26);
}

template <int W>
__global__ void oracle_decide_kernel(const DevTable T, const SpecDev* specs, int n_specs, const int32_t* stream_spec,
                                     const double* s, const double* idle, const double* goal, uint32_t* decision,
                                     long long n, bool fp64_all) {
  auto tile = cg::tiled_partition<W>(cg::this_thread_block());
  const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / W;
  if (i >= n) return;
  const int si = stream_spec ? stream_spec[i] : (int)(i % n_specs);
  Decision d = oracle_decide(T, T.cellA, T.cellB, T.c64, T.any_cols, tile, specs + si, s[i], idle[i], goal[i], fp64_all);
  if (tile.thread_rank() == 0) decision[i] = (uint32_t)cell_cand(T.cellB[d.cell]) | ((uint32_t)d.level << 16);
}


// launchers (defined per W in alert_inst_w*.cu)
template <int W>
cudaError_t launch_run(int pf, const RunParams& P, int tpb, size_t smem, cudaStream_t st);
template <int W>
cudaError_t launch_decide(const StepParams& P, uint32_t* out, int tpb, size_t smem, cudaStream_t st);
template <int W>
cudaError_t launch_oracle(const DevTable& T, const SpecDev* specs, int n_specs, const int32_t* stream_spec,
                          const double* s, const double* idle, const double* goal, uint32_t* decision,
                          long long n, int tpb, unsigned flags, cudaStream_t st);

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
  cudaError_t launch_oracle<W>(const DevTable& T, const SpecDev* specs, int n_specs,                  \
                               const int32_t* stream_spec, const double* s, const double* idle,       \
                               const double* goal, uint32_t* decision, long long n, int tpb,         \
                               unsigned flags, cudaStream_t st) {                                     \
    long long blocks = (n * W + tpb - 1) / tpb;                                                       \
    oracle_decide_kernel<W><<<(unsigned)blocks, tpb, 0, st>>>(T, specs, n_specs, stream_spec, s, idle, goal, \
                                                             decision, n, flags & ALERT_FLAG_FP64_ALL);  \
    return cudaGetLastError();                                                                        \
  }

}  // namespace alert
