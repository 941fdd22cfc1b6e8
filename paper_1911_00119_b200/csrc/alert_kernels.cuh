// alert_kernels.cuh — kernel templates of the fused scheduling loop and the
// per-step decide / oracle kernels; instantiated per lane width W in
// alert_inst_w*.cu (compiled in parallel) and dispatched from alert_capi.cu.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

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
  int min_energy_only;                 // every spec minimises energy: MS_MIN_ENERGY kernel
  int any_min_energy;                  // some spec minimises energy (per-tile z-threshold slots needed)
  int max_accuracy_only;               // every spec maximises accuracy: MS_MAX_ACCURACY kernel (W = 1, 8)
  int spec_shared;                     // all specs staged once per block (few specs), not per tile
  // min-energy fast scan: per (spec, traditional DNN) z-thresholds, row
  // stride n_tdnn + 1 (last = pr_threshold bound), from zlo_kernel; null = off
  const float* zlo;
  int fast_smem;  // host: shared-memory slots for the fast scan staged
  int fast_rows;  // fast scan in row mode (large tables): no staged rows / thresholds
  int units_smem; // max-accuracy fast scan: bound-sorted units staged in shared memory
  long long stream_begin, stream_end, step_begin, step_end;
  // persistent scheduling: warps claim the next 32 / W streams from this
  // counter (zeroed per launch) as they finish; null = static grid stride
  unsigned long long* work;
  // Idle-filter gains (estimator.py:123-125) do not depend on the data: the
  // sequence M_k (state after k updates from m0) and W_k reaches an exact FP64
  // fixed point at k = idle_fix; M/W are precomputed on the host with the
  // reference's operations.  idle_fix < 0: table unused (division path).
  int idle_fix;
  double idle_w[kIdleTab];
  double idle_m[kIdleTab];
};

// Per-thread cold state of run_kernel (shared memory): touched at segment
// changes, by group specs, and once per step for the idle power.
struct ColdState {
  double budget, idle;
  long long seg0, gseg0;
  int count, seg, nseg, phase;
  int gseg, ngseg, gend, si;  // goal-change cursor (AlertTrace.goal_*), current spec index
};

// Goal changes (AlertTrace.goal_*): the segment of `row` holding step n and its end.
__device__ __forceinline__ int goal_seek(const AlertTrace& tr, long long gseg0, int ng, int g, long long n) {
  while (g + 1 < ng && n >= tr.goal_seg_end[gseg0 + g]) ++g;
  return g;
}
__device__ __forceinline__ int goal_end(const AlertTrace& tr, long long gseg0, int ng, int g) {
  return g + 1 < ng ? tr.goal_seg_end[gseg0 + g] : 0x7fffffff;
}

// Shared-memory layout of run_kernel (host and device compute it identically).
struct SmemLayout {
  size_t B, col, spec, c64, ratio, agg, sv, fz, ff, wst, un, cold, slot, total;
  __host__ __device__ static size_t up16(size_t x) { return (x + 15) & ~size_t(15); }
  // pad = look-ahead rows past the end of the cell / column tables for a tile
  // width W: 2 chunks of 4 cells (see cell_pass), so 8 W + 8.
  __host__ __device__ static int pad_rows(int W) { return 8 * W + 8; }
  __host__ __device__ SmemLayout(int n_cells, int n_cols, int n_spec, int n_c64, int n_tiles, int n_ratio,
                                 size_t agg_bytes, int n_sv, int W, int n_fz = 0, int n_ff = 0,
                                 bool flat = false, int n_un = 0, int n_sq = 0) {
    B = sizeof(float4) * (size_t)(n_cells + pad_rows(W));
    col = B + sizeof(float4) * (size_t)n_cells;
    spec = up16(col + sizeof(int2) * (size_t)(n_cols + pad_rows(W)));
    c64 = up16(spec + sizeof(SpecDev) * (size_t)n_spec);
    ratio = up16(c64 + sizeof(Cell64) * (size_t)n_c64);
    agg = up16(ratio + sizeof(double) * (size_t)n_tiles * (size_t)n_ratio);
    sv = up16(agg + agg_bytes * (size_t)n_tiles);
    fz = up16(sv + sizeof(float) * (size_t)n_tiles * (size_t)n_sv);  // [n_fz][n_tiles]: the tiles' z' copies
    ff = up16(fz + sizeof(float) * (size_t)n_tiles * (size_t)n_fz);  // fast-scan traditional cells
    wst = up16(ff + (flat ? sizeof(float4) * (size_t)(n_ff + pad_rows(W)) : 0));
    un = up16(wst + (flat ? sizeof(unsigned) * (size_t)(n_cells / 32 + 2) : 0));  // sequence, units, lbs
    cold = up16(un + 2 * sizeof(float4) * (size_t)n_sq + (sizeof(int2) + sizeof(float)) * (size_t)n_un);
    slot = up16(cold + sizeof(ColdState) * (size_t)n_tiles * (size_t)W);
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
  int dn, dvl, dva, dve;    // current segment counts
  int l1, l2, ref, full;    // launch totals
  int tvl, tva, tve, seen;  // ALERT_FLAG_FRESH: violation totals, phases whose slot is written
};
struct TileAggOr : TileAgg {  // + the oracle alongside (PF_BOTH kernels only)
  double oe, oec, oa, oac;
  int ovl, ova, ove, osame;
};

enum { PF_ALERT = 0, PF_ORACLE = 1, PF_BOTH = 2 };  // policy families


// Close the current segment: per-phase slot (phase ids < ALERT_MAX_PHASES) and
// overall violation counts.
// With ALERT_FLAG_FRESH the block is written, never read: a phase slot's
// first flush stores, a recurring phase's adds to what this launch stored,
// the overall counts stay in the tile until the end (finish_fresh).
__device__ __forceinline__ void flush_segment(TileAgg& g, double* agg, int phase, bool fresh) {
  if (phase >= 0 && phase < ALERT_MAX_PHASES) {
    double* p = agg + ALERT_AGG_PHASE_BASE + ALERT_AGG_PHASE_STRIDE * phase;
    if (fresh && !((g.seen >> phase) & 1)) {
      p[0] = (double)g.dn;
      p[5] = (double)g.dvl; p[6] = (double)g.dva; p[7] = (double)g.dve;
      g.seen |= 1 << phase;
    } else {
      p[0] += (double)g.dn;
      p[5] += (double)g.dvl; p[6] += (double)g.dva; p[7] += (double)g.dve;
    }
    p[1] = g.pe; p[2] = g.pec; p[3] = g.pa; p[4] = g.pac;
  }
  if (fresh) {
    g.tvl += g.dvl; g.tva += g.dva; g.tve += g.dve;
  } else {
    agg[ALERT_AGG_VIOL_LAT] += (double)g.dvl;
    agg[ALERT_AGG_VIOL_ACC] += (double)g.dva;
    agg[ALERT_AGG_VIOL_ENERGY] += (double)g.dve;
  }
  g.dn = g.dvl = g.dva = g.dve = 0;
}
__device__ __forceinline__ void open_segment(TileAgg& g, const double* agg, int phase, bool fresh) {
  if (fresh && phase >= 0 && phase < ALERT_MAX_PHASES && !((g.seen >> phase) & 1)) {
    g.pe = g.pec = g.pa = g.pac = 0.0;
  } else if (phase >= 0 && phase < ALERT_MAX_PHASES) {
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
  tile.sync();  // every lane is done reading the previous segment's ratios (racecheck)
  for (int j = tile.thread_rank(); j < T.n_powers; j += Tile::num_threads())
    r[j] = py_min(1.0, xdiv(idle, T.power_cap64[j]));
  tile.sync();
}

// The fused closed loop (simulator.run, simulator.py:461-507): one tile of W
// lanes per stream, filter state in registers for the whole step range.
// Register budget: 128 (16 warps / SM).  ALERT_MINE_REGS overrides it for
// the min-energy-only kernel; 144 was measured slower (the register file is
// split per SMSP, so 144 leaves 3 warps / scheduler and c2 needs two waves).
#ifndef ALERT_MINE_REGS
#define ALERT_MINE_REGS 128
#endif
#ifndef ALERT_ALL_REGS
#define ALERT_ALL_REGS 128
#endif
template <int W, int PF, int MS>
__global__ void __launch_bounds__(512) __maxnreg__(MS == MS_MIN_ENERGY ? ALERT_MINE_REGS : ALERT_ALL_REGS)
    run_kernel(const RunParams P) {
  extern __shared__ float4 smem[];
  const DevTable& T = P.T;
  const int n_tiles = blockDim.x / W;
  const int n_tdnn = T.n_trad / T.n_powers;
  using Agg = typename std::conditional<PF == PF_BOTH, TileAggOr, TileAgg>::type;
  const SmemLayout L(T.n_cells, T.n_any_cols, P.spec_shared ? P.n_specs : n_tiles, P.c64_smem ? T.n_cells : 0,
                     n_tiles, P.ratio_smem ? T.n_powers : 0, sizeof(Agg), P.sv_smem ? T.n_cells : 0, W,
                     (P.zlo && !P.fast_rows && P.any_min_energy) ? T.n_trad : 0, (P.zlo && !P.fast_rows) ? T.n_trad : 0,
                     P.zlo && !P.fast_rows, P.units_smem ? T.n_units : 0, P.units_smem ? T.n_seq : 0);
  char* base = reinterpret_cast<char*>(smem);
  float4* sA = smem;
  float4* sB = reinterpret_cast<float4*>(base + L.B);
  int2* sCol = reinterpret_cast<int2*>(base + L.col);
  SpecDev* sSpec = reinterpret_cast<SpecDev*>(base + L.spec);
  Cell64* sC64 = reinterpret_cast<Cell64*>(base + L.c64);
  double* sRatio = reinterpret_cast<double*>(base + L.ratio);
  Agg* sAgg = reinterpret_cast<Agg*>(base + L.agg);
  if (P.spec_shared)  // few specs: one shared copy per block, a tile's spec is a pointer into it
    for (int i = threadIdx.x; i < P.n_specs * (int)(sizeof(SpecDev) / 16); i += blockDim.x)
      reinterpret_cast<float4*>(sSpec)[i] = reinterpret_cast<const float4*>(P.specs)[i];
  float* sV = reinterpret_cast<float*>(base + L.sv);
  ColdState* sCold = reinterpret_cast<ColdState*>(base + L.cold);
  load_table_smem(T, sA, sB, sCol);
  if (P.c64_smem)
    for (int i = threadIdx.x; i < T.n_cells; i += blockDim.x) sC64[i] = T.c64[i];
  float4* sF = reinterpret_cast<float4*>(base + L.ff);
  if (P.zlo && !P.fast_rows)  // fast-scan rows {1/t, cap t, byte offset of the DNN threshold, (c / W) & 7}, padded
    for (int i = threadIdx.x; i < T.n_trad + SmemLayout::pad_rows(W); i += blockDim.x) {
      const bool in = i < T.n_trad;
      const int off = in ? (i / T.n_powers) * n_tiles * (int)sizeof(float) : 0;
      sF[i] = make_float4(in ? T.cellA[i].x : 0.f, in ? T.cellA[i].y : 0.f, __int_as_float(off),
                          __int_as_float((i / W) & 7));
    }
  float4* sQA = reinterpret_cast<float4*>(base + L.un);
  float4* sQM = sQA + (P.units_smem ? T.n_seq : 0);
  int2* sUn = reinterpret_cast<int2*>(sQM + (P.units_smem ? T.n_seq : 0));
  const int n_seq = T.n_seqk[P.kinds & 3];  // the policy's kinds sequence
  float* sLb = reinterpret_cast<float*>(sUn + (P.units_smem ? T.n_units : 0));
  if (P.units_smem) {
    for (int i = threadIdx.x; i < T.n_units; i += blockDim.x) {
      sUn[i] = T.units[i];
      sLb[i] = T.unit_lb[i];
    }
    const int off = ((P.kinds & 3) - 1) * T.n_seq;
    for (int i = threadIdx.x; i < n_seq; i += blockDim.x) {
      sQA[i] = T.useqA[off + i];
      sQM[i] = T.useqM[off + i];
    }
  }
  unsigned* sWst = reinterpret_cast<unsigned*>(base + L.wst);
  if (P.zlo && !P.fast_rows)  // column-start bits of the anytime cells, per 32-cell window
    for (int w = threadIdx.x; w * 32 < T.n_cells - T.n_trad; w += blockDim.x) {
      unsigned b = 0;
      for (int u = 0; u < 32 && T.n_trad + w * 32 + u < T.n_cells; ++u)
        b |= (unsigned)(T.cellA[T.n_trad + w * 32 + u].w >= 0.0f) << u;
      sWst[w] = b;
    }
  __syncthreads();
  const Cell64* C64 = P.c64_smem ? sC64 : T.c64;

  auto tile = cg::tiled_partition<W>(cg::this_thread_block());
  // Persistent: the grid is sized to the resident blocks (launch_persistent),
  // the table is staged once per block, and each tile runs stream after
  // stream: warps claim the next 32 / W streams from a per-launch counter
  // (P.work) as they finish, or grid-stride when it is null.  The loop body
  // is written inline (a lambda here is not always inlined: a call with a
  // 3 KB stack frame in the oracle-alongside kernel).
  const bool dyn = P.work != nullptr;
  const int tw = (threadIdx.x & 31) / W;  // tile index within the warp
  auto claim = [&]() -> long long {  // dynamic: the warp's next 32 / W streams
    unsigned long long b = 0;
    if ((threadIdx.x & 31) == 0) b = atomicAdd(P.work, (unsigned long long)(32 / W));
    return (long long)__shfl_sync(0xffffffffu, b, 0);
  };
  const long long span = (long long)gridDim.x * (blockDim.x / W);
  for (long long cur = dyn ? claim() : P.stream_begin + ((long long)blockIdx.x * blockDim.x + threadIdx.x) / W;;
       cur = dyn ? claim() : cur + span) {
  // dynamic: the warp stops together once its claim starts past the end
  const long long stream_ll = dyn ? P.stream_begin + cur + tw : cur;
  if (dyn ? P.stream_begin + cur >= P.stream_end : stream_ll >= P.stream_end) break;
  if (stream_ll >= P.stream_end) continue;  // the claim's last warp: tiles past the end idle
  const int stream = (int)stream_ll;  // < 2^31 (checked on the host)
  const bool writer = tile.thread_rank() == 0;
  const int tid = threadIdx.x / W;  // tile index in the block
  Agg& G = sAgg[tid];
  // Cold per-stream state (group budget, segment cursor, idle power) lives in
  // the thread's shared slots, not in registers across the step loop: the
  // step loop's register budget goes to the scan.
  ColdState& cs = sCold[threadIdx.x];
  const unsigned sv_tile = (unsigned)__cvta_generic_to_shared(sV + (size_t)tid * T.n_cells);

  const AlertTrace& tr = P.tr;
  const long long row = tr.stream_row ? tr.stream_row[stream] : stream_ll;
  // goal changes: the row's spec segment at step_begin overrides stream_spec
  cs.ngseg = tr.n_goal_segments ? tr.n_goal_segments[row] : 0;
  cs.gseg0 = row * (long long)tr.max_goal_segments;
  cs.gseg = cs.ngseg ? goal_seek(tr, cs.gseg0, cs.ngseg, 0, P.step_begin) : 0;
  cs.gend = cs.ngseg ? goal_end(tr, cs.gseg0, cs.ngseg, cs.gseg) : 0x7fffffff;
  cs.si = cs.ngseg ? tr.goal_seg_spec[cs.gseg0 + cs.gseg]
                   : (P.stream_spec ? P.stream_spec[stream] : (int)(stream_ll % P.n_specs));
  // the stream's spec, copied into the tile's shared slot (all per-step spec
  // reads are then shared-memory loads); again at every goal change.
  // min-energy fast scan: the spec's z-thresholds, copied into the tile's
  // interleaved shared slots (element d at [d * n_tiles + tile])
  const SpecDev* spec = sSpec + tid;
  bool fast = false, fast_me = false;
  float zpr = -kInfF;
  auto stage_spec = [&](int si) {
    if (P.spec_shared) {
      spec = sSpec + si;
    } else {
      const float4* src = reinterpret_cast<const float4*>(P.specs + si);
      float4* dst = reinterpret_cast<float4*>(sSpec + tid);
      tile.sync();  // every lane is done with the previous spec
      for (int k = tile.thread_rank(); k < (int)(sizeof(SpecDev) / 16); k += W) dst[k] = src[k];
      tile.sync();
      spec = sSpec + tid;
    }
    fast = P.zlo && (spec->mode == ALERT_MODE_MIN_ENERGY || T.units);
    fast_me = fast && spec->mode == ALERT_MODE_MIN_ENERGY;  // per-DNN thresholds needed
    zpr = -kInfF;
    if (fast) {
      const float* zrow = P.zlo + (size_t)si * (n_tdnn + 1);
      zpr = zrow[n_tdnn];
      if (!P.fast_rows && fast_me) {
        float* fzZ = reinterpret_cast<float*>(base + L.fz) + tid;
        // one copy per traditional cell (not per DNN): the scan's threshold
        // address does not depend on the cell row it loads
        for (int c = tile.thread_rank(); c < T.n_trad; c += W) fzZ[c * n_tiles] = zrow[c / T.n_powers];
        if (W > 1) tile.sync();
      }
    }
  };
  stage_spec(cs.si);

  // ALERT_FLAG_FRESH: slowdown_init / idle_power_init (estimator.py:47-56,
  // policies.py:90-91) here instead of reading alert_state_init's arrays
  const bool fresh = P.flags & ALERT_FLAG_FRESH;
  Filter f;
  if (fresh) {
    f.mu = P.cfg.mu0;
    f.sigma2 = P.cfg.sigma2_0;
    f.k_gain = P.cfg.k0;
    f.q_noise = P.cfg.q0;
    f.innov = 0.0;
    f.phi = T.phi0;
    f.m_var = P.cfg.m0;
  } else {
    f.mu = P.st.mu[stream];
    f.sigma2 = P.st.sigma2[stream];
    f.k_gain = P.st.k_gain[stream];
    f.q_noise = P.st.q_noise[stream];
    f.innov = P.st.innov[stream];
    f.phi = P.st.phi[stream];
    f.m_var = P.st.m_var[stream];
  }
  bool k_valid = false;  // k_gain == sigma2 / (sigma2 + r) holds after one update here
  int ik = -1;           // position in the idle-filter gain table
  if (P.idle_fix >= 0)
    for (int k = 0; k <= P.idle_fix; ++k)
      if (P.idle_m[k] == f.m_var) { ik = k; break; }
  cs.budget = fresh ? 0.0 : P.st.group_budget[stream];
  cs.count = fresh ? 0 : P.st.group_count[stream];

  // segment (phase) tracking; only cur_end stays in a register
  {
    const int nseg = tr.n_segments[row];
    const long long seg0 = row * tr.max_segments;
    int seg = 0;
    while (seg + 1 < nseg && P.step_begin >= tr.seg_end[seg0 + seg]) ++seg;
    cs.seg0 = seg0;
    cs.nseg = nseg;
    cs.seg = seg;
    cs.phase = tr.seg_phase[seg0 + seg];
    cs.idle = tr.seg_idle[seg0 + seg];
  }
  int cur_end = min(cs.seg + 1 < cs.nseg ? tr.seg_end[cs.seg0 + cs.seg] : 0x7fffffff, cs.gend);
  if (P.ratio_smem) fill_ratios(T, tile, sRatio + (size_t)tid * T.n_powers, cs.idle);

  const bool has_agg = P.out.agg != nullptr;
  if (writer && has_agg) {
    double* agg = P.out.agg + stream_ll * ALERT_AGG_FIELDS;
    G = Agg{};
    if (!fresh) {  // FRESH: the sums start at zero, the block is only written (at the end)
      G.e = agg[ALERT_AGG_ENERGY]; G.ec = agg[ALERT_AGG_ENERGY_C];
      G.a = agg[ALERT_AGG_ACC]; G.ac = agg[ALERT_AGG_ACC_C];
      if constexpr (PF == PF_BOTH) {
        G.oe = agg[ALERT_AGG_OR_ENERGY]; G.oec = agg[ALERT_AGG_OR_ENERGY_C];
        G.oa = agg[ALERT_AGG_OR_ACC]; G.oac = agg[ALERT_AGG_OR_ACC_C];
      }
    }
    open_segment(G, agg, cs.phase, fresh);
  }

  // Trace prefetch: the next step's slow-down is copied global -> shared with
  // cp.async (LDGSTS) into one of two per-thread slots, so no register is held
  // across the step and the load latency hides behind a whole step of work.
  const unsigned slot_sa =
      (unsigned)__cvta_generic_to_shared(reinterpret_cast<unsigned long long*>(base + L.slot) + 2 * threadIdx.x);
  const bool f64 = tr.slowdown_dtype == ALERT_DTYPE_F64;
  const int esz = f64 ? 8 : 4;
  const char* sptr = static_cast<const char*>(tr.slowdown) +
                     (row * tr.row_stride + (P.step_begin - tr.step_offset) * tr.step_stride) * esz;
  prefetch_s(slot_sa, sptr, f64);
  const int n_end = (int)P.step_end;
  for (int n = (int)P.step_begin; n < n_end; ++n) {
    const unsigned par = (unsigned)(n - (int)P.step_begin) & 1u;
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    unsigned long long s_raw;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(s_raw) : "r"(slot_sa + 8u * par) : "memory");
    if (n + 1 < n_end) {
      sptr += tr.step_stride * esz;
      prefetch_s(slot_sa + 8u * (par ^ 1u), sptr, f64);
    }
    if (n >= cur_end) {  // segment change (rare): cursor, phase, idle power; goal change
      int seg = cs.seg;
      const int nseg = cs.nseg;
      const long long seg0 = cs.seg0;
      if (seg + 1 < nseg && n >= tr.seg_end[seg0 + seg]) {
        if (has_agg && writer) flush_segment(G, P.out.agg + stream_ll * ALERT_AGG_FIELDS, cs.phase, fresh);
        while (seg + 1 < nseg && n >= tr.seg_end[seg0 + seg]) ++seg;
        cs.seg = seg;
        cs.phase = tr.seg_phase[seg0 + seg];
        cs.idle = tr.seg_idle[seg0 + seg];
        if (P.ratio_smem) fill_ratios(T, tile, sRatio + (size_t)tid * T.n_powers, cs.idle);
        if (has_agg && writer) open_segment(G, P.out.agg + stream_ll * ALERT_AGG_FIELDS, cs.phase, fresh);
      }
      if (n >= cs.gend) {  // goal change: the row's next spec (policy.spec swapped)
        cs.gseg = goal_seek(tr, cs.gseg0, cs.ngseg, cs.gseg, n);
        cs.gend = goal_end(tr, cs.gseg0, cs.ngseg, cs.gseg);
        const int si = tr.goal_seg_spec[cs.gseg0 + cs.gseg];
        if (si != cs.si) {
          cs.si = si;
          stage_spec(si);
        }
      }
      cur_end = min(seg + 1 < nseg ? tr.seg_end[seg0 + seg] : 0x7fffffff, cs.gend);
    }
    // adjust_goal (selector.py:48-70) with group budgets (simulator.py:473-483)
    double goal, period;
    const int group_size = spec->group_size;
    if (group_size > 0) {
      if (cs.count == 0) {
        cs.budget = xmul((double)group_size, spec->t_goal);
        cs.count = group_size;
      }
      goal = py_max(xsub(xdiv(cs.budget, (double)cs.count), spec->oh), 0.001);
      period = xadd(goal, spec->oh);
    } else {
      goal = spec->goal0;
      period = spec->period0;
    }

    Decision d;
    double s;  // true slow-down of this input: consumed only after the decision
    if (PF == PF_ORACLE) {
      s = s_of_raw(tr, s_raw);
      d = oracle_decide(T, sA, sB, C64, sCol, tile, spec, s, cs.idle, goal, P.flags & ALERT_FLAG_FP64_ALL,
                         P.flags & (ALERT_FLAG_NO_FAST | ALERT_FLAG_NO_ORACLE_FAST));
    } else {
      StepCtx x;
      make_ctx(x, spec, C64, f.mu, f.sigma2, f.phi, goal, P.flags & ALERT_FLAG_FP64_ALL);
      x.sv = sv_tile;
      x.has_sv = P.sv_smem;
      if (fast && !x.fp64_all) {
        x.fast = true;
        x.sF = sF;
        x.wst = sWst;
        x.any_window = P.flags & ALERT_FLAG_ANY_WINDOW;
        if (P.units_smem) {
          x.su = sUn;
          x.slb = sLb;
          if (n_seq) {
            x.sqA = sQA;
            x.sqM = sQM;
            x.n_seq = n_seq;
          }
        }
        float* fzZ = reinterpret_cast<float*>(base + L.fz) + tid;
        fast_prep(x, tile, fzZ, fzZ + (size_t)n_tiles * n_tdnn, n_tiles, fast_me ? n_tdnn : 0, zpr,
                  P.fast_rows ? P.zlo + (size_t)P.n_specs * (n_tdnn + 1) + (size_t)cs.si * n_tdnn : nullptr);
      }
      d = alert_decide<MS>(T, sA, sB, sCol, tile, x, P.kinds, P.flags & ALERT_FLAG_NO_REFINE);
      s = s_of_raw(tr, s_raw);
    }
    int exec_cell = d.cell;
    if (P.out.forced) {
      const int fc = P.out.forced[stream_ll * P.out.stream_stride + (long long)n * P.out.step_stride];
      if (fc >= 0) exec_cell = T.cell_of_cand[fc];
    }
    const double idle = cs.idle;
    const Outcome o = execute_measure(sB, C64, spec, exec_cell, s, goal, period, idle);
    if (PF != PF_ORACLE) {  // AlertPolicy.observe, policies.py:105-108
      slowdown_update(P.cfg, f, o.fb_latency, o.fb_t_prof, k_valid);
      const int pw = __float_as_uint(sB[exec_cell].y) >> 20;  // power index from the tie key
      const double ratio = P.ratio_smem ? sRatio[(size_t)tid * T.n_powers + pw]
                                        : py_min(1.0, xdiv(idle, C64[exec_cell].cap));
      idle_update(P.cfg, f, ratio, ik, P.idle_fix, P.idle_w, P.idle_m);
    }
    if (group_size > 0) {  // simulator.py:501-503
      cs.budget = xsub(cs.budget, o.latency);
      cs.count -= 1;
    }
    const AlertOutputs& out = P.out;
    if (writer && out.fb_latency) {  // StepRecord feedback pair (xi diagnostics), goal, phi
      const long long oidx = stream_ll * out.stream_stride + (long long)n * out.step_stride;
      out.fb_latency[oidx] = o.fb_latency;
      out.fb_t_prof[oidx] = o.fb_t_prof;
      if (out.plan_goal) out.plan_goal[oidx] = goal;
      if (out.phi) out.phi[oidx] = f.phi;
    }
    if (writer && out.decision) {
      const long long oidx = stream_ll * out.stream_stride + (long long)n * out.step_stride;
      out.decision[oidx] = pack_decision(cell_cand(sB[d.cell]), d.level, o, d.refined, cs.phase, d.level == 0);
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
    if (writer && has_agg) {  // aggregates in step order (CPython 3.12 sum() semantics)
      neumaier(G.e, G.ec, o.energy);
      neumaier(G.a, G.ac, o.delivered);
      neumaier(G.pe, G.pec, o.energy);
      neumaier(G.pa, G.pac, o.delivered);
      G.dn += 1;
      G.dvl += o.vl; G.dva += o.va; G.dve += o.ve;
      G.l1 += d.level == 1; G.l2 += d.level == 2;
      G.ref += d.refined;
      G.full += d.full;
    }
    if (PF == PF_BOTH) {  // OraclePolicy alongside on the same step
      Decision od = oracle_decide(T, sA, sB, C64, sCol, tile, spec, s, idle, goal, P.flags & ALERT_FLAG_FP64_ALL,
                         P.flags & (ALERT_FLAG_NO_FAST | ALERT_FLAG_NO_ORACLE_FAST));
      const Outcome oo = execute_measure(sB, C64, spec, od.cell, s, goal, period, idle);
      if constexpr (PF == PF_BOTH) if (writer && has_agg) {
        neumaier(G.oe, G.oec, oo.energy);
        neumaier(G.oa, G.oac, oo.delivered);
        G.ovl += oo.vl; G.ova += oo.va; G.ove += oo.ve;
        G.osame += od.cell == exec_cell;
      }
      if (writer && out.oracle_decision)
        out.oracle_decision[stream_ll * out.stream_stride + (long long)n * out.step_stride] =
            pack_decision(cell_cand(sB[od.cell]), od.level, oo, false, cs.phase, od.level == 0);
    }
  }
  if (!writer) continue;
  P.st.mu[stream] = f.mu;
  P.st.sigma2[stream] = f.sigma2;
  P.st.k_gain[stream] = f.k_gain;
  P.st.q_noise[stream] = f.q_noise;
  P.st.innov[stream] = f.innov;
  P.st.phi[stream] = f.phi;
  P.st.m_var[stream] = f.m_var;
  P.st.group_budget[stream] = cs.budget;
  P.st.group_count[stream] = cs.count;
  if (fresh && P.st.policy_aux) P.st.policy_aux[stream] = -1;  // as alert_state_init (comparison schemes only)
  if (has_agg) {
    double* agg = P.out.agg + stream_ll * ALERT_AGG_FIELDS;
    flush_segment(G, agg, cs.phase, fresh);
    const double steps = (double)(P.step_end - P.step_begin);
    // counters: added to the block, or (FRESH) stored — every field written
    // once and none read, the unvisited phase slots and the spare fields zeroed
    auto put = [&](int k, double v) {
      if (fresh) agg[k] = v;
      else agg[k] += v;
    };
    if (fresh) {
      agg[ALERT_AGG_VIOL_LAT] = (double)G.tvl;
      agg[ALERT_AGG_VIOL_ACC] = (double)G.tva;
      agg[ALERT_AGG_VIOL_ENERGY] = (double)G.tve;
      for (int k = ALERT_AGG_FULL_SCAN + 1; k < ALERT_AGG_PHASE_BASE; ++k) agg[k] = 0.0;
      for (int ph = 0; ph < ALERT_MAX_PHASES; ++ph)
        if (!((G.seen >> ph) & 1))
          for (int k = 0; k < ALERT_AGG_PHASE_STRIDE; ++k) agg[ALERT_AGG_PHASE_BASE + ALERT_AGG_PHASE_STRIDE * ph + k] = 0.0;
    }
    put(ALERT_AGG_N, steps);
    agg[ALERT_AGG_ENERGY] = G.e; agg[ALERT_AGG_ENERGY_C] = G.ec;
    agg[ALERT_AGG_ACC] = G.a; agg[ALERT_AGG_ACC_C] = G.ac;
    put(ALERT_AGG_LEVEL0, steps - (double)G.l1 - (double)G.l2);
    put(ALERT_AGG_LEVEL1, (double)G.l1);
    put(ALERT_AGG_LEVEL2, (double)G.l2);
    put(ALERT_AGG_REFINED, (double)G.ref);
    put(ALERT_AGG_FULL_SCAN, (double)G.full);
    if constexpr (PF == PF_BOTH) {
      agg[ALERT_AGG_OR_ENERGY] = G.oe; agg[ALERT_AGG_OR_ENERGY_C] = G.oec;
      agg[ALERT_AGG_OR_ACC] = G.oa; agg[ALERT_AGG_OR_ACC_C] = G.oac;
      put(ALERT_AGG_OR_VIOL_LAT, (double)G.ovl);
      put(ALERT_AGG_OR_VIOL_ACC, (double)G.ova);
      put(ALERT_AGG_OR_VIOL_ENERGY, (double)G.ove);
      put(ALERT_AGG_OR_SAME, (double)G.osame);
    } else if (fresh) {
      for (int k = ALERT_AGG_OR_ENERGY; k <= ALERT_AGG_OR_SAME; ++k) agg[k] = 0.0;
    }
  }
  }  // stream loop
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
    decision[i] = (uint32_t)cell_cand(sB[d.cell]) | ((uint32_t)d.level << 16) | ((uint32_t)d.refined << 26) |
                  ((uint32_t)(d.level == 0) << 30);
}

template <int W>
__global__ void oracle_decide_kernel(const DevTable T, const SpecDev* specs, int n_specs, const int32_t* stream_spec,
                                     const double* s, const double* idle, const double* goal, uint32_t* decision,
                                     AlertPrediction* exact, long long n, bool fp64_all) {
  auto tile = cg::tiled_partition<W>(cg::this_thread_block());
  const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / W;
  if (i >= n) return;
  const int si = stream_spec ? stream_spec[i] : (int)(i % n_specs);
  Decision d = oracle_decide(T, T.cellA, T.cellB, T.c64, T.any_cols, tile, specs + si, s[i], idle[i], goal[i], fp64_all);
  if (tile.thread_rank() == 0) {
    decision[i] = (uint32_t)cell_cand(T.cellB[d.cell]) | ((uint32_t)d.level << 16) | ((uint32_t)(d.level == 0) << 30);
    if (exact) {  // _exact_pred of the choice (policies.py:172-205): its exact outcome, period = goal + overhead
      const Outcome o = execute_measure(T.cellB, T.c64, specs + si, d.cell, s[i], goal[i],
                                        xadd(goal[i], specs[si].oh), idle[i]);
      AlertPrediction p;
      p.latency_mean = o.latency;
      p.latency_sigma = 0.0;
      p.pr_deadline = o.met ? 1.0 : 0.0;
      p.expected_accuracy = o.delivered;
      p.energy = o.energy;
      p.dnn_index = p.power_index = p.target_stage = p._pad = 0;
      exact[i] = p;
    }
  }
}


// launchers (defined per W in alert_inst_w*.cu)
template <int W>
cudaError_t launch_run(int pf, const RunParams& P, int tpb, size_t smem, cudaStream_t st);
template <int W>
cudaError_t launch_decide(const StepParams& P, uint32_t* out, int tpb, size_t smem, cudaStream_t st);
template <int W>
cudaError_t launch_oracle(const DevTable& T, const SpecDev* specs, int n_specs, const int32_t* stream_spec,
                          const double* s, const double* idle, const double* goal, uint32_t* decision,
                          AlertPrediction* exact, long long n, int tpb, unsigned flags, cudaStream_t st);

template <class K>
inline cudaError_t set_smem(K kern, size_t smem) {
  if (smem > 48 * 1024) return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return cudaSuccess;
}

// Persistent launch of run_kernel: as many blocks as are resident at once
// (occupancy x SMs, at most one per tile group of streams); the blocks
// grid-stride over the streams.
template <class K>
inline cudaError_t launch_persistent(K kern, const RunParams& P, long long blocks, int tpb, size_t smem,
                                     cudaStream_t st) {
  cudaError_t e;
  if ((e = set_smem(kern, smem))) return e;
  int dev = 0, sms = 0, per_sm = 0;
  if ((e = cudaGetDevice(&dev)) || (e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) ||
      (e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, tpb, smem)))
    return e;
  const long long resident = (long long)std::max(1, per_sm) * std::max(1, sms);
  // A/B knobs: ALERT_NO_PERSIST (one tile group per block), ALERT_STATIC_PERSIST (grid stride)
  static const bool no_persist = std::getenv("ALERT_NO_PERSIST") != nullptr;
  static const bool static_persist = std::getenv("ALERT_STATIC_PERSIST") != nullptr;
  RunParams Q = P;
  if (no_persist || static_persist || blocks <= resident) Q.work = nullptr;
  else if (Q.work && (e = cudaMemsetAsync(Q.work, 0, sizeof(unsigned long long), st))) return e;
  kern<<<(unsigned)(no_persist ? blocks : std::min(blocks, resident)), tpb, smem, st>>>(Q);
  return cudaGetLastError();
}

#define ALERT_INSTANTIATE(W)                                                                          \
  template <>                                                                                         \
  cudaError_t launch_run<W>(int pf, const RunParams& P, int tpb, size_t smem, cudaStream_t st) {      \
    const long long blocks = ((P.stream_end - P.stream_begin) * W + tpb - 1) / tpb;                  \
    if (pf == PF_ORACLE) return launch_persistent(run_kernel<W, PF_ORACLE, MS_ALL>, P, blocks, tpb, smem, st); \
    if (pf == PF_BOTH) return launch_persistent(run_kernel<W, PF_BOTH, MS_ALL>, P, blocks, tpb, smem, st); \
    if (P.min_energy_only)                                                                            \
      return launch_persistent(run_kernel<W, PF_ALERT, MS_MIN_ENERGY>, P, blocks, tpb, smem, st);     \
    if constexpr (W == 1 || W == 8)  /* the widths the library picks by default */                    \
      if (P.max_accuracy_only)                                                                        \
        return launch_persistent(run_kernel<W, PF_ALERT, MS_MAX_ACCURACY>, P, blocks, tpb, smem, st);   \
    return launch_persistent(run_kernel<W, PF_ALERT, MS_ALL>, P, blocks, tpb, smem, st);              \
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
                               const double* goal, uint32_t* decision, AlertPrediction* exact,        \
                               long long n, int tpb, unsigned flags, cudaStream_t st) {              \
    long long blocks = (n * W + tpb - 1) / tpb;                                                       \
    oracle_decide_kernel<W><<<(unsigned)blocks, tpb, 0, st>>>(T, specs, n_specs, stream_spec, s, idle, goal, \
                                                             decision, exact, n, flags & ALERT_FLAG_FP64_ALL); \
    return cudaGetLastError();                                                                        \
  }

}  // namespace alert
