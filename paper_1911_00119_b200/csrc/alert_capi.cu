// alert_capi.cu — kernels and the C ABI (include/alert_b200.h) of the B200
// ALERT scheduling step.  Build: see __graft_entry__.py (nvcc, sm_100a).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "alert_baselines.cuh"

#include <curand_kernel.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: named ranges for nsys / ncu --nvtx

using namespace alert;

// NVTX range for the duration of an entry point (SURVEY §5 tracing)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// ==========================================================================
// error plumbing
static thread_local std::string g_last_error;

static int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define CUDA_TRY(expr)                                                               \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      return fail(ALERT_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(_e)); \
  } while (0)

struct AlertContext {
  int device = 0;
  int lanes = 0;  // 0 = auto
  int tpb = 64;
  bool tpb_auto = true;  // alert_set_launch(.., 0): pick the block size from the shared-memory footprint
  int n_sm = 148;
  int max_smem = 227 * 1024;
  std::atomic<long long> launches{0};
};

struct AlertTable {
  DevTable dev{};
  void* buf = nullptr;  // one device allocation holding every array
  int n_cand = 0;
  std::vector<int32_t> cand_dnn, cand_power, cand_stage;
  std::vector<double> acc_levels;  // distinct accuracies, descending (rank order)
  int n_any_cols = 0;
  int device = 0;
};

// ==========================================================================
// kernels

// predict_all for n streams: out[i][candidate] in reference order, FP64 exact.
__global__ void predict_kernel(const StepParams P, AlertPrediction* out, const int32_t* cand_dnn,
                               const int32_t* cand_power, const int32_t* cand_stage) {
  const long long total = P.n * P.T.n_cells;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (long long)gridDim.x * blockDim.x) {
    const long long i = g / P.T.n_cells;
    const int c = (int)(g % P.T.n_cells);  // candidate index
    const int cell = P.T.cell_of_cand[c];
    const int si = P.stream_spec ? P.stream_spec[i] : (int)(i % P.n_specs);
    StepCtx x;
    make_ctx(x, P.specs + si, P.T.c64, P.st.mu[i], P.st.sigma2[i], P.st.phi[i], P.goal[i], true);
    ensure_fp64(x);
    Pred64 q = eval64(P.T, x, cell);
    AlertPrediction r;
    double t = P.T.c64[cell].t;
    r.latency_mean = xmul(x.mu, t);
    r.latency_sigma = xmul(x.sig, t);
    r.pr_deadline = q.pr;
    r.expected_accuracy = q.acc;
    r.energy = q.energy;
    r.dnn_index = cand_dnn[c];
    r.power_index = cand_power[c];
    r.target_stage = cand_stage[c];
    r._pad = 0;
    out[g] = r;
  }
}

__global__ void observe_kernel(const DevTable T, const AlertFilterConfig cfg, AlertState st, const double* fb_lat,
                               const double* fb_t, const double* idle, const int32_t* power, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Filter f{st.mu[i], st.sigma2[i], st.k_gain[i], st.q_noise[i], st.innov[i], st.phi[i], st.m_var[i]};
  bool k_valid = false;
  int ik = -1;
  slowdown_update(cfg, f, fb_lat[i], fb_t[i], k_valid);
  idle_update(cfg, f, py_min(1.0, xdiv(idle[i], T.power_cap64[power[i]])), ik, -1, nullptr, nullptr);
  st.mu[i] = f.mu; st.sigma2[i] = f.sigma2; st.k_gain[i] = f.k_gain; st.q_noise[i] = f.q_noise;
  st.innov[i] = f.innov; st.phi[i] = f.phi; st.m_var[i] = f.m_var;
}

// z-thresholds of the min-energy fast scan, one thread per (spec, traditional
// DNN) (+ one per spec for the pr_threshold bound).  feasible at level 0
// (selector.py:73-84 with accuracy_blend, predictor.py:68-70) means
//   fl(fl(Pr a) + fl(fl(1 - Pr) q_fail)) >= q_goal  and  Pr >= pr_th,
// with Pr = fl(0.5 fl(1 + erf(x / sqrt 2))) (predictor.py:56-65).  In exact
// arithmetic that implies Phi(z) >= thr - delta, delta covering the FP64
// roundings of the blend (4 ulp of the largest operand / (a - q_fail)) and of
// Pr (erf <= 1 ulp, x, the final rounding: 1e-15 absolute), hence
// z >= Phi^-1(thr - delta) - margin (normcdfinv error).  Results are lower
// bounds (never excluding a feasible cell); -inf = always possible, 1e10 =
// never; capped at 7.5 where Pr can round to exactly 1.  Stored in FP32 as
// z' = z - 20 eps |z| (the margin of fast_prep, alert_device.cuh).
__device__ inline double zlo_of_prob(double p) {
  if (!(p > 0.0)) return -kInf;
  double z = p >= 1.0 ? 7.5 : fmin(normcdfinv(p), 7.5);
  return z - 1e-9 * (1.0 + fabs(z));
}
// z' of spec s, traditional DNN d (d == n_tdnn: the pr_threshold bound)
__device__ float zlo_value(const SpecDev& sp, const Cell64* c64, int P, int n_tdnn, int d) {
  const double zpr = sp.has_pr ? zlo_of_prob(sp.pr_th - 1e-15) : -kInf;
  double z;
  if (d == n_tdnn) {
    z = zpr;
  } else {
    const double a = c64[(size_t)d * P].a, qf = c64[(size_t)d * P].qf, q = sp.q_goal;
    if (!(a > qf)) {
      z = -kInf;  // accuracy not increasing in Pr: leave it to the certification
    } else if (q > a * (1.0 + 1e-14) && q > a + 1e-300) {
      z = kInf;   // acc <= max(a, q_fail) (1 + 4 ulp) < q_goal: never feasible
    } else {
      const double m = fmax(1.0, fmax(fabs(a), fmax(fabs(qf), fabs(q))));
      const double delta = 8.0 * 1.1102230246251565e-16 * m / (a - qf) + 1e-15;
      z = zlo_of_prob((q - qf) / (a - qf) - delta);
    }
    z = fmax(z, zpr);
  }
  const float zf = z == kInf ? 1e10f : (float)z;
  return fmaf(-20.0f * kEps, fabsf(zf), zf);
}
// out: [n_specs][n_tdnn + 1] by DNN, then (rows != null, row mode)
// [n_specs][n_tdnn] in the scan's row order (rows[r].x = DNN bits)
__global__ void zlo_kernel(const SpecDev* specs, int n_specs, const Cell64* c64, int P, int n_tdnn,
                           const float4* rows, float* out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int stride = n_tdnn + 1;
  const long long n1 = (long long)n_specs * stride;
  if (i < n1) {
    out[i] = zlo_value(specs[i / stride], c64, P, n_tdnn, (int)(i % stride));
  } else if (rows && n_tdnn > 0 && i < n1 + (long long)n_specs * n_tdnn) {
    const long long j = i - n1;
    out[i] = zlo_value(specs[j / n_tdnn], c64, P, n_tdnn, __float_as_int(rows[j % n_tdnn].x));
  }
}


// ==========================================================================
// xi diagnostics (simulator.py:521-543): numpy.histogram(xi, 40) + mean / std
// with numpy's exact arithmetic (linspace edges, index correction, pairwise
// summation order; see alert_xi_stats).
__device__ __forceinline__ double xi_at(const double* num, const double* den, long long i) {
  return den ? xdiv(num[i], den[i]) : num[i];
}

__global__ void xi_minmax_kernel(const double* num, const double* den, long long n, int bins, double* edges,
                                 double* scratch) {
  __shared__ double smin[1024], smax[1024];
  double mn = kInf, mx = -kInf;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = xi_at(num, den, i);
    mn = fmin(mn, v);
    mx = fmax(mx, v);
  }
  smin[threadIdx.x] = mn;
  smax[threadIdx.x] = mx;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      smin[threadIdx.x] = fmin(smin[threadIdx.x], smin[threadIdx.x + w]);
      smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + w]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double first = smin[0], last = smax[0];
    if (first == last) {  // _get_outer_edges: expand an empty range
      first = xsub(first, 0.5);
      last = xadd(last, 0.5);
    }
    // np.linspace(first, last, bins + 1): y = arange * step + start, y[-1] = stop
    const double delta = xsub(last, first), step = xdiv(delta, (double)bins);
    for (int i = 0; i < bins; ++i)
      edges[i] = step == 0.0 ? xadd(xmul(xdiv((double)i, (double)bins), delta), first)
                             : xadd(xmul((double)i, step), first);
    edges[bins] = last;
    scratch[0] = first;
    scratch[1] = last;
  }
}

__global__ void xi_hist_kernel(const double* num, const double* den, long long n, int bins, const double* edges,
                               const double* scratch, unsigned long long* counts) {
  const double first = scratch[0], last = scratch[1];
  const double denom = xsub(last, first);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double v = xi_at(num, den, i);
    if (!(v >= first && v <= last)) continue;
    long long k = (long long)xmul(xdiv(xsub(v, first), denom), (double)bins);
    if (k == bins) k -= 1;
    if (v < edges[k]) k -= 1;
    if (v >= edges[k + 1] && k != bins - 1) k += 1;
    atomicAdd(counts + k, 1ull);
  }
}

// numpy's pairwise_sum (loops_utils.h) on one leaf (n <= 128)
__device__ double np_leaf_sum(const double* num, const double* den, long long off, long long n, int mode,
                              double mean) {
  auto val = [&](long long i) {
    const double v = xi_at(num, den, off + i);
    if (mode == 0) return v;
    const double d = xsub(v, mean);
    return xmul(d, d);
  };
  if (n < 8) {
    double res = 0.0;
    for (long long i = 0; i < n; ++i) res = xadd(res, val(i));
    return res;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = val(j);
  long long i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = xadd(r[j], val(i + j));
  double res = xadd(xadd(xadd(r[0], r[1]), xadd(r[2], r[3])), xadd(xadd(r[4], r[5]), xadd(r[6], r[7])));
  for (; i < n; ++i) res = xadd(res, val(i));
  return res;
}

__global__ void xi_leaf_kernel(const double* num, const double* den, const long long* leaves, int n_leaves, int mode,
                               const double* mean_sd, double* leaf_sums) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_leaves) return;
  leaf_sums[k] = np_leaf_sum(num, den, leaves[2 * k], leaves[2 * k + 1], mode, mode ? mean_sd[0] : 0.0);
}

// replays the pairwise recursion: prog = post-order of leaf pushes (>= 0)
// and additions (-1); mode 0 -> mean, mode 1 -> sd
__global__ void xi_combine_kernel(const int* prog, int n_prog, const double* leaf_sums, long long n, int mode,
                                  double* mean_sd) {
  double stack[80];
  int sp = 0;
  for (int i = 0; i < n_prog; ++i) {
    const int op = prog[i];
    if (op >= 0) {
      stack[sp++] = leaf_sums[op];
    } else {
      const double b = stack[--sp], a = stack[--sp];
      stack[sp++] = xadd(a, b);
    }
  }
  const double q = xdiv(stack[0], (double)n);
  if (mode == 0) mean_sd[0] = q;
  else mean_sd[1] = sqrt(q);
}

__global__ void state_init_kernel(AlertState st, AlertFilterConfig cfg, double phi0, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  st.mu[i] = cfg.mu0;  // slowdown_init, estimator.py:47-56
  st.sigma2[i] = cfg.sigma2_0;
  st.k_gain[i] = cfg.k0;
  st.q_noise[i] = cfg.q0;
  st.innov[i] = 0.0;
  st.phi[i] = phi0;  // idle_power_init(phi0), policies.py:90-91
  st.m_var[i] = cfg.m0;
  st.group_budget[i] = 0.0;
  st.group_count[i] = 0;
  if (st.policy_aux) st.policy_aux[i] = -1;  // comparison schemes: begin() pending
}

// Deterministic reduction: fixed chunks of streams per block, fixed order.
constexpr int kReduceChunk = 4096;
constexpr int kReduceRep = 3;  // threads per field
__global__ void reduce_partial_kernel(const double* agg, long long n, double* partial) {
  __shared__ double sh[kReduceRep * ALERT_AGG_FIELDS];
  const int t = threadIdx.x;  // blockDim = kReduceRep * FIELDS
  const int field = t % ALERT_AGG_FIELDS, rep = t / ALERT_AGG_FIELDS;
  const long long s0 = (long long)blockIdx.x * kReduceChunk;
  const long long s1 = min(n, s0 + kReduceChunk);
  double acc = 0.0;
  for (long long s = s0 + rep; s < s1; s += kReduceRep) acc = xadd(acc, agg[s * ALERT_AGG_FIELDS + field]);
  sh[t] = acc;
  __syncthreads();
  if (rep == 0) {
    double v = sh[field];
    for (int r = 1; r < kReduceRep; ++r) v = xadd(v, sh[r * ALERT_AGG_FIELDS + field]);
    partial[(long long)blockIdx.x * ALERT_AGG_FIELDS + field] = v;
  }
}

__global__ void reduce_final_kernel(const double* partial, long long nb, double* out) {
  const int field = threadIdx.x;
  if (field >= ALERT_AGG_FIELDS) return;
  double v = 0.0;
  for (long long b = 0; b < nb; ++b) v = xadd(v, partial[b * ALERT_AGG_FIELDS + field]);
  out[field] = v;
}

// ==========================================================================
// host side

int alert_abi_version(void) { return ALERT_ABI_VERSION; }

const char* alert_strerror(int status) {
  switch (status) {
    case ALERT_OK: return "ok";
    case ALERT_ERR_INVALID_ARGUMENT: return "invalid argument";
    case ALERT_ERR_INVALID_SPACE: return "invalid config space";
    case ALERT_ERR_INVALID_SPEC: return "invalid constraint spec";
    case ALERT_ERR_INVALID_TRACE: return "invalid trace";
    case ALERT_ERR_CUDA: return "CUDA error";
    case ALERT_ERR_UNSUPPORTED: return "unsupported size";
    case ALERT_ERR_NO_CANDIDATE: return "no candidate of the requested kinds";
    default: return "unknown status";
  }
}

const char* alert_last_error(void) { return g_last_error.c_str(); }

int alert_create(AlertContext** out, int device) {
  if (!out) return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_create: out is NULL");
  int n = 0;
  CUDA_TRY(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_create: bad device index");
  CUDA_TRY(cudaSetDevice(device));
  AlertContext* c = new AlertContext();
  c->device = device;
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  c->n_sm = prop.multiProcessorCount;
  c->max_smem = (int)prop.sharedMemPerBlockOptin;
  *out = c;
  return ALERT_OK;
}

int alert_destroy(AlertContext* ctx) {
  delete ctx;
  return ALERT_OK;
}

int alert_set_launch(AlertContext* ctx, int lanes, int tpb) {
  if (!ctx) return fail(ALERT_ERR_INVALID_ARGUMENT, "ctx is NULL");
  if (lanes != 0 && lanes != 1 && lanes != 2 && lanes != 4 && lanes != 8 && lanes != 16 && lanes != 32)
    return fail(ALERT_ERR_INVALID_ARGUMENT, "lanes_per_stream must be 0 or a power of two <= 32");
  if (tpb != 0 && (tpb < 32 || tpb > 512 || tpb % 32))
    return fail(ALERT_ERR_INVALID_ARGUMENT, "threads_per_block must be a multiple of 32 in [32, 256]");
  ctx->lanes = lanes;
  ctx->tpb = tpb ? tpb : 64;
  ctx->tpb_auto = tpb == 0;
  return ALERT_OK;
}

int alert_get_launch(AlertContext* ctx, int* lanes, int* tpb) {
  if (!ctx) return fail(ALERT_ERR_INVALID_ARGUMENT, "ctx is NULL");
  if (lanes) *lanes = ctx->lanes;
  if (tpb) *tpb = ctx->tpb;
  return ALERT_OK;
}

int64_t alert_launch_count(AlertContext* ctx) { return ctx ? (int64_t)ctx->launches.load() : -1; }

// model.validate (model.py:100-163), first problem only
static std::string validate_space(const AlertSpaceDesc* d) {
  char buf[256];
  if (d->n_powers < 1) return "power axis is empty";
  if (d->n_dnns < 1) return "DNN axis is empty";
  if (!(d->p_idle_prof > 0)) return "p_idle_prof must be positive";
  double prev = 0.0;
  for (int j = 0; j < d->n_powers; ++j) {
    if (!(d->power_cap[j] > prev)) {
      snprintf(buf, sizeof buf, "power[%d]: cap %g W not strictly above previous", j, d->power_cap[j]);
      return buf;
    }
    prev = d->power_cap[j];
  }
  int off = 0;
  for (int i = 0; i < d->n_dnns; ++i) {
    int ns = d->dnn_n_stages[i];
    int kind = d->dnn_kind[i];
    if (kind != ALERT_KIND_TRADITIONAL && kind != ALERT_KIND_ANYTIME) return "unknown DNN kind";
    if (kind == ALERT_KIND_TRADITIONAL && ns != 1) return "traditional profile must have exactly 1 stage";
    if (kind == ALERT_KIND_ANYTIME && ns < 2) return "anytime profile needs >= 2 stages";
    if (ns > ALERT_MAX_STAGES) return "too many stages (ALERT_MAX_STAGES)";
    double qf = d->dnn_q_fail[i];
    if (!(qf >= 0.0 && qf <= 1.0)) return "q_fail outside [0,1]";
    if (qf > d->stage_accuracy[off]) return "q_fail exceeds first-stage accuracy";
    double pa = -1.0;
    for (int k = 0; k < ns; ++k) {
      double a = d->stage_accuracy[off + k];
      if (!(a >= 0.0 && a <= 1.0)) return "stage accuracy outside [0,1]";
      if (kind == ALERT_KIND_ANYTIME && a <= pa) return "anytime accuracies not increasing";
      pa = a;
      const double* t = d->stage_t_prof + (size_t)(off + k) * d->n_powers;
      for (int j = 0; j < d->n_powers; ++j) {
        if (!(t[j] > 0)) return "latency not positive";
        if (j > 0 && t[j] > t[j - 1]) return "latency increases with the power cap";
        if (kind == ALERT_KIND_ANYTIME && k > 0 && t[j] <= t[j - d->n_powers])
          return "anytime stage latencies not strictly increasing";
      }
    }
    off += ns;
  }
  return "";
}

int alert_table_create(AlertContext* ctx, const AlertSpaceDesc* d, AlertTable** out) {
  if (!ctx || !d || !out) return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_table_create: NULL argument");
  if (!d->dnn_kind || !d->dnn_n_stages || !d->dnn_q_fail || !d->stage_accuracy || !d->stage_t_prof || !d->power_cap)
    return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_table_create: NULL array in AlertSpaceDesc");
  std::string prob = validate_space(d);
  if (!prob.empty()) return fail(ALERT_ERR_INVALID_SPACE, "invalid profile: " + prob);
  const int P = d->n_powers;
  std::vector<int> stage_off(d->n_dnns);
  int off = 0;
  for (int i = 0; i < d->n_dnns; ++i) { stage_off[i] = off; off += d->dnn_n_stages[i]; }
  // candidate enumeration (policies.py:59-67) and the cell order (traditional first)
  AlertTable* tb = new AlertTable();
  std::vector<int> trad_cells, any_cells;  // values = candidate index
  std::vector<int2> cols;
  int c = 0;
  for (int i = 0; i < d->n_dnns; ++i)
    for (int j = 0; j < P; ++j) {
      bool trad = d->dnn_kind[i] == ALERT_KIND_TRADITIONAL;
      int nt = trad ? 1 : d->dnn_n_stages[i];
      for (int k = 0; k < nt; ++k, ++c) {
        tb->cand_dnn.push_back(i);
        tb->cand_power.push_back(j);
        tb->cand_stage.push_back(trad ? 0 : k + 1);
        (trad ? trad_cells : any_cells).push_back(c);
      }
    }
  const int n = c;
  if (n > ALERT_MAX_CANDIDATES || P > 1023 || d->n_dnns > 4095 || d->n_dnns * (ALERT_MAX_STAGES + 1) > 65535) {
    delete tb;
    return fail(ALERT_ERR_UNSUPPORTED, "table too large for the packed tie-break key / shared memory");
  }
  std::vector<int> order(trad_cells);
  for (size_t q = 0; q < any_cells.size();) {  // columns of consecutive stages
    int cand = any_cells[q];
    int ns = d->dnn_n_stages[tb->cand_dnn[cand]];
    cols.push_back(make_int2((int)order.size(), ns));
    for (int k = 0; k < ns; ++k) order.push_back(any_cells[q + k]);
    q += ns;
  }
  // exact accuracy classes: every distinct stage accuracy / q_fail value,
  // descending; rank 0 = most accurate (oracle FP32 scan compares ranks)
  std::vector<double> levels;
  for (int i = 0; i < d->n_dnns; ++i) {
    levels.push_back(d->dnn_q_fail[i]);
    for (int k = 0; k < d->dnn_n_stages[i]; ++k) levels.push_back(d->stage_accuracy[stage_off[i] + k]);
  }
  std::sort(levels.begin(), levels.end(), [](double x, double y) { return x > y; });
  levels.erase(std::unique(levels.begin(), levels.end()), levels.end());
  auto rank_of = [&](double v) {
    return (uint32_t)(std::lower_bound(levels.begin(), levels.end(), v, [](double x, double y) { return x > y; }) -
                      levels.begin());
  };
  tb->acc_levels = levels;
  std::vector<float4> A(n), B(n);
  std::vector<Cell64> c64(n);
  std::vector<int> cell_of_cand(n);
  double max_cap = d->power_cap[P - 1];
  for (int cell = 0; cell < n; ++cell) {
    int cand = order[cell];
    int i = tb->cand_dnn[cand], j = tb->cand_power[cand], st = tb->cand_stage[cand];
    int k0 = st == 0 ? 0 : st - 1;
    double t = d->stage_t_prof[(size_t)(stage_off[i] + k0) * P + j];
    double a = d->stage_accuracy[stage_off[i] + k0];
    double qf = d->dnn_q_fail[i];
    double prev = k0 == 0 ? qf : d->stage_accuracy[stage_off[i] + k0 - 1];
    uint32_t key = ((uint32_t)j << 20) | ((uint32_t)i << 8) | (uint32_t)st;
    // .w = base of the running expected accuracy: q_fail for a traditional cell
    // or the first stage of an anytime column, -1 (= "carry the previous
    // stage's value") for later stages
    A[cell] = make_float4((float)(1.0 / t), (float)(d->power_cap[j] * t), (float)(a - prev),
                          k0 == 0 ? (float)qf : -1.0f);
    // .z = candidate | stage << 16; .w = rank(stage accuracy) | rank(q_fail) << 16
    const uint32_t cs = (uint32_t)cand | ((uint32_t)st << 16);
    const uint32_t rk = rank_of(a) | (rank_of(qf) << 16);
    float kb, cb, rb;
    memcpy(&kb, &key, 4);
    memcpy(&cb, &cs, 4);
    memcpy(&rb, &rk, 4);
    B[cell] = make_float4((float)t, kb, cb, rb);
    c64[cell] = Cell64{t, a, qf, d->power_cap[j]};
    cell_of_cand[cand] = cell;
  }
  size_t bytes = 0;
  auto place = [&](size_t sz) { size_t o = (bytes + 255) & ~size_t(255); bytes = o + sz; return o; };
  size_t oA = place(sizeof(float4) * n), oB = place(sizeof(float4) * n), oC = place(sizeof(int2) * (cols.size() + 1));
  size_t oC64 = place(sizeof(Cell64) * n), oCell = place(4 * n);
  size_t oPw = place(8 * P);
  size_t oSys = place(4 * P), oApp = place(4 * P);
  // max-accuracy fast scan units: traditional cells and anytime columns,
  // sorted by accuracy upper bound (max of q_fail and the stage accuracies)
  struct Unit { int first, n; double bound; };
  std::vector<Unit> units;
  for (int cell = 0; cell < (int)trad_cells.size(); ++cell)
    units.push_back({cell, 1, std::max(c64[cell].a, c64[cell].qf)});
  for (const int2& cd : cols) {
    double b = c64[cd.x].qf;
    for (int k = 0; k < cd.y; ++k) b = std::max(b, c64[cd.x + k].a);
    units.push_back({cd.x, cd.y | (1 << 16), b});
  }
  std::stable_sort(units.begin(), units.end(), [](const Unit& a, const Unit& b) { return a.bound > b.bound; });
  std::vector<int2> unit_v(units.size());
  std::vector<float> unit_lb(units.size());
  for (size_t k = 0; k < units.size(); ++k) {
    unit_v[k] = make_int2(units[k].first, units[k].n);
    unit_lb[k] = (float)(2.0 - units[k].bound) - 1e-5f;
  }
  // the same order flattened to one entry per cell for the W = 1 scan
  // (fast_max_accuracy_flat, tables of <= 64 cells), one sequence per DNN-kinds
  // filter (1 traditional, 2 anytime, 3 both; the excluded units are left
  // out): the cell's cellA row (.w = q_fail at a unit start, 0 after: the
  // running accuracy restarts by acc * carry + .w) and the metadata {unit lb,
  // dead-group multiplier (1 at a unit start whose group the deadline bound
  // can kill, else 0), carry (0 at a unit start, else 1), k | cell << 8 |
  // (skip to - 1) << 16 | (chain out to - 1) << 24}.  A group = the run of
  // units of one DNN (equal bounds), re-ordered by latency ascending: a unit
  // whose deadline-probability bound fails makes every later unit of the
  // group fail too (1/t only falls), so the scan skips the group; an anytime
  // unit's first cell can kill its group only with monotone stage latencies
  // (any_mono), which is also when a surely infeasible stage ends its chain.
  bool mono = true;
  for (const int2& cd : cols)
    for (int k = 1; k < cd.y; ++k)
      if (!(c64[cd.x + k].t >= c64[cd.x + k - 1].t)) mono = false;
  std::vector<float4> seqA[3], seqM[3];
  if (n <= 64) {
    for (int kinds = 1; kinds <= 3; ++kinds) {
      std::vector<Unit> ku;
      for (const Unit& u : units)
        if ((kinds >> ((u.n >> 16) ? 1 : 0)) & 1) ku.push_back(u);
      auto& SA = seqA[kinds - 1];
      auto& SM = seqM[kinds - 1];
      for (size_t g0 = 0; g0 < ku.size();) {
        const int dnn = tb->cand_dnn[order[ku[g0].first]];
        size_t g1 = g0 + 1;
        while (g1 < ku.size() && tb->cand_dnn[order[ku[g1].first]] == dnn) ++g1;
        std::vector<Unit> grp(ku.begin() + g0, ku.begin() + g1);
        std::stable_sort(grp.begin(), grp.end(),
                         [&](const Unit& a, const Unit& b) { return c64[a.first].t < c64[b.first].t; });
        int cells = 0;
        for (const Unit& u : grp) cells += u.n & 0xFFFF;
        const int next_group = (int)SM.size() + cells;
        for (const Unit& u : grp) {
          const int m = u.n & 0xFFFF, next = (int)SM.size() + m;
          const bool any = (u.n >> 16) != 0;
          const float lb = (float)(2.0 - u.bound) - 1e-5f;
          for (int k = 0; k < m; ++k) {
            const int here = (int)SM.size();
            float4 a = A[u.first + k];
            a.w = k == 0 ? a.w : 0.0f;
            SA.push_back(a);
            const int out_to = (any && mono) ? next : here + 1;
            const uint32_t w = (uint32_t)k | ((uint32_t)(u.first + k) << 8) | ((uint32_t)(next_group - 1) << 16) |
                               ((uint32_t)(out_to - 1) << 24);
            float wf;
            memcpy(&wf, &w, 4);
            SM.push_back(make_float4(lb, (k == 0 && (!any || mono)) ? 1.0f : 0.0f, k == 0 ? 0.0f : 1.0f, wf));
          }
        }
        g0 = g1;
      }
    }
  }
  const size_t n_seq = std::max(seqM[0].size(), std::max(seqM[1].size(), seqM[2].size()));
  // min-energy row mode: traditional DNN rows {dnn bits, smallest cap * t,
  // largest 1/t, 0} by their smallest cap * t, ascending
  std::vector<float4> trows;
  if (P > 0 && !trad_cells.empty()) {
    for (int dn = 0; dn < (int)trad_cells.size() / P; ++dn) {
      float m = A[(size_t)dn * P].y, ax = A[(size_t)dn * P].x;
      for (int j = 1; j < P; ++j) {
        m = std::min(m, A[(size_t)dn * P + j].y);
        ax = std::max(ax, A[(size_t)dn * P + j].x);
      }
      float dnf;
      memcpy(&dnf, &dn, 4);
      trows.push_back(make_float4(dnf, m, ax, 0.0f));
    }
    std::stable_sort(trows.begin(), trows.end(), [](const float4& a, const float4& b) { return a.y < b.y; });
  }
  // oracle max-accuracy fast scan: traditional DNN rows {first cell, rank of
  // the DNN's accuracy, smallest FP32 latency of the row, 0} by rank, best first
  std::vector<float4> orows;
  if (P > 0 && !trad_cells.empty()) {
    for (int dn = 0; dn < (int)trad_cells.size() / P; ++dn) {
      float tmin = B[(size_t)dn * P].x;
      for (int j = 1; j < P; ++j) tmin = std::min(tmin, B[(size_t)dn * P + j].x);
      uint32_t rk;
      memcpy(&rk, &B[(size_t)dn * P].w, 4);
      const int first = dn * P, rank = (int)(rk & 0xFFFF);
      float ff, rf;
      memcpy(&ff, &first, 4);
      memcpy(&rf, &rank, 4);
      orows.push_back(make_float4(ff, rf, tmin, 0.0f));
    }
    std::stable_sort(orows.begin(), orows.end(), [](const float4& a, const float4& b) {
      int ra, rb;
      memcpy(&ra, &a.y, 4);
      memcpy(&rb, &b.y, 4);
      return ra < rb;
    });
  }
  size_t oOrows = place(sizeof(float4) * orows.size());
  size_t oTrows = place(sizeof(float4) * trows.size());
  size_t oUnit = place(sizeof(int2) * units.size()), oUlb = place(4 * units.size());
  size_t oSeqA = place(sizeof(float4) * 3 * n_seq), oSeqM = place(sizeof(float4) * 3 * n_seq);
  // comparison-scheme cells (policies.py:283-454): per power, the sys-only
  // DNN's cell and the first cell of the app-only DNN's column
  std::vector<int> sys_cells(P, -1), app_first(P, -1);
  int app_stages = 0;
  if (d->sys_dnn >= 0 && d->sys_dnn < d->n_dnns && d->dnn_kind[d->sys_dnn] == ALERT_KIND_TRADITIONAL)
    for (int c2 = 0; c2 < n; ++c2)
      if (tb->cand_dnn[c2] == d->sys_dnn) sys_cells[tb->cand_power[c2]] = cell_of_cand[c2];
  if (d->app_dnn >= 0 && d->app_dnn < d->n_dnns && d->dnn_kind[d->app_dnn] == ALERT_KIND_ANYTIME) {
    app_stages = d->dnn_n_stages[d->app_dnn];
    for (int c2 = 0; c2 < n; ++c2)
      if (tb->cand_dnn[c2] == d->app_dnn && tb->cand_stage[c2] == 1) app_first[tb->cand_power[c2]] = cell_of_cand[c2];
  }
  CUDA_TRY(cudaSetDevice(ctx->device));
  char* buf = nullptr;
  cudaError_t e = cudaMalloc(&buf, bytes);
  if (e != cudaSuccess) {
    delete tb;
    return fail(ALERT_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  }
  std::vector<char> h(bytes, 0);
  memcpy(&h[oA], A.data(), sizeof(float4) * n);
  memcpy(&h[oB], B.data(), sizeof(float4) * n);
  if (!cols.empty()) memcpy(&h[oC], cols.data(), sizeof(int2) * cols.size());
  memcpy(&h[oC64], c64.data(), sizeof(Cell64) * n);
  memcpy(&h[oCell], cell_of_cand.data(), 4 * n);
  memcpy(&h[oPw], d->power_cap, 8 * P);
  memcpy(&h[oSys], sys_cells.data(), 4 * P);
  if (!units.empty()) {
    memcpy(&h[oUnit], unit_v.data(), sizeof(int2) * units.size());
    memcpy(&h[oUlb], unit_lb.data(), 4 * units.size());
  }
  if (!trows.empty()) memcpy(&h[oTrows], trows.data(), sizeof(float4) * trows.size());
  if (!orows.empty()) memcpy(&h[oOrows], orows.data(), sizeof(float4) * orows.size());
  for (int v = 0; v < 3; ++v)
    if (!seqM[v].empty()) {
      memcpy(&h[oSeqA + sizeof(float4) * v * n_seq], seqA[v].data(), sizeof(float4) * seqA[v].size());
      memcpy(&h[oSeqM + sizeof(float4) * v * n_seq], seqM[v].data(), sizeof(float4) * seqM[v].size());
    }
  memcpy(&h[oApp], app_first.data(), 4 * P);
  e = cudaMemcpy(buf, h.data(), bytes, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(buf);
    delete tb;
    return fail(ALERT_ERR_CUDA, std::string("cudaMemcpy: ") + cudaGetErrorString(e));
  }
  DevTable& T = tb->dev;
  T.n_cells = n;
  T.n_trad = (int)trad_cells.size();
  T.n_any_cols = (int)cols.size();
  T.n_powers = P;
  T.cellA = reinterpret_cast<const float4*>(buf + oA);
  T.cellB = reinterpret_cast<const float4*>(buf + oB);
  T.any_cols = reinterpret_cast<const int2*>(buf + oC);
  T.c64 = reinterpret_cast<const Cell64*>(buf + oC64);
  T.cell_of_cand = reinterpret_cast<const int*>(buf + oCell);
  double r = d->p_idle_prof / max_cap;
  T.phi0 = (1.0 < r) ? 1.0 : r;  // min(1.0, p_idle_prof / max cap), policies.py:90
  T.power_cap64 = reinterpret_cast<const double*>(buf + oPw);
  T.sys_cells = sys_cells[0] >= 0 ? reinterpret_cast<const int*>(buf + oSys) : nullptr;
  T.units = units.empty() ? nullptr : reinterpret_cast<const int2*>(buf + oUnit);
  T.unit_lb = units.empty() ? nullptr : reinterpret_cast<const float*>(buf + oUlb);
  T.n_units = (int)units.size();
  T.useqA = n_seq ? reinterpret_cast<const float4*>(buf + oSeqA) : nullptr;
  T.useqM = n_seq ? reinterpret_cast<const float4*>(buf + oSeqM) : nullptr;
  T.n_seq = (int)n_seq;
  T.n_seqk[0] = 0;
  for (int v = 0; v < 3; ++v) T.n_seqk[v + 1] = (int)seqM[v].size();
  T.trad_rows = trows.empty() ? nullptr : reinterpret_cast<const float4*>(buf + oTrows);
  T.or_rows = orows.empty() ? nullptr : reinterpret_cast<const float4*>(buf + oOrows);
  T.app_first = app_stages > 0 ? reinterpret_cast<const int*>(buf + oApp) : nullptr;
  T.app_stages = app_stages;
  T.cap_max = (float)max_cap;
  T.cap_min = (float)d->power_cap[0];
  for (int j = 1; j < P; ++j) T.cap_min = std::min(T.cap_min, (float)d->power_cap[j]);
  T.any_mono = mono;  // fast scans' anytime skips: stage latencies non-decreasing
  tb->buf = buf;
  tb->n_cand = n;
  tb->n_any_cols = (int)cols.size();
  tb->device = ctx->device;
  *out = tb;
  return ALERT_OK;
}

int alert_table_destroy(AlertTable* tb) {
  if (!tb) return ALERT_OK;
  cudaSetDevice(tb->device);
  cudaFree(tb->buf);
  delete tb;
  return ALERT_OK;
}

int alert_table_num_candidates(const AlertTable* tb) { return tb ? tb->n_cand : -1; }

int alert_table_candidate(const AlertTable* tb, int c, int32_t* dnn, int32_t* power, int32_t* stage) {
  if (!tb || c < 0 || c >= tb->n_cand) return fail(ALERT_ERR_INVALID_ARGUMENT, "candidate index out of range");
  if (dnn) *dnn = tb->cand_dnn[c];
  if (power) *power = tb->cand_power[c];
  if (stage) *stage = tb->cand_stage[c];
  return ALERT_OK;
}

// ConstraintSpec invariants (model.py:81-97) + group size
static int check_specs(const AlertSpec* specs, int n) {
  if (!specs || n < 1) return fail(ALERT_ERR_INVALID_ARGUMENT, "specs: need at least one spec");
  for (int k = 0; k < n; ++k) {
    const AlertSpec& s = specs[k];
    char where[64];
    snprintf(where, sizeof where, "spec[%d]: ", k);
    if (s.mode != ALERT_MODE_MIN_ENERGY && s.mode != ALERT_MODE_MAX_ACCURACY)
      return fail(ALERT_ERR_INVALID_SPEC, std::string(where) + "unknown mode");
    if (!(s.overhead_budget >= 0)) return fail(ALERT_ERR_INVALID_SPEC, std::string(where) + "overhead_budget must be >= 0");
    if (!(s.t_goal > s.overhead_budget))
      return fail(ALERT_ERR_INVALID_SPEC, std::string(where) + "t_goal must exceed overhead_budget");
    if (s.mode == ALERT_MODE_MAX_ACCURACY && !(s.e_goal > 0))
      return fail(ALERT_ERR_INVALID_SPEC, std::string(where) + "e_goal must be positive");
    if (s.mode == ALERT_MODE_MIN_ENERGY && !(s.q_goal > 0))
      return fail(ALERT_ERR_INVALID_SPEC, std::string(where) + "q_goal must be positive");
    if (s.has_pr && !(s.pr_threshold > 0.0 && s.pr_threshold < 1.0))
      return fail(ALERT_ERR_INVALID_SPEC, std::string(where) + "pr_threshold must lie in (0, 1)");
    if (s.group_size < 0) return fail(ALERT_ERR_INVALID_SPEC, std::string(where) + "group_size must be >= 0");
  }
  return ALERT_OK;
}

static int kinds_of(int policy, const AlertTable* tb) {
  int k = policy == ALERT_POLICY_ALERT_ANY ? 2 : policy == ALERT_POLICY_ALERT_TRAD ? 1 : 3;
  int have = (tb->dev.n_trad > 0 ? 1 : 0) | (tb->dev.n_any_cols > 0 ? 2 : 0);
  return (k & have) ? k : 0;
}

static size_t table_smem(const AlertTable* tb, int W) {
  return SmemLayout(tb->dev.n_cells, tb->dev.n_any_cols, 0, 0, 0, 0, 0, 0, W).total;
}

// Staging decisions of run_kernel: specs, FP64 cells and the per-segment
// idle-ratio table go to shared memory when small (see SmemLayout).
static void run_staging(const AlertTable* tb, const AlertSpec* specs, int n_specs, int tpb, int W, RunParams& P,
                        int policy = ALERT_POLICY_ALERT, unsigned flags = 0) {
  const DevTable& T = tb->dev;
  P.policy = policy;
  // min-energy fast scan (fast_min_energy): needs some min-energy spec, row /
  // column indices that fit the 6-bit key field, and the ALERT policy family
  bool any_min_energy = false, all_min_energy = true;
  for (int k = 0; k < n_specs; ++k) {
    any_min_energy |= specs[k].mode == ALERT_MODE_MIN_ENERGY;
    all_min_energy &= specs[k].mode == ALERT_MODE_MIN_ENERGY;
  }
  P.min_energy_only = all_min_energy;
  P.any_min_energy = any_min_energy;
  P.max_accuracy_only = !any_min_energy;
  // few specs: staged once per block (a tile's spec is a pointer), else one copy per tile
  static const bool no_shared_specs = std::getenv("ALERT_NO_SPEC_SHARED") != nullptr;  // A/B knob
  P.spec_shared = !no_shared_specs && n_specs <= kSpecSmemMax && n_specs < tpb / W;
  const int n_tdnn = T.n_powers > 0 ? T.n_trad / T.n_powers : 0;
  P.zlo = nullptr;
  P.fast_smem = 0;
  // row mode for large tables (no staged per-cell rows / per-tile thresholds)
  P.fast_rows = T.n_trad > 512 || (flags & ALERT_FLAG_FAST_ROWS);
  P.units_smem = 0;
  const bool any_max_accuracy = !all_min_energy;
  if ((any_min_energy || any_max_accuracy) && policy != ALERT_POLICY_ORACLE &&
      !(flags & (ALERT_FLAG_NO_FAST | ALERT_FLAG_FP64_ALL)) &&
      ALERT_MAX_STAGES <= 8 &&
      (P.fast_rows || !any_min_energy || (size_t)(tpb / W) * (size_t)T.n_trad * sizeof(float) <= 16 * 1024))
    P.fast_smem = 1;  // alert_run computes the thresholds (zlo_kernel) and sets P.zlo
  // max-accuracy fast scan needs its sorted units in shared memory
  // (alert_run drops the staging again if the block's shared memory exceeds the limit)
  if (P.fast_smem && any_max_accuracy && T.units && T.n_units <= 4096) P.units_smem = 1;
  P.c64_smem = T.n_cells <= kC64SmemMax;
  P.ratio_smem = T.n_powers <= kRatioSmemMax &&
                 (size_t)(tpb / W) * (size_t)T.n_powers * sizeof(double) <= 16 * 1024;
  // stored objectives pay off only where FP64 re-ranks are frequent:
  // max-accuracy with a completion-probability threshold (SURVEY §7 hard part 1)
  bool refine_heavy = false;
  for (int k = 0; k < n_specs; ++k)
    refine_heavy |= specs[k].mode == ALERT_MODE_MAX_ACCURACY && specs[k].has_pr;
  // (not with the one-lane flat max-accuracy scan: it keeps no per-cell
  // objectives, and the slots would only cost occupancy)
  const bool flat = W == 1 && T.n_seq > 0 && P.units_smem;
  P.sv_smem = refine_heavy && !flat && (size_t)(tpb / W) * (size_t)T.n_cells * sizeof(float) <= 32 * 1024;
}

// the flat W = 1 max-accuracy scan needs its staged sequence; larger unit
// tables can be read through L1 when shared memory is short
static bool T_units_large(const AlertTable* tb) { return tb->dev.n_seq == 0; }

static size_t run_smem(const AlertTable* tb, int n_specs, int tpb, int W, const RunParams& P) {
  const DevTable& T = tb->dev;
  const size_t agg_bytes = P.policy == ALERT_POLICY_ALERT_WITH_ORACLE ? sizeof(TileAggOr) : sizeof(TileAgg);
  SmemLayout L(T.n_cells, T.n_any_cols, P.spec_shared ? n_specs : tpb / W, P.c64_smem ? T.n_cells : 0, tpb / W,
               P.ratio_smem ? T.n_powers : 0, agg_bytes, P.sv_smem ? T.n_cells : 0, W,
               (P.fast_smem && !P.fast_rows && P.any_min_energy) ? T.n_trad : 0,
               (P.fast_smem && !P.fast_rows) ? T.n_trad : 0, P.fast_smem && !P.fast_rows,
               P.units_smem ? T.n_units : 0, P.units_smem ? T.n_seq : 0);
  return L.total;
}

static int pick_lanes(const AlertContext* ctx, const AlertTable* tb) {
  if (ctx->lanes) return ctx->lanes;
  // measured on B200 (profiles/r01b_lanes_c4.txt): one lane per stream for
  // small tables (no redundant per-step work), 8-lane tiles for the
  // 2,144-candidate table (c4: 2 / 4 / 8 / 16 / 32 lanes -> 2.37 / 2.03 /
  // 2.55 / 2.05 / 1.20 e8 decisions/s; 4 streams per warp bound the wait
  // for the slowest stream's row scan)
  return tb->n_cand <= 256 ? 1 : 8;
}

// Upload host specs to stream-ordered device memory (freed after the launch).
// AlertSpec -> SpecDev (device form): goal0 / period0 with the reference's
// operations (selector.py:48-70: max(t_goal - overhead, 0.001); simulator.py:483),
// FP32 copies for the scan.
static SpecDev spec_dev(const AlertSpec& a, const AlertTable* tb) {
  SpecDev d{};
  d.t_goal = a.t_goal;
  d.e_goal = a.e_goal;
  d.q_goal = a.q_goal;
  d.pr_th = a.pr_threshold;
  d.zq = a.z_q;
  d.oh = a.overhead_budget;
  volatile double g = a.t_goal - a.overhead_budget;  // no contraction / reassociation
  double goal = (0.001 > g) ? 0.001 : (double)g;
  d.goal0 = goal;
  d.period0 = goal + a.overhead_budget;
  d.q_f = (float)a.q_goal;
  d.e_f = (float)a.e_goal;
  d.th_f = (float)a.pr_threshold;
  d.zq_f = (float)a.z_q;
  d.mode = a.mode;
  d.has_pr = a.has_pr;
  d.group_size = a.group_size;
  // delivered >= q_goal  <=>  rank(delivered) < rank_q  (ranks are descending)
  int rq = 0;
  while (rq < (int)tb->acc_levels.size() && tb->acc_levels[rq] >= a.q_goal) ++rq;
  d.rank_q = rq;
  return d;
}

// Upload host specs to stream-ordered device memory (freed after the launch).
static int upload_specs(const AlertSpec* specs, int n, const AlertTable* tb, cudaStream_t st, SpecDev** dev) {
  std::vector<SpecDev> h(n);
  for (int k = 0; k < n; ++k) h[k] = spec_dev(specs[k], tb);
  CUDA_TRY(cudaMallocAsync((void**)dev, sizeof(SpecDev) * n, st));
  CUDA_TRY(cudaMemcpyAsync(*dev, h.data(), sizeof(SpecDev) * n, cudaMemcpyHostToDevice, st));
  // pageable source: the copy is staged before cudaMemcpyAsync returns
  return ALERT_OK;
}

// Idle-filter gain table (see RunParams): M_0 = m0, W_k = (M_k+s)/(M_k+s+v),
// M_{k+1} = (1-W_k)(M_k+s), until M_{k+1} == M_k exactly.
static void idle_table(const AlertFilterConfig& c, RunParams& P) {
  P.idle_fix = -1;
  volatile double m = c.m0;
  for (int k = 0; k + 1 < kIdleTab; ++k) {
    volatile double ms = m + c.s;
    volatile double den = ms + c.v;
    volatile double w = ms / den;
    volatile double omw = 1.0 - w;
    volatile double mn = omw * ms;
    P.idle_m[k] = m;
    P.idle_w[k] = w;
    if (mn == m) {
      P.idle_fix = k;
      return;
    }
    m = mn;
  }
}

static int dispatch_run(int W, int pf, const RunParams& P, int tpb, size_t smem, cudaStream_t st) {
  cudaError_t e;
  switch (W) {
    case 1: e = launch_run<1>(pf, P, tpb, smem, st); break;
    case 2: e = launch_run<2>(pf, P, tpb, smem, st); break;
    case 4: e = launch_run<4>(pf, P, tpb, smem, st); break;
    case 8: e = launch_run<8>(pf, P, tpb, smem, st); break;
    case 16: e = launch_run<16>(pf, P, tpb, smem, st); break;
    default: e = launch_run<32>(pf, P, tpb, smem, st); break;
  }
  if (e != cudaSuccess) return fail(ALERT_ERR_CUDA, std::string("run_kernel: ") + cudaGetErrorString(e));
  return ALERT_OK;
}

int alert_state_init(AlertContext* ctx, const AlertTable* tb, const AlertFilterConfig* cfg, AlertState st,
                     int64_t n, void* cuda_stream) {
  if (!ctx || !tb || !cfg) return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_state_init: NULL argument");
  if (n < 0) return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_state_init: n < 0");
  if (!st.mu || !st.sigma2 || !st.k_gain || !st.q_noise || !st.innov || !st.phi || !st.m_var || !st.group_budget ||
      !st.group_count)
    return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_state_init: NULL state array");
  if (n == 0) return ALERT_OK;
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  state_init_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(st, *cfg, tb->dev.phi0, n);
  CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return ALERT_OK;
}

// Comparison schemes (alert_baselines.cuh): oracle-static's begin() for the
// streams whose policy_aux is still -1, then the one-thread-per-stream loop.
static int run_baseline(AlertContext* ctx, const AlertTable* tb, const AlertFilterConfig* cfg,
                        const AlertSpec* specs, int n_specs, const int32_t* stream_spec, const AlertTrace* tr,
                        AlertState st, const AlertOutputs* out, int policy, int64_t stream_begin,
                        int64_t stream_end, int64_t step_begin, int64_t step_end, cudaStream_t s) {
  CUDA_TRY(cudaSetDevice(ctx->device));
  SpecDev* dspecs = nullptr;
  int r = upload_specs(specs, n_specs, tb, s, &dspecs);
  if (r) return r;
  BaseParams B;
  B.T = tb->dev;
  B.cfg = *cfg;
  B.specs = dspecs;
  B.n_specs = n_specs;
  B.stream_spec = stream_spec;
  B.tr = *tr;
  B.st = st;
  B.out = *out;
  B.policy = policy;
  B.stream_begin = stream_begin;
  B.stream_end = stream_end;
  B.step_begin = step_begin;
  B.step_end = step_end;
  const long long n = stream_end - stream_begin;
  if (policy == ALERT_POLICY_ORACLE_STATIC) {
    static_choice_kernel<<<(unsigned)n, 128, 0, s>>>(B);
    CUDA_TRY(cudaGetLastError());
    ctx->launches++;
  }
  const unsigned grid = (unsigned)((n + 127) / 128);
  switch (policy) {
    case ALERT_POLICY_ORACLE_STATIC: baseline_kernel<ALERT_POLICY_ORACLE_STATIC><<<grid, 128, 0, s>>>(B); break;
    case ALERT_POLICY_SYS_ONLY: baseline_kernel<ALERT_POLICY_SYS_ONLY><<<grid, 128, 0, s>>>(B); break;
    case ALERT_POLICY_APP_ONLY: baseline_kernel<ALERT_POLICY_APP_ONLY><<<grid, 128, 0, s>>>(B); break;
    default: baseline_kernel<ALERT_POLICY_NO_COORD><<<grid, 128, 0, s>>>(B); break;
  }
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(dspecs, s);
  if (e != cudaSuccess) return fail(ALERT_ERR_CUDA, std::string("baseline_kernel: ") + cudaGetErrorString(e));
  ctx->launches++;
  return ALERT_OK;
}

int alert_run(AlertContext* ctx, const AlertTable* tb, const AlertFilterConfig* cfg, const AlertSpec* specs,
              int32_t n_specs, const int32_t* stream_spec, const AlertTrace* tr, AlertState st,
              const AlertOutputs* out, int32_t policy, uint32_t flags, int64_t stream_begin, int64_t stream_end,
              int64_t step_begin, int64_t step_end, void* cuda_stream) {
  NvtxRange nvtx_range("alert_run");
  if (!ctx || !tb || !cfg || !tr || !out) return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_run: NULL argument");
  int r = check_specs(specs, n_specs);
  if (r) return r;
  if (policy < ALERT_POLICY_ALERT || policy > ALERT_POLICY_NO_COORD)
    return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_run: unknown policy");
  const bool baseline = policy >= ALERT_POLICY_ORACLE_STATIC;
  if (policy == ALERT_POLICY_SYS_ONLY && !tb->dev.sys_cells)
    return fail(ALERT_ERR_NO_CANDIDATE, "alert_run: sys-only needs a traditional DNN (AlertSpaceDesc.sys_dnn)");
  if ((policy == ALERT_POLICY_APP_ONLY || policy == ALERT_POLICY_NO_COORD) && !tb->dev.app_first)
    return fail(ALERT_ERR_NO_CANDIDATE, "alert_run: space has no anytime DNN (AlertSpaceDesc.app_dnn)");
  if ((policy == ALERT_POLICY_ORACLE_STATIC || policy == ALERT_POLICY_NO_COORD) && !st.policy_aux)
    return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_run: this policy needs AlertState.policy_aux");
  int kinds = baseline ? 3 : kinds_of(policy, tb);
  if (!kinds) return fail(ALERT_ERR_NO_CANDIDATE, "alert_run: space has no DNN of the policy's kinds");
  if (!tr->slowdown || !tr->n_segments || !tr->seg_end || !tr->seg_phase || !tr->seg_idle || tr->max_segments < 1)
    return fail(ALERT_ERR_INVALID_TRACE, "alert_run: incomplete trace description");
  if (tr->n_goal_segments && (!tr->goal_seg_end || !tr->goal_seg_spec || tr->max_goal_segments < 1))
    return fail(ALERT_ERR_INVALID_TRACE, "alert_run: incomplete goal-change description");
  if (tr->slowdown_dtype != ALERT_DTYPE_F32 && tr->slowdown_dtype != ALERT_DTYPE_F64)
    return fail(ALERT_ERR_INVALID_TRACE, "alert_run: unknown slowdown dtype");
  if (step_begin < tr->step_offset || step_end < step_begin || step_end > tr->step_offset + tr->n_steps)
    return fail(ALERT_ERR_INVALID_TRACE, "alert_run: step range outside the trace buffer");
  if (stream_begin < 0 || stream_end < stream_begin)
    return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_run: bad stream range");
  if (stream_end > 0x7fffffffLL || step_end > 0x7fffffffLL)
    return fail(ALERT_ERR_UNSUPPORTED, "alert_run: stream / step indices must fit in 31 bits");
  if (!tr->stream_row && stream_end > tr->n_rows)
    return fail(ALERT_ERR_INVALID_TRACE, "alert_run: more streams than trace rows and no stream_row map");
  if (!st.mu || !st.sigma2 || !st.k_gain || !st.q_noise || !st.innov || !st.phi || !st.m_var || !st.group_budget ||
      !st.group_count)
    return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_run: NULL state array");
  if ((out->decision || out->energy || out->accuracy || out->latency || out->mu || out->sigma2 ||
       out->oracle_decision || out->forced) &&
      (out->stream_stride == 0 && out->step_stride == 0))
    return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_run: per-step outputs need strides");
  if (stream_end == stream_begin || step_end == step_begin) return ALERT_OK;
  if (baseline && (flags & ALERT_FLAG_FRESH)) {  // the fused comparison schemes read state / accumulate
    CUDA_TRY(cudaSetDevice(ctx->device));
    const long long nr = stream_end - stream_begin;
    AlertState sub = st;
    sub.mu += stream_begin; sub.sigma2 += stream_begin; sub.k_gain += stream_begin; sub.q_noise += stream_begin;
    sub.innov += stream_begin; sub.phi += stream_begin; sub.m_var += stream_begin;
    sub.group_budget += stream_begin; sub.group_count += stream_begin;
    if (sub.policy_aux) sub.policy_aux += stream_begin;
    state_init_kernel<<<(unsigned)((nr + 255) / 256), 256, 0, (cudaStream_t)cuda_stream>>>(sub, *cfg, tb->dev.phi0, nr);
    CUDA_TRY(cudaGetLastError());
    ctx->launches++;
    if (out->agg)
      CUDA_TRY(cudaMemsetAsync(out->agg + stream_begin * ALERT_AGG_FIELDS, 0, sizeof(double) * ALERT_AGG_FIELDS * nr,
                               (cudaStream_t)cuda_stream));
  }
  if (baseline) return run_baseline(ctx, tb, cfg, specs, n_specs, stream_spec, tr, st, out, policy, stream_begin,
                                    stream_end, step_begin, step_end, (cudaStream_t)cuda_stream);
  int W = pick_lanes(ctx, tb);
  RunParams P;
  auto stage = [&](int tpb) {
    run_staging(tb, specs, n_specs, tpb, W, P, policy, flags);
    size_t sm = run_smem(tb, n_specs, tpb, W, P);
    if (P.units_smem && T_units_large(tb)) {
      // large unit tables are read through L1 instead when staging them
      // would not fit or would cost resident blocks (128 registers/thread)
      int sm_per_sm = 0, dev = ctx->device;
      cudaDeviceGetAttribute(&sm_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
      P.units_smem = 0;
      const size_t without = run_smem(tb, n_specs, tpb, W, P);
      const int by_regs = 65536 / (128 * tpb);
      auto resident = [&](size_t b) { return std::min(by_regs, (int)((size_t)sm_per_sm / (b + 1024))); };
      if ((int)sm <= ctx->max_smem && resident(sm) >= resident(without)) P.units_smem = 1;
      else sm = without;
    }
    if ((int)sm > ctx->max_smem && P.fast_smem) {  // no room for the fast-scan tables
      P.fast_smem = 0;
      sm = run_smem(tb, n_specs, tpb, W, P);
    }
    return sm;
  };
  // Block size: 64 threads by default (fine-grained waves for ~10^4-10^5
  // streams); a large table (shared memory per block > 40 KB) with enough
  // streams gets 512-thread blocks so the staged table is shared by 8x more
  // tiles and occupancy is not capped by shared memory.
  int tpb = ctx->tpb;
  size_t smem = stage(tpb);
  if (ctx->tpb_auto && smem > 40 * 1024 && (stream_end - stream_begin) * W >= 148LL * 2 * 256) {
    // one 512-thread block per SM holds the table once (two 256-thread
    // blocks hold it twice) at the same 16 warps: room for the unit table
    // (c4: +6%, c5: +4% measured); 256 when 512 does not fit
    tpb = 512;
    smem = stage(tpb);
    if ((int)smem > ctx->max_smem) {
      tpb = 256;
      smem = stage(tpb);
    }
  }
  if ((int)smem > ctx->max_smem) return fail(ALERT_ERR_UNSUPPORTED, "alert_run: table exceeds shared memory");
  idle_table(*cfg, P);
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  SpecDev* dspecs = nullptr;
  r = upload_specs(specs, n_specs, tb, s, &dspecs);
  if (r) return r;
  P.T = tb->dev;
  P.cfg = *cfg;
  P.specs = dspecs;
  P.n_specs = n_specs;
  P.stream_spec = stream_spec;
  P.tr = *tr;
  P.st = st;
  P.out = *out;
  P.policy = policy;
  P.flags = flags;
  P.kinds = kinds;
  P.stream_begin = stream_begin;
  P.stream_end = stream_end;
  P.step_begin = step_begin;
  P.step_end = step_end;
  int pf = policy == ALERT_POLICY_ORACLE ? PF_ORACLE : policy == ALERT_POLICY_ALERT_WITH_ORACLE ? PF_BOTH : PF_ALERT;
  float* dzlo = nullptr;
  if (P.fast_smem) {  // fast scan staged by run_staging: compute the thresholds on the stream
    const int n_tdnn = tb->dev.n_trad / tb->dev.n_powers;
    const float4* rows = P.fast_rows ? tb->dev.trad_rows : nullptr;
    const long long nz = (long long)n_specs * (n_tdnn + 1) + (rows ? (long long)n_specs * n_tdnn : 0);
    CUDA_TRY(cudaMallocAsync((void**)&dzlo, sizeof(float) * nz, s));
    zlo_kernel<<<(unsigned)((nz + 127) / 128), 128, 0, s>>>(dspecs, n_specs, tb->dev.c64, tb->dev.n_powers, n_tdnn,
                                                          rows, dzlo);
    CUDA_TRY(cudaGetLastError());
    ctx->launches++;
    P.zlo = dzlo;
  }
  P.work = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&P.work, sizeof(unsigned long long), s));  // persistent work counter
  r = dispatch_run(W, pf, P, tpb, smem, s);
  cudaFreeAsync(P.work, s);
  cudaFreeAsync(dspecs, s);
  if (dzlo) cudaFreeAsync(dzlo, s);
  if (r) return r;
  ctx->launches++;
  return ALERT_OK;
}

int alert_static_choice(AlertContext* ctx, const AlertTable* tb, const AlertSpec* specs, int32_t n_specs,
                        const int32_t* stream_spec, const AlertTrace* tr, AlertState st, int64_t stream_begin,
                        int64_t stream_end, int64_t step_begin, int64_t step_end, void* cuda_stream) {
  if (!ctx || !tb || !tr) return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_static_choice: NULL argument");
  int r = check_specs(specs, n_specs);
  if (r) return r;
  if (!st.policy_aux) return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_static_choice: needs AlertState.policy_aux");
  if (!tr->slowdown || !tr->n_segments || !tr->seg_end || !tr->seg_phase || !tr->seg_idle || tr->max_segments < 1)
    return fail(ALERT_ERR_INVALID_TRACE, "alert_static_choice: incomplete trace description");
  if (tr->n_goal_segments && (!tr->goal_seg_end || !tr->goal_seg_spec || tr->max_goal_segments < 1))
    return fail(ALERT_ERR_INVALID_TRACE, "alert_static_choice: incomplete goal-change description");
  if (step_begin < tr->step_offset || step_end <= step_begin || step_end > tr->step_offset + tr->n_steps)
    return fail(ALERT_ERR_INVALID_TRACE, "alert_static_choice: step range outside the trace buffer");
  if (stream_begin < 0 || stream_end < stream_begin || stream_end > 0x7fffffffLL)
    return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_static_choice: bad stream range");
  if (!tr->stream_row && stream_end > tr->n_rows)
    return fail(ALERT_ERR_INVALID_TRACE, "alert_static_choice: more streams than trace rows and no stream_row map");
  if (stream_end == stream_begin) return ALERT_OK;
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  SpecDev* dspecs = nullptr;
  r = upload_specs(specs, n_specs, tb, s, &dspecs);
  if (r) return r;
  BaseParams B{};
  B.T = tb->dev;
  B.specs = dspecs;
  B.n_specs = n_specs;
  B.stream_spec = stream_spec;
  B.tr = *tr;
  B.st = st;
  B.policy = ALERT_POLICY_ORACLE_STATIC;
  B.stream_begin = stream_begin;
  B.stream_end = stream_end;
  B.step_begin = step_begin;
  B.step_end = step_end;
  static_choice_kernel<<<(unsigned)(stream_end - stream_begin), 128, 0, s>>>(B);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(dspecs, s);
  if (e != cudaSuccess) return fail(ALERT_ERR_CUDA, std::string("static_choice_kernel: ") + cudaGetErrorString(e));
  ctx->launches++;
  return ALERT_OK;
}

int alert_baseline_decide(AlertContext* ctx, const AlertTable* tb, const AlertSpec* specs, int32_t n_specs,
                          const int32_t* stream_spec, AlertState st, const double* plan_goal, int32_t policy,
                          uint32_t* decision, int64_t n, void* cuda_stream) {
  if (!ctx || !tb || !plan_goal || !decision)
    return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_baseline_decide: NULL argument");
  int r = check_specs(specs, n_specs);
  if (r) return r;
  if (policy < ALERT_POLICY_ORACLE_STATIC || policy > ALERT_POLICY_NO_COORD)
    return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_baseline_decide: policy must be a comparison scheme");
  if (policy == ALERT_POLICY_SYS_ONLY && !tb->dev.sys_cells)
    return fail(ALERT_ERR_NO_CANDIDATE, "alert_baseline_decide: sys-only needs a traditional DNN");
  if ((policy == ALERT_POLICY_APP_ONLY || policy == ALERT_POLICY_NO_COORD) && !tb->dev.app_first)
    return fail(ALERT_ERR_NO_CANDIDATE, "alert_baseline_decide: space has no anytime DNN");
  if ((policy == ALERT_POLICY_ORACLE_STATIC || policy == ALERT_POLICY_NO_COORD) && !st.policy_aux)
    return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_baseline_decide: this policy needs AlertState.policy_aux");
  if ((policy != ALERT_POLICY_ORACLE_STATIC) && (!st.mu || !st.sigma2 || !st.phi))
    return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_baseline_decide: NULL state array");
  if (n <= 0) return n < 0 ? fail(ALERT_ERR_INVALID_ARGUMENT, "alert_baseline_decide: n < 0") : ALERT_OK;
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  baseline_decide_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(tb->dev, nullptr, n_specs, stream_spec, st,
                                                                     plan_goal, policy, decision, n);
  CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return ALERT_OK;
}

int alert_decide(AlertContext* ctx, const AlertTable* tb, const AlertSpec* specs, int32_t n_specs,
                 const int32_t* stream_spec, AlertState st, const double* plan_goal, int32_t policy, uint32_t flags,
                 uint32_t* decision, int64_t n, void* cuda_stream) {
  if (!ctx || !tb || !plan_goal || !decision) return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_decide: NULL argument");
  int r = check_specs(specs, n_specs);
  if (r) return r;
  if (policy < ALERT_POLICY_ALERT || policy > ALERT_POLICY_ALERT_TRAD)
    return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_decide: policy must be alert, alert-any or alert-trad");
  int kinds = kinds_of(policy, tb);
  if (!kinds) return fail(ALERT_ERR_NO_CANDIDATE, "alert_decide: space has no DNN of the policy's kinds");
  if (n <= 0) return n < 0 ? fail(ALERT_ERR_INVALID_ARGUMENT, "alert_decide: n < 0") : ALERT_OK;
  size_t smem = table_smem(tb, pick_lanes(ctx, tb));
  if ((int)smem > ctx->max_smem) return fail(ALERT_ERR_UNSUPPORTED, "alert_decide: table exceeds shared memory");
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  SpecDev* dspecs = nullptr;
  r = upload_specs(specs, n_specs, tb, s, &dspecs);
  if (r) return r;
  StepParams P{};
  P.T = tb->dev;
  P.specs = dspecs;
  P.n_specs = n_specs;
  P.stream_spec = stream_spec;
  P.st = st;
  P.goal = plan_goal;
  P.policy = policy;
  P.flags = flags;
  P.kinds = kinds;
  P.n = n;
  cudaError_t e;
  switch (pick_lanes(ctx, tb)) {
    case 1: e = launch_decide<1>(P, decision, std::min(ctx->tpb, 256), smem, s); break;
    case 2: e = launch_decide<2>(P, decision, std::min(ctx->tpb, 256), smem, s); break;
    case 4: e = launch_decide<4>(P, decision, std::min(ctx->tpb, 256), smem, s); break;
    case 8: e = launch_decide<8>(P, decision, std::min(ctx->tpb, 256), smem, s); break;
    case 16: e = launch_decide<16>(P, decision, std::min(ctx->tpb, 256), smem, s); break;
    default: e = launch_decide<32>(P, decision, std::min(ctx->tpb, 256), smem, s); break;
  }
  if (e != cudaSuccess) r = fail(ALERT_ERR_CUDA, std::string("decide_kernel: ") + cudaGetErrorString(e));
  cudaFreeAsync(dspecs, s);
  if (r) return r;
  ctx->launches++;
  return ALERT_OK;
}

int alert_predict(AlertContext* ctx, const AlertTable* tb, const AlertSpec* specs, int32_t n_specs,
                  const int32_t* stream_spec, AlertState st, const double* plan_goal, AlertPrediction* out,
                  int64_t n, void* cuda_stream) {
  if (!ctx || !tb || !plan_goal || !out) return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_predict: NULL argument");
  int r = check_specs(specs, n_specs);
  if (r) return r;
  if (n <= 0) return n < 0 ? fail(ALERT_ERR_INVALID_ARGUMENT, "alert_predict: n < 0") : ALERT_OK;
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  SpecDev* dspecs = nullptr;
  r = upload_specs(specs, n_specs, tb, s, &dspecs);
  if (r) return r;
  // per-candidate (dnn, power, stage) arrays in stream-ordered scratch
  int nc = tb->n_cand;
  int32_t* meta = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&meta, sizeof(int32_t) * 3 * nc, s));
  CUDA_TRY(cudaMemcpyAsync(meta, tb->cand_dnn.data(), 4 * nc, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(meta + nc, tb->cand_power.data(), 4 * nc, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(meta + 2 * nc, tb->cand_stage.data(), 4 * nc, cudaMemcpyHostToDevice, s));
  StepParams P{};
  P.T = tb->dev;
  P.specs = dspecs;
  P.n_specs = n_specs;
  P.stream_spec = stream_spec;
  P.st = st;
  P.goal = plan_goal;
  P.n = n;
  long long total = n * nc;
  unsigned blocks = (unsigned)std::min<long long>((total + 255) / 256, 65535LL * 4);
  predict_kernel<<<blocks, 256, 0, s>>>(P, out, meta, meta + nc, meta + 2 * nc);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(meta, s);
  cudaFreeAsync(dspecs, s);
  if (e != cudaSuccess) return fail(ALERT_ERR_CUDA, std::string("predict_kernel: ") + cudaGetErrorString(e));
  ctx->launches++;
  return ALERT_OK;
}

int alert_observe(AlertContext* ctx, const AlertTable* tb, const AlertFilterConfig* cfg, AlertState st,
                  const double* fb_latency, const double* fb_t_prof, const double* idle, const int32_t* power,
                  int64_t n, void* cuda_stream) {
  if (!ctx || !tb || !cfg || !fb_latency || !fb_t_prof || !idle || !power)
    return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_observe: NULL argument");
  if (n <= 0) return n < 0 ? fail(ALERT_ERR_INVALID_ARGUMENT, "alert_observe: n < 0") : ALERT_OK;
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  observe_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(tb->dev, *cfg, st, fb_latency, fb_t_prof, idle, power, n);
  CUDA_TRY(cudaGetLastError());
  ctx->launches++;
  return ALERT_OK;
}

int alert_oracle_decide(AlertContext* ctx, const AlertTable* tb, const AlertSpec* specs, int32_t n_specs,
                        const int32_t* stream_spec, const double* sd, const double* idle, const double* plan_goal,
                        uint32_t flags, uint32_t* decision, AlertPrediction* exact, int64_t n, void* cuda_stream) {
  if (!ctx || !tb || !sd || !idle || !plan_goal || !decision)
    return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_oracle_decide: NULL argument");
  int r = check_specs(specs, n_specs);
  if (r) return r;
  if (n <= 0) return n < 0 ? fail(ALERT_ERR_INVALID_ARGUMENT, "alert_oracle_decide: n < 0") : ALERT_OK;
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  SpecDev* dspecs = nullptr;
  r = upload_specs(specs, n_specs, tb, s, &dspecs);
  if (r) return r;
  int W = pick_lanes(ctx, tb);
  int tpb = ctx->tpb;
  cudaError_t e;
  switch (W) {
    case 1: e = launch_oracle<1>(tb->dev, dspecs, n_specs, stream_spec, sd, idle, plan_goal, decision, exact, n, tpb, flags, s); break;
    case 2: e = launch_oracle<2>(tb->dev, dspecs, n_specs, stream_spec, sd, idle, plan_goal, decision, exact, n, tpb, flags, s); break;
    case 4: e = launch_oracle<4>(tb->dev, dspecs, n_specs, stream_spec, sd, idle, plan_goal, decision, exact, n, tpb, flags, s); break;
    case 8: e = launch_oracle<8>(tb->dev, dspecs, n_specs, stream_spec, sd, idle, plan_goal, decision, exact, n, tpb, flags, s); break;
    case 16: e = launch_oracle<16>(tb->dev, dspecs, n_specs, stream_spec, sd, idle, plan_goal, decision, exact, n, tpb, flags, s); break;
    default: e = launch_oracle<32>(tb->dev, dspecs, n_specs, stream_spec, sd, idle, plan_goal, decision, exact, n, tpb, flags, s); break;
  }
  cudaFreeAsync(dspecs, s);
  if (e != cudaSuccess) return fail(ALERT_ERR_CUDA, std::string("oracle_decide_kernel: ") + cudaGetErrorString(e));
  ctx->launches++;
  return ALERT_OK;
}

int alert_reduce(AlertContext* ctx, const double* agg, int64_t n, double* out, void* cuda_stream) {
  if (!ctx || !agg || !out) return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_reduce: NULL argument");
  if (n < 0) return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_reduce: n < 0");
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  long long nb = (n + kReduceChunk - 1) / kReduceChunk;
  if (nb == 0) {
    CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double) * ALERT_AGG_FIELDS, s));
    return ALERT_OK;
  }
  double* partial = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&partial, sizeof(double) * ALERT_AGG_FIELDS * nb, s));
  reduce_partial_kernel<<<(unsigned)nb, kReduceRep * ALERT_AGG_FIELDS, 0, s>>>(agg, n, partial);
  reduce_final_kernel<<<1, 128, 0, s>>>(partial, nb, out);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(partial, s);
  if (e != cudaSuccess) return fail(ALERT_ERR_CUDA, std::string("reduce: ") + cudaGetErrorString(e));
  ctx->launches += 2;
  return ALERT_OK;
}

// numpy pairwise_sum recursion (n > 128: split at n/2 rounded down to a
// multiple of 8) as leaves + a post-order program
static void np_pairwise_plan(long long off, long long n, std::vector<long long>& leaves, std::vector<int>& prog) {
  if (n <= 128) {
    prog.push_back((int)(leaves.size() / 2));
    leaves.push_back(off);
    leaves.push_back(n);
    return;
  }
  long long n2 = n / 2;
  n2 -= n2 % 8;
  np_pairwise_plan(off, n2, leaves, prog);
  np_pairwise_plan(off + n2, n - n2, leaves, prog);
  prog.push_back(-1);
}

int alert_xi_stats(AlertContext* ctx, const double* num, const double* den, int64_t n, int32_t bins,
                   int64_t* counts, double* edges, double* mean_sd, void* cuda_stream) {
  if (!ctx || !num || !counts || !edges || !mean_sd) return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_xi_stats: NULL argument");
  if (n < 1 || bins < 1) return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_xi_stats: need n >= 1 values and bins >= 1");
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  std::vector<long long> leaves;
  std::vector<int> prog;
  np_pairwise_plan(0, n, leaves, prog);
  const int n_leaves = (int)(leaves.size() / 2);
  char* buf = nullptr;
  const size_t b_leaves = sizeof(long long) * leaves.size(), b_prog = sizeof(int) * prog.size();
  const size_t bytes = b_leaves + b_prog + sizeof(double) * (size_t)n_leaves + 2 * sizeof(double) + 64;
  CUDA_TRY(cudaMallocAsync((void**)&buf, bytes, s));
  long long* d_leaves = reinterpret_cast<long long*>(buf);
  int* d_prog = reinterpret_cast<int*>(buf + b_leaves);
  double* d_sums = reinterpret_cast<double*>(buf + ((b_leaves + b_prog + 15) & ~size_t(15)));
  double* d_scr = d_sums + n_leaves;
  CUDA_TRY(cudaMemcpyAsync(d_leaves, leaves.data(), b_leaves, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(d_prog, prog.data(), b_prog, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(int64_t) * bins, s));
  xi_minmax_kernel<<<1, 1024, 0, s>>>(num, den, n, bins, edges, d_scr);
  xi_hist_kernel<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 8), 256, 0, s>>>(
      num, den, n, bins, edges, d_scr, reinterpret_cast<unsigned long long*>(counts));
  for (int mode = 0; mode < 2; ++mode) {
    xi_leaf_kernel<<<(n_leaves + 127) / 128, 128, 0, s>>>(num, den, d_leaves, n_leaves, mode, mean_sd, d_sums);
    xi_combine_kernel<<<1, 1, 0, s>>>(d_prog, (int)prog.size(), d_sums, n, mode, mean_sd);
  }
  CUDA_TRY(cudaGetLastError());
  cudaFreeAsync(buf, s);
  ctx->launches += 6;
  return ALERT_OK;
}

// On-device realization (simulator.py:221-235 recipe, Philox streams).
__global__ void realize_kernel(const AlertPhaseDesc* ph, int n_ph, unsigned long long seed, long long off,
                               long long n, void* out, int f64) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  curandStatePhilox4_32_10_t rs;
  curand_init(seed, (unsigned long long)(off + k), 0ull, &rs);
  long long step = 0;
  for (int p = 0; p < n_ph; ++p) {
    const AlertPhaseDesc d = ph[p];
    for (long long i = 0; i < d.length; ++i, ++step) {
      double s;
      switch (d.dist) {
        case ALERT_DIST_CONSTANT: s = d.a; break;
        case ALERT_DIST_GAUSSIAN: s = d.a + d.b * curand_normal_double(&rs); break;
        case ALERT_DIST_LOGNORMAL: s = exp(d.a + d.b * curand_normal_double(&rs)); break;
        default: s = d.a + (d.b - d.a) * curand_uniform_double(&rs); break;
      }
      if (d.input_noise_sd > 0.0) s *= 1.0 + d.input_noise_sd * curand_normal_double(&rs);
      s = fmax(s, 0.01);  // MIN_SLOWDOWN, simulator.py:28
      if (f64) static_cast<double*>(out)[step * n + k] = s;
      else static_cast<float*>(out)[step * n + k] = (float)s;
    }
  }
}

int alert_realize(AlertContext* ctx, const AlertPhaseDesc* phases, int32_t n_phases, uint64_t seed,
                  int64_t stream_offset, int64_t n_streams, void* out, int32_t dtype, void* cuda_stream) {
  if (!ctx || !phases || !out || n_phases < 1) return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_realize: bad argument");
  if (dtype != ALERT_DTYPE_F32 && dtype != ALERT_DTYPE_F64)
    return fail(ALERT_ERR_INVALID_ARGUMENT, "alert_realize: unknown dtype");
  for (int p = 0; p < n_phases; ++p)
    if (phases[p].length < 0 || phases[p].dist < 0 || phases[p].dist > ALERT_DIST_UNIFORM)
      return fail(ALERT_ERR_INVALID_TRACE, "alert_realize: bad phase description");
  if (n_streams <= 0) return n_streams < 0 ? fail(ALERT_ERR_INVALID_ARGUMENT, "alert_realize: n < 0") : ALERT_OK;
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  AlertPhaseDesc* d = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&d, sizeof(AlertPhaseDesc) * n_phases, s));
  CUDA_TRY(cudaMemcpyAsync(d, phases, sizeof(AlertPhaseDesc) * n_phases, cudaMemcpyHostToDevice, s));
  realize_kernel<<<(unsigned)((n_streams + 127) / 128), 128, 0, s>>>(d, n_phases, seed, stream_offset, n_streams, out,
                                                                    dtype == ALERT_DTYPE_F64);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(d, s);
  if (e != cudaSuccess) return fail(ALERT_ERR_CUDA, std::string("realize_kernel: ") + cudaGetErrorString(e));
  ctx->launches++;
  return ALERT_OK;
}
