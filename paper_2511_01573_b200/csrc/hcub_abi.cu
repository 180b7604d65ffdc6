// Host runtime behind include/hcub_b200.h: region-store workers, the
// device-resident single-worker loop (ref pkg/src/hcub/driver.py:237-323) and
// the operator-level entry points.  No CPU fallback: every numeric result
// comes from the kernels in k1_eval.cuh / store_kernels.cuh.
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl is dlopen()ed (hcub_comm_init)

#include <algorithm>
#include <atomic>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges for nsys timelines
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hcub_b200.h"
#include "k1_table.cuh"
#include "k1_gm9.cuh"
#include "k1_gk.cuh"
#include "store_kernels.cuh"

// ---------------------------------------------------------------------------
// errors

static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) {                                                                  \
      return fail(e_ == cudaErrorMemoryAllocation ? HCUB_E_OOM : HCUB_E_CUDA, "%s: %s (%s:%d)", #call, \
                  cudaGetErrorString(e_), __FILE__, __LINE__);                                \
    }                                                                                         \
  } while (0)

#define TRY(call)            \
  do {                       \
    int r_ = (call);         \
    if (r_) return r_;       \
  } while (0)

// ---------------------------------------------------------------------------
// K1 launchers (one TU per integrand kind, see k1_inst.cu)

#define DECL(FN)                                                                                                \
  extern "C" cudaError_t hcub_launch_k1_fn##FN(int, const K1Args*, const RuleC*, const FnParams*, unsigned, unsigned, \
                                               cudaStream_t);                                                  \
  extern "C" cudaError_t hcub_launch_points_fn##FN(int, const double*, int64_t, double*, const FnParams*, cudaStream_t);
DECL(1) DECL(2) DECL(3) DECL(4) DECL(5) DECL(6) DECL(7) DECL(8)
#undef DECL

#define DECLT(FN) \
  extern "C" cudaError_t hcub_launch_k1t_fn##FN(int, const K1Args*, const TableArgs*, const FnParams*, unsigned, unsigned, \
                                                cudaStream_t);
DECLT(1) DECLT(2) DECLT(3) DECLT(4) DECLT(5) DECLT(6) DECLT(7) DECLT(8)
#undef DECLT
typedef cudaError_t (*k1t_launcher)(int, const K1Args*, const TableArgs*, const FnParams*, unsigned, unsigned,
                                    cudaStream_t);
static const k1t_launcher K1T_LAUNCH[9] = {nullptr, hcub_launch_k1t_fn1, hcub_launch_k1t_fn2, hcub_launch_k1t_fn3,
                                           hcub_launch_k1t_fn4, hcub_launch_k1t_fn5, hcub_launch_k1t_fn6,
                                           hcub_launch_k1t_fn7, hcub_launch_k1t_fn8};
#define DECL9(FN) \
  extern "C" cudaError_t hcub_launch_k9_fn##FN(int, const K1Args*, const Rule9C*, const FnParams*, cudaStream_t);
DECL9(1) DECL9(2) DECL9(3) DECL9(4) DECL9(5) DECL9(6) DECL9(7) DECL9(8)
#undef DECL9
typedef cudaError_t (*k9_launcher)(int, const K1Args*, const Rule9C*, const FnParams*, cudaStream_t);
static const k9_launcher K9_LAUNCH[9] = {nullptr, hcub_launch_k9_fn1, hcub_launch_k9_fn2, hcub_launch_k9_fn3,
                                         hcub_launch_k9_fn4, hcub_launch_k9_fn5, hcub_launch_k9_fn6,
                                         hcub_launch_k9_fn7, hcub_launch_k9_fn8};
#define DECLG(FN) \
  extern "C" cudaError_t hcub_launch_k1gk_fn##FN(int, const K1Args*, const GkArgs*, const FnParams*, int64_t, int64_t, \
                                                 double*, cudaStream_t);
DECLG(1) DECLG(2) DECLG(3) DECLG(4) DECLG(5) DECLG(6) DECLG(7) DECLG(8)
#undef DECLG
typedef cudaError_t (*k1gk_launcher)(int, const K1Args*, const GkArgs*, const FnParams*, int64_t, int64_t, double*,
                                     cudaStream_t);
static const k1gk_launcher K1GK_LAUNCH[9] = {nullptr, hcub_launch_k1gk_fn1, hcub_launch_k1gk_fn2,
                                             hcub_launch_k1gk_fn3, hcub_launch_k1gk_fn4, hcub_launch_k1gk_fn5,
                                             hcub_launch_k1gk_fn6, hcub_launch_k1gk_fn7, hcub_launch_k1gk_fn8};

// 15-point Kronrod extension of the 7-point Gauss rule on [-1, 1]: the
// standard abscissae/weights (ref rules.py:287-329), ascending order.
static GkArgs make_gk(int d) {
  static const double xh[8] = {0.991455371120812639206854697526329, 0.949107912342758524526189684047851,
                               0.864864423359769072789712788640926, 0.741531185599394439863864773280788,
                               0.586087235467691130294144838258730, 0.405845151377397166906606412076961,
                               0.207784955007898467600689403773245, 0.0};
  static const double wkh[8] = {0.022935322010529224963732008058970, 0.063092092629978553290700663189204,
                                0.104790010322250183839876322541518, 0.140653259715525918745189590510238,
                                0.169004726639267902826583426598550, 0.190350578064785409913256402421014,
                                0.204432940075298892414161999234649, 0.209482141084727828012999174891714};
  static const double wgh[8] = {0.0, 0.129484966168869693270611432679082, 0.0, 0.279705391489276667901467771423780,
                                0.0, 0.381830050505118944950369775488975, 0.0, 0.417959183673469387755102040816327};
  GkArgs g{};
  for (int q = 0; q < 15; ++q) {
    const int h = q < 8 ? q : 14 - q;  // mirror: nodes -xh[0..6], +xh[7..0]
    g.node[q] = q < 7 ? -xh[h] : xh[h];
    g.wk[q] = wkh[h];
    g.ratio[q] = wgh[h] / wkh[h];
  }
  int K = 1;
  for (int j = 0; j < d; ++j) K *= 15;
  g.K = K;
  g.chunks = (K + GK_CHUNK - 1) / GK_CHUNK;
  g.twod = std::ldexp(1.0, d);
  return g;
}

typedef cudaError_t (*k1_launcher)(int, const K1Args*, const RuleC*, const FnParams*, unsigned, unsigned, cudaStream_t);
typedef cudaError_t (*pt_launcher)(int, const double*, int64_t, double*, const FnParams*, cudaStream_t);
static const k1_launcher K1_LAUNCH[9] = {nullptr, hcub_launch_k1_fn1, hcub_launch_k1_fn2, hcub_launch_k1_fn3,
                                         hcub_launch_k1_fn4, hcub_launch_k1_fn5, hcub_launch_k1_fn6,
                                         hcub_launch_k1_fn7, hcub_launch_k1_fn8};
static const pt_launcher PT_LAUNCH[9] = {nullptr, hcub_launch_points_fn1, hcub_launch_points_fn2,
                                         hcub_launch_points_fn3, hcub_launch_points_fn4, hcub_launch_points_fn5,
                                         hcub_launch_points_fn6, hcub_launch_points_fn7, hcub_launch_points_fn8};

// lanes per region: enough threads to cover the machine several times over
// (hcub_set_k1_lanes overrides the choice process-wide; tests use it to put
// small golden batches through the one-lane-per-region path).
static std::atomic<int> g_k1_log2g{-1};
static int pick_log2g(int64_t n, int sms) {
  const int forced = g_k1_log2g.load(std::memory_order_relaxed);
  if (forced >= 0) return forced;
  const int64_t target = (int64_t)sms * 2048;
  int lg = 0;
  while (lg < 5 && n * (1ll << lg) < target) ++lg;
  return lg;
}

// ---------------------------------------------------------------------------
// descriptors

// Rule tables on the device: host table -> device copy + kernel arguments.
struct DevTable {
  TableArgs args{};
  double* buf = nullptr;  // pts | w | we
  int dev = 0;
  void release() {
    if (buf) { cudaSetDevice(dev); cudaFree(buf); }
    buf = nullptr;
  }
};

static int upload_table(const hcub_rule* r, int device, cudaStream_t st, DevTable* t) {
  if (r->K < 1 || r->K > (1 << 26) || !r->points || !r->weights || !r->embedded_weights)
    return fail(HCUB_E_ARG, "bad rule table");
  const int d = r->d;
  const size_t n = (size_t)r->K * (d + 2);
  t->dev = device;
  CK(cudaMalloc(&t->buf, n * sizeof(double)));
  CK(cudaMemcpyAsync(t->buf, r->points, (size_t)r->K * d * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(t->buf + (size_t)r->K * d, r->weights, (size_t)r->K * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(t->buf + (size_t)r->K * (d + 1), r->embedded_weights, (size_t)r->K * 8, cudaMemcpyHostToDevice, st));
  TableArgs& a = t->args;
  a.pts = t->buf;
  a.w = t->buf + (size_t)r->K * d;
  a.we = t->buf + (size_t)r->K * (d + 1);
  a.K = (int)r->K;
  a.has_pairs = r->has_axis_pairs;
  a.center = r->center_index;
  for (int k = 0; k < HCUB_MAXD; ++k)
    for (int q = 0; q < 4; ++q) a.pairs[k][q] = r->axis_pairs[k][q];
  a.ratio = r->fourth_diff_ratio;
  a.null_center = r->null_center_weight;
  a.null_axis = r->null_axis_weight;
  a.twod = std::ldexp(1.0, d);
  return 0;
}

static int make_rule9(const hcub_rule* r, Rule9C* out);

static int make_rule(const hcub_rule* r, RuleC* rc) {
  if (!r) return fail(HCUB_E_ARG, "rule is NULL");
  if (r->kind == 2) {  // tensor Gauss-Kronrod (ref rules.py:332-357)
    if (r->d < 1 || r->d > 6) return fail(HCUB_E_DIM, "tensor Gauss-Kronrod rule is capped at d <= 6, got %d", r->d);
    memset(rc, 0, sizeof *rc);
    rc->twod = std::ldexp(1.0, r->d);
    return 0;
  }
  if (r->kind == 3) {  // degree-9 generator form (make_rule9 checks the table)
    Rule9C tmp;
    TRY(make_rule9(r, &tmp));
    memset(rc, 0, sizeof *rc);
    rc->twod = std::ldexp(1.0, r->d);
    return 0;
  }
  if (r->kind == 1) {
    if (r->d < 1 || r->d > HCUB_MAX_DIM) return fail(HCUB_E_DIM, "rule tables support 1 <= d <= %d, got %d", HCUB_MAX_DIM, r->d);
    if (r->has_axis_pairs && (r->center_index < 0 || r->center_index >= r->K)) return fail(HCUB_E_ARG, "bad center index");
    memset(rc, 0, sizeof *rc);
    rc->twod = std::ldexp(1.0, r->d);
    return 0;
  }
  if (r->d < 2 || r->d > HCUB_MAX_DIM)
    return fail(HCUB_E_DIM, "fully symmetric rule supports 2 <= d <= %d, got %d", HCUB_MAX_DIM, r->d);
  rc->lam2 = r->lam2; rc->lam3 = r->lam3; rc->lam4 = r->lam4; rc->lam5 = r->lam5;
  for (int i = 0; i < 5; ++i) { rc->w[i] = r->w[i]; rc->we[i] = r->we[i]; }
  rc->ratio = r->fourth_diff_ratio;
  rc->null_center = r->null_center_weight;
  rc->null_axis = r->null_axis_weight;
  rc->twod = std::ldexp(1.0, r->d);
  return 0;
}

// kind 3: the degree-9 table of rule9.py (parse_rule_table of gm9_rule_text)
// -> generator form.  The orbit layout is fixed (rule9.py order); every
// orbit's nodes must carry one weight pair and the expected magnitudes, so a
// table that is not that family is rejected instead of mis-evaluated.
static int make_rule9(const hcub_rule* r, Rule9C* out) {
  const int d = r->d;
  if (d < 2 || d > 10) return fail(HCUB_E_DIM, "degree-9 generator kernel supports 2 <= d <= 10, got %d (use the node table)", d);
  const int64_t n3 = d >= 3 ? 4ll * d * (d - 1) * (d - 2) / 3 : 0;
  const int64_t size[O9_N] = {1, 2ll * d, 2ll * d, 2ll * d, 2ll * d, 2ll * d * (d - 1), 4ll * d * (d - 1), n3, 1ll << d};
  int64_t start[O9_N + 1] = {0};
  for (int o = 0; o < O9_N; ++o) start[o + 1] = start[o] + size[o];
  if (!r->points || !r->weights || !r->embedded_weights || r->K != start[O9_N] || !r->has_axis_pairs)
    return fail(HCUB_E_ARG, "not a degree-9 (rule9) table: %lld nodes", (long long)r->K);
  memset(out, 0, sizeof *out);
  for (int o = 0; o < O9_N; ++o) {
    if (!size[o]) continue;
    const int64_t s0 = start[o];
    out->w[o] = r->weights[s0];
    out->we[o] = r->embedded_weights[s0];
    for (int64_t i = s0; i < start[o + 1]; ++i)
      if (r->weights[i] != out->w[o] || r->embedded_weights[i] != out->we[o])
        return fail(HCUB_E_ARG, "not a degree-9 (rule9) table: orbit %d weights differ", o);
  }
  auto mag = [&](int o, int which) {  // which = 0: largest, 1: smallest nonzero |coordinate| of the orbit's first node
    double hi = 0.0, lo = INFINITY;
    for (int j = 0; j < d; ++j) {
      const double v = std::fabs(r->points[start[o] * d + j]);
      if (v > 0.0) { hi = std::max(hi, v); lo = std::min(lo, v); }
    }
    return which ? lo : hi;
  };
  out->g[0] = mag(O9_A0, 0);
  out->g[1] = mag(O9_A1, 0);
  out->g[2] = mag(O9_A2, 0);
  out->g[3] = mag(O9_A3, 0);
  if (mag(O9_CORNER, 0) != out->g[0] || mag(O9_P11, 0) != out->g[1] || mag(O9_P12, 0) != out->g[1] ||
      mag(O9_P12, 1) != out->g[2] || (n3 && mag(O9_T111, 0) != out->g[1]) || !(out->g[2] < out->g[0]))
    return fail(HCUB_E_ARG, "not a degree-9 (rule9) table: generator magnitudes");
  out->ratio = r->fourth_diff_ratio;
  out->null_center = r->null_center_weight;
  out->null_axis = r->null_axis_weight;
  out->twod = std::ldexp(1.0, d);
  return 0;
}

static int make_fn(const hcub_integrand* f, int d, FnParams* fp) {
  if (!f) return fail(HCUB_E_ARG, "integrand is NULL");
  if (f->kind < HCUB_F1 || f->kind > HCUB_PRODUCT_PEAK) return fail(HCUB_E_ARG, "unknown integrand kind %d", f->kind);
  if (f->d != d) return fail(HCUB_E_DIM, "integrand is for d=%d, rule for d=%d", f->d, d);
  memset(fp, 0, sizeof *fp);
  fp->a = (f->kind == HCUB_F2) ? std::pow(50.0, -2.0) : f->a;
  for (int j = 0; j < HCUB_MAXD; ++j) {
    fp->ctr[j] = (f->kind == HCUB_PRODUCT_PEAK) ? f->center[j] : 0.5;
    fp->coef[j] = (f->kind == HCUB_F6) ? (j + 1) + 4.0 : (double)(j + 1);
    fp->thr[j] = (3.0 + (j + 1)) / 10.0;
  }
  return 0;
}

// ---------------------------------------------------------------------------
// worker

// Caching device allocator for the (large, growing) store buffers: blocks
// are kept per device after release and reused best-fit, so repeated runs
// and the geometric growth of a store do not pay cudaMalloc/cudaFree (which
// synchronise the device) on the steady-state path.  On allocation failure
// the cache is returned to the driver and the request retried once.
#include <map>
#include <mutex>
struct Arena {
  std::mutex mu;
  std::multimap<size_t, void*> cached[64];  // per device: size -> block
  std::map<void*, size_t> sizes[64];
};
static Arena g_arena;

static cudaError_t arena_alloc(int dev, size_t bytes, void** p) {
  bytes = (bytes + 511) & ~(size_t)511;
  if (bytes == 0) bytes = 512;
  {
    std::lock_guard<std::mutex> lk(g_arena.mu);
    auto& c = g_arena.cached[dev];
    auto it = c.lower_bound(bytes);
    if (it != c.end() && it->first <= bytes * 2 + (64 << 20)) {  // avoid hoarding huge blocks for tiny asks
      *p = it->second;
      c.erase(it);
      return cudaSuccess;
    }
  }
  cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    std::lock_guard<std::mutex> lk(g_arena.mu);
    for (auto& kv : g_arena.cached[dev]) { cudaFree(kv.second); g_arena.sizes[dev].erase(kv.second); }
    g_arena.cached[dev].clear();
    e = cudaMalloc(p, bytes);
    if (e != cudaSuccess) { cudaGetLastError(); return e; }
  }
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_arena.mu);
  g_arena.sizes[dev][*p] = bytes;
  return cudaSuccess;
}

static void arena_free(int dev, void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_arena.mu);
  auto it = g_arena.sizes[dev].find(p);
  if (it == g_arena.sizes[dev].end()) { cudaFree(p); return; }
  g_arena.cached[dev].emplace(it->second, p);
}

struct hcub_worker {
  int dev = 0, d = 0, fn = 0, sms = 148;
  cudaStream_t st = nullptr;
  RuleC rc{};
  FnParams fp{};
  int64_t K = 0;
  double dom_lo[HCUB_MAXD]{}, dom_hi[HCUB_MAXD]{}, dext[HCUB_MAXD]{}, dvol = 0;
  int64_t n = 0;
  Cols buf[2]{};
  int64_t bcap[2]{};     // rows each SoA buffer holds
  int cur = 0;
  int64_t rows_cap = 0;  // rows of the per-row scratch below
  int64_t max_cap = 0;   // fixed capacity (explicit request) or 0 = grow on demand
  double* vol = nullptr;
  double* aext = nullptr;
  signed char* axis = nullptr;
  signed char* axis2 = nullptr;  // fused-split loop: children's axes while the parents' are read
  int64_t* pidx = nullptr;       // fused-split loop: survivor (parent) indices
  int64_t n_virtual = -1;        // worker mode: pending virtual children (>= 0) of the current store
  // virtual children a take_top removed (the next K1 / k3_expand skip them):
  // S[j] = R[j] - j over the sorted removed indices R, nrm entries
  int64_t* rmS = nullptr;
  int64_t rm_cap = 0;
  int64_t nrm = 0;
  unsigned long long* cand_k = nullptr;  // K4 candidates of the threshold bucket
  long long* cand_i = nullptr;
  int64_t cand_cap = 0;
  bool table = false;            // rule given as an explicit node table (k1_table_eval)
  DevTable tab;
  bool gk = false;               // tensor Gauss-Kronrod rule (k1_gk_partial / finalize)
  GkArgs gka{};
  double* gk_part = nullptr;     // per-chunk partial sums scratch
  int64_t gk_part_len = 0;
  unsigned char* removed = nullptr;
  int64_t* tiles = nullptr;
  int64_t* scratch_i64 = nullptr;  // [2]
  SAcc* acc = nullptr;             // [ACC_N]
  SAcc* kacc = nullptr;            // [2 * K1_SHARDS] fused-K2 shards
  int64_t eval_rows = 0;           // rows covered by the last K1 over the store
  bool pending = false;            // evaluate_begin issued, evaluate_end not yet
  DevStatus* dst = nullptr;
  DevStatus* hst = nullptr;  // pinned mirror
  double* dI = nullptr;      // device scalar: global integral for classify
  unsigned int* hist = nullptr;
  unsigned long long* ck = nullptr;
  long long* ci = nullptr;
  int64_t take_cap = 0;
  double* stage = nullptr;  // row staging (append / take)
  int64_t stage_rows = 0;
  bool evaluated = false;
  // classify could not grow the spare buffer for the split (capacity): the
  // store still holds the evaluated parents, the carry already holds the
  // finalized rows, and acc[ACC_HALF_*] the exact sums of the survivors'
  // provisional children halves.  A settle must then count carry + halves
  // (+ rows appended afterwards), as the reference does after its split.
  bool settle_halves = false;
  int64_t halves_rows = 0;
  // timing
  bool rule9 = false;  // degree-9 family in generator form (k1_gm9_eval)
  Rule9C r9{};
  cudaEvent_t ev[10]{};
  // one-sync protocol: evaluate_end_async left its K1/K2 timings to collect,
  // a speculative classify is waiting for commit / discard
  bool timings_pending = false, pending_tail = false, spec = false;
  double k1_ms = 0, k2_ms = 0, k3_ms = 0;
  int64_t k1_launches = 0, launches = 0;
  int64_t cap() const { return bcap[cur]; }
};

#define AK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      return fail(e_ == cudaErrorMemoryAllocation ? HCUB_E_CAPACITY : HCUB_E_CUDA, "%s: %s", #call, \
                  cudaGetErrorString(e_));                                                        \
  } while (0)

static void free_buffer(hcub_worker* w, int b) {
  arena_free(w->dev, w->buf[b].lo); arena_free(w->dev, w->buf[b].hi);
  arena_free(w->dev, w->buf[b].I); arena_free(w->dev, w->buf[b].E);
  w->buf[b] = Cols{};
  w->bcap[b] = 0;
}

// (re)allocate buffer b for `rows` rows; contents are not preserved
static int alloc_buffer(hcub_worker* w, int b, int64_t rows) {
  CK(cudaStreamSynchronize(w->st));  // previous users of the block are done
  free_buffer(w, b);
  const size_t r = (size_t)rows, d = (size_t)w->d;
  AK(arena_alloc(w->dev, r * d * 8, (void**)&w->buf[b].lo));
  AK(arena_alloc(w->dev, r * d * 8, (void**)&w->buf[b].hi));
  AK(arena_alloc(w->dev, r * 8, (void**)&w->buf[b].I));
  AK(arena_alloc(w->dev, r * 8, (void**)&w->buf[b].E));
  w->bcap[b] = rows;
  return 0;
}

// per-row scratch.  Every per-row column K1 writes and K3 reads (volume,
// split-axis extent, split axes, survivor indices) keeps its contents: the
// overlapped distributed order (evaluate_begin -> append arrivals ->
// evaluate_end) and the fused-split loop grow it between the K1 that wrote
// the first rows and the classify that reads them.  Only the flag/tile
// scratch is dead across calls.
static int ensure_rows_to(hcub_worker* w, int64_t r) {
  CK(cudaStreamSynchronize(w->st));
  const int64_t old = w->rows_cap;
  // new blocks first: a failed allocation leaves the worker's columns intact
  unsigned char* removed = nullptr;
  int64_t* tiles = nullptr;
  AK(arena_alloc(w->dev, r, (void**)&removed));
  {
    const cudaError_t e = arena_alloc(w->dev, (r / TILE + 2) * 8, (void**)&tiles);
    if (e != cudaSuccess) {
      arena_free(w->dev, removed);
      return fail(e == cudaErrorMemoryAllocation ? HCUB_E_CAPACITY : HCUB_E_CUDA, "per-row scratch: %s",
                  cudaGetErrorString(e));
    }
  }
  // one column at a time (new block, copy, free the old one): the transient
  // peak is one column, and a failure part-way leaves every column holding at
  // least its old rows (rows_cap is only raised at the end)
  void** cols[5] = {(void**)&w->vol, (void**)&w->aext, (void**)&w->axis, (void**)&w->axis2, (void**)&w->pidx};
  const size_t elem[5] = {8, 8, 1, 1, 8};
  for (int i = 0; i < 5; ++i) {
    void* np = nullptr;
    const cudaError_t e = arena_alloc(w->dev, (size_t)r * elem[i], &np);
    if (e != cudaSuccess) {
      arena_free(w->dev, removed);
      arena_free(w->dev, tiles);
      return fail(e == cudaErrorMemoryAllocation ? HCUB_E_CAPACITY : HCUB_E_CUDA, "per-row scratch: %s",
                  cudaGetErrorString(e));
    }
    if (*cols[i] && old > 0) CK(cudaMemcpyAsync(np, *cols[i], (size_t)old * elem[i], cudaMemcpyDeviceToDevice, w->st));
    CK(cudaStreamSynchronize(w->st));
    arena_free(w->dev, *cols[i]);
    *cols[i] = np;
  }
  arena_free(w->dev, w->removed);
  arena_free(w->dev, w->tiles);
  w->removed = removed;
  w->tiles = tiles;
  w->rows_cap = r;
  return 0;
}

static int ensure_rows(hcub_worker* w, int64_t rows) {
  if (rows <= w->rows_cap) return 0;
  // 1.5x geometric growth; near the end of HBM settle for exactly `rows`
  const int64_t r = std::max<int64_t>(rows, w->rows_cap + w->rows_cap / 2);
  const int rc = ensure_rows_to(w, r);
  if (rc == HCUB_E_CAPACITY && r > rows) return ensure_rows_to(w, rows);
  return rc;
}

static int64_t grow_target(hcub_worker* w, int64_t need, int64_t have) {
  int64_t t = std::max<int64_t>(need, have + have / 2);  // 1.5x geometric growth
  t = std::max<int64_t>(t, 1 << 16);
  if (w->max_cap > 0) t = std::min(t, w->max_cap);
  return (t + 63) & ~(int64_t)63;  // even leading dimension: children are written as double2
}

// the spare buffer must hold `need` rows (contents dead)
static int ensure_next(hcub_worker* w, int64_t need) {
  const int nb = w->cur ^ 1;
  // the capacity check comes first: a pooled shell may hold larger buffers
  if (w->max_cap > 0 && need > w->max_cap)
    return fail(HCUB_E_CAPACITY, "%lld rows exceed the fixed store capacity %lld", (long long)need, (long long)w->max_cap);
  if (need <= w->bcap[nb]) return 0;
  return alloc_buffer(w, nb, grow_target(w, need, w->bcap[nb]));
}

// the current buffer must hold `need` rows, preserving its n rows
static int ensure_cur(hcub_worker* w, int64_t need) {
  if (w->max_cap > 0 && need > w->max_cap)
    return fail(HCUB_E_CAPACITY, "%lld rows exceed the fixed store capacity %lld", (long long)need, (long long)w->max_cap);
  if (need <= w->cap()) return 0;
  const int nb = w->cur ^ 1;
  if (w->bcap[nb] < need) TRY(alloc_buffer(w, nb, grow_target(w, need, w->cap())));
  if (w->n > 0) {
    Cols& s = w->buf[w->cur];
    Cols& t = w->buf[nb];
    const size_t row = (size_t)w->n * 8;
    CK(cudaMemcpy2DAsync(t.lo, w->bcap[nb] * 8, s.lo, w->cap() * 8, row, w->d, cudaMemcpyDeviceToDevice, w->st));
    CK(cudaMemcpy2DAsync(t.hi, w->bcap[nb] * 8, s.hi, w->cap() * 8, row, w->d, cudaMemcpyDeviceToDevice, w->st));
    CK(cudaMemcpyAsync(t.I, s.I, row, cudaMemcpyDeviceToDevice, w->st));
    CK(cudaMemcpyAsync(t.E, s.E, row, cudaMemcpyDeviceToDevice, w->st));
  }
  w->cur = nb;
  return 0;
}

// small per-worker resources (stream, events, status, accumulators)
static int shell_alloc(hcub_worker* w) {
  CK(cudaStreamCreateWithFlags(&w->st, cudaStreamNonBlocking));
  CK(cudaMalloc(&w->scratch_i64, 2 * sizeof(int64_t)));
  CK(cudaMalloc(&w->acc, ACC_N * sizeof(SAcc)));
  CK(cudaMalloc(&w->kacc, 2 * K1_SHARDS * sizeof(SAcc)));
  CK(cudaMalloc(&w->dst, sizeof(DevStatus)));
  CK(cudaMallocHost(&w->hst, sizeof(DevStatus)));
  CK(cudaMalloc(&w->dI, sizeof(double)));
  CK(cudaMalloc(&w->hist, 4096 * sizeof(unsigned int)));  // k4v_hist12 bins (k4_hist uses the first 256)
  CK(cudaMemsetAsync(w->hist, 0, 4096 * sizeof(unsigned int), w->st));
  for (auto& e : w->ev) CK(cudaEventCreate(&e));
  return 0;
}

static void worker_free(hcub_worker* w) {
  if (!w) return;
  cudaSetDevice(w->dev);
  if (w->st) cudaStreamSynchronize(w->st);
  w->tab.release();
  free_buffer(w, 0);
  free_buffer(w, 1);
  arena_free(w->dev, w->vol); arena_free(w->dev, w->axis); arena_free(w->dev, w->removed); arena_free(w->dev, w->tiles);
  arena_free(w->dev, w->aext); arena_free(w->dev, w->axis2); arena_free(w->dev, w->pidx);
  arena_free(w->dev, w->gk_part);
  cudaFree(w->scratch_i64);
  cudaFree(w->acc); cudaFree(w->kacc); cudaFree(w->dst); cudaFreeHost(w->hst); cudaFree(w->dI); cudaFree(w->hist);
  arena_free(w->dev, w->ck); arena_free(w->dev, w->ci); arena_free(w->dev, w->stage);
  arena_free(w->dev, w->rmS); arena_free(w->dev, w->cand_k); arena_free(w->dev, w->cand_i);
  for (auto& e : w->ev) if (e) cudaEventDestroy(e);
  if (w->st) cudaStreamDestroy(w->st);
  delete w;
}

// Idle worker shells per device: a run re-uses stream, events, pinned status
// and its grown store buffers instead of re-creating them (these host-side
// CUDA calls cost milliseconds per run otherwise).
static std::mutex g_pool_mu;
static std::vector<hcub_worker*> g_pool[64];
static int g_sms[64];

static hcub_worker* pool_take(int dev, int d) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  auto& p = g_pool[dev & 63];
  for (size_t i = 0; i < p.size(); ++i)
    if (p[i]->d == d) { hcub_worker* w = p[i]; p.erase(p.begin() + i); return w; }
  if (!p.empty()) {  // other dimension: keep the shell, drop its d-sized buffers
    hcub_worker* w = p.back();
    p.pop_back();
    free_buffer(w, 0);
    free_buffer(w, 1);
    arena_free(w->dev, w->stage);  // (2d+2) doubles per row
    w->stage = nullptr;
    w->stage_rows = 0;
    return w;
  }
  return nullptr;
}

static void worker_release(hcub_worker* w) {
  if (!w) return;
  cudaSetDevice(w->dev);
  cudaStreamSynchronize(w->st);
  w->tab.release();
  w->table = false;
  w->gk = false;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  auto& p = g_pool[w->dev & 63];
  if (p.size() < 8) p.push_back(w);
  else worker_free(w);
}

static int device_sms(int dev) {
  if (!g_sms[dev & 63]) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    g_sms[dev & 63] = v;
  }
  return g_sms[dev & 63];
}

static int worker_init(int device, const hcub_rule* rule, const hcub_integrand* f, const double* dom_lo,
                       const double* dom_hi, int64_t capacity, hcub_worker** out) {
  if (!out) return fail(HCUB_E_ARG, "out is NULL");
  *out = nullptr;
  RuleC rc;
  TRY(make_rule(rule, &rc));
  FnParams fp;
  TRY(make_fn(f, rule->d, &fp));
  if (!dom_lo || !dom_hi) return fail(HCUB_E_ARG, "domain is NULL");
  double dext[HCUB_MAXD], vol = 1.0;
  for (int j = 0; j < rule->d; ++j) {
    dext[j] = dom_hi[j] - dom_lo[j];
    if (!(dext[j] > 0) || !std::isfinite(dext[j])) return fail(HCUB_E_ARG, "every axis needs lo < hi");
    vol = (j == 0) ? dext[0] : vol * dext[j];  // float(np.prod(domain.hi - domain.lo))
  }
  CK(cudaSetDevice(device));
  hcub_worker* w = pool_take(device, rule->d);
  if (!w) {
    w = new hcub_worker();
    w->dev = device;
    int rc2 = shell_alloc(w);
    if (rc2) { std::string m = g_err; worker_free(w); g_err = m; return rc2; }
  }
  w->d = rule->d;
  w->fn = f->kind;
  w->rc = rc;
  w->fp = fp;
  w->K = (1ll << w->d) + 2ll * w->d * w->d + 2ll * w->d + 1;
  w->table = rule->kind == 1;
  w->gk = rule->kind == 2;
  w->rule9 = rule->kind == 3;
  if (w->rule9) {  // generator kernel for one region per lane, the node table for lane groups (small stores)
    w->K = rule->K;
    int r9 = make_rule9(rule, &w->r9);
    if (!r9) r9 = upload_table(rule, device, w->st, &w->tab);
    if (r9) { std::string m = g_err; worker_free(w); g_err = m; return r9; }
  }
  if (w->gk) {
    w->gka = make_gk(rule->d);
    w->K = w->gka.K;
  }
  if (w->table) {
    w->K = rule->K;
    const int rt = upload_table(rule, device, w->st, &w->tab);
    if (rt) { std::string m = g_err; worker_free(w); g_err = m; return rt; }
  }
  for (int j = 0; j < w->d; ++j) { w->dom_lo[j] = dom_lo[j]; w->dom_hi[j] = dom_hi[j]; w->dext[j] = dext[j]; }
  w->dvol = vol;
  w->sms = device_sms(device);
  w->n = 0;
  w->n_virtual = -1;
  w->nrm = 0;
  w->evaluated = false;
  w->pending = false;
  w->settle_halves = false;
  w->eval_rows = 0;
  w->k1_ms = w->k2_ms = w->k3_ms = 0;
  w->k1_launches = w->launches = 0;
  if (capacity > 0) capacity = (capacity + 63) & ~(int64_t)63;
  w->max_cap = capacity > 0 ? capacity : 0;
  int rc3 = 0;
  if (cudaMemsetAsync(w->dst, 0, sizeof(DevStatus), w->st) != cudaSuccess) rc3 = fail(HCUB_E_CUDA, "memset failed");
  const int64_t first = capacity > 0 ? capacity : (1 << 16);
  if (!rc3 && w->cap() < first) {
    if (w->bcap[w->cur ^ 1] >= first) w->cur ^= 1;
    else rc3 = alloc_buffer(w, w->cur, first);
  }
  if (!rc3 && capacity > 0 && w->bcap[w->cur ^ 1] < capacity) rc3 = alloc_buffer(w, w->cur ^ 1, capacity);
  if (!rc3) rc3 = ensure_rows(w, first);
  if (rc3) { std::string m = g_err; worker_free(w); g_err = m; return rc3; }
  *out = w;
  return 0;
}

static int ensure_stage(hcub_worker* w, int64_t rows) {
  if (rows <= w->stage_rows) return 0;
  CK(cudaStreamSynchronize(w->st));
  arena_free(w->dev, w->stage);
  w->stage = nullptr;
  const int64_t r = std::max<int64_t>(rows, 1024);
  AK(arena_alloc(w->dev, (size_t)r * (2 * w->d + 2) * sizeof(double), (void**)&w->stage));
  w->stage_rows = r;
  return 0;
}

static int ensure_take(hcub_worker* w, int64_t m) {
  if (m <= w->take_cap) return 0;
  CK(cudaStreamSynchronize(w->st));
  arena_free(w->dev, w->ck); arena_free(w->dev, w->ci);
  w->ck = nullptr; w->ci = nullptr;
  const int64_t r = std::max<int64_t>(m, 1024);
  AK(arena_alloc(w->dev, r * sizeof(unsigned long long), (void**)&w->ck));
  AK(arena_alloc(w->dev, r * sizeof(long long), (void**)&w->ci));
  w->take_cap = r;
  return 0;
}

static unsigned grid_for(int64_t threads, int block) { return (unsigned)((threads + block - 1) / block); }

// K1 launch shape: one thread per (region, lane), 128-thread blocks.
// (Tried: two sibling regions per lane so the second child's parent loads
// hit L1 - 6 % slower at d = 8, neutral at d = 5.)
static void k1_geometry(const K1Args& a, int64_t threads, int sms, unsigned* grid, unsigned* block) {
  (void)a;
  (void)sms;
  *block = K1_BLOCK;
  *grid = grid_for(threads, K1_BLOCK);
}

// K1 dispatch: Genz-Malik generator kernel or explicit-table kernel
static const int64_t GK_SCRATCH = 16 << 20;  // doubles of chunk partials per launch (128 MB)

static cudaError_t launch_gk(int fn, int d, const K1Args& a, const GkArgs& g, const FnParams& fp, double* part,
                             int64_t part_len, cudaStream_t st) {
  const int64_t per = (int64_t)g.chunks * (d + 3);
  const int64_t batch = std::max<int64_t>(1, part_len / per);
  for (int64_t r0 = 0; r0 < a.n; r0 += batch) {
    const cudaError_t e = K1GK_LAUNCH[fn](d, &a, &g, &fp, r0, std::min(batch, a.n - r0), part, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

#ifndef K9_MIN_ROWS_PER_SM
#define K9_MIN_ROWS_PER_SM 128  // rows per SM from which the degree-9 generator kernel takes over (measured: 128 < 512 < 2048)
#endif

static cudaError_t launch_k1(hcub_worker* w, const K1Args& a, int64_t threads) {
  if (w->gk) {
    const int64_t need = std::min<int64_t>(GK_SCRATCH, std::max<int64_t>(a.n, 1) * w->gka.chunks * (w->d + 3));
    if (w->gk_part_len < need) {
      cudaStreamSynchronize(w->st);
      arena_free(w->dev, w->gk_part);
      w->gk_part = nullptr;
      w->gk_part_len = 0;
      const cudaError_t e = arena_alloc(w->dev, need * 8, (void**)&w->gk_part);
      if (e != cudaSuccess) return e;
      w->gk_part_len = need;
    }
    return launch_gk(w->fn, w->d, a, w->gka, w->fp, w->gk_part, w->gk_part_len, w->st);
  }
  if (w->rule9) {
    // the generator kernel (one region per lane) once it has ~4 blocks per SM;
    // below that the node table with lane groups keeps the machine busy
    if (a.n >= (int64_t)w->sms * K9_MIN_ROWS_PER_SM || a.log2g == 0) {
      K1Args b = a;
      b.log2g = 0;
      return K9_LAUNCH[w->fn](w->d, &b, &w->r9, &w->fp, w->st);
    }
    return K1T_LAUNCH[w->fn](w->d, &a, &w->tab.args, &w->fp, grid_for(threads, K1_BLOCK), K1_BLOCK, w->st);
  }
  if (w->table) return K1T_LAUNCH[w->fn](w->d, &a, &w->tab.args, &w->fp, grid_for(threads, K1_BLOCK), K1_BLOCK, w->st);
  unsigned grid, block;
  k1_geometry(a, threads, w->sms, &grid, &block);
  return K1_LAUNCH[w->fn](w->d, &a, &w->rc, &w->fp, grid, block, w->st);
}

// Genz-Malik generator kernels accumulate the exact column sums themselves
// (fused K2); the table and Gauss-Kronrod kernels leave them to k2_reduce.
static bool k1_fused_sums(const hcub_worker* w) { return !w->gk; }

// Exact column sums of the n evaluated rows -> status.I/E = fsum([carry,
// *column]): merge of K1's per-SM shards (fused), or k2_reduce + round.
static int launch_finish_sums(hcub_worker* w) {
  if (w->n > 0 && k1_fused_sums(w)) {
    k2_merge_round<<<1, K2M_THREADS, 0, w->st>>>(w->kacc, K1_SHARDS, w->acc, w->dst);
  } else {
    if (w->n > 0) {
      Cols& c = w->buf[w->cur];
      const unsigned g2 = (unsigned)std::max<int64_t>(1, std::min<int64_t>(grid_for(w->n, 512 * 8), (int64_t)w->sms * 8));
      k2_reduce<<<g2, 256, 0, w->st>>>(c.I, c.E, w->n, w->acc);
      CK(cudaGetLastError());
      w->launches += 1;
    }
    k2_round<<<1, 64, 0, w->st>>>(w->acc, w->dst);
  }
  CK(cudaGetLastError());
  CK(cudaEventRecord(w->ev[2], w->st));
  w->launches += 1;
  return 0;
}

// K1 over the current store, then (finish) K2 and the rounding kernel:
// status.I/E = fsum([carry, *column]).  Asynchronous.  With finish = false
// the sums stay in the accumulators so rows appended later can be added by
// a tail K1 before launch_finish_sums (hcub_worker_evaluate_begin/_end).
static int launch_evaluate(hcub_worker* w, bool finish = true) {
  Cols& c = w->buf[w->cur];
  w->settle_halves = false;
  CK(cudaMemsetAsync(&w->acc[ACC_I], 0, 2 * sizeof(SAcc), w->st));
  const bool fused = k1_fused_sums(w);
  if (fused) CK(cudaMemsetAsync(w->kacc, 0, 2 * K1_SHARDS * sizeof(SAcc), w->st));
  w->eval_rows = w->n;
  if (w->n > 0) {
    TRY(ensure_rows(w, w->n));
    K1Args a{};
    a.lo = c.lo; a.hi = c.hi; a.ld = w->cap(); a.n = w->n;
    a.integral = c.I; a.error = c.E; a.vol = w->vol; a.axis = w->axis; a.aext = w->aext;
    a.log2g = pick_log2g(w->n, w->sms);
    if (fused) a.kacc = w->kacc;
    const int64_t threads = w->n << a.log2g;
    CK(cudaEventRecord(w->ev[0], w->st));
    CK(launch_k1(w, a, threads));
    CK(cudaEventRecord(w->ev[1], w->st));
    w->k1_launches += 1;
    w->launches += 1;
  } else {
    CK(cudaEventRecord(w->ev[0], w->st));
    CK(cudaEventRecord(w->ev[1], w->st));
  }
  return finish ? launch_finish_sums(w) : 0;
}

// Fused split: K1 over the 2*n_split children of the current store's
// survivors (w->pidx), materialising them into the spare buffer, then K2.
static int launch_evaluate_children(hcub_worker* w, int64_t n_children, bool finish = true) {
  w->settle_halves = false;
  TRY(ensure_next(w, n_children));
  TRY(ensure_rows(w, std::max<int64_t>(n_children, w->n)));
  const int nb = w->cur ^ 1;
  Cols& par = w->buf[w->cur];
  Cols& kid = w->buf[nb];
  const bool fused = k1_fused_sums(w);
  CK(cudaMemsetAsync(&w->acc[ACC_I], 0, 2 * sizeof(SAcc), w->st));
  if (fused) CK(cudaMemsetAsync(w->kacc, 0, 2 * K1_SHARDS * sizeof(SAcc), w->st));
  CK(cudaEventRecord(w->ev[0], w->st));
  if (n_children > 0) {
    K1Args a{};
    a.lo = kid.lo; a.hi = kid.hi; a.ld = w->bcap[nb]; a.n = n_children;
    a.integral = kid.I; a.error = kid.E; a.vol = w->vol; a.axis = w->axis2; a.aext = w->aext;
    a.pidx = w->pidx; a.plo = par.lo; a.phi = par.hi; a.pld = w->cap(); a.pax = w->axis;
    a.rmS = w->rmS; a.nrm = w->nrm;
    a.clo = kid.lo; a.chi = kid.hi;
    a.log2g = pick_log2g(n_children, w->sms);
    if (fused) a.kacc = w->kacc;
    CK(launch_k1(w, a, n_children << a.log2g));
  }
  CK(cudaEventRecord(w->ev[1], w->st));
  if (n_children > 0) {
    w->k1_launches += 1;
    w->launches += 1;
  }
  std::swap(w->axis, w->axis2);
  w->nrm = 0;
  w->cur = nb;
  w->n = n_children;
  w->eval_rows = n_children;
  w->evaluated = true;
  return finish ? launch_finish_sums(w) : 0;
}

// worker mode: turn pending virtual children into real rows
static int materialize(hcub_worker* w) {
  if (w->n_virtual < 0) return 0;
  const int64_t nc = w->n_virtual - w->nrm;
  w->n_virtual = -1;
  TRY(ensure_next(w, nc));
  const int nb = w->cur ^ 1;
  if (nc > 0) {
    const unsigned g = (unsigned)std::min<int64_t>(grid_for(nc, 256), (int64_t)w->sms * 16);
    k3_expand<<<g, 256, 0, w->st>>>(w->pidx, nc, w->buf[w->cur], w->cap(), w->axis, w->buf[nb], w->bcap[nb], w->d,
                                    w->rmS, w->nrm);
    CK(cudaGetLastError());
    w->launches += 1;
  }
  w->nrm = 0;
  w->cur = nb;
  w->n = nc;
  w->evaluated = false;
  return 0;
}

static ClassifyArgs classify_args(hcub_worker* w, const double* gI, const hcub_driver_cfg* cfg) {
  ClassifyArgs a{};
  Cols& c = w->buf[w->cur];
  a.cur = c; a.cap = w->cap(); a.vol = w->vol; a.axis = w->axis; a.aext = w->aext; a.n = w->n; a.gI = gI;
  a.tau = cfg->tau_rel; a.floor = cfg->abs_floor; a.safety = cfg->safety; a.dvol = w->dvol;
  {  // exact reciprocal of a power-of-two domain volume (k3_vfrac)
    int e = 0;
    const double m = std::frexp(w->dvol, &e);
    a.inv_dvol = (m == 0.5 && e - 1 > -1022 && e - 1 < 1022) ? std::ldexp(1.0, 1 - e) : 0.0;
  }
  const double g = cfg->min_width_ulp_factor * 2.220446049250313e-16;  // (factor * eps) * extent
  for (int j = 0; j < w->d; ++j) a.guard[j] = g * w->dext[j];
  a.d = w->d;
  a.tile_counts = w->tiles;
  a.acc = w->acc;
  a.st = w->dst;
  return a;
}

// K3a: classification counts + finalized carry + tile scan.  Asynchronous.
static int launch_classify(hcub_worker* w, const double* gI, const hcub_driver_cfg* cfg, bool compact = false) {
  CK(cudaMemsetAsync(&w->acc[ACC_FIN_I], 0, 2 * sizeof(SAcc), w->st));
  CK(cudaMemsetAsync(&w->dst->n_split, 0, 3 * sizeof(long long), w->st));
  const int64_t tiles = (w->n + TILE - 1) / TILE;
  if (tiles > 0) {
    ClassifyArgs a = classify_args(w, gI, cfg);
    if (compact) a.flags = w->removed;
    CK(cudaMemsetAsync(w->tiles, 0, tiles * sizeof(int64_t), w->st));
    k3_classify<<<(unsigned)std::min<int64_t>(tiles, (int64_t)w->sms * 8), TILE_THREADS, 0, w->st>>>(a);
    CK(cudaGetLastError());
    // tile scan + finalized-sum rounding in one single-block launch
    k_scan_tiles<<<1, 1024, 0, w->st>>>(w->tiles, tiles, w->scratch_i64, w->acc, w->dst, gI, cfg->tau_rel,
                                        cfg->abs_floor);
    CK(cudaGetLastError());
    w->launches += 2;
    if (compact) {  // survivors -> parent list of the next (virtual) store
      k3_compact<<<(unsigned)tiles, TILE_THREADS, 0, w->st>>>(w->removed, w->n, w->tiles, w->pidx);
      CK(cudaGetLastError());
      w->launches += 1;
    }
  } else {
    k3_round<<<1, 64, 0, w->st>>>(w->acc, w->dst, gI, cfg->tau_rel, cfg->abs_floor);
    CK(cudaGetLastError());
    w->launches += 1;
  }
  CK(cudaEventRecord(w->ev[3], w->st));
  return 0;
}

static int launch_split(hcub_worker* w, const double* gI, const hcub_driver_cfg* cfg, int64_t n_split,
                        bool write_estimates = true) {
  TRY(ensure_next(w, 2 * n_split));
  const int64_t tiles = (w->n + TILE - 1) / TILE;
  const int nb = w->cur ^ 1;
  CK(cudaEventRecord(w->ev[4], w->st));
  if (tiles > 0 && n_split > 0) {
    SplitArgs s{};
    s.c = classify_args(w, gI, cfg);
    s.nxt = w->buf[nb];
    s.cap_next = w->bcap[nb];
    s.tile_offsets = w->tiles;
    s.write_estimates = write_estimates ? 1 : 0;
    k3_split<<<(unsigned)tiles, TILE_THREADS, 0, w->st>>>(s);
    CK(cudaGetLastError());
    w->launches += 1;
  }
  CK(cudaEventRecord(w->ev[5], w->st));
  w->cur = nb;
  w->n = 2 * n_split;
  w->evaluated = false;
  return 0;
}

static void add_timings(hcub_worker* w, bool with_split, bool with_classify) {
  float a = 0, b = 0, c = 0, e = 0;
  cudaEventElapsedTime(&a, w->ev[0], w->ev[1]);
  cudaEventElapsedTime(&b, w->ev[1], w->ev[2]);
  if (with_classify) cudaEventElapsedTime(&c, w->ev[2], w->ev[3]);
  w->k1_ms += a;
  w->k2_ms += b;
  w->k3_ms += c;
  if (with_split) {
    cudaEventElapsedTime(&e, w->ev[4], w->ev[5]);
    w->k3_ms += e;
  }
}

// ---------------------------------------------------------------------------
// C ABI

extern "C" {

int hcub_abi_version(void) { return HCUB_ABI_VERSION; }
const char* hcub_last_error(void) { return g_err.c_str(); }

int hcub_set_k1_lanes(int log2_lanes) {
  if (log2_lanes < -1 || log2_lanes > 5) return fail(HCUB_E_ARG, "log2_lanes must be -1 (auto) or 0..5");
  g_k1_log2g.store(log2_lanes, std::memory_order_relaxed);
  return 0;
}

int hcub_device_count(int* out) {
  if (!out) return fail(HCUB_E_ARG, "out is NULL");
  CK(cudaGetDeviceCount(out));
  return 0;
}

int hcub_worker_create(int device, const hcub_rule* rule, const hcub_integrand* f, const double* dom_lo,
                       const double* dom_hi, int64_t capacity, hcub_worker** out) {
  return worker_init(device, rule, f, dom_lo, dom_hi, capacity, out);
}

void hcub_worker_destroy(hcub_worker* w) { worker_release(w); }

int hcub_worker_size(hcub_worker* w, int64_t* n, int64_t* capacity) {
  if (!w) return fail(HCUB_E_ARG, "worker is NULL");
  if (n) *n = w->n_virtual >= 0 ? w->n_virtual - w->nrm : w->n;
  if (capacity) *capacity = w->max_cap > 0 ? w->max_cap : w->cap();
  return 0;
}

int hcub_worker_append(hcub_worker* w, const double* lo, const double* hi, const double* integral,
                       const double* error, int64_t m, int on_device) {
  if (!w || m < 0) return fail(HCUB_E_ARG, "bad arguments");
  if (m == 0) return 0;
  if (!lo || !hi) return fail(HCUB_E_ARG, "lo/hi are NULL");
  CK(cudaSetDevice(w->dev));
  TRY(materialize(w));
  TRY(ensure_cur(w, w->n + m));
  const double *dlo = lo, *dhi = hi, *dI = integral, *dE = error;
  if (!on_device) {
    // validate lo < hi (ref regions.py:204-205) on the host copy we were given
    for (int64_t i = 0; i < m * w->d; ++i)
      if (!(lo[i] < hi[i])) return fail(HCUB_E_ARG, "every appended region needs lo < hi on all axes");
    TRY(ensure_stage(w, m));
    const size_t rb = (size_t)m * w->d * sizeof(double);
    double* s = w->stage;
    CK(cudaMemcpyAsync(s, lo, rb, cudaMemcpyHostToDevice, w->st));
    CK(cudaMemcpyAsync(s + m * w->d, hi, rb, cudaMemcpyHostToDevice, w->st));
    dlo = s;
    dhi = s + m * w->d;
    dI = dE = nullptr;
    if (integral) { CK(cudaMemcpyAsync(s + 2 * m * w->d, integral, m * 8, cudaMemcpyHostToDevice, w->st)); dI = s + 2 * m * w->d; }
    if (error) { CK(cudaMemcpyAsync(s + 2 * m * w->d + m, error, m * 8, cudaMemcpyHostToDevice, w->st)); dE = s + 2 * m * w->d + m; }
  }
  const unsigned g = (unsigned)std::min<int64_t>(grid_for(m, 256), 4096);
  long long* bad = on_device ? &w->dst->pad[0] : nullptr;  // host rows were checked above
  if (bad) CK(cudaMemsetAsync(bad, 0, sizeof(long long), w->st));
  k5_append_rows<<<g, 256, 0, w->st>>>(dlo, dhi, m, w->d, w->buf[w->cur], w->cap(), w->n, dI, dE, bad);
  CK(cudaGetLastError());
  w->launches += 1;
  long long nbad = 0;
  if (bad) CK(cudaMemcpyAsync(&nbad, bad, sizeof nbad, cudaMemcpyDeviceToHost, w->st));
  CK(cudaStreamSynchronize(w->st));
  // rows written past n are dead until n moves: a rejected append leaves the store as it was
  if (nbad) return fail(HCUB_E_ARG, "every appended region needs lo < hi on all axes (%lld device rows violate it)", nbad);
  w->n += m;
  w->evaluated = false;
  return 0;
}

int hcub_worker_read(hcub_worker* w, double* lo, double* hi, double* integral, double* error, int64_t* axis) {
  if (w && w->pending) return fail(HCUB_E_ARG, "an evaluation is pending (call hcub_worker_evaluate_end)");
  if (!w) return fail(HCUB_E_ARG, "worker is NULL");
  CK(cudaSetDevice(w->dev));
  TRY(materialize(w));
  const int64_t n = w->n;
  if (n == 0) return 0;
  Cols& c = w->buf[w->cur];
  if (lo || hi) {
    TRY(ensure_stage(w, n));
    const unsigned g = (unsigned)std::min<int64_t>(grid_for(n, 256), 4096);
    k_read_rows<<<g, 256, 0, w->st>>>(c, w->cap(), n, w->d, w->stage, w->stage + n * w->d);
    CK(cudaGetLastError());
    if (lo) CK(cudaMemcpyAsync(lo, w->stage, n * w->d * 8, cudaMemcpyDeviceToHost, w->st));
    if (hi) CK(cudaMemcpyAsync(hi, w->stage + n * w->d, n * w->d * 8, cudaMemcpyDeviceToHost, w->st));
  }
  if (integral) CK(cudaMemcpyAsync(integral, c.I, n * 8, cudaMemcpyDeviceToHost, w->st));
  if (error) CK(cudaMemcpyAsync(error, c.E, n * 8, cudaMemcpyDeviceToHost, w->st));
  std::vector<signed char> ax;
  if (axis) {
    ax.resize(n);
    if (w->evaluated) CK(cudaMemcpyAsync(ax.data(), w->axis, n, cudaMemcpyDeviceToHost, w->st));
    else std::fill(ax.begin(), ax.end(), (signed char)-1);
  }
  CK(cudaStreamSynchronize(w->st));
  if (axis) for (int64_t i = 0; i < n; ++i) axis[i] = ax[i];
  return 0;
}

int hcub_worker_set_carry(hcub_worker* w, double fi, double fe) {
  if (!w) return fail(HCUB_E_ARG, "worker is NULL");
  CK(cudaSetDevice(w->dev));
  double v[2] = {fi, fe};
  CK(cudaMemcpyAsync(&w->dst->fin_I, v, 2 * sizeof(double), cudaMemcpyHostToDevice, w->st));
  CK(cudaStreamSynchronize(w->st));
  return 0;
}

int hcub_worker_get_carry(hcub_worker* w, double* fi, double* fe) {
  if (!w) return fail(HCUB_E_ARG, "worker is NULL");
  CK(cudaSetDevice(w->dev));
  double v[2];
  CK(cudaMemcpyAsync(v, &w->dst->fin_I, 2 * sizeof(double), cudaMemcpyDeviceToHost, w->st));
  CK(cudaStreamSynchronize(w->st));
  if (fi) *fi = v[0];
  if (fe) *fe = v[1];
  return 0;
}

int hcub_worker_evaluate(hcub_worker* w, double* pi, double* pe, int64_t* evals) {
  if (w && w->pending) return fail(HCUB_E_ARG, "an evaluation is pending (call hcub_worker_evaluate_end)");
  if (!w) return fail(HCUB_E_ARG, "worker is NULL");
  CK(cudaSetDevice(w->dev));
  if (w->n_virtual >= 0) {  // fused split: K1 materialises the children while evaluating them
    const int64_t nc = w->n_virtual - w->nrm;
    w->n_virtual = -1;
    TRY(launch_evaluate_children(w, nc));
  } else {
    TRY(launch_evaluate(w));
  }
  CK(cudaMemcpyAsync(w->hst, w->dst, sizeof(DevStatus), cudaMemcpyDeviceToHost, w->st));
  CK(cudaStreamSynchronize(w->st));
  float a = 0, b = 0;
  cudaEventElapsedTime(&a, w->ev[0], w->ev[1]);
  cudaEventElapsedTime(&b, w->ev[1], w->ev[2]);
  w->k1_ms += a;
  w->k2_ms += b;
  w->evaluated = true;
  if (pi) *pi = w->hst->I;
  if (pe) *pe = w->hst->E;
  if (evals) *evals = w->n * w->K;
  return 0;
}

int hcub_worker_evaluate_begin(hcub_worker* w) {
  if (!w) return fail(HCUB_E_ARG, "worker is NULL");
  if (w->pending) return fail(HCUB_E_ARG, "evaluate_begin already pending");
  CK(cudaSetDevice(w->dev));
  if (w->n_virtual >= 0) {
    const int64_t nc = w->n_virtual - w->nrm;
    w->n_virtual = -1;
    TRY(launch_evaluate_children(w, nc, /*finish=*/false));
  } else {
    TRY(launch_evaluate(w, /*finish=*/false));
  }
  w->evaluated = false;
  w->pending = true;
  return 0;
}

// the launch half of evaluate_end: tail K1 over rows appended since
// evaluate_begin, then the exact sums (status.I/E on the device)
static int evaluate_end_launch(hcub_worker* w) {
  w->pending = false;
  const int64_t start = w->eval_rows, m = w->n - start;
  w->pending_tail = m > 0;
  if (m > 0) {  // rows appended since evaluate_begin: one more K1 into the same accumulators
    TRY(ensure_rows(w, w->n));
    Cols& c = w->buf[w->cur];
    K1Args a{};
    a.lo = c.lo + start; a.hi = c.hi + start; a.ld = w->cap(); a.n = m;
    a.integral = c.I + start; a.error = c.E + start; a.vol = w->vol + start; a.axis = w->axis + start;
    a.aext = w->aext + start;
    a.log2g = pick_log2g(m, w->sms);
    if (k1_fused_sums(w)) a.kacc = w->kacc;
    CK(cudaEventRecord(w->ev[6], w->st));
    CK(launch_k1(w, a, m << a.log2g));
    CK(cudaEventRecord(w->ev[7], w->st));
    w->k1_launches += 1;
    w->launches += 1;
  }
  w->eval_rows = w->n;
  TRY(launch_finish_sums(w));
  w->evaluated = true;
  w->timings_pending = true;
  return 0;
}

// K1 / K2 times of the last evaluation (its events have completed)
static void collect_eval_timings(hcub_worker* w) {
  if (!w->timings_pending) return;
  float a = 0, b = 0, t = 0;
  cudaEventElapsedTime(&a, w->ev[0], w->ev[1]);
  cudaEventElapsedTime(&b, w->ev[1], w->ev[2]);
  if (w->pending_tail) cudaEventElapsedTime(&t, w->ev[6], w->ev[7]);
  w->k1_ms += a + t;
  w->k2_ms += b - t;
  w->timings_pending = false;
}

int hcub_worker_evaluate_end(hcub_worker* w, double* pi, double* pe, int64_t* evals) {
  if (!w) return fail(HCUB_E_ARG, "worker is NULL");
  if (!w->pending) return fail(HCUB_E_ARG, "evaluate_end without evaluate_begin");
  CK(cudaSetDevice(w->dev));
  TRY(evaluate_end_launch(w));
  CK(cudaMemcpyAsync(w->hst, w->dst, sizeof(DevStatus), cudaMemcpyDeviceToHost, w->st));
  CK(cudaStreamSynchronize(w->st));
  collect_eval_timings(w);
  if (pi) *pi = w->hst->I;
  if (pe) *pe = w->hst->E;
  if (evals) *evals = w->n * w->K;
  return 0;
}

int hcub_worker_evaluate_end_async(hcub_worker* w, int64_t* evals) {
  if (!w) return fail(HCUB_E_ARG, "worker is NULL");
  if (!w->pending) return fail(HCUB_E_ARG, "evaluate_end without evaluate_begin");
  CK(cudaSetDevice(w->dev));
  TRY(evaluate_end_launch(w));
  if (evals) *evals = w->n * w->K;
  return 0;
}

int hcub_worker_stream(hcub_worker* w, void** stream) {
  if (!w || !stream) return fail(HCUB_E_ARG, "bad arguments");
  *stream = (void*)w->st;
  return 0;
}

int hcub_worker_record_partials(hcub_worker* w, double* dev_dst) {
  if (!w || !dev_dst) return fail(HCUB_E_ARG, "bad arguments");
  if (w->pending) return fail(HCUB_E_ARG, "an evaluation is pending (call hcub_worker_evaluate_end)");
  CK(cudaSetDevice(w->dev));
  CK(cudaMemcpyAsync(dev_dst, &w->dst->I, 2 * sizeof(double), cudaMemcpyDeviceToDevice, w->st));
  return 0;
}

int hcub_worker_reserve(hcub_worker* w, int64_t rows, int32_t* ok) {
  if (!w || rows < 0 || !ok) return fail(HCUB_E_ARG, "bad arguments");
  if (w->pending) return fail(HCUB_E_ARG, "reserve while an evaluation is pending");
  *ok = 0;
  CK(cudaSetDevice(w->dev));
  int rc = ensure_next(w, rows);
  if (!rc) rc = ensure_rows(w, std::max<int64_t>(rows, w->n));  // and the per-row columns of the split
  if (rc && rc != HCUB_E_CAPACITY) return rc;
  *ok = rc == 0;
  return 0;
}

// host half of classify, after the status mirror (w->hst) holds the K3
// results: grow / materialise / keep the children virtual, report
static int classify_finish(hcub_worker* w, const hcub_driver_cfg* cfg, int split, hcub_classify_out* out,
                           cudaEvent_t k3_start) {
  float c = 0;
  cudaEventElapsedTime(&c, k3_start, w->ev[3]);
  w->k3_ms += c;
  const int64_t ns = w->hst->n_split;
  int done = 0;
  int grow = split ? ensure_next(w, 2 * ns) : 0;
  if (grow && grow != HCUB_E_CAPACITY) return grow;
  const bool materialise = split && !grow;
  if (!materialise && w->n > 0) {  // children stay virtual: their provisional sums for a settle
    CK(cudaMemsetAsync(&w->acc[ACC_HALF_I], 0, 2 * sizeof(SAcc), w->st));
    ClassifyArgs ca = classify_args(w, w->dI, cfg);
    k3_child_sums<<<(unsigned)std::min<int64_t>(grid_for(w->n, TILE_THREADS), (int64_t)w->sms * 8), TILE_THREADS, 0, w->st>>>(ca);
    k3_round_halves<<<1, 64, 0, w->st>>>(w->acc, w->dst);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&w->hst->half_I, &w->dst->half_I, 2 * sizeof(double), cudaMemcpyDeviceToHost, w->st));
    CK(cudaStreamSynchronize(w->st));
    if (split) {  // the split was wanted but could not be stored
      w->settle_halves = true;
      w->halves_rows = w->n;
    }
  } else {
    w->hst->half_I = w->hst->half_E = 0.0;
  }
  if (materialise && split == 2) {  // children stay virtual until evaluated or needed as rows
    w->n_virtual = 2 * ns;
    w->nrm = 0;
    done = 1;
  } else if (materialise) {
    TRY(launch_split(w, w->dI, cfg, ns));
    CK(cudaStreamSynchronize(w->st));
    float e = 0;
    cudaEventElapsedTime(&e, w->ev[4], w->ev[5]);
    w->k3_ms += e;
    done = 1;
  }
  if (out) {
    out->n_split = ns;
    out->n_finalized = w->hst->n_final;
    out->width_guard_hits = w->hst->n_wall;
    out->finalized_integral = w->hst->fin_I;
    out->finalized_error = w->hst->fin_E;
    out->children_integral = w->hst->half_I;
    out->children_error = w->hst->half_E;
    out->split_done = done;
  }
  return 0;
}

int hcub_worker_classify(hcub_worker* w, double global_integral, const hcub_driver_cfg* cfg, int split,
                         hcub_classify_out* out) {
  if (!w || !cfg) return fail(HCUB_E_ARG, "bad arguments");
  if (w->pending) return fail(HCUB_E_ARG, "classify while an evaluation is pending");
  if (w->spec) return fail(HCUB_E_ARG, "a speculative classify is waiting for commit / discard");
  if (!w->evaluated && w->n > 0) return fail(HCUB_E_ARG, "classify needs an evaluated store");
  CK(cudaSetDevice(w->dev));
  w->settle_halves = false;
  CK(cudaMemcpyAsync(w->dI, &global_integral, sizeof(double), cudaMemcpyHostToDevice, w->st));
  CK(cudaEventRecord(w->ev[2], w->st));
  TRY(launch_classify(w, w->dI, cfg, /*compact=*/split == 2));
  CK(cudaMemcpyAsync(w->hst, w->dst, sizeof(DevStatus), cudaMemcpyDeviceToHost, w->st));
  CK(cudaStreamSynchronize(w->st));
  collect_eval_timings(w);
  return classify_finish(w, cfg, split, out, w->ev[2]);
}

// One-sync distributed protocol (distributed.py, NCCL): the global integral
// is reduced on the device from the all-gathered records and classify runs
// against it before the host has seen the records; the status mirror comes
// back with the caller's single stream synchronisation.  Nothing host-side
// changes until commit; discard (the loop stopped: converged or out of
// iterations) restores the finalized carry the speculative K3 advanced.
static int classify_launch_dev(hcub_worker* w, const double* dev_rows, int ranks, int width, int col_integral,
                               int col_bound, const hcub_driver_cfg* cfg) {
  CK(cudaMemcpyAsync(&w->dst->saved_fin_I, &w->dst->fin_I, 2 * sizeof(double), cudaMemcpyDeviceToDevice, w->st));
  k_record_reduce<<<1, 32, 0, w->st>>>(dev_rows, ranks, width, col_integral, col_bound, w->dI, w->dst);
  CK(cudaGetLastError());
  CK(cudaEventRecord(w->ev[8], w->st));
  TRY(launch_classify(w, w->dI, cfg, /*compact=*/true));
  CK(cudaMemcpyAsync(w->hst, w->dst, sizeof(DevStatus), cudaMemcpyDeviceToHost, w->st));
  w->launches += 1;
  w->spec = true;
  return 0;
}

int hcub_worker_classify_launch(hcub_worker* w, const double* dev_rows, int ranks, int width, int col_integral,
                                int col_bound, const hcub_driver_cfg* cfg) {
  if (!w || !cfg || !dev_rows || ranks < 1 || col_integral < 0 || col_bound < 0 || col_integral >= width ||
      col_bound >= width)
    return fail(HCUB_E_ARG, "bad arguments");
  if (w->pending) return fail(HCUB_E_ARG, "classify while an evaluation is pending");
  if (w->spec) return fail(HCUB_E_ARG, "a speculative classify is already waiting");
  if (!w->evaluated && w->n > 0) return fail(HCUB_E_ARG, "classify needs an evaluated store");
  CK(cudaSetDevice(w->dev));
  return classify_launch_dev(w, dev_rows, ranks, width, col_integral, col_bound, cfg);
}

int hcub_worker_classify_commit(hcub_worker* w, double global_integral, const hcub_driver_cfg* cfg,
                                hcub_classify_out* out) {
  if (!w || !cfg) return fail(HCUB_E_ARG, "bad arguments");
  if (!w->spec) return fail(HCUB_E_ARG, "no speculative classify to commit");
  CK(cudaSetDevice(w->dev));
  CK(cudaStreamSynchronize(w->st));  // normally a no-op: the caller synchronised the stream
  w->spec = false;
  collect_eval_timings(w);
  if (w->hst->spec_gI != global_integral && !(std::isnan(w->hst->spec_gI) && std::isnan(global_integral)))
    return fail(HCUB_E_PROTOCOL, "device-reduced global integral %.17g differs from the host's %.17g",
                w->hst->spec_gI, global_integral);
  w->settle_halves = false;
  return classify_finish(w, cfg, 2, out, w->ev[8]);
}

int hcub_worker_classify_discard(hcub_worker* w) {
  if (!w) return fail(HCUB_E_ARG, "worker is NULL");
  CK(cudaSetDevice(w->dev));
  if (w->spec)
    CK(cudaMemcpyAsync(&w->dst->fin_I, &w->dst->saved_fin_I, 2 * sizeof(double), cudaMemcpyDeviceToDevice, w->st));
  CK(cudaStreamSynchronize(w->st));
  w->spec = false;
  collect_eval_timings(w);
  return 0;
}

// ---------------------------------------------------------------------------
// Native NCCL communicator for the per-iteration record exchange (SURVEY.md
// 8b hcub_comm_init; ref distributed.py:325-346 metadata_reduce is the
// collective it carries).  libnccl.so.2 is resolved at run time - the copy
// torch already loaded when present - so the library has no link-time NCCL
// dependency and single-GPU use never touches it.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
  bool ok = false;
};
static NcclApi* nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.GetErrorString;
  });
  return api.ok ? &api : nullptr;
}
#define NK(call)                                                                                 \
  do {                                                                                           \
    ncclResult_t r_ = (call);                                                                    \
    if (r_ != ncclSuccess) return fail(HCUB_E_PROTOCOL, "NCCL: %s (%s:%d)", nccl_api()->GetErrorString(r_), \
                                       __FILE__, __LINE__);                                      \
  } while (0)

struct hcub_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 0, dev = 0, width = 0;
  double* drow = nullptr;   // own row + gathered rows (device)
  double* hbuf = nullptr;   // pinned host staging: own row, then the gathered rows
};

static void comm_free_bufs(hcub_comm* c) {
  if (c->drow) cudaFree(c->drow);
  if (c->hbuf) cudaFreeHost(c->hbuf);
  c->drow = nullptr;
  c->hbuf = nullptr;
  c->width = 0;
}

int hcub_nccl_unique_id(void* id128) {
  if (!id128) return fail(HCUB_E_ARG, "bad arguments");
  NcclApi* api = nccl_api();
  if (!api) return fail(HCUB_E_PROTOCOL, "libnccl.so.2 not found");
  ncclUniqueId id;
  NK(api->GetUniqueId(&id));
  memcpy(id128, id.internal, sizeof id.internal);
  return 0;
}

int hcub_comm_init(int device, int rank, int nranks, const void* id128, hcub_comm** out) {
  if (!out || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return fail(HCUB_E_ARG, "bad arguments");
  *out = nullptr;
  NcclApi* api = nccl_api();
  if (!api) return fail(HCUB_E_PROTOCOL, "libnccl.so.2 not found");
  CK(cudaSetDevice(device));
  ncclUniqueId id;
  memcpy(id.internal, id128, sizeof id.internal);
  hcub_comm* c = new hcub_comm();
  c->rank = rank;
  c->nranks = nranks;
  c->dev = device;
  const ncclResult_t r = api->CommInitRank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(HCUB_E_PROTOCOL, "ncclCommInitRank: %s", api->GetErrorString(r));
  }
  *out = c;
  return 0;
}

void hcub_comm_destroy(hcub_comm* c) {
  if (!c) return;
  cudaSetDevice(c->dev);
  comm_free_bufs(c);
  if (c->comm && nccl_api()) nccl_api()->CommDestroy(c->comm);
  delete c;
}

int hcub_worker_exchange_records(hcub_worker* w, hcub_comm* c, const double* row, int width, int col_partial,
                                 int col_bound, const hcub_driver_cfg* cfg, double* rows_out) {
  if (!w || !c || !row || !rows_out || width < 1 || col_partial < 0 || col_partial + 1 >= width || col_bound < 0 ||
      col_bound >= width)
    return fail(HCUB_E_ARG, "bad arguments");
  if (w->pending) return fail(HCUB_E_ARG, "an evaluation is pending (call hcub_worker_evaluate_end)");
  if (w->dev != c->dev) return fail(HCUB_E_ARG, "worker and communicator are on different devices");
  if (cfg && w->spec) return fail(HCUB_E_ARG, "a speculative classify is already waiting");
  CK(cudaSetDevice(w->dev));
  const int P = c->nranks;
  if (c->width != width) {
    CK(cudaStreamSynchronize(w->st));
    comm_free_bufs(c);
    CK(cudaMalloc(&c->drow, sizeof(double) * width * (P + 1)));
    CK(cudaHostAlloc(&c->hbuf, sizeof(double) * width * (P + 1), cudaHostAllocDefault));
    c->width = width;
  }
  double* drows = c->drow + width;
  memcpy(c->hbuf, row, sizeof(double) * width);
  CK(cudaMemcpyAsync(c->drow, c->hbuf, sizeof(double) * width, cudaMemcpyHostToDevice, w->st));
  CK(cudaMemcpyAsync(c->drow + col_partial, &w->dst->I, 2 * sizeof(double), cudaMemcpyDeviceToDevice, w->st));
  NK(nccl_api()->AllGather(c->drow, drows, (size_t)width, ncclFloat64, c->comm, w->st));
  if (cfg) TRY(classify_launch_dev(w, drows, P, width, col_partial, col_bound, cfg));
  CK(cudaMemcpyAsync(c->hbuf + width, drows, sizeof(double) * width * P, cudaMemcpyDeviceToHost, w->st));
  CK(cudaStreamSynchronize(w->st));
  memcpy(rows_out, c->hbuf + width, sizeof(double) * width * P);
  return 0;
}

}  // extern "C"

// take_top on virtual children (after classify(split=2)): selection over the
// survivors' columns, no child rows are built and nothing is compacted - the
// removed children are skipped by the next K1 / k3_expand (w->rmS).  Device
// traffic: two passes over the survivors (8 B index + 8 B error gather each)
// plus the threshold bucket's candidates, instead of expanding, radix-sorting
// and rewriting the whole store.
static const int64_t VT_MAX_TAKE = 8192;  // k4v_gather ranks the picks by O(m^2) comparisons

static int take_top_virtual(hcub_worker* w, int64_t n, double* lo, double* hi, double* error, double* integral,
                            int on_device) {
  const int64_t ns = w->n_virtual / 2;  // survivors; n <= 2 * ns
  const int64_t m = (n + 1) / 2;         // survivors giving children
  TRY(ensure_take(w, m));
  if (!on_device) TRY(ensure_stage(w, n));
  if (w->rm_cap < n || w->cand_cap < ns) {
    CK(cudaStreamSynchronize(w->st));
    if (w->rm_cap < n) {
      arena_free(w->dev, w->rmS);
      w->rmS = nullptr;
      w->rm_cap = std::max<int64_t>(n, 1024);
      AK(arena_alloc(w->dev, w->rm_cap * sizeof(int64_t), (void**)&w->rmS));
    }
    if (w->cand_cap < ns) {
      arena_free(w->dev, w->cand_k); arena_free(w->dev, w->cand_i);
      w->cand_k = nullptr; w->cand_i = nullptr;
      w->cand_cap = std::max<int64_t>(ns + ns / 2, 1 << 16);
      AK(arena_alloc(w->dev, w->cand_cap * sizeof(unsigned long long), (void**)&w->cand_k));
      AK(arena_alloc(w->dev, w->cand_cap * sizeof(long long), (void**)&w->cand_i));
    }
  }
  Cols& c = w->buf[w->cur];
  const unsigned g = (unsigned)std::min<int64_t>(grid_for(ns, 256), (int64_t)w->sms * 8);
  k4v_hist12<<<g, 256, 0, w->st>>>(w->pidx, c.E, ns, w->hist);
  k4v_pick12<<<1, 32, 0, w->st>>>(w->hist, m, w->dst);
  k4v_collect<<<g, 256, 0, w->st>>>(w->pidx, c.E, ns, w->dst, w->ck, w->ci, w->cand_k, w->cand_i, w->cand_cap);
  // exact (key, survivor index) selection among the bucket's candidates
  const unsigned gc = (unsigned)std::min<int64_t>(grid_for(ns, 256), (int64_t)w->sms * 2);
  for (int shift = 48; shift >= 0; shift -= 8) {
    k4c_hist<<<gc, 256, 0, w->st>>>(w->cand_k, w->cand_i, w->dst, 0, shift, w->hist);
    k4_pick<<<1, 1, 0, w->st>>>(w->hist, 0, shift, w->dst);
  }
  int idx_bytes = 1;
  while (idx_bytes < 8 && (ns >> (8 * idx_bytes)) > 0) ++idx_bytes;
  for (int shift = 8 * (idx_bytes - 1); shift >= 0; shift -= 8) {
    k4c_hist<<<gc, 256, 0, w->st>>>(w->cand_k, w->cand_i, w->dst, 1, shift, w->hist);
    k4_pick<<<1, 1, 0, w->st>>>(w->hist, 1, shift, w->dst);
  }
  k4c_collect<<<gc, 256, 0, w->st>>>(w->cand_k, w->cand_i, w->dst, w->ck, w->ci);
  double* olo = on_device ? lo : w->stage;
  double* ohi = on_device ? hi : w->stage + n * w->d;
  double* oE = on_device ? error : w->stage + 2 * n * w->d;
  double* oI = on_device ? integral : w->stage + 2 * n * w->d + n;
  k4v_gather<<<(unsigned)grid_for(m, 256), 256, 0, w->st>>>(w->ck, w->ci, m, n, w->pidx, c, w->cap(), w->axis, w->d,
                                                            olo, ohi, oE, oI, w->rmS);
  CK(cudaGetLastError());
  w->launches += 5 + 2 * (7 + idx_bytes);
  if (!on_device) {
    if (lo) CK(cudaMemcpyAsync(lo, olo, n * w->d * 8, cudaMemcpyDeviceToHost, w->st));
    if (hi) CK(cudaMemcpyAsync(hi, ohi, n * w->d * 8, cudaMemcpyDeviceToHost, w->st));
    if (error) CK(cudaMemcpyAsync(error, oE, n * 8, cudaMemcpyDeviceToHost, w->st));
    if (integral) CK(cudaMemcpyAsync(integral, oI, n * 8, cudaMemcpyDeviceToHost, w->st));
  }
  long long cnt = 0;
  CK(cudaMemcpyAsync(&cnt, &w->dst->take_count, sizeof cnt, cudaMemcpyDeviceToHost, w->st));
  CK(cudaStreamSynchronize(w->st));
  if (cnt != m) return fail(HCUB_E_PROTOCOL, "take_top selected %lld survivors, expected %lld", cnt, (long long)m);
  w->nrm = n;
  w->evaluated = false;  // the store holds parents plus virtual children: evaluate next
  return 0;
}

extern "C" int hcub_worker_take_top(hcub_worker* w, int64_t n, double* lo, double* hi, double* error,
                                    double* integral, int on_device, int64_t* taken) {
  if (w && w->pending) return fail(HCUB_E_ARG, "an evaluation is pending (call hcub_worker_evaluate_end)");
  if (!w || n < 0) return fail(HCUB_E_ARG, "bad arguments");
  if (taken) *taken = 0;
  CK(cudaSetDevice(w->dev));
  if (w->n_virtual >= 0 && w->nrm == 0 && n > 0) {
    const int64_t nn = std::min<int64_t>(n, w->n_virtual);
    if (nn > 0 && nn <= VT_MAX_TAKE) {
      TRY(take_top_virtual(w, nn, lo, hi, error, integral, on_device));
      if (taken) *taken = nn;
      return 0;
    }
  }
  TRY(materialize(w));
  n = std::min<int64_t>(n, w->n);
  if (n == 0) return 0;
  CK(cudaSetDevice(w->dev));
  TRY(ensure_take(w, n));
  TRY(ensure_stage(w, n));
  TRY(ensure_next(w, w->n - n));
  TRY(ensure_rows(w, w->n));
  Cols& c = w->buf[w->cur];
  const unsigned g = (unsigned)std::min<int64_t>(grid_for(w->n, 256), (int64_t)w->sms * 8);
  // MSB radix select of the n-th smallest key, then of the index among ties
  {
    DevStatus init{};
    CK(cudaMemcpyAsync(&w->dst->take_count, &init.take_count, 4 * sizeof(long long), cudaMemcpyHostToDevice, w->st));
    long long rank = n;
    CK(cudaMemcpyAsync(&w->dst->sel_rank, &rank, sizeof rank, cudaMemcpyHostToDevice, w->st));
  }
  for (int shift = 56; shift >= 0; shift -= 8) {
    k4_hist<<<g, 256, 0, w->st>>>(c.E, w->n, 0, shift, w->dst, w->hist);
    k4_pick<<<1, 1, 0, w->st>>>(w->hist, 0, shift, w->dst);
  }
  int idx_bytes = 1;
  while (idx_bytes < 8 && (w->n >> (8 * idx_bytes)) > 0) ++idx_bytes;
  for (int shift = 8 * (idx_bytes - 1); shift >= 0; shift -= 8) {
    k4_hist<<<g, 256, 0, w->st>>>(c.E, w->n, 1, shift, w->dst, w->hist);
    k4_pick<<<1, 1, 0, w->st>>>(w->hist, 1, shift, w->dst);
  }
  k4_collect<<<g, 256, 0, w->st>>>(c.E, w->n, w->dst, w->ck, w->ci, w->removed);
  double* olo = on_device ? lo : w->stage;
  double* ohi = on_device ? hi : w->stage + n * w->d;
  double* oE = on_device ? error : w->stage + 2 * n * w->d;
  double* oI = on_device ? integral : w->stage + 2 * n * w->d + n;
  k4_rank_gather<<<(unsigned)grid_for(n, 256), 256, 0, w->st>>>(w->ck, w->ci, n, c, w->cap(), w->d, olo, ohi, oE, oI);
  CK(cudaGetLastError());
  // order-preserving removal into the other buffer
  const int64_t tiles = (w->n + TILE - 1) / TILE;
  const int nb = w->cur ^ 1;
  k_keep_count<<<(unsigned)tiles, TILE_THREADS, 0, w->st>>>(w->removed, w->n, w->tiles);
  k_scan_tiles<<<1, 1024, 0, w->st>>>(w->tiles, tiles, w->scratch_i64);
  k_keep_scatter<<<(unsigned)tiles, TILE_THREADS, 0, w->st>>>(w->removed, w->n, c, w->cap(), w->buf[nb], w->bcap[nb], w->d, w->tiles);
  CK(cudaGetLastError());
  w->launches += 2 * (8 + idx_bytes) + 5;
  if (!on_device) {
    if (lo) CK(cudaMemcpyAsync(lo, olo, n * w->d * 8, cudaMemcpyDeviceToHost, w->st));
    if (hi) CK(cudaMemcpyAsync(hi, ohi, n * w->d * 8, cudaMemcpyDeviceToHost, w->st));
    if (error) CK(cudaMemcpyAsync(error, oE, n * 8, cudaMemcpyDeviceToHost, w->st));
    if (integral) CK(cudaMemcpyAsync(integral, oI, n * 8, cudaMemcpyDeviceToHost, w->st));
  }
  long long cnt = 0;
  CK(cudaMemcpyAsync(&cnt, &w->dst->take_count, sizeof cnt, cudaMemcpyDeviceToHost, w->st));
  CK(cudaStreamSynchronize(w->st));
  if (cnt != n) return fail(HCUB_E_PROTOCOL, "take_top selected %lld rows, expected %lld", cnt, (long long)n);
  w->cur = nb;
  w->n -= n;
  w->evaluated = false;
  if (taken) *taken = n;
  return 0;
}

extern "C" int hcub_worker_exact_partial(hcub_worker* w, int which, int64_t* slots68, int32_t* specials3) {
  if (w && w->pending) return fail(HCUB_E_ARG, "an evaluation is pending (call hcub_worker_evaluate_end)");
  if (!w || (which != 0 && which != 1) || !slots68) return fail(HCUB_E_ARG, "bad arguments");
  CK(cudaSetDevice(w->dev));
  TRY(materialize(w));
  Cols& c = w->buf[w->cur];
  CK(cudaMemsetAsync(&w->acc[ACC_I], 0, 2 * sizeof(SAcc), w->st));
  // unsplit store after a capacity failure: the parents' rows are replaced
  // by their children's provisional halves (acc[ACC_HALF_*]); rows appended
  // since then count in full
  const int64_t r0 = w->settle_halves ? std::min(w->halves_rows, w->n) : 0;
  if (w->n > r0) {
    const int64_t m = w->n - r0;
    const unsigned g2 = (unsigned)std::min<int64_t>(grid_for(m, 256), (int64_t)w->sms * 8);
    k2_reduce<<<g2, 256, 0, w->st>>>(c.I + r0, c.E + r0, m, w->acc);
    CK(cudaGetLastError());
  }
  SAcc h, hh{};
  CK(cudaMemcpyAsync(&h, &w->acc[ACC_I + which], sizeof(SAcc), cudaMemcpyDeviceToHost, w->st));
  if (w->settle_halves)
    CK(cudaMemcpyAsync(&hh, &w->acc[ACC_HALF_I + which], sizeof(SAcc), cudaMemcpyDeviceToHost, w->st));
  CK(cudaStreamSynchronize(w->st));
  for (int k = 0; k < SA_SLOTS; ++k) slots68[k] = (int64_t)(h.slot[k] + hh.slot[k]);  // slot-wise, exact
  if (specials3) {
    specials3[0] = h.nan_count + hh.nan_count;
    specials3[1] = h.pinf_count + hh.pinf_count;
    specials3[2] = h.ninf_count + hh.ninf_count;
  }
  return 0;
}

extern "C" int hcub_worker_timings(hcub_worker* w, double* k1, double* k2, double* k3, int64_t* k1n, int64_t* nl) {
  if (!w) return fail(HCUB_E_ARG, "worker is NULL");
  if (k1) *k1 = w->k1_ms;
  if (k2) *k2 = w->k2_ms;
  if (k3) *k3 = w->k3_ms;
  if (k1n) *k1n = w->k1_launches;
  if (nl) *nl = w->launches;
  return 0;
}

// ---------------------------------------------------------------------------
// single-worker loop (ref driver.py:237-323)

extern "C" int hcub_integrate(int device, const hcub_rule* rule, const hcub_integrand* f, const double* dom_lo,
                              const double* dom_hi, const double* lo0, const double* hi0, int64_t n0,
                              const hcub_driver_cfg* cfg, int64_t capacity, hcub_trace_fn trace, void* user,
                              hcub_result* out) {
  if (!cfg || !out || n0 < 1 || !lo0 || !hi0) return fail(HCUB_E_ARG, "bad arguments");
  if (!(cfg->tau_rel > 0)) return fail(HCUB_E_ARG, "tau_rel must be positive");
  if (cfg->max_regions < 1 || cfg->max_iterations < 1) return fail(HCUB_E_ARG, "max_regions and max_iterations must be >= 1");
  memset(out, 0, sizeof *out);
  hcub_worker* w = nullptr;
  TRY(worker_init(device, rule, f, dom_lo, dom_hi, capacity, &w));
  struct Guard { hcub_worker* w; ~Guard() { worker_release(w); } } guard{w};
  TRY(hcub_worker_append(w, lo0, hi0, nullptr, nullptr, n0, 0));

  cudaEvent_t t0, t1;
  CK(cudaEventCreate(&t0));
  CK(cudaEventCreate(&t1));
  CK(cudaEventRecord(t0, w->st));
  int64_t it = 0, evals = 0, peak = w->n, n_children = 0;
  int reason = -1;
  bool conv = false;
  double I = 0, E = 0;
  struct Range {  // one NVTX range per iteration (K1 -> sums -> K3 -> status read)
    Range() { nvtxRangePushA("hcub.integrate.iteration"); }
    ~Range() { nvtxRangePop(); }
  };
  while (true) {
    Range range;
    ++it;
    if (it == 1) TRY(launch_evaluate(w));
    else TRY(launch_evaluate_children(w, n_children));  // fused split: K1 builds the children
    const bool last = it >= cfg->max_iterations;
    // speculative (needs only device scalars): classify, tile scan, survivor list
    if (!last) TRY(launch_classify(w, &w->dst->I, cfg, /*compact=*/true));
    CK(cudaMemcpyAsync(w->hst, w->dst, sizeof(DevStatus), cudaMemcpyDeviceToHost, w->st));
    CK(cudaStreamSynchronize(w->st));
    add_timings(w, false, !last);
    I = w->hst->I;
    E = w->hst->E;
    evals += w->n * w->K;
    peak = std::max(peak, w->n);
    if (trace && trace(user, it, w->n, I, E, evals) != 0)
      return fail(HCUB_E_ABORTED, "trace callback aborted the integration at iteration %lld", (long long)it);
    if (E <= std::max(cfg->abs_floor, std::fabs(I) * cfg->tau_rel)) { reason = HCUB_TOLERANCE; conv = true; break; }
    if (it >= cfg->max_iterations) { reason = HCUB_MAX_ITERATIONS; break; }
    const int64_t ns = w->hst->n_split;
    if (ns == 0) {
      I = w->hst->fin_I;
      E = w->hst->fin_E;
      conv = E <= std::max(cfg->abs_floor, std::fabs(I) * cfg->tau_rel);
      reason = conv ? HCUB_TOLERANCE : HCUB_WIDTH_GUARD_EXHAUSTED;
      break;
    }
    if (2 * ns > cfg->max_regions) { reason = HCUB_MAX_REGIONS; break; }
    int grow = ensure_next(w, 2 * ns);
    if (!grow) grow = ensure_rows(w, 2 * ns);  // the children's per-row columns too
    if (grow == HCUB_E_CAPACITY) { reason = HCUB_MAX_REGIONS; out->capacity_limited = 1; break; }
    if (grow) return grow;
    n_children = 2 * ns;
  }
  CK(cudaEventRecord(t1, w->st));
  CK(cudaEventSynchronize(t1));
  float ms = 0;
  cudaEventElapsedTime(&ms, t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  out->integral = I;
  out->error = E;
  out->converged = conv;
  out->termination_reason = reason;
  out->iterations = it;
  out->total_f_evals = evals;
  out->peak_regions = peak;
  out->device_ms = ms;
  out->k1_ms = w->k1_ms;
  out->k2_ms = w->k2_ms;
  out->k3_ms = w->k3_ms;
  out->k1_launches = w->k1_launches;
  out->launches = w->launches;
  return 0;
}

// ---------------------------------------------------------------------------
// operator-level entry points

extern "C" int hcub_apply_rule_batch(int device, const hcub_rule* rule, const hcub_integrand* f, const double* lo,
                                     const double* hi, int64_t n, double* integral, double* error, double* scores,
                                     int64_t* axis, int64_t* evals) {
  RuleC rc;
  TRY(make_rule(rule, &rc));
  FnParams fp;
  TRY(make_fn(f, rule->d, &fp));
  const int d = rule->d;
  const int64_t K = (rule->kind == 1 || rule->kind == 3) ? rule->K
                    : rule->kind == 2 ? (int64_t)make_gk(d).K
                                      : (1ll << d) + 2ll * d * d + 2ll * d + 1;
  if (evals) *evals = n * K;
  if (n == 0) return 0;
  if (n < 0 || !lo || !hi || !integral || !error) return fail(HCUB_E_ARG, "bad arguments");
  CK(cudaSetDevice(device));
  const int sms = device_sms(device);
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct SG { cudaStream_t s; ~SG() { cudaStreamSynchronize(s); cudaStreamDestroy(s); } } sg{st};
  const size_t rb = (size_t)n * d * sizeof(double);
  double *rows = nullptr, *soa = nullptr, *out = nullptr, *dsc = nullptr;
  int64_t* dax = nullptr;
  CK(cudaMallocAsync(&rows, 2 * rb, st));
  CK(cudaMallocAsync(&soa, 2 * rb, st));
  CK(cudaMallocAsync(&out, 2 * n * sizeof(double), st));
  CK(cudaMallocAsync(&dax, n * sizeof(int64_t), st));
  if (scores) CK(cudaMallocAsync(&dsc, rb, st));
  CK(cudaMemcpyAsync(rows, lo, rb, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(rows + n * d, hi, rb, cudaMemcpyHostToDevice, st));
  Cols c{soa, soa + n * d, out, out + n};
  k5_append_rows<<<(unsigned)std::min<int64_t>(grid_for(n, 256), 4096), 256, 0, st>>>(rows, rows + n * d, n, d, c, n, 0,
                                                                                       nullptr, nullptr);
  CK(cudaGetLastError());
  K1Args a{};
  a.lo = c.lo; a.hi = c.hi; a.ld = n; a.n = n;
  a.integral = out; a.error = out + n; a.axis64 = dax; a.scores = dsc;
  a.log2g = pick_log2g(n, sms);
  DevTable tab;
  struct TG { DevTable* t; ~TG() { t->release(); } } tg{&tab};
  if (rule->kind == 2) {
    const GkArgs g = make_gk(d);
    const int64_t len = std::min<int64_t>(GK_SCRATCH, n * (int64_t)g.chunks * (d + 3));
    double* part = nullptr;
    CK(cudaMallocAsync(&part, len * 8, st));
    CK(launch_gk(f->kind, d, a, g, fp, part, len, st));
    cudaFreeAsync(part, st);
  } else if (rule->kind == 1) {
    TRY(upload_table(rule, device, st, &tab));
    CK(K1T_LAUNCH[f->kind](d, &a, &tab.args, &fp, grid_for(n << a.log2g, K1_BLOCK), K1_BLOCK, st));
  } else if (rule->kind == 3) {
    Rule9C r9;
    TRY(make_rule9(rule, &r9));
    a.log2g = 0;
    CK(K9_LAUNCH[f->kind](d, &a, &r9, &fp, st));
  } else {
    unsigned grid, block;
    k1_geometry(a, n << a.log2g, sms, &grid, &block);
    CK(K1_LAUNCH[f->kind](d, &a, &rc, &fp, grid, block, st));
  }
  CK(cudaMemcpyAsync(integral, out, n * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(error, out + n, n * 8, cudaMemcpyDeviceToHost, st));
  if (axis) CK(cudaMemcpyAsync(axis, dax, n * 8, cudaMemcpyDeviceToHost, st));
  if (scores) CK(cudaMemcpyAsync(scores, dsc, rb, cudaMemcpyDeviceToHost, st));
  cudaFreeAsync(rows, st); cudaFreeAsync(soa, st); cudaFreeAsync(out, st); cudaFreeAsync(dax, st);
  if (dsc) cudaFreeAsync(dsc, st);
  CK(cudaStreamSynchronize(st));
  return 0;
}

extern "C" int hcub_eval_points(int device, const hcub_integrand* f, const double* pts, int64_t m, double* outv) {
  if (!f || (m > 0 && (!pts || !outv))) return fail(HCUB_E_ARG, "bad arguments");
  if (f->d < 1 || f->d > HCUB_MAX_DIM) return fail(HCUB_E_DIM, "dimension %d unsupported", f->d);
  if (m == 0) return 0;
  FnParams fp;
  TRY(make_fn(f, f->d, &fp));
  CK(cudaSetDevice(device));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct SG { cudaStream_t s; ~SG() { cudaStreamSynchronize(s); cudaStreamDestroy(s); } } sg{st};
  double *dp = nullptr, *dv = nullptr;
  CK(cudaMallocAsync(&dp, m * f->d * 8, st));
  CK(cudaMallocAsync(&dv, m * 8, st));
  CK(cudaMemcpyAsync(dp, pts, m * f->d * 8, cudaMemcpyHostToDevice, st));
  CK(PT_LAUNCH[f->kind](f->d, dp, m, dv, &fp, st));
  CK(cudaMemcpyAsync(outv, dv, m * 8, cudaMemcpyDeviceToHost, st));
  cudaFreeAsync(dp, st);
  cudaFreeAsync(dv, st);
  CK(cudaStreamSynchronize(st));
  return 0;
}

extern "C" int hcub_exact_sum(int device, const double* x, int64_t n, double carry, double* out) {
  if (!out || (n > 0 && !x) || n < 0) return fail(HCUB_E_ARG, "bad arguments");
  CK(cudaSetDevice(device));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct SG { cudaStream_t s; ~SG() { cudaStreamSynchronize(s); cudaStreamDestroy(s); } } sg{st};
  double* dx = nullptr;
  SAcc* acc = nullptr;
  DevStatus* dst = nullptr;
  CK(cudaMallocAsync(&dx, (n > 0 ? n : 1) * 8, st));
  CK(cudaMallocAsync(&acc, 2 * sizeof(SAcc), st));
  CK(cudaMallocAsync(&dst, sizeof(DevStatus), st));
  CK(cudaMemsetAsync(acc, 0, 2 * sizeof(SAcc), st));
  CK(cudaMemsetAsync(dst, 0, sizeof(DevStatus), st));
  if (n > 0) {
    CK(cudaMemcpyAsync(dx, x, n * 8, cudaMemcpyHostToDevice, st));
    const unsigned g = (unsigned)std::min<int64_t>(grid_for(n, 256), 1024);
    k2_reduce<<<g, 256, 0, st>>>(dx, dx, n, acc);  // I and E both sum x
    CK(cudaGetLastError());
  }
  CK(cudaMemcpyAsync(&dst->fin_I, &carry, 8, cudaMemcpyHostToDevice, st));
  k2_round<<<1, 64, 0, st>>>(acc, dst);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, &dst->I, 8, cudaMemcpyDeviceToHost, st));
  cudaFreeAsync(dx, st); cudaFreeAsync(acc, st); cudaFreeAsync(dst, st);
  CK(cudaStreamSynchronize(st));
  return 0;
}

extern "C" int hcub_worker_evaluate_tail(hcub_worker* w, int64_t start, int64_t* evals) {
  if (w && w->pending) return fail(HCUB_E_ARG, "an evaluation is pending (call hcub_worker_evaluate_end)");
  if (!w) return fail(HCUB_E_ARG, "bad arguments");
  CK(cudaSetDevice(w->dev));
  TRY(materialize(w));
  if (start < 0 || start > w->n) return fail(HCUB_E_ARG, "bad arguments");
  const int64_t m = w->n - start;
  if (evals) *evals = m * w->K;
  if (m == 0) return 0;
  TRY(ensure_rows(w, w->n));
  Cols& c = w->buf[w->cur];
  K1Args a{};
  a.lo = c.lo + start; a.hi = c.hi + start; a.ld = w->cap(); a.n = m;
  a.integral = c.I + start; a.error = c.E + start; a.vol = w->vol + start; a.axis = w->axis + start;
  a.aext = w->aext + start;
  a.log2g = pick_log2g(m, w->sms);
  CK(launch_k1(w, a, m << a.log2g));
  CK(cudaStreamSynchronize(w->st));
  w->k1_launches += 1;
  w->launches += 1;
  return 0;
}

extern "C" int hcub_trim(int device) {
  CK(cudaSetDevice(device));
  std::vector<hcub_worker*> idle;
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    idle.swap(g_pool[device & 63]);
  }
  for (auto* w : idle) worker_free(w);
  std::lock_guard<std::mutex> lk(g_arena.mu);
  for (auto& kv : g_arena.cached[device & 63]) { cudaFree(kv.second); g_arena.sizes[device & 63].erase(kv.second); }
  g_arena.cached[device & 63].clear();
  return 0;
}
