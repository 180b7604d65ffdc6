/* hcub_b200.h - C ABI of the B200-native h-adaptive cubature library.
 *
 * The reference (`hcub`, pkg/src/hcub/) is pure Python/NumPy and has no FFI
 * of its own.  These entry points are what its hot path would bind through
 * ctypes (INTEGRATION.md shows the binding); each names the reference
 * function it replaces.  Plain C types only; every pointer argument says
 * whether it is host or device memory.  All functions return 0 on success or
 * an HCUB_E_* code; hcub_last_error() then holds a message (thread local).
 *
 * Layouts: region bounds cross the ABI row-major (n, d) like the reference's
 * numpy arrays; inside the library the store is structure-of-arrays in HBM.
 */
#ifndef HCUB_B200_H
#define HCUB_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HCUB_ABI_VERSION 2
#define HCUB_MAX_DIM 13

/* return codes (the Python shim maps them onto the reference's exceptions) */
enum {
  HCUB_OK = 0,
  HCUB_E_DIM = 1,      /* UnsupportedDimensionError  (ref rules.py:67-68, 266-269) */
  HCUB_E_ARG = 2,      /* ValueError                 (ref driver.py:97-101) */
  HCUB_E_CUDA = 3,     /* CUDA runtime failure */
  HCUB_E_PROTOCOL = 4, /* ProtocolError              (ref distributed.py:72-73) */
  HCUB_E_OOM = 5,      /* device memory exhausted */
  HCUB_E_CAPACITY = 6, /* store capacity exceeded */
  HCUB_E_ABORTED = 7   /* the trace callback asked to stop (it raised, ref driver.py:264-273) */
};

/* integrand kinds: BenchmarkIntegrand.id f1..f7 (ref integrands.py:32) and
 * make_product_peak (ref integrands.py:194-210) */
enum { HCUB_F1 = 1, HCUB_F2, HCUB_F3, HCUB_F4, HCUB_F5, HCUB_F6, HCUB_F7, HCUB_PRODUCT_PEAK };

typedef struct {
  int32_t kind; /* HCUB_F1 .. HCUB_PRODUCT_PEAK */
  int32_t d;
  double a;                    /* product peak: 1/sharpness^2 (f2: 50.0**-2) */
  double center[HCUB_MAX_DIM]; /* product-peak centers */
} hcub_integrand;

/* Fully symmetric degree-7/5 Genz-Malik table in generator form
 * (ref rules.py:257-282; axis bookkeeping rules.py:206-250). */
typedef struct {
  int32_t d;
  int32_t node_count;
  double lam2, lam3, lam4, lam5;
  double w[5], we[5]; /* per-node weights: center, lam2, lam3, lam4 pairs, lam5 corners */
  double fourth_diff_ratio, null_center_weight, null_axis_weight;
  /* kind 1: an explicit fully symmetric node table (parse_rule_table /
   * load_rule_table, ref rules.py:377-405) - custom families such as a
   * degree-9 Genz-Malik table.  Host pointers; copied to the device. */
  int32_t kind;           /* 0 = Genz-Malik generator form above, 1 = node table below,
                             2 = tensor Gauss(7)/Kronrod(15) rule, d <= 6 (ref rules.py:332-357),
                             3 = the degree-9 table of rule9.py given as a node table (below),
                                 evaluated in generator form (orbit layout checked) */
  int32_t has_axis_pairs; /* table carries the on-axis bookkeeping (ref rules.py:206-250) */
  int32_t center_index;
  int32_t axis_pairs[HCUB_MAX_DIM][4]; /* per axis: +inner, -inner, +outer, -outer node ids */
  int64_t K;
  const double* points;           /* (K, d) reference-cube nodes */
  const double* weights;          /* (K) */
  const double* embedded_weights; /* (K) */
} hcub_rule;

/* DriverConfig (ref driver.py:79-102) + VolumeBudgetClassifier.safety (:70) */
typedef struct {
  double tau_rel, abs_floor, min_width_ulp_factor, safety;
  int64_t max_iterations, max_regions;
} hcub_driver_cfg;

/* IntegrationResult (ref driver.py:115-123) plus device timings */
enum { HCUB_TOLERANCE = 0, HCUB_MAX_ITERATIONS = 1, HCUB_MAX_REGIONS = 2, HCUB_WIDTH_GUARD_EXHAUSTED = 3 };
typedef struct {
  double integral, error;
  int32_t converged, termination_reason;
  int64_t iterations, total_f_evals, peak_regions;
  int32_t capacity_limited; /* MAX_REGIONS fired on device capacity, not cfg.max_regions */
  int32_t pad;
  double device_ms;         /* CUDA-event time of the whole loop */
  double k1_ms, k2_ms, k3_ms;
  int64_t k1_launches, launches;
} hcub_result;

/* ClassifyOutcome (ref driver.py:137-144) + settle partials */
typedef struct {
  int64_t n_split, n_finalized, width_guard_hits;
  double finalized_integral, finalized_error;
  double children_integral, children_error; /* exact sums of the children's provisional halves */
  int32_t split_done; /* children materialised (0 when not requested or over capacity) */
  int32_t pad;
} hcub_classify_out;

/* IterationTrace sink (ref driver.py:126-134).  Returns 0 to continue; any
 * other value stops hcub_integrate at once with HCUB_E_ABORTED (the reference
 * propagates an exception raised by its trace callable immediately). */
typedef int (*hcub_trace_fn)(void* user, int64_t iteration, int64_t active_regions, double integral, double error,
                              int64_t f_evals);

typedef struct hcub_worker hcub_worker;

int hcub_abi_version(void);
const char* hcub_last_error(void);
int hcub_device_count(int* out);
/* Lanes per region of the Genz-Malik evaluation kernel, as log2 (0 = one
 * region per lane ... 5 = one region per warp); -1 (default) picks from the
 * batch size.  Process-wide; a tuning/testing knob with no reference
 * counterpart - results agree across settings to summation-order rounding,
 * scores and split axes bit for bit. */
int hcub_set_k1_lanes(int log2_lanes);

/* apply_rule_batch (ref rules.py:459-536 + driver.py:164).  Host pointers.
 * lo, hi: (n, d) row-major.  scores (n, d) and axis (n) may be NULL. */
int hcub_apply_rule_batch(int device, const hcub_rule* rule, const hcub_integrand* f, const double* lo,
                          const double* hi, int64_t n, double* integral, double* error, double* scores,
                          int64_t* axis, int64_t* evals);

/* exact_sum / exact_sum_with (ref driver.py:43-50): math.fsum([carry, *x])
 * computed on the device by the same superaccumulator the driver uses
 * (exactly rounded, order independent).  Host pointer x (n). */
int hcub_exact_sum(int device, const double* x, int64_t n, double carry, double* out);

/* BenchmarkIntegrand.__call__ (ref integrands.py:45-46): f at m points (m, d), host pointers */
int hcub_eval_points(int device, const hcub_integrand* f, const double* pts, int64_t m, double* out);

/* integrate (ref driver.py:237-323): the whole single-worker loop on device.
 * lo0/hi0: initial partition (n0, d) row-major host (uniform_partition,
 * ref regions.py:92-111, done by the caller).  capacity 0 = size from cfg and
 * free HBM.  trace may be NULL. */
int hcub_integrate(int device, const hcub_rule* rule, const hcub_integrand* f, const double* dom_lo,
                   const double* dom_hi, const double* lo0, const double* hi0, int64_t n0,
                   const hcub_driver_cfg* cfg, int64_t capacity, hcub_trace_fn trace, void* user, hcub_result* out);

/* ---- worker: one region store on one device (one rank of run_distributed,
 *      ref distributed.py:195-225).  Calls on one worker are serialised by
 *      the caller; distinct workers are independent (re-entrant). ---- */
int hcub_worker_create(int device, const hcub_rule* rule, const hcub_integrand* f, const double* dom_lo,
                       const double* dom_hi, int64_t capacity, hcub_worker** out);
void hcub_worker_destroy(hcub_worker* w);
int hcub_worker_size(hcub_worker* w, int64_t* n, int64_t* capacity);
/* RegionStore.append_batch (ref regions.py:182-218) / _deliver (distributed.py:400-403):
 * rows (m, d) row-major; on_device != 0 means lo/hi are device pointers.
 * integral/error may be NULL (zeros).  Every row needs lo < hi on every axis
 * (ref regions.py:204-205), checked on both paths (device rows by K5's flag
 * reduction): HCUB_E_ARG and nothing appended otherwise. */
int hcub_worker_append(hcub_worker* w, const double* lo, const double* hi, const double* integral,
                       const double* error, int64_t m, int on_device);
/* copy the store out (host pointers, row-major; any may be NULL) */
int hcub_worker_read(hcub_worker* w, double* lo, double* hi, double* integral, double* error, int64_t* axis);
/* finalized carry (WorkerState.finalized_*) */
int hcub_worker_set_carry(hcub_worker* w, double fin_integral, double fin_error);
int hcub_worker_get_carry(hcub_worker* w, double* fin_integral, double* fin_error);
/* evaluate_batch (ref driver.py:147-171) + WorkerState.record partials
 * (distributed.py:217-225): K1 over the store, exact sums with the carry. */
int hcub_worker_evaluate(hcub_worker* w, double* partial_integral, double* partial_error, int64_t* f_evals);
/* evaluate split in two so rows can arrive while K1 runs (round-robin
 * transfers overlapped with evaluation): _begin launches K1
 * over the current store (or the virtual children of the last classify)
 * and returns at once; rows appended meanwhile (hcub_worker_append) are
 * evaluated by _end with one more K1 into the same exact accumulators, then
 * the partials are rounded as hcub_worker_evaluate would: same per-row
 * estimates, same exact sums, same store order as delivering first and
 * evaluating after (ref distributed.py:482-499).  Between the two only
 * append is allowed. */
int hcub_worker_evaluate_begin(hcub_worker* w);
int hcub_worker_evaluate_end(hcub_worker* w, double* partial_integral, double* partial_error, int64_t* f_evals);
/* One-sync protocol (run_distributed over NCCL; no reference counterpart - the
 * reference's simulated ranks need no device synchronisation):
 *   evaluate_end_async  - evaluate_end without the host read; the partials
 *                         stay in device status (f_evals is host-known)
 *   stream              - the worker's cudaStream_t (collectives are enqueued on it)
 *   record_partials     - enqueue a device copy of (partial integral, partial
 *                         error) to dev_dst[0..1] (the caller's record row)
 *   classify_launch     - global integral = exact sum of columns col_integral
 *                         and col_bound of the all-gathered records
 *                         (ref distributed.py:338-345) reduced on the device,
 *                         then classify against it (ref :521-534) and the
 *                         status copied back - all asynchronous
 *   classify_commit     - after the caller synchronised the stream: checks the
 *                         device value equals the host's metadata_reduce,
 *                         then does classify's host half (split = 2)
 *   classify_discard    - the loop stopped: restore the finalized carry (with
 *                         no speculative classify: only settles the last
 *                         evaluation's timings) */
int hcub_worker_evaluate_end_async(hcub_worker* w, int64_t* f_evals);
int hcub_worker_stream(hcub_worker* w, void** stream);
int hcub_worker_record_partials(hcub_worker* w, double* dev_dst);
int hcub_worker_classify_launch(hcub_worker* w, const double* dev_rows, int ranks, int width, int col_integral,
                                int col_bound, const hcub_driver_cfg* cfg);
int hcub_worker_classify_commit(hcub_worker* w, double global_integral, const hcub_driver_cfg* cfg,
                                hcub_classify_out* out);
int hcub_worker_classify_discard(hcub_worker* w);

/* Native NCCL communicator (SURVEY.md 8b hcub_comm_init): libnccl.so.2 is
 * resolved at run time.  Rank 0 creates the 128-byte unique id, the caller
 * distributes it (run_distributed: torch.distributed broadcast), every rank
 * calls hcub_comm_init collectively. */
typedef struct hcub_comm hcub_comm;
int hcub_nccl_unique_id(void* id128);
int hcub_comm_init(int device, int rank, int nranks, const void* id128, hcub_comm** out);
void hcub_comm_destroy(hcub_comm* c);
/* The whole per-iteration record exchange of the one-sync protocol in one
 * call (replaces ref distributed.py:503-504 / 719-723): the host words of
 * `row` (width doubles) plus the worker's partials at columns
 * col_partial..col_partial+1 (from the device status left by
 * evaluate_end_async) are all-gathered over NCCL on the worker's stream; with
 * cfg != NULL the global integral (exact sum of columns col_partial and
 * col_bound) is reduced on the device and classify launched speculatively
 * (commit / discard as above); the nranks x width rows land in rows_out
 * after one stream synchronisation. */
int hcub_worker_exchange_records(hcub_worker* w, hcub_comm* c, const double* row, int width, int col_partial,
                                 int col_bound, const hcub_driver_cfg* cfg, double* rows_out);
/* _settle's evaluation of late arrivals (ref distributed.py:418-428): K1 over
 * rows [start, n) only; estimates of earlier rows are kept. */
int hcub_worker_evaluate_tail(hcub_worker* w, int64_t start, int64_t* f_evals);
/* make room for a split of up to `rows` children without growing later:
 * *ok = 1 if the spare buffer now holds them, 0 if the store capacity does
 * not allow it (the classify of such a store may then report split_done = 0).
 * run_distributed reserves 2n rows before the metadata exchange, so every
 * rank can prove from the gathered records that no split can overflow and
 * skip the reference's post-split count exchange (ref distributed.py:535-537). */
int hcub_worker_reserve(hcub_worker* w, int64_t rows, int32_t* ok);
/* classify_filter_split (ref driver.py:178-234) against a given global integral:
 * finalizes into the carry, counts, and replaces the store by the children
 * unless 2*n_split exceeds the capacity (then split_done = 0 and the store is
 * left evaluated; the caller terminates with MAX_REGIONS).  split: 0 = count
 * only, 1 = materialise the children now (K3 split), 2 = keep them virtual
 * (survivor list) - the next evaluate derives them inside K1, and any call
 * that needs rows (append / read / take_top / exact sums) materialises them. */
int hcub_worker_classify(hcub_worker* w, double global_integral, const hcub_driver_cfg* cfg, int split,
                         hcub_classify_out* out);
/* take_top (ref distributed.py:381-392): remove the n rows with the largest
 * provisional error (numpy stable argsort(-error) order) and write them to
 * lo/hi (n, d) row-major, error/integral (n); on_device selects pointer space. */
int hcub_worker_take_top(hcub_worker* w, int64_t n, double* lo, double* hi, double* error, double* integral,
                         int on_device, int64_t* taken);
/* exact (unrounded) sum of the store's integral (which = 0) or error
 * (which = 1) column as 68 signed 32-bit-digit slots in units of 2^-1074 plus
 * nan/+inf/-inf counts; lets the host combine ranks with one rounding, like
 * _settle's single math.fsum (distributed.py:430-437).  The finalized carry is
 * NOT included: the caller adds hcub_worker_get_carry's value exactly (the
 * Python shim does, worker.py ExactPartial).  After a classify whose split
 * could not be stored (split_done = 0) the evaluated parents count as their
 * children's provisional halves (ref driver.py:224-226), as the reference's
 * settle sees them; rows appended afterwards count in full. */
int hcub_worker_exact_partial(hcub_worker* w, int which, int64_t* slots68, int32_t* specials3);
/* drop the cached device memory (idle worker shells and allocator blocks) */
int hcub_trim(int device);
/* accumulated device timings of this worker */
int hcub_worker_timings(hcub_worker* w, double* k1_ms, double* k2_ms, double* k3_ms, int64_t* k1_launches,
                        int64_t* launches);

#ifdef __cplusplus
}
#endif
#endif
