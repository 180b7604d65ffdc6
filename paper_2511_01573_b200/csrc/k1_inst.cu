// One translation unit per integrand kind (compiled with -DHCUB_FN=<kind>):
// instantiates K1 for d = 2..13 and exposes a launcher switch.
#include <atomic>

#include "k1_table.cuh"
#include "k1_gm9.cuh"
#include "k1_gk.cuh"

#ifndef HCUB_FN
#error "compile with -DHCUB_FN=<FnKind>"
#endif

#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)

extern "C" cudaError_t CAT(hcub_launch_k1_fn, HCUB_FN)(int d, const K1Args* a, const RuleC* rc, const FnParams* fp,
                                                       unsigned grid, unsigned block, cudaStream_t st) {
  if (block == 0) return cudaErrorInvalidValue;
  // the caller sized grid x block threads; each dimension launches its own
  // block size (K1_BLOCK_OF) over the same thread range.  Only the G > 1 path
  // stages on-axis coordinates in shared memory.
  const unsigned long long threads = (unsigned long long)grid * block;
  switch (d) {
#define CASE(D) \
  case D: {                                                                                                 \
    constexpr int KB = K1_BLOCK_OF(D);                                                                        \
    const int smem = a->log2g ? 4 * D * KB * (int)sizeof(double) : 0;                                         \
    static std::atomic<unsigned long long> attr{0}; /* function attributes are per device */                 \
    int dev = 0;                                                                                              \
    cudaGetDevice(&dev);                                                                                      \
    if (!(attr.load() >> (dev & 63) & 1ull)) {                                                                \
      cudaFuncSetAttribute(k1_gm_eval<D, HCUB_FN>, cudaFuncAttributeMaxDynamicSharedMemorySize,               \
                           4 * D * KB * (int)sizeof(double));                                                 \
      attr.fetch_or(1ull << (dev & 63));                                                                      \
    }                                                                                                         \
    k1_gm_eval<D, HCUB_FN><<<(unsigned)((threads + KB - 1) / KB), KB, smem, st>>>(*a, *rc, *fp);              \
    break;                                                                                                    \
  }
    CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13)
#undef CASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// degree-9 family in generator form: one region per lane, a->n lanes
extern "C" cudaError_t CAT(hcub_launch_k9_fn, HCUB_FN)(int d, const K1Args* a, const Rule9C* r9, const FnParams* fp,
                                                       cudaStream_t st) {
  switch (d) {
#define CASE(D)                                                                              \
  case D: {                                                                                  \
    constexpr int KB = K1_BLOCK_OF(D);                                                       \
    k1_gm9_eval<D, HCUB_FN><<<(unsigned)((a->n + KB - 1) / KB), KB, 0, st>>>(*a, *r9, *fp);  \
    break;                                                                                   \
  }
    CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10)  /* d > 10: the node-table kernel (rules.py) */
#undef CASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

extern "C" cudaError_t CAT(hcub_launch_points_fn, HCUB_FN)(int d, const double* pts, int64_t m, double* out,
                                                           const FnParams* fp, cudaStream_t st) {
  const unsigned grid = (unsigned)((m + 255) / 256);
  switch (d) {
#define CASE(D) \
  case D: k_eval_points<D, HCUB_FN><<<grid, 256, 0, st>>>(pts, m, out, *fp); break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13)
#undef CASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

extern "C" cudaError_t CAT(hcub_launch_k1t_fn, HCUB_FN)(int d, const K1Args* a, const TableArgs* t, const FnParams* fp,
                                                        unsigned grid, unsigned block, cudaStream_t st) {
  switch (d) {
#define CASE(D) \
  case D: k1_table_eval<D, HCUB_FN><<<grid, block, 0, st>>>(*a, *t, *fp); break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13)
#undef CASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// tensor Gauss-Kronrod: partial sums for regions [r0, r0+nb), then finalize
extern "C" cudaError_t CAT(hcub_launch_k1gk_fn, HCUB_FN)(int d, const K1Args* a, const GkArgs* gk, const FnParams* fp,
                                                         int64_t r0, int64_t nb, double* part, cudaStream_t st) {
  const int64_t warps = nb * gk->chunks;
  const unsigned grid = (unsigned)((warps * 32 + 127) / 128);
  const unsigned fgrid = (unsigned)((nb * 32 + 127) / 128);
  switch (d) {
#define CASE(D)                                                                   \
  case D:                                                                         \
    k1_gk_partial<D, HCUB_FN><<<grid, 128, 0, st>>>(*a, *gk, *fp, r0, nb, part);  \
    k1_gk_finalize<D><<<fgrid, 128, 0, st>>>(*a, *gk, r0, nb, part);              \
    break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6)
#undef CASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
