// HBM-bound kernels over the SoA region store.
//
//  K2  k2_reduce          exact sums of integral/error columns
//                          (ref driver.py:48-50, 166-167; distributed.py:217-225)
//  K3  k3_classify        volume-budget classification, width guard, finalized
//                          carry sums, per-tile split counts
//                          (ref driver.py:72-76, 178-204)
//      k_scan_tiles       exclusive scan of per-tile counts (single block)
//      k3_split           order-preserving bisection of the survivors into the
//                          other buffer, children interleaved [2i]=lower,
//                          [2i+1]=upper, provisional half estimates
//                          (ref driver.py:206-226)
//  K4  k4_hist / k4_pick / k4_collect / k4_rank
//                          exact top-n by provisional error with numpy's
//                          stable argsort(-error) order
//                          (ref distributed.py:381-392), MSB radix select
//      k_keep_count/k_keep_scatter
//                          order-preserving removal (ref regions.py:226-261)
//  K5  k5_append_rows     receiver appends coordinate rows at the tail
//                          (ref distributed.py:400-403, regions.py:182-218)
#pragma once
#include "hcub_device.cuh"

#define TILE_THREADS 256
#define TILE_ITEMS 4  // even: k3_classify reads row pairs
#define TILE (TILE_THREADS * TILE_ITEMS)

struct Cols {        // one SoA buffer of the store
  double* lo;        // [d][cap]
  double* hi;        // [d][cap]
  double* I;         // [cap]
  double* E;         // [cap]
};

struct DevStatus {
  double I, E;             // partial estimate incl. finalized carry (evaluate)
  double fin_I, fin_E;     // finalized carry (classify)
  double half_I, half_E;   // sum of the children's provisional halves (settle)
  long long n_split, n_final, n_wall;
  double budget;           // max(floor, |I|*tau) of the last classify
  long long take_count;    // K4 candidates collected
  unsigned long long sel_key, sel_idx;
  long long sel_rank;      // remaining rank inside the current prefix bucket
  double saved_fin_I, saved_fin_E;  // carry before a speculative classify (restored on discard)
  double spec_gI;                   // global integral a speculative classify ran against
  long long pad[4];
};

enum { ACC_I = 0, ACC_E, ACC_FIN_I, ACC_FIN_E, ACC_HALF_I, ACC_HALF_E, ACC_N };

// ---------------------------------------------------------------------------
// K2

__global__ void __launch_bounds__(256) k2_reduce(const double* __restrict__ I, const double* __restrict__ E, int64_t n,
                                                 SAcc* acc /* [ACC_I], [ACC_E] */) {
  __shared__ SAcc s[2];
  for (int k = threadIdx.x; k < SA_SLOTS * 2; k += blockDim.x) s[k / SA_SLOTS].slot[k % SA_SLOTS] = 0ull;
  if (threadIdx.x < 2) { s[threadIdx.x].nan_count = s[threadIdx.x].pinf_count = s[threadIdx.x].ninf_count = 0; }
  __syncthreads();
  // each warp walks contiguous chunks of 32 x 16 rows: every load is 32
  // consecutive rows, and a lane's successive rows are 32 apart (siblings of
  // similar magnitude), so the per-lane windows rarely miss
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  SaLane wi, we;
  for (int64_t ch = warp * 512; ch < n; ch += nwarps * 512) {
    // two batches of 8 rows per lane: all 16 loads of a batch are issued
    // before the (integer-heavy) accumulation, so HBM latency overlaps
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      double vi[8], ve[8];
#pragma unroll
      for (int s2 = 0; s2 < 8; ++s2) {
        const int64_t i = ch + (b * 8 + s2) * 32 + lane;
        vi[s2] = i < n ? __ldcs(I + i) : 0.0;  // +-0 adds nothing
        ve[s2] = i < n ? __ldcs(E + i) : 0.0;
      }
#pragma unroll
      for (int s2 = 0; s2 < 8; ++s2) {
        wi.add(&s[0], vi[s2]);
        we.add(&s[1], ve[s2]);
      }
    }
    wi.flush(&s[0]);
    we.flush(&s[1]);
  }
  __syncthreads();
  if (threadIdx.x == 0) sa_normalise(&s[0]);
  if (threadIdx.x == 32) sa_normalise(&s[1]);
  __syncthreads();
  sa_merge_atomic(&acc[ACC_I], &s[0], threadIdx.x, blockDim.x);
  sa_merge_atomic(&acc[ACC_E], &s[1], threadIdx.x, blockDim.x);
}

// Global integral of the distributed protocol from the all-gathered metadata
// records, on the device: exact sum of the partial integrals plus the
// in-flight integral bounds (ref distributed.py:338-345, rank order is
// immaterial for an exactly rounded sum) -> *out and st->spec_gI.  <<<1, 32>>>
__global__ void k_record_reduce(const double* rows, int ranks, int width, int ca, int cb, double* out,
                                DevStatus* st) {
  __shared__ SAcc s;
  for (int k = threadIdx.x; k < SA_SLOTS; k += blockDim.x) s.slot[k] = 0ull;
  if (threadIdx.x == 0) s.nan_count = s.pinf_count = s.ninf_count = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * ranks; i += blockDim.x) sa_add_atomic(&s, rows[(i >> 1) * width + ((i & 1) ? cb : ca)]);
  __syncthreads();
  if (threadIdx.x == 0) {
    const double v = sa_round(&s, 0.0);
    *out = v;
    st->spec_gI = v;
  }
}

// Fused-K2 variant of k2_round: sum the per-SM shards K1 accumulated into
// acc[ACC_I], acc[ACC_E] (slot-wise integer sums, exact), then round.
// <<<1, K2M_THREADS>>>: K2M_PARTS threads per (column, slot) each sum a
// strided subset of the shards, combined in shared memory.
#define K2M_PARTS 4
#define K2M_THREADS (2 * SA_SLOTS * K2M_PARTS)
__global__ void __launch_bounds__(K2M_THREADS) k2_merge_round(const SAcc* shards, int nshards, SAcc* acc,
                                                               DevStatus* st) {
  __shared__ unsigned long long part[K2M_THREADS];
  __shared__ unsigned specials[2][3];  // nan / +inf / -inf counts of the two columns
  const int t = threadIdx.x, cs = t / K2M_PARTS, q = t % K2M_PARTS;
  const int c = cs / SA_SLOTS, k = cs % SA_SLOTS;
  if (t < 6) specials[t / 3][t % 3] = 0;
  unsigned long long v = 0;
#pragma unroll 8
  for (int s = q; s < nshards; s += K2M_PARTS) v += shards[2 * s + c].slot[k];
  part[t] = v;
  __syncthreads();
  // special-value counts: one (shard, column) pair per thread, not a serial
  // walk over the shards (that walk was most of this kernel's time)
  for (int i = t; i < 2 * nshards; i += K2M_THREADS) {
    const SAcc& sh = shards[i];
    if (sh.nan_count) atomicAdd(&specials[i & 1][0], sh.nan_count);
    if (sh.pinf_count) atomicAdd(&specials[i & 1][1], sh.pinf_count);
    if (sh.ninf_count) atomicAdd(&specials[i & 1][2], sh.ninf_count);
  }
  __syncthreads();
  if (t < 2) {
    acc[ACC_I + t].nan_count = specials[t][0];
    acc[ACC_I + t].pinf_count = specials[t][1];
    acc[ACC_I + t].ninf_count = specials[t][2];
  }
  __syncthreads();
  if (q == 0) {
    unsigned long long sum = 0;
#pragma unroll
    for (int j = 0; j < K2M_PARTS; ++j) sum += part[t + j];
    acc[ACC_I + c].slot[k] = sum;
  }
  __syncthreads();
  if (t == 0) st->I = sa_round(&acc[ACC_I], st->fin_I);
  if (t == 32) st->E = sa_round(&acc[ACC_E], st->fin_E);
}

// partial = fsum([carry, *column]) for I and E   (one thread each)
__global__ void k2_round(const SAcc* acc, DevStatus* st) {  // <<<1, 64>>>: one warp per value
  if (threadIdx.x == 0) st->I = sa_round(&acc[ACC_I], st->fin_I);
  if (threadIdx.x == 32) st->E = sa_round(&acc[ACC_E], st->fin_E);
}

// ---------------------------------------------------------------------------
// K3

struct ClassifyArgs {
  Cols cur;
  int64_t cap;
  const double* vol;
  const signed char* axis;
  const double* aext;   // extent of the split axis (from K1)
  int64_t n;
  const double* gI;     // device pointer to the global integral estimate
  double tau, floor, safety, dvol;
  double inv_dvol;      // 1/dvol when that is exact (dvol a power of two), else 0
  double guard[HCUB_MAXD];  // ulp_factor * eps * domain_extent[axis]
  int d;
  int64_t* tile_counts;
  SAcc* acc;
  DevStatus* st;
  unsigned char* flags;  // [n] 1 = split (optional)
};

// vol_r / vol_domain as numpy rounds it: a multiplication by the exact
// reciprocal when the domain volume is a power of two (the same correctly
// rounded quotient, without the division's instruction sequence)
__device__ __forceinline__ double k3_vfrac(const ClassifyArgs& a, double vol) {
  return a.inv_dvol != 0.0 ? mul_rn(vol, a.inv_dvol) : __ddiv_rn(vol, a.dvol);
}

// ref driver.py:72-76 and 192-201
__device__ __forceinline__ bool k3_finalize(const ClassifyArgs& a, double bs, int64_t i, bool& wall) {
  const int ax = a.axis[i];
  wall = a.aext[i] <= a.guard[ax];  // (hi - lo)[axis] <= ulp_factor * eps * domain_extent[axis]
  const double thr = mul_rn(bs, k3_vfrac(a, a.vol[i]));
  return (a.cur.E[i] <= thr) || wall;
}

__device__ __forceinline__ double k3_bs(const ClassifyArgs& a) {
  const double I = *a.gI;
  const double budget = fmax(a.floor, mul_rn(fabs(I), a.tau));  // max(cfg.abs_floor, |I|*tau)
  return mul_rn(budget, a.safety);
}

// A tile's rows are taken in row pairs: pair (it, t) = rows tile*TILE +
// 2*(it*TILE_THREADS + t) + {0, 1}, so every column is read with one 128-bit
// load per pair and a warp's load covers 64 consecutive rows (512 B).
// Columns are 512-byte aligned allocations (arena) read from row 0.
constexpr int K3_PAIRS = TILE_ITEMS / 2;
__device__ __forceinline__ double2 k3_ld2(const double* p, int64_t i, int64_t n) {
  if (i + 1 < n) return __ldcs(reinterpret_cast<const double2*>(p + i));
  return make_double2(i < n ? __ldcs(p + i) : 0.0, 0.0);
}
#ifndef K3_MINB
#define K3_MINB 4  // measured f2 d=5 to tolerance, K3 total: 2 blocks 3.95 ms, 3 -> 3.63, 4 -> 3.32
#endif
__global__ void __launch_bounds__(TILE_THREADS, K3_MINB) k3_classify(ClassifyArgs a) {
  __shared__ SAcc s[2];
  __shared__ unsigned long long cnt[3];
  __shared__ double guard[HCUB_MAXD];  // per-axis width guard (divergent axes: no constant-bank serialisation)
  if (threadIdx.x < HCUB_MAXD) guard[threadIdx.x] = a.guard[threadIdx.x];
  for (int k = threadIdx.x; k < SA_SLOTS * 2; k += blockDim.x) s[k / SA_SLOTS].slot[k % SA_SLOTS] = 0ull;
  if (threadIdx.x < 2) { s[threadIdx.x].nan_count = s[threadIdx.x].pinf_count = s[threadIdx.x].ninf_count = 0; }
  if (threadIdx.x < 3) cnt[threadIdx.x] = 0;
  __syncthreads();
  const double bs = k3_bs(a);
  const int64_t tiles = (a.n + TILE - 1) / TILE;
  int nfin = 0, nwall = 0;
  long long nsplit_all = 0;  // lane 0 of each warp
  SaLane wi, we;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {  // persistent over tiles
    int nsplit = 0;
    // every load of the tile is issued before any is used (one HBM round
    // trip per tile; I is read for all items, finalized or not), then the
    // integer-heavy exact accumulation
    bool fin[TILE_ITEMS];
    double fi[TILE_ITEMS], fe[TILE_ITEMS], fv[TILE_ITEMS], fx[TILE_ITEMS];
    int fa[TILE_ITEMS];
#pragma unroll
    for (int p = 0; p < K3_PAIRS; ++p) {
      const int64_t i = tile * TILE + 2 * (p * TILE_THREADS + threadIdx.x);
      const double2 e = k3_ld2(a.cur.E, i, a.n), v = k3_ld2(a.cur.I, i, a.n);
      const double2 vo = k3_ld2(a.vol, i, a.n), x = k3_ld2(a.aext, i, a.n);
      fe[2 * p] = e.x; fe[2 * p + 1] = e.y;
      fi[2 * p] = v.x; fi[2 * p + 1] = v.y;
      fv[2 * p] = vo.x; fv[2 * p + 1] = vo.y;
      fx[2 * p] = x.x; fx[2 * p + 1] = x.y;
      if (i + 1 < a.n) {
        const char2 ax = __ldcs(reinterpret_cast<const char2*>(a.axis + i));
        fa[2 * p] = ax.x; fa[2 * p + 1] = ax.y;
      } else {
        fa[2 * p] = i < a.n ? (int)__ldcs(a.axis + i) : 0;
        fa[2 * p + 1] = 0;
      }
    }
#pragma unroll
    for (int it = 0; it < TILE_ITEMS; ++it) {
      const int64_t i = tile * TILE + 2 * ((it >> 1) * TILE_THREADS + threadIdx.x) + (it & 1);
      const bool in = i < a.n;
      // ref driver.py:72-76, 192-201
      const bool wall = in && fx[it] <= guard[fa[it]];
      const double thr = mul_rn(bs, k3_vfrac(a, fv[it]));
      fin[it] = in && ((fe[it] <= thr) || wall);
      nfin += fin[it];
      nsplit += in && !fin[it];
      nwall += wall;
    }
    if (a.flags) {
#pragma unroll
      for (int p = 0; p < K3_PAIRS; ++p) {
        const int64_t i = tile * TILE + 2 * (p * TILE_THREADS + threadIdx.x);
        if (i + 1 < a.n)
          *reinterpret_cast<uchar2*>(a.flags + i) = make_uchar2(!fin[2 * p], !fin[2 * p + 1]);
        else if (i < a.n)
          a.flags[i] = (unsigned char)!fin[2 * p];
      }
    }
#pragma unroll
    for (int it = 0; it < TILE_ITEMS; ++it)
      if (fin[it]) {
        wi.add(&s[0], fi[it]);
        we.add(&s[1], fe[it]);
      }
    // per-warp split counts straight into the (zeroed) tile counter: no
    // block barrier inside the tile loop, so loads of the next tile overlap
    for (int o = 16; o; o >>= 1) nsplit += __shfl_xor_sync(0xffffffffu, nsplit, o);
    if ((threadIdx.x & 31) == 0 && nsplit) {
      atomicAdd((unsigned long long*)&a.tile_counts[tile], (unsigned long long)nsplit);
      nsplit_all += nsplit;
    }
  }
  // lane windows are flushed once per block (a lane adds at most 4 values per
  // tile it visits: far below the 2^31 addends an int64 slot absorbs)
  wi.flush(&s[0]);
  we.flush(&s[1]);
  for (int o = 16; o; o >>= 1) {
    nfin += __shfl_xor_sync(0xffffffffu, nfin, o);
    nwall += __shfl_xor_sync(0xffffffffu, nwall, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&cnt[0], (unsigned long long)nsplit_all);
    atomicAdd(&cnt[1], (unsigned long long)nfin);
    atomicAdd(&cnt[2], (unsigned long long)nwall);
  }
  __syncthreads();
  if (threadIdx.x == 0) sa_normalise(&s[0]);
  if (threadIdx.x == 32) sa_normalise(&s[1]);
  if (threadIdx.x == 64) {
    atomicAdd((unsigned long long*)&a.st->n_split, cnt[0]);
    atomicAdd((unsigned long long*)&a.st->n_final, cnt[1]);
    atomicAdd((unsigned long long*)&a.st->n_wall, cnt[2]);
  }
  __syncthreads();
  sa_merge_atomic(&a.acc[ACC_FIN_I], &s[0], threadIdx.x, blockDim.x);
  sa_merge_atomic(&a.acc[ACC_FIN_E], &s[1], threadIdx.x, blockDim.x);
}

// Survivor flags of k3_classify -> stable list of survivor indices (the
// parents of the next store in the fused-split loop).
__global__ void __launch_bounds__(TILE_THREADS) k3_compact(const unsigned char* __restrict__ flags, int64_t n,
                                                           const int64_t* tile_offsets, int64_t* out_idx);

// Tile-local ranks of flagged striped items in tile order (it-major, then
// thread): warp ballots plus a 32-entry prefix over (item row, warp).
struct TileRanks {
  int warp_off[TILE_ITEMS][TILE_THREADS / 32];
};
__device__ __forceinline__ void tile_rank(const bool (&flag)[TILE_ITEMS], int (&rank)[TILE_ITEMS], TileRanks& sm) {
  const unsigned lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  unsigned bal[TILE_ITEMS];
#pragma unroll
  for (int it = 0; it < TILE_ITEMS; ++it) {
    bal[it] = __ballot_sync(0xffffffffu, flag[it]);
    if (lane == 0) sm.warp_off[it][w] = __popc(bal[it]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int it = 0; it < TILE_ITEMS; ++it)
      for (int q = 0; q < TILE_THREADS / 32; ++q) { const int c = sm.warp_off[it][q]; sm.warp_off[it][q] = run; run += c; }
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int it = 0; it < TILE_ITEMS; ++it) rank[it] = sm.warp_off[it][w] + __popc(bal[it] & lt);
}

// exact sums of the children's provisional halves (2 x 0.5*parent) of the
// survivors - only the distributed settle after MAX_REGIONS needs them
__global__ void __launch_bounds__(TILE_THREADS) k3_child_sums(ClassifyArgs a) {
  __shared__ SAcc s[2];
  for (int k = threadIdx.x; k < SA_SLOTS * 2; k += blockDim.x) s[k / SA_SLOTS].slot[k % SA_SLOTS] = 0ull;
  if (threadIdx.x < 2) { s[threadIdx.x].nan_count = s[threadIdx.x].pinf_count = s[threadIdx.x].ninf_count = 0; }
  __syncthreads();
  const double bs = k3_bs(a);
  SaWindow hi_, he;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
    bool wall;
    if (!k3_finalize(a, bs, i, wall)) {
      const double h1 = 0.5 * a.cur.I[i], h2 = 0.5 * a.cur.E[i];
      hi_.add(&s[0], h1); hi_.add(&s[0], h1);
      he.add(&s[1], h2); he.add(&s[1], h2);
    }
  }
  hi_.finish(&s[0]); he.finish(&s[1]);
  __syncthreads();
  if (threadIdx.x == 0) sa_normalise(&s[0]);
  if (threadIdx.x == 32) sa_normalise(&s[1]);
  __syncthreads();
  sa_merge_atomic(&a.acc[ACC_HALF_I], &s[0], threadIdx.x, blockDim.x);
  sa_merge_atomic(&a.acc[ACC_HALF_E], &s[1], threadIdx.x, blockDim.x);
}

// fin = fsum([fin, *finalized]); halves = exact sum of children provisional values
__global__ void k3_round(const SAcc* acc, DevStatus* st, const double* gI, double tau, double floor_) {
  // <<<1, 64>>>: one warp per value
  if (threadIdx.x == 0) st->fin_I = sa_round(&acc[ACC_FIN_I], st->fin_I);
  if (threadIdx.x == 32) st->fin_E = sa_round(&acc[ACC_FIN_E], st->fin_E);
  if (threadIdx.x == 1) st->budget = fmax(floor_, mul_rn(fabs(*gI), tau));
}

__global__ void k3_round_halves(const SAcc* acc, DevStatus* st) {  // <<<1, 64>>>
  if (threadIdx.x == 0) st->half_I = sa_round(&acc[ACC_HALF_I], 0.0);
  if (threadIdx.x == 32) st->half_E = sa_round(&acc[ACC_HALF_E], 0.0);
}

// exclusive scan of `counts[0..m)` in place, single block of 1024 threads.
// With `acc` set it also does k3_round's work afterwards (one launch less
// per iteration in the classify sequence).
__global__ void __launch_bounds__(1024) k_scan_tiles(int64_t* counts, int64_t m, int64_t* total,
                                                     const SAcc* acc = nullptr, DevStatus* st = nullptr,
                                                     const double* gI = nullptr, double tau = 0.0,
                                                     double floor_ = 0.0) {
  __shared__ long long warp_sums[32];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < m; base += 1024) {
    const int64_t i = base + threadIdx.x;
    long long v = (i < m) ? counts[i] : 0;
    long long x = v;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[w] = x;
    __syncthreads();
    if (w == 0) {
      long long s = warp_sums[lane];
      for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      warp_sums[lane] = s;
    }
    __syncthreads();
    const long long incl = x + (w ? warp_sums[w - 1] : 0) + carry;
    if (i < m) counts[i] = incl - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry = incl;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
  if (acc) {  // == k3_round
    if (threadIdx.x == 0) st->fin_I = sa_round(&acc[ACC_FIN_I], st->fin_I);
    if (threadIdx.x == 32) st->fin_E = sa_round(&acc[ACC_FIN_E], st->fin_E);
    if (threadIdx.x == 64) st->budget = fmax(floor_, mul_rn(fabs(*gI), tau));
  }
}

// block-level exclusive scan of one value per thread; returns the prefix
__device__ __forceinline__ int block_excl_scan(int v, int* smem_warp /*[TILE_THREADS/32]*/) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    int s = (lane < (int)(blockDim.x >> 5)) ? smem_warp[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    smem_warp[lane] = s;
  }
  __syncthreads();
  return x - v + (w ? smem_warp[w - 1] : 0);
}

struct SplitArgs {
  ClassifyArgs c;
  Cols nxt;
  int64_t cap_next;
  const int64_t* tile_offsets;  // exclusive scan of tile_counts
  int write_estimates;          // children's provisional 1/2 estimates (only take_top reads them)
};

__global__ void __launch_bounds__(TILE_THREADS) k3_split(SplitArgs s) {
  __shared__ TileRanks sm;
  const ClassifyArgs& a = s.c;
  const double bs = k3_bs(a);
  const int64_t tile0 = (int64_t)blockIdx.x * TILE;
  bool flag[TILE_ITEMS];
  int rank[TILE_ITEMS];
#pragma unroll
  for (int it = 0; it < TILE_ITEMS; ++it) {
    const int64_t i = tile0 + it * TILE_THREADS + threadIdx.x;
    bool wall;
    flag[it] = i < a.n && !k3_finalize(a, bs, i, wall);
  }
  tile_rank(flag, rank, sm);
  const int64_t off = s.tile_offsets[blockIdx.x];
  const int d = a.d;
#pragma unroll
  for (int it = 0; it < TILE_ITEMS; ++it) {
    if (!flag[it]) continue;
    const int64_t i = tile0 + it * TILE_THREADS + threadIdx.x;
    const int ax = a.axis[i];
    const int64_t c0 = 2 * (off + rank[it]);
    for (int j = 0; j < d; ++j) {
      const double l = a.cur.lo[(int64_t)j * a.cap + i], u = a.cur.hi[(int64_t)j * a.cap + i];
      double l1 = l, u0 = u;
      if (j == ax) {
        const double mid = add_rn(l, mul_rn(0.5, sub_rn(u, l)));  // ref driver.py:211
        u0 = mid;
        l1 = mid;
      }
      // children are adjacent: one 16-byte store per column, coalesced across the warp
      *reinterpret_cast<double2*>(&s.nxt.lo[(int64_t)j * s.cap_next + c0]) = make_double2(l, l1);
      *reinterpret_cast<double2*>(&s.nxt.hi[(int64_t)j * s.cap_next + c0]) = make_double2(u0, u);
    }
    if (s.write_estimates) {
      const double hI = 0.5 * a.cur.I[i], hE = 0.5 * a.cur.E[i];
      *reinterpret_cast<double2*>(&s.nxt.I[c0]) = make_double2(hI, hI);
      *reinterpret_cast<double2*>(&s.nxt.E[c0]) = make_double2(hE, hE);
    }
  }
}

// ---------------------------------------------------------------------------
// K4: exact top-n by provisional error (stable, numpy argsort(-E) order)

__device__ __forceinline__ unsigned long long k4_key(double e) {
  double v = -e;
  if (v == 0.0) v = 0.0;  // -0.0 and +0.0 compare equal in numpy's sort
  if (isnan(v)) return ~0ull;
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | (1ull << 63));
}

struct SelState {          // lives in DevStatus
  unsigned long long key;  // sel_key: selected prefix / final threshold key
  unsigned long long idx;  // sel_idx: index threshold among equal keys
  long long rank;          // sel_rank: 1-based rank still to locate
};

// histogram of digit `shift` among rows whose higher digits equal the prefix
__global__ void __launch_bounds__(256) k4_hist(const double* __restrict__ E, int64_t n, int phase, int shift,
                                               const DevStatus* st, unsigned int* hist) {
  __shared__ unsigned int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const unsigned long long key_pref = st->sel_key, idx_pref = st->sel_idx;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = k4_key(E[i]);
    unsigned long long v;
    if (phase == 0) {
      const unsigned long long hm = (shift == 56) ? 0ull : (~0ull << (shift + 8));
      if ((k & hm) != (key_pref & hm)) continue;
      v = k;
    } else {
      if (k != key_pref) continue;
      const unsigned long long hm = (shift == 56) ? 0ull : (~0ull << (shift + 8));
      if (((unsigned long long)i & hm) != (idx_pref & hm)) continue;
      v = (unsigned long long)i;
    }
    atomicAdd(&h[(v >> shift) & 0xff], 1u);
  }
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}

// choose the digit bucket holding the remaining rank; one thread
__global__ void k4_pick(unsigned int* hist, int phase, int shift, DevStatus* st) {
  long long r = st->sel_rank;
  int b = 0;
  for (; b < 256; ++b) {
    if (r <= (long long)hist[b]) break;
    r -= hist[b];
  }
  if (b == 256) b = 255;  // unreachable when rank <= population
  if (phase == 0) st->sel_key |= (unsigned long long)b << shift;
  else st->sel_idx |= (unsigned long long)b << shift;
  st->sel_rank = r;
  for (int i = 0; i < 256; ++i) hist[i] = 0;
}

// collect (key, idx) of every selected row (order fixed later by k4_rank)
__global__ void __launch_bounds__(256) k4_collect(const double* __restrict__ E, int64_t n, DevStatus* st,
                                                  unsigned long long* ck, long long* ci, unsigned char* removed) {
  const unsigned long long K = st->sel_key, T = st->sel_idx;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = k4_key(E[i]);
    const bool take = (k < K) || (k == K && (unsigned long long)i <= T);
    removed[i] = take;
    if (take) {
      const long long slot = atomicAdd((unsigned long long*)&st->take_count, 1ull);
      ck[slot] = k;
      ci[slot] = i;
    }
  }
}

// rank sort of m <= a few thousand candidates and gather into row-major output
__global__ void __launch_bounds__(256) k4_rank_gather(const unsigned long long* ck, const long long* ci, int64_t m,
                                                      Cols cur, int64_t cap, int d, double* out_lo, double* out_hi,
                                                      double* out_E, double* out_I) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = ck[p];
    const long long i = ci[p];
    int64_t pos = 0;
    for (int64_t q = 0; q < m; ++q) pos += (ck[q] < k) || (ck[q] == k && ci[q] < i);
    for (int j = 0; j < d; ++j) {
      out_lo[pos * d + j] = cur.lo[(int64_t)j * cap + i];
      out_hi[pos * d + j] = cur.hi[(int64_t)j * cap + i];
    }
    if (out_E) out_E[pos] = cur.E[i];
    if (out_I) out_I[pos] = cur.I[i];
  }
}

// ---------------------------------------------------------------------------
// K4 on virtual children (donor side of a transfer after classify(split=2)):
// the post-split store's child c is half c & 1 of parent pidx[c >> 1] with
// provisional error 0.5 * E[parent] (ref driver.py:224-226), so siblings
// share a key and sit next to each other, and numpy's stable
// argsort(-error)[:n] (ref distributed.py:381-392) is the first n entries of
// "children 2i, 2i+1 of the survivors i in (key, i) order".  The top
// m = ceil(n/2) survivors are selected from the parents' columns (no child
// rows are built); the chosen children are emitted in that order and their
// virtual indices recorded (sorted, as S[j] = R[j] - j) so the next K1 /
// k3_expand skip them.  Full passes over the survivors: one 12-bit
// histogram and one collection; the rest works on the few candidates that
// share the threshold bucket.

__device__ __forceinline__ unsigned long long k4v_key(const int64_t* __restrict__ pidx, const double* __restrict__ E,
                                                      int64_t i) {
  return k4_key(0.5 * E[pidx[i]]);  // the child's provisional error, exactly as k3_expand writes it
}

__global__ void __launch_bounds__(256) k4v_hist12(const int64_t* __restrict__ pidx, const double* __restrict__ E,
                                                  int64_t ns, unsigned int* hist /* [4096] */) {
  __shared__ unsigned int h[4096];
  for (int b = threadIdx.x; b < 4096; b += blockDim.x) h[b] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&h[k4v_key(pidx, E, i) >> 52], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < 4096; b += blockDim.x)
    if (h[b]) atomicAdd(&hist[b], h[b]);
}

// bucket B holding rank m: sel_key = B << 52, sel_rank = rank inside B,
// take_count / cand_count (pad[1]) reset; the histogram is cleared
__global__ void k4v_pick12(unsigned int* hist, long long m, DevStatus* st) {
  __shared__ unsigned long long part[32];
  const int lane = threadIdx.x;  // one warp; lane owns bins [128*lane, 128*lane + 128)
  unsigned long long c = 0;
  for (int b = 0; b < 128; ++b) c += hist[128 * lane + b];
  part[lane] = c;
  __syncwarp();
  if (lane == 0) {
    long long r = m;
    int w = 0;
    for (; w < 32; ++w) {
      if (r <= (long long)part[w]) break;
      r -= (long long)part[w];
    }
    int b = 128 * w;
    for (; b < 128 * w + 127; ++b) {
      if (r <= (long long)hist[b]) break;
      r -= hist[b];
    }
    st->sel_key = (unsigned long long)b << 52;
    st->sel_idx = 0;
    st->sel_rank = r;
    st->take_count = 0;
    st->pad[1] = 0;
  }
  __syncwarp();
  for (int b = lane; b < 4096; b += 32) hist[b] = 0;
}

// survivors below the bucket are taken; those in it become candidates
// (key, survivor index) for the exact selection; cand overflow -> pad[2]
__global__ void __launch_bounds__(256) k4v_collect(const int64_t* __restrict__ pidx, const double* __restrict__ E,
                                                   int64_t ns, DevStatus* st, unsigned long long* ck, long long* ci,
                                                   unsigned long long* cand_k, long long* cand_i, int64_t cand_cap) {
  const unsigned long long B = st->sel_key >> 52;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = k4v_key(pidx, E, i);
    const unsigned long long b = k >> 52;
    if (b < B) {
      const long long slot = atomicAdd((unsigned long long*)&st->take_count, 1ull);
      ck[slot] = k;
      ci[slot] = i;
    } else if (b == B) {
      const long long slot = atomicAdd((unsigned long long*)&st->pad[1], 1ull);
      if (slot < cand_cap) { cand_k[slot] = k; cand_i[slot] = i; }
      else st->pad[2] = 1;
    }
  }
}

// exact radix select over the candidates: digit `shift` of the key (phase 0)
// or of the survivor index among equal keys (phase 1), like k4_hist
__global__ void __launch_bounds__(256) k4c_hist(const unsigned long long* __restrict__ cand_k,
                                                const long long* __restrict__ cand_i, const DevStatus* st, int phase,
                                                int shift, unsigned int* hist) {
  __shared__ unsigned int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t nc = st->pad[1];
  const unsigned long long key_pref = st->sel_key, idx_pref = st->sel_idx;
  const unsigned long long hm = (shift == 56) ? 0ull : (~0ull << (shift + 8));
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nc; q += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = cand_k[q];
    unsigned long long v;
    if (phase == 0) {
      if ((k & hm) != (key_pref & hm)) continue;
      v = k;
    } else {
      if (k != key_pref) continue;
      v = (unsigned long long)cand_i[q];
      if ((v & hm) != (idx_pref & hm)) continue;
    }
    atomicAdd(&h[(v >> shift) & 0xff], 1u);
  }
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}

__global__ void __launch_bounds__(256) k4c_collect(const unsigned long long* __restrict__ cand_k,
                                                   const long long* __restrict__ cand_i, DevStatus* st,
                                                   unsigned long long* ck, long long* ci) {
  const int64_t nc = st->pad[1];
  const unsigned long long K = st->sel_key, T = st->sel_idx;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nc; q += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = cand_k[q];
    const unsigned long long i = (unsigned long long)cand_i[q];
    if ((k < K) || (k == K && i <= T)) {
      const long long slot = atomicAdd((unsigned long long*)&st->take_count, 1ull);
      ck[slot] = k;
      ci[slot] = (long long)i;
    }
  }
}

// the m selected survivors -> the n children in (key, index) order, written
// row-major; their virtual indices as the sorted skip list S (k1_load_region)
__global__ void __launch_bounds__(256) k4v_gather(const unsigned long long* __restrict__ ck,
                                                  const long long* __restrict__ ci, int64_t m, int64_t n,
                                                  const int64_t* __restrict__ pidx, Cols par, int64_t pcap,
                                                  const signed char* __restrict__ pax, int d, double* out_lo,
                                                  double* out_hi, double* out_E, double* out_I, int64_t* rmS) {
  const bool odd = n & 1;  // the last survivor in key order gives only its lower child
  // survivor index of that last one: the (key, index) maximum
  long long cut = -1;
  if (odd) {
    unsigned long long bk = 0;
    for (int64_t t = 0; t < m; ++t)
      if (cut < 0 || ck[t] > bk || (ck[t] == bk && ci[t] > cut)) { bk = ck[t]; cut = ci[t]; }
  }
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = ck[q];
    const long long i = ci[q];
    int64_t pos = 0, rho = 0;
    for (int64_t t = 0; t < m; ++t) {
      pos += (ck[t] < k) || (ck[t] == k && ci[t] < i);
      rho += ci[t] < i;
    }
    const int64_t p = pidx[i];
    const int ax = pax[p];
    const bool both = !(odd && i == cut);
    for (int s = 0; s < (both ? 2 : 1); ++s) {
      const int64_t row = 2 * pos + s;
      for (int j = 0; j < d; ++j) {
        double l = par.lo[(int64_t)j * pcap + p], u = par.hi[(int64_t)j * pcap + p];
        if (j == ax) {
          const double mid = add_rn(l, mul_rn(0.5, sub_rn(u, l)));  // ref driver.py:211
          if (s) l = mid; else u = mid;
        }
        out_lo[row * d + j] = l;
        out_hi[row * d + j] = u;
      }
      if (out_E) out_E[row] = 0.5 * par.E[p];
      if (out_I) out_I[row] = 0.5 * par.I[p];
    }
    // removed virtual children in index order: 2 per survivor before this
    // one, minus the cut survivor's missing upper child if it comes earlier
    const int64_t j0 = 2 * rho - ((odd && cut >= 0 && cut < i) ? 1 : 0);
    rmS[j0] = 2 * i - j0;
    if (both) rmS[j0 + 1] = 2 * i + 1 - (j0 + 1);
  }
}

// order-preserving removal: count kept rows per tile, then scatter
// (striped tiles, ballot ranks: every access of a warp is 32 consecutive rows)
__global__ void __launch_bounds__(TILE_THREADS) k_keep_count(const unsigned char* removed, int64_t n, int64_t* tile_counts) {
  __shared__ int tot;
  if (threadIdx.x == 0) tot = 0;
  __syncthreads();
  int c = 0;
#pragma unroll
  for (int it = 0; it < TILE_ITEMS; ++it) {
    const int64_t i = (int64_t)blockIdx.x * TILE + it * TILE_THREADS + threadIdx.x;
    c += (i < n && !removed[i]);
  }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&tot, c);
  __syncthreads();
  if (threadIdx.x == 0) tile_counts[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(TILE_THREADS) k_keep_scatter(const unsigned char* removed, int64_t n, Cols cur,
                                                               int64_t cap, Cols nxt, int64_t cap_next, int d,
                                                               const int64_t* tile_offsets) {
  __shared__ TileRanks sm;
  const int64_t tile0 = (int64_t)blockIdx.x * TILE;
  bool flag[TILE_ITEMS];
  int rank[TILE_ITEMS];
#pragma unroll
  for (int it = 0; it < TILE_ITEMS; ++it) {
    const int64_t i = tile0 + it * TILE_THREADS + threadIdx.x;
    flag[it] = i < n && !removed[i];
  }
  tile_rank(flag, rank, sm);
  const int64_t off = tile_offsets[blockIdx.x];
#pragma unroll
  for (int it = 0; it < TILE_ITEMS; ++it) {
    if (!flag[it]) continue;
    const int64_t i = tile0 + it * TILE_THREADS + threadIdx.x;
    const int64_t o = off + rank[it];
    for (int j = 0; j < d; ++j) {
      nxt.lo[(int64_t)j * cap_next + o] = cur.lo[(int64_t)j * cap + i];
      nxt.hi[(int64_t)j * cap_next + o] = cur.hi[(int64_t)j * cap + i];
    }
    nxt.I[o] = cur.I[i];
    nxt.E[o] = cur.E[i];
  }
}

// ---------------------------------------------------------------------------
// K5 / store I/O

// rows (m, d) row-major -> SoA tail at [n0, n0+m); estimates zero
__global__ void k5_append_rows(const double* __restrict__ lo, const double* __restrict__ hi, int64_t m, int d,
                               Cols cur, int64_t cap, int64_t n0, const double* I, const double* E,
                               long long* bad = nullptr) {
  // bad != nullptr: count rows violating lo < hi on some axis (ref
  // regions.py:204-205); the caller rejects the append if any
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    bool ok = true;
    for (int j = 0; j < d; ++j) {
      const double l = lo[r * d + j], h = hi[r * d + j];
      ok &= l < h;
      cur.lo[(int64_t)j * cap + n0 + r] = l;
      cur.hi[(int64_t)j * cap + n0 + r] = h;
    }
    cur.I[n0 + r] = I ? I[r] : 0.0;
    cur.E[n0 + r] = E ? E[r] : 0.0;
    if (bad && !ok) atomicAdd((unsigned long long*)bad, 1ull);
  }
}

// SoA -> row-major (store dump / RegionStore view)
__global__ void k_read_rows(Cols cur, int64_t cap, int64_t n, int d, double* lo, double* hi) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    for (int j = 0; j < d; ++j) {
      lo[r * d + j] = cur.lo[(int64_t)j * cap + r];
      hi[r * d + j] = cur.hi[(int64_t)j * cap + r];
    }
}

__global__ void __launch_bounds__(TILE_THREADS) k3_compact(const unsigned char* __restrict__ flags, int64_t n,
                                                           const int64_t* tile_offsets, int64_t* out_idx) {
  __shared__ TileRanks sm;
  const int64_t tile0 = (int64_t)blockIdx.x * TILE;
  bool flag[TILE_ITEMS];
  int rank[TILE_ITEMS];
#pragma unroll
  for (int it = 0; it < TILE_ITEMS; ++it) {
    const int64_t i = tile0 + it * TILE_THREADS + threadIdx.x;
    flag[it] = i < n && flags[i];
  }
  tile_rank(flag, rank, sm);
  const int64_t off = tile_offsets[blockIdx.x];
#pragma unroll
  for (int it = 0; it < TILE_ITEMS; ++it)
    if (flag[it]) out_idx[off + rank[it]] = tile0 + it * TILE_THREADS + threadIdx.x;
}

// Materialise the virtual children of a fused-split store (worker mode, before
// a take_top / read / append needs real rows): child c = half (c & 1) of
// parent pidx[c >> 1], provisional estimates 0.5 * parent (ref driver.py:206-226).
__global__ void k3_expand(const int64_t* __restrict__ pidx, int64_t nc, Cols par, int64_t pcap,
                          const signed char* __restrict__ pax, Cols kid, int64_t kcap, int d,
                          const int64_t* __restrict__ rmS, int64_t nrm) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = nrm ? c + rm_skip(rmS, nrm, c) : c;  // virtual child of output row c
    const int64_t p = pidx[v >> 1];
    const int ax = pax[p];
    const bool upper = v & 1;
    for (int j = 0; j < d; ++j) {
      double l = par.lo[(int64_t)j * pcap + p], u = par.hi[(int64_t)j * pcap + p];
      if (j == ax) {
        const double mid = add_rn(l, mul_rn(0.5, sub_rn(u, l)));
        if (upper) l = mid; else u = mid;
      }
      kid.lo[(int64_t)j * kcap + c] = l;
      kid.hi[(int64_t)j * kcap + c] = u;
    }
    kid.I[c] = 0.5 * par.I[p];
    kid.E[c] = 0.5 * par.E[p];
  }
}
