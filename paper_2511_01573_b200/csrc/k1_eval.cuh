// K1 gm_eval: fused Genz-Malik rule evaluation, error cascade, fourth-difference
// axis scores, split-axis argmax and non-finite guard for a batch of regions.
//
// Replaces ref pkg/src/hcub/rules.py:495-536 (_apply_symmetric_batch), 428-451
// (estimate_error), 480-492 (_guard_nonfinite) and the argmax of
// ref driver.py:164 / rules.py:454-456.
//
// Work mapping: a group of G lanes (G = 1..32, power of two, chosen per launch
// from n so small stores still fill the machine) owns one region.  Nodes are
// generated on the fly from the five generators; no node table exists.
//  * G = 1 (k1_region_g1, every large store): node coordinates are shared
//    registers (c, c +- lam h) at compile-time positions - an axis loop with
//    selects for the exact on-axis nodes, a switch on the lam4 pair, the low
//    corner bits unrolled - with block barriers between the phases.
//  * G > 1 (k1_region, small stores): nodes strided over the lanes, orbit
//    sums combined with warp shuffles.
// Every node goes through the integrand functor on its own coordinate vector
// with its own fence value (fz, hcub_device.cuh), so no part of one node's
// evaluation is hoisted or shared with another (SURVEY.md 8d integrity rule).
//
// Parity: the 4d+1 on-axis nodes (center, +-lam2 e_k, +-lam3 e_k) are
// evaluated with numpy's operation order (x = c + h*p with separate
// rounding, Fn::exact), and the score arithmetic uses explicit _rn
// intrinsics, so scores and split axes are bit-identical to the reference
// for f2 / product-peak.  Everything else tolerates reassociation.
#pragma once
#include "hcub_device.cuh"
#include "l4_cases.inc"

// k<l pairs ordered by l then k: the first d(d-1)/2 entries are exactly the
// pairs of dimension d, for every d <= HCUB_MAXD.
struct PairTab {
  unsigned char k[HCUB_MAXD * (HCUB_MAXD - 1) / 2];
  unsigned char l[HCUB_MAXD * (HCUB_MAXD - 1) / 2];
};
constexpr PairTab make_pair_tab() {
  PairTab t{};
  int p = 0;
  for (int l = 1; l < HCUB_MAXD; ++l)
    for (int k = 0; k < l; ++k) { t.k[p] = (unsigned char)k; t.l[p] = (unsigned char)l; ++p; }
  return t;
}
__constant__ PairTab c_pairs = make_pair_tab();

// lam4 node e = 4*pair + signs: bit j of the low half marks the two nonzero
// axes (k, l), bit j of the high half the negated ones.  Entries for pairs of
// dimension d come first, so one table serves every d.
struct L4Tab {
  unsigned int m[2 * HCUB_MAXD * (HCUB_MAXD - 1)];
};
constexpr L4Tab make_l4_tab() {
  L4Tab t{};
  int p = 0;
  for (int l = 1; l < HCUB_MAXD; ++l)
    for (int k = 0; k < l; ++k, ++p)
      for (int s = 0; s < 4; ++s) {
        const unsigned on = (1u << k) | (1u << l);
        const unsigned neg = ((unsigned)(s & 1) << k) | ((unsigned)((s >> 1) & 1) << l);
        t.m[4 * p + s] = on | (neg << 16);
      }
  return t;
}
__constant__ L4Tab c_l4 = make_l4_tab();

// c +- o materialised as opaque values: the compiler must not re-derive node
// coordinates as c + select(o, -o) per node (two extra DADD per coordinate)
__device__ __forceinline__ double opaque_add(double a, double b) {
  double r;
  asm("add.rn.f64 %0, %1, %2;" : "=d"(r) : "d"(a), "d"(b));
  return r;
}
__device__ __forceinline__ double opaque_sub(double a, double b) {
  double r;
  asm("sub.rn.f64 %0, %1, %2;" : "=d"(r) : "d"(a), "d"(b));
  return r;
}

struct K1Args {
  const double* lo;   // SoA: lo[j*ld + i]
  const double* hi;
  int64_t ld;         // leading dimension (store capacity or n)
  int64_t n;          // regions
  double* integral;   // [n]
  double* error;      // [n]
  double* vol;        // [n] or null
  signed char* axis;  // [n] or null
  int64_t* axis64;    // [n] or null (apply_rule_batch surface)
  double* scores;     // row-major [n][d] or null
  double* aext;       // [n] extent of the split axis (K3 width guard) or null
  // Fused split (single-worker loop): region r is child (r & 1) of parent
  // pidx[r >> 1] of the previous store (plo/phi, leading dim pld, split axes
  // pax); the child box is derived on the fly and materialised into clo/chi
  // (leading dim ld).  pidx == null: regions are read from lo/hi.
  const int64_t* pidx;
  const double* plo;
  const double* phi;
  int64_t pld;
  const signed char* pax;
  double* clo;
  double* chi;
  // virtual children removed by take_top (donor side of a transfer): S[j] =
  // R[j] - j for the sorted removed virtual-child indices R; output row r is
  // virtual child r + #{j : S[j] <= r} (null / 0: none removed)
  const int64_t* rmS;
  int64_t nrm;
  unsigned long long zero;  // always 0 at run time; opaque to the compiler (see node_copy)
  // Fused K2: exact sums of the integral / error column accumulated in the
  // epilogue into per-SM shards (kacc[2*s] = integral, kacc[2*s+1] = error,
  // s = SM id % K1_SHARDS); null = the caller runs k2_reduce instead.
  SAcc* kacc;
  int log2g;          // lanes per region = 1 << log2g
};

// A per-node private copy of a shared coordinate: XOR with a run-time zero
// that differs per node and per iteration, so neither NVVM (hoisting) nor
// ptxas (CSE) can merge the integrand work of two nodes that happen to share
// a coordinate value.  Costs two integer LOP3s, no FP64 work.
__device__ __forceinline__ double node_copy(double v, unsigned long long z) {
  return __longlong_as_double(__double_as_longlong(v) ^ (long long)z);
}

// numpy.argmax ordering: the first NaN wins, otherwise the first maximum.
__device__ __forceinline__ bool score_better(double s, int k, double bs, int bk) {
  if (bk < 0) return true;
  if (k < 0) return false;
  bool sn = isnan(s), bn = isnan(bs);
  if (sn || bn) return sn && (!bn || k < bk);
  return s > bs || (s == bs && k < bk);
}

#ifndef K1_BLOCK
#define K1_BLOCK 128
#endif
// Threads per block of k1_gm_eval at dimension D.  Larger blocks put more of
// an SM's warps behind one phase barrier (K1_SYNC), so fewer distinct phases
// (switch cases, corner loop) compete for the instruction cache at a time.
#ifndef K1_B5
#define K1_B5 256  // d <= 5 (measured f2 d=5: 128 -> 5.43e11, 256 -> 5.51e11, 512 -> 5.41e11)
#endif
#ifndef K1_B8
#define K1_B8 128  // 6 <= d <= 8 (f2 d=8: 128 -> 5.26e11, 256 -> 5.15e11, 384 -> 5.11e11)
#endif
#define K1_BLOCK_OF(D) ((D) <= 5 ? K1_B5 : (D) <= 8 ? K1_B8 : K1_BLOCK)
// Build-time tuning knobs (measured alternatives in DESIGN.md section 4):
// lam4 nodes per switch case (4 = one pair per case)
#ifndef K1_L4_NODES
#define K1_L4_NODES 4
#endif
// K1_AXIS_SWITCH: on-axis nodes through a switch on the axis (compile-time
// positions, 4 nodes per case) instead of run-time selects
#ifndef K1_AXIS_SWITCH
#define K1_AXIS_SWITCH 0
#endif
#define K1_SHARDS 160  // >= SM count: one exact-sum shard per SM
// axes per iteration of the exact on-axis loop (4 exact nodes each)
#ifndef K1_AXIS_UNROLL
#define K1_AXIS_UNROLL 2  // measured: 1 -> 5.22e11, 2 -> 5.26e11, 4 -> 4.90e11 (f2 d=8)
#endif
// corner-index bits unrolled per iteration of the corner loop (16 nodes)
#ifndef K1_CORNER_BITS
#define K1_CORNER_BITS 4
#endif
// d <= 5: the whole axis loop and all 2^d corners straight-line (small code;
// measured configs[1] f2 d=5 K1 39.88 ms -> 39.03 ms with the axis loop
// unrolled, 38.83 ms with the corners too, profiles/r02_k1d5_variants.txt)
#ifndef K1_AXIS_UNROLL_OF
#define K1_AXIS_UNROLL_OF(D) ((D) <= 5 ? (D) : K1_AXIS_UNROLL)
#endif
#ifndef K1_CORNER_BITS_OF
#define K1_CORNER_BITS_OF(D) ((D) <= 5 ? (D) : K1_CORNER_BITS)
#endif
// K1_SYNC: barrier between the phases of a region (one-region-per-lane path)
// so the block's warps run the same code at the same time: the lam4 switch is
// larger than the instruction cache, and warps drifting through different
// cases stall on instruction fetch (measured: +5 % K1 throughput)
#ifndef K1_SYNC
#define K1_SYNC(D) 1
#endif
#define K1_PHASE_SYNC() \
  do {                   \
    if (K1_SYNC(D)) __syncthreads(); \
  } while (0)
// Resident 128-thread blocks per SM: more warps hide the FP64/MUFU latency
// chains of the one-lane path better than the extra registers help (f2 d=8:
// 4 blocks/128 regs 5.05e11, 5/96 5.20e11, 6/80 5.26e11, 7/72 5.26e11,
// 8/64 5.20e11 evaluations/s; d = 5: 6 blocks 5.29e11, 8 blocks 5.37e11);
// large d needs the registers.
// d <= 5 (straight-line code): 5 x 256 threads at 48 registers beat 4 x 256 at
// 64 despite the spills (configs[1] K1 38.97 -> 38.68 ms; 6 blocks at 40
// registers 39.58 ms); the degree-9 kernel at d = 5 prefers 4 (4.63 vs 4.68 ms).
#ifndef K1_MIN_BLOCKS
#define K1_MIN_BLOCKS(D) ((D) <= 5 ? 1280 / K1_B5 : (D) <= 8 ? 768 / K1_B8 : (D) <= 10 ? 5 : 4)
#endif
// per integrand: f3 at d = 10 (BASELINE configs[3]; one FMA per coordinate,
// cheap nodes) runs best with 6 blocks at 80 registers (K1 1052.8 -> 1038 ms),
// f2 at d = 10 with 5 (6: +0.2 %, 4: +3.7 %)
#define K1_MINB(D, FN) (((FN) == FN_F3 && (D) == 10) ? 6 : K1_MIN_BLOCKS(D))
#ifndef K9_MIN_BLOCKS
#define K9_MIN_BLOCKS(D) ((D) <= 5 ? 1024 / K1_B5 : K1_MIN_BLOCKS(D))
#endif

// Region r's box (materialised, or derived from its parent in the fused-split
// loop and then materialised by `writer`): centers, half widths, extents and
// volume with numpy's operation order (ref rules.py:497-500, driver.py:211-221).
template <int D>
__device__ __forceinline__ void k1_load_region(const K1Args& a, const int64_t r, const bool writer, double (&c)[D],
                                               double (&h)[D], double (&ext)[D], double& vol) {
  int64_t par = 0;
  int pax = -1, upper = 0;
  if (a.pidx) {
    const int64_t v = a.nrm ? r + rm_skip(a.rmS, a.nrm, r) : r;
    par = a.pidx[v >> 1];
    pax = a.pax[par];
    upper = (int)(v & 1);
  }
  vol = 1.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    double l, u;
    if (a.pidx) {
      l = a.plo[j * a.pld + par];
      u = a.phi[j * a.pld + par];
      if (j == pax) {  // mid = lo + 0.5*(hi-lo); [2i] lower, [2i+1] upper half
        const double mid = add_rn(l, mul_rn(0.5, sub_rn(u, l)));
        if (upper) l = mid; else u = mid;
      }
      if (writer) {
        a.clo[j * a.ld + r] = l;
        a.chi[j * a.ld + r] = u;
      }
    } else {
      l = a.lo[j * a.ld + r];
      u = a.hi[j * a.ld + r];
    }
    ext[j] = sub_rn(u, l);
    h[j] = mul_rn(0.5, ext[j]);
    c[j] = add_rn(l, h[j]);
    vol = (j == 0) ? ext[0] : mul_rn(vol, ext[j]);
  }
}

// Error cascade (ref rules.py:443-451) with numpy's NaN semantics.
__device__ __forceinline__ double cascade_error(double main, double emb, double low, double lowest) {
  const double e1 = fabs(main - emb), e2 = fabs(emb - low), e3 = fabs(low - lowest);
  double err = e1;
  if (e2 > 0.0 && e3 > 0.0) {
    const double r1 = e1 / e2, r2 = e2 / e3;
    const double rr = (isnan(r1) || isnan(r2)) ? r1 + r2 : fmax(r1, r2);
    const double sc = (rr >= 1.0) ? 10.0 : (isnan(rr) ? rr : fmin(fmax(4.0 * rr, 0.05), 1.0));
    err = sc * e1;
  }
  return err;
}

// Fused K2 (ref driver.py:166-167): the region's integral and error go into
// the SM's shard of the exact superaccumulator; lanes of a warp with the same
// slot window are combined by shuffles first (all 32 lanes must call).
__device__ __forceinline__ void k1_accumulate(const K1Args& a, bool valid, double integ, double err) {
  if (!a.kacc) return;
  unsigned smid;
  asm("mov.u32 %0, %%smid;" : "=r"(smid));
  SAcc* sh = a.kacc + 2 * (smid % K1_SHARDS);
  sa_warp_add(sh, integ, valid);
  sa_warp_add(sh + 1, err, valid);
}

// Non-finite guard, rare path (ref rules.py:480-492): a non-finite node value
// makes some orbit sum non-finite, so finite sums prove every node was finite.
// Otherwise re-walk every node with explicit checks (sums may also have
// overflowed from finite values, which the reference does not guard).  Any
// non-finite node: integral 0, error 1e30*vol, widest axis, scores = extents.
template <int D, int FN>
__device__ __forceinline__ void k1_nonfinite(const K1Args& a, const RuleC& rc, const FnParams& fp, const int64_t r,
                                          double& integ, double& err, int& axis, double& e_ax) {
  using F = Fn<FN, D>;
  double c[D], h[D], ext[D], vol;
  k1_load_region<D>(a, r, false, c, h, ext, vol);
  bool bad = !isfinite(F::exact(c, fp));
  for (int k = 0; k < D && !bad; ++k)
    for (int s = 0; s < 4 && !bad; ++s) {
      const double lam = (s < 2) ? rc.lam2 : rc.lam3;
      double x[D];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const double off = mul_rn(h[j], lam);
        x[j] = (j != k) ? c[j] : ((s & 1) ? sub_rn(c[j], off) : add_rn(c[j], off));
      }
      bad = !isfinite(F::exact(x, fp));
    }
  for (int e = 0; e < 2 * D * (D - 1) && !bad; ++e) {
    const int p = e >> 2;
    const int k = c_pairs.k[p], l = c_pairs.l[p];
    double x[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double o = rc.lam4 * h[j];
      const bool neg = (j == k) ? (e & 1) : ((e >> 1) & 1);
      x[j] = (j == k || j == l) ? (neg ? c[j] - o : c[j] + o) : c[j];
    }
    bad = !isfinite(F::fast(x, fp));
  }
  for (unsigned m = 0; m < (1u << D) && !bad; ++m) {
    double x[D];
#pragma unroll
    for (int j = 0; j < D; ++j) x[j] = c[j] + (((m >> j) & 1u) ? -1.0 : 1.0) * (rc.lam5 * h[j]);
    bad = !isfinite(F::fast(x, fp));
  }
  if (!bad) return;
  integ = 0.0;
  err = 1e30 * vol;  // NONFINITE_ERROR_SCALE, ref rules.py:61
  int bk = 0;
  double bv = ext[0];
#pragma unroll
  for (int j = 1; j < D; ++j)
    if (ext[j] > bv) { bv = ext[j]; bk = j; }
  axis = bk;
  e_ax = bv;
  if (a.scores)
#pragma unroll
    for (int j = 0; j < D; ++j) a.scores[r * D + j] = ext[j];
}

// One region per group of G lanes; lane 0 of the group writes the outputs
// and feeds the exact-sum windows.
template <int D, int FN>
__device__ __forceinline__ void k1_region(const K1Args& a, const RuleC& rc, const FnParams& fp, const int64_t rid,
                                          const int g, const int G, double* xq, SAcc* sacc) {
  constexpr int KB = K1_BLOCK_OF(D);  // xq stride: one column per thread of the block
  using F = Fn<FN, D>;
  const bool live = rid < a.n;
  const int64_t r = live ? rid : a.n - 1;  // idle lanes shadow a real region (shuffles stay full-warp)
  const unsigned zs = (unsigned)a.zero;

  // geometry: exactly as numpy (ref rules.py:497-500)
  double c[D], h[D], ext[D];
  double vol;
  k1_load_region<D>(a, r, g == 0 && live, c, h, ext, vol);
  const double scale = __ddiv_rn(vol, rc.twod);

  // ---- on-axis nodes: exact path -------------------------------------------
  // The 4d on-axis coordinates c_k +- h_k*lam (numpy order: product, then sum)
  // are staged per thread in shared memory so each node fetches its moving
  // coordinate with one load; the other coordinates are the center.
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if ((k & (G - 1)) != g) continue;  // only the lane that owns axis k needs it
    const double o2 = mul_rn(h[k], rc.lam2), o3 = mul_rn(h[k], rc.lam3);
    xq[(4 * k + 0) * KB] = add_rn(c[k], o2);
    xq[(4 * k + 1) * KB] = sub_rn(c[k], o2);
    xq[(4 * k + 2) * KB] = add_rn(c[k], o3);
    xq[(4 * k + 3) * KB] = sub_rn(c[k], o3);
  }
  const double fc = F::exact(c, fp);
  bool safe = false;
  if constexpr (HasSafe<F>::value) safe = F::safe_range(c, h, rc.lam3, fp);
  safe = __all_sync(0xffffffffu, safe);  // warp-uniform choice of the exact path
  double S2 = 0.0, S3 = 0.0;
  int best_k = -1;
  double best_s = 0.0;
  {
    const int naxes = (D - g + G - 1) / G;  // axes k = g, g+G, ...
    double vin = 0.0;
    const double two_fc = 2.0 * fc;
    // two independent nodes per iteration (c_k + off, c_k - off); each gets
    // its own opaque copy of the center so they share no work
#pragma unroll 1
    for (int q = 0; q < 2 * naxes; ++q) {
      const int k = g + (q >> 1) * G;
      const int s = q & 1;  // 0: lam2 pair, 1: lam3 pair
      const double xp = xq[(4 * k + 2 * s) * KB];
      const double xm = xq[(4 * k + 2 * s + 1) * KB];
      const unsigned onehot = 1u << k;
      const unsigned long long z1 = (unsigned long long)q * a.zero, z2 = z1 + a.zero;
      double x1[D], x2[D];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const bool mv = (onehot >> j) & 1u;
        x1[j] = mv ? xp : node_copy(c[j], z1);
        x2[j] = mv ? xm : node_copy(c[j], z2);
      }
      double v1, v2;
      if constexpr (HasSafe<F>::value) {
        if (safe) { v1 = F::exact_safe(x1, fp); v2 = F::exact_safe(x2, fp); }
        else { v1 = F::exact(x1, fp); v2 = F::exact(x2, fp); }
      } else {
        v1 = F::exact(x1, fp);
        v2 = F::exact(x2, fp);
      }
      const double v = add_rn(v1, v2);  // vals[plus] + vals[minus]
      if (s == 0) {
        vin = v;
      } else {
        // ref rules.py:520-524: |(v_in - 2fc) - ratio*(v_out - 2fc)|
        const double sc = fabs(sub_rn(sub_rn(vin, two_fc), mul_rn(rc.ratio, sub_rn(v, two_fc))));
        if (score_better(sc, k, best_s, best_k)) { best_s = sc; best_k = k; }
        if (a.scores && live) a.scores[r * D + k] = sc;
        S2 += vin;
        S3 += v;
      }
    }
  }

  // ---- lam4 orbit: 2d(d-1) nodes, fast path --------------------------------
  double S4 = 0.0;
  {
    double p4[D], m4[D];
#pragma unroll
    for (int j = 0; j < D; ++j) { const double o = rc.lam4 * h[j]; p4[j] = opaque_add(c[j], o); m4[j] = opaque_sub(c[j], o); }
    const int n4 = 2 * D * (D - 1);
#pragma unroll 1
    for (int e = g; e < n4; e += G) {
      const unsigned msk = c_l4.m[e];
      const unsigned on = msk & 0xffffu, neg = msk >> 16;
      double x[D];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const double pm = ((neg >> j) & 1u) ? m4[j] : p4[j];
        x[j] = ((on >> j) & 1u) ? pm : c[j];
      }
      S4 += F::fast(x, fp, (unsigned)e * zs);
    }
  }

  // ---- lam5 orbit: 2^d corner nodes, fast path -----------------------------
  double S5 = 0.0;
  {
    double p5[D], m5[D];
#pragma unroll
    for (int j = 0; j < D; ++j) { const double o = rc.lam5 * h[j]; p5[j] = opaque_add(c[j], o); m5[j] = opaque_sub(c[j], o); }
    // corner m and its complement share no coordinate: two independent
    // nodes per iteration
    const unsigned nh = 1u << (D - 1);
#pragma unroll 1
    for (unsigned m = g; m < nh; m += G) {
      double x1[D], x2[D];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const bool bit = (m >> j) & 1u;
        x1[j] = bit ? m5[j] : p5[j];
        x2[j] = bit ? p5[j] : m5[j];
      }
      S5 += F::fast(x1, fp, (2u * m + 1u) * zs) + F::fast(x2, fp, (2u * m + 2u) * zs);
    }
  }

  // ---- combine the G lanes of a region -------------------------------------
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    if (o >= G) break;
    S2 += __shfl_xor_sync(0xffffffffu, S2, o);
    S3 += __shfl_xor_sync(0xffffffffu, S3, o);
    S4 += __shfl_xor_sync(0xffffffffu, S4, o);
    S5 += __shfl_xor_sync(0xffffffffu, S5, o);
    const double os = __shfl_xor_sync(0xffffffffu, best_s, o);
    const int ok = __shfl_xor_sync(0xffffffffu, best_k, o);
    if (score_better(os, ok, best_s, best_k)) { best_s = os; best_k = ok; }
  }
  double integ = 0.0, err = 0.0;
  if (g == 0 && live) {
    const double main = (rc.w[0] * fc + rc.w[1] * S2 + rc.w[2] * S3 + rc.w[3] * S4 + rc.w[4] * S5) * scale;
    const double emb = (rc.we[0] * fc + rc.we[1] * S2 + rc.we[2] * S3 + rc.we[3] * S4 + rc.we[4] * S5) * scale;
    // degree-3 / degree-1 companions (ref rules.py:525-526)
    const double low = (rc.null_center * fc + rc.null_axis * S3) * scale;
    const double lowest = (rc.twod * fc) * scale;
    err = cascade_error(main, emb, low, lowest);
    integ = main;
    int axis = best_k;
    double e_ax = ext[0];
#pragma unroll
    for (int j = 1; j < D; ++j)
      if (j == axis) e_ax = ext[j];
    // non-finite guard (ref rules.py:480-492)
    if (!(isfinite(fc) && isfinite(S2) && isfinite(S3) && isfinite(S4) && isfinite(S5)))
      k1_nonfinite<D, FN>(a, rc, fp, r, integ, err, axis, e_ax);
    a.integral[r] = integ;
    a.error[r] = err;
    if (a.vol) a.vol[r] = vol;
    if (a.axis) a.axis[r] = (signed char)axis;
    if (a.axis64) a.axis64[r] = axis;
    if (a.aext) a.aext[r] = e_ax;
  }
  k1_accumulate(a, g == 0 && live, integ, err);
  (void)sacc;
}

template <class F, bool SAFE, int D>
__device__ __forceinline__ double exact_eval(const double (&x)[D], const FnParams& fp, unsigned z) {
  if constexpr (SAFE) return F::exact_safe(x, fp, z);
  else return F::exact(x, fp, z);
}

// On-axis nodes of one region, one lane per region (G = 1): for each axis k
// the four nodes c +- lam2 h_k e_k, c +- lam3 h_k e_k on the exact path
// (numpy order: x = c + h*p, product then sum), then the fourth-difference
// score (ref rules.py:519-524).  The axis is a run-time loop index and the
// moving coordinate is placed by selects, which keeps the code small (these
// nodes are FP64-heavy, so the selects cost no FP64 throughput).
#if K1_AXIS_SWITCH
// Switch over the axis k (compile-time positions inside each case).
#define HCUB_AX_CASES(D, BODY)                                   \
  case 0: if constexpr (0 < D) { BODY(0); } break;               \
  case 1: if constexpr (1 < D) { BODY(1); } break;               \
  case 2: if constexpr (2 < D) { BODY(2); } break;               \
  case 3: if constexpr (3 < D) { BODY(3); } break;               \
  case 4: if constexpr (4 < D) { BODY(4); } break;               \
  case 5: if constexpr (5 < D) { BODY(5); } break;               \
  case 6: if constexpr (6 < D) { BODY(6); } break;               \
  case 7: if constexpr (7 < D) { BODY(7); } break;               \
  case 8: if constexpr (8 < D) { BODY(8); } break;               \
  case 9: if constexpr (9 < D) { BODY(9); } break;               \
  case 10: if constexpr (10 < D) { BODY(10); } break;            \
  case 11: if constexpr (11 < D) { BODY(11); } break;            \
  case 12: if constexpr (12 < D) { BODY(12); } break;            \
  default: break;

template <int D, int FN, bool SAFE>
__device__ __forceinline__ void k1_axes_g1(const RuleC& rc, const FnParams& fp, const double (&c)[D],
                                           const double (&h)[D], const double fc, unsigned& zc, const unsigned zs,
                                           double& S2, double& S3, double& best_s, int& best_k, double* srow) {
  using F = Fn<FN, D>;
  const double two_fc = 2.0 * fc;
#pragma unroll 1
  for (int k = 0; k < D; ++k) {
    double vin = 0.0, vout = 0.0;
    switch (k) {
#define HCUB_AX_BODY(K)                                                                       \
  {                                                                                           \
    double x[D];                                                                              \
    _Pragma("unroll") for (int j = 0; j < D; ++j) x[j] = c[j];                                \
    const double o2 = mul_rn(h[K], rc.lam2), o3 = mul_rn(h[K], rc.lam3);                      \
    double v[4];                                                                              \
    _Pragma("unroll") for (int s = 0; s < 4; ++s) {                                           \
      const double o = (s < 2) ? o2 : o3;                                                     \
      x[K] = (s & 1) ? sub_rn(c[K], o) : add_rn(c[K], o);                                     \
      zc += zs;                                                                               \
      v[s] = exact_eval<F, SAFE>(x, fp, zc);                                                  \
    }                                                                                         \
    vin = add_rn(v[0], v[1]);                                                                 \
    vout = add_rn(v[2], v[3]);                                                                \
  }
      HCUB_AX_CASES(D, HCUB_AX_BODY)
#undef HCUB_AX_BODY
    }
    // ref rules.py:520-524: |(v_in - 2fc) - ratio*(v_out - 2fc)|
    const double sc = fabs(sub_rn(sub_rn(vin, two_fc), mul_rn(rc.ratio, sub_rn(vout, two_fc))));
    if (score_better(sc, k, best_s, best_k)) { best_s = sc; best_k = k; }
    if (srow) srow[k] = sc;
    S2 += vin;
    S3 += vout;
  }
}
#else
template <int D, int FN, bool SAFE>
__device__ __forceinline__ void k1_axes_g1(const RuleC& rc, const FnParams& fp, const double (&c)[D],
                                           const double (&h)[D], const double fc, unsigned& zc, const unsigned zs,
                                           double& S2, double& S3, double& best_s, int& best_k, double* srow) {
  using F = Fn<FN, D>;
  const double two_fc = 2.0 * fc;
  constexpr int kAxisUnroll = K1_AXIS_UNROLL_OF(D);
#pragma unroll (kAxisUnroll)
  for (int k = 0; k < D; ++k) {
    double ck = c[0], hk = h[0];
#pragma unroll
    for (int j = 1; j < D; ++j)
      if (j == k) { ck = c[j]; hk = h[j]; }
    const double o2 = mul_rn(hk, rc.lam2), o3 = mul_rn(hk, rc.lam3);
    double v[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const double o = (s < 2) ? o2 : o3;
      const double xk = (s & 1) ? sub_rn(ck, o) : add_rn(ck, o);
      double x[D];
#pragma unroll
      for (int j = 0; j < D; ++j) x[j] = (j == k) ? xk : c[j];
      zc += zs;
      v[s] = exact_eval<F, SAFE>(x, fp, zc);
    }
    const double vin = add_rn(v[0], v[1]);  // vals[plus] + vals[minus]
    const double vout = add_rn(v[2], v[3]);
    // ref rules.py:520-524: |(v_in - 2fc) - ratio*(v_out - 2fc)|
    const double sc = fabs(sub_rn(sub_rn(vin, two_fc), mul_rn(rc.ratio, sub_rn(vout, two_fc))));
    if (score_better(sc, k, best_s, best_k)) { best_s = sc; best_k = k; }
    if (srow) srow[k] = sc;
    S2 += vin;
    S3 += vout;
  }
}

#endif

// One region per lane.  Node coordinates are shared register values (center,
// c +- lam h per axis); every node's integrand evaluation starts from a
// constant fenced with its own run-time zero (fz), so the nodes share no
// arithmetic while the generator spends no per-coordinate selects or copies.
template <int D, int FN>
__device__ __forceinline__ void k1_region_g1_body(const K1Args& a, const RuleC& rc, const FnParams& fp,
                                                  const int64_t r, const bool live, const double (&c)[D],
                                                  const double (&h)[D], const double (&ext)[D], const double vol) {
  using F = Fn<FN, D>;
  const unsigned zs = (unsigned)a.zero;
  unsigned zc = zs;
  const double scale = __ddiv_rn(vol, rc.twod);

  // ---- center + on-axis nodes: exact path ----------------------------------
  const double fc = F::exact(c, fp, zc);
  double S2 = 0.0, S3 = 0.0, best_s = 0.0;
  int best_k = -1;
  double* srow = (a.scores && live) ? a.scores + r * D : nullptr;
  bool safe = false;
  if constexpr (HasSafe<F>::value) safe = F::safe_range(c, h, rc.lam3, fp);
  if (__all_sync(0xffffffffu, safe)) {  // warp-uniform choice
    if constexpr (HasSafe<F>::value) k1_axes_g1<D, FN, true>(rc, fp, c, h, fc, zc, zs, S2, S3, best_s, best_k, srow);
  } else {
    k1_axes_g1<D, FN, false>(rc, fp, c, h, fc, zc, zs, S2, S3, best_s, best_k, srow);
  }
  double e_ax = ext[0];
#pragma unroll
  for (int j = 1; j < D; ++j)
    if (j == best_k) e_ax = ext[j];
  K1_PHASE_SYNC();

  // ---- lam4 orbit: 2d(d-1) nodes, one per case of a switch on (k, l) -------
  double S4 = 0.0;
  {
    double p4[D], m4[D];
#pragma unroll
    for (int j = 0; j < D; ++j) { const double o = rc.lam4 * h[j]; p4[j] = c[j] + o; m4[j] = c[j] - o; }
    // node e = 4*pair + signs; K1_L4_NODES nodes per case of the switch
    // (fewer: smaller code; more: more independent work per case)
    constexpr int NPC = K1_L4_NODES;
#pragma unroll 1
    for (int e = 0; e < 2 * D * (D - 1); e += NPC) {
      switch (e >> 2) {
#define HCUB_L4G1_BODY(K, L)                                       \
  {                                                                \
    double x[D];                                                   \
    _Pragma("unroll") for (int j = 0; j < D; ++j) x[j] = c[j];     \
    _Pragma("unroll") for (int q = 0; q < NPC; ++q) {              \
      const int sg = (e + q) & 3;                                  \
      x[K] = (sg & 1) ? m4[K] : p4[K];                             \
      x[L] = (sg & 2) ? m4[L] : p4[L];                             \
      zc += zs;                                                    \
      S4 += F::fast(x, fp, zc);                                    \
    }                                                              \
  }
        HCUB_L4_CASES(D, HCUB_L4G1_BODY)
#undef HCUB_L4G1_BODY
      }
    }
  }
  K1_PHASE_SYNC();

  // ---- lam5 orbit: 2^d corners; low KLO bits unrolled, high bits looped ----
  double S5a = 0.0, S5b = 0.0;
  {
    double p5[D], m5[D];
#pragma unroll
    for (int j = 0; j < D; ++j) { const double o = rc.lam5 * h[j]; p5[j] = c[j] + o; m5[j] = c[j] - o; }
    constexpr int KLO = D < K1_CORNER_BITS_OF(D) ? D : K1_CORNER_BITS_OF(D);
    constexpr unsigned NHI = 1u << (D - KLO);
#pragma unroll 1
    for (unsigned mh = 0; mh < NHI; ++mh) {
      double xh[D];
#pragma unroll
      for (int j = KLO; j < D; ++j) xh[j] = ((mh >> (j - KLO)) & 1u) ? m5[j] : p5[j];
#pragma unroll
      for (unsigned ml = 0; ml < (1u << KLO); ++ml) {
        double x[D];
#pragma unroll
        for (int j = 0; j < D; ++j) x[j] = (j < KLO) ? (((ml >> j) & 1u) ? m5[j] : p5[j]) : xh[j];
        zc += zs;
        if (ml & 1u) S5b += F::fast(x, fp, zc);
        else S5a += F::fast(x, fp, zc);
      }
    }
  }
  const double S5 = S5a + S5b;
  double integ = 0.0, err = 0.0;
  if (live) {
    const double main = (rc.w[0] * fc + rc.w[1] * S2 + rc.w[2] * S3 + rc.w[3] * S4 + rc.w[4] * S5) * scale;
    const double emb = (rc.we[0] * fc + rc.we[1] * S2 + rc.we[2] * S3 + rc.we[3] * S4 + rc.we[4] * S5) * scale;
    const double low = (rc.null_center * fc + rc.null_axis * S3) * scale;  // ref rules.py:525-526
    const double lowest = (rc.twod * fc) * scale;
    err = cascade_error(main, emb, low, lowest);
    integ = main;
    int axis = best_k;
    if (!(isfinite(fc) && isfinite(S2) && isfinite(S3) && isfinite(S4) && isfinite(S5)))
      k1_nonfinite<D, FN>(a, rc, fp, r, integ, err, axis, e_ax);
    a.integral[r] = integ;
    a.error[r] = err;
    if (a.vol) a.vol[r] = vol;
    if (a.axis) a.axis[r] = (signed char)axis;
    if (a.axis64) a.axis64[r] = axis;
    if (a.aext) a.aext[r] = e_ax;
  }
  k1_accumulate(a, live, integ, err);
}

template <int D, int FN>
__device__ __forceinline__ void k1_region_g1(const K1Args& a, const RuleC& rc, const FnParams& fp, const int64_t rid) {
  const bool live = rid < a.n;
  const int64_t r = live ? rid : a.n - 1;
  double c[D], h[D], ext[D], vol;
  k1_load_region<D>(a, r, live, c, h, ext, vol);
  k1_region_g1_body<D, FN>(a, rc, fp, r, live, c, h, ext, vol);
}

// One region per group of G lanes (grid covers n << log2g threads).
template <int D, int FN>
__global__ void __launch_bounds__(K1_BLOCK_OF(D), K1_MINB(D, FN)) k1_gm_eval(K1Args a, RuleC rc, FnParams fp) {
  extern __shared__ double k1_smem[];
  const int G = 1 << a.log2g;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (G == 1) k1_region_g1<D, FN>(a, rc, fp, t);
  else k1_region<D, FN>(a, rc, fp, t >> a.log2g, (int)(t & (G - 1)), G, k1_smem + threadIdx.x, nullptr);
}

// Plain point evaluation (BenchmarkIntegrand.__call__ surface), fast path.
template <int D, int FN>
__global__ void k_eval_points(const double* pts, int64_t m, double* out, FnParams fp) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double x[D];
#pragma unroll
  for (int j = 0; j < D; ++j) x[j] = pts[i * D + j];
  out[i] = Fn<FN, D>::exact(x, fp);
}
