// K1 for the degree-9 fully symmetric family (rule9.py: DCUHRE D09HRE node
// set, embedded degree 7) in generator form - the table of
// parse_rule_table(gm9_rule_text(d)) evaluated without a node table, the
// way k1_gm_eval evaluates the degree-7 rule.  Same results as k1_table_eval
// on that table (ref rules.py:495-536 semantics: scores from the two
// smallest on-axis orbits, here g2 = lam_in and g0 = lam_out, on the exact
// path; degree-3 companion on {center, g0 axis}).
//
// One region per lane.  Orbits (rule9.py order):
//   center | axis g0 | axis g1 | axis g2 | axis g3 | (g1,g1) pairs |
//   (g1,g2) ordered pairs | (g1,g1,g1) triples | g0 corners
// Exact path: center, +-g2, +-g0 on every axis (k1_axes_g1 with lam2 := g2,
// lam3 := g0).  Fast path: the rest, every node through the functor on its
// own coordinate vector with its own fence (no cross-node sharing, SURVEY.md
// 8d).  Coordinates: the g1/g3 axis nodes by selects (4d nodes), pairs at
// compile-time positions (a switch case per pair, 12 nodes each), triples by
// pair case + a run-time third axis placed with selects over the axes above
// the pair, corners as in k1_gm_eval.
#pragma once
#include "k1_eval.cuh"

// sign loops of the pair / triple switch cases, unrolled at d <= 5 and
// partly rolled above: code per case vs the instruction cache, which the
// switches far exceed at d = 8 (measured in profiles/r02_gm9_generator_variants.txt:
// d = 8 3.5e11 -> 4.1e11 evaluations/s rolled, d = 5 4.35e11 unrolled vs 4.0e11)
#ifndef K9_PU6
#define K9_PU6 1
#endif
#ifndef K9_TU6
#define K9_TU6 2
#endif

enum { O9_CENTER = 0, O9_A0, O9_A1, O9_A2, O9_A3, O9_P11, O9_P12, O9_T111, O9_CORNER, O9_N };

struct Rule9C {
  double g[4];                  // generator magnitudes g0..g3 (g_i = sqrt(lam_i))
  double w[O9_N], we[O9_N];     // per-node main / embedded weight of each orbit (x 2^d)
  double ratio, null_center, null_axis, twod;  // (g2/g0)^2, degree-3 companion, 2^d
};

// k<l<m triples ordered by m, then l, then k: the first C(d,3) entries are
// exactly the triples of dimension d
struct TripleTab {
  unsigned char k[286], l[286], m[286];  // C(13,3)
};
constexpr TripleTab make_triple_tab() {
  TripleTab t{};
  int p = 0;
  for (int m = 2; m < HCUB_MAXD; ++m)
    for (int l = 1; l < m; ++l)
      for (int k = 0; k < l; ++k) { t.k[p] = (unsigned char)k; t.l[p] = (unsigned char)l; t.m[p] = (unsigned char)m; ++p; }
  return t;
}
__constant__ TripleTab c_triples = make_triple_tab();

// x = c with up to three coordinates replaced (run-time positions, selects)
template <int D>
__device__ __forceinline__ void place3(double (&x)[D], const double (&c)[D], int k, double vk, int l, double vl,
                                       int m, double vm) {
#pragma unroll
  for (int j = 0; j < D; ++j) x[j] = (j == k) ? vk : (j == l) ? vl : (j == m) ? vm : c[j];
}
// c[k] for a run-time k (select chain: no local-memory indexing)
template <int D>
__device__ __forceinline__ double pick(const double (&v)[D], int k) {
  double r = v[0];
#pragma unroll
  for (int j = 1; j < D; ++j)
    if (j == k) r = v[j];
  return r;
}

// The fast-path orbits of one region, weighted-sum mode (CHECK = false) or
// the rare non-finite re-walk (CHECK = true: returns whether any node value
// is non-finite; its pairs and triples use run-time selects - small code).
template <int D, int FN, bool CHECK>
__device__ __forceinline__ bool gm9_fast_orbits(const Rule9C& r9, const FnParams& fp, const double (&c)[D],
                                                const double (&h)[D], unsigned& zc, const unsigned zs, double& sA1,
                                                double& sA3, double& sP11, double& sP12, double& sT, double& sC) {
  using F = Fn<FN, D>;
  bool bad = false;
  auto acc = [&](double& s, double v) {
    if (CHECK) bad |= !isfinite(v);
    else s += v;
  };
  const double g0 = r9.g[0], g1 = r9.g[1], g2 = r9.g[2], g3 = r9.g[3];
  constexpr int kPairU = D <= 5 ? 4 : K9_PU6, kTriU = D <= 5 ? 8 : K9_TU6;
  // ---- g1 / g3 on the axes: 4 nodes per axis ----
#pragma unroll 1
  for (int k = 0; k < D; ++k) {
    const double ck = pick<D>(c, k), hk = pick<D>(h, k);
    const double o1 = g1 * hk, o3 = g3 * hk;
    double x[D];
    place3<D>(x, c, k, ck + o1, -1, 0.0, -1, 0.0);
    zc += zs; acc(sA1, F::fast(x, fp, zc));
    place3<D>(x, c, k, ck - o1, -1, 0.0, -1, 0.0);
    zc += zs; acc(sA1, F::fast(x, fp, zc));
    place3<D>(x, c, k, ck + o3, -1, 0.0, -1, 0.0);
    zc += zs; acc(sA3, F::fast(x, fp, zc));
    place3<D>(x, c, k, ck - o3, -1, 0.0, -1, 0.0);
    zc += zs; acc(sA3, F::fast(x, fp, zc));
  }
  if (!CHECK) K1_PHASE_SYNC();  // (the rare re-walk runs divergently: no barriers)
  // ---- pairs k < l: (g1, g1) x 4 signs, (g1, g2) and (g2, g1) x 4 signs;
  //      one switch case per pair (compile-time coordinate positions) ----
  if constexpr (CHECK) {
#pragma unroll 1
    for (int p = 0; p < D * (D - 1) / 2; ++p) {
      const int k = c_pairs.k[p], l = c_pairs.l[p];
      const double ck = pick<D>(c, k), hk = pick<D>(h, k), cl = pick<D>(c, l), hl = pick<D>(h, l);
      for (int s = 0; s < 4; ++s) {
        const double sk = (s & 1) ? -1.0 : 1.0, sl = (s & 2) ? -1.0 : 1.0;
        double x[D];
        place3<D>(x, c, k, fma(sk, g1 * hk, ck), l, fma(sl, g1 * hl, cl), -1, 0.0);
        acc(sP11, F::fast(x, fp));
        place3<D>(x, c, k, fma(sk, g1 * hk, ck), l, fma(sl, g2 * hl, cl), -1, 0.0);
        acc(sP12, F::fast(x, fp));
        place3<D>(x, c, k, fma(sk, g2 * hk, ck), l, fma(sl, g1 * hl, cl), -1, 0.0);
        acc(sP12, F::fast(x, fp));
      }
    }
    if constexpr (D >= 3) {
#pragma unroll 1
      for (int t = 0; t < D * (D - 1) * (D - 2) / 6; ++t) {
        const int k = c_triples.k[t], l = c_triples.l[t], m = c_triples.m[t];
        const double ck = pick<D>(c, k), cl = pick<D>(c, l), cm = pick<D>(c, m);
        const double ak = g1 * pick<D>(h, k), al = g1 * pick<D>(h, l), am = g1 * pick<D>(h, m);
        for (int s = 0; s < 8; ++s) {
          double x[D];
          place3<D>(x, c, k, (s & 1) ? ck - ak : ck + ak, l, (s & 2) ? cl - al : cl + al, m,
                    (s & 4) ? cm - am : cm + am);
          acc(sT, F::fast(x, fp));
        }
      }
    }
  } else {
#pragma unroll 1
  for (int p = 0; p < D * (D - 1) / 2; ++p) {
    switch (p) {
#define HCUB_P9_BODY(K, L)                                                                   \
  {                                                                                          \
    double x[D];                                                                             \
    _Pragma("unroll") for (int j = 0; j < D; ++j) x[j] = c[j];                               \
    const double a1 = g1 * h[K], b1 = g1 * h[L], a2 = g2 * h[K], b2 = g2 * h[L];             \
    _Pragma("unroll (kPairU)") for (int s = 0; s < 4; ++s) {                                 \
      const double sk = (s & 1) ? -1.0 : 1.0, sl = (s & 2) ? -1.0 : 1.0;                     \
      x[K] = fma(sk, a1, c[K]); x[L] = fma(sl, b1, c[L]);                                    \
      zc += zs; acc(sP11, F::fast(x, fp, zc));                                               \
      x[L] = fma(sl, b2, c[L]);                                                              \
      zc += zs; acc(sP12, F::fast(x, fp, zc));                                               \
      x[K] = fma(sk, a2, c[K]); x[L] = fma(sl, b1, c[L]);                                    \
      zc += zs; acc(sP12, F::fast(x, fp, zc));                                               \
    }                                                                                        \
  }
      HCUB_L4_CASES(D, HCUB_P9_BODY)
#undef HCUB_P9_BODY
    }
  }
  K1_PHASE_SYNC();
  // ---- triples k < l < m: (g1, g1, g1) x 8 signs; a switch case per (k, l)
  //      (compile-time), m > l a run-time loop placed by selects over j > l ----
  if constexpr (D >= 3) {
#pragma unroll 1
    for (int p = 0; p < D * (D - 1) / 2; ++p) {
      switch (p) {
#define HCUB_T9_BODY(K, L)                                                                   \
  {                                                                                          \
    const double ak = g1 * h[K], al = g1 * h[L];                                             \
    _Pragma("unroll 1") for (int m = L + 1; m < D; ++m) {                                    \
      const double cm = pick<D>(c, m), am = g1 * pick<D>(h, m);                              \
      _Pragma("unroll (kTriU)") for (int s = 0; s < 8; ++s) {                                 \
        const double vm = (s & 4) ? cm - am : cm + am;                                       \
        double x[D];                                                                         \
        _Pragma("unroll") for (int j = 0; j < D; ++j)                                        \
          x[j] = (j == K) ? ((s & 1) ? c[K] - ak : c[K] + ak)                                \
               : (j == L) ? ((s & 2) ? c[L] - al : c[L] + al)                                \
               : (j > L && j == m) ? vm : c[j];                                              \
        zc += zs; acc(sT, F::fast(x, fp, zc));                                               \
      }                                                                                      \
    }                                                                                        \
  }
        HCUB_L4_CASES(D, HCUB_T9_BODY)
#undef HCUB_T9_BODY
      }
    }
  }
  K1_PHASE_SYNC();
  }
  // ---- 2^d corners at g0: low bits unrolled (compile-time patterns) ----
  {
    double p0[D], m0[D];
#pragma unroll
    for (int j = 0; j < D; ++j) { const double o = g0 * h[j]; p0[j] = c[j] + o; m0[j] = c[j] - o; }
    constexpr int KLO = D < K1_CORNER_BITS_OF(D) ? D : K1_CORNER_BITS_OF(D);
    constexpr unsigned NHI = 1u << (D - KLO);
#pragma unroll 1
    for (unsigned mh = 0; mh < NHI; ++mh) {
      double xh[D];
#pragma unroll
      for (int j = KLO; j < D; ++j) xh[j] = ((mh >> (j - KLO)) & 1u) ? m0[j] : p0[j];
#pragma unroll
      for (unsigned ml = 0; ml < (1u << KLO); ++ml) {
        double x[D];
#pragma unroll
        for (int j = 0; j < D; ++j) x[j] = (j < KLO) ? (((ml >> j) & 1u) ? m0[j] : p0[j]) : xh[j];
        zc += zs;
        acc(sC, F::fast(x, fp, zc));
      }
    }
  }
  return bad;
}

// Rare path (ref rules.py:480-492): does any node of the region evaluate to
// a non-finite value?  Out of line, so its registers never burden the main path.
template <int D, int FN>
__device__ __noinline__ bool gm9_any_nonfinite(const K1Args& a, const Rule9C& r9, const FnParams& fp, int64_t r) {
  using F = Fn<FN, D>;
  double c[D], h[D], ext[D], vol;
  k1_load_region<D>(a, r, false, c, h, ext, vol);
  bool bad = !isfinite(F::exact(c, fp));
  for (int k = 0; k < D && !bad; ++k)
    for (int s = 0; s < 4 && !bad; ++s) {
      const double lam = (s < 2) ? r9.g[2] : r9.g[0];
      double x[D];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const double off = mul_rn(h[j], lam);
        x[j] = (j != k) ? c[j] : ((s & 1) ? sub_rn(c[j], off) : add_rn(c[j], off));
      }
      bad = !isfinite(F::exact(x, fp));
    }
  if (!bad) {
    unsigned z = 0u;
    double d0, d1, d2, d3, d4, d5;
    bad = gm9_fast_orbits<D, FN, true>(r9, fp, c, h, z, 0u, d0, d1, d2, d3, d4, d5);
  }
  return bad;
}

template <int D, int FN>
__global__ void __launch_bounds__(K1_BLOCK_OF(D), K9_MIN_BLOCKS(D)) k1_gm9_eval(K1Args a, Rule9C r9, FnParams fp) {
  using F = Fn<FN, D>;
  const int64_t rid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = rid < a.n;
  const int64_t r = live ? rid : a.n - 1;
  const unsigned zs = (unsigned)a.zero;
  unsigned zc = zs;
  double c[D], h[D], ext[D], vol;
  k1_load_region<D>(a, r, live, c, h, ext, vol);
  const double scale = __ddiv_rn(vol, r9.twod);

  // ---- exact path: center, +-g2 (lam_in) and +-g0 (lam_out) on every axis ----
  RuleC rx{};
  rx.lam2 = r9.g[2];
  rx.lam3 = r9.g[0];
  rx.ratio = r9.ratio;
  const double fc = F::exact(c, fp, zc);
  double S2 = 0.0, S0 = 0.0, best_s = 0.0;  // sums of the g2 / g0 axis orbits
  int best_k = -1;
  double* srow = (a.scores && live) ? a.scores + r * D : nullptr;
  bool safe = false;
  if constexpr (HasSafe<F>::value) safe = F::safe_range(c, h, fmax(r9.g[0], r9.g[2]), fp);
  if (__all_sync(0xffffffffu, safe)) {
    if constexpr (HasSafe<F>::value) k1_axes_g1<D, FN, true>(rx, fp, c, h, fc, zc, zs, S2, S0, best_s, best_k, srow);
  } else {
    k1_axes_g1<D, FN, false>(rx, fp, c, h, fc, zc, zs, S2, S0, best_s, best_k, srow);
  }
  double e_ax = ext[0];
#pragma unroll
  for (int j = 1; j < D; ++j)
    if (j == best_k) e_ax = ext[j];
  K1_PHASE_SYNC();

  double sA1 = 0.0, sA3 = 0.0, sP11 = 0.0, sP12 = 0.0, sT = 0.0, sC = 0.0;
  gm9_fast_orbits<D, FN, false>(r9, fp, c, h, zc, zs, sA1, sA3, sP11, sP12, sT, sC);

  double integ = 0.0, err = 0.0;
  if (live) {
    const double S[O9_N] = {fc, S0, sA1, S2, sA3, sP11, sP12, sT, sC};
    double m = 0.0, e = 0.0;
#pragma unroll
    for (int o = 0; o < O9_N; ++o) { m += r9.w[o] * S[o]; e += r9.we[o] * S[o]; }
    const double main = m * scale, emb = e * scale;
    const double low = (r9.null_center * fc + r9.null_axis * S0) * scale;  // ref rules.py:525-526
    const double lowest = (r9.twod * fc) * scale;
    err = cascade_error(main, emb, low, lowest);
    integ = main;
    int axis = best_k;
    bool finite = isfinite(fc) && isfinite(S0) && isfinite(S2);
#pragma unroll
    for (int o = 2; o < O9_N; ++o) finite &= isfinite(S[o]);
    if (!finite) {  // rare path: a non-finite node, or overflowing sums of finite ones
      const bool bad = gm9_any_nonfinite<D, FN>(a, r9, fp, r);
      if (bad) {
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
    }
    a.integral[r] = integ;
    a.error[r] = err;
    if (a.vol) a.vol[r] = vol;
    if (a.axis) a.axis[r] = (signed char)axis;
    if (a.axis64) a.axis64[r] = axis;
    if (a.aext) a.aext[r] = e_ax;
  }
  k1_accumulate(a, live, integ, err);
}
