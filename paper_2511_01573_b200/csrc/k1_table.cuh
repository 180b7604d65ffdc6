// K1 for explicit fully symmetric node tables (parse_rule_table /
// load_rule_table, ref pkg/src/hcub/rules.py:377-405 + 178-250, applied by
// _apply_symmetric_batch rules.py:495-536): the route for custom rule families
// such as the paper's degree-9 Genz-Malik tables (SPEC.md 170/185).
//
// The table (nodes on the reference cube, per-node main/embedded weights)
// lives in device memory; every node is one full functor evaluation
// x = c + h*p.  Tables carrying the axis bookkeeping (unique center node, two
// distinct on-axis orbits) get the 4th-difference scores and the null-rule
// cascade exactly as the reference computes them (center and on-axis nodes on
// the exact path); others use |main - embedded| and the widest axis.
#pragma once
#include "k1_eval.cuh"

struct TableArgs {
  const double* pts;   // [K][d] reference-cube nodes
  const double* w;     // [K] main weights (x 2^d convention, like the reference)
  const double* we;    // [K] embedded weights
  int K;
  int has_pairs;
  int center;
  int pairs[HCUB_MAXD][4];  // node ids: +in, -in, +out, -out per axis
  double ratio, null_center, null_axis, twod;
};

template <int D, int FN>
__device__ __forceinline__ void k1_table_epilogue(const K1Args& a, const TableArgs& t, const FnParams& fp, int64_t r,
                                                  const double (&c)[D], const double (&h)[D], const double (&ext)[D],
                                                  double vol, double scale, double sm, double se, bool finite,
                                                  double& integ_out, double& err_out);

template <int D, int FN>
__global__ void __launch_bounds__(K1_BLOCK) k1_table_eval(K1Args a, TableArgs t, FnParams fp) {
  using F = Fn<FN, D>;
  const int G = 1 << a.log2g;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t rid = tid >> a.log2g;
  const int g = (int)(tid & (G - 1));
  const bool live = rid < a.n;
  const int64_t r = live ? rid : a.n - 1;
  double c[D], h[D], ext[D], vol;
  k1_load_region<D>(a, r, g == 0 && live, c, h, ext, vol);
  const double scale = __ddiv_rn(vol, t.twod);

  // weighted sums over every node (fast functor), nodes strided over the group
  double sm = 0.0, se = 0.0;
  bool finite = true;
#pragma unroll 1
  for (int i = g; i < t.K; i += G) {
    const double* p = t.pts + (int64_t)i * D;
    double x[D];
#pragma unroll
    for (int j = 0; j < D; ++j) x[j] = fma(h[j], p[j], c[j]);
    const double v = F::fast(x, fp);
    finite &= isfinite(v);
    sm = fma(t.w[i], v, sm);
    se = fma(t.we[i], v, se);
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    if (o >= G) break;
    sm += __shfl_xor_sync(0xffffffffu, sm, o);
    se += __shfl_xor_sync(0xffffffffu, se, o);
    finite = __shfl_xor_sync(0xffffffffu, (int)finite, o) && finite;
  }
  double integ = 0.0, err = 0.0;
  if (g == 0 && live) {
    k1_table_epilogue<D, FN>(a, t, fp, r, c, h, ext, vol, scale, sm, se, finite, integ, err);
  }
  k1_accumulate(a, g == 0 && live, integ, err);  // fused K2 (all lanes of the warp take part)
}

// scores / cascade / guard / outputs of one region (lane 0 of its group)
template <int D, int FN>
__device__ __forceinline__ void k1_table_epilogue(const K1Args& a, const TableArgs& t, const FnParams& fp, int64_t r,
                                                  const double (&c)[D], const double (&h)[D], const double (&ext)[D],
                                                  double vol, double scale, double sm, double se, bool finite,
                                                  double& integ_out, double& err_out) {
  using F = Fn<FN, D>;
  // exact on-axis nodes (numpy order x = c + h*p) for the scores / cascade
  auto exact_node = [&](int id) {
    const double* p = t.pts + (int64_t)id * D;
    double x[D];
#pragma unroll
    for (int j = 0; j < D; ++j) x[j] = add_rn(c[j], mul_rn(h[j], p[j]));
    return F::exact(x, fp);
  };
  const double main = sm * scale, emb = se * scale;
  double err;
  int axis = 0;
  if (t.has_pairs) {
    const double fc = exact_node(t.center);
    const double two_fc = 2.0 * fc;
    double sout = 0.0, best = 0.0;
    int bk = -1;
    for (int k = 0; k < D; ++k) {
      const double vin = add_rn(exact_node(t.pairs[k][0]), exact_node(t.pairs[k][1]));
      const double vout = add_rn(exact_node(t.pairs[k][2]), exact_node(t.pairs[k][3]));
      const double sc = fabs(sub_rn(sub_rn(vin, two_fc), mul_rn(t.ratio, sub_rn(vout, two_fc))));
      if (score_better(sc, k, best, bk)) { best = sc; bk = k; }
      if (a.scores) a.scores[r * D + k] = sc;
      sout += vout;
    }
    axis = bk;
    const double low = (t.null_center * fc + t.null_axis * sout) * scale;
    const double lowest = (t.twod * fc) * scale;
    err = cascade_error(main, emb, low, lowest);
  } else {  // no on-axis bookkeeping: widest axis, plain embedded difference
    err = fabs(main - emb);
    double bv = ext[0];
#pragma unroll
    for (int j = 1; j < D; ++j)
      if (ext[j] > bv) { bv = ext[j]; axis = j; }
    if (a.scores)
#pragma unroll
      for (int j = 0; j < D; ++j) a.scores[r * D + j] = ext[j];
  }
  double integ = main;
  if (!finite) {  // non-finite guard (ref rules.py:480-492)
    integ = 0.0;
    err = 1e30 * vol;
    double bv = ext[0];
    axis = 0;
#pragma unroll
    for (int j = 1; j < D; ++j)
      if (ext[j] > bv) { bv = ext[j]; axis = j; }
    if (a.scores)
#pragma unroll
      for (int j = 0; j < D; ++j) a.scores[r * D + j] = ext[j];
  }
  a.integral[r] = integ;
  a.error[r] = err;
  if (a.vol) a.vol[r] = vol;
  if (a.axis) a.axis[r] = (signed char)axis;
  if (a.axis64) a.axis64[r] = axis;
  if (a.aext) {
    double e_ax = ext[0];
#pragma unroll
    for (int j = 1; j < D; ++j)
      if (j == axis) e_ax = ext[j];
    a.aext[r] = e_ax;
  }
  integ_out = integ;
  err_out = err;
}
