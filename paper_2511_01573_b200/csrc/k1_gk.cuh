// K1 for the tensor-product Gauss(7)/Kronrod(15) rule, d <= 6
// (ref pkg/src/hcub/rules.py:285-357 build_gk_tensor_rule, 539-633
// _apply_tensor_gk_batch; get_rule("gm", 1) resolves here too).
//
// 15^d nodes per region, decoded on the fly from the node index (axis 0 the
// slowest digit, numpy meshgrid 'ij' / kron order).  Work unit: one warp per
// (region, chunk of GK_CHUNK nodes); each warp reduces its partial sums
// (main, embedded, d per-axis mixed sums) with shuffles and stores them; a
// second kernel sums the chunks of a region in a fixed order (deterministic)
// and forms integral, error = |main - emb|, per-axis scores
// |axis_i * scale - main| and the split axis, with the non-finite guard.
#pragma once
#include "k1_eval.cuh"

#define GK_CHUNK 512  // nodes per warp work unit (16 per lane)

struct GkArgs {
  double node[15];   // 1-D Kronrod abscissae on [-1, 1], ascending
  double wk[15];     // Kronrod weights
  double ratio[15];  // Gauss / Kronrod weight (0 at Kronrod-only nodes)
  int K;             // 15^d
  int chunks;        // ceil(K / GK_CHUNK)
  double twod;
};

template <int D, int FN>
__global__ void __launch_bounds__(128) k1_gk_partial(K1Args a, GkArgs gk, FnParams fp, int64_t r0, int64_t nb,
                                                     double* __restrict__ part) {
  using F = Fn<FN, D>;
  const int lane = threadIdx.x & 31;
  const int64_t unit = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // warp id
  const int64_t reg = unit / gk.chunks;
  const int chunk = (int)(unit % gk.chunks);
  const bool active = reg < nb;  // warp-uniform; inactive warps still reach the barrier
  const int64_t r = r0 + (active ? reg : 0);
  double c[D], h[D], ext[D], vol;
  k1_load_region<D>(a, r, active && chunk == 0 && lane == 0, c, h, ext, vol);
  // per-axis node coordinates (numpy order c + h*p) and 1-D weights in
  // shared memory, indexed by each node's digits
  __shared__ double wks[16], rts[16];
  __shared__ double xs_all[4][D][16];  // 4 warps per 128-thread block
  if (threadIdx.x < 15) { wks[threadIdx.x] = gk.wk[threadIdx.x]; rts[threadIdx.x] = gk.ratio[threadIdx.x]; }
  double (*xs)[16] = xs_all[threadIdx.x >> 5];
  for (int q = lane; q < 15 * D; q += 32) {
    const int j = q / 15, k = q % 15;
    double cj = c[0], hj = h[0];
#pragma unroll
    for (int jj = 1; jj < D; ++jj)
      if (jj == j) { cj = c[jj]; hj = h[jj]; }
    xs[j][k] = add_rn(cj, mul_rn(hj, gk.node[k]));
  }
  __syncthreads();
  double sm = 0.0, se = 0.0, sa[D];
#pragma unroll
  for (int j = 0; j < D; ++j) sa[j] = 0.0;
  bool finite = true;
  const int n0 = chunk * GK_CHUNK, n1 = active ? min(gk.K, n0 + GK_CHUNK) : n0;
#pragma unroll 1
  for (int n = n0 + lane; n < n1; n += 32) {
    int dig[D];
    int rem = n;
#pragma unroll
    for (int j = D - 1; j >= 0; --j) { dig[j] = rem % 15; rem /= 15; }
    double x[D];
    double wm = 1.0, rp = 1.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      x[j] = xs[j][dig[j]];
      wm *= wks[dig[j]];
      rp *= rts[dig[j]];
    }
    const double v = F::fast(x, fp);
    finite &= isfinite(v);
    const double wv = wm * v;
    sm += wv;
    se += wv * rp;  // Gauss product weight = Kronrod product * prod(Gauss/Kronrod)
#pragma unroll
    for (int j = 0; j < D; ++j) sa[j] += wv * rts[dig[j]];  // axis j on Gauss weights, others Kronrod
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sm += __shfl_xor_sync(0xffffffffu, sm, o);
    se += __shfl_xor_sync(0xffffffffu, se, o);
#pragma unroll
    for (int j = 0; j < D; ++j) sa[j] += __shfl_xor_sync(0xffffffffu, sa[j], o);
    finite = __shfl_xor_sync(0xffffffffu, (int)finite, o) && finite;
  }
  if (lane == 0 && active) {
    double* p = part + (reg * gk.chunks + chunk) * (D + 3);
    p[0] = sm;
    p[1] = se;
#pragma unroll
    for (int j = 0; j < D; ++j) p[2 + j] = sa[j];
    p[2 + D] = finite ? 0.0 : 1.0;
  }
}

// one warp per region: fixed-order sum of its chunks, then the outputs
template <int D>
__global__ void __launch_bounds__(128) k1_gk_finalize(K1Args a, GkArgs gk, int64_t r0, int64_t nb,
                                                      const double* __restrict__ part) {
  const int lane = threadIdx.x & 31;
  const int64_t reg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (reg >= nb) return;
  const int64_t r = r0 + reg;
  double acc[D + 3];
#pragma unroll
  for (int q = 0; q < D + 3; ++q) acc[q] = 0.0;
  for (int ch = lane; ch < gk.chunks; ch += 32) {
    const double* p = part + (reg * gk.chunks + ch) * (D + 3);
#pragma unroll
    for (int q = 0; q < D + 3; ++q) acc[q] += p[q];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1)
#pragma unroll
    for (int q = 0; q < D + 3; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
  if (lane != 0) return;
  double ext[D], vol = 1.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    ext[j] = sub_rn(a.hi[j * a.ld + r], a.lo[j * a.ld + r]);
    vol = (j == 0) ? ext[0] : mul_rn(vol, ext[j]);
  }
  const double scale = __ddiv_rn(vol, gk.twod);
  const double main = acc[0] * scale, emb = acc[1] * scale;
  double integ = main, err = fabs(main - emb), sc[D];
#pragma unroll
  for (int j = 0; j < D; ++j) sc[j] = fabs(acc[2 + j] * scale - main);
  if (acc[2 + D] != 0.0) {  // non-finite guard (ref rules.py:480-492)
    integ = 0.0;
    err = 1e30 * vol;
#pragma unroll
    for (int j = 0; j < D; ++j) sc[j] = ext[j];
  }
  int axis = -1;
  double best = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j)
    if (score_better(sc[j], j, best, axis)) { best = sc[j]; axis = j; }
  if (a.scores)
#pragma unroll
    for (int j = 0; j < D; ++j) a.scores[r * D + j] = sc[j];
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
}
