// eig_topr.cuh -- the top-R eigenpairs of an ne x ne symmetric matrix (ne <= 512) for the
// NG-SGD initialisation (B.3.2): S_0 = X_0^T X_0 / N, or the Gram matrix
// X_0 X_0^T / N when N < D.  FP64, one CTA of 1024 threads, the matrix in global memory
// (2 MB at ne = 512: L2-resident):
//
//   1. Householder tridiagonalisation A = Q T Q^T (LAPACK dsytd2 'L' order): per column,
//      the reflector (block reduction), p = A_22 v (a warp per row, coalesced), w, and the
//      rank-2 update of the trailing matrix (full symmetric storage).  Reflector k is kept
//      as row k of V (v_k[k+1] = 1), tau_k in tau.
//   2. The R largest eigenvalues of T by multisection on the Sturm count (a group of
//      threads per eigenvalue, 2^-52 relative bracket), then their eigenvectors by inverse
//      iteration (LU with partial pivoting of T - lambda I, three solves), each relative
//      cluster (|lambda_i - lambda_j| <= 1e-9 ||T||) orthogonalised by modified Gram-Schmidt.
//   3. Back-transformation u = Q x (the reflectors applied to every eigenvector, a warp per
//      vector, no barriers).
//
// Replaces the one-CTA cyclic Jacobi of the whole ne x ne matrix (~1 s per state at
// ne = 512) with O(ne^3) Householder work plus O(R ne) per eigenpair.
#pragma once

#include "ng_common.cuh"

namespace ng {

constexpr int kToprMaxN = 512;
constexpr int kToprMaxR = 128;

struct ToprWork {        // global-memory workspace (device), sizes for ne, R
  double* A;             // ne x ne (in: the matrix; destroyed)
  double* V;             // ne x ne: reflector rows
  double* tau;           // ne
  double* d;             // ne
  double* e;             // ne
  double* X;             // R x ne: eigenvectors of T, then of A (rows)
  double* lam;           // R: eigenvalues, descending
  double* scr;           // (1 + 3 R) ne: e_i^2 and the inverse-iteration factors
};

__device__ __forceinline__ int topr_sturm(const double* __restrict__ d, const double* __restrict__ e2, int n,
                                          double x, double pivmin) {
  // number of eigenvalues of T below x
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += q < 0.0;
  for (int i = 1; i < n; ++i) {
    q = (d[i] - x) - e2[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

// Solve (T - lam I) x = b in place (b -> x): Gaussian elimination with partial pivoting on
// the tridiagonal (LAPACK dgttrf order: the upper factor gets one fill-in diagonal), pivots
// below `tiny` in magnitude replaced by `tiny` (inverse iteration only needs a direction).
__device__ void topr_tri_solve(const double* __restrict__ d, const double* __restrict__ e, int n, double lam,
                               double tiny, double* __restrict__ x, double* __restrict__ u0,
                               double* __restrict__ u1, double* __restrict__ u2) {
  double a = d[0] - lam, b = n > 1 ? e[0] : 0.0, c = 0.0;   // current row: cols i, i+1, i+2
  for (int i = 0; i + 1 < n; ++i) {
    const double sub = e[i], nd = d[i + 1] - lam, ns = (i + 2 < n) ? e[i + 1] : 0.0;
    double na, nb;
    if (fabs(sub) > fabs(a)) {            // row i+1 is the pivot row
      const double m = a / sub;
      u0[i] = sub; u1[i] = nd; u2[i] = ns;
      const double xi = x[i];
      x[i] = x[i + 1];
      x[i + 1] = xi - m * x[i];
      na = b - m * nd;
      nb = c - m * ns;
    } else {
      if (fabs(a) < tiny) a = copysign(tiny, a);
      const double m = sub / a;
      u0[i] = a; u1[i] = b; u2[i] = c;
      x[i + 1] -= m * x[i];
      na = nd - m * b;
      nb = ns - m * c;
    }
    a = na; b = nb; c = 0.0;
  }
  if (fabs(a) < tiny) a = copysign(tiny, a);
  u0[n - 1] = a; u1[n - 1] = 0.0; u2[n - 1] = 0.0;
  for (int i = n - 1; i >= 0; --i) {
    double t = x[i];
    if (i + 1 < n) t -= u1[i] * x[i + 1];
    if (i + 2 < n) t -= u2[i] * x[i + 2];
    x[i] = t / u0[i];
  }
}

// All three phases; every thread of the CTA calls it.  R <= min(ne, kToprMaxR).
__device__ void eig_topr(int ne, int R, const ToprWork& W) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  __shared__ double red[32];
  __shared__ double vs[kToprMaxN], ps[kToprMaxN];
  __shared__ double sh_tau, sh_alpha_scale;
  double* A = W.A;
  const int n = ne;
  // ---- 1. tridiagonalisation
  for (int k = 0; k + 2 < n; ++k) {
    const int m0 = k + 1;   // trailing block starts here
    // reflector of column k, rows k+1 .. n-1
    double s = 0.0;
    for (int i = m0 + 1 + tid; i < n; i += nt) { const double a = A[(int64_t)i * n + k]; s = fma(a, a, s); }
    s = block_sum(s, red);
    if (tid == 0) {
      const double alpha = A[(int64_t)m0 * n + k];
      double beta, tau, scal;
      if (s == 0.0) { beta = alpha; tau = 0.0; scal = 0.0; }
      else {
        beta = -copysign(sqrt(alpha * alpha + s), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      W.d[k] = A[(int64_t)k * n + k];
      W.e[k] = beta;
      W.tau[k] = tau;
      sh_tau = tau; sh_alpha_scale = scal;
    }
    __syncthreads();
    const double tau = sh_tau, scal = sh_alpha_scale;
    for (int i = tid; i < n; i += nt) {
      const double v = (i < m0) ? 0.0 : (i == m0 ? 1.0 : A[(int64_t)i * n + k] * scal);
      vs[i] = v;
      W.V[(int64_t)k * n + i] = v;
    }
    __syncthreads();
    // p = A_22 v (a warp per row)
    for (int i = m0 + warp; i < n; i += nw) {
      const double* Ai = A + (int64_t)i * n;
      double acc = 0.0;
      for (int j = m0 + lane; j < n; j += 32) acc = fma(Ai[j], vs[j], acc);
      acc = warp_sum(acc);
      if (lane == 0) ps[i] = acc;
    }
    __syncthreads();
    double pv = 0.0;
    for (int i = m0 + tid; i < n; i += nt) pv = fma(ps[i], vs[i], pv);
    pv = block_sum(pv, red);
    const double hk = 0.5 * tau * pv;
    for (int i = m0 + tid; i < n; i += nt) ps[i] = tau * (ps[i] - hk * vs[i]);   // w
    __syncthreads();
    // rank-2 update of the trailing block (full symmetric storage)
    const int r = n - m0;
    for (int idx = tid; idx < r * r; idx += nt) {
      const int i = m0 + idx / r, j = m0 + idx % r;
      A[(int64_t)i * n + j] -= vs[i] * ps[j] + ps[i] * vs[j];
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (n >= 2) {
      W.d[n - 2] = A[(int64_t)(n - 2) * n + (n - 2)];
      W.e[n - 2] = A[(int64_t)(n - 1) * n + (n - 2)];
    }
    W.d[n - 1] = A[(int64_t)(n - 1) * n + (n - 1)];
  }
  __syncthreads();
  // ---- 2. eigenvalues (top R) by multisection, then inverse iteration
  double* e2 = W.scr;                       // n (shared by all threads): e_i^2
  for (int i = tid; i + 1 < n; i += nt) e2[i] = W.e[i] * W.e[i];
  double tn = 0.0;
  for (int i = tid; i < n; i += nt) tn = fmax(tn, fabs(W.d[i]) + (i + 1 < n ? fabs(W.e[i]) : 0.0) + (i > 0 ? fabs(W.e[i - 1]) : 0.0));
  tn = block_max(tn, red);
  __syncthreads();
  const double pivmin = 1e-300 * fmax(1.0, tn * tn);
  const double eps = 2.220446049250313e-16;
  {
    // 8 threads per eigenvalue (groups aligned inside warps): 9-section of the bracket of
    // the (q+1)-th largest eigenvalue until it is 2 eps relative wide; every lane of a warp
    // keeps iterating until the whole warp is done (the shuffles need all of them)
    const int q = tid >> 3, g = tid & 7;
    const bool act = q < R;
    const int target = n - 1 - q;          // ascending index
    double lo = -tn - 1e-300, hi = tn + 1e-300;
    bool done = !act;
    for (int it = 0; it < 400; ++it) {
      if (__all_sync(0xffffffffu, done)) break;
      const double x = lo + (hi - lo) * (double)(g + 1) * (1.0 / 9.0);
      const int c = act ? topr_sturm(W.d, e2, n, x, pivmin) : 0;
      double nlo = lo, nhi = hi;
#pragma unroll
      for (int gg = 0; gg < 8; ++gg) {
        const double xg = __shfl_sync(0xffffffffu, x, (lane & ~7) + gg);
        const int cg = __shfl_sync(0xffffffffu, c, (lane & ~7) + gg);
        if (cg <= target) nlo = fmax(nlo, xg);
        else nhi = fmin(nhi, xg);
      }
      if (!done) { lo = nlo; hi = nhi; }
      done = done || (hi - lo <= 2.0 * eps * fmax(fabs(lo), fabs(hi)) + pivmin);
    }
    if (act && g == 0) W.lam[q] = 0.5 * (lo + hi);
  }
  __syncthreads();
  // eigenvectors: one thread per eigenvalue, three inverse-iteration solves from a
  // deterministic start, normalised
  for (int q = tid; q < R; q += nt) {
    double* x = W.X + (int64_t)q * n;
    double* sc = W.scr + n + (int64_t)q * 3 * n;
    const double lam = W.lam[q];
    for (int i = 0; i < n; ++i) x[i] = 1.0 + 0.001 * (double)((i * 7919 + q * 104729) % 997) / 997.0;
    for (int it = 0; it < 3; ++it) {
      topr_tri_solve(W.d, W.e, n, lam, eps * tn + pivmin, x, sc, sc + n, sc + 2 * n);
      double nn = 0.0;
      for (int i = 0; i < n; ++i) nn = fma(x[i], x[i], nn);
      const double inv = 1.0 / sqrt(nn);
      for (int i = 0; i < n; ++i) x[i] *= inv;
    }
  }
  __syncthreads();
  // clusters: MGS in descending order against every earlier member within 1e-9 ||T||
  for (int q = 1; q < R; ++q) {
    for (int p = 0; p < q; ++p) {
      if (fabs(W.lam[p] - W.lam[q]) > 1e-9 * tn) continue;   // uniform branch
      const double* xp = W.X + (int64_t)p * n;
      double* xq = W.X + (int64_t)q * n;
      double dt = 0.0;
      for (int i = tid; i < n; i += nt) dt = fma(xp[i], xq[i], dt);
      dt = block_sum(dt, red);
      for (int i = tid; i < n; i += nt) xq[i] -= dt * xp[i];
      __syncthreads();
      double nn = 0.0;
      for (int i = tid; i < n; i += nt) nn = fma(xq[i], xq[i], nn);
      nn = block_sum(nn, red);
      const double inv = 1.0 / sqrt(fmax(nn, 1e-300));
      for (int i = tid; i < n; i += nt) xq[i] *= inv;
      __syncthreads();
    }
  }
  // ---- 3. u = Q x = H_0 H_1 ... H_{n-3} x: a warp per vector, reflectors applied last-first
  for (int q = warp; q < R; q += nw) {
    double* x = W.X + (int64_t)q * n;
    for (int k = n - 3; k >= 0; --k) {
      const double* v = W.V + (int64_t)k * n;
      double dt = 0.0;
      for (int i = k + 1 + lane; i < n; i += 32) dt = fma(v[i], x[i], dt);
      dt = warp_sum(dt) * W.tau[k];
      for (int i = k + 1 + lane; i < n; i += 32) x[i] = fma(-dt, v[i], x[i]);
    }
  }
  __syncthreads();
}

}  // namespace ng
