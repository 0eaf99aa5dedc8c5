// eig_dc.cuh -- dense symmetric eigendecomposition for the R x R refresh:
// Householder tridiagonalisation + divide-and-conquer, FP64, ONE CTA of 1024 threads.
//
//   Z = Q_h T Q_h^T   (T tridiagonal; Q_h = H_0 ... H_{n-3}, reflectors kept in A)
//   T = Q_t diag(lam) Q_t^T by Cuppen's method: every boundary of T is torn up front
//       (T = blockdiag + sum rho_b v_b v_b^T), the 1 x 1 leaves are merged bottom-up; a
//       merge solves D + rho z z^T with LAPACK-style deflation (small rho z_i, and close
//       d_i via a Givens rotation), the secular equation for each remaining root as an
//       offset tau from its nearer pole (bisection, then safeguarded Newton), and the
//       Gu-Eisenstat z-hat so the eigenvectors are numerically orthogonal.
//   U = Q_h Q_t.
// Accuracy is absolute (|lam err| ~ eps ||Z||, like LAPACK's syevd that the oracle calls);
// tools/dc_proto.py is the NumPy prototype this follows step by step.  Merges of a level run
// concurrently, one group of warps each (named barriers); a merge of k = nl + nr costs one
// O(k) serial deflation scan, K secular solves (a warp each, lanes split the sum), O(k^2)
// z-hat / vectors and the k x k x k update of the block's eigenvector columns.
#pragma once

#include "ng_common.cuh"

namespace ng {

constexpr int kDCMax = 80;           // n <= kDCMax (shared-memory plan below)
__device__ unsigned long long g_dc_clk[16];   // phase timing (ng_debug_eig_clocks out[8..23])
constexpr bool kDCTiming = true;              // thread 0 accumulates phase cycles (a few atomics per solve)

__device__ __forceinline__ void dc_gsync(int G, int bar_id) {
  if (G == 1) {
    __syncwarp();
  } else if (G == 32) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(32 * G) : "memory");
  }
}


// FP64 reciprocal / divide / square root from the hardware approximations (MUFU.RCP64H,
// MUFU.RSQ64H) plus Newton steps: ~1 ulp, a fraction of the latency of the IEEE-rounded
// library sequences -- the secular iterations and the Householder step are chains of them.
__device__ __forceinline__ double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double fdiv(double a, double b) {
  const double r = frcp(b);
  const double q = a * r;
  return fma(fma(-b, q, a), r, q);
}
__device__ __forceinline__ double fsqrt(double x) {   // x >= 0
  if (!(x > 0.0)) return 0.0;
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-0.5 * x * y, y, 1.5);
  y = y * fma(-0.5 * x * y, y, 1.5);
  const double s = x * y;
  return fma(0.5 * y, fma(-s, s, x), s);
}

// Shared-memory plan (doubles unless noted), n <= kDCMax.
struct DCPlan {
  int n, lda;
  size_t oA, oQ, oV, oa, oe, obeta, op, olam, od, oz, ozh, otau, orc, ors, owork, oint, total;
};
__host__ __device__ inline DCPlan dc_plan(int n) {
  DCPlan p;
  p.n = n;
  p.lda = n + 1;
  size_t o = 0;
  p.oA = o; o += (size_t)n * p.lda;   // Householder work / reflectors; at the end U^T (rows)
  p.oQ = o; o += (size_t)n * n;       // eigenvectors of T (columns), block diagonal during D&C
  p.oV = o; o += (size_t)n * n;       // per-merge k x k secular eigenvectors (block offsets)
  p.oa = o; o += n;
  p.oe = o; o += n;
  p.obeta = o; o += n;
  p.op = o; o += n;
  p.olam = o; o += n;                 // eigenvalues of the current blocks (ascending per block)
  p.od = o; o += n;                   // merge scratch, indexed by the block's positions
  p.oz = o; o += n;
  p.ozh = o; o += n;
  p.otau = o; o += n;
  p.orc = o; o += n;                  // deflation rotations (c, s)
  p.ors = o; o += n;
  p.owork = o; o += 32 * (size_t)kDCMax;   // per-warp row staging
  p.oint = o;                          // ints: perm, colmap, defl, nd, org, rot (6 n), spare 2 n, counters 2 n
  p.total = sizeof(double) * o + sizeof(int) * (10 * (size_t)n + 64);
  return p;
}


// All K roots of the secular equation 1 + rho sum_i z_i^2 / (d_i - lam) = 0 (dk ascending,
// compact arrays), each as origin pole o (the nearer end of its interval) and offset tau.
// The group's T threads are cut into segments of L lanes (power of two, <= 32); segment s
// solves roots s, s + T/L, ...; its lanes split the sums and reduce with xor shuffles.  The
// "middle way" iteration (Li / LAPACK dlaed4 family): the poles left of the root (i <= j)
// and right of it (i > j) are each replaced by one pole at the nearest d plus a constant,
// matching value and slope at t; the quadratic gives the next t.  Bracketed by the sign of
// f (increasing in t); bisection if a step leaves the bracket.
__device__ __forceinline__ double seg_sum(double v, int L) {
  for (int o = L >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ void dc_roots(int K, const double* __restrict__ dk, const double* __restrict__ zk, double rho,
                         double zsq, int tg, int T, int* __restrict__ org, double* __restrict__ tau) {
  constexpr double kEps = 2.220446049250313e-16;
  int L = 32;
  while (L > 1 && L * K > T) L >>= 1;
  const int seg = tg / L, sl = tg - (tg / L) * L, nseg = T / L;
  for (int jb = 0; jb < K; jb += nseg) {          // uniform trip count over the group
    const int j = min(jb + seg, K - 1);
    const bool act = jb + seg < K;
    int o;
    double lo, hi;
    // f at the interval midpoint picks the nearer pole (every lane runs the shuffles: the
    // segments of one warp may hold interior and last roots)
    const bool interior = j < K - 1;
    const double dj = dk[j], mid = interior ? 0.5 * (dk[j + 1] - dj) : 1.0;
    double fm = 0.0;
#pragma unroll 4
    for (int i = sl; i < K; i += L) fm += zk[i] * zk[i] * frcp((dk[i] - dj) - mid);
    fm = 1.0 + rho * seg_sum(fm, L);
    if (interior) {
      if (fm >= 0.0) { o = j; lo = 0.0; hi = mid; } else { o = j + 1; lo = -mid; hi = 0.0; }
    } else {
      o = K - 1; lo = 0.0; hi = rho * zsq;
    }
    const double dpo = dk[o];
    const double DLp = dk[j] - dpo;
    const double DRp = (j < K - 1) ? dk[j + 1] - dpo : 0.0;
    double t = 0.5 * (lo + hi);
    bool done = false;
    for (int it = 0; it < 64; ++it) {
      double psi = 0.0, dpsi = 0.0, phi = 0.0, dphi = 0.0;
#pragma unroll 4
      for (int i = sl; i < K; i += L) {
        const double inv = frcp((dk[i] - dpo) - t);
        const double q = zk[i] * zk[i] * inv;
        if (i <= j) { psi += q; dpsi += q * inv; } else { phi += q; dphi += q * inv; }
      }
      psi = rho * seg_sum(psi, L);
      dpsi = rho * seg_sum(dpsi, L);
      phi = rho * seg_sum(phi, L);
      dphi = rho * seg_sum(dphi, L);
      if (!done) {
        const double f = 1.0 + psi + phi;
        if (f > 0.0) hi = t; else lo = t;
        if (f == 0.0) {
          done = true;
        } else {
          const double DL = DLp - t;
          const double b1 = dpsi * DL * DL, a1 = psi - b1 * frcp(DL);
          double u;
          if (j == K - 1) {
            u = DL + fdiv(b1, 1.0 + a1);
          } else {
            const double DR = DRp - t;
            const double b2 = dphi * DR * DR, a2 = phi - b2 * frcp(DR);
            const double c = 1.0 + a1 + a2;
            const double B = -(c * (DL + DR) + b1 + b2), C = c * DL * DR + b1 * DR + b2 * DL;
            const double disc = fmax(B * B - 4.0 * c * C, 0.0);
            const double q = -0.5 * (B + copysign(fsqrt(disc), B));
            const double u1 = (c != 0.0) ? fdiv(q, c) : 1e300, u2 = (q != 0.0) ? fdiv(C, q) : 1e300;
            u = (u1 > lo - t && u1 < hi - t) ? u1 : u2;
          }
          double tn = t + u;
          if (!(tn > lo && tn < hi)) tn = 0.5 * (lo + hi);
          done = fabs(tn - t) <= 4.0 * kEps * fabs(tn) || hi - lo <= 4.0 * kEps * fmax(fabs(lo), fabs(hi));
          t = tn;
        }
      }
      if (__all_sync(0xffffffffu, done)) break;
    }
    if (act && sl == 0) { org[jb + seg] = o; tau[jb + seg] = t; }
  }
}

// One merge of blocks [l0, s) and [s, r1): eigen of [T1 0; 0 T2] + rho_s v v^T, given
// lam[l0..r1) (ascending per half) and the block-diagonal columns Q[:, l0..r1).  Executed
// by a group of G warps (thread index tg in [0, 32G)); gsync synchronises the group.
__device__ void dc_merge(double* __restrict__ sm, const DCPlan& P, int l0, int s, int r1, double rho_signed,
                         int tg, int G, int bar_id) {
  const int n = P.n, T = 32 * G, k = r1 - l0, nl = s - l0;
  double* Q = sm + P.oQ;
  double* V = sm + P.oV;
  double* lam = sm + P.olam;
  double* d = sm + P.od + l0;     // all merge scratch lives at the block's positions
  double* z = sm + P.oz + l0;
  double* zh = sm + P.ozh + l0;
  double* tau = sm + P.otau + l0;
  double* rc = sm + P.orc + l0;
  double* rs = sm + P.ors + l0;
  int* ib = reinterpret_cast<int*>(sm + P.oint);
  int* perm = ib + l0;            // sorted position -> local index
  int* colmap = ib + n + l0;      // sorted position -> global column
  int* defl = ib + 2 * n + l0;
  int* nd = ib + 3 * n + l0;      // compact index -> sorted position
  int* org = ib + 4 * n + l0;     // root j -> compact index of its origin pole
  int* rot = ib + 5 * n + l0;     // deflation rotation j: (prev << 16) | cur (sorted positions)
  int* cnt = ib + 8 * n;          // [2*merge slot] counters: K, nrot (per block start)
  const int lane = tg & 31, wg = tg >> 5;
  const double sgn = rho_signed >= 0.0 ? 1.0 : -1.0;
  // 1. z = [last row of Q_L; +-first row of Q_R] (columns of each half), its norm
  for (int i = tg; i < k; i += T) {
    const double zi = (i < nl) ? Q[(s - 1) * n + l0 + i] : sgn * Q[s * n + l0 + i];
    z[i] = zi;
  }
  dc_gsync(G, bar_id);
  double zz = 0.0;
  for (int i = lane; i < k; i += 32) zz += z[i] * z[i];
  zz = warp_sum(zz);                                  // every warp computes the same norm
  const double zn = fsqrt(zz);
  const double rho = fabs(rho_signed) * zz;
  // 2. merge the two ascending halves: rank of each entry in the combined order
  for (int i = tg; i < k; i += T) {
    const double di = lam[l0 + i];
    int r;
    if (i < nl) {   // count right entries < di
      int lo = 0, hi = k - nl;
      while (lo < hi) { const int mid = (lo + hi) >> 1; if (lam[s + mid] < di) lo = mid + 1; else hi = mid; }
      r = i + lo;
    } else {        // count left entries <= di
      int lo = 0, hi = nl;
      while (lo < hi) { const int mid = (lo + hi) >> 1; if (lam[l0 + mid] <= di) lo = mid + 1; else hi = mid; }
      r = (i - nl) + lo;
    }
    perm[r] = i;
  }
  dc_gsync(G, bar_id);
  // sorted d, z (normalised), column map; scratch copies so lam can be overwritten later
  for (int r = tg; r < k; r += T) {
    const int i = perm[r];
    d[r] = lam[l0 + i];
    zh[r] = fdiv(z[i], zn);          // (z is re-read below: stage the sorted z in zh first)
    colmap[r] = l0 + i;
  }
  dc_gsync(G, bar_id);
  for (int r = tg; r < k; r += T) z[r] = zh[r];
  dc_gsync(G, bar_id);
  // 3-5. deflation scan (serial, thread 0 of the group) and the compact list
  if (tg == 0) {
    double dmax = 0.0, zmax = 0.0;
    for (int r = 0; r < k; ++r) { dmax = fmax(dmax, fabs(d[r])); zmax = fmax(zmax, fabs(z[r])); }
    const double tol = 8.0 * 2.220446049250313e-16 * fmax(dmax, rho * zmax);
    int prev = -1, nrot = 0, K = 0;
    for (int r = 0; r < k; ++r) {
      defl[r] = (rho * fabs(z[r]) <= tol) ? 1 : 0;
      if (defl[r]) continue;
      if (prev >= 0) {
        const double rr = fsqrt(z[prev] * z[prev] + z[r] * z[r]);
        const double irr = frcp(rr), c = z[r] * irr, sn = -z[prev] * irr;
        if (fabs((d[r] - d[prev]) * c * sn) <= tol) {
          const double t = d[prev] * c * c + d[r] * sn * sn;
          d[r] = d[prev] * sn * sn + d[r] * c * c;
          d[prev] = t;
          z[r] = rr;
          z[prev] = 0.0;
          defl[prev] = 1;
          rot[nrot] = (prev << 16) | r;
          rc[nrot] = c;
          rs[nrot] = sn;
          ++nrot;
        }
      }
      prev = r;
    }
    for (int r = 0; r < k; ++r)
      if (!defl[r]) nd[K++] = r;
    cnt[2 * l0] = K;
    cnt[2 * l0 + 1] = nrot;
  }
  dc_gsync(G, bar_id);
  const int K = cnt[2 * l0], nrot = cnt[2 * l0 + 1];
  // deflation rotations on the block's columns (every row applies them in order)
  if (nrot > 0)
    for (int row = l0 + tg; row < r1; row += T) {
      double* qr = Q + row * n;
      for (int t = 0; t < nrot; ++t) {
        const int a = colmap[rot[t] >> 16], b = colmap[rot[t] & 0xFFFF];
        const double qa = qr[a], qb = qr[b], c = rc[t], sn = rs[t];
        qr[a] = c * qa + sn * qb;
        qr[b] = -sn * qa + c * qb;
      }
    }
  // 6. secular roots: warp wg solves roots j = wg, wg + G, ...; lanes split the sum
  double zsq = 0.0;
  for (int i = lane; i < K; i += 32) { const double zi = z[nd[i]]; zsq += zi * zi; }
  zsq = warp_sum(zsq);
  // compact copies of the non-deflated d, z (rc / rs are free once the rotations are done)
  dc_gsync(G, bar_id);
  double* dk = rc;
  double* zk = rs;
  for (int i = tg; i < K; i += T) { dk[i] = d[nd[i]]; zk[i] = z[nd[i]]; }
  dc_gsync(G, bar_id);
  if (K > 0) dc_roots(K, dk, zk, rho, zsq, tg, T, org, tau);
  dc_gsync(G, bar_id);
  // 7. Gu-Eisenstat z-hat: prod_j (lam_j - d_i) = rho zhat_i^2 prod_{j != i} (d_j - d_i)
  for (int i = tg; i < K; i += T) {
    const double di = dk[i];
    double pr[4] = {1.0, 1.0, 1.0, 1.0};   // four independent chains of ratios
    for (int j = 0; j < K; ++j) {
      const double num = (dk[org[j]] - di) + tau[j];
      pr[j & 3] *= (j != i) ? fdiv(num, dk[j] - di) : num;
    }
    const double num = (pr[0] * pr[1]) * (pr[2] * pr[3]);
    zh[i] = copysign(fsqrt(fmax(fdiv(num, rho), 0.0)), zk[i]);
  }
  dc_gsync(G, bar_id);
  // 8. k x k eigenvector matrix in sorted-position space: V[r][c] (ld n, block offset l0)
  double* Vb = V + l0 * n + l0;
  for (int idx = tg; idx < k * k; idx += T) {
    const int r = idx / k, c = idx - (idx / k) * k;
    Vb[r * n + c] = 0.0;
  }
  dc_gsync(G, bar_id);
  for (int r = tg; r < k; r += T)
    if (defl[r]) Vb[r * n + r] = 1.0;
  for (int j = tg; j < K; j += T) {
    const double dpo = dk[org[j]], tj = tau[j];
    double nrm = 0.0;
    for (int i = 0; i < K; ++i) {
      const double v = fdiv(zh[i], (dk[i] - dpo) - tj);
      nrm += v * v;
    }
    const double inv = frcp(fsqrt(nrm));
    const int c = nd[j];
    for (int i = 0; i < K; ++i) Vb[nd[i] * n + c] = fdiv(zh[i], (dk[i] - dpo) - tj) * inv;
  }
  dc_gsync(G, bar_id);
  // new eigenvalues at sorted position c: deflated d[c], else root j with nd[j] = c
  for (int j = tg; j < K; j += T) tau[j] = dk[org[j]] + tau[j];   // tau := lambda_j
  dc_gsync(G, bar_id);
  for (int j = tg; j < K; j += T) zh[nd[j]] = tau[j];
  for (int r = tg; r < k; r += T)
    if (defl[r]) zh[r] = d[r];
  dc_gsync(G, bar_id);
  // ascending order of the k new eigenvalues: rank -> perm (reuse), then lam
  for (int c = tg; c < k; c += T) {
    const double v = zh[c];
    int rk = 0;
    for (int c2 = 0; c2 < k; ++c2) { const double w = zh[c2]; rk += (w < v) || (w == v && c2 < c); }
    perm[rk] = c;
  }
  dc_gsync(G, bar_id);
  // 9. Q[row, l0 + rk] = sum_r Q[row, colmap[r]] V[r][perm[rk]], one warp per row (the old
  // row is staged in the warp's own slot first: the update is in place)
  double* st = sm + P.owork + (size_t)(threadIdx.x >> 5) * kDCMax;
  for (int row = l0 + wg; row < r1; row += G) {
    for (int r = lane; r < k; r += 32) st[r] = Q[row * n + colmap[r]];
    __syncwarp();
    for (int rk = lane; rk < k; rk += 32) {
      const int c = perm[rk];
      double acc = 0.0;
      for (int r = 0; r < k; ++r) acc += st[r] * Vb[r * n + c];
      Q[row * n + l0 + rk] = acc;
    }
    __syncwarp();
  }
  for (int rk = tg; rk < k; rk += T) lam[l0 + rk] = zh[perm[rk]];
  dc_gsync(G, bar_id);
}

// Eigendecomposition of the n x n symmetric Z (row stride ldz, shared or global; may be
// this plan's own A region, ld n+1) into ascending eigenvalues lam_out[n] and eigenvector
// ROWS Vt (row i = eigenvector of lam_i, row stride ldvt; may be this plan's V region).
// sm: P.total bytes of shared memory; all threads of the CTA (1024).
__device__ void eig_dc(double* __restrict__ sm, const DCPlan& P, const double* __restrict__ Zin, int ldz,
                       double* __restrict__ lam_out, double* __restrict__ Vt, int ldvt) {
  const int n = P.n, lda = P.lda, tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = nt >> 5;
  double* A = sm + P.oA;
  double* Q = sm + P.oQ;
  double* a = sm + P.oa;
  double* e = sm + P.oe;
  double* beta = sm + P.obeta;
  double* p = sm + P.op;
  double* lam = sm + P.olam;
  long long ck0 = clock64();
  if (Zin != A || ldz != lda) {   // (the refresh builds Z_t directly in A)
    for (int idx = tid; idx < n * n; idx += nt) {
      const int i = idx / n, j = idx - (idx / n) * n;
      A[i * lda + j] = Zin[i * ldz + j];
    }
  }
  __syncthreads();
  // ---- Householder tridiagonalisation (Golub-Van Loan 5.1.1 / 8.3.1)
  for (int k = 0; k + 2 < n; ++k) {
    const int m = n - k - 1;
    double* xr = A + k * lda + k + 1;   // x = A[k][k+1 ..], reflector v[1..] stored here after
    if (warp == 0) {
      double sg = 0.0;
      for (int i = 1 + lane; i < m; i += 32) sg += xr[i] * xr[i];
      sg = warp_sum(sg);
      const double x0 = xr[0];
      double bt = 0.0, ek = x0, v0 = 1.0;
      if (sg != 0.0) {
        const double mu = fsqrt(x0 * x0 + sg);
        v0 = (x0 <= 0.0) ? x0 - mu : -fdiv(sg, x0 + mu);
        bt = fdiv(2.0 * v0 * v0, sg + v0 * v0);
        ek = mu;
      }
      const double iv0 = frcp(v0);
      __syncwarp();
      if (sg != 0.0)
        for (int i = 1 + lane; i < m; i += 32) xr[i] *= iv0;
      if (lane == 0) { beta[k] = bt; e[k] = ek; a[k] = A[k * lda + k]; xr[0] = 1.0; }
    }
    __syncthreads();
    const double bt = beta[k];
    if (bt != 0.0) {
      // p = beta S v, S = A[k+1.., k+1..]: 8 threads per row, partial sums over every 8th
      // column, reduced inside the 8-lane group
      {
        const int i = tid >> 3, c = tid & 7;
        double acc = 0.0;
        if (i < m) {
          const double* srow = A + (k + 1 + i) * lda + k + 1;
          for (int j = c; j < m; j += 8) acc += srow[j] * xr[j];
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        acc += __shfl_xor_sync(0xffffffffu, acc, 4);
        if (i < m && c == 0) p[i] = bt * acc;
      }
      __syncthreads();
      double pv = 0.0;
      for (int i = lane; i < m; i += 32) pv += p[i] * xr[i];
      const double K = 0.5 * bt * warp_sum(pv);
      for (int i = warp; i < m; i += nwarps) {
        const double vi = xr[i], wi = p[i] - K * vi;
        double* arow = A + (k + 1 + i) * lda + k + 1;
        for (int j = lane; j < m; j += 32) {
          const double vj = xr[j], wj = p[j] - K * vj;
          arow[j] -= vi * wj + wi * vj;
        }
      }
      __syncthreads();
    }
  }
  if (tid == 0) {
    if (n >= 2) {
      a[n - 2] = A[(n - 2) * lda + n - 2];
      e[n - 2] = A[(n - 2) * lda + n - 1];
    }
    a[n - 1] = A[(n - 1) * lda + n - 1];
    if (n >= 2) beta[n - 2] = 0.0;
  }
  __syncthreads();
  long long ck1 = clock64();
  // ---- divide and conquer on (a, e): tear every boundary, 1 x 1 leaves, Q = I
  for (int i = tid; i < n; i += nt) {
    double ai = a[i];
    if (i > 0) ai -= fabs(e[i - 1]);
    if (i + 1 < n) ai -= fabs(e[i]);
    lam[i] = ai;
  }
  for (int idx = tid; idx < n * n; idx += nt) Q[idx] = ((idx / n) == (idx % n)) ? 1.0 : 0.0;
  __syncthreads();
  for (int w = 1; w < n; w *= 2) {
    const int nm = (n - w + 2 * w - 1) / (2 * w);   // merges at this width
    // group size: whole warps, powers of two, at most 8 concurrent groups with G > 1
    int G = 1;
    if (nm < nwarps) { G = nwarps / nm; int g2 = 1; while (g2 * 2 <= G) g2 *= 2; G = g2; if (G > 1 && nwarps / G > 8) G = nwarps / 8; }
    const int ngroups = nwarps / G;
    const int grp = warp / G, tg = tid - grp * 32 * G;
    long long cl = clock64();
    for (int mi = grp; mi < nm; mi += ngroups) {
      const int l0 = mi * 2 * w, s = l0 + w, r1 = min(n, l0 + 2 * w);
      dc_merge(sm, P, l0, s, r1, e[s - 1], tg, G, 1 + grp);
    }
    __syncthreads();
    if (kDCTiming && tid == 0) {
      int lv = 0;
      for (int ww = 1; ww < w; ww *= 2) ++lv;
      if (lv < 12) atomicAdd(&g_dc_clk[4 + lv], (unsigned long long)(clock64() - cl));
    }
  }
  long long ck2 = clock64();
  // ---- U = Q_h Q_t: apply H_{n-3}, ..., H_0 from the left (v in A's rows)
  for (int k = n - 3; k >= 0; --k) {
    const double bt = beta[k];
    if (bt == 0.0) continue;
    const int m = n - k - 1;
    const double* v = A + k * lda + k + 1;
    // p[j] = beta sum_i v_i Q[k+1+i][j]: 8 threads per column, reduced in the 8-lane group
    {
      const int j = tid >> 3, c = tid & 7;
      double acc = 0.0;
      if (j < n)
        for (int i = c; i < m; i += 8) acc += v[i] * Q[(k + 1 + i) * n + j];
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      if (j < n && c == 0) p[j] = bt * acc;
    }
    __syncthreads();
    for (int i = warp; i < m; i += nwarps) {
      const double vi = v[i];
      double* qrow = Q + (k + 1 + i) * n;
      for (int j = lane; j < n; j += 32) qrow[j] -= vi * p[j];
    }
    __syncthreads();
  }
  long long ck3 = clock64();
  if (kDCTiming && tid == 0) {
    atomicAdd(&g_dc_clk[0], (unsigned long long)(ck1 - ck0));
    atomicAdd(&g_dc_clk[1], (unsigned long long)(ck2 - ck1));
    atomicAdd(&g_dc_clk[2], (unsigned long long)(ck3 - ck2));
    atomicAdd(&g_dc_clk[3], 1ull);
  }
  for (int i = tid; i < n; i += nt) lam_out[i] = lam[i];
  for (int idx = tid; idx < n * n; idx += nt) {
    const int i = idx / n, j = idx - (idx / n) * n;   // Vt[i][j] = U[j][i]
    Vt[i * ldvt + j] = Q[j * n + i];
  }
  __syncthreads();
}

}  // namespace ng
