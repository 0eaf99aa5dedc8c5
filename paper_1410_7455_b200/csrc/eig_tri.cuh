// eig_tri.cuh -- dense symmetric eigendecomposition for the R x R refresh (eqn:zt:eig:repeat,
// P:1382-1384): Z = U C U^T.  FP64, ONE CTA (1024 threads), n <= kTriMax.
//
//   1. Householder tridiagonalisation Z = Q T Q^T (LAPACK dsytd2 'L' order) with the
//      trailing matrix resident in registers (tri_reduce_reg): one pass per column applies
//      the previous reflector's rank-2 update and forms A_22 v; one warp then forms w, the
//      next column and the next reflector.  2 barriers per column; the reflectors are kept
//      and applied to the eigenvectors at the end (tri_backtransform_reg, barrier-free).
//   2. T is split where an off-diagonal is negligible (relative to its diagonal neighbours,
//      or to eps ||T||).  Each block gets a positive definite root representation
//      L D L^T = T_b - sigma_b I (sigma_b = 0 when T_b factors with D > 0, which Z = Y Y^T
//      makes the usual case), which determines its eigenvalues to high RELATIVE accuracy
//      (Demmel-Kahan).  One thread per eigenvalue: bisection on the stationary-qd negcount
//      until the eigenvalue is isolated, then Rayleigh-quotient steps from the twisted
//      factorisation (stationary top-down + progressive bottom-up qd, twist r = argmin
//      |gamma_r|), safeguarded by the bisection bracket.  The eigenvector is the twisted
//      solve z_r = 1 at the converged shift (Dhillon-Parlett "getvec"); its error is
//      O(n eps / relgap), so the graded tails of Z_t (eigenvalues over 8-20 decades, tiny
//      absolute but large relative gaps) come out orthogonal without any Gram-Schmidt.
//   3. Safety net: X X^T is formed and the solve reports failure when max |X X^T - I| >
//      kTriOrthTol (tight relative clusters, noise-level eigenvalues of a numerically
//      indefinite block); the caller then runs the cyclic Jacobi solver instead.
//   4. The eigenvectors of Z are V = X Q^T (rows): the n-2 reflectors applied to the rows of
//      X in registers.
//
// This replaces 8-13 Jacobi sweeps (79 barrier rounds each at R = 80) with ~2n barriers and
// per-thread qd recurrences.  scratch/ prototypes: tools/tri_proto.py.
#pragma once

#include "ng_common.cuh"

namespace ng {

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


constexpr int kTriMax = 80;
// Threads of a CTA that runs eig_tri: 22 warps (the register-resident tridiagonalisation
// needs 21: a serial warp + 20 warps of four rows each; the multisection 8n = 640 lanes).
// Registers are handed out per 4 warps, so 21-24 warps allow 80 registers per thread against
// 64 at 1024 threads, which removes most of the solver's spills (local memory that misses L1
// once the refresh's shared memory takes most of the unified L1 / shared storage); 96
// registers at 672 threads are refused at launch (24 x 32 x 96 > 65536).
constexpr int kTriThreads = 704;
constexpr int kTriChunks = 5;   // column chunks of the Householder pass
constexpr double kTriOrthTol = 1e-6;   // ~ the Jacobi solver's 1e-7 rotation threshold; W is FP32
constexpr int kTriCoarse = 64;        // coarse negcount points per block (ratio 8 apart)
constexpr int kTriCoarseBlocks = 16;  // blocks of >= kTriCoarseMin indices that get them
constexpr int kTriCoarseMin = 8;
constexpr double kTriClusterTol = 1e-7;   // relative gap below which twisted vectors are redone
                                          // (above it their error n eps / relgap < 2e-7)
__device__ long long g_tri_clk[8];
__device__ long long g_tri_dbg[8];   // finer phase-2 stamps of the last solve (ng_debug_eig_tri ok[8..15])
__device__ unsigned long long g_tri_rqimax;   // slowest eigenvalue's RQI loop (cycles)
__device__ int g_tri_maxit;
__device__ double g_tri_fail_z[kTriMax * kTriMax];   // last Z_t whose solve fell back (ng_debug_tri_fail)
__device__ int g_tri_fail_n, g_tri_fail_count, g_tri_fail_why, g_tri_maxpos;   // thread 0's phase stamps of the last solve (ng_debug_eig_tri)

// Shared-memory plan (offsets in doubles from a 16-byte aligned base), n <= kTriMax.
struct TriPlan {
  int n, lda;
  __host__ __device__ int ldq() const { return kTriMax; }   // reflector rows, zero-padded to 80
  size_t oA, oQ, oX, od, oe, oD, oL, oDL, oDL2, ogu, osig, olam, omu, ov, ow, opb, oqb, otau, ored, oint, total;
};
__host__ __device__ inline TriPlan tri_plan(int n) {
  TriPlan p;
  p.n = n;
  p.lda = n + 1;   // odd row stride: column walks across lanes stay conflict-free
  size_t o = 0;
  auto al = [&]() { o = (o + 1) & ~(size_t)1; };   // 16-byte aligned arrays
  p.oA = o; o += (size_t)n * p.lda; al();   // Householder work; then per-eigenvalue qd scratch; then V
  p.oQ = o; o += (size_t)n * p.ldq(); al();   // reflector rows v_k, zero-padded to kTriMax (16-byte rows)
  p.oX = o; o += (size_t)n * p.lda; al();   // eigenvectors of T (rows)
  p.od = o; o += n; al();                   // diag(T)
  p.oe = o; o += n; al();                   // offdiag(T)
  p.oD = o; o += n; al();                   // root representation D (per block)
  p.oL = o; o += n; al();                   // root representation L
  p.oDL = o; o += n; al();                  // D_i L_i
  p.oDL2 = o; o += n; al();                 // D_i L_i^2
  p.ogu = o; o += n; al();                  // Gershgorin upper bound of the block's L D L^T, per index
  p.osig = o; o += n; al();                 // block shift sigma, per index
  p.olam = o; o += n; al();                 // eigenvalues (index order, unscaled)
  p.omu = o; o += n; al();                  // eigenvalues of the block representations
  p.ov = o; o += 3 * (size_t)n; al();       // reflector vectors (triple buffer)
  p.ow = o; o += 2 * (size_t)kTriMax; al();  // w vectors (double buffer, zero-padded to kTriMax)
  p.opb = o; o += (size_t)kTriChunks * n; al();       // partial sums of A_22 v
  p.oqb = o; o += 2 * (size_t)kTriChunks * n; al();   // partial sums of Q v (double buffer)
  p.otau = o; o += kTriMax; al();           // tau_k of the kept reflectors
  p.ored = o; o += 64; al();
  p.oint = o;   // ints: bstart[n], bend[n], crow[n], cpos[n], status[4], blo[kTriCoarseBlocks], coarse counts
  p.total = sizeof(double) * o + sizeof(int) * (4 * (size_t)n + 4 + kTriCoarseBlocks * (kTriCoarse + 1));
  return p;
}

// Register layout of an n-vector inside a warp: index i lives in lane (i & 31), slot i >> 5.
__device__ __forceinline__ double tri_bcast(const double (&r)[3], int i) {   // i warp-uniform
  const int c = i >> 5;
  const double x = (c == 0) ? r[0] : (c == 1 ? r[1] : r[2]);
  return __shfl_sync(0xffffffffu, x, i & 31);
}


// Reflector from the (already updated) column c held in registers (col[i], i >= c), LAPACK
// dlarfg on rows c+1..n-1: H = I - tau v v^T, H x = beta e_1, v_{c+1} = 1.  One warp;
// writes v (smem), tau, d[c] = col_c, e[c] = beta.
__device__ __forceinline__ void tri_reflect(const double (&col)[3], int c, int n, double* __restrict__ vout,
                                            double* __restrict__ tau_out, double* __restrict__ d,
                                            double* __restrict__ e, int lane) {
  const double alpha = tri_bcast(col, c + 1);
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int i = lane + 32 * q;
    if (i >= c + 2 && i < n) s = fma(col[q], col[q], s);
  }
  s = warp_sum(s);
  double beta, scal, tau;
  if (s == 0.0) {
    beta = alpha; tau = 0.0; scal = 0.0;
  } else {
    beta = -copysign(fsqrt(fma(alpha, alpha, s)), alpha);
    tau = fdiv(beta - alpha, beta);
    scal = frcp(alpha - beta);
  }
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int i = lane + 32 * q;
    if (i < n) vout[i] = (i >= c + 2) ? col[q] * scal : (i == c + 1 ? 1.0 : 0.0);
  }
  const double dc = tri_bcast(col, c);
  if (lane == 0) { d[c] = dc; e[c] = beta; *tau_out = tau; }
}

// Register layout of tri_reduce_reg / tri_backtransform_reg: lane = 8a + b; thread (warp w,
// a, b) owns row i = 4w + a (tri_reduce_reg: 4(w - 1) + a, warp 0 being the serial warp),
// columns j = 10b .. 10b + 9 (n <= 80: 20 warps hold rows).
// A row reduction is then a 3-level shuffle inside an 8-lane group, and every thread reads
// its ten entries of a column vector with five 16-byte shared-memory loads.
constexpr int kTrCols = 10;

__device__ __forceinline__ double tr_rowsum(double x) {   // sum over the 8 lanes of a row group
  x += __shfl_xor_sync(0xffffffffu, x, 1);
  x += __shfl_xor_sync(0xffffffffu, x, 2);
  x += __shfl_xor_sync(0xffffffffu, x, 4);
  return x;
}

// The last columns of the reduction, once the trailing block has at most g_tri_tail rows
// (<= 32 RPL): ONE warp (warp 0) finishes it from shared memory with shuffles and __syncwarp
// only -- the CTA-wide pass of tri_reduce_reg costs two 1024-thread barriers per column,
// which is most of its time when the block is small.  Same dsytd2 'L' steps and outputs as
// tri_reduce_reg: T (= the A region, ld lda) holds A after updates 0..k0-1 in rows / columns
// >= k0 + 1 and reflector k0 is built; writes reflectors k0+1.., taus, d, e.  Lane L owns
// rows g = k0 + 1 + L + 32 r.
template <int RPL>
__device__ __forceinline__ void tri_reduce_tail(const TriPlan& P, double* __restrict__ sm, int k0, int lane) {
  const int n = P.n, lda = P.lda;
  constexpr int ldq = kTriMax;
  double* T = sm + P.oA;
  double* Q = sm + P.oQ;
  double* taus = sm + P.otau;
  double* d = sm + P.od;
  double* e = sm + P.oe;
  double* wsm = sm + P.ow;
  for (int k = k0; k + 2 < n; ++k) {
    const double* v = Q + k * ldq;
    const double tau = taus[k];
    double p[RPL], vg[RPL], w[RPL];
    double dot = 0.0;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int g = k0 + 1 + lane + 32 * r;
      const bool act = g >= k + 1 && g < n;
      double a0 = 0.0, a1 = 0.0;
      if (act) {
        const double* Tg = T + g * lda;
        for (int j = k + 1; j < n; j += 4) {
          double tq[4], vq[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const bool in = j + q < n;
            tq[q] = in ? Tg[j + q] : 0.0;
            vq[q] = in ? v[j + q] : 0.0;
          }
          a0 = fma(tq[0], vq[0], a0);
          a1 = fma(tq[1], vq[1], a1);
          a0 = fma(tq[2], vq[2], a0);
          a1 = fma(tq[3], vq[3], a1);
        }
      }
      p[r] = a0 + a1;
      vg[r] = act ? v[g] : 0.0;
      dot = fma(p[r], vg[r], dot);
    }
    dot = warp_sum(dot);
    const double hk = 0.5 * tau * dot;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int g = k0 + 1 + lane + 32 * r;
      w[r] = tau * fma(-hk, vg[r], p[r]);
      if (g >= k + 1 && g < n) wsm[g] = w[r];
    }
    __syncwarp();
    // A_22 -= v w^T + w v^T
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int g = k0 + 1 + lane + 32 * r;
      if (g >= k + 1 && g < n) {
        double* Tg = T + g * lda;
        // chunks of 4: the loads of a chunk issue together (the stores may alias them)
        for (int j = k + 1; j < n; j += 4) {
          double tq[4], vq[4], wq[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const bool in = j + q < n;
            tq[q] = in ? Tg[j + q] : 0.0;
            vq[q] = in ? v[j + q] : 0.0;
            wq[q] = in ? wsm[j + q] : 0.0;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (j + q < n) Tg[j + q] = fma(-vg[r], wq[q], fma(-w[r], vq[q], tq[q]));
        }
      }
    }
    __syncwarp();
    const int c = k + 1;
    if (c + 2 < n) {
      // reflector of column c (rows c+1..n-1), as tri_reflect
      const double alpha = T[(c + 1) * lda + c];
      double s = 0.0, x[RPL];
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int g = k0 + 1 + lane + 32 * r;
        x[r] = (g >= c + 2 && g < n) ? T[g * lda + c] : 0.0;
        s = fma(x[r], x[r], s);
      }
      s = warp_sum(s);
      double beta, scal, tc;
      if (s == 0.0) {
        beta = alpha; tc = 0.0; scal = 0.0;
      } else {
        beta = -copysign(fsqrt(fma(alpha, alpha, s)), alpha);
        tc = fdiv(beta - alpha, beta);
        scal = frcp(alpha - beta);
      }
      double* vo = Q + c * ldq;
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int g = k0 + 1 + lane + 32 * r;
        if (g >= c + 2 && g < n) vo[g] = x[r] * scal;
      }
      if (lane == 0) { vo[c + 1] = 1.0; d[c] = T[c * lda + c]; e[c] = beta; taus[c] = tc; }
    } else if (lane == 0) {
      d[c] = T[c * lda + c];
      e[c] = T[(n - 1) * lda + c];
      d[n - 1] = T[(n - 1) * lda + n - 1];
    }
    __syncwarp();
  }
}
constexpr int kTriTailRPL = 1;   // rows per lane of the one-warp tail
__device__ int g_tri_tail = 32 * kTriTailRPL;   // tail size (rows); 0 = CTA-wide pass throughout (NG_TUNE_TRI_TAIL)

// Step 1 (register-resident): A (n x n symmetric, ld lda, scaled, in shared memory) ->
// d, e; the reflectors are kept, not accumulated: v_k in row k of the Q region (v_k[i] at
// Q[k kTriMax + i], v_k[k+1] = 1, zero elsewhere up to kTriMax), tau_k at taus[k].  The
// trailing matrix lives in registers for the whole reduction (layout above), so it never
// touches shared memory; every column vector is zero-padded to kTriMax so the pass is
// branch-free 16-byte loads.  Per column k, ONE pass applies update k-1 (A -= v w^T + w v^T)
// and forms p = A v_k, and the owner of column k+1 publishes it; then warp 0 (which holds
// no rows) forms w_k = tau (p - (tau/2)(p.v) v), updates column k+1 by it and builds
// reflector k+1.  Two barriers per column (LAPACK dsytd2 'L' order).
__device__ __noinline__ void tri_reduce_reg(const TriPlan& P, double* __restrict__ sm) {
  const int n = P.n, lda = P.lda, tid = threadIdx.x, nt = blockDim.x;
  constexpr int ldq = kTriMax;
  const int lane = tid & 31, warp = tid >> 5, ra = lane >> 3, cb = lane & 7;
  // warp 0 runs the serial part and holds no rows (its registers go to the reflector)
  const int row = 4 * (warp - 1) + ra, j0 = kTrCols * cb;
  const bool rwarp = warp >= 1 && 4 * (warp - 1) < n;
  const double* A = sm + P.oA;
  double* Q = sm + P.oQ;        // reflector rows
  double* taus = sm + P.otau;
  double* d = sm + P.od;
  double* e = sm + P.oe;
  double* wb = sm + P.ow;       // w by parity
  double* pA = sm + P.opb;      // p = A_22 v_k
  double* colb = sm + P.oqb;    // column k+1 after updates 0..k-1
  double* ann = sm + P.ored;    // A[n-1][n-1] after updates 0..k-1
  if (n <= 2) {
    if (tid == 0) {
      d[0] = A[0];
      if (n == 2) { d[1] = A[lda + 1]; e[0] = A[lda]; }
    }
    __syncthreads();
    return;
  }
  for (int i = tid; i < n * ldq; i += nt) Q[i] = 0.0;
  for (int i = tid; i < 2 * ldq; i += nt) wb[i] = 0.0;
  const bool own = rwarp && row < n;
  // columns k >= k0 (trailing block <= g_tri_tail rows) go to the one-warp tail
  const int k0 = max(0, n - 1 - min(g_tri_tail, 32 * kTriTailRPL));
  double M[kTrCols];
#pragma unroll
  for (int g = 0; g < kTrCols; ++g) M[g] = (own && j0 + g < n && k0 > 0) ? A[row * lda + j0 + g] : 0.0;
  __syncthreads();
  if (warp == 0) {
    double col[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int i = lane + 32 * q;
      col[q] = (i < n) ? A[i * lda] : 0.0;
    }
    tri_reflect(col, 0, n, Q, taus, d, e, lane);
  }
  __syncthreads();
  for (int k = 0; k + 2 < n; ++k) {
    const int cur = k & 1, prv = cur ^ 1;
    const double* v = Q + k * ldq;
    if (k == k0) {
      // hand over: apply update k0-1 and store rows / columns >= k0+1 back into the A region
      // (at k0 = 0 it still holds the input), then warp 0 finishes alone
      if (k0 > 0 && rwarp && 4 * (warp - 1) + 3 >= k + 1) {
        const double vr = own ? Q[(k - 1) * ldq + row] : 0.0;
        const double wr = own ? wb[prv * ldq + row] : 0.0;
        const double* vp = Q + (k - 1) * ldq + j0;
        const double* wp = wb + prv * ldq + j0;
        double* Aw = sm + P.oA;
#pragma unroll
        for (int g = 0; g < kTrCols; ++g) {
          const double x = fma(-vr, wp[g], fma(-wr, vp[g], M[g]));
          if (own && row >= k + 1 && j0 + g >= k + 1 && j0 + g < n) Aw[row * lda + j0 + g] = x;
        }
      }
      __syncthreads();
      if (warp == 0) tri_reduce_tail<kTriTailRPL>(P, sm, k0, lane);
      __syncthreads();
      return;
    }
    // warp-uniform: the row-group shuffles need every lane of the warp; warps whose rows
    // are all above the trailing block (<= k) are finished and skip the pass
    if (rwarp && 4 * (warp - 1) + 3 >= k + 1) {
      // column vectors streamed from shared memory two entries at a time (holding them
      // would need 60 more registers than a 1024-thread CTA allows)
      const double2* v2 = reinterpret_cast<const double2*>(v + j0);
      const double2* vp2 = reinterpret_cast<const double2*>(Q + (k > 0 ? k - 1 : 0) * ldq + j0);
      const double2* wp2 = reinterpret_cast<const double2*>(wb + prv * ldq + j0);
      // (at k = 0 both w buffers are still zero, so the update is a no-op)
      const double vr = own ? Q[(k > 0 ? k - 1 : 0) * ldq + row] : 0.0;
      const double wr = own ? wb[prv * ldq + row] : 0.0;
      double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
      for (int q = 0; q < kTrCols / 2; ++q) {
        const double2 x = v2[q], y = vp2[q], z = wp2[q];
        M[2 * q] = fma(-vr, z.x, fma(-wr, y.x, M[2 * q]));
        M[2 * q + 1] = fma(-vr, z.y, fma(-wr, y.y, M[2 * q + 1]));
        acc0 = fma(M[2 * q], x.x, acc0);
        acc1 = fma(M[2 * q + 1], x.y, acc1);
      }
      const double acc = tr_rowsum(acc0 + acc1);
      if (own && cb == 0) pA[row] = acc;
      // publish column k+1 (slot selected with compile-time indices: a runtime M[g] would
      // move M to local memory) and A[n-1][n-1]
      const int c = k + 1;
      if (own && c / kTrCols == cb) {
        double x = 0.0;
#pragma unroll
        for (int g = 0; g < kTrCols; ++g) if (j0 + g == c) x = M[g];
        colb[row] = x;
      }
      if (row == n - 1 && (n - 1) / kTrCols == cb) {
        double x = 0.0;
#pragma unroll
        for (int g = 0; g < kTrCols; ++g) if (j0 + g == n - 1) x = M[g];
        *ann = x;
      }
    }
    __syncthreads();
    if (warp == 0) {
      // w_k = tau (p - (tau/2)(p.v) v), column c = k+1 after update k, reflector c
      const int c = k + 1;
      const double tau = taus[k];
      double pr[3], vr[3], w[3], col[3];
      double dot = 0.0;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int i = lane + 32 * q;
        const bool in = i >= c && i < n;
        pr[q] = in ? pA[i] : 0.0;
        vr[q] = in ? v[i] : 0.0;
        col[q] = in ? colb[i] : 0.0;
        dot = fma(pr[q], vr[q], dot);
      }
      dot = warp_sum(dot);
      const double hk = 0.5 * tau * dot;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        w[q] = tau * fma(-hk, vr[q], pr[q]);
        const int i = lane + 32 * q;
        if (i < n) wb[cur * ldq + i] = w[q];
      }
      const double vc = tri_bcast(vr, c), wc = tri_bcast(w, c);
#pragma unroll
      for (int q = 0; q < 3; ++q) col[q] = fma(-vr[q], wc, fma(-w[q], vc, col[q]));
      if (c + 2 < n) {
        tri_reflect(col, c, n, Q + c * ldq, taus + c, d, e, lane);
      } else {
        const int l = n - 1;
        const double dc = tri_bcast(col, c), el = tri_bcast(col, l);
        const double vl = tri_bcast(vr, l), wl = tri_bcast(w, l);
        if (lane == 0) {
          d[c] = dc;
          e[c] = el;
          d[l] = fma(-2.0 * vl, wl, *ann);
        }
      }
    }
    __syncthreads();
  }
}

// V = X Q^T with Q = H_0 H_1 ... H_{n-3} (the reflectors tri_reduce_reg keeps): row i of
// V is the i-th eigenvector of Z.  Rows of X in registers (layout above); V <- V H_k for
// k = n-3 .. 0.  Every row reduction stays inside an 8-lane group: no barrier at all.
// Writes V into `out` (ld lda).
__device__ __forceinline__ void tri_backtransform_reg(const TriPlan& P, const double* __restrict__ sm,
                                                      const double* __restrict__ X, double* __restrict__ out) {
  const int n = P.n, lda = P.lda, tid = threadIdx.x;
  constexpr int ldq = kTriMax;
  const int lane = tid & 31, warp = tid >> 5, ra = lane >> 3, cb = lane & 7;
  const int row = 4 * warp + ra, j0 = kTrCols * cb;
  const double* Q = sm + P.oQ;
  const double* taus = sm + P.otau;
  if (4 * warp >= n) return;   // warp-uniform: the row-group shuffles need every lane
  const bool own = row < n;
  double M[kTrCols];
#pragma unroll
  for (int g = 0; g < kTrCols; ++g) M[g] = (own && j0 + g < n) ? X[row * lda + j0 + g] : 0.0;
  for (int k = n - 3; k >= 0; --k) {
    const double2* v2 = reinterpret_cast<const double2*>(Q + k * ldq + j0);
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int q = 0; q < kTrCols / 2; ++q) {
      const double2 x = v2[q];
      s0 = fma(M[2 * q], x.x, s0);
      s1 = fma(M[2 * q + 1], x.y, s1);
    }
    const double s = -taus[k] * tr_rowsum(s0 + s1);
#pragma unroll
    for (int q = 0; q < kTrCols / 2; ++q) {
      const double2 x = v2[q];
      M[2 * q] = fma(s, x.x, M[2 * q]);
      M[2 * q + 1] = fma(s, x.y, M[2 * q + 1]);
    }
  }
#pragma unroll
  for (int g = 0; g < kTrCols; ++g)
    if (own && j0 + g < n) out[row * lda + j0 + g] = M[g];
}

// Reciprocal from MUFU.RCP64H plus one Newton step (relative error ~2^-44): the negcount
// only needs the signs of the D+_i, and a 2^-44 relative perturbation of each ratio is a
// tiny relative perturbation of the representation's entries (Demmel-Kahan), so the count
// stays that of a representation relatively close to L D L^T.
__device__ __forceinline__ double rcp1(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return fma(r, fma(-x, r, 1.0), r);
}

// Stationary qd (dstqds) negcount of L D L^T - lam on block [lo, hi): the number of
// eigenvalues of the block's representation below lam.  DL2_i = D_i L_i^2.
__device__ __forceinline__ int tri_negcount(const double* __restrict__ D, const double* __restrict__ DL2, int lo, int hi,
                                            double lam, double pivmin) {
  int neg = 0;
  double s = -lam;
  for (int i = lo; i < hi - 1; ++i) {
    double dp = D[i] + s;
    if (fabs(dp) < pivmin) dp = -pivmin;
    neg += dp < 0.0;
    s = fma(DL2[i] * rcp1(dp), s, -lam);
  }
  double dp = D[hi - 1] + s;
  if (fabs(dp) < pivmin) dp = -pivmin;
  return neg + (dp < 0.0);
}

// Twisted factorisation of L D L^T - lam on [lo, hi) (Dhillon-Parlett): stationary qd
// top-down (L+_i -> x[i], s_i -> sc[i]), progressive qd bottom-up (U-_i overwrites sc[i]
// once gamma_i = s_i + p_i + lam is formed), twist r = argmin |gamma_i|; z_r = 1,
// z_i = -L+_i z_{i+1} (i < r), z_{i+1} = -U-_i z_i (i >= r).  z -> x[lo..hi-1].  Returns the
// negcount; gamma_r and ||z||^2 out.
__device__ __forceinline__ int tri_twisted(const double* __restrict__ D, const double* __restrict__ L,
                                           const double* __restrict__ DL, const double* __restrict__ DL2, int lo,
                                           int hi, double lam, double pivmin, double* __restrict__ x,
                                           double* __restrict__ sc, double* gamma_out, double* znorm2_out) {
  int neg = 0;
  double s = -lam;
  for (int i = lo; i < hi - 1; ++i) {
    sc[i] = s;
    double dp = D[i] + s;
    if (fabs(dp) < pivmin) dp = -pivmin;
    neg += dp < 0.0;
    const double lp = fdiv(DL[i], dp);
    x[i] = lp;
    s = fma(lp * L[i], s, -lam);
  }
  {
    double dp = D[hi - 1] + s;
    if (fabs(dp) < pivmin) dp = -pivmin;
    neg += dp < 0.0;
  }
  double p = D[hi - 1] - lam;
  int r = hi - 1;
  double gbest = s + p + lam;
  for (int i = hi - 2; i >= lo; --i) {
    double dm = DL2[i] + p;
    if (fabs(dm) < pivmin) dm = -pivmin;
    const double rd = frcp(dm);
    const double si = sc[i];
    sc[i] = DL[i] * rd;                 // U-_i = D_i L_i / D-_{i+1}
    p = fma(p, D[i] * rd, -lam);
    const double g = si + p + lam;
    if (fabs(g) < fabs(gbest)) { gbest = g; r = i; }
  }
  double nrm = 1.0, zn = 1.0, znn = 0.0;   // z_{i+1}, z_{i+2} on the upward walk
  for (int i = r - 1; i >= lo; --i) {
    double z = -x[i] * zn;
    if (zn == 0.0 && i + 2 < hi) z = -fdiv(DL[i + 1], DL[i]) * znn;   // restart across a zero (dlar1v)
    x[i] = z;
    nrm = fma(z, z, nrm);
    znn = zn;
    zn = z;
  }
  x[r] = 1.0;
  zn = 1.0;
  znn = 0.0;
  for (int i = r; i < hi - 1; ++i) {
    double z = -sc[i] * zn;
    if (zn == 0.0 && i > lo) z = -fdiv(DL[i - 1], DL[i]) * znn;
    x[i + 1] = z;
    nrm = fma(z, z, nrm);
    znn = zn;
    zn = z;
  }
  *gamma_out = gbest;
  *znorm2_out = nrm;
  return neg;
}

// tri_twisted on TWO threads of one warp (role 0 = lane `base`, role 1 = lane `base + 1`,
// both in `pmask`): the stationary top-down and the progressive bottom-up qd recurrences are
// independent, so role 0 runs the top-down walk and role 1 the bottom-up one, meeting at
// m = lo + (hi - 1 - lo) / 2.  Phase 1: role 0 does i < m (s_i kept in sc[i], L+_i in x[i]),
// role 1 does i >= m (U-_i in sc[i], p_i parked in x[i]).  Phase 2 (after a __syncwarp):
// role 0 does i >= m, reading p_i and forming gamma_i = s_i + p_i + lam before it writes L+_i
// over it; role 1 does i < m, reading s_i before it writes U-_i.  Every recurrence value and
// every gamma_i is the same arithmetic as tri_twisted; the twist r is the same argmin (ties:
// the largest index).  The two halves of the vector walk (up from r, down from r) run on the
// two roles as well; only the summation order of ||z||^2 differs from tri_twisted.  Both roles
// return the same neg / gamma / ||z||^2.
__device__ __forceinline__ int tri_twisted2(int role, unsigned pmask, int base, const double* __restrict__ D,
                                            const double* __restrict__ L, const double* __restrict__ DL,
                                            const double* __restrict__ DL2, int lo, int hi, double lam,
                                            double pivmin, double* __restrict__ x, double* __restrict__ sc,
                                            double* gamma_out, double* znorm2_out) {
  const int m = lo + (hi - 1 - lo) / 2;
  int neg = 0, r = hi - 1;
  double gbest = 0.0, s = -lam, p = D[hi - 1] - lam;
  if (role == 0) {
    for (int i = lo; i < m; ++i) {
      sc[i] = s;
      double dp = D[i] + s;
      if (fabs(dp) < pivmin) dp = -pivmin;
      neg += dp < 0.0;
      const double lp = fdiv(DL[i], dp);
      x[i] = lp;
      s = fma(lp * L[i], s, -lam);
    }
  } else {
    x[hi - 1] = p;
    for (int i = hi - 2; i >= m; --i) {
      double dm = DL2[i] + p;
      if (fabs(dm) < pivmin) dm = -pivmin;
      const double rd = frcp(dm);
      sc[i] = DL[i] * rd;
      p = fma(p, D[i] * rd, -lam);
      x[i] = p;
    }
  }
  __syncwarp(pmask);
  if (role == 0) {
    bool first = true;
    for (int i = m; i < hi - 1; ++i) {
      const double g = s + x[i] + lam;
      if (first || fabs(g) <= fabs(gbest)) { gbest = g; r = i; first = false; }
      double dp = D[i] + s;
      if (fabs(dp) < pivmin) dp = -pivmin;
      neg += dp < 0.0;
      const double lp = fdiv(DL[i], dp);
      x[i] = lp;
      s = fma(lp * L[i], s, -lam);
    }
    {
      double dp = D[hi - 1] + s;
      if (fabs(dp) < pivmin) dp = -pivmin;
      neg += dp < 0.0;
      const double g = s + x[hi - 1] + lam;
      if (first || fabs(g) <= fabs(gbest)) { gbest = g; r = hi - 1; }
    }
  } else {
    bool first = true;
    for (int i = m - 1; i >= lo; --i) {
      double dm = DL2[i] + p;
      if (fabs(dm) < pivmin) dm = -pivmin;
      const double rd = frcp(dm);
      const double si = sc[i];
      sc[i] = DL[i] * rd;
      p = fma(p, D[i] * rd, -lam);
      const double g = si + p + lam;
      if (first || fabs(g) < fabs(gbest)) { gbest = g; r = i; first = false; }
    }
    if (first) r = -1;   // empty lower half
  }
  // combine: the upper half (role 0) wins ties
  const double g0 = __shfl_sync(pmask, gbest, base), g1 = __shfl_sync(pmask, gbest, base + 1);
  const int r0 = __shfl_sync(pmask, r, base), r1 = __shfl_sync(pmask, r, base + 1);
  neg = __shfl_sync(pmask, neg, base);
  if (r1 >= 0 && fabs(g1) < fabs(g0)) { gbest = g1; r = r1; } else { gbest = g0; r = r0; }
  __syncwarp(pmask);   // x (L+, p_{hi-1}) and sc (U-) complete before the walks
  double part = 0.0;
  if (role == 0) {
    double zn = 1.0, znn = 0.0;   // z_{i+1}, z_{i+2} on the upward walk
    for (int i = r - 1; i >= lo; --i) {
      double z = -x[i] * zn;
      if (zn == 0.0 && i + 2 < hi) z = -fdiv(DL[i + 1], DL[i]) * znn;   // restart across a zero (dlar1v)
      x[i] = z;
      part = fma(z, z, part);
      znn = zn;
      zn = z;
    }
    x[r] = 1.0;
  } else {
    double zn = 1.0, znn = 0.0;
    for (int i = r; i < hi - 1; ++i) {
      double z = -sc[i] * zn;
      if (zn == 0.0 && i > lo) z = -fdiv(DL[i - 1], DL[i]) * znn;
      x[i + 1] = z;
      part = fma(z, z, part);
      znn = zn;
      zn = z;
    }
  }
  const double u0 = __shfl_sync(pmask, part, base), u1 = __shfl_sync(pmask, part, base + 1);
  __syncwarp(pmask);
  *gamma_out = gbest;
  *znorm2_out = 1.0 + u0 + u1;
  return neg;
}

// C[i][j] = sum_k A[i][k] B[j][k] (n x n, FP64, shared memory, ld ldx), 4 x 4 per thread with
// rows i = ti + g a, columns j = tj + g b (g = ceil(n / 4)).  Returns max |C - I| over the
// block when `dev_only` (C not written), else writes C.
__device__ __forceinline__ double tri_gemm_nt(const double* __restrict__ Am, const double* __restrict__ Bm, int n,
                                              int ldx, double* __restrict__ C, int ldc, bool dev_only,
                                              double* __restrict__ red) {
  const int g = (n + 3) >> 2;
  const int tid = threadIdx.x;
  double dev = 0.0;
  for (int t = tid; t < g * g; t += blockDim.x) {
    const int ti = t / g, tj = t - ti * g;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    int ia[4], jb[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      ia[a] = min(ti + g * a, n - 1);
      jb[a] = min(tj + g * a, n - 1);
    }
    for (int k = 0; k < n; ++k) {
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) { av[a] = Am[ia[a] * ldx + k]; bv[a] = Bm[jb[a] * ldx + k]; }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = ti + g * a;
      if (i >= n) continue;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int j = tj + g * b;
        if (j >= n) continue;
        if (dev_only) {
          const double x = acc[a][b] - (i == j ? 1.0 : 0.0);
          dev = (x == x) ? fmax(dev, fabs(x)) : INFINITY;
        } else {
          C[i * ldc + j] = acc[a][b];
        }
      }
    }
  }
  if (dev_only) return block_max(dev, red);
  return 0.0;
}

// Full solve.  On entry A (= sm + P.oA, ld P.lda) holds the symmetric matrix.  On success
// (return 1): lam[i] (sm + P.olam, unordered) and eigenvector rows V = sm + P.oA (ld P.lda).
// Returns 0 when the orthogonality check fails (the caller falls back to Jacobi).
__device__ __noinline__ int eig_tri(const TriPlan& P, double* __restrict__ sm, long long* stamps = nullptr) {
  const int n = P.n, lda = P.lda, tid = threadIdx.x, nt = blockDim.x;
  double* A = sm + P.oA;
  double* X = sm + P.oX;
  double* d = sm + P.od;
  double* e = sm + P.oe;
  double* Dr = sm + P.oD;
  double* Lr = sm + P.oL;
  double* sig = sm + P.osig;
  double* lam = sm + P.olam;
  double* red = sm + P.ored;
  int* bstart = reinterpret_cast<int*>(sm + P.oint);
  int* bend = bstart + n;
  int* crow = bend + n;                        // coarse row of the block starting here (-1: none)
  int* cpos = crow + n;                        // position in a relative cluster (0: first / none)
  int* status = cpos + n;                      // [0] ok, [1] max cluster position, [2] coarse rows
  int* blo = status + 4;                       // block start of coarse row b
  int* ccnt = blo + kTriCoarseBlocks;          // coarse counts [kTriCoarseBlocks][kTriCoarse]
  constexpr double eps = 2.220446049250313e-16;
  // scale to max |a_ij| ~ 1 by a power of two (exact)
  double amax = 0.0;
  for (int idx = tid; idx < n * n; idx += nt) {
    const int i = idx / n, j = idx - i * n;
    amax = fmax(amax, fabs(A[i * lda + j]));
  }
  amax = block_max(amax, red);
  if (!(amax > 0.0) || !isfinite(amax)) {
    if (!isfinite(amax)) return 0;
    for (int i = tid; i < n; i += nt) lam[i] = 0.0;
    for (int idx = tid; idx < n * n; idx += nt) {
      const int i = idx / n, j = idx - i * n;
      A[i * lda + j] = (i == j) ? 1.0 : 0.0;
    }
    __syncthreads();
    return 1;
  }
  int ex;
  frexp(amax, &ex);
  const double scale = ldexp(1.0, -ex), unscale = ldexp(1.0, ex);
  for (int idx = tid; idx < n * n; idx += nt) {
    const int i = idx / n, j = idx - i * n;
    A[i * lda + j] *= scale;
  }
  __syncthreads();
  if (tid == 0) g_tri_clk[0] = clock64();
  if (tid == 0 && stamps) stamps[0] = clock64();
  tri_reduce_reg(P, sm);
  if (tid == 0 && stamps) stamps[1] = clock64();
  if (tid == 0) g_tri_clk[1] = clock64();
  // ||T|| and the split
  double tn = 0.0;
  for (int i = tid; i < n; i += nt) tn = fmax(tn, fmax(fabs(d[i]), i + 1 < n ? fabs(e[i]) : 0.0));
  tn = block_max(tn, red);
  // the negligibility test of every off-diagonal in parallel (cpos[] holds the flags until
  // the cluster pass reuses it), then thread 0 walks the flags
  for (int i = tid; i < n; i += nt) {
    bool cut = (i == n - 1);
    if (!cut) {
      const double ei = fabs(e[i]);
      cut = ei <= eps * sqrt(fabs(d[i])) * sqrt(fabs(d[i + 1])) || ei <= 2.0 * eps * tn;
      if (cut) e[i] = 0.0;
    }
    cpos[i] = cut ? 1 : 0;
  }
  __syncthreads();
  if (tid == 0) {
    int s0 = 0;
    status[0] = 1;
    status[2] = 0;
    for (int i = 0; i < n; ++i) {
      const bool cut = cpos[i] != 0;
      if (cut) {
        for (int k = s0; k <= i; ++k) { bstart[k] = s0; bend[k] = i + 1; }
        crow[s0] = -1;
        if (i + 1 - s0 >= kTriCoarseMin && status[2] < kTriCoarseBlocks) {
          crow[s0] = status[2];
          blo[status[2]++] = s0;
        }
        s0 = i + 1;
      }
    }
  }
  __syncthreads();
  if (tid == 0) g_tri_dbg[0] = clock64();
  const double pivmin = 1e-290;
  // root representation per block, L D L^T = T_b - sigma I positive definite
  double* DL = sm + P.oDL;
  double* DL2 = sm + P.oDL2;
  double* gub = sm + P.ogu;
  if (tid < n && bstart[tid] == tid) {
    const int lo = tid, hi = bend[tid];
    double sigma = 0.0;
    bool ok = false;
    for (int attempt = 0; attempt < 64 && !ok; ++attempt) {
      ok = true;
      double di = d[lo] - sigma;
      for (int i = lo; i < hi - 1; ++i) {
        if (!(di > 0.0)) { ok = false; break; }
        Dr[i] = di;
        const double li = fdiv(e[i], di);
        Lr[i] = li;
        DL[i] = e[i];                            // D_i L_i = e_i
        DL2[i] = e[i] * li;
        di = (d[i + 1] - sigma) - DL2[i];
      }
      if (ok && !(di > 0.0)) ok = false;
      if (ok) Dr[hi - 1] = di;
      else sigma = (sigma == 0.0) ? -4.0 * (hi - lo) * eps * tn : 2.0 * sigma;
    }
    if (!ok) { status[0] = 0; g_tri_fail_why = 1; }
    // Gershgorin upper bound of the representation (= of T_b - sigma)
    double gu = 0.0;
    for (int i = lo; i < hi; ++i) {
      double rad = 0.0;
      if (i > lo) rad += fabs(e[i - 1]);
      if (i < hi - 1) rad += fabs(e[i]);
      gu = fmax(gu, (d[i] - sigma) + rad);
    }
    gu *= 1.0 + 4.0 * (hi - lo) * eps;
    for (int i = lo; i < hi; ++i) { sig[i] = sigma; gub[i] = gu; }
  }
  __syncthreads();
  if (tid == 0) g_tri_dbg[1] = clock64();
  if (status[0] == 0) return 0;
  // coarse pass: negcounts of each big block at gu 8^-k, k = 0..kTriCoarse-1 (a thread each)
  for (int t = tid; t < status[2] * kTriCoarse; t += nt) {
    const int b = t / kTriCoarse, k = t - b * kTriCoarse;
    const int lo = blo[b], hi = bend[lo];
    ccnt[b * kTriCoarse + k] = (k == 0) ? (hi - lo) : tri_negcount(Dr, DL2, lo, hi, ldexp(gub[lo], -3 * k), pivmin);
  }
  __syncthreads();
  if (tid == 0) g_tri_clk[5] = clock64();
  // eight threads per eigenvalue: eigenvalue jj (ascending) of the block containing index j.
  // 9-section (8 negcounts per round, geometric spacing while the bracket spans > 2^9) until
  // isolated and 1e-6 wide, then safeguarded RQI by the group's first thread (one Rayleigh
  // correction from there is accurate to ~eps, the second twisted solve gives the vector).
  {
    const int j = tid >> 3, g8 = tid & 7;
    const unsigned gmask = 0xffu << (tid & 24);
    double a = 0.0, b = 0.0;
    int na = 0, nbc = 0;
    if (j < n) {
      const int lo = bstart[j], hi = bend[j], nb = hi - lo, jj = j - lo;
      double* x = X + j * lda;
      for (int c = g8; c < n; c += 8) x[c] = 0.0;
      __syncwarp(gmask);
      if (nb == 1) {
        if (g8 == 0) x[lo] = 1.0;
      } else {
        const double gu = gub[lo];
        a = gu * 1e-300;
        b = gu;
        nbc = nb;
        if (crow[lo] >= 0) {   // tightest coarse bracket of eigenvalue jj
          const int* cc = ccnt + crow[lo] * kTriCoarse;
          for (int k = 1; k < kTriCoarse; ++k) {
            const int c = cc[k];
            const double xk = ldexp(gu, -3 * k);
            if (c <= jj) { a = xk; na = c; break; }
            b = xk; nbc = c;
          }
        }
        for (int it = 0; it < 64; ++it) {
          const bool iso = (na == jj) && (nbc == jj + 1);
          if (iso && (b - a) <= 1e-6 * a) break;
          double xg;
          const int ea = ilogb(a), eb = ilogb(b);
          if (eb - ea >= 9) xg = ldexp(a, ((g8 + 1) * (eb - ea)) / 9);
          else xg = fma((double)(g8 + 1) * (1.0 / 9.0), b - a, a);
          if (!(xg > a && xg < b)) xg = 0.5 * (a + b);
          const int cg = tri_negcount(Dr, DL2, lo, hi, xg, pivmin);
          const unsigned bits = (__ballot_sync(gmask, cg <= jj) >> (tid & 24)) & 0xffu;
          const int f = __ffs(~bits & 0x1ffu) - 1;   // first point with count > jj (8: none)
          const int base = tid & 24;
          const double xa = __shfl_sync(gmask, xg, base + max(f - 1, 0));
          const int ca = __shfl_sync(gmask, cg, base + max(f - 1, 0));
          const double xb = __shfl_sync(gmask, xg, base + min(f, 7));
          const int cb = __shfl_sync(gmask, cg, base + min(f, 7));
          if (f > 0) { a = xa; na = ca; }
          if (f < 8) { b = xb; nbc = cb; }
        }
        if (g8 == 0) {   // the bracket, for the densely packed RQI threads below
          sm[P.ov + j] = a;
          sm[P.ov + n + j] = b;
          sm[P.ov + 2 * n + j] = (double)(na * 256 + nbc);
        }
      }
    }
    __syncthreads();
    if (tid == 0) g_tri_clk[6] = clock64();
    if (tid == 0 && stamps) stamps[2] = clock64();
    // RQI: TWO adjacent lanes per eigenvalue (tri_twisted2 splits each twisted factorisation
    // between them), eigenvalues packed densely over the first 2n threads: the FP64 pipe
    // issues a whole warp per instruction, so one active lane per 8-lane group (the
    // multisection layout) wasted 7/8 of it on these long sequential chains.
    if (tid < 2 * n) {
      const int jr = tid >> 1, role = tid & 1;
      const unsigned pmask = 3u << (tid & 31 & ~1);
      const int pbase = tid & 31 & ~1;
      const int lo = bstart[jr], hi = bend[jr], nb = hi - lo, jj = jr - lo;
      double* x = X + jr * lda;
      double lj = 0.0;
      if (nb == 1) {
        lj = Dr[lo];
      } else {
        double a = sm[P.ov + jr], b = sm[P.ov + n + jr];
        const int pk = (int)sm[P.ov + 2 * n + jr];
        int na = pk >> 8, nbc = pk & 255;
        {
          const long long rq0 = clock64();
          double lc = -1.0, lam_v = 0.0, gm = 0.0, nz = 1.0;
          bool have_vec = false, conv = false;
          double* ss = A + jr * lda;
          int it_used = 0, ntw = 0;
          for (int it = 0; it < 400 && !conv; ++it) {
            ++it_used;
            const bool iso = (na == jj) && (nbc == jj + 1);
            const bool rqi = iso && (b - a) <= 0.5 * a;
            ntw += rqi;
            double l;
            if (rqi && lc > a && lc < b) l = lc;
            else if (b > 4.0 * a) l = sqrt(a) * sqrt(b);
            else l = 0.5 * (a + b);
            int neg;
            if (rqi) {
              neg = tri_twisted2(role, pmask, pbase, Dr, Lr, DL, DL2, lo, hi, l, pivmin, x, ss, &gm, &nz);
              have_vec = true;
              lam_v = l;
            } else {
              neg = tri_negcount(Dr, DL2, lo, hi, l, pivmin);
            }
            if (neg <= jj) { a = l; na = neg; } else { b = l; nbc = neg; }
            if (rqi) {
              const double dl = fdiv(gm, nz);
              lc = l + dl;
              // |dl| <= 64 eps l: the vector solved at l is within 64 eps / relgap (< 2e-7 outside
              // relative clusters) of the eigenvector; the usual rounding floor of gamma / |z|^2
              // is a few n eps, so 4 eps cost a third solve on most eigenvalues
              if (fabs(dl) <= 64.0 * eps * l || (b - a) <= 4.0 * eps * a) conv = true;
            } else if (iso && (b - a) <= 4.0 * eps * a) {
              conv = true;
            }
          }
          if (role == 0) atomicMax(&g_tri_maxit, 1000 * it_used + ntw);
          if (!have_vec || !conv) {
            lam_v = have_vec ? lam_v : 0.5 * (a + b);
            tri_twisted2(role, pmask, pbase, Dr, Lr, DL, DL2, lo, hi, lam_v, pivmin, x, ss, &gm, &nz);
            if (!conv && role == 0) { atomicAnd(status, 0); g_tri_fail_why = 2; }
          }
          lj = lam_v;
          const double inv = rsqrt(nz);
          for (int c = lo + role; c < hi; c += 2) x[c] *= inv;
          if (role == 0) atomicMax(&g_tri_rqimax, (unsigned long long)(clock64() - rq0));
        }
      }
      if (role == 0) {
        lam[jr] = (lj + sig[lo]) * unscale;
        sm[P.omu + jr] = lj;
      }
    }
  }
  __syncthreads();
  if (tid == 0) g_tri_dbg[2] = clock64();
  if (tid == 0 && stamps) stamps[3] = clock64();
  // relative clusters (relgap < kTriClusterTol within a block): the twisted vectors of the
  // members are not reliable (error ~ n eps / relgap).  Every member redoes its vector by two
  // steps of inverse iteration from its own pseudo-random start (in parallel), then each
  // cluster is orthonormalised by modified Gram-Schmidt run twice, one member per step
  // (every later member projects out the current one; one barrier per step).
  {
    const double* mu = sm + P.omu;
    if (tid == 0) {
      int mx = 0;
      for (int j = 0; j < n; ++j) {
        int pos = 0;
        if (j > bstart[j] && fabs(mu[j] - mu[j - 1]) <= kTriClusterTol * fabs(mu[j - 1])) pos = cpos[j - 1] + 1;
        cpos[j] = pos;
        mx = max(mx, pos);
      }
      // a cluster's first member (pos 0 followed by pos 1) is redone too: mark it -1
      for (int j = 0; j + 1 < n; ++j)
        if (cpos[j] == 0 && cpos[j + 1] == 1) cpos[j] = -1;
      status[1] = mx;
      atomicMax(&g_tri_maxpos, mx);
    }
    __syncthreads();
    const int mx = status[1];
    if (mx > 0) {
      if (tid < n && cpos[tid] != 0) {
        const int j = tid, lo = bstart[j], hi = bend[j];
        double* y = X + j * lda;
        double* lp = A + j * lda;             // L+ of the stationary factorisation
        const double l = mu[j];
        uint32_t hsh = 0x9e3779b9u * (uint32_t)(j + 1);
        for (int i = lo; i < hi; ++i) {
          hsh ^= hsh << 13; hsh ^= hsh >> 17; hsh ^= hsh << 5;
          y[i] = (double)(hsh & 0xffffu) * (1.0 / 65536.0) - 0.5;
        }
        for (int it = 0; it < 2; ++it) {
          // (L D L^T - l I) y <- y via L+ D+ L+^T: the stationary factorisation and the
          // forward substitution + diagonal scaling in one top-down walk, then backward
          double sst = -l, yp = 0.0;
          for (int i = lo; i < hi; ++i) {
            double dp = Dr[i] + sst;
            if (fabs(dp) < pivmin) dp = -pivmin;
            const double yi = (i > lo) ? fma(-lp[i - 1], yp, y[i]) : y[i];
            yp = yi;
            y[i] = fdiv(yi, dp);
            if (i < hi - 1) {
              const double q = fdiv(DL[i], dp);
              lp[i] = q;
              sst = fma(q * Lr[i], sst, -l);
            }
          }
          double ymax = fabs(y[hi - 1]);
          for (int i = hi - 2; i >= lo; --i) { y[i] = fma(-lp[i], y[i + 1], y[i]); ymax = fmax(ymax, fabs(y[i])); }
          const double isc = (ymax > 0.0 && isfinite(ymax)) ? 1.0 / ymax : 1.0;
          for (int i = lo; i < hi; ++i) y[i] *= isc;
        }
      }
      __syncthreads();
      // MGS twice over cluster positions: at step p the member at position p-1 of every
      // cluster is final (normalised); the members after it project it out.  A warp per
      // member (members j = warp, warp + 32, ...), lanes over the vector's entries.
      const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
      for (int rep = 0; rep < 2; ++rep) {
        for (int p = 0; p <= mx; ++p) {
          for (int j = warp; j < n; j += nwarp) {
            if (cpos[j] == 0) continue;   // warp-uniform
            const int lo = bstart[j], hi = bend[j];
            const int pj = cpos[j] < 0 ? 0 : cpos[j];
            if (pj != p) continue;
            double* y = X + j * lda;
            double nr = 0.0;
            for (int i = lo + lane; i < hi; i += 32) nr = fma(y[i], y[i], nr);
            nr = warp_sum(nr);
            const double inr = nr > 0.0 ? rsqrt(nr) : 0.0;
            for (int i = lo + lane; i < hi; i += 32) y[i] *= inr;
          }
          __syncthreads();
          for (int j = warp; j < n; j += nwarp) {
            if (cpos[j] == 0) continue;
            const int lo = bstart[j], hi = bend[j];
            const int pj = cpos[j] < 0 ? 0 : cpos[j];
            if (pj <= p) continue;
            const double* xq = X + (j - (pj - p)) * lda;   // the member at position p
            double* y = X + j * lda;
            double dt = 0.0;
            for (int i = lo + lane; i < hi; i += 32) dt = fma(xq[i], y[i], dt);
            dt = warp_sum(dt);
            for (int i = lo + lane; i < hi; i += 32) y[i] = fma(-dt, xq[i], y[i]);
          }
          __syncthreads();
        }
      }
    }
  }
  if (tid == 0) g_tri_clk[2] = clock64();
  if (tid == 0 && stamps) stamps[4] = clock64();
  if (status[0] == 0) return 0;
  // safety net: orthogonality of the eigenvectors of T
  const double dev = tri_gemm_nt(X, X, n, lda, nullptr, 0, true, red);
  if (tid == 0) g_tri_clk[3] = clock64();
  if (!(dev <= kTriOrthTol)) { if (tid == 0) g_tri_fail_why = 3; return 0; }
  // V = X Q^T (rows = eigenvectors of Z), into the A region
  tri_backtransform_reg(P, sm, X, A);
  __syncthreads();
  if (tid == 0) g_tri_clk[4] = clock64();
  return 1;
}

}  // namespace ng
