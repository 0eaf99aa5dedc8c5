// eig_jacobi.cuh -- one-CTA symmetric eigensolver (cyclic parallel Jacobi, FP64).
//
// Used for Z_t = U_t C_t U_t^T (eqn:zt:eig, P:990-993 / P:1121-1124), which the paper
// ran on the CPU "in O(R^2)" plus an eigendecomposition; here
// it runs on the device in one CTA so the step never crosses to the host.  Also used
// once per state for the initial top-R eigenpairs of S_0 (B.3.2).
//
// Algorithm: Jacobi rotations in round-robin ("circle") ordering: each round applies
// floor(n/2) disjoint plane rotations simultaneously.  A' = J^T A J is done as
// independent 2x2 block updates  A'[P,Q] = G_P^T A[P,Q] G_Q  (P, Q index rotation
// pairs), so one round costs one barrier after computing the rotations and one after
// the update.  The rotation angle is computed in FP32 and turned into an exactly
// orthogonal FP64 rotation (c = rsqrt(1 + t^2), s = t c), so convergence is governed by
// the FP64 skip threshold while the per-round latency chain stays short.  Eigenvectors are accumulated as ROWS of Vt (Vt = U^T).  Sweeps stop when
// a full sweep performs no rotation (|a_pq| <= rel_tol sqrt(|a_pp a_qq|), rel_tol =
// 1e-12 by default, or below an absolute floor), or after max_sweeps.
//
// A and Vt may live in shared or global memory (generic addressing).
#pragma once

#include <type_traits>

#include "ng_common.cuh"

namespace ng {

struct JacobiScratch {  // shared memory, sized for m = ceil(n/2) pairs
  int* pp;
  int* qq;
  double* c;
  double* s;
  double* t;
  int* nrot;
};

__device__ __forceinline__ void jacobi_pair(int round, int k, int npad, int& p, int& q) {
  // circle method: player npad-1 fixed; the other npad-1 rotate.
  const int m1 = npad - 1;
  if (k == 0) { p = m1; q = round % m1; }
  else { p = (round + k) % m1; q = (round - k + m1) % m1; }
  if (p > q) { int tmp = p; p = q; q = tmp; }
}

// Eigen-decompose the symmetric n x n matrix A (row-major, lda) in place: on return
// the diagonal of A holds the eigenvalues (unsorted), Vt (n x n, ldv) holds the
// eigenvectors as rows.  Must be called by all threads of the CTA.
__device__ void jacobi_eig(double* A, int lda, double* Vt, int ldv, int n, JacobiScratch sc,
                           int max_sweeps, double abs_floor, double rel_tol = 1e-12) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int npad = n + (n & 1);
  const int m = npad / 2;
  for (int idx = tid; idx < n * n; idx += nt) {
    const int i = idx / n, j = idx % n;
    Vt[(int64_t)i * ldv + j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  if (n <= 1) return;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (tid == 0) *sc.nrot = 0;
    __syncthreads();
    for (int round = 0; round < npad - 1; ++round) {
      // ---- rotation parameters for the m disjoint pairs of this round
      for (int k = tid; k < m; k += nt) {
        int p, q;
        jacobi_pair(round, k, npad, p, q);
        double c = 1.0, s = 0.0, t = 0.0;
        if (q < n) {
          const double app = A[(int64_t)p * lda + p], aqq = A[(int64_t)q * lda + q];
          const double apq = A[(int64_t)p * lda + q];
          const double thr = fmax(rel_tol * sqrt(fabs(app * aqq)), abs_floor);
          if (fabs(apq) > thr) {
            // tan of the annihilating angle in FP32 (short latency chain), then an exactly
            // orthogonal FP64 rotation from it: the residual a'_pq ~ 1e-7 a_pq is removed
            // by the next sweep.
            const double thd = (aqq - app) / (2.0 * apq);
            float tf;
            if (fabs(thd) > 1e18) {
              tf = (float)(0.5 / thd);
            } else {
              const float th = (float)thd;
              tf = copysignf(1.f, th) / (fabsf(th) + sqrtf(fmaf(th, th, 1.f)));
            }
            t = (double)tf;
            c = rsqrt(fma(t, t, 1.0));
            s = t * c;
            atomicAdd(sc.nrot, 1);
          }
        }
        sc.pp[k] = p; sc.qq[k] = q; sc.c[k] = c; sc.s[k] = s; sc.t[k] = t;
      }
      __syncthreads();
      // ---- A' = J^T A J as 2x2 block updates over pairs (ka <= kb), mirrored.
      for (int idx = tid; idx < m * m; idx += nt) {
        const int ka = idx % m, kb = idx / m;
        if (ka > kb) continue;
        const int p1 = sc.pp[ka], q1 = sc.qq[ka], p2 = sc.pp[kb], q2 = sc.qq[kb];
        const double c1 = sc.c[ka], s1 = sc.s[ka], c2 = sc.c[kb], s2 = sc.s[kb];
        if (s1 == 0.0 && s2 == 0.0) continue;
        const bool v1 = q1 < n, v2 = q2 < n;
        if (ka == kb) {
          // diagonal block: G^T [[a, b], [b, d]] G
          const double a = A[(int64_t)p1 * lda + p1], d = A[(int64_t)q1 * lda + q1];
          const double b = A[(int64_t)p1 * lda + q1];
          const double cc = c1 * c1, ss = s1 * s1, cs = c1 * s1;
          const double an = cc * a - 2.0 * cs * b + ss * d;
          const double dn = ss * a + 2.0 * cs * b + cc * d;
          const double bn = (cc - ss) * b + cs * (a - d);
          A[(int64_t)p1 * lda + p1] = an;
          A[(int64_t)q1 * lda + q1] = dn;
          A[(int64_t)p1 * lda + q1] = bn;
          A[(int64_t)q1 * lda + p1] = bn;
          continue;
        }
        const double m00 = A[(int64_t)p1 * lda + p2];
        const double m01 = v2 ? A[(int64_t)p1 * lda + q2] : 0.0;
        const double m10 = v1 ? A[(int64_t)q1 * lda + p2] : 0.0;
        const double m11 = (v1 && v2) ? A[(int64_t)q1 * lda + q2] : 0.0;
        // T = G1^T M   (G = [[c, s], [-s, c]])
        const double t00 = c1 * m00 - s1 * m10, t01 = c1 * m01 - s1 * m11;
        const double t10 = s1 * m00 + c1 * m10, t11 = s1 * m01 + c1 * m11;
        // T G2
        const double r00 = c2 * t00 - s2 * t01, r01 = s2 * t00 + c2 * t01;
        const double r10 = c2 * t10 - s2 * t11, r11 = s2 * t10 + c2 * t11;
        A[(int64_t)p1 * lda + p2] = r00; A[(int64_t)p2 * lda + p1] = r00;
        if (v2) { A[(int64_t)p1 * lda + q2] = r01; A[(int64_t)q2 * lda + p1] = r01; }
        if (v1) { A[(int64_t)q1 * lda + p2] = r10; A[(int64_t)p2 * lda + q1] = r10; }
        if (v1 && v2) { A[(int64_t)q1 * lda + q2] = r11; A[(int64_t)q2 * lda + q1] = r11; }
      }
      // ---- Vt rows: row'_p = c row_p - s row_q, row'_q = s row_p + c row_q
      for (int idx = tid; idx < m * n; idx += nt) {
        const int k = idx / n, j = idx % n;
        const double s = sc.s[k];
        if (s == 0.0) continue;
        const double c = sc.c[k];
        const int p = sc.pp[k], q = sc.qq[k];
        const double vp = Vt[(int64_t)p * ldv + j], vq = Vt[(int64_t)q * ldv + j];
        Vt[(int64_t)p * ldv + j] = c * vp - s * vq;
        Vt[(int64_t)q * ldv + j] = s * vp + c * vq;
      }
      __syncthreads();
    }
    const int rot = *sc.nrot;
    __syncthreads();
    if (rot == 0) break;
  }
}

// Sort eigenpairs descending: writes eigenvalues to lam_out[n] and the permuted rows of
// Vt into Vt_out (n x n, ldo).  Ties keep ascending original index (reading R7/R12).
__device__ void eig_sort_desc(const double* A, int lda, const double* Vt, int ldv, int n,
                              double* lam_out, double* Vt_out, int ldo, int* rank_scratch) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < n; i += nt) {
    const double li = A[(int64_t)i * lda + i];
    int r = 0;
    for (int j = 0; j < n; ++j) {
      const double lj = A[(int64_t)j * lda + j];
      r += (lj > li) || (lj == li && j < i);
    }
    rank_scratch[i] = r;
    lam_out[r] = li;
  }
  __syncthreads();
  for (int idx = tid; idx < n * n; idx += nt) {
    const int i = idx / n, j = idx % n;
    Vt_out[(int64_t)rank_scratch[i] * ldo + j] = Vt[(int64_t)i * ldv + j];
  }
  __syncthreads();
}

}  // namespace ng

namespace ng {

// ---------------------------------------------------------------------------------------
// Lean shared-memory variant for the per-update R x R refresh (R <= 112), templated on
// the element type (double in the FP32 path, float in the TF32 path -- the paper ran
// this eigendecomposition in single precision).  The pair table of every round
// and the list of 2x2 blocks are precomputed once, eigenvector rows are rotated with
// contiguous, conflict-free accesses over all threads, warp-uniform skips drop converged
// pairs.  Rotation test without square roots:  a_pq^2 > tol^2 |a_pp a_qq|  and
// a_pq^2 > floor^2.  The angle comes from FP32 and is turned into an exactly orthogonal
// rotation (c = rsqrt(1 + t^2), s = t c) in T.  Stopping: a sweep with no rotation, or a
// sweep whose largest relative off-diagonal was below sqrt(tol) (the rotations of that
// sweep leave O(tol) behind: Jacobi converges quadratically).
//   A: n x n, row stride lda (shared);  Vt: n x n, row stride ldv (shared, 16-byte
//   aligned rows: ldv * sizeof(T) % 16 == 0).  Pairs of round r come from the circle
//   method by arithmetic; each thread's <= 2 blocks (ka <= kb) are decoded once.
// ---------------------------------------------------------------------------------------
template <typename T>
struct JacobiSmem {
  T* c;
  T* s;
  int* nrot;
  float* offmax;
};

template <typename T>
__device__ __forceinline__ T rsqrt_t(T x);
template <>
__device__ __forceinline__ double rsqrt_t<double>(double x) { return rsqrt(x); }
template <>
__device__ __forceinline__ float rsqrt_t<float>(float x) { return rsqrtf(x); }

__device__ __forceinline__ void circle_pair(int r, int k, int m1, int& p, int& q) {
  if (k == 0) { p = m1; q = r; }
  else {
    p = r + k; if (p >= m1) p -= m1;
    q = r - k; if (q < 0) q += m1;
  }
  if (p > q) { const int t = p; p = q; q = t; }
}

template <typename T>
__device__ __forceinline__ int jacobi_eig_smem(T* __restrict__ A, int lda, T* __restrict__ Vt, int ldv, int n,
                                               JacobiSmem<T> sc, int max_sweeps, double abs_floor, double rel_tol,
                                               int dbg = 0) {
  // ldv * sizeof(T) must be a multiple of 16 (vectorised eigenvector rows)
  constexpr int VEC = 16 / sizeof(T);
  using V = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
  using CS = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
  const int npad = n + (n & 1);
  const int m = npad / 2, m1 = npad - 1;
  const int rounds = npad - 1;
  const int nblk = m * (m + 1) / 2;
  const T tol2 = (T)(rel_tol * rel_tol), flo2 = (T)(abs_floor * abs_floor);
  const float stop2 = (float)rel_tol;
  CS* cs2 = reinterpret_cast<CS*>(sc.c);          // (c, s) of pair k, m entries
  int* pqt = sc.nrot + 64;                         // p | q << 16 of pair k (this round)
  // this thread's 2x2 blocks (ka <= kb), decoded once
  int bka[2], bkb[2], nb = 0;   // nblk <= 2 * blockDim (R <= 112 with 1024 threads)
  for (int bb = tid; bb < nblk && nb < 2; bb += nt) {
    int kb = (int)((sqrtf(8.f * bb + 1.f) - 1.f) * 0.5f);
    while (kb * (kb + 1) / 2 > bb) --kb;
    while ((kb + 1) * (kb + 2) / 2 <= bb) ++kb;
    bka[nb] = bb - kb * (kb + 1) / 2;
    bkb[nb] = kb;
    ++nb;
  }
  for (int idx = tid; idx < n * ldv; idx += nt) {
    const int i = idx / ldv, j = idx - i * ldv;
    Vt[idx] = (i == j) ? T(1) : T(0);
  }
  __syncthreads();
  if (n <= 1) return 0;
  const int nvec = (n + VEC - 1) / VEC;   // vectors per eigenvector row
  // this thread's eigenvector items (pair k, vector column j), decoded once
  int vk[4], vj[4], nvi = 0;    // m * nvec <= 4 * blockDim
  for (int it = tid; it < m * nvec && nvi < 4; it += nt) { vk[nvi] = it / nvec; vj[nvi] = it - vk[nvi] * nvec; ++nvi; }
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    int my_rot = 0;          // per-thread counters, reduced once per sweep (no atomics)
    float my_off = 0.f;
    for (int round = 0; round < rounds; ++round) {
      if (tid < m) {
        const int k = tid;
        int p, q;
        circle_pair(round, k, m1, p, q);
        T c = T(1), s = T(0);
        if (q < n) {
          const T app = A[p * lda + p], aqq = A[q * lda + q], apq = A[p * lda + q];
          const T apq2 = apq * apq, dd = fabs(app * aqq);
          if (apq2 > tol2 * dd && apq2 > flo2) {
            my_off = fmaxf(my_off, __fdividef((float)apq2, (float)dd));
            // MUFU-based angle (the FP32 angle only has to be ~1e-7 accurate)
            const float th = __fdividef((float)(aqq - app), 2.f * (float)apq);
            float tf;
            if (!(fabsf(th) < 1e18f)) {
              tf = __fdividef(0.5f, th);
            } else {
              const float r2 = fmaf(th, th, 1.f);
              tf = copysignf(__fdividef(1.f, fabsf(th) + r2 * rsqrtf(r2)), th);
            }
            const T t = (T)tf;
            const T x = t * t + T(1);
            const T c0 = (T)rsqrtf((float)x);
            c = c0 * (T(1.5) - T(0.5) * x * c0 * c0);      // one Newton step: ~1e-14 relative
            s = t * c;
            ++my_rot;
          }
        }
        CS v;
        v.x = c;
        v.y = s;
        cs2[k] = v;
        pqt[k] = p | (q << 16);
      }
      __syncthreads();
      // A' = J^T A J, 2x2 blocks (ka <= kb), mirrored
      for (int i = 0; i < ((dbg & 1) ? 0 : nb); ++i) {
        const int ka = bka[i], kb = bkb[i];
        const CS r1 = cs2[ka], r2 = cs2[kb];
        const T c1 = r1.x, s1 = r1.y, c2 = r2.x, s2 = r2.y;
        if (s1 == T(0) && s2 == T(0)) continue;
        const int pq1 = pqt[ka], pq2 = pqt[kb];
        const int p1 = pq1 & 0xFFFF, q1 = pq1 >> 16, p2 = pq2 & 0xFFFF, q2 = pq2 >> 16;
        const int rp1 = p1 * lda, rq1 = q1 * lda;
        if (ka == kb) {
          const T a = A[rp1 + p1], d = A[rq1 + q1], bb = A[rp1 + q1];
          const T cc = c1 * c1, ss = s1 * s1, csx = c1 * s1;
          const T bn = (cc - ss) * bb + csx * (a - d);
          A[rp1 + p1] = cc * a - T(2) * csx * bb + ss * d;
          A[rq1 + q1] = ss * a + T(2) * csx * bb + cc * d;
          A[rp1 + q1] = bn;
          A[rq1 + p1] = bn;
          continue;
        }
        const int rp2 = p2 * lda, rq2 = q2 * lda;
        const bool v1 = q1 < n, v2 = q2 < n;
        const T m00 = A[rp1 + p2];
        const T m01 = v2 ? A[rp1 + q2] : T(0);
        const T m10 = v1 ? A[rq1 + p2] : T(0);
        const T m11 = (v1 && v2) ? A[rq1 + q2] : T(0);
        const T t00 = c1 * m00 - s1 * m10, t01 = c1 * m01 - s1 * m11;
        const T t10 = s1 * m00 + c1 * m10, t11 = s1 * m01 + c1 * m11;
        const T r00 = c2 * t00 - s2 * t01, r01 = s2 * t00 + c2 * t01;
        const T r10 = c2 * t10 - s2 * t11, r11 = s2 * t10 + c2 * t11;
        A[rp1 + p2] = r00; A[rp2 + p1] = r00;
        if (v2) { A[rp1 + q2] = r01; A[rq2 + p1] = r01; }
        if (v1) { A[rq1 + p2] = r10; A[rp2 + q1] = r10; }
        if (v1 && v2) { A[rq1 + q2] = r11; A[rq2 + q1] = r11; }
      }
      // eigenvector rows p, q of each rotating pair: (pair, vector column) items spread
      // evenly over all threads
      for (int i = 0; i < ((dbg & 2) ? 0 : nvi); ++i) {
        const int k = vk[i], j = vj[i];
        const CS r = cs2[k];
        const T c = r.x, s = r.y;
        if (s == T(0)) continue;
        const int pq = pqt[k];
        V* vp = reinterpret_cast<V*>(Vt + (pq & 0xFFFF) * ldv) + j;
        V* vq = reinterpret_cast<V*>(Vt + (pq >> 16) * ldv) + j;
        const V a = *vp, b = *vq;
        V na, nb2;
        if constexpr (VEC == 2) {
          na.x = c * a.x - s * b.x; na.y = c * a.y - s * b.y;
          nb2.x = s * a.x + c * b.x; nb2.y = s * a.y + c * b.y;
        } else {
          na.x = c * a.x - s * b.x; na.y = c * a.y - s * b.y; na.z = c * a.z - s * b.z; na.w = c * a.w - s * b.w;
          nb2.x = s * a.x + c * b.x; nb2.y = s * a.y + c * b.y; nb2.z = s * a.z + c * b.z; nb2.w = s * a.w + c * b.w;
        }
        *vp = na;
        *vq = nb2;
      }
      __syncthreads();
    }
    // sweep totals (threads >= m contribute 0)
    my_rot = warp_sum(my_rot);
    my_off = warp_max(my_off);
    if (lane == 0) { sc.nrot[warp] = my_rot; sc.offmax[warp] = my_off; }
    __syncthreads();
    int rot = 0;
    float om = 0.f;
    for (int w = 0; w < nwarps; ++w) { rot += sc.nrot[w]; om = fmaxf(om, sc.offmax[w]); }
    __syncthreads();
    if (rot == 0 || om < stop2 || ((dbg & 4) && sweep + 1 >= 5)) { ++sweep; break; }
  }
  return sweep;
}

}  // namespace ng
