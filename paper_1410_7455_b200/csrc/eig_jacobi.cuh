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

// ---------------------------------------------------------------------------------------
// Permuted ping-pong variant (double, n <= kJacobiPPMax): the cyclic circle-method
// Jacobi of jacobi_eig_smem with the data MOVED instead of the pairing: pair k of every
// round is always storage slots (2k, 2k+1), and after each round every row / column goes
// from slot s to slot sigma(s) (T[k] = slot 2k, B[k] = slot 2k+1; T[0] stays, the others
// turn one place: T[k] -> T[k+1], T[m-1] -> B[m-1], B[k] -> B[k-1], B[0] -> T[1]) -- the
// same round-robin tournament, so every pair still meets once per sweep.  Every thread's
// read and write addresses are therefore fixed for the whole solve (no per-round index
// arithmetic), and round g reads buffer g&1 and writes buffer (g+1)&1 (one block barrier
// per round).  Z is stored by 2x2 blocks of slot pairs, upper block triangle only:
// element (r, c), r/2 <= c/2, at (r/2) * ldp + 2c + (r&1); a block is 4 contiguous
// doubles.  Eigenvector rows (Vt) live in slot order too and move with their slot.  The
// rotations of round g+1 are computed during round g by m "angle" threads from the
// round-g inputs and rotations (the entries they need are fixed linear combinations).
// The rotation rule, angle formula and stopping rule are those of jacobi_eig_smem.
// An odd n is padded with a zero row / column (it never rotates).
// ---------------------------------------------------------------------------------------
constexpr int kJacobiPPMax = 80;

__host__ __device__ constexpr int pp_ldp(int npad) { return 2 * npad + 2; }   // 16 B odd multiple

__device__ __forceinline__ int pp_sigma(int s, int m) {
  if (m == 1 || s == 0) return s;
  const int k = s >> 1;
  if ((s & 1) == 0) return (k < m - 1) ? s + 2 : s + 1;
  return (k > 0) ? s - 2 : 2;
}

__device__ __forceinline__ int pp_addr(int r, int c, int ldp) {
  if ((r >> 1) > (c >> 1)) { const int t = r; r = c; c = t; }
  return (r >> 1) * ldp + 2 * c + (r & 1);
}

struct JacobiPPBuf {
  double* Z[2];    // m * ldp each (Z[0] holds the input)
  double* V[2];    // npad * npad each (eigenvector rows by slot)
  double2* cs;     // 2 x m rotations
  int* nrot;       // 32 per-warp counters
  float* offmax;   // 32 per-warp maxima
};

// shared-space accesses by 32-bit byte address (offsets are fixed per thread)
__device__ __forceinline__ uint32_t sh_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ double2 lds_d2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds_d(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_d(uint32_t a, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v)); }
__device__ __forceinline__ void sts_d2(uint32_t a, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y));
}

// ---- thread-block-cluster helpers (the V-split refresh, ngsgd.cu)
__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cl_map(uint32_t local_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mb_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_arm(uint32_t bar, uint32_t bytes) {   // local arrive + expect_tx
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// (default .release.cta semantics, as CUTLASS's cluster pipelines: a cluster-scope release
// would put a MEMBAR.GPU on every round)
__device__ __forceinline__ void mb_arrive_remote(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void mb_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAITC_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void st_async_d2(uint32_t cluster_addr, double2 v, uint32_t cluster_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                   cluster_addr),
               "d"(v.x), "d"(v.y), "r"(cluster_bar)
               : "memory");
}
__device__ __forceinline__ void st_async_u32(uint32_t cluster_addr, uint32_t v, uint32_t cluster_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];" ::"r"(cluster_addr),
               "r"(v), "r"(cluster_bar)
               : "memory");
}
__device__ __forceinline__ double ld_cluster_d(uint32_t cluster_addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(cluster_addr) : "memory");
  return v;
}
__device__ __forceinline__ int ld_cluster_i(uint32_t cluster_addr) {
  int v;
  asm volatile("ld.shared::cluster.b32 %0, [%1];" : "=r"(v) : "r"(cluster_addr) : "memory");
  return v;
}

// Rotation hand-off from the Z CTA (cluster rank 0) to the eigenvector CTAs (ranks
// 1..nv): a ring of `ring` rounds; slot s holds the m rotations of one round plus a
// command word (CONTINUE / STOP).  All addresses are local shared addresses of the
// same-offset arrays (identical layout in every CTA of the cluster).
// round timing (ng_debug_eig_clocks), recorded when dbg & 64
__device__ unsigned long long g_eig_clk[8];

struct PPCluster {
  int nv, ring;
  uint32_t cs_ring;    // V CTAs: ring x m double2
  uint32_t cmd_ring;   // V CTAs: ring x u32
  uint32_t full_bar;   // V CTAs: ring mbarriers (1 local arrive + m*16+4 tx bytes)
  uint32_t empty_bar;  // Z CTA: ring mbarriers (nv remote arrives)
};
constexpr uint32_t kPPContinue = 1u, kPPStop = 2u;

__device__ __forceinline__ void pp_push_cs(const PPCluster& cl, int m, int gn, int kk, double2 v) {
  const int s = gn % cl.ring;
  if (gn >= cl.ring) mb_wait(cl.empty_bar + 8u * s, (uint32_t)((gn / cl.ring) - 1) & 1u);
  for (int r = 1; r <= cl.nv; ++r)
    st_async_d2(cl_map(cl.cs_ring + 16u * (s * m + kk), r), v, cl_map(cl.full_bar + 8u * s, r));
}
__device__ __forceinline__ void pp_push_cmd(const PPCluster& cl, int gn, uint32_t cmd) {
  const int s = gn % cl.ring;
  for (int r = 1; r <= cl.nv; ++r) st_async_u32(cl_map(cl.cmd_ring + 4u * s, r), cmd, cl_map(cl.full_bar + 8u * s, r));
}

// Returns the sweep count; *fb = buffer index holding the result, *phantom = slot of the
// padding row (-1 if n is even).  Thread roles: threads [0, m) own the diagonal blocks,
// [m, m + m(m-1)/2) the off-diagonal blocks (no divergence between the two kinds inside
// a warp), the last m threads compute the next round's rotations; eigenvector items are
// spread over all threads.  Requires m(m+1)/2 <= blockDim - m.
// VLOCAL = false: the eigenvector rows live in the cluster's V CTAs (jacobi_pp_vworker);
// the angle threads push every round's rotations to them through `cl`.
template <bool VLOCAL>
__device__ __forceinline__ int jacobi_pp(JacobiPPBuf b, int n, int max_sweeps, double abs_floor, double rel_tol,
                                         int* fb, int* phantom, int dbg, const PPCluster cl) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
  const int npad = n + (n & 1), m = npad / 2, rounds = npad - 1, ldp = pp_ldp(npad);
  const int noff = m * (m - 1) / 2;
  const double tol2 = rel_tol * rel_tol, flo2 = abs_floor * abs_floor;
  const float stop2 = (float)rel_tol;
  if (VLOCAL)
    for (int idx = tid; idx < npad * npad; idx += nt) {
      const int i = idx / npad, j = idx - i * npad;
      b.V[0][idx] = (i == j && i < n) ? 1.0 : 0.0;
    }
  const uint32_t zb = sh_addr(b.Z[0]), zd = sh_addr(b.Z[1]) - zb;
  const uint32_t vb = VLOCAL ? sh_addr(b.V[0]) : 0u, vd = VLOCAL ? sh_addr(b.V[1]) - vb : 0u;
  const uint32_t csb = sh_addr(b.cs);
  // ---- block role: byte offsets within a Z buffer, fixed for the whole solve
  const bool is_diag = tid < m;
  const bool is_off = tid >= m && tid < m + noff;
  int ka = 0, kb = 0;
  if (is_diag) {
    ka = kb = tid;
  } else if (is_off) {
    const int bb = tid - m;                // strictly upper block triangle, kb >= 1
    kb = (int)((sqrtf(8.f * bb + 1.f) + 1.f) * 0.5f);
    while (kb * (kb - 1) / 2 > bb) --kb;
    while ((kb + 1) * kb / 2 <= bb) ++kb;
    ka = bb - kb * (kb - 1) / 2;
  }
  uint32_t boff = 0, w00 = 0, w01 = 0, w10 = 0, w11 = 0, x00 = 0, x01 = 0, x10 = 0, x11 = 0;
  uint32_t ca = csb + 16u * ka, cbk = csb + 16u * kb;
  int dup = 0;
  if (is_diag || is_off) {
    boff = 8u * (ka * ldp + 4 * kb);
    const int r0 = pp_sigma(2 * ka, m), r1 = pp_sigma(2 * ka + 1, m);
    const int c0 = pp_sigma(2 * kb, m), c1 = pp_sigma(2 * kb + 1, m);
    w00 = 8u * pp_addr(r0, c0, ldp);
    w01 = 8u * pp_addr(r0, c1, ldp);
    w10 = 8u * pp_addr(r1, c0, ldp);
    w11 = 8u * pp_addr(r1, c1, ldp);
    // an off-diagonal element landing inside a next-round diagonal block is stored twice
    if ((r0 >> 1) == (c0 >> 1) && r0 != c0) { dup |= 1; x00 = 8u * pp_addr(c0, r0, ldp); }
    if ((r0 >> 1) == (c1 >> 1) && r0 != c1) { dup |= 2; x01 = 8u * pp_addr(c1, r0, ldp); }
    if ((r1 >> 1) == (c0 >> 1) && r1 != c0) { dup |= 4; x10 = 8u * pp_addr(c0, r1, ldp); }
    if ((r1 >> 1) == (c1 >> 1) && r1 != c1) { dup |= 8; x11 = 8u * pp_addr(c1, r1, ldp); }
  }
  // ---- angle role: pair k of the next round from the slots that move into 2k, 2k+1
  const int angle0 = nt - m;
  const bool is_angle = tid >= angle0;
  const int kk = tid - angle0;
  uint32_t du = 0, dv = 0, mbo = 0, cu = 0, cv = 0;
  int mtr = 0, iu = 0, iv = 0;
  if (is_angle) {
    int u = 0, v = 0;
    for (int s2 = 0; s2 < npad; ++s2) {
      const int t = pp_sigma(s2, m);
      if (t == 2 * kk) u = s2;
      if (t == 2 * kk + 1) v = s2;
    }
    const int pu = u >> 1, pv = v >> 1;
    iu = u & 1; iv = v & 1;
    du = 8u * (pu * ldp + 4 * pu);
    dv = 8u * (pv * ldp + 4 * pv);
    mtr = pu > pv;
    mbo = 8u * (mtr ? pv * ldp + 4 * pu : pu * ldp + 4 * pv);
    cu = 16u * pu;
    cv = 16u * pv;
  }
  // ---- eigenvector items (pair k, double2 column j): rows 2k, 2k+1 -> sigma(2k), sigma(2k+1)
  const int nv2 = npad / 2;
  uint32_t vr[2], vw0[2], vw1[2], vcs[2];
  int nvi = 0;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int it = tid + i * nt;
    vr[i] = vw0[i] = vw1[i] = vcs[i] = 0;
    if (VLOCAL && it < m * nv2) {
      const int k = it / nv2, j = it - k * nv2;
      vcs[i] = 16u * k;
      vr[i] = 8u * ((2 * k) * npad + 2 * j);
      vw0[i] = 8u * (pp_sigma(2 * k, m) * npad + 2 * j);
      vw1[i] = 8u * (pp_sigma(2 * k + 1, m) * npad + 2 * j);
      nvi = i + 1;
    }
  }
  const uint32_t vrow = 8u * npad;
  int rot_cur = 0, rot_next = 0;
  float off_cur = 0.f, off_next = 0.f;
  auto angle = [&](double app, double aqq, double apq, int& rot, float& off) -> double2 {
    double2 r;
    r.x = 1.0;
    r.y = 0.0;
    const double apq2 = apq * apq, dd = fabs(app * aqq);
    if (apq2 > tol2 * dd && apq2 > flo2) {
      off = fmaxf(off, __fdividef((float)apq2, (float)dd));
      const float th = __fdividef((float)(aqq - app), 2.f * (float)apq);
      float tf;
      if (!(fabsf(th) < 1e18f)) {
        tf = __fdividef(0.5f, th);
      } else {
        const float r2 = fmaf(th, th, 1.f);
        tf = copysignf(__fdividef(1.f, fabsf(th) + r2 * rsqrtf(r2)), th);
      }
      const double t = (double)tf;
      const double x = t * t + 1.0;
      const double c0 = (double)rsqrtf((float)x);
      const double c = c0 * (1.5 - 0.5 * x * c0 * c0);
      r.x = c;
      r.y = t * c;
      ++rot;
    }
    return r;
  };
  if (tid == 0) *phantom = (n & 1) ? n : -1;
  __syncthreads();   // input Z[0] complete (caller), V[0] initialised
  if (is_angle) {
    const double* z = b.Z[0] + kk * ldp + 4 * kk;
    const double2 r0 = angle(z[0], z[3], z[2], rot_cur, off_cur);
    b.cs[kk] = r0;
    if (!VLOCAL) {
      pp_push_cs(cl, m, 0, kk, r0);
      if (kk == 0) pp_push_cmd(cl, 0, kPPContinue);
    }
  }
  __syncthreads();
  int sweep = 0, g = 0;
  const uint32_t csd = 16u * m;
  const bool timing = (dbg & 64) != 0;
  unsigned long long ck[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const bool t_angle = timing && is_angle && kk == 0, t_blk = timing && tid == m + 1, t_zero = timing && tid == 0;
  for (; sweep < max_sweeps; ++sweep) {
    for (int round = 0; round < rounds; ++round, ++g) {
      const bool odd = g & 1;
      long long c0 = 0;
      if (timing) c0 = clock64();
      const uint32_t zc = zb + (odd ? zd : 0u), zn = zb + (odd ? 0u : zd);
      const uint32_t vc = vb + (odd ? vd : 0u), vn = vb + (odd ? 0u : vd);
      const uint32_t cc_ = odd ? csd : 0u;
      if (is_off && !(dbg & 16)) {
        const double2 r1 = lds_d2(ca + cc_), r2 = lds_d2(cbk + cc_);
        const double2 u = lds_d2(zc + boff);          // (2ka, 2kb), (2ka+1, 2kb)
        const double2 w = lds_d2(zc + boff + 16u);    // (2ka, 2kb+1), (2ka+1, 2kb+1)
        const double c1 = r1.x, s1 = r1.y, c2 = r2.x, s2 = r2.y;
        const double m00 = u.x, m10 = u.y, m01 = w.x, m11 = w.y;
        long long c1t = 0;
        if (t_blk) {
          asm volatile("" ::"d"(m00), "d"(m11), "d"(c1), "d"(s2));
          c1t = clock64();
          ck[4] += c1t - c0;
        }
        const double t00 = c1 * m00 - s1 * m10, t01 = c1 * m01 - s1 * m11;
        const double t10 = s1 * m00 + c1 * m10, t11 = s1 * m01 + c1 * m11;
        const double r00 = c2 * t00 - s2 * t01, r01 = s2 * t00 + c2 * t01;
        const double r10 = c2 * t10 - s2 * t11, r11 = s2 * t10 + c2 * t11;
        sts_d(zn + w00, r00);
        sts_d(zn + w01, r01);
        sts_d(zn + w10, r10);
        sts_d(zn + w11, r11);
        if (t_blk) ck[5] += clock64() - c1t;
        if (dup) {
          if (dup & 1) sts_d(zn + x00, r00);
          if (dup & 2) sts_d(zn + x01, r01);
          if (dup & 4) sts_d(zn + x10, r10);
          if (dup & 8) sts_d(zn + x11, r11);
        }
      } else if (is_diag && !(dbg & 16)) {
        const double2 r1 = lds_d2(ca + cc_);
        const double2 u = lds_d2(zc + boff);
        const double2 w = lds_d2(zc + boff + 16u);
        const double c1 = r1.x, s1 = r1.y;
        const double a = u.x, bb = w.x, d = w.y;
        const double cc = c1 * c1, ss = s1 * s1, csx = c1 * s1;
        const double bn = (cc - ss) * bb + csx * (a - d);
        sts_d(zn + w00, cc * a - 2.0 * csx * bb + ss * d);
        sts_d(zn + w11, ss * a + 2.0 * csx * bb + cc * d);
        sts_d(zn + w01, bn);
        if (dup & 2) sts_d(zn + x01, bn);   // m == 1 only
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        if (i >= nvi) break;
        const double2 r = lds_d2(csb + vcs[i] + cc_);
        const double2 a = lds_d2(vc + vr[i]);
        const double2 bq = lds_d2(vc + vr[i] + vrow);
        double2 na, nb2;
        na.x = r.x * a.x - r.y * bq.x; na.y = r.x * a.y - r.y * bq.y;
        nb2.x = r.y * a.x + r.x * bq.x; nb2.y = r.y * a.y + r.x * bq.y;
        sts_d2(vn + vw0[i], na);
        sts_d2(vn + vw1[i], nb2);
      }
      if (is_angle) {
        // new row (slot u) = x0 row(2pu) + x1 row(2pu+1), with R = [[c, -s], [s, c]]
        const double2 rP = lds_d2(csb + cu + cc_), rQ = lds_d2(csb + cv + cc_);
        const double xu0 = iu ? rP.y : rP.x, xu1 = iu ? rP.x : -rP.y;
        const double xv0 = iv ? rQ.y : rQ.x, xv1 = iv ? rQ.x : -rQ.y;
        const double2 zu0 = lds_d2(zc + du), zu1 = lds_d2(zc + du + 16u);
        const double2 zv0 = lds_d2(zc + dv), zv1 = lds_d2(zc + dv + 16u);
        const double2 zm0 = lds_d2(zc + mbo), zm1 = lds_d2(zc + mbo + 16u);
        const double app = xu0 * xu0 * zu0.x + 2.0 * xu0 * xu1 * zu1.x + xu1 * xu1 * zu1.y;
        const double aqq = xv0 * xv0 * zv0.x + 2.0 * xv0 * xv1 * zv1.x + xv1 * xv1 * zv1.y;
        // M(i, j) = Z[2pu+i][2pv+j]: stored (i, j) at 2j+i, or transposed at 2i+j
        const double m00 = zm0.x, m11 = zm1.y;
        const double m10 = mtr ? zm1.x : zm0.y, m01 = mtr ? zm0.y : zm1.x;
        const double apq = xu0 * (m00 * xv0 + m01 * xv1) + xu1 * (m10 * xv0 + m11 * xv1);
        const bool wrap = round + 1 == rounds;
        long long a1t = 0;
        if (t_angle) {
          asm volatile("" ::"d"(zu0.x), "d"(zv1.y), "d"(zm0.x), "d"(zm1.y), "d"(rP.x), "d"(rQ.y));
          a1t = clock64();
          ck[1] += a1t - c0;
        }
        double2 rn;
        if (dbg & 32) {   // profiling: fixed rotation, no angle chain
          rn.x = 0.8;
          rn.y = 0.6;
        } else {
          rn = wrap ? angle(app, aqq, apq, rot_next, off_next) : angle(app, aqq, apq, rot_cur, off_cur);
        }
        long long a2t = 0;
        if (t_angle) {
          asm volatile("" ::"d"(rn.x), "d"(rn.y));
          a2t = clock64();
          ck[2] += a2t - a1t;
        }
        sts_d2(csb + (odd ? 0u : csd) + 16u * kk, rn);
        if (!VLOCAL) {
          pp_push_cs(cl, m, g + 1, kk, rn);
          if (kk == 0 && !wrap) pp_push_cmd(cl, g + 1, kPPContinue);
        }
        if (t_angle) { ck[3] += clock64() - a2t; ck[0] += 1; }
      }
      if (tid == 0 && *phantom >= 0) *phantom = pp_sigma(*phantom, m);
      __syncthreads();
      if (t_zero) ck[6] += clock64() - c0;
    }
    int my_rot = warp_sum(rot_cur);
    float my_off = warp_max(off_cur);
    if (lane == 0) { b.nrot[warp] = my_rot; b.offmax[warp] = my_off; }
    rot_cur = rot_next; off_cur = off_next; rot_next = 0; off_next = 0.f;
    __syncthreads();
    int rot = 0;
    float om = 0.f;
    for (int w = 0; w < nwarps; ++w) { rot += b.nrot[w]; om = fmaxf(om, b.offmax[w]); }
    __syncthreads();
    const bool stop = rot == 0 || om < stop2 || ((dbg & 4) && sweep + 1 >= 5) || sweep + 1 >= max_sweeps;
    // the next round's rotations were already pushed; its command decides
    if (!VLOCAL && is_angle && kk == 0) pp_push_cmd(cl, g, stop ? kPPStop : kPPContinue);
    if (stop) { ++sweep; break; }
  }
  if (timing) {
    if (t_angle) for (int i = 0; i < 4; ++i) atomicAdd(&g_eig_clk[i], ck[i]);
    if (t_blk) { atomicAdd(&g_eig_clk[4], ck[4]); atomicAdd(&g_eig_clk[5], ck[5]); }
    if (t_zero) atomicAdd(&g_eig_clk[6], ck[6]);
  }
  *fb = g & 1;
  return sweep;
}

// The eigenvector side of the cluster solve (ranks 1..nv): columns [j0, j0 + w) of the
// slot-ordered eigenvector rows, ping-pong V0/V1 (npad x w, row stride w), rotations of
// round g from ring slot g % ring.  Returns the number of rounds applied (the final
// buffer is rounds & 1).
__device__ __forceinline__ int jacobi_pp_vworker(double* V0, double* V1, int n, int j0, int w,
                                                 const double2* cs_ring, const uint32_t* cmd_ring, const PPCluster cl) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int npad = n + (n & 1), m = npad / 2;
  const int nw2 = w / 2;
  for (int idx = tid; idx < npad * w; idx += nt) {
    const int i = idx / w, j = j0 + (idx - (idx / w) * w);
    V0[idx] = (i == j && i < n) ? 1.0 : 0.0;
  }
  // items (pair k, double2 column j) -- one per thread (m * w / 2 <= blockDim)
  const bool has = tid < m * nw2;
  uint32_t vr = 0, vw0 = 0, vw1 = 0, kcs = 0;
  if (has) {
    const int k = tid / nw2, j = tid - k * nw2;
    kcs = 16u * k;
    vr = 8u * ((2 * k) * w + 2 * j);
    vw0 = 8u * (pp_sigma(2 * k, m) * w + 2 * j);
    vw1 = 8u * (pp_sigma(2 * k + 1, m) * w + 2 * j);
  }
  const uint32_t vb = sh_addr(V0), vd = sh_addr(V1) - vb, vrow = 8u * w;
  const uint32_t csr = sh_addr(cs_ring);
  const uint32_t tx = 16u * m + 4u;
  __syncthreads();
  int g = 0;
  for (;; ++g) {
    const int s = g % cl.ring;
    mb_wait(cl.full_bar + 8u * s, (uint32_t)(g / cl.ring) & 1u);
    if (cmd_ring[s] == kPPStop) break;
    if (has) {
      const bool odd = g & 1;
      const uint32_t vc = vb + (odd ? vd : 0u), vn = vb + (odd ? 0u : vd);
      const double2 r = lds_d2(csr + 16u * (s * m) + kcs);
      const double2 a = lds_d2(vc + vr);
      const double2 bq = lds_d2(vc + vr + vrow);
      double2 na, nb2;
      na.x = r.x * a.x - r.y * bq.x; na.y = r.x * a.y - r.y * bq.y;
      nb2.x = r.y * a.x + r.x * bq.x; nb2.y = r.y * a.y + r.x * bq.y;
      sts_d2(vn + vw0, na);
      sts_d2(vn + vw1, nb2);
    }
    __syncthreads();
    if (tid == 0) {
      mb_arm(cl.full_bar + 8u * s, tx);                 // next use of this slot
      mb_arrive_remote(cl_map(cl.empty_bar + 8u * s, 0));
    }
  }
  return g;
}

}  // namespace ng
