// gemm_simt.cuh -- generic CUDA-core GEMM used by the FP32 ("paper-faithful")
// path and by the FP64 initialisation.  C = op(A) * op(B), results handed element by
// element to an epilogue functor.  The BF16 path uses the tcgen05 kernels in
// gemm_tc.cuh instead.
//
//   A is M x K:  A_K (K-major)  -> A[m][k] = A[m*lda + k]
//                !A_K (M-major) -> A[m][k] = A[k*lda + m]
//   B is K x N:  B_K (K-major)  -> B[k][n] = B[n*ldb + k]
//                !B_K (N-major) -> B[k][n] = B[k*ldb + n]
//
// Split-K: blockIdx.z covers k in [z*k_split, min(K,(z+1)*k_split)); the epilogue
// receives z so partial sums can be written to separate slices and reduced in a
// fixed order (deterministic, no atomics).
// Gating: if `gate` is non-NULL and *gate == 0 the whole launch is a no-op (used for the
// rarely-taken B.3.1 re-orthogonalisation so the host never synchronises).
#pragma once

#include "ng_common.cuh"

namespace ng {

template <typename T, bool A_K, bool B_K, int BM, int BN, int BK, int TM, int TN, class Epi>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
gemm_simt_kernel(int M, int N, int K, const T* __restrict__ A, int64_t lda,
                 const T* __restrict__ B, int64_t ldb, Epi epi, const int* gate, int k_split) {
  if (gate != nullptr && *gate == 0) return;
  constexpr int NT = (BM / TM) * (BN / TN);
  __shared__ T As[BK][BM + 4];
  __shared__ T Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kb = blockIdx.z * k_split;
  const int ke = min(K, kb + k_split);

  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

  for (int k0 = kb; k0 < ke; k0 += BK) {
    // ---- stage A tile (BM x BK) as As[k][m]
    for (int idx = tid; idx < BM * BK; idx += NT) {
      int mm, kk;
      if (A_K) { mm = idx / BK; kk = idx % BK; } else { kk = idx / BM; mm = idx % BM; }
      const int gm = m0 + mm, gk = k0 + kk;
      T v = T(0);
      if (gm < M && gk < ke) v = A_K ? A[(int64_t)gm * lda + gk] : A[(int64_t)gk * lda + gm];
      As[kk][mm] = v;
    }
    // ---- stage B tile (BK x BN) as Bs[k][n]
    for (int idx = tid; idx < BN * BK; idx += NT) {
      int nn, kk;
      if (B_K) { nn = idx / BK; kk = idx % BK; } else { kk = idx / BN; nn = idx % BN; }
      const int gn = n0 + nn, gk = k0 + kk;
      T v = T(0);
      if (gn < N && gk < ke) v = B_K ? B[(int64_t)gn * ldb + gk] : B[(int64_t)gk * ldb + gn];
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[kk][ty + i * (BM / TM)];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx + j * (BN / TN)];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int gm = m0 + ty + i * (BM / TM);
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int gn = n0 + tx + j * (BN / TN);
      if (gn < N) epi(gm, gn, acc[i][j], (int)blockIdx.z);
    }
  }
}

// Host launcher.  splits >= 1; k_split is rounded to a multiple of BK.
template <typename T, bool A_K, bool B_K, class Epi>
ng_status gemm_simt(cudaStream_t st, int M, int N, int K, const T* A, int64_t lda, const T* B,
                    int64_t ldb, Epi epi, int splits = 1, const int* gate = nullptr) {
  constexpr int BM = 64, BN = 64, BK = 16, TM = 4, TN = 4;
  if (M <= 0 || N <= 0) return NG_OK;
  if (splits < 1) splits = 1;
  int k_split = (int)round_up(ceil_div(K > 0 ? K : 1, splits), BK);
  splits = ceil_div(K > 0 ? K : 1, k_split);
  dim3 grid(ceil_div(N, BN), ceil_div(M, BM), splits);
  gemm_simt_kernel<T, A_K, B_K, BM, BN, BK, TM, TN, Epi>
      <<<grid, (BM / TM) * (BN / TN), 0, st>>>(M, N, K, A, lda, B, ldb, epi, gate, k_split);
  return check_launch("gemm_simt");
}

// Number of splits actually used by gemm_simt for a given K / requested splits.
inline int gemm_simt_splits(int K, int splits) {
  if (splits < 1) splits = 1;
  int k_split = (int)round_up(ceil_div(K > 0 ? K : 1, splits), 16);
  return ceil_div(K > 0 ? K : 1, k_split);
}

// ------------------------------------------------------------------ epilogues

template <typename T>
struct EpiStore {  // C[m][n] = alpha * acc
  T* C; int64_t ldc; T alpha;
  __device__ void operator()(int m, int n, T acc, int) const { C[(int64_t)m * ldc + n] = alpha * acc; }
};

template <typename T>
struct EpiStoreSplit {  // C[z][m][n] = acc  (partials for a fixed-order reduction)
  T* C; int64_t ldc; int64_t zstride;
  __device__ void operator()(int m, int n, T acc, int z) const {
    C[(int64_t)z * zstride + (int64_t)m * ldc + n] = acc;
  }
};

struct EpiAxpyDevScale {  // C[m][n] += (*scale) * acc    (weight update, eqn:add:w)
  float* C; int64_t ldc; const float* scale;
  __device__ void operator()(int m, int n, float acc, int) const {
    C[(int64_t)m * ldc + n] += (*scale) * acc;
  }
};

}  // namespace ng
