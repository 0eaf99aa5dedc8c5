// gemm_tc.cuh -- tcgen05 (5th-gen tensor core) GEMM for sm_100a: TMA-fed operands in
// 128B-swizzled shared memory, accumulators in TMEM, tcgen05.ld epilogue.
//
//   C[M x N] (epilogue)= A[M x K] * B[K x N]
//   A K-major : A[m][k] = A[m*lda + k]      A MN-major : A[m][k] = A[k*lda + m]
//   B K-major : B[k][n] = B[n*ldb + k]      B MN-major : B[k][n] = B[k*ldb + n]
//
// Operands are FP32 in HBM and are consumed by the tensor core as TF32 (kind::tf32,
// FP32 accumulation): no conversion pass and no shadow copies; the same FP32 buffers feed
// the NG-SGD kernels.  split3 = 3xTF32: every landed stage is split in shared memory into
// hi (TF32) + lo (the rest) and A_lo B_hi + A_hi B_lo + A_hi B_hi accumulate in TMEM --
// FP32-grade products on the tensor cores at 3x the MMA work.
#pragma once

#include <cuda.h>

#include "ng_common.cuh"

namespace ng {

enum TcEpiKind : int {
  TC_EPI_STORE = 0,     // C[m][n] = acc
  TC_EPI_AXPY = 1,      // C[m][n] += (*scale) * acc          (weight update, eqn:add:w)
  TC_EPI_PARTIAL = 2,   // C[z][m][n] = acc                    (split-K partials)
  TC_EPI_NGAPPLY = 3,   // C[m][n] -= acc, with per-row partial sums of old^2 / new^2 of this
                        // column tile in xx / pp [blockIdx.x * part_ld + m]  (NG apply)
  TC_EPI_PNORM = 4,     // C[m][n] = acc and the p-norm of each group of 10 columns:
                        // y[m][n/10] = sqrt(sum z^2); the last column tile also writes y[m][N/10]
                        // = 1 (bias input of the next layer) and zeros up to ldy (BN = 80 only)
};

struct TcEpilogue {
  int kind = TC_EPI_STORE;
  float* C = nullptr;
  int64_t ldc = 0;
  int64_t zstride = 0;        // TC_EPI_PARTIAL: elements between split slices
  const float* scale = nullptr;
  float* xx = nullptr;        // TC_EPI_NGAPPLY partial ||x_i||^2
  float* pp = nullptr;        // TC_EPI_NGAPPLY partial ||x_hat_i||^2
  int64_t part_ld = 0;
  float* y = nullptr;         // TC_EPI_PNORM next-layer input [a, 1, 0...], row stride ldy
  int64_t ldy = 0;
};

// Launch one GEMM on `st`.  bn in {32, 64, 128}; splits >= 1 (K split evenly over 32-wide
// k-blocks; with splits > 1 the epilogue must be TC_EPI_PARTIAL).  Pointers must be 16B
// aligned and lda/ldb multiples of 4 (TMA).  Returns the number of splits used via
// *splits_used (may be smaller than requested).
ng_status tc_gemm_tf32(cudaStream_t st, int M, int N, int K, const float* A, int64_t lda, bool a_kmajor,
                       const float* B, int64_t ldb, bool b_kmajor, const TcEpilogue& epi, int bn = 128,
                       int splits = 1, int* splits_used = nullptr, bool split3 = false);

// ---- grouped launch: several independent problems (same majors / epilogue kind / BN)
// in ONE kernel launch; each CTA finds its problem from the tile index.
constexpr int kTcGroupMax = 16;

struct TcGroupDesc {       // host-side description of one problem
  int M, N, K, splits;
  const float* A; int64_t lda;
  const float* B; int64_t ldb;
  TcEpilogue epi;
  int* splits_used;         // optional out
};

struct alignas(64) TcProblem {
  CUtensorMap tmA, tmB;
  int M, N, K, kbps, tile_begin, pad_[3];
  TcEpilogue epi;
};

struct TcGroup {
  TcProblem p[kTcGroupMax];
  int count;
  int nstages;              // smem ring depth = min(kStages, max k-blocks per tile)
};

ng_status tc_gemm_tf32_grouped(cudaStream_t st, const TcGroupDesc* desc, int count, bool a_kmajor, bool b_kmajor,
                               int epi_kind, int bn, bool split3 = false);

// The weight update of every layer, C_g += (*scale_g) A_g B_g (both operands MN-major, TF32):
// a persistent kernel, one CTA per SM, two TMEM accumulators so the read-modify-write
// epilogue of one tile overlaps the mainloop of the next.
ng_status tc_gemm_tf32_axpy_persistent(cudaStream_t st, const TcGroupDesc* desc, int count);

// Forward affine layer fused with the p-norm (G = 10): Z = Y W^T (both K-major,
// Z row stride ldz) and Ynext = [pnorm(Z), 1, 0 ...] (row stride ldy >= N/10 + 1).  N must be
// a multiple of 10.  80-column tiles (8 whole groups each).
ng_status tc_gemm_tf32_pnorm(cudaStream_t st, int M, int N, int K, const float* A, int64_t lda, const float* B,
                             int64_t ldb, float* Z, int64_t ldz, float* Ynext, int64_t ldy, bool split3 = false);

// Split count actually used for a requested split count.
int tc_splits(int K, int splits);

}  // namespace ng
