// simple_ng.cu -- the simple natural-gradient preconditioner of Appendix A,
// efficient form A.3, on sm_100a, FP64 arithmetic on FP32 data:
//
//   beta = alpha max(tr X^T X, 1e-20) / (N D)
//   column space (N > D):  Q = X (beta I + X^T X / (N-1))^{-1}
//   row space (N <= D):    Q = (beta I + X X^T / (N-1))^{-1} X
//   a_i = x_i^T q_i,  b_i = 1 + a_i / (N - 1 - a_i),  x_hat_i = b_i q_i
//   gamma = sqrt(tr X^T X / tr X_hat^T X_hat)  (1 if the denominator is 0)
//
// The m x m system (m = min-side, strict N > D for the column space, reading R11) is SPD
// and well conditioned (cond <= 1 + N D / (alpha (N - 1))); it is formed (FP64 Gram),
// factored (FP64 Cholesky, one CTA per problem) and solved (FP64 forward / backward
// substitution, one thread per right-hand side) on the device.  Every kernel takes a job
// table, so the 2I preconditioning calls of a DNN step run as one launch per phase.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "ng_common.cuh"
#include "simple_ng_impl.cuh"

namespace ng {

constexpr int kSimpleMaxJobs = 16;
constexpr int kGramTile = 32;     // 32 x 32 output tile, 256 threads (4 outputs each)
constexpr int kGramK = 32;        // k-chunk staged in shared memory

struct SimpleJob {
  float* X;         // n x D, ld (in place: X -> X_hat)
  int64_t ld;
  int n, D, m, col; // col != 0: column space (m = D, right-hand sides = rows); else row space (m = n)
  double* G;        // m x m: Gram, then beta I + G/(n-1), then its lower Cholesky factor
  double* Y;        // m x rhs: the solves (element (i, r) at Y[i * rhs + r])
  double* rowpart;  // 2 x n: ||x_r||^2, ||x_hat_r||^2
  double* stats;    // [0] tr X^T X [1] beta [2] sum ||x||^2 [3] sum p
  float* gamma;     // 1
  float* p;         // n: ||x_hat_r||^2 (unscaled by gamma)
  int* flags;       // [0] error bits
  float alpha;
  int rhs;
};
struct SimpleJobs {
  SimpleJob j[kSimpleMaxJobs];
  int count;
};

// G = X^T X (column space) or X X^T (row space), FP64 accumulation of the FP32 data; only
// tiles on or below the diagonal (the factorisation reads the lower triangle).
__global__ void __launch_bounds__(256) simple_gram_kernel(const __grid_constant__ SimpleJobs jb) {
  const SimpleJob& J = jb.j[blockIdx.y];
  const int tiles = (J.m + kGramTile - 1) / kGramTile;
  const int ti = blockIdx.x / tiles, tj = blockIdx.x % tiles;   // grid.x = max tiles^2
  if (ti >= tiles || tj > ti) return;
  __shared__ double As[kGramK][kGramTile + 1], Bs[kGramK][kGramTile + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;   // 16 x 16 threads, 2 x 2 outputs
  const int i0 = ti * kGramTile, j0 = tj * kGramTile;
  const int K = J.col ? J.n : J.D;
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int k0 = 0; k0 < K; k0 += kGramK) {
    for (int idx = threadIdx.x; idx < kGramK * kGramTile; idx += 256) {
      const int kk = idx / kGramTile, c = idx % kGramTile, k = k0 + kk;
      double a = 0.0, b = 0.0;
      if (k < K) {
        if (J.col) {   // G[i][j] = sum_r X[r][i] X[r][j]
          if (i0 + c < J.m) a = J.X[(int64_t)k * J.ld + i0 + c];
          if (j0 + c < J.m) b = J.X[(int64_t)k * J.ld + j0 + c];
        } else {       // G[i][j] = sum_c X[i][c] X[j][c]
          if (i0 + c < J.m) a = J.X[(int64_t)(i0 + c) * J.ld + k];
          if (j0 + c < J.m) b = J.X[(int64_t)(j0 + c) * J.ld + k];
        }
      }
      As[kk][c] = a;
      Bs[kk][c] = b;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < kGramK; ++kk) {
      const double a0 = As[kk][ty], a1 = As[kk][ty + 16], b0 = Bs[kk][tx], b1 = Bs[kk][tx + 16];
      acc[0][0] = fma(a0, b0, acc[0][0]);
      acc[0][1] = fma(a0, b1, acc[0][1]);
      acc[1][0] = fma(a1, b0, acc[1][0]);
      acc[1][1] = fma(a1, b1, acc[1][1]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int i = i0 + ty + 16 * u, j = j0 + tx + 16 * v;
      if (i < J.m && j < J.m && j <= i) J.G[(int64_t)i * J.m + j] = acc[u][v];
    }
}

// beta, A = beta I + G/(n-1) and its Cholesky factor A = L L^T (lower, in place, row-major),
// one CTA per job, right-looking and blocked by kCholB columns: the diagonal block is
// factored in shared memory, the panel below it solved against it (a thread per row), then
// the whole panel (<= 512 x kCholB doubles) is staged in shared memory for the trailing
// update A_22 -= P P^T of the lower triangle (every element a kCholB-long dot product).
constexpr int kCholB = 32;
__global__ void __launch_bounds__(1024) simple_chol_kernel(const __grid_constant__ SimpleJobs jb) {
  const SimpleJob& J = jb.j[blockIdx.x];
  const int m = J.m, tid = threadIdx.x, nt = blockDim.x;
  double* G = J.G;
  extern __shared__ __align__(16) double chs[];
  double* Lkk = chs;                      // kCholB x (kCholB + 1)
  double* P = chs + kCholB * (kCholB + 1);  // m x (kCholB + 1): the current panel
  __shared__ double red[32];
  double tr = 0.0;
  for (int i = tid; i < m; i += nt) tr += G[(int64_t)i * m + i];
  tr = block_sum(tr, red);
  const double beta = (double)J.alpha * fmax(tr, 1e-20) / ((double)J.n * (double)J.D);
  const double inv_n1 = 1.0 / (double)(J.n - 1);
  for (int idx = tid; idx < m * m; idx += nt) {
    const int i = idx / m, j = idx % m;
    if (j <= i) G[idx] = G[idx] * inv_n1 + (i == j ? beta : 0.0);
  }
  if (tid == 0) { J.stats[0] = tr; J.stats[1] = beta; }
  __syncthreads();
  constexpr int LD = kCholB + 1;
  for (int k0 = 0; k0 < m; k0 += kCholB) {
    const int bk = min(kCholB, m - k0);
    // (a) the diagonal block, unblocked in shared memory
    for (int idx = tid; idx < bk * bk; idx += nt) {
      const int i = idx / bk, j = idx % bk;
      Lkk[i * LD + j] = (j <= i) ? G[(int64_t)(k0 + i) * m + k0 + j] : 0.0;
    }
    __syncthreads();
    for (int k = 0; k < bk; ++k) {
      if (tid == 0) {
        const double d = Lkk[k * LD + k];
        if (!(d > 0.0)) atomicOr(reinterpret_cast<unsigned*>(J.flags), kErrNotPD);
        Lkk[k * LD + k] = sqrt(fmax(d, 1e-300));
      }
      __syncthreads();
      const double inv = 1.0 / Lkk[k * LD + k];
      for (int i = k + 1 + tid; i < bk; i += nt) Lkk[i * LD + k] *= inv;
      __syncthreads();
      const int r = bk - k - 1;
      for (int idx = tid; idx < r * r; idx += nt) {
        const int i = k + 1 + idx / r, j = k + 1 + idx % r;
        if (j <= i) Lkk[i * LD + j] -= Lkk[i * LD + k] * Lkk[j * LD + k];
      }
      __syncthreads();
    }
    for (int idx = tid; idx < bk * bk; idx += nt) {
      const int i = idx / bk, j = idx % bk;
      if (j <= i) G[(int64_t)(k0 + i) * m + k0 + j] = Lkk[i * LD + j];
    }
    // (b) the panel below: row r solves x L_kk^T = a (a thread per row, x kept in P)
    const int rows = m - k0 - bk;
    for (int r = tid; r < rows; r += nt) {
      const int gi = k0 + bk + r;
      double* x = P + r * LD;
      for (int j = 0; j < bk; ++j) {
        double s2 = G[(int64_t)gi * m + k0 + j];
        for (int t = 0; t < j; ++t) s2 = fma(-x[t], Lkk[j * LD + t], s2);
        x[j] = s2 / Lkk[j * LD + j];
      }
      for (int j = 0; j < bk; ++j) G[(int64_t)gi * m + k0 + j] = x[j];
    }
    __syncthreads();
    // (c) trailing update of the lower triangle: A_ij -= sum_t P_it P_jt
    for (int idx = tid; idx < rows * rows; idx += nt) {
      const int i = idx / rows, j = idx % rows;
      if (j > i) continue;
      double acc = 0.0;
      for (int t = 0; t < bk; ++t) acc = fma(P[i * LD + t], P[j * LD + t], acc);
      G[(int64_t)(k0 + bk + i) * m + k0 + bk + j] -= acc;
    }
    __syncthreads();
  }
}

// kSolveCols right-hand sides per CTA (a row of X in the column space, a column in the row
// space), their vectors in shared memory; L y = b then L^T q = y, eight rows (forward) or
// eight columns (backward) of L staged in shared memory at a time (coalesced, one L2 round
// trip per eight steps), every dot product split over kSolveSplit lanes (3-level shuffle).
// q -> Y (element (i, r) at Y[i * rhs + r]).
constexpr int kSolveCols = 32, kSolveSplit = 8, kSolveBlk = 8;
__global__ void __launch_bounds__(kSolveCols * kSolveSplit) simple_solve_kernel(const __grid_constant__ SimpleJobs jb) {
  const SimpleJob& J = jb.j[blockIdx.y];
  const int m = J.m, rhs = J.rhs, tid = threadIdx.x, nt = blockDim.x;
  const int c = tid / kSolveSplit, g = tid % kSolveSplit;
  if ((int)(blockIdx.x * kSolveCols) >= rhs) return;   // uniform per CTA
  // y of right-hand side c at ys[c * ldy + k] (ldy = m + 1: the eight lanes of a group read
  // consecutive k, the four groups of a warp land on different banks)
  const int ldy = m + 1;
  extern __shared__ __align__(16) double ys[];
  double* Lb = ys + (size_t)kSolveCols * ldy;       // kSolveBlk x m: rows (forward) / columns (backward) of L
  const double* L = J.G;
  for (int idx = tid; idx < m * kSolveCols; idx += nt) {
    const int i = idx / kSolveCols, cc = idx % kSolveCols, rr = blockIdx.x * kSolveCols + cc;
    double b = 0.0;
    if (rr < rhs) b = J.col ? (double)J.X[(int64_t)rr * J.ld + i] : (double)J.X[(int64_t)i * J.ld + rr];
    ys[cc * ldy + i] = b;
  }
  double* y = ys + (size_t)c * ldy;
  for (int i0 = 0; i0 < m; i0 += kSolveBlk) {       // forward: y_i = (b_i - sum_{k<i} L_ik y_k) / L_ii
    const int bi = min(kSolveBlk, m - i0);
    __syncthreads();
    for (int idx = tid; idx < bi * (i0 + bi); idx += nt) {
      const int r = idx / (i0 + bi), k = idx % (i0 + bi);
      Lb[r * m + k] = L[(int64_t)(i0 + r) * m + k];
    }
    __syncthreads();
    for (int ii = 0; ii < bi; ++ii) {
      const int i = i0 + ii;
      const double* Li = Lb + ii * m;
      double s0 = 0.0, s1 = 0.0;
      int k = g;
      for (; k + kSolveSplit < i; k += 2 * kSolveSplit) {
        s0 = fma(Li[k], y[k], s0);
        s1 = fma(Li[k + kSolveSplit], y[k + kSolveSplit], s1);
      }
      if (k < i) s0 = fma(Li[k], y[k], s0);
      double s = s0 + s1;
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      s += __shfl_xor_sync(0xffffffffu, s, 4);
      if (g == 0) y[i] = (y[i] - s) / Li[i];
      __syncwarp();
    }
  }
  for (int i1 = m; i1 > 0; i1 -= kSolveBlk) {       // backward: q_i = (y_i - sum_{k>i} L_ki q_k) / L_ii
    const int i0 = max(0, i1 - kSolveBlk), bi = i1 - i0;
    __syncthreads();
    for (int idx = tid; idx < (m - i0) * bi; idx += nt) {   // global reads: 8 consecutive columns per row
      const int k = i0 + idx / bi, j = idx % bi;
      Lb[j * m + k] = L[(int64_t)k * m + i0 + j];
    }
    __syncthreads();
    for (int ii = bi - 1; ii >= 0; --ii) {
      const int i = i0 + ii;
      const double* Lc = Lb + ii * m;                 // column i of L, rows k
      double s0 = 0.0, s1 = 0.0;
      int k = i + 1 + g;
      for (; k + kSolveSplit < m; k += 2 * kSolveSplit) {
        s0 = fma(Lc[k], y[k], s0);
        s1 = fma(Lc[k + kSolveSplit], y[k + kSolveSplit], s1);
      }
      if (k < m) s0 = fma(Lc[k], y[k], s0);
      double s = s0 + s1;
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      s += __shfl_xor_sync(0xffffffffu, s, 4);
      if (g == 0) y[i] = (y[i] - s) / Lc[i];
      __syncwarp();
    }
  }
  __syncthreads();
  for (int idx = tid; idx < m * kSolveCols; idx += nt) {
    const int i = idx / kSolveCols, cc = idx % kSolveCols, rr = blockIdx.x * kSolveCols + cc;
    if (rr < rhs) J.Y[(int64_t)i * rhs + rr] = ys[cc * ldy + i];
  }
}

// Row r: a_r = x_r . q_r, b_r = 1 + a_r / (n - 1 - a_r), x_hat_r = b_r q_r (in place, FP32),
// ||x_r||^2 and ||x_hat_r||^2 (FP64).  One CTA per row; grid (max n, jobs).
__global__ void __launch_bounds__(256) simple_rows_kernel(const __grid_constant__ SimpleJobs jb) {
  const SimpleJob& J = jb.j[blockIdx.y];
  const int r = blockIdx.x;
  if (r >= J.n) return;
  __shared__ double red[32];
  float* x = J.X + (int64_t)r * J.ld;
  auto q_at = [&](int c) -> double {
    return J.col ? J.Y[(int64_t)c * J.rhs + r] : J.Y[(int64_t)r * J.rhs + c];
  };
  double a = 0.0, xx = 0.0;
  for (int c = threadIdx.x; c < J.D; c += blockDim.x) {
    const double xv = x[c];
    a = fma(xv, q_at(c), a);
    xx = fma(xv, xv, xx);
  }
  a = block_sum(a, red);
  xx = block_sum(xx, red);
  const double b = 1.0 + a / ((double)(J.n - 1) - a);
  double pp = 0.0;
  __syncthreads();   // every x read before the row is overwritten
  for (int c = threadIdx.x; c < J.D; c += blockDim.x) {
    const float xh = (float)(b * q_at(c));
    x[c] = xh;
    pp = fma((double)xh, (double)xh, pp);
  }
  pp = block_sum(pp, red);
  if (threadIdx.x == 0) {
    J.rowpart[r] = xx;
    J.rowpart[J.n + r] = pp;
    J.p[r] = (float)pp;
  }
}

// gamma = sqrt(sum ||x||^2 / sum ||x_hat||^2) (1 if 0), fixed-order sums over rows.
__global__ void __launch_bounds__(256) simple_gamma_kernel(const __grid_constant__ SimpleJobs jb) {
  const SimpleJob& J = jb.j[blockIdx.x];
  __shared__ double red[32];
  double sx = 0.0, sp = 0.0;
  for (int r = threadIdx.x; r < J.n; r += blockDim.x) { sx += J.rowpart[r]; sp += J.rowpart[J.n + r]; }
  sx = block_sum(sx, red);
  sp = block_sum(sp, red);
  if (threadIdx.x == 0) {
    J.stats[2] = sx;
    J.stats[3] = sp;
    *J.gamma = (sp > 0.0) ? (float)sqrt(sx / sp) : 1.0f;
    if (!isfinite(sx) || !isfinite(sp)) atomicOr(reinterpret_cast<unsigned*>(J.flags), kErrNonFinite);
  }
}

}  // namespace ng

using namespace ng;

static ng_status simple_alloc(void** p, size_t bytes) {
  if (cudaMalloc(p, std::max<size_t>(bytes, 16)) != cudaSuccess) {
    set_error("ngsimple: cudaMalloc failed");
    return NG_ENOMEM;
  }
  return NG_OK;
}

void ngsimple_destroy_impl(ngsimple_ctx* h) {
  if (!h) return;
  if (h->G) cudaFree(h->G);
  if (h->Y) cudaFree(h->Y);
  if (h->rowpart) cudaFree(h->rowpart);
  if (h->stats) cudaFree(h->stats);
  if (h->gamma) cudaFree(h->gamma);
  if (h->p) cudaFree(h->p);
  if (h->flags) cudaFree(h->flags);
  delete h;
}

ng_status ngsimple_create_impl(int dim, int max_rows, float alpha, cudaStream_t st, ngsimple_ctx** out) {
  NG_REQUIRE(out != nullptr, NG_EINVAL, "NULL argument");
  NG_REQUIRE(dim >= 1 && max_rows >= 2, NG_ESHAPE, "ngsimple: dim >= 1 and max_rows >= 2 (hold-out, P:815-819)");
  NG_REQUIRE(alpha > 0.f, NG_EINVAL, "ngsimple: alpha must be > 0");
  ngsimple_ctx* h = new ngsimple_ctx();
  h->dim = dim;
  h->max_rows = max_rows;
  h->alpha = alpha;
  h->st = st;
  // column space (n > D) needs D x D, row space (n <= D) needs n x n: never more than min(D, max_rows)
  const size_t m = (size_t)std::min(dim, max_rows);
  ng_status s = simple_alloc((void**)&h->G, sizeof(double) * m * m);
  if (s == NG_OK) s = simple_alloc((void**)&h->Y, sizeof(double) * (size_t)dim * max_rows);
  if (s == NG_OK) s = simple_alloc((void**)&h->rowpart, sizeof(double) * 2 * max_rows);
  if (s == NG_OK) s = simple_alloc((void**)&h->stats, sizeof(double) * 4);
  if (s == NG_OK) s = simple_alloc((void**)&h->gamma, sizeof(float));
  if (s == NG_OK) s = simple_alloc((void**)&h->p, sizeof(float) * max_rows);
  if (s == NG_OK) s = simple_alloc((void**)&h->flags, sizeof(int) * 4);
  if (s == NG_OK && cudaMemsetAsync(h->flags, 0, sizeof(int) * 4, st) != cudaSuccess) s = NG_ECUDA;
  if (s != NG_OK) { ngsimple_destroy_impl(h); return s; }
  *out = h;
  return NG_OK;
}

namespace ng {
ng_status ngsimple_precondition_group_impl(const SimpleCall* calls, int count) {
  NG_REQUIRE(calls != nullptr && count >= 0, NG_EINVAL, "NULL argument");
  for (int b = 0; b < count; b += kSimpleMaxJobs) {
    const int cnt = std::min(kSimpleMaxJobs, count - b);
    SimpleJobs jb;
    std::memset(&jb, 0, sizeof(jb));
    jb.count = cnt;
    cudaStream_t st = nullptr;
    int max_tiles = 1, max_n = 1, max_rhs = 1;
    for (int q = 0; q < cnt; ++q) {
      const SimpleCall& c = calls[b + q];
      ngsimple_ctx* h = c.h;
      NG_REQUIRE(h != nullptr && c.x != nullptr, NG_EINVAL, "NULL argument");
      NG_REQUIRE(c.n >= 2 && c.n <= h->max_rows, NG_ESHAPE, "ngsimple: n must be in [2, max_rows] (S:56)");
      NG_REQUIRE(c.ld >= h->dim, NG_ESHAPE, "ngsimple: ld < dim");
      NG_REQUIRE(q == 0 || h->st == st, NG_EINVAL, "ngsimple: grouped calls must share a stream");
      st = h->st;
      SimpleJob& J = jb.j[q];
      J.X = c.x; J.ld = c.ld; J.n = c.n; J.D = h->dim;
      J.col = c.n > h->dim ? 1 : 0;                       // strict N > D (reading R11)
      J.m = J.col ? h->dim : c.n;
      J.rhs = J.col ? c.n : h->dim;
      J.G = h->G; J.Y = h->Y; J.rowpart = h->rowpart; J.stats = h->stats;
      J.gamma = c.gamma_out ? c.gamma_out : h->gamma;
      J.p = c.p_out ? c.p_out : h->p;
      J.flags = h->flags; J.alpha = h->alpha;
      const int t = (J.m + kGramTile - 1) / kGramTile;
      max_tiles = std::max(max_tiles, t * t);
      max_n = std::max(max_n, c.n);
      max_rhs = std::max(max_rhs, J.rhs);
    }
    if (cnt == 0) continue;
    simple_gram_kernel<<<dim3(max_tiles, cnt), 256, 0, st>>>(jb);
    NG_TRY(check_launch("simple_gram_kernel"));
    int max_m = 1;
    for (int q = 0; q < cnt; ++q) max_m = std::max(max_m, jb.j[q].m);
    const size_t chol_smem = sizeof(double) * ((size_t)kCholB * (kCholB + 1) + (size_t)max_m * (kCholB + 1));
    const size_t solve_smem = sizeof(double) * ((size_t)kSolveCols * (max_m + 1) + (size_t)max_m * kSolveBlk);
    static bool attr = false;
    if (!attr) {
      NG_CUDA_TRY(cudaFuncSetAttribute(simple_chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      NG_CUDA_TRY(cudaFuncSetAttribute(simple_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr = true;
    }
    NG_REQUIRE(chol_smem <= 200u * 1024u && solve_smem <= 200u * 1024u, NG_ESHAPE,
               "ngsimple: min(n, dim) too large for the shared-memory panels (<= 740)");
    simple_chol_kernel<<<cnt, 1024, chol_smem, st>>>(jb);
    NG_TRY(check_launch("simple_chol_kernel"));
    simple_solve_kernel<<<dim3(ceil_div(max_rhs, kSolveCols), cnt), kSolveCols * kSolveSplit, solve_smem, st>>>(jb);
    NG_TRY(check_launch("simple_solve_kernel"));
    simple_rows_kernel<<<dim3(max_n, cnt), 256, 0, st>>>(jb);
    NG_TRY(check_launch("simple_rows_kernel"));
    simple_gamma_kernel<<<cnt, 256, 0, st>>>(jb);
    NG_TRY(check_launch("simple_gamma_kernel"));
  }
  return NG_OK;
}
}  // namespace ng

extern "C" {

ng_status ngsimple_create(int32_t dim, int32_t max_rows, float alpha, void* cuda_stream, ngsimple_t* out) {
  return ngsimple_create_impl(dim, max_rows, alpha, (cudaStream_t)cuda_stream, out);
}

ng_status ngsimple_destroy(ngsimple_t h) {
  NG_REQUIRE(h != nullptr, NG_EINVAL, "NULL argument");
  cudaStreamSynchronize(h->st);
  ngsimple_destroy_impl(h);
  return NG_OK;
}

ng_status ngsimple_precondition(ngsimple_t h, int32_t n, float* x, int64_t ld, float* gamma_out, float* row_sq_out) {
  NG_REQUIRE(h != nullptr && x != nullptr, NG_EINVAL, "NULL argument");
  SimpleCall c{h, n, x, ld, gamma_out, row_sq_out};
  return ngsimple_precondition_group_impl(&c, 1);
}

ng_status ngsimple_read_flags(ngsimple_t h) {
  NG_REQUIRE(h != nullptr, NG_EINVAL, "NULL argument");
  int f = 0;
  NG_CUDA_TRY(cudaStreamSynchronize(h->st));
  NG_CUDA_TRY(cudaMemcpy(&f, h->flags, sizeof(int), cudaMemcpyDeviceToHost));
  return status_from_flags((uint32_t)f, "ngsimple");
}

}  // extern "C"
