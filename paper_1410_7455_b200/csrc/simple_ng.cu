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
  double* DI;       // ceil(m / kTsB) x kTsB x kTsB: inverses of the diagonal blocks of L
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

// The two triangular solves L y = b, L^T q = y as GEMMs (round 2; the substitution kernel
// before it did one dot product per row and reached ~1% of the FP64 rate): L is cut into
// kTsB-row blocks whose diagonal blocks are inverted once (simple_diaginv_kernel); then,
// for a tile of kTsC right-hand sides per CTA,
//   forward,  block b ascending:  T = y_b - L[b, <b] y[<b],      y_b = L_bb^{-1} T
//   backward, block b descending: T = y_b - L[>b, b]^T q[>b],    q_b = L_bb^{-T} T
// every product a register-tiled FP64 GEMM (4 x 4 outputs per thread, kTsK-deep chunks
// staged in shared memory).  y and q live in Y (L2-resident); the tiles are independent.
constexpr int kTsB = 64;    // row block (diagonal blocks inverted)
constexpr int kTsC = 64;    // right-hand sides per CTA
constexpr int kTsK = 8;     // k-chunk staged in shared memory

// DI[b] = L_bb^{-1} (kTsB x kTsB row-major; zero above the diagonal and outside the block):
// thread c forms column c by forward substitution on e_c.
__global__ void __launch_bounds__(kTsB) simple_diaginv_kernel(const __grid_constant__ SimpleJobs jb) {
  const SimpleJob& J = jb.j[blockIdx.y];
  const int m = J.m, b = blockIdx.x, i0 = b * kTsB;
  if (i0 >= m) return;
  const int bs = min(kTsB, m - i0), c = threadIdx.x;
  extern __shared__ __align__(16) double dis[];   // L_bb, then the inverse (2 x kTsB x (kTsB + 1))
  double (*Ls)[kTsB + 1] = reinterpret_cast<double (*)[kTsB + 1]>(dis);
  double (*xs)[kTsB + 1] = reinterpret_cast<double (*)[kTsB + 1]>(dis + kTsB * (kTsB + 1));
  for (int idx = c; idx < kTsB * kTsB; idx += kTsB) {
    const int i = idx / kTsB, j = idx % kTsB;
    Ls[i][j] = (i < bs && j <= i) ? J.G[(int64_t)(i0 + i) * m + i0 + j] : 0.0;
  }
  __syncthreads();
  for (int i = 0; i < kTsB; ++i) {
    double x = 0.0;
    if (i < bs && i >= c) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = c; k < i; ++k) s = fma(-Ls[i][k], xs[k][c], s);
      x = s / Ls[i][i];
    }
    xs[i][c] = x;
  }
  __syncthreads();
  double* DI = J.DI + (size_t)b * kTsB * kTsB;
  for (int idx = c; idx < kTsB * kTsB; idx += kTsB) DI[idx] = xs[idx / kTsB][idx % kTsB];
}

// acc += A B over one staged chunk: A as As[kk][row] (rows 4 tr .. 4 tr + 3), B rows at
// B + kk * ldb (columns 4 tc .. 4 tc + 3), both 16-byte aligned.
__device__ __forceinline__ void ts_chunk(const double (*As)[kTsB + 2], const double* B, int ldb, int tr, int tc,
                                         double (&acc)[4][4]) {
#pragma unroll
  for (int kk = 0; kk < kTsK; ++kk) {
    const double2 a01 = *reinterpret_cast<const double2*>(&As[kk][4 * tr]);
    const double2 a23 = *reinterpret_cast<const double2*>(&As[kk][4 * tr + 2]);
    const double2 b01 = *reinterpret_cast<const double2*>(B + kk * ldb + 4 * tc);
    const double2 b23 = *reinterpret_cast<const double2*>(B + kk * ldb + 4 * tc + 2);
    const double a[4] = {a01.x, a01.y, a23.x, a23.y}, bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], bv[j], acc[i][j]);
  }
}

__global__ void __launch_bounds__(256) simple_trsm_kernel(const __grid_constant__ SimpleJobs jb) {
  const SimpleJob& J = jb.j[blockIdx.y];
  const int m = J.m, rhs = J.rhs, c0 = blockIdx.x * kTsC;
  if (c0 >= rhs) return;   // uniform per CTA
  const int tid = threadIdx.x, tr = tid >> 4, tc = tid & 15;
  constexpr int LDS = kTsC + 2;   // 16-byte aligned rows
  __shared__ __align__(16) double As[kTsK][kTsB + 2];
  __shared__ __align__(16) double Bs[kTsK][LDS];
  __shared__ __align__(16) double Ts[kTsB][LDS];
  double* Y = J.Y;
  const double* L = J.G;
  const int nb = (m + kTsB - 1) / kTsB;
  // b (this tile's right-hand sides) into Y, FP64
  for (int idx = tid; idx < m * kTsC; idx += blockDim.x) {
    int i, cc;
    if (J.col) { cc = idx / m; i = idx - cc * m; } else { i = idx / kTsC; cc = idx - i * kTsC; }
    const int c = c0 + cc;
    if (c < rhs) Y[(int64_t)i * rhs + c] = J.col ? (double)J.X[(int64_t)c * J.ld + i] : (double)J.X[(int64_t)i * J.ld + c];
  }
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {   // 0: L y = b, 1: L^T q = y
    for (int s = 0; s < nb; ++s) {
      const int b = pass == 0 ? s : nb - 1 - s;
      const int i0 = b * kTsB, bs = min(kTsB, m - i0);
      const int kb = pass == 0 ? 0 : i0 + bs, ke = pass == 0 ? i0 : m;
      double acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
      for (int k0 = kb; k0 < ke; k0 += kTsK) {
        for (int idx = tid; idx < kTsK * kTsB; idx += blockDim.x) {
          int kk, r;
          double v = 0.0;
          if (pass == 0) {
            r = idx / kTsK; kk = idx - r * kTsK;
            if (r < bs && k0 + kk < ke) v = L[(int64_t)(i0 + r) * m + k0 + kk];
          } else {
            kk = idx / kTsB; r = idx - kk * kTsB;
            if (r < bs && k0 + kk < ke) v = L[(int64_t)(k0 + kk) * m + i0 + r];
          }
          As[kk][r] = v;
        }
        for (int idx = tid; idx < kTsK * kTsC; idx += blockDim.x) {
          const int kk = idx / kTsC, cc = idx - kk * kTsC, c = c0 + cc;
          Bs[kk][cc] = (k0 + kk < ke && c < rhs) ? __ldcg(Y + (int64_t)(k0 + kk) * rhs + c) : 0.0;
        }
        __syncthreads();
        ts_chunk(As, &Bs[0][0], LDS, tr, tc, acc);
        __syncthreads();
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = 4 * tr + i, cc = 4 * tc + j, c = c0 + cc;
          Ts[r][cc] = (r < bs && c < rhs) ? __ldcg(Y + (int64_t)(i0 + r) * rhs + c) - acc[i][j] : 0.0;
          acc[i][j] = 0.0;
        }
      __syncthreads();
      const double* DI = J.DI + (size_t)b * kTsB * kTsB;
      for (int k0 = 0; k0 < kTsB; k0 += kTsK) {
        for (int idx = tid; idx < kTsK * kTsB; idx += blockDim.x) {
          int kk, r;
          if (pass == 0) { r = idx / kTsK; kk = idx - r * kTsK; As[kk][r] = DI[r * kTsB + k0 + kk]; }
          else { kk = idx / kTsB; r = idx - kk * kTsB; As[kk][r] = DI[(k0 + kk) * kTsB + r]; }
        }
        __syncthreads();
        ts_chunk(As, &Ts[k0][0], LDS, tr, tc, acc);
        __syncthreads();
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = 4 * tr + i, c = c0 + 4 * tc + j;
          if (r < bs && c < rhs) Y[(int64_t)(i0 + r) * rhs + c] = acc[i][j];
        }
      __syncthreads();
    }
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
  if (h->DI) cudaFree(h->DI);
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
  if (s == NG_OK) s = simple_alloc((void**)&h->DI, sizeof(double) * (size_t)((m + kTsB - 1) / kTsB) * kTsB * kTsB);
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
      J.G = h->G; J.Y = h->Y; J.DI = h->DI; J.rowpart = h->rowpart; J.stats = h->stats;
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
    static bool attr = false;
    if (!attr) {
      NG_CUDA_TRY(cudaFuncSetAttribute(simple_chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      NG_CUDA_TRY(cudaFuncSetAttribute(simple_diaginv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(sizeof(double) * 2 * kTsB * (kTsB + 1))));
      attr = true;
    }
    NG_REQUIRE(chol_smem <= 200u * 1024u, NG_ESHAPE,
               "ngsimple: min(n, dim) too large for the shared-memory panels (<= 740)");
    simple_chol_kernel<<<cnt, 1024, chol_smem, st>>>(jb);
    NG_TRY(check_launch("simple_chol_kernel"));
    simple_diaginv_kernel<<<dim3(ceil_div(max_m, kTsB), cnt), kTsB, sizeof(double) * 2 * kTsB * (kTsB + 1), st>>>(jb);
    NG_TRY(check_launch("simple_diaginv_kernel"));
    simple_trsm_kernel<<<dim3(ceil_div(max_rhs, kTsC), cnt), 256, 0, st>>>(jb);
    NG_TRY(check_launch("simple_trsm_kernel"));
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
