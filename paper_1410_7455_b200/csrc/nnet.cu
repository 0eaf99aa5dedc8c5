// nnet.cu -- p-norm/softmax DNN training step with online NG-SGD (arXiv 1410.7455) and
// the every-K parameter average (section 3.1), on sm_100a.
//
//   forward:   Y_1 = [frames, 1];  Z_l = Y_l W_l^T;  Y_{l+1} = [pnorm(Z_l), 1]
//              (P:281-283), optionally renormalised to unit-RMS rows
//              (R32);  output log-softmax, objective, X_L = onehot - p
//
//   backward:  g = X_l W_l[:, :D_in];  (renorm: g <- s (g - y y^T g / D));
//              X_{l-1} = g[k/G] z_k / a_{k/G}
//   update:    X_hat, gamma_x = NG_out(X_l); Y_hat, gamma_y = NG_in(Y_l);
//              alpha_t = min(1, N max_change / (lr gamma_x gamma_y sum_i sqrt(p_i^x p_i^y)))
//              (C.3);  W_l += alpha_t lr gamma_x gamma_y X_hat^T Y_hat
//              (eqn:add:w)
//   average:   W <- tree_sum_r(W^r) / n over NCCL
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "gemm_simt.cuh"
#include "gemm_tc.cuh"
#include "ngsgd_impl.cuh"
#include "simple_ng_impl.cuh"

using namespace ng;

constexpr int kMaxRowWidth = 50000;   // widest activation row staged in shared memory
constexpr int kBwdSplits = 8;
constexpr int kMaxRanks = 64;      // nnet_average: jobs per communicator   // split-K of the TF32 backward-data GEMM (K = 3000..5000)

struct nnet_ctx {
  nnet_config cfg{};
  cudaStream_t st = nullptr;
  int L = 0;                                 // number of weight matrices I
  std::vector<int> rows, cols, ldp;          // W_l is rows x cols (cols = D_in + 1)
  std::vector<size_t> off;                   // offset of W_l in the arena (floats)
  float* arena = nullptr;                    // all W_l, FP32 master copy
  size_t arena_count = 0;
  std::vector<float*> Y, Z, X;               // per layer activations / derivatives
  std::vector<ngsgd_ctx*> ng_in, ng_out;
  std::vector<ngsimple_ctx*> sn_in, sn_out;   // precond = 2: simple NG-SGD (Appendix A)
  float* gam = nullptr;       // 2L: gamma_in, gamma_out per layer
  float* pbuf = nullptr;      // 2L x max_minibatch: p_in, p_out per layer
  float* scale = nullptr;     // L: alpha_t lr gamma_x gamma_y
  float* stats = nullptr;     // L x 4: alpha_t, gamma_in, gamma_out, bound
  double* objrows = nullptr;  // max_minibatch
  float* rscale = nullptr;    // (L-1) x max_minibatch: renormalisation scale s per hidden layer row
  int32_t* lab = nullptr;     // max_minibatch: labels of a gathered minibatch
  double* obj = nullptr;      // 1
  int* eflags = nullptr;      // sticky error bits
  int n_last = 0;
  bool have_fb = false;
  // tensor-core (TF32) path: split-K partials of the backward-data GEMM
  std::vector<int> ldr;                      // leading dimension of Z_l / X_l (rows padded to 8)
  float* gpart = nullptr;
  size_t gpart_count = 0;
  // NCCL
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  float* recvbuf = nullptr;     // nranks x shard: shard `rank` of every rank
  float* gatherbuf = nullptr;   // nranks x shard: averaged shards (all-gather target)
  double* objbuf = nullptr;     // nranks: all-gathered objectives (nnet_select_best)
  float* localsum = nullptr;    // nnet_average_local: the averaged arena
  float* gradbuf = nullptr;     // arena-sized: X_l^T Y_l of every layer (model combination)
  double* cgpart = nullptr;     // L x P: combination gradient
  size_t shard = 0;
};

// ------------------------------------------------------------------------------------
// kernels
// ------------------------------------------------------------------------------------

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// C.6: W ~ N(0, 1/fan-in) (fan-in includes the bias column, reading R20),
// counter-based (splitmix64 + Box-Muller) so the init is reproducible from the seed.
__global__ void init_weights_kernel(float* W, int rows, int cols, int ld, uint64_t seed, int layer, float stddev) {
  const int64_t total = (int64_t)rows * ld;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / ld), c = (int)(i % ld);
    float v = 0.f;
    if (c < cols && stddev > 0.f) {
      const uint64_t key = seed * 0x100000001B3ull + ((uint64_t)layer << 48) + (uint64_t)r * cols + c;
      const uint64_t a = splitmix64(2 * key), b = splitmix64(2 * key + 1);
      const double u1 = ((a >> 11) + 1.0) * (1.0 / 9007199254740992.0);
      const double u2 = (b >> 11) * (1.0 / 9007199254740992.0);
      v = (float)(stddev * sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
    }
    W[i] = v;
  }
}

// Y_1 = [frames, 1], zero padding columns.  Frames are FP32, or 1-byte codes
// decoded as x = float(lo_c + step_c q) (C.2, reading R36); row r of the
// minibatch is row rows[r] of the frame array when rows != NULL (a block of the N x M
// randomisation), whose label is copied to lab_out[r].
__global__ void input_kernel(int n, int din, const void* __restrict__ f, int fmt, int64_t ldf,
                             const double* __restrict__ lo, const double* __restrict__ step,
                             const int32_t* __restrict__ rows, const int32_t* __restrict__ lab_in,
                             int32_t* __restrict__ lab_out, float* __restrict__ Y, int ldy, int* eflags) {
  pdl_trigger();
  pdl_wait();   // launched with launch_pdl: inputs come from the previous kernel
  const int64_t total = (int64_t)n * ldy;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / ldy), c = (int)(i % ldy);
    const int64_t src = rows ? (int64_t)rows[r] : (int64_t)r;
    float v = 0.f;
    if (c < din) {
      if (fmt == 1) {
        const uint8_t q = reinterpret_cast<const uint8_t*>(f)[src * ldf + c];
        v = (float)(lo[c] + step[c] * (double)q);
      } else {
        v = reinterpret_cast<const float*>(f)[src * ldf + c];
      }
      if (!isfinite(v)) atomicOr(reinterpret_cast<unsigned*>(eflags), kErrNonFinite);
    } else if (c == din) {
      v = 1.f;
      if (lab_out) lab_out[r] = lab_in[src];
    }
    Y[i] = v;
  }
}

// 1-byte compression (R36), column c: lo = min_r x[r, c], step = (max - min) / 255
// (FP64 from the FP32 extremes).  One CTA per column, fixed-order reductions.
__global__ void __launch_bounds__(256)
compress_range_kernel(int n, int D, const float* __restrict__ x, int64_t ldx, double* __restrict__ lo,
                      double* __restrict__ step) {
  __shared__ float sc[32];
  const int c = blockIdx.x;
  float mn = INFINITY, mx = -INFINITY;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    const float v = x[(int64_t)r * ldx + c];
    mn = fminf(mn, v);
    mx = fmaxf(mx, v);
  }
  mx = block_max(mx, sc);
  __syncthreads();
  mn = -block_max(-mn, sc);
  if (threadIdx.x == 0) {
    lo[c] = (double)mn;
    step[c] = ((double)mx - (double)mn) / 255.0;
  }
}

// q = clamp(rint((x - lo) / step), 0, 255) in FP64 (0 where step = 0)  (R36)
__global__ void compress_codes_kernel(int n, int D, const float* __restrict__ x, int64_t ldx,
                                      const double* __restrict__ lo, const double* __restrict__ step,
                                      uint8_t* __restrict__ q, int64_t ldq) {
  const int64_t total = (int64_t)n * D;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / D), c = (int)(i % D);
    const double s = step[c];
    const double t = s > 0.0 ? ((double)x[(int64_t)r * ldx + c] - lo[c]) / s : 0.0;
    q[(int64_t)r * ldq + c] = (uint8_t)fmin(255.0, fmax(0.0, rint(t)));
  }
}

// One row of Z staged in shared memory with 16-byte loads (rows are 16B aligned: ld % 8 == 0).
__device__ __forceinline__ void stage_row(float* __restrict__ dst, const float* __restrict__ src, int cnt) {
  const int c4 = cnt >> 2;
  for (int i = threadIdx.x; i < c4; i += blockDim.x)
    reinterpret_cast<float4*>(dst)[i] = __ldg(reinterpret_cast<const float4*>(src) + i);
  for (int i = (c4 << 2) + threadIdx.x; i < cnt; i += blockDim.x) dst[i] = __ldg(src + i);
}

// p-norm, p = 2: a_j = sqrt(sum_{k in group j} z_k^2); Y_next = [a, 1].
// One CTA per row; the row of Z is read once, coalesced, into shared memory.
__global__ void __launch_bounds__(256)
pnorm_kernel(int n, int dout, int ldz, int G, const float* __restrict__ Z, float* __restrict__ Yn, int ldy) {
  extern __shared__ __align__(16) unsigned char nn_smem[];
  float* zs = reinterpret_cast<float*>(nn_smem);
  const int r = blockIdx.x, dp = dout / G;
  stage_row(zs, Z + (int64_t)r * ldz, dout);
  __syncthreads();
  float* y = Yn + (int64_t)r * ldy;
  for (int c = threadIdx.x; c < ldy; c += blockDim.x) {
    float v = 0.f;
    if (c < dp) {
      float s = 0.f;
      for (int k = 0; k < G; ++k) s = fmaf(zs[c * G + k], zs[c * G + k], s);
      v = sqrtf(s);
    } else if (c == dp) {
      v = 1.f;
    }
    y[c] = v;
  }
}

// Renormalisation layer after a p-norm layer (reading R32): row i of
// Y[:, :D] is scaled in place by s_i = sqrt(D / ||a_i||^2) (0 for an all-zero row) and s_i
// is kept for the backward pass.  One warp per row, 16-byte accesses when aligned, FP64
// sum of squares.
__global__ void __launch_bounds__(256)
renorm_kernel(int n, int D, float* __restrict__ Y, int ldy, float* __restrict__ rs) {
  pdl_trigger();
  pdl_wait();   // launched with launch_pdl: Y comes from the previous kernel
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= n) return;
  float* y = Y + (int64_t)r * ldy;
  const bool vec = ((ldy & 3) == 0) && ((reinterpret_cast<uintptr_t>(Y) & 15) == 0);
  const int d4 = vec ? (D >> 2) : 0;
  double ss = 0.0;
  for (int i = lane; i < d4; i += 32) {
    const float4 v = reinterpret_cast<const float4*>(y)[i];
    ss += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
  }
  for (int j = 4 * d4 + lane; j < D; j += 32) ss += (double)y[j] * y[j];
  ss = warp_sum(ss);
  const float s = ss > 0.0 ? (float)sqrt((double)D / ss) : 0.f;
  for (int i = lane; i < d4; i += 32) {
    float4 v = reinterpret_cast<const float4*>(y)[i];
    v.x *= s; v.y *= s; v.z *= s; v.w *= s;
    reinterpret_cast<float4*>(y)[i] = v;
  }
  for (int j = 4 * d4 + lane; j < D; j += 32) y[j] *= s;
  if (lane == 0) rs[r] = s;
}

// log p(y|x) = z_y - logsumexp(z); X_L = onehot(y) - softmax(z); one CTA per row,
// the row staged once in shared memory.
__global__ void __launch_bounds__(256)
softmax_kernel(int n, int C, int ld, const float* __restrict__ Z, const int32_t* __restrict__ labels,
               float* __restrict__ X, double* __restrict__ objrows, int* eflags) {
  pdl_trigger();
  pdl_wait();   // launched with launch_pdl: inputs come from the previous kernel
  extern __shared__ __align__(16) unsigned char nn_smem[];
  __shared__ float sc[32];
  float* zs = reinterpret_cast<float*>(nn_smem);
  const int r = blockIdx.x;
  stage_row(zs, Z + (int64_t)r * ld, C);
  __syncthreads();
  float m = -INFINITY;
  for (int j = threadIdx.x; j < C; j += blockDim.x) m = fmaxf(m, zs[j]);
  m = block_max(m, sc);
  float s = 0.f;
  for (int j = threadIdx.x; j < C; j += blockDim.x) s += expf(zs[j] - m);
  s = block_sum(s, sc);
  const float lse = m + logf(s);
  int y = labels[r];
  if (y < 0 || y >= C) {
    if (threadIdx.x == 0) atomicOr(reinterpret_cast<unsigned*>(eflags), kErrLabel);
    y = -1;
  }
  float* x = X + (int64_t)r * ld;
  const int c4 = C >> 2;
  for (int i = threadIdx.x; i < c4; i += blockDim.x) {
    const float4 z = reinterpret_cast<const float4*>(zs)[i];
    const int j = i << 2;
    reinterpret_cast<float4*>(x)[i] =
        make_float4((j == y ? 1.f : 0.f) - expf(z.x - lse), (j + 1 == y ? 1.f : 0.f) - expf(z.y - lse),
                    (j + 2 == y ? 1.f : 0.f) - expf(z.z - lse), (j + 3 == y ? 1.f : 0.f) - expf(z.w - lse));
  }
  for (int j = (c4 << 2) + threadIdx.x; j < C; j += blockDim.x) x[j] = (j == y ? 1.f : 0.f) - expf(zs[j] - lse);
  if (threadIdx.x == 0) {
    objrows[r] = (y >= 0) ? (double)(zs[y] - lse) : 0.0;
    if (!isfinite(lse)) atomicOr(reinterpret_cast<unsigned*>(eflags), kErrNonFinite);
  }
}

__global__ void objsum_kernel(int n, const double* __restrict__ rows, double* __restrict__ out) {
  pdl_trigger();
  pdl_wait();   // launched with launch_pdl: inputs come from the previous kernel
  __shared__ double sc[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += rows[i];
  s = block_sum(s, sc);
  if (threadIdx.x == 0) *out = s;
}

// p-norm backward fused into the backward-data GEMM epilogue: for output (i, j) of
// g = X_l W_l[:, :D_in]:  X_{l-1}[i, jG+q] = g z_{jG+q} / a_j  (0 if a_j = 0).
struct EpiPnormBack {
  float* Xp; const float* Zp; const float* Yl; int ldx; int ldy; int G;
  __device__ void operator()(int i, int j, float g, int) const {
    const float a = Yl[(int64_t)i * ldy + j];
    const float* z = Zp + (int64_t)i * ldx + (int64_t)j * G;
    float* xo = Xp + (int64_t)i * ldx + (int64_t)j * G;
    if (a > 0.f) {
      const float ga = g / a;
      for (int q = 0; q < G; ++q) xo[q] = ga * z[q];
    } else {
      for (int q = 0; q < G; ++q) xo[q] = 0.f;
    }
  }
};

// TF32 path: g = sum_z partial_z (fixed order), then the p-norm backward of EpiPnormBack.
// One CTA per row: g / a_j for the row's din groups into shared memory, then the row of
// X_{l-1} = (g/a) z with 16-byte coalesced loads of Z and stores of X.
__global__ void __launch_bounds__(256)
pnorm_back_kernel(const float* __restrict__ part, int splits, int n, int din, const float* __restrict__ Zp,
                  const float* __restrict__ Yl, float* __restrict__ Xp, int ldx, int ldy, int G,
                  const float* __restrict__ rs) {
  pdl_trigger();
  pdl_wait();   // launched with launch_pdl: inputs come from the previous kernel
  extern __shared__ __align__(16) unsigned char nn_smem[];
  float* ga = reinterpret_cast<float*>(nn_smem);
  const int r = blockIdx.x;
  const int64_t total = (int64_t)n * din;
  // the row of Z (last phase) does not depend on g: its loads are issued first so their
  // latency overlaps the split-K sum and the renormalisation backward
  constexpr int kZP = 4;
  const int dout = din * G;
  const int c4 = dout >> 2;
  const float* zr = Zp + (int64_t)r * ldx;
  const bool zpre = (dout & 3) == 0 && (ldx & 3) == 0 && c4 <= kZP * (int)blockDim.x;
  float4 zq[kZP];
#pragma unroll
  for (int q = 0; q < kZP; ++q) {
    const int i = threadIdx.x + q * blockDim.x;
    zq[q] = (zpre && i < c4) ? __ldg(reinterpret_cast<const float4*>(zr) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (rs != nullptr) {
    // renormalisation layer between: y = s a (R32).  g_a = s (g - y (y^T g) / D), then the
    // p-norm derivative divides by a = y / s (0 where a = 0).  g (the fixed-order sum of
    // the split-K partials) is staged in shared memory with 16-byte loads, y^T g reduced in
    // FP64.
    __shared__ double sc[32];
    double dot = 0.0;
    const float* yrow = Yl + (int64_t)r * ldy;
    if ((din & 3) == 0 && (total & 3) == 0 && (ldy & 3) == 0 && splits <= 8) {
      const int d4 = din >> 2;
      for (int j4 = threadIdx.x; j4 < d4; j4 += blockDim.x) {
        const int64_t i4 = ((int64_t)r * din >> 2) + j4;
        float4 pv[8];
#pragma unroll
        for (int z = 0; z < 8; ++z)
          if (z < splits) pv[z] = __ldg(reinterpret_cast<const float4*>(part + (int64_t)z * total) + i4);
        float4 g = pv[0];
#pragma unroll
        for (int z = 1; z < 8; ++z)
          if (z < splits) { g.x += pv[z].x; g.y += pv[z].y; g.z += pv[z].z; g.w += pv[z].w; }
        reinterpret_cast<float4*>(ga)[j4] = g;
        const float4 y = __ldg(reinterpret_cast<const float4*>(yrow) + j4);
        dot += (double)y.x * g.x + (double)y.y * g.y + (double)y.z * g.z + (double)y.w * g.w;
      }
    } else {
      for (int j = threadIdx.x; j < din; j += blockDim.x) {
        const int64_t i = (int64_t)r * din + j;
        float g = 0.f;
        for (int z = 0; z < splits; ++z) g += part[(int64_t)z * total + i];
        ga[j] = g;
        dot += (double)yrow[j] * g;
      }
    }
    dot = block_sum(dot, sc);   // (contains the barrier that publishes ga)
    const float s = rs[r];
    const float yg = (float)(dot / (double)din);
    for (int j = threadIdx.x; j < din; j += blockDim.x) {
      const float y = yrow[j];
      const float a = s > 0.f ? y / s : 0.f;
      ga[j] = a > 0.f ? (s * (ga[j] - y * yg)) / a : 0.f;
    }
  } else if ((din & 3) == 0 && (total & 3) == 0 && splits <= 8) {
    // 16-byte loads of the split-K partials, all splits issued before the fixed-order sum
    const int d4 = din >> 2;
    for (int j4 = threadIdx.x; j4 < d4; j4 += blockDim.x) {
      const int64_t i4 = ((int64_t)r * din >> 2) + j4;
      float4 pv[8];
#pragma unroll
      for (int z = 0; z < 8; ++z)
        if (z < splits) pv[z] = __ldg(reinterpret_cast<const float4*>(part + (int64_t)z * total) + i4);
      float4 g = pv[0];
#pragma unroll
      for (int z = 1; z < 8; ++z)
        if (z < splits) { g.x += pv[z].x; g.y += pv[z].y; g.z += pv[z].z; g.w += pv[z].w; }
      const float* ar = Yl + (int64_t)r * ldy + 4 * j4;
      const float a0 = ar[0], a1 = ar[1], a2 = ar[2], a3 = ar[3];
      ga[4 * j4 + 0] = a0 > 0.f ? g.x / a0 : 0.f;
      ga[4 * j4 + 1] = a1 > 0.f ? g.y / a1 : 0.f;
      ga[4 * j4 + 2] = a2 > 0.f ? g.z / a2 : 0.f;
      ga[4 * j4 + 3] = a3 > 0.f ? g.w / a3 : 0.f;
    }
  } else {
    for (int j = threadIdx.x; j < din; j += blockDim.x) {
      const int64_t i = (int64_t)r * din + j;
      float g = 0.f;
      for (int z = 0; z < splits; ++z) g += part[(int64_t)z * total + i];
      const float a = Yl[(int64_t)r * ldy + j];
      ga[j] = a > 0.f ? g / a : 0.f;
    }
  }
  __syncthreads();
  float* xr = Xp + (int64_t)r * ldx;
  if (zpre) {
#pragma unroll
    for (int q = 0; q < kZP; ++q) {
      const int i = threadIdx.x + q * blockDim.x;
      if (i < c4) {
        const float4 z = zq[q];
        const int k = i << 2;
        reinterpret_cast<float4*>(xr)[i] =
            make_float4(ga[k / G] * z.x, ga[(k + 1) / G] * z.y, ga[(k + 2) / G] * z.z, ga[(k + 3) / G] * z.w);
      }
    }
    return;
  }
  for (int i = threadIdx.x; i < c4; i += blockDim.x) {
    const float4 z = __ldg(reinterpret_cast<const float4*>(zr) + i);
    const int k = i << 2;
    reinterpret_cast<float4*>(xr)[i] =
        make_float4(ga[k / G] * z.x, ga[(k + 1) / G] * z.y, ga[(k + 2) / G] * z.z, ga[(k + 3) / G] * z.w);
  }
  for (int k = (c4 << 2) + threadIdx.x; k < dout; k += blockDim.x) xr[k] = ga[k / G] * zr[k];
}

// plain SGD (precond = 0): p_i = ||row_i||^2, gamma = 1
__global__ void rowsq_kernel(int n, int D, const float* __restrict__ X, int64_t ld, float* __restrict__ p,
                             float* __restrict__ gamma) {
  __shared__ float sc[32];
  const int r = blockIdx.x;
  float s = 0.f;
  for (int j = threadIdx.x; j < D; j += blockDim.x) { const float x = X[(int64_t)r * ld + j]; s = fmaf(x, x, s); }
  s = block_sum(s, sc);
  if (threadIdx.x == 0) { p[r] = s; if (r == 0) *gamma = 1.f; }
}

// C.3: bound = lr gamma_x gamma_y sum_i sqrt(p^x_i p^y_i) on the
// preconditioned rows; alpha_t = min(1, N max_change_per_sample / bound), 1 if bound = 0.
// One CTA per layer.
__global__ void __launch_bounds__(256)
maxchange_kernel(int n, int maxmb, float lr, float mc, const float* __restrict__ gam, const float* __restrict__ pbuf,
                 float* __restrict__ scale, float* __restrict__ stats) {
  pdl_trigger();
  pdl_wait();   // launched with launch_pdl: inputs come from the previous kernel
  __shared__ double sc[32];
  const int l = blockIdx.x;
  const float gy = gam[2 * l], gx = gam[2 * l + 1];
  const float* py = pbuf + (int64_t)(2 * l) * maxmb;
  const float* px = pbuf + (int64_t)(2 * l + 1) * maxmb;
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += sqrt((double)px[i] * (double)py[i]);
  s = block_sum(s, sc);
  if (threadIdx.x == 0) {
    const double bound = (double)lr * gx * gy * s;
    const double limit = (double)n * mc;
    const double alpha = (bound > 0.0) ? fmin(1.0, limit / bound) : 1.0;
    scale[l] = (float)(alpha * lr * gx * gy);
    stats[4 * l + 0] = (float)alpha;
    stats[4 * l + 1] = gy;
    stats[4 * l + 2] = gx;
    stats[4 * l + 3] = (float)bound;
  }
}

// Deterministic average of one shard (R18): out[i] = tree_sum_r(recv[r*stride + i])
// * inv over r = 0..nr-1 in the oracle's fixed pairwise order (level by level, an unpaired
// last element carried up; oracle/training.py tree_sum).  That order equals complete
// binary trees over the blocks given by the binary digits of nr (largest block first),
// folded right to left: e.g. nr = 7 = 4+2+1 -> (((0+1)+(2+3)) + ((4+5) + 6)).  Each block
// is a compile-time recursion, so every partial sum stays in registers (nr <= 127).
template <int K>
__device__ __forceinline__ float tree_block(const float* __restrict__ p, size_t stride) {
  if constexpr (K == 0) {
    return __ldg(p);
  } else {
    const float a = tree_block<K - 1>(p, stride);
    const float b = tree_block<K - 1>(p + ((size_t)1 << (K - 1)) * stride, stride);
    return a + b;
  }
}

__device__ __forceinline__ float tree_block_dyn(int k, const float* __restrict__ p, size_t stride) {
  switch (k) {
    case 0: return tree_block<0>(p, stride);
    case 1: return tree_block<1>(p, stride);
    case 2: return tree_block<2>(p, stride);
    case 3: return tree_block<3>(p, stride);
    case 4: return tree_block<4>(p, stride);
    case 5: return tree_block<5>(p, stride);
    default: return tree_block<6>(p, stride);
  }
}

__global__ void __launch_bounds__(256)
tree_avg_kernel(int nr, size_t count, size_t stride, const float* __restrict__ recv, float* __restrict__ out,
                float inv) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    bool have = false;
    for (int k = 0; k < 7; ++k) {            // blocks from the right end (lowest binary digit)
      if (!((nr >> k) & 1)) continue;
      const size_t start = (size_t)(nr & ~((2 << k) - 1));
      const float b = tree_block_dyn(k, recv + start * stride + i, stride);
      acc = have ? b + acc : b;
      have = true;
    }
    out[i] = acc * inv;
  }
}

// Generalised model combination (C.4): W_l = sum_p w[l][p] W_l^(p) over the
// arena range of layer l (blockIdx.y), and grad[l][p] = <G_l, W_l^(p)> with G_l = X_l^T Y_l
// (one CTA per (l, p), fixed-order reduction).
constexpr int kCombMax = 32;
struct CombineArgs {
  const float* model[kCombMax];
  float w[16 * kCombMax];          // L x P
  int64_t off[17];                 // layer ranges in the arena
  int P;
};
__global__ void __launch_bounds__(256) combine_kernel(const __grid_constant__ CombineArgs a, float* __restrict__ out) {
  const int l = blockIdx.y;
  for (int64_t i = a.off[l] + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.off[l + 1];
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int p = 0; p < a.P; ++p) acc = fmaf(a.w[l * kCombMax + p], a.model[p][i], acc);
    out[i] = acc;
  }
}
__global__ void __launch_bounds__(256) combine_grad_kernel(const __grid_constant__ CombineArgs a,
                                                           const float* __restrict__ G, double* __restrict__ grad) {
  __shared__ double sc[32];
  const int l = blockIdx.y, p = blockIdx.x;
  double acc = 0.0;
  for (int64_t i = a.off[l] + threadIdx.x; i < a.off[l + 1]; i += blockDim.x)
    acc = fma((double)G[i], (double)a.model[p][i], acc);
  acc = block_sum(acc, sc);
  if (threadIdx.x == 0) grad[l * kCombMax + p] = acc;
}

static ng_status launch_tree_avg(cudaStream_t st, int nr, size_t count, size_t stride, const float* recv, float* out) {
  if (count == 0) return NG_OK;
  const int blocks = (int)std::min<size_t>(4 * 148, (count + 255) / 256);
  tree_avg_kernel<<<blocks, 256, 0, st>>>(nr, count, stride, recv, out, 1.0f / (float)nr);
  return check_launch("tree_avg_kernel");
}

__global__ void scale_kernel(float* x, size_t n, float s) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) x[i] *= s;
}

// ------------------------------------------------------------------------------------
// host
// ------------------------------------------------------------------------------------

static void nnet_free(nnet_ctx* h) {
  if (!h) return;
  for (auto* p : h->ng_in) ngsgd_destroy_impl(p);
  for (auto* p : h->ng_out) ngsgd_destroy_impl(p);
  for (auto* p : h->sn_in) ngsimple_destroy_impl(p);
  for (auto* p : h->sn_out) ngsimple_destroy_impl(p);
  for (auto* p : h->Y) if (p) cudaFree(p);
  for (auto* p : h->Z) if (p) cudaFree(p);
  for (auto* p : h->X) if (p) cudaFree(p);
  if (h->arena) cudaFree(h->arena);
  if (h->gam) cudaFree(h->gam);
  if (h->pbuf) cudaFree(h->pbuf);
  if (h->scale) cudaFree(h->scale);
  if (h->stats) cudaFree(h->stats);
  if (h->objrows) cudaFree(h->objrows);
  if (h->rscale) cudaFree(h->rscale);
  if (h->lab) cudaFree(h->lab);
  if (h->obj) cudaFree(h->obj);
  if (h->eflags) cudaFree(h->eflags);
  if (h->recvbuf) cudaFree(h->recvbuf);
  if (h->gatherbuf) cudaFree(h->gatherbuf);
  if (h->objbuf) cudaFree(h->objbuf);
  if (h->localsum) cudaFree(h->localsum);
  if (h->gradbuf) cudaFree(h->gradbuf);
  if (h->cgpart) cudaFree(h->cgpart);
  if (h->comm) ncclCommDestroy(h->comm);
  if (h->gpart) cudaFree(h->gpart);
  delete h;
}

template <typename T>
static ng_status nalloc(T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) { set_error(std::string("cudaMalloc: ") + cudaGetErrorString(e)); return NG_ENOMEM; }
  return NG_OK;
}

static ng_status read_eflags(nnet_ctx* h, const char* where) {
  int f = 0;
  NG_CUDA_TRY(cudaMemcpy(&f, h->eflags, sizeof(int), cudaMemcpyDeviceToHost));
  return status_from_flags((uint32_t)f, where);
}

extern "C" {

ng_status nnet_create(const nnet_config* cfg, void* cuda_stream, nnet_t* out) {
  NG_REQUIRE(cfg != nullptr && out != nullptr, NG_EINVAL, "NULL argument");
  NG_REQUIRE(cfg->input_dim >= 1 && cfg->num_hidden >= 0 && cfg->num_classes >= 2 && cfg->max_minibatch >= 1,
             NG_ESHAPE, "bad network dimensions");
  NG_REQUIRE(cfg->num_hidden == 0 || (cfg->pnorm_group >= 1 && cfg->hidden_dim >= cfg->pnorm_group &&
                                      cfg->hidden_dim % cfg->pnorm_group == 0),
             NG_ESHAPE, "hidden_dim must be a multiple of pnorm_group");
  NG_REQUIRE(cfg->precision == NG_FP32 || cfg->precision == NG_TF32 || cfg->precision == NG_FP32_SIMT, NG_EINVAL,
             "precision must be NG_FP32, NG_TF32 or NG_FP32_SIMT (NG_BF16 is reserved)");
  NG_REQUIRE(cfg->num_hidden + 1 <= 16, NG_EINVAL, "at most 16 weight matrices");
  NG_REQUIRE(cfg->precond >= 0 && cfg->precond <= 2, NG_EINVAL, "precond must be 0 (none), 1 (online) or 2 (simple)");
  NG_REQUIRE(cfg->precond != 2 || cfg->max_minibatch >= 2, NG_ESHAPE, "simple NG needs max_minibatch >= 2");
  NG_REQUIRE(cfg->hidden_dim <= kMaxRowWidth && cfg->num_classes <= kMaxRowWidth, NG_ESHAPE,
             "hidden_dim and num_classes must be <= 50000 (one row staged in shared memory)");
  {
    static bool attr = false;
    if (!attr) {
      const int b = (int)(sizeof(float) * kMaxRowWidth);
      NG_CUDA_TRY(cudaFuncSetAttribute(pnorm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
      NG_CUDA_TRY(cudaFuncSetAttribute(softmax_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
      NG_CUDA_TRY(cudaFuncSetAttribute(pnorm_back_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
      attr = true;
    }
  }
  nnet_ctx* h = new nnet_ctx();
  h->cfg = *cfg;
  h->st = (cudaStream_t)cuda_stream;
  h->L = cfg->num_hidden + 1;
  int din = cfg->input_dim;
  size_t off = 0;
  for (int l = 0; l < h->L; ++l) {
    const int r = (l == h->L - 1) ? cfg->num_classes : cfg->hidden_dim;
    h->rows.push_back(r);
    h->cols.push_back(din + 1);
    h->ldp.push_back((int)round_up(din + 1, 8));
    h->ldr.push_back((int)round_up(r, 8));
    h->off.push_back(off);
    off += (size_t)r * h->ldp.back();
    off = (size_t)round_up((int64_t)off, 64);
    din = (l == h->L - 1) ? 0 : cfg->hidden_dim / cfg->pnorm_group;
  }
  h->arena_count = (size_t)round_up((int64_t)off, 8 * 64);
  const int N = cfg->max_minibatch;
  ng_status s = nalloc(&h->arena, h->arena_count);
  for (int l = 0; l < h->L && s == NG_OK; ++l) {
    float *y = nullptr, *z = nullptr, *x = nullptr;
    s = nalloc(&y, (size_t)N * h->ldp[l]);
    if (s == NG_OK) s = nalloc(&z, (size_t)N * h->ldr[l]);
    if (s == NG_OK) s = nalloc(&x, (size_t)N * h->ldr[l]);
    h->Y.push_back(y); h->Z.push_back(z); h->X.push_back(x);
    if (s == NG_OK && cfg->precond == 2) {
      ngsimple_ctx *a = nullptr, *b = nullptr;
      s = ngsimple_create_impl(h->cols[l], N, cfg->ng_in.alpha, h->st, &a);
      if (s == NG_OK) s = ngsimple_create_impl(h->rows[l], N, cfg->ng_out.alpha, h->st, &b);
      h->sn_in.push_back(a); h->sn_out.push_back(b);
    } else if (s == NG_OK && cfg->precond) {
      ngsgd_ctx *a = nullptr, *b = nullptr;
      s = ngsgd_create_impl(h->cols[l], N, &cfg->ng_in, h->st, &a);
      if (s == NG_OK) s = ngsgd_create_impl(h->rows[l], N, &cfg->ng_out, h->st, &b);
      h->ng_in.push_back(a); h->ng_out.push_back(b);
    }
  }
  if (s == NG_OK) s = nalloc(&h->gam, 2 * h->L);
  if (s == NG_OK) s = nalloc(&h->pbuf, (size_t)2 * h->L * N);
  if (s == NG_OK) s = nalloc(&h->scale, h->L);
  if (s == NG_OK) s = nalloc(&h->stats, 4 * h->L);
  if (s == NG_OK) s = nalloc(&h->objrows, N);
  if (s == NG_OK) s = nalloc(&h->lab, N);
  if (s == NG_OK && cfg->renorm) s = nalloc(&h->rscale, (size_t)std::max(1, h->L - 1) * N);
  if (s == NG_OK) s = nalloc(&h->obj, 1);
  if (s == NG_OK) s = nalloc(&h->eflags, 1);
  if (s == NG_OK && (cfg->precision != NG_FP32_SIMT || cfg->renorm)) {
    size_t mx = 0;
    for (int l = 1; l < h->L; ++l) mx = std::max(mx, (size_t)kBwdSplits * N * (h->cols[l] - 1));
    h->gpart_count = mx;
    s = nalloc(&h->gpart, mx);
  }
  if (s == NG_OK) {
    cudaMemsetAsync(h->arena, 0, h->arena_count * sizeof(float), h->st);
    cudaMemsetAsync(h->eflags, 0, sizeof(int), h->st);
    for (int l = 0; l < h->L; ++l) {
      const bool last = (l == h->L - 1);
      const float sd = last ? 0.f : (float)(1.0 / std::sqrt((double)h->cols[l]));
      const int64_t tot = (int64_t)h->rows[l] * h->ldp[l];
      init_weights_kernel<<<std::min(2048, ceil_div(tot, 256)), 256, 0, h->st>>>(
          h->arena + h->off[l], h->rows[l], h->cols[l], h->ldp[l], cfg->seed, l, sd);
    }
    s = check_launch("init_weights_kernel");
  }
  if (s == NG_OK && cudaStreamSynchronize(h->st) != cudaSuccess) { set_error("nnet_create: sync failed"); s = NG_ECUDA; }
  if (s != NG_OK) { nnet_free(h); return s; }
  *out = h;
  return NG_OK;
}

ng_status nnet_destroy(nnet_t h) {
  if (!h) return NG_EINVAL;
  nnet_join(h);
  cudaStreamSynchronize(h->st);
  nnet_free(h);
  return NG_OK;
}

ng_status nnet_objective_async(nnet_t h, double* host_out) {
  NG_REQUIRE(h != nullptr && host_out != nullptr, NG_EINVAL, "NULL argument");
  NG_REQUIRE(h->have_fb, NG_ESTATE, "nnet_objective_async before nnet_forward_backward");
  cudaStream_t st = h->st;
  NG_CUDA_TRY(launch_pdl(objsum_kernel, dim3(1), dim3(512), 0, st, h->n_last, (const double*)h->objrows, h->obj));
  NG_TRY(check_launch("objsum_kernel"));
  NG_CUDA_TRY(cudaMemcpyAsync(host_out, h->obj, sizeof(double), cudaMemcpyDeviceToHost, st));
  return NG_OK;
}

ng_status nnet_join(nnet_t h) {
  NG_REQUIRE(h != nullptr, NG_EINVAL, "NULL argument");
  for (auto* p : h->ng_in) NG_TRY(ngsgd_join_impl(p));
  for (auto* p : h->ng_out) NG_TRY(ngsgd_join_impl(p));
  return NG_OK;
}

ng_status nnet_num_layers(nnet_t h, int32_t* out) {
  NG_REQUIRE(h && out, NG_EINVAL, "NULL argument");
  *out = h->L;
  return NG_OK;
}

ng_status nnet_layer_shape(nnet_t h, int32_t layer, int32_t* rows, int32_t* cols) {
  NG_REQUIRE(h && rows && cols, NG_EINVAL, "NULL argument");
  NG_REQUIRE(layer >= 0 && layer < h->L, NG_EINVAL, "layer out of range");
  *rows = h->rows[layer];
  *cols = h->cols[layer];
  return NG_OK;
}

ng_status nnet_forward_backward(nnet_t h, const float* frames, int64_t ld, const int32_t* labels, int32_t n,
                                double* objective_out) {
  NG_REQUIRE(h && frames && labels, NG_EINVAL, "NULL argument");
  nnet_input in;
  std::memset(&in, 0, sizeof(in));
  in.frames = frames; in.format = 0; in.ld = ld; in.labels = labels;
  return nnet_forward_backward_ex(h, &in, n, objective_out);
}

ng_status nnet_forward_backward_ex(nnet_t h, const nnet_input* in, int32_t n, double* objective_out) {
  NG_REQUIRE(h && in && in->frames && in->labels, NG_EINVAL, "NULL argument");
  NG_REQUIRE(in->format == 0 || in->format == 1, NG_EINVAL, "format must be 0 (float32) or 1 (uint8 codes)");
  NG_REQUIRE(in->format == 0 || (in->lo && in->step), NG_EINVAL, "uint8 frames need lo and step");
  NG_REQUIRE(n >= 1 && n <= h->cfg.max_minibatch, NG_ESHAPE, "n must be in [1, max_minibatch]");
  NG_REQUIRE(in->ld >= h->cfg.input_dim, NG_ESHAPE, "ld < input_dim");
  cudaStream_t st = h->st;
  const int L = h->L, G = h->cfg.pnorm_group;
  const bool tc = h->cfg.precision != NG_FP32_SIMT;   // tcgen05 (TF32, or 3xTF32 in NG_FP32)
  const bool s3 = h->cfg.precision == NG_FP32;
  const int32_t* labels = in->rows ? h->lab : in->labels;
  {
    const int64_t tot = (int64_t)n * h->ldp[0];
    NG_CUDA_TRY(launch_pdl(input_kernel, dim3(std::min(4096, ceil_div(tot, 256))), dim3(256), 0, st, n,
                           h->cfg.input_dim, in->frames, (int)in->format, in->ld, in->lo, in->step, in->rows,
                           in->labels, in->rows ? h->lab : (int32_t*)nullptr, h->Y[0], h->ldp[0], h->eflags));
    NG_TRY(check_launch("input_kernel"));
  }
  // forward
  for (int l = 0; l < L; ++l) {
    const float* W = h->arena + h->off[l];
    const double R_ = h->rows[l], C_ = h->cols[l];
    ProfScope ps(NG_PROF_FWD_GEMM, st, 2.0 * n * R_ * C_, 4.0 * (n * C_ + R_ * C_ + n * R_));
    static const int fuse_pnorm = tune_int("NG_TUNE_FWD_PNORM", 1);
    const bool fused = tc && fuse_pnorm && l < L - 1 && G == 10 && h->rows[l] % 10 == 0;
    if (fused) {
      // affine + p-norm in one tensor-core launch (80-column tiles = 8 whole groups)
      NG_TRY(tc_gemm_tf32_pnorm(st, n, h->rows[l], h->cols[l], h->Y[l], h->ldp[l], W, h->ldp[l], h->Z[l], h->ldr[l],
                                h->Y[l + 1], h->ldp[l + 1], s3));
    } else if (tc) {
      TcEpilogue e;
      e.kind = TC_EPI_STORE; e.C = h->Z[l]; e.ldc = h->ldr[l];
      static const int bn = tune_int("NG_TUNE_FWD_BN", 128);
      NG_TRY(tc_gemm_tf32(st, n, h->rows[l], h->cols[l], h->Y[l], h->ldp[l], true, W, h->ldp[l], true, e, bn, 1,
                          nullptr, s3));
    } else {
      NG_TRY((gemm_simt<float, true, true>(st, n, h->rows[l], h->cols[l], h->Y[l], h->ldp[l], W, h->ldp[l],
                                           EpiStore<float>{h->Z[l], h->ldr[l], 1.f})));
    }
    if (l < L - 1 && !fused) {
      pnorm_kernel<<<n, 256, sizeof(float) * h->rows[l], st>>>(n, h->rows[l], h->ldr[l], G, h->Z[l], h->Y[l + 1],
                                                               h->ldp[l + 1]);
      NG_TRY(check_launch("pnorm_kernel"));
    }
    if (l < L - 1 && h->cfg.renorm) {
      NG_CUDA_TRY(launch_pdl(renorm_kernel, dim3(ceil_div(n, 8)), dim3(256), 0, st, n, h->cols[l + 1] - 1,
                             h->Y[l + 1], h->ldp[l + 1], h->rscale + (size_t)l * h->cfg.max_minibatch));
      NG_TRY(check_launch("renorm_kernel"));
    }
  }
  NG_CUDA_TRY(launch_pdl(softmax_kernel, dim3(n), dim3(256), sizeof(float) * h->rows[L - 1], st, n, h->rows[L - 1],
                         h->ldr[L - 1], (const float*)h->Z[L - 1], labels, h->X[L - 1], h->objrows, h->eflags));
  NG_TRY(check_launch("softmax_kernel"));
  // backward with the pre-update weights (reading R21)
  for (int l = L - 1; l >= 1; --l) {
    const float* W = h->arena + h->off[l];
    EpiPnormBack epi{h->X[l - 1], h->Z[l - 1], h->Y[l], h->ldr[l - 1], h->ldp[l], G};
    const double R_ = h->rows[l], C_ = h->cols[l], Rp = h->rows[l - 1];
    const float* rs = h->cfg.renorm ? h->rscale + (size_t)(l - 1) * h->cfg.max_minibatch : nullptr;
    ProfScope ps(NG_PROF_BWD_GEMM, st, 2.0 * n * R_ * (C_ - 1), 4.0 * (n * R_ + R_ * C_ + 2.0 * n * Rp + n * C_));
    if (tc) {
      const int din = h->cols[l] - 1;
      TcEpilogue e;
      e.kind = TC_EPI_PARTIAL; e.C = h->gpart; e.ldc = din; e.zstride = (int64_t)n * din;
      int sp = 1;
      static const int bn = tune_int("NG_TUNE_BWD_BN", 128);   // measured +2% over 64 (tools/tune_sweep3.sh)
      static const int splits = std::min(kBwdSplits, std::max(1, tune_int("NG_TUNE_BWD_SPLITS", kBwdSplits)));
      NG_TRY(tc_gemm_tf32(st, n, din, h->rows[l], h->X[l], h->ldr[l], true, W, h->ldp[l], false, e, bn, splits,
                          &sp, s3));
      const int64_t tot = (int64_t)n * din;
      (void)tot;
      NG_CUDA_TRY(launch_pdl(pnorm_back_kernel, dim3(n), dim3(256), sizeof(float) * din, st, (const float*)h->gpart, sp,
                             n, din, (const float*)h->Z[l - 1], (const float*)h->Y[l], h->X[l - 1], h->ldr[l - 1],
                             h->ldp[l], G, rs));
      NG_TRY(check_launch("pnorm_back_kernel"));
    } else if (rs != nullptr) {
      // FP32 with renormalisation: g to a buffer, then the renorm + p-norm backward per row
      const int din = h->cols[l] - 1;
      NG_TRY((gemm_simt<float, true, false>(st, n, din, h->rows[l], h->X[l], h->ldr[l], W, h->ldp[l],
                                            EpiStore<float>{h->gpart, din, 1.f})));
      NG_CUDA_TRY(launch_pdl(pnorm_back_kernel, dim3(n), dim3(256), sizeof(float) * din, st, (const float*)h->gpart, 1,
                             n, din, (const float*)h->Z[l - 1], (const float*)h->Y[l], h->X[l - 1], h->ldr[l - 1],
                             h->ldp[l], G, rs));
      NG_TRY(check_launch("pnorm_back_kernel"));
    } else {
      NG_TRY((gemm_simt<float, true, false>(st, n, h->cols[l] - 1, h->rows[l], h->X[l], h->ldr[l], W, h->ldp[l],
                                            epi)));
    }
  }
  h->n_last = n;
  h->have_fb = true;
  if (objective_out) {
    NG_CUDA_TRY(launch_pdl(objsum_kernel, dim3(1), dim3(512), 0, st, n, (const double*)h->objrows, h->obj));
    NG_TRY(check_launch("objsum_kernel"));
    NG_CUDA_TRY(cudaMemcpyAsync(objective_out, h->obj, sizeof(double), cudaMemcpyDeviceToHost, st));
    NG_CUDA_TRY(cudaStreamSynchronize(st));
    NG_TRY(read_eflags(h, "nnet_forward_backward"));
  }
  return NG_OK;
}

ng_status nnet_update(nnet_t h, float lr, float max_change_per_sample, nnet_update_stats* stats_out) {
  NG_REQUIRE(h != nullptr, NG_EINVAL, "NULL argument");
  NG_REQUIRE(h->have_fb, NG_ESTATE, "nnet_update before nnet_forward_backward");
  cudaStream_t st = h->st;
  const int L = h->L, n = h->n_last, N = h->cfg.max_minibatch;
  int upd_in[16] = {0}, upd_out[16] = {0};
  if (h->cfg.precond == 2) {
    // simple NG-SGD (Appendix A) on both sides of every matrix: one launch per phase
    NG_REQUIRE(n >= 2, NG_ESHAPE, "simple NG needs n >= 2 (held-out estimate, S:56)");
    std::vector<SimpleCall> sc;
    for (int l = 0; l < L; ++l) {
      float* py = h->pbuf + (size_t)(2 * l) * N;
      float* px = h->pbuf + (size_t)(2 * l + 1) * N;
      sc.push_back(SimpleCall{h->sn_out[l], n, h->X[l], h->ldr[l], h->gam + 2 * l + 1, px});
      sc.push_back(SimpleCall{h->sn_in[l], n, h->Y[l], h->ldp[l], h->gam + 2 * l, py});
    }
    // algorithmic FP64 work (A.3): Gram m(m+1) K, Cholesky m^3/3, the two
    // triangular solves 2 m^2 rhs, the rows 4 n D (m = min side, rhs / K = the other side)
    double flops = 0.0;
    for (const SimpleCall& c : sc) {
      const double D = c.h->dim, m = (c.n > c.h->dim) ? D : (double)c.n, o = (c.n > c.h->dim) ? (double)c.n : D;
      flops += m * (m + 1.0) * o + m * m * m / 3.0 + 2.0 * m * m * o + 4.0 * c.n * D;
    }
    ProfScope ps(NG_PROF_NG_APPLY, st, flops, 0.0);
    NG_TRY(ngsimple_precondition_group_impl(sc.data(), (int)sc.size()));
  } else if (h->cfg.precond) {
    // all 2I preconditioning calls of the step as one group: one launch per
    // NG phase for every tensor-core-eligible state
    std::vector<NgCall> calls;
    for (int l = 0; l < L; ++l) {
      float* py = h->pbuf + (size_t)(2 * l) * N;
      float* px = h->pbuf + (size_t)(2 * l + 1) * N;
      calls.push_back(NgCall{h->ng_out[l], n, h->X[l], h->ldr[l], h->gam + 2 * l + 1, px, -1, &upd_out[l]});
      calls.push_back(NgCall{h->ng_in[l], n, h->Y[l], h->ldp[l], h->gam + 2 * l, py, -1, &upd_in[l]});
    }
    NG_TRY(ngsgd_precondition_group_impl(calls.data(), (int)calls.size()));
  }
  for (int l = 0; l < L; ++l) {
    float* py = h->pbuf + (size_t)(2 * l) * N;
    float* px = h->pbuf + (size_t)(2 * l + 1) * N;
    if (h->cfg.precond) {
    } else {
      rowsq_kernel<<<n, 256, 0, st>>>(n, h->rows[l], h->X[l], h->ldr[l], px, h->gam + 2 * l + 1);
      rowsq_kernel<<<n, 256, 0, st>>>(n, h->cols[l], h->Y[l], h->ldp[l], py, h->gam + 2 * l);
      NG_TRY(check_launch("rowsq_kernel"));
    }
  }
  NG_CUDA_TRY(launch_pdl(maxchange_kernel, dim3(L), dim3(256), 0, st, n, N, lr, max_change_per_sample,
                         (const float*)h->gam, (const float*)h->pbuf, h->scale, h->stats));
  NG_TRY(check_launch("maxchange_kernel"));
  const bool tc = h->cfg.precision != NG_FP32_SIMT;
  const bool s3 = h->cfg.precision == NG_FP32;
  static const int upd_grouped = tune_int("NG_TUNE_UPD_GROUPED", 1);
  if (tc && upd_grouped && L <= kTcGroupMax) {
    // all L weight updates W_l += s_l X_l^T Y_l (eqn:add:w) in ONE tensor-core launch
    std::vector<TcGroupDesc> d(L);
    double flops = 0, bytes = 0;
    for (int l = 0; l < L; ++l) {
      const double R_ = h->rows[l], C_ = h->cols[l];
      flops += 2.0 * n * R_ * C_;
      bytes += 4.0 * (n * R_ + n * C_ + 2.0 * R_ * C_);
      TcGroupDesc& q = d[l];
      std::memset(&q, 0, sizeof(q));
      q.M = h->rows[l]; q.N = h->cols[l]; q.K = n; q.splits = 1;
      q.A = h->X[l]; q.lda = h->ldr[l]; q.B = h->Y[l]; q.ldb = h->ldp[l];
      q.epi.kind = TC_EPI_AXPY; q.epi.C = h->arena + h->off[l]; q.epi.ldc = h->ldp[l]; q.epi.scale = h->scale + l;
      q.splits_used = nullptr;
    }
    static const int bn = tune_int("NG_TUNE_UPD_BN", 128);   // with BWD_BN 128: +3.7% (tools/tune_sweep3.sh)
    ProfScope ps(NG_PROF_UPD_GEMM, st, flops, bytes);
    // persistent double-buffered variant: measured on par (0.138 vs 0.136 ms NG+update phase), off
    static const int persistent = tune_int("NG_TUNE_UPD_PERSISTENT", 0);
    if (!s3 && persistent && bn == 128)
      NG_TRY(tc_gemm_tf32_axpy_persistent(st, d.data(), L));
    else
      NG_TRY(tc_gemm_tf32_grouped(st, d.data(), L, false, false, TC_EPI_AXPY, bn, s3));
  } else
  for (int l = 0; l < L; ++l) {
    float* W = h->arena + h->off[l];
    const double R_ = h->rows[l], C_ = h->cols[l];
    ProfScope ps(NG_PROF_UPD_GEMM, st, 2.0 * n * R_ * C_, 4.0 * (n * R_ + n * C_ + 2.0 * R_ * C_));
    if (tc) {
      TcEpilogue e;
      e.kind = TC_EPI_AXPY; e.C = W; e.ldc = h->ldp[l]; e.scale = h->scale + l;
      static const int bn = tune_int("NG_TUNE_UPD_BN", 128);   // with BWD_BN 128: +3.7% (tools/tune_sweep3.sh)
      NG_TRY(tc_gemm_tf32(st, h->rows[l], h->cols[l], n, h->X[l], h->ldr[l], false, h->Y[l], h->ldp[l], false, e, bn,
                          1, nullptr, s3));
    } else {
      NG_TRY((gemm_simt<float, false, false>(st, h->rows[l], h->cols[l], n, h->X[l], h->ldr[l], h->Y[l], h->ldp[l],
                                             EpiAxpyDevScale{W, h->ldp[l], h->scale + l})));
    }
  }
  h->have_fb = false;
  if (stats_out) {
    std::vector<float> sv(4 * L);
    NG_CUDA_TRY(cudaMemcpyAsync(sv.data(), h->stats, sizeof(float) * 4 * L, cudaMemcpyDeviceToHost, st));
    NG_CUDA_TRY(cudaStreamSynchronize(st));
    std::memset(stats_out, 0, sizeof(*stats_out));
    for (int l = 0; l < L; ++l) {
      stats_out->alpha_t[l] = sv[4 * l + 0];
      stats_out->gamma_in[l] = sv[4 * l + 1];
      stats_out->gamma_out[l] = sv[4 * l + 2];
      stats_out->updated_in[l] = upd_in[l];
      stats_out->updated_out[l] = upd_out[l];
    }
    NG_TRY(read_eflags(h, "nnet_update"));
  }
  return NG_OK;
}

ng_status nnet_get_params(nnet_t h, int32_t layer, float* host, int64_t count) {
  NG_REQUIRE(h && host, NG_EINVAL, "NULL argument");
  NG_REQUIRE(layer >= 0 && layer < h->L, NG_EINVAL, "layer out of range");
  NG_REQUIRE(count == (int64_t)h->rows[layer] * h->cols[layer], NG_ESHAPE, "count != rows*cols");
  NG_TRY(nnet_join(h));
  NG_CUDA_TRY(cudaStreamSynchronize(h->st));
  NG_CUDA_TRY(cudaMemcpy2D(host, sizeof(float) * h->cols[layer], h->arena + h->off[layer], sizeof(float) * h->ldp[layer],
                           sizeof(float) * h->cols[layer], h->rows[layer], cudaMemcpyDeviceToHost));
  return read_eflags(h, "nnet_get_params");
}

ng_status nnet_set_params(nnet_t h, int32_t layer, const float* host, int64_t count) {
  NG_REQUIRE(h && host, NG_EINVAL, "NULL argument");
  NG_REQUIRE(layer >= 0 && layer < h->L, NG_EINVAL, "layer out of range");
  NG_REQUIRE(count == (int64_t)h->rows[layer] * h->cols[layer], NG_ESHAPE, "count != rows*cols");
  NG_CUDA_TRY(cudaStreamSynchronize(h->st));
  NG_CUDA_TRY(cudaMemcpy2D(h->arena + h->off[layer], sizeof(float) * h->ldp[layer], host, sizeof(float) * h->cols[layer],
                           sizeof(float) * h->cols[layer], h->rows[layer], cudaMemcpyHostToDevice));
  return NG_OK;
}

ng_status nnet_get_ngsgd(nnet_t h, int32_t layer, int32_t side, ngsgd_t* out) {
  NG_REQUIRE(h && out, NG_EINVAL, "NULL argument");
  NG_REQUIRE(h->cfg.precond == 1, NG_ESTATE, "network has no online NG-SGD preconditioners");
  NG_REQUIRE(layer >= 0 && layer < h->L && (side == 0 || side == 1), NG_EINVAL, "bad layer/side");
  *out = side == 0 ? h->ng_in[layer] : h->ng_out[layer];
  return NG_OK;
}

int32_t nnet_comm_id_bytes(void) { return (int32_t)sizeof(ncclUniqueId); }

ng_status nnet_comm_get_unique_id(void* id_out) {
  NG_REQUIRE(id_out != nullptr, NG_EINVAL, "NULL argument");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) { set_error(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r)); return NG_ENCCL; }
  std::memcpy(id_out, &id, sizeof(id));
  return NG_OK;
}

ng_status nnet_comm_init(nnet_t h, const void* nccl_unique_id, int32_t rank, int32_t nranks) {
  NG_REQUIRE(h && nccl_unique_id, NG_EINVAL, "NULL argument");
  NG_REQUIRE(nranks >= 1 && nranks <= kMaxRanks && rank >= 0 && rank < nranks, NG_EINVAL,
             "bad rank/nranks (1 <= nranks <= 64)");
  NG_REQUIRE(h->comm == nullptr, NG_ESTATE, "communicator already initialised");
  ncclUniqueId id;
  std::memcpy(&id, nccl_unique_id, sizeof(id));
  ncclResult_t r = ncclCommInitRank(&h->comm, nranks, id, rank);
  if (r != ncclSuccess) { set_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r)); h->comm = nullptr; return NG_ENCCL; }
  h->rank = rank;
  h->nranks = nranks;
  // any nranks: equal shards of ceil(count / n) rounded up to 64 floats; the last shard(s)
  // are ragged (possibly empty) in the arena and padded in the gather buffer
  h->shard = (size_t)round_up((int64_t)((h->arena_count + nranks - 1) / nranks), 64);
  NG_TRY(nalloc(&h->recvbuf, h->shard * nranks));
  NG_TRY(nalloc(&h->gatherbuf, h->shard * nranks));
  NG_CUDA_TRY(cudaMemsetAsync(h->gatherbuf, 0, sizeof(float) * h->shard * nranks, h->st));
  return NG_OK;
}

ng_status nnet_average(nnet_t h, int32_t mode) {
  NG_REQUIRE(h != nullptr, NG_EINVAL, "NULL argument");
  NG_REQUIRE(h->comm != nullptr, NG_ENCCL, "nnet_comm_init not called");
  cudaStream_t st = h->st;
  const int nr = h->nranks;
  ncclResult_t r = ncclSuccess;
  ProfScope ps(NG_PROF_AVERAGE, st, 0.0, 4.0 * 2.0 * h->arena_count);
  if (mode == 0) {
    // shard p of every rank goes to rank p (all-to-all), rank p sums it in the fixed tree
    // order, then an in-place all-gather of the padded shards and one copy back
    auto len = [&](int p) -> size_t {
      const size_t lo = (size_t)p * h->shard;
      return lo >= h->arena_count ? 0 : std::min(h->shard, h->arena_count - lo);
    };
    const size_t mine = len(h->rank);
    r = ncclGroupStart();
    for (int p = 0; p < nr && r == ncclSuccess; ++p) {
      if (len(p) > 0) r = ncclSend(h->arena + (size_t)p * h->shard, len(p), ncclFloat, p, h->comm, st);
      if (r == ncclSuccess && mine > 0)
        r = ncclRecv(h->recvbuf + (size_t)p * h->shard, mine, ncclFloat, p, h->comm, st);
    }
    ncclResult_t r2 = ncclGroupEnd();
    if (r == ncclSuccess) r = r2;
    if (r == ncclSuccess) {
      NG_TRY(launch_tree_avg(st, nr, mine, h->shard, h->recvbuf, h->gatherbuf + (size_t)h->rank * h->shard));
      r = ncclAllGather(h->gatherbuf + (size_t)h->rank * h->shard, h->gatherbuf, h->shard, ncclFloat, h->comm, st);
    }
    if (r == ncclSuccess)
      NG_CUDA_TRY(cudaMemcpyAsync(h->arena, h->gatherbuf, sizeof(float) * h->arena_count, cudaMemcpyDeviceToDevice, st));
  } else {
    r = ncclAllReduce(h->arena, h->arena, h->arena_count, ncclFloat, ncclSum, h->comm, st);
    if (r == ncclSuccess) {
      scale_kernel<<<std::min<size_t>(4096, (h->arena_count + 255) / 256), 256, 0, st>>>(h->arena, h->arena_count,
                                                                                          1.0f / (float)nr);
      NG_TRY(check_launch("scale_kernel"));
    }
  }
  if (r != ncclSuccess) { set_error(std::string("nnet_average: ") + ncclGetErrorString(r)); return NG_ENCCL; }
  NG_CUDA_TRY(cudaStreamSynchronize(st));
  return read_eflags(h, "nnet_average");
}

ng_status nnet_select_best(nnet_t h, double objective, int32_t* winner_out) {
  NG_REQUIRE(h != nullptr, NG_EINVAL, "NULL argument");
  NG_REQUIRE(h->comm != nullptr, NG_ENCCL, "nnet_comm_init not called");
  NG_REQUIRE(std::isfinite(objective), NG_EINVAL, "objective must be finite");
  cudaStream_t st = h->st;
  const int nr = h->nranks;
  if (!h->objbuf) NG_TRY(nalloc(&h->objbuf, 2 * (size_t)nr));
  NG_CUDA_TRY(cudaMemcpyAsync(h->objbuf + nr, &objective, sizeof(double), cudaMemcpyHostToDevice, st));
  ncclResult_t r = ncclAllGather(h->objbuf + nr, h->objbuf, 1, ncclDouble, h->comm, st);
  if (r != ncclSuccess) { set_error(std::string("nnet_select_best: ") + ncclGetErrorString(r)); return NG_ENCCL; }
  std::vector<double> all(nr);
  NG_CUDA_TRY(cudaMemcpyAsync(all.data(), h->objbuf, sizeof(double) * nr, cudaMemcpyDeviceToHost, st));
  NG_CUDA_TRY(cudaStreamSynchronize(st));
  int win = 0;                                  // the best objective; ties -> the lowest rank
  for (int p = 1; p < nr; ++p)
    if (all[p] > all[win]) win = p;
  r = ncclBroadcast(h->arena, h->arena, h->arena_count, ncclFloat, win, h->comm, st);
  if (r != ncclSuccess) { set_error(std::string("nnet_select_best: ") + ncclGetErrorString(r)); return NG_ENCCL; }
  NG_CUDA_TRY(cudaStreamSynchronize(st));
  if (winner_out) *winner_out = win;
  return read_eflags(h, "nnet_select_best");
}

ng_status nnet_average_local(nnet_t* nets, int32_t n) {
  NG_REQUIRE(nets != nullptr && n >= 1 && n <= kMaxRanks, NG_EINVAL, "bad network list (1 <= n <= 64)");
  nnet_ctx* h0 = nets[0];
  NG_REQUIRE(h0 != nullptr, NG_EINVAL, "NULL network");
  for (int q = 1; q < n; ++q) {
    NG_REQUIRE(nets[q] != nullptr && nets[q]->arena_count == h0->arena_count, NG_ESHAPE,
               "nnet_average_local: networks of different shapes");
    NG_TRY(nnet_join(nets[q]));
    NG_CUDA_TRY(cudaStreamSynchronize(nets[q]->st));
  }
  NG_TRY(nnet_join(h0));
  const size_t count = h0->arena_count;
  cudaStream_t st = h0->st;
  // stack the arenas (rank order) and sum them in the fixed tree of nnet_average
  float* stack = nullptr;
  NG_CUDA_TRY(cudaMallocAsync((void**)&stack, sizeof(float) * count * (n + 1), st));
  for (int q = 0; q < n; ++q)
    NG_CUDA_TRY(cudaMemcpyAsync(stack + (size_t)q * count, nets[q]->arena, sizeof(float) * count,
                                cudaMemcpyDeviceToDevice, st));
  ng_status s = launch_tree_avg(st, n, count, count, stack, stack + (size_t)n * count);
  for (int q = 0; q < n && s == NG_OK; ++q)
    if (cudaMemcpyAsync(nets[q]->arena, stack + (size_t)n * count, sizeof(float) * count, cudaMemcpyDeviceToDevice,
                        st) != cudaSuccess) s = NG_ECUDA;
  cudaFreeAsync(stack, st);
  if (s != NG_OK) return s;
  NG_CUDA_TRY(cudaStreamSynchronize(st));
  return NG_OK;
}

ng_status nnet_arena_size(nnet_t h, int64_t* count) {
  NG_REQUIRE(h && count, NG_EINVAL, "NULL argument");
  *count = (int64_t)h->arena_count;
  return NG_OK;
}

ng_status nnet_copy_arena(nnet_t h, float* dev, int32_t direction) {
  NG_REQUIRE(h && dev, NG_EINVAL, "NULL argument");
  NG_TRY(nnet_join(h));
  const size_t bytes = sizeof(float) * h->arena_count;
  NG_CUDA_TRY(cudaMemcpyAsync(direction ? h->arena : dev, direction ? dev : h->arena, bytes, cudaMemcpyDeviceToDevice,
                              h->st));
  return NG_OK;
}

static ng_status comb_args(nnet_ctx* h, const float* const* models, int P, const float* w, CombineArgs* a) {
  NG_REQUIRE(models != nullptr && P >= 1 && P <= kCombMax, NG_EINVAL, "1 <= P <= 32 models");
  std::memset(a, 0, sizeof(*a));
  a->P = P;
  for (int p = 0; p < P; ++p) { NG_REQUIRE(models[p] != nullptr, NG_EINVAL, "NULL model"); a->model[p] = models[p]; }
  if (w)
    for (int l = 0; l < h->L; ++l)
      for (int p = 0; p < P; ++p) a->w[l * kCombMax + p] = w[l * P + p];
  for (int l = 0; l < h->L; ++l) a->off[l] = (int64_t)h->off[l];
  a->off[h->L] = (int64_t)h->arena_count;
  return NG_OK;
}

ng_status nnet_set_combination(nnet_t h, const float* const* models, int32_t P, const float* weights) {
  NG_REQUIRE(h && weights, NG_EINVAL, "NULL argument");
  CombineArgs a;
  NG_TRY(comb_args(h, models, P, weights, &a));
  NG_TRY(nnet_join(h));
  combine_kernel<<<dim3(std::min<int64_t>(1024, ceil_div(h->arena_count, 256)), h->L), 256, 0, h->st>>>(a, h->arena);
  return check_launch("combine_kernel");
}

ng_status nnet_combination_grad(nnet_t h, const float* const* models, int32_t P, double* grad) {
  NG_REQUIRE(h && grad, NG_EINVAL, "NULL argument");
  NG_REQUIRE(h->have_fb, NG_ESTATE, "nnet_combination_grad before nnet_forward_backward");
  CombineArgs a;
  NG_TRY(comb_args(h, models, P, nullptr, &a));
  cudaStream_t st = h->st;
  if (!h->gradbuf) {
    NG_TRY(nalloc(&h->gradbuf, h->arena_count));
    NG_TRY(nalloc(&h->cgpart, (size_t)16 * kCombMax));
    NG_CUDA_TRY(cudaMemsetAsync(h->gradbuf, 0, sizeof(float) * h->arena_count, st));
  }
  const int n = h->n_last;
  // G_l = X_l^T Y_l (the gradient of the objective w.r.t. W_l) for every layer
  for (int l = 0; l < h->L; ++l) {
    float* Gl = h->gradbuf + h->off[l];
    if (h->cfg.precision != NG_FP32_SIMT) {
      TcEpilogue e;
      e.kind = TC_EPI_STORE; e.C = Gl; e.ldc = h->ldp[l];
      NG_TRY(tc_gemm_tf32(st, h->rows[l], h->cols[l], n, h->X[l], h->ldr[l], false, h->Y[l], h->ldp[l], false, e, 128,
                          1, nullptr, h->cfg.precision == NG_FP32));
    } else {
      NG_TRY((gemm_simt<float, false, false>(st, h->rows[l], h->cols[l], n, h->X[l], h->ldr[l], h->Y[l], h->ldp[l],
                                             EpiStore<float>{Gl, h->ldp[l], 1.f})));
    }
  }
  combine_grad_kernel<<<dim3(P, h->L), 256, 0, st>>>(a, h->gradbuf, h->cgpart);
  NG_TRY(check_launch("combine_grad_kernel"));
  std::vector<double> g((size_t)16 * kCombMax);
  NG_CUDA_TRY(cudaMemcpyAsync(g.data(), h->cgpart, sizeof(double) * g.size(), cudaMemcpyDeviceToHost, st));
  NG_CUDA_TRY(cudaStreamSynchronize(st));
  for (int l = 0; l < h->L; ++l)
    for (int p = 0; p < P; ++p) grad[l * P + p] = g[l * kCombMax + p];
  return read_eflags(h, "nnet_combination_grad");
}

ng_status ng_compress_frames(int32_t n, int32_t dim, const float* x, int64_t ldx, uint8_t* q, int64_t ldq, double* lo,
                             double* step, void* stream) {
  NG_REQUIRE(x && q && lo && step, NG_EINVAL, "NULL argument");
  NG_REQUIRE(n >= 1 && dim >= 1 && ldx >= dim && ldq >= dim, NG_ESHAPE, "bad shape");
  cudaStream_t st = (cudaStream_t)stream;
  compress_range_kernel<<<dim, 256, 0, st>>>(n, dim, x, ldx, lo, step);
  NG_TRY(check_launch("compress_range_kernel"));
  compress_codes_kernel<<<std::min(4096, ceil_div((int64_t)n * dim, 256)), 256, 0, st>>>(n, dim, x, ldx, lo, step, q,
                                                                                       ldq);
  return check_launch("compress_codes_kernel");
}

ng_status ng_debug_tree_avg(int32_t nr, int64_t count, const float* in, float* out, void* stream) {
  NG_REQUIRE(in && out, NG_EINVAL, "NULL argument");
  NG_REQUIRE(nr >= 1 && nr <= kMaxRanks && count >= 0, NG_EINVAL, "bad nr / count");
  return launch_tree_avg((cudaStream_t)stream, nr, (size_t)count, (size_t)count, in, out);
}

}  // extern "C"
