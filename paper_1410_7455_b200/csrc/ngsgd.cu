// ngsgd.cu -- online natural-gradient preconditioner (Appendix B of arXiv 1410.7455)
// on sm_100a.  Every step of B.5 runs in the kernels below; the paper's
// CPU part (Z_t, its eigendecomposition, rho/D/E/A_t) runs
// in ONE CTA on the device (refresh_kernel), so a step never crosses to the host.
//
// Per call (non-update):  proj (H partials) -> reduce H -> apply (X_hat, partial row
//   norms) -> finalize (p_i, tr(X X^T), sum p, gamma)
// Per call (update):      proj -> reduce H -> J = H^T X -> K = J J^T, L -> apply ->
//   finalize -> refresh (Z, Jacobi eig, floors, rho', D', E', A_t) -> B_t = J + s.W ->
//   W' = A_t B_t -> [gated] W'W'^T -> [gated] check/Cholesky -> [gated] M W'.
#include <math.h>

#include <cmath>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "eig_jacobi.cuh"
#include "eig_tri.cuh"
#include "eig_topr.cuh"
#include "gemm_simt.cuh"
#include "gemm_tc.cuh"
#include "ngsgd_impl.cuh"

namespace ng {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }

// ---- instrumentation -------------------------------------------------------------
static std::atomic<int64_t> g_launches{0};
static uint32_t g_prof_mask = 0;
static std::vector<cudaEvent_t> g_ev0, g_ev1;
static std::vector<int> g_ev_group;
static int g_ev_used = 0;
static ng_profile_stats g_prof{};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static void prof_flush() {
  for (int i = 0; i < g_ev_used; ++i) {
    float ms = 0.f;
    cudaEventSynchronize(g_ev1[i]);
    if (cudaEventElapsedTime(&ms, g_ev0[i], g_ev1[i]) == cudaSuccess) g_prof.ms[g_ev_group[i]] += ms;
  }
  g_ev_used = 0;
}

ProfScope::ProfScope(int grp, cudaStream_t s, double flops, double bytes) {
  if (!((g_prof_mask >> grp) & 1u)) return;
  if (g_ev_used == (int)g_ev0.size()) prof_flush();
  group = grp;
  st = s;
  slot = g_ev_used++;
  g_ev_group[slot] = grp;
  g_prof.launches[grp] += 1;
  g_prof.flops[grp] += flops;
  g_prof.bytes[grp] += bytes;
  cudaEventRecord(g_ev0[slot], s);
}

ProfScope::~ProfScope() {
  if (slot >= 0) cudaEventRecord(g_ev1[slot], st);
}

ng_status status_from_flags(uint32_t f, const char* where) {
  if (f & kErrNotPD) { set_error(std::string(where) + ": Cholesky of O_t failed (corrupted NG state, B.3.1)"); return NG_ENOTPD; }
  if (f & kErrLabel) { set_error(std::string(where) + ": label out of range"); return NG_ELABEL; }
  if (f & kErrNonFinite) { set_error(std::string(where) + ": non-finite value in device data"); return NG_ENONFINITE; }
  return NG_OK;
}

constexpr int kApplyRows = 16, kApplyCols = 128;
int rr_chunks(int D);
// The refresh chain (side stream) only gates the state's next call; give its small,
// dependent kernels the highest stream priority so that they are not queued behind the
// main stream's full-GPU GEMMs (NG_TUNE_SIDE_PRIORITY=0 keeps the default priority).
inline int refresh_priority() {
  static int v = 1;
  static bool done = false;
  if (!done) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    v = tune_int("NG_TUNE_SIDE_PRIORITY", 1) ? hi : lo;
    done = true;
  }
  return v;
}
// Column tile of the tensor-core NG apply (NG_TUNE_APPLY_BN: 32, 64 or 128).
inline int apply_bn() {
  static const int v = tune_int("NG_TUNE_APPLY_BN", 128);
  return (v == 32 || v == 64) ? v : 128;
}
constexpr int kTcMaxSplits = 32;   // split-K capacity (H, K, L) of the tensor-core path
constexpr int kTcJSplits = 4;      // split-K of J = H^T X (K = N)
constexpr int kMaxRank = 112;

// ------------------------------------------------------------------------------------
// kernels: apply / finalize / reductions
// ------------------------------------------------------------------------------------

// X_hat = X - H W (eqn:hatxt:compute:2), in place; partial row sums of
// x_i^2 (for tr(X X^T)) and x_hat_i^2 (p_i, eqn:pi) over this column tile.
__global__ void __launch_bounds__(256)
apply_kernel(int n, int D, int R, float* __restrict__ X, int64_t ldx, const float* __restrict__ H,
             const float* __restrict__ W, int64_t ldw, float* __restrict__ xxpart,
             float* __restrict__ ppart, int64_t part_ld) {
  extern __shared__ __align__(16) unsigned char ng_smem[];
  float* sm = reinterpret_cast<float*>(ng_smem);
  float* Hs = sm;                          // kApplyRows x R
  float* Ws = sm + kApplyRows * R;         // R x kApplyCols
  const int r0 = blockIdx.x * kApplyRows, c0 = blockIdx.y * kApplyCols;
  for (int i = threadIdx.x; i < kApplyRows * R; i += blockDim.x) {
    const int rr = i / R, k = i % R;
    Hs[i] = (r0 + rr < n) ? H[(int64_t)(r0 + rr) * R + k] : 0.f;
  }
  for (int i = threadIdx.x; i < R * kApplyCols; i += blockDim.x) {
    const int k = i / kApplyCols, cc = i % kApplyCols;
    Ws[i] = (c0 + cc < D) ? W[(int64_t)k * ldw + c0 + cc] : 0.f;
  }
  __syncthreads();
  const int row = threadIdx.x >> 4, l16 = threadIdx.x & 15;
  const int gr = r0 + row;
  float xx = 0.f, pp = 0.f;
#pragma unroll
  for (int j = 0; j < kApplyCols / 16; ++j) {
    const int cc = l16 + 16 * j, gc = c0 + cc;
    float acc = 0.f;
    for (int k = 0; k < R; ++k) acc = fmaf(Hs[row * R + k], Ws[k * kApplyCols + cc], acc);
    if (gr < n && gc < D) {
      float* px = X + (int64_t)gr * ldx + gc;
      const float x = *px;
      xx = fmaf(x, x, xx);
      const float xn = x - acc;
      *px = xn;
      pp = fmaf(xn, xn, pp);
    }
  }
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
    xx += __shfl_xor_sync(0xffffffffu, xx, o);
    pp += __shfl_xor_sync(0xffffffffu, pp, o);
  }
  if (l16 == 0 && gr < n) {
    xxpart[(int64_t)blockIdx.y * part_ld + gr] = xx;
    ppart[(int64_t)blockIdx.y * part_ld + gr] = pp;
  }
}

// R == 0: X_hat = X; partial row norms only.
__global__ void rownorm_part_kernel(int n, int D, const float* __restrict__ X, int64_t ldx,
                                    float* __restrict__ xxpart, float* __restrict__ ppart) {
  const int row = blockIdx.x;
  float s = 0.f;
  for (int j = threadIdx.x; j < D; j += blockDim.x) { const float x = X[(int64_t)row * ldx + j]; s = fmaf(x, x, s); }
  __shared__ float sc[32];
  s = block_sum(s, sc);
  if (threadIdx.x == 0) { xxpart[row] = s; ppart[row] = s; }
}

// p_i = sum over tiles (fixed order); tr(X X^T) and sum p_i with the same tree (reading
// R27); gamma = sqrt(tr(X X^T)/sum p) or 1 (eqn:gammat).
__global__ void __launch_bounds__(512)
finalize_kernel(int n, int tiles, const float* __restrict__ xxpart, const float* __restrict__ ppart,
                int64_t part_ld, float* __restrict__ p_int, float* __restrict__ p_out,
                double* __restrict__ sums, float* __restrict__ gamma_int,
                float* __restrict__ gamma_out, int* __restrict__ flags) {
  __shared__ double sc[32];
  double sxx = 0.0, spp = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    // the same summation tree as finalize_group_kernel
    float xa[4] = {0.f, 0.f, 0.f, 0.f}, pa[4] = {0.f, 0.f, 0.f, 0.f};
    int t = 0;
    for (; t + 4 <= tiles; t += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        xa[u] += xxpart[(int64_t)(t + u) * part_ld + i];
        pa[u] += ppart[(int64_t)(t + u) * part_ld + i];
      }
    }
    for (; t < tiles; ++t) { xa[0] += xxpart[(int64_t)t * part_ld + i]; pa[0] += ppart[(int64_t)t * part_ld + i]; }
    const float xx = (xa[0] + xa[1]) + (xa[2] + xa[3]), pp = (pa[0] + pa[1]) + (pa[2] + pa[3]);
    p_int[i] = pp;
    if (p_out) p_out[i] = pp;
    sxx += (double)xx;
    spp += (double)pp;
  }
  sxx = block_sum(sxx, sc);
  spp = block_sum(spp, sc);
  if (threadIdx.x == 0) {
    sums[0] = sxx;
    sums[1] = spp;
    const float g = (spp > 0.0) ? (float)sqrt(sxx / spp) : 1.0f;
    *gamma_int = g;
    if (gamma_out) *gamma_out = g;
    if (!isfinite(sxx) || !isfinite(spp)) atomicOr(reinterpret_cast<unsigned*>(flags + 3), kErrNonFinite);
  }
}

// out[i] = sum_z part[z * zstride + i], fixed order.
__global__ void reduce_splits_kernel(float* __restrict__ out, const float* __restrict__ part, int64_t count,
                                     int splits, int64_t zstride, const int* gate) {
  if (gate && *gate == 0) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    float a4[4] = {0.f, 0.f, 0.f, 0.f};   // the summation tree of seg_reduce_kernel
    int z = 0;
    for (; z + 4 <= splits; z += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) a4[u] += part[(int64_t)(z + u) * zstride + i];
    }
    for (; z < splits; ++z) a4[0] += part[(int64_t)z * zstride + i];
    out[i] = (a4[0] + a4[1]) + (a4[2] + a4[3]);
  }
}

// out[r][j] = sum_z part[z][r][j] (row-strided 2D, fixed order).
__global__ void reduce_rows_kernel(float* __restrict__ out, int64_t ld, const float* __restrict__ part, int64_t zstride,
                                   int splits, int R, int D) {
  const int64_t total = (int64_t)R * D;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t off = (i / D) * ld + (i % D);
    float a4[4] = {0.f, 0.f, 0.f, 0.f};   // the summation tree of seg_reduce_kernel
    int z = 0;
    for (; z + 4 <= splits; z += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) a4[u] += part[(int64_t)(z + u) * zstride + off];
    }
    for (; z < splits; ++z) a4[0] += part[(int64_t)z * zstride + off];
    out[off] = (a4[0] + a4[1]) + (a4[2] + a4[3]);
  }
}

// B_t = J_t + (N(1-eta)/eta)(D_t + rho_t I) W_t, in J's buffer.
__global__ void bscale_kernel(int R, int D, float* __restrict__ J, const float* __restrict__ W,
                              int64_t ldw, const float* __restrict__ s) {
  const int64_t total = (int64_t)R * D;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / D), j = (int)(i % D);
    J[(int64_t)r * ldw + j] = fmaf(s[r], W[(int64_t)r * ldw + j], J[(int64_t)r * ldw + j]);
  }
}

__global__ void copy_gated_kernel(int R, int D, float* __restrict__ dst, const float* __restrict__ src,
                                  int64_t ld, const int* gate) {
  if (gate && *gate == 0) return;
  const int64_t total = (int64_t)R * D;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / D), j = (int)(i % D);
    dst[(int64_t)r * ld + j] = src[(int64_t)r * ld + j];
  }
}

// ------------------------------------------------------------------------------------
// refresh: the R x R part of the update, one CTA, FP64
// ------------------------------------------------------------------------------------

// Eigensolver variants of refresh_kernel:
//   REFRESH_INPLACE  one CTA, in-place two-barrier Jacobi (any R <= kMaxRank)
//   REFRESH_TRI      one CTA, Householder + relatively robust representation + twisted
//                    factorisation eigenvectors (eig_tri.cuh), falling back to the in-place
//                    Jacobi when its orthogonality check fails (default, 2 <= R <= 80)
// (Round-1/2 alternatives measured slower and removed -- a permuted ping-pong Jacobi, its
// thread-block-cluster split and a divide-and-conquer solver.)
enum RefreshMode : int { REFRESH_INPLACE = 0, REFRESH_TRI = 4 };

// Shared-memory plan (offsets in doubles from the 16-byte aligned dynamic base).
struct RefreshSmem {
  int R, npad, LD, LDV, mp, mode;
  size_t o_d, o_lam, o_z0, o_v0, o_cs, o_ring, o_int, total_bytes;
};
__host__ __device__ inline RefreshSmem refresh_plan(int R, int mode) {
  RefreshSmem p;
  p.R = R;
  p.npad = R + (R & 1);
  p.LD = R + 1;
  p.LDV = (R + 3) / 4 * 4;
  p.mp = R / 2 + 1;
  p.mode = mode;
  size_t o = 0;
  p.o_d = o;    o += 5 * (size_t)R + 40;               // d, emh, dr, c, dn, red[32], scalars[8]
  p.o_lam = o;  o += (size_t)p.npad + 2;               // eigenvalues
  o = (o + 1) & ~(size_t)1;                            // 16-byte alignment
  if (mode == REFRESH_TRI) {   // eig_tri's plan; Z_t in its A region (ld R + 1)
    const TriPlan tp = tri_plan(R);
    p.o_ring = o;
    p.o_z0 = o + tp.oA;
    p.o_v0 = o + tp.oX;                    // Jacobi fallback: eigenvector rows (ld LDV)
    p.o_cs = o + tp.oQ;                    // Jacobi fallback: (c, s) scratch
    o += ((tp.total + 15) / 16) * 2;
  } else {
    p.o_z0 = o; o += ((size_t)R * p.LD + 1) & ~(size_t)1;
    p.o_v0 = o; o += (size_t)R * p.LDV;
    p.o_cs = o; o += 2 * (size_t)p.mp + 2;
    p.o_ring = o;
  }
  p.o_int = o;
  // ints: perm[npad], nrot[64 + 2 mp], iflag, phantom, fb, offmax[32] (float)
  p.total_bytes = sizeof(double) * o + sizeof(int) * ((size_t)p.npad + 64 + 2 * p.mp + 3 + 32) + 64;
  return p;
}

__device__ unsigned long long g_ref_t[256][9];   // refresh timing (ng_debug_refresh_times): R, start, end ns, eig, phase cycles
__device__ unsigned int g_ref_n;

// One state's refresh job (the grouped launch passes a table of them).
struct RefreshJob {
  int R, D, N, pad_;
  double eta, alpha, eps;
  const float* KL;
  double* dstate;
  const double* sums;
  float* Amat;
  float* svec;
  int* flags;
};

// The refresh in three calls -- refresh_pre (Z_t), the eigensolver, refresh_post (everything
// after it) -- with nothing but the job and a few shared-memory scalars carried across: the
// eigensolver is a separate (non-inlined) function, and values live across a call cost it
// registers (measured: its tridiagonalisation 182 -> 148 us in the grouped kernel).
// Shared scalars after red[32]: [0] sum d, [1] max |z_ii|, [2] t_start, [3] t_eig0 (ns).
__device__ __forceinline__ double refresh_zval(const RefreshJob& J, const double* emh, const double* dr, int i, int j) {
  const int R = J.R;
  const float* K = J.KL;
  const float* L = J.KL + R * R;
  const double a1 = J.eta * J.eta / ((double)J.N * J.N), a2 = (1.0 - J.eta) * (1.0 - J.eta);
  const double a3 = J.eta * (1.0 - J.eta) / J.N;
  const double ks = 0.5 * ((double)K[i * R + j] + (double)K[j * R + i]);
  const double ls = 0.5 * ((double)L[i * R + j] + (double)L[j * R + i]);
  double z = a1 * emh[i] * ks * emh[j] + a3 * emh[i] * ls * emh[j] * (dr[i] + dr[j]);
  if (i == j) z += a2 * dr[i] * dr[i];
  return z;
}

template <int MODE>
__device__ __noinline__ void refresh_pre(const RefreshJob& J) {
  extern __shared__ __align__(16) unsigned char ng_smem[];
  double* sm = reinterpret_cast<double*>(ng_smem);
  unsigned long long t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  const int R = J.R;
  const RefreshSmem P = refresh_plan(R, MODE);
  double* d = sm + P.o_d;               // R   old d
  double* emh = d + R;                  // R   E_t^{-1/2}
  double* dr = emh + R;                 // R   d + rho
  double* red = dr + 3 * R;             // 32 reduction scratch, then the scalars
  int* iflag = reinterpret_cast<int*>(sm + P.o_int) + P.npad + 64 + 2 * P.mp;
  const int tid = threadIdx.x, nt = blockDim.x;
  const double rho = J.dstate[0];
  for (int i = tid; i < R; i += nt) d[i] = J.dstate[1 + i];
  __syncthreads();
  // beta_t (eqn:beta2) and e_tii (eqn:etii)
  double sd = 0.0;
  for (int i = tid; i < R; i += nt) sd += d[i];
  sd = block_sum(sd, red);
  const double beta = rho * (1.0 + J.alpha) + (J.alpha / J.D) * sd;
  for (int i = tid; i < R; i += nt) {
    const double e = 1.0 / (beta / d[i] + 1.0);
    emh[i] = 1.0 / sqrt(e);
    dr[i] = d[i] + rho;
  }
  if (tid == 0) *iflag = 0;
  __syncthreads();
  // Z_t by eqn:zt:compute, symmetrised
  double* Z = sm + P.o_z0;
  for (int idx = tid; idx < R * R; idx += nt) {
    const int i = idx / R, j = idx % R;
    Z[i * P.LD + j] = refresh_zval(J, emh, dr, i, j);
  }
  double zmax = 0.0;
  for (int i = tid; i < R; i += nt) zmax = fmax(zmax, fabs(refresh_zval(J, emh, dr, i, i)));
  zmax = block_max(zmax, red);   // (its barriers also complete Z)
  if (tid == 0) {
    unsigned long long t_eig0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_eig0));
    red[32] = sd;
    red[33] = zmax;
    reinterpret_cast<unsigned long long*>(red)[34] = t_start;
    reinterpret_cast<unsigned long long*>(red)[35] = t_eig0;
  }
  __syncthreads();
}

// eig_ok: the default solver's result (REFRESH_TRI); 0 runs the in-place Jacobi on Z_t (the
// fallback, and REFRESH_INPLACE's solver).  Z = U C U^T (eqn:zt:eig:repeat); Jacobi rel_tol
// 1e-7: rotations stop once every |z_pq| <= 1e-7 sqrt(z_pp z_qq) (eigenvector error ~1e-7 /
// relative gap, far below the FP32 storage of A_t and W_{t+1}).
template <int MODE>
__device__ __noinline__ void refresh_post(const RefreshJob& J, int dbg_mask, int eig_ok, const long long* eig_st) {
  extern __shared__ __align__(16) unsigned char ng_smem[];
  double* sm = reinterpret_cast<double*>(ng_smem);
  const int R = J.R, D = J.D, N = J.N;
  const double eta = J.eta, alpha = J.alpha, eps = J.eps;
  const RefreshSmem P = refresh_plan(R, MODE);
  double* d = sm + P.o_d;
  double* emh = d + R;
  double* dr = emh + R;
  double* c = dr + R;                   // R   sorted eigenvalues
  double* dn = c + R;                   // R   new d
  double* red = dn + R;
  double* lam = sm + P.o_lam;           // eigenvalues
  int* perm = reinterpret_cast<int*>(sm + P.o_int);   // npad
  int* nrot = perm + P.npad;            // 32 per-warp sweep counts, 32 spare, then 2*mp pair table
  int* iflag = nrot + 64 + 2 * P.mp;    // floored
  float* offmax = reinterpret_cast<float*>(iflag + 3);  // 32 (per-warp max ratio)
  const int tid = threadIdx.x, nt = blockDim.x;
  const double rho = J.dstate[0];
  const double sd = red[32], zmax = red[33];
  double* Z = sm + P.o_z0;
  int sweeps;
  const double* V;   // eigenvector rows (index order), row stride ldv
  int ldv;
  if (MODE == REFRESH_TRI && eig_ok) {
    const TriPlan tp = tri_plan(R);
    const double* tb = sm + P.o_ring;
    for (int i = tid; i < R; i += nt) lam[i] = tb[tp.olam + i];
    sweeps = 0;
    V = tb + tp.oA;
    ldv = tp.lda;
  } else {
    if (MODE == REFRESH_TRI) {
      // fallback: Z_t again (the solve overwrote it), in-place cyclic Jacobi
      __syncthreads();
      for (int idx = tid; idx < R * R; idx += nt) {
        const int i = idx / R, j = idx % R;
        Z[i * P.LD + j] = refresh_zval(J, emh, dr, i, j);
        g_tri_fail_z[idx] = Z[i * P.LD + j];
      }
      if (tid == 0) { g_tri_fail_n = R; atomicAdd(&g_tri_fail_count, 1); }
      __syncthreads();
    }
    JacobiSmem<double> scr{sm + P.o_cs, sm + P.o_cs + P.mp, nrot, offmax};
    sweeps = jacobi_eig_smem<double>(Z, P.LD, sm + P.o_v0, P.LDV, R, scr, 20, 1e-15 * zmax, 1e-7, dbg_mask);
    if (MODE == REFRESH_TRI && sweeps == 0) sweeps = 1;   // flags[4] > 0 marks the fallback
    for (int i = tid; i < R; i += nt) lam[i] = Z[i * P.LD + i];
    V = sm + P.o_v0;
    ldv = P.LDV;
  }
  unsigned long long t_eig1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_eig1));
  __syncthreads();
  // descending order
  for (int i = tid; i < R; i += nt) {
    const double li = lam[i];
    int r = 0;
    for (int j = 0; j < R; ++j) { const double lj = lam[j]; r += (lj > li) || (lj == li && j < i); }
    perm[r] = i;
  }
  __syncthreads();
  // floor C at (1-eta)^2 rho_t^2 (reading R13)
  const double cf = (1.0 - eta) * (1.0 - eta) * rho * rho;
  for (int r = tid; r < R; r += nt) {
    double cr = lam[perm[r]];
    if (cr < cf) { cr = cf; atomicOr(iflag, 1); }
    c[r] = cr;
  }
  __syncthreads();
  // rho'_{t+1} (eqn:rhodash2), D_{t+1} (eqn:dt1), rho_{t+1} (eqn:rhot1)
  const double trX = J.sums[0];
  double ssc = 0.0;
  for (int r = tid; r < R; r += nt) ssc += sqrt(c[r]);
  ssc = block_sum(ssc, red);
  const double rho_dash = ((eta / N) * trX + (1.0 - eta) * (D * rho + sd) - ssc) / (double)(D - R);
  const double rho_new = fmax(eps, rho_dash);
  for (int r = tid; r < R; r += nt) dn[r] = fmax(sqrt(c[r]) - rho_dash, eps);
  __syncthreads();
  double sdn = 0.0;
  for (int r = tid; r < R; r += nt) sdn += dn[r];
  sdn = block_sum(sdn, red);
  const double beta_new = rho_new * (1.0 + alpha) + (alpha / D) * sdn;
  // A_t = (eta/N) E_{t+1}^{1/2} C^{-1/2} U^T E_t^{-1/2}
  for (int idx = tid; idx < R * R; idx += nt) {
    const int r = idx / R, j = idx % R;
    const double en = 1.0 / (beta_new / dn[r] + 1.0);
    J.Amat[idx] = (float)((eta / N) * sqrt(en) / sqrt(c[r]) * V[perm[r] * ldv + j] * emh[j]);
  }
  // row scale of B_t with the OLD d, rho
  for (int k = tid; k < R; k += nt) J.svec[k] = (float)((N * (1.0 - eta) / eta) * dr[k]);
  double cmax = 0.0, cmin = 1e300;
  for (int r = tid; r < R; r += nt) { cmax = fmax(cmax, c[r]); cmin = fmin(cmin, c[r]); }
  cmax = block_max(cmax, red);
  cmin = -block_max(-cmin, red);
  __syncthreads();
  // commit the new state
  if (tid == 0) J.dstate[0] = rho_new;
  for (int r = tid; r < R; r += nt) {
    J.dstate[1 + r] = dn[r];
    J.dstate[1 + R + r] = 1.0 / (beta_new / dn[r] + 1.0);
  }
  if (tid == 0) {
    const int fl = *iflag;
    int* flags = J.flags;
    flags[0] = fl;
    flags[1] = (fl || cmax / cmin > 1e6) ? 1 : 0;     // B.3.1 trigger
    flags[2] = 0;
    flags[4] = sweeps;
    if (!isfinite(rho_new) || !isfinite(sdn)) atomicOr(reinterpret_cast<unsigned*>(flags + 3), kErrNonFinite);
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    const unsigned slot = atomicAdd(&g_ref_n, 1u) & 255u;
    const unsigned long long* ts = reinterpret_cast<const unsigned long long*>(red);
    g_ref_t[slot][0] = (unsigned long long)R | ((unsigned long long)D << 16);
    g_ref_t[slot][1] = ts[34];
    g_ref_t[slot][2] = t_end;
    g_ref_t[slot][3] = ts[35];
    g_ref_t[slot][4] = t_eig1;
    if (MODE == REFRESH_TRI) {   // cycles: tridiagonalisation, split..multisection, RQI + vectors, clusters + check + back
      g_ref_t[slot][5] = (unsigned long long)(eig_st[1] - eig_st[0]);
      g_ref_t[slot][6] = (unsigned long long)(eig_st[2] - eig_st[1]);
      g_ref_t[slot][7] = (unsigned long long)(eig_st[3] - eig_st[2]);
      g_ref_t[slot][8] = (unsigned long long)(eig_st[4] - eig_st[3]);
    }
  }
}

template <int MODE>
__device__ __forceinline__ void refresh_body(const RefreshJob& J, int dbg_mask) {
  extern __shared__ __align__(16) unsigned char ng_smem[];
  __shared__ long long eig_st[8];   // eigensolver phase stamps (thread 0)
  refresh_pre<MODE>(J);
  int ok = 0;
  if (MODE == REFRESH_TRI) {
    double* sm = reinterpret_cast<double*>(ng_smem);
    ok = eig_tri(tri_plan(J.R), sm + refresh_plan(J.R, MODE).o_ring, eig_st);
  }
  refresh_post<MODE>(J, dbg_mask, ok, eig_st);
}

template <int MODE>
__global__ void __launch_bounds__(MODE == REFRESH_TRI ? kTriThreads : 1024, 1)
refresh_kernel(int R, int D, int N, double eta, double alpha, double eps,
               const float* __restrict__ KL, double* __restrict__ dstate,
               const double* __restrict__ sums, float* __restrict__ Amat,
               float* __restrict__ svec, int* __restrict__ flags, int dbg_mask) {
  const RefreshJob J{R, D, N, 0, eta, alpha, eps, KL, dstate, sums, Amat, svec, flags};
  refresh_body<MODE>(J, dbg_mask);
}

// Grouped refresh: every updating state of a step in ONE launch, one CTA per state
// (Householder + RRR eigensolver, 2 <= R <= kTriMax), on one side stream.
constexpr int kRefreshGroupMax = 16;
struct RefreshGroup {
  RefreshJob j[kRefreshGroupMax];
  int count, dbg;
};
__global__ void __launch_bounds__(kTriThreads, 1) refresh_group_kernel(const __grid_constant__ RefreshGroup g) {
  refresh_body<REFRESH_TRI>(g.j[blockIdx.x], g.dbg);
}

// B_t = J_t + (N(1-eta)/eta)(D_t + rho_t I) W_t of every job (blockIdx.y), in J's buffer.
struct BscaleGroup {
  float* J[kRefreshGroupMax];
  const float* W[kRefreshGroupMax];
  const float* s[kRefreshGroupMax];
  int64_t ldw[kRefreshGroupMax];
  int R[kRefreshGroupMax], D[kRefreshGroupMax];
};
__global__ void __launch_bounds__(256) bscale_group_kernel(const __grid_constant__ BscaleGroup g) {
  const int q = blockIdx.y, R = g.R[q], D = g.D[q];
  const int64_t total = (int64_t)R * D, ldw = g.ldw[q];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / D), j = (int)(i % D);
    g.J[q][(int64_t)r * ldw + j] = fmaf(g.s[q][r], g.W[q][(int64_t)r * ldw + j], g.J[q][(int64_t)r * ldw + j]);
  }
}

// B.3.1 (reading R5): O = E^{-1/2} (W W^T) E^{-1/2} for the NEW state; if
// max |O - I| > 1e-3: O = C C^T, M = E^{1/2} C^{-1} E^{-1/2} (flags[2] = 1).
__device__ __forceinline__ void reorth_check_body(int R, const float* __restrict__ WW, const double* __restrict__ dstate,
                                                  double* __restrict__ Cfac, int* __restrict__ flags) {
  if (flags[1] == 0) return;
  extern __shared__ __align__(16) unsigned char ng_smem[];
  double* sm = reinterpret_cast<double*>(ng_smem);
  double* O = sm;             // R*R
  double* eh = O + R * R;     // R    e^{1/2}
  double* red = eh + R;       // 32
  __shared__ int fail;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) fail = 0;
  for (int i = tid; i < R; i += nt) eh[i] = sqrt(dstate[1 + R + i]);
  __syncthreads();
  double dev = 0.0;
  for (int idx = tid; idx < R * R; idx += nt) {
    const int i = idx / R, j = idx % R;
    const double w = 0.5 * ((double)WW[i * R + j] + (double)WW[j * R + i]);
    const double o = w / (eh[i] * eh[j]);
    O[idx] = o;
    dev = fmax(dev, fabs(o - (i == j ? 1.0 : 0.0)));
  }
  dev = block_max(dev, red);
  if (dev <= 1e-3) { if (tid == 0) flags[2] = 0; return; }
  // Cholesky O = C C^T (lower), right-looking; column k is scaled by every thread from the
  // pivot it reads itself (one barrier per column for the pivot, one for the update)
  for (int k = 0; k < R; ++k) {
    const double okk = O[k * R + k];
    if (!(okk > 0.0)) { fail = 1; break; }   // uniform: every thread reads the same pivot
    const double ckk = sqrt(okk);
    const double inv = 1.0 / ckk;
    const int m = R - k - 1;
    // rank-1 update of the trailing lower triangle with the scaled column
    for (int idx = tid; idx < m * m; idx += nt) {
      const int i = k + 1 + idx / m, j = k + 1 + idx % m;
      if (j <= i) O[i * R + j] -= (O[i * R + k] * inv) * (O[j * R + k] * inv);
    }
    __syncthreads();
    for (int i = k + 1 + tid; i < R; i += nt) O[i * R + k] *= inv;
    if (tid == 0) O[k * R + k] = ckk;
    __syncthreads();
  }
  if (fail) {
    if (tid == 0) { flags[2] = 0; atomicOr(reinterpret_cast<unsigned*>(flags + 3), kErrNotPD); }
    return;
  }
  for (int idx = tid; idx < R * R; idx += nt) {
    const int i = idx / R, j = idx % R;
    Cfac[idx] = (j <= i) ? O[idx] : 0.0;
  }
  if (tid == 0) flags[2] = 1;
}

// B.3.1 repair W' <- M W' with M = E'^{1/2} C^{-1} E'^{-1/2} (reading R5), as an
// FP64 forward substitution per column of W' (no explicit C^{-1}): column j of W' is
// y = C^{-1} (E'^{-1/2} w_j), then w_j <- E'^{1/2} y.  In place, gated on flags[2].
// 128 columns per CTA; the factor and the 128 right-hand sides live in shared memory.
constexpr int kTrsmCols = 128;
__device__ __forceinline__ void reorth_trsm_body(int blk, int R, int D, float* __restrict__ W, int64_t ldw,
                                                 const double* __restrict__ Cfac, const double* __restrict__ dstate,
                                                 const int* __restrict__ flag) {
  if (*flag == 0) return;
  extern __shared__ __align__(16) unsigned char ng_smem[];
  double* C = reinterpret_cast<double*>(ng_smem);    // R*R
  double* eh = C + R * R;                            // R
  double* Y = eh + R;                                // R x kTrsmCols
  const int tid = threadIdx.x;
  for (int i = tid; i < R * R; i += blockDim.x) C[i] = Cfac[i];
  for (int i = tid; i < R; i += blockDim.x) eh[i] = sqrt(dstate[1 + R + i]);
  __syncthreads();
  const int j = blk * kTrsmCols + tid;
  if (j >= D) return;
  for (int i = 0; i < R; ++i) {
    const double* ci = C + i * R;
    double s0 = (double)W[(int64_t)i * ldw + j] / eh[i], s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int k = 0;
    for (; k + 4 <= i; k += 4) {
      s0 -= ci[k] * Y[k * kTrsmCols + tid];
      s1 -= ci[k + 1] * Y[(k + 1) * kTrsmCols + tid];
      s2 -= ci[k + 2] * Y[(k + 2) * kTrsmCols + tid];
      s3 -= ci[k + 3] * Y[(k + 3) * kTrsmCols + tid];
    }
    for (; k < i; ++k) s0 -= ci[k] * Y[k * kTrsmCols + tid];
    Y[i * kTrsmCols + tid] = ((s0 + s1) + (s2 + s3)) / ci[i];
  }
  for (int i = 0; i < R; ++i) W[(int64_t)i * ldw + j] = (float)(eh[i] * Y[i * kTrsmCols + tid]);
}

__global__ void __launch_bounds__(1024)
reorth_check_kernel(int R, const float* __restrict__ WW, const double* __restrict__ dstate,
                    double* __restrict__ Cfac, int* __restrict__ flags) {
  reorth_check_body(R, WW, dstate, Cfac, flags);
}
__global__ void __launch_bounds__(kTrsmCols)
reorth_trsm_kernel(int R, int D, float* __restrict__ W, int64_t ldw, const double* __restrict__ Cfac,
                   const double* __restrict__ dstate, const int* __restrict__ flag) {
  reorth_trsm_body(blockIdx.x, R, D, W, ldw, Cfac, dstate, flag);
}

// Grouped B.3.1 check (one CTA per job) and repair (the jobs' column blocks stacked).
struct ReorthGroup {
  const float* WW[kRefreshGroupMax];
  const double* dstate[kRefreshGroupMax];
  double* Cfac[kRefreshGroupMax];
  int* flags[kRefreshGroupMax];
  float* W[kRefreshGroupMax];
  int64_t ldw[kRefreshGroupMax];
  int R[kRefreshGroupMax], D[kRefreshGroupMax], blk_begin[kRefreshGroupMax + 1];
  int count;
};
__global__ void __launch_bounds__(1024) reorth_check_group_kernel(const __grid_constant__ ReorthGroup g) {
  const int q = blockIdx.x;
  reorth_check_body(g.R[q], g.WW[q], g.dstate[q], g.Cfac[q], g.flags[q]);
}
__global__ void __launch_bounds__(kTrsmCols) reorth_trsm_group_kernel(const __grid_constant__ ReorthGroup g) {
  int q = 0;
  while (q + 1 < g.count && (int)blockIdx.x >= g.blk_begin[q + 1]) ++q;
  reorth_trsm_body((int)blockIdx.x - g.blk_begin[q], g.R[q], g.D[q], g.W[q], g.ldw[q], g.Cfac[q], g.dstate[q],
                   g.flags[q] + 2);
}

// ------------------------------------------------------------------------------------
// initialisation kernels (B.3.2): once per state, host-synchronising
// ------------------------------------------------------------------------------------

__global__ void sumsq_kernel(int n, int D, const float* __restrict__ X, int64_t ldx, double* out) {
  __shared__ double sc[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < (int64_t)n * D; i += blockDim.x) {
    const float x = X[(i / D) * ldx + (i % D)];
    s += (double)x * x;
  }
  s = block_sum(s, sc);
  if (threadIdx.x == 0) *out = s;
}

__global__ void to_double_kernel(int n, int D, const float* __restrict__ X, int64_t ldx, double* __restrict__ Y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)n * D; i += (int64_t)gridDim.x * blockDim.x)
    Y[i] = (double)X[(i / D) * ldx + (i % D)];
}

// Top eigenpairs of the symmetric ne x ne matrix A (global memory): sorted eigenvalues
// -> lam, eigenvector rows -> Vs (ne x ne).
__global__ void __launch_bounds__(1024)
init_eig_kernel(int ne, double* A, double* Vt, double* Vs, double* lam, int* ws_int, double* ws_dbl) {
  __shared__ double red[32];
  const int m = ne / 2 + 1;
  JacobiScratch scr{ws_int, ws_int + m, ws_dbl, ws_dbl + m, ws_dbl + 2 * m, ws_int + 2 * m};
  double amax = 0.0;
  for (int i = threadIdx.x; i < ne; i += blockDim.x) amax = fmax(amax, fabs(A[(int64_t)i * ne + i]));
  amax = block_max(amax, red);
  jacobi_eig(A, ne, Vt, ne, ne, scr, 30, 1e-15 * amax);
  eig_sort_desc(A, ne, Vt, ne, ne, lam, Vs, ne, ws_int + 2 * m + 1);
}

// Top-R eigenpairs of the init matrix (eig_topr.cuh), one CTA: lam (descending) and the
// eigenvector rows X (R x ne).
__global__ void __launch_bounds__(1024) init_topr_kernel(int ne, int R, ToprWork w) { eig_topr(ne, R, w); }

// rho_0, d_0, E_0 and W_0 = E_0^{1/2} R_0.  R0 (R x D,
// double) holds either eigenvector rows of S_0 (gram = 0) or rows X^T v (gram = 1),
// which are normalised here by 1/sqrt(N lambda); numerically-null directions are
// completed to an orthonormal set (their eigenvectors are arbitrary, reading R7).
__global__ void __launch_bounds__(512)
init_finalize_kernel(int R, int D, int N, int n_avail, int gram, double trS, double alpha, double eps,
                     const double* __restrict__ lam, double* __restrict__ R0, float* __restrict__ W,
                     int64_t ldw, double* __restrict__ dstate) {
  __shared__ double red[32];
  __shared__ double lr[kMaxRank];
  const int tid = threadIdx.x, nt = blockDim.x;
  const double lam0 = n_avail > 0 ? fmax(lam[0], 0.0) : 0.0;
  for (int r = tid; r < R; r += nt) lr[r] = (r < n_avail) ? fmax(lam[r], 0.0) : 0.0;
  __syncthreads();
  for (int r = 0; r < R; ++r) {
    const bool valid = (r < n_avail) && (lr[r] > 1e-12 * lam0) && (lr[r] > 0.0);
    double* row = R0 + (int64_t)r * D;
    if (gram && valid) {
      const double sc = 1.0 / sqrt((double)N * lr[r]);
      for (int j = tid; j < D; j += nt) row[j] *= sc;
      __syncthreads();
      continue;
    }
    if (!gram && r < n_avail) continue;   // S_0 eigenvectors are already orthonormal
    // completion: e_j orthogonalised against previous rows (twice), first that survives
    for (int attempt = 0; attempt < D; ++attempt) {
      const int jj = (int)(((int64_t)r * 7919 + attempt * 104729) % D);
      for (int j = tid; j < D; j += nt) row[j] = (j == jj) ? 1.0 : 0.0;
      __syncthreads();
      for (int pass = 0; pass < 2; ++pass) {
        for (int s = 0; s < R; ++s) {
          if (s == r) continue;
          if (s > r) break;
          const double* o = R0 + (int64_t)s * D;
          double dot = 0.0;
          for (int j = tid; j < D; j += nt) dot += o[j] * row[j];
          dot = block_sum(dot, red);
          for (int j = tid; j < D; j += nt) row[j] -= dot * o[j];
          __syncthreads();
        }
      }
      double nn = 0.0;
      for (int j = tid; j < D; j += nt) nn += row[j] * row[j];
      nn = block_sum(nn, red);
      if (nn > 0.25) {
        const double sc = 1.0 / sqrt(nn);
        for (int j = tid; j < D; j += nt) row[j] *= sc;
        __syncthreads();
        break;
      }
      __syncthreads();
    }
  }
  // rho_0 = max((tr S_0 - sum lambda)/(D - R), eps); d_0 = max(eps, lambda - rho_0)
  double sl = 0.0;
  for (int r = tid; r < R; r += nt) sl += lr[r];
  sl = block_sum(sl, red);
  const double rho0 = fmax((trS - sl) / (double)(D - R), eps);
  double sd = 0.0;
  for (int r = tid; r < R; r += nt) sd += fmax(eps, lr[r] - rho0);
  sd = block_sum(sd, red);
  const double beta0 = rho0 * (1.0 + alpha) + (alpha / D) * sd;
  for (int64_t idx = tid; idx < (int64_t)R * D; idx += nt) {
    const int r = (int)(idx / D), j = (int)(idx % D);
    const double d0 = fmax(eps, lr[r] - rho0);
    const double e0 = 1.0 / (beta0 / d0 + 1.0);
    W[(int64_t)r * ldw + j] = (float)(sqrt(e0) * R0[idx]);
  }
  if (tid == 0) dstate[0] = rho0;
  for (int r = tid; r < R; r += nt) {
    const double d0 = fmax(eps, lr[r] - rho0);
    dstate[1 + r] = d0;
    dstate[1 + R + r] = 1.0 / (beta0 / d0 + 1.0);
  }
}

__global__ void passthrough_kernel(int n, float* p, float* p_out, float* g, float* g_out) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) { p[i] = 0.f; if (p_out) p_out[i] = 0.f; }
  if (threadIdx.x == 0) { *g = 1.f; if (g_out) *g_out = 1.f; }
}

// ------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------

static size_t reorth_smem_bytes(int R) { return sizeof(double) * (R * R + R + 32); }
static size_t trsm_smem_bytes(int R) { return sizeof(double) * ((size_t)R * R + R + (size_t)R * kTrsmCols); }

template <typename T>
static ng_status dalloc(T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) { set_error(std::string("cudaMalloc: ") + cudaGetErrorString(e)); return NG_ENOMEM; }
  return NG_OK;
}

static ng_status set_kernel_attrs() {
  static bool done = false;
  if (done) return NG_OK;
  {
    const int tail = tune_int("NG_TUNE_TRI_TAIL", 32 * kTriTailRPL);   // one-warp tail of the tridiagonalisation
    NG_CUDA_TRY(cudaMemcpyToSymbol(g_tri_tail, &tail, sizeof(tail)));
  }
  NG_CUDA_TRY(cudaFuncSetAttribute(refresh_kernel<REFRESH_INPLACE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)refresh_plan(kMaxRank, REFRESH_INPLACE).total_bytes));
  NG_CUDA_TRY(cudaFuncSetAttribute(refresh_kernel<REFRESH_TRI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)refresh_plan(kTriMax, REFRESH_TRI).total_bytes));
  NG_CUDA_TRY(cudaFuncSetAttribute(refresh_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  NG_CUDA_TRY(cudaFuncSetAttribute(reorth_check_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)reorth_smem_bytes(kMaxRank)));
  NG_CUDA_TRY(cudaFuncSetAttribute(reorth_trsm_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)trsm_smem_bytes(kMaxRank)));
  NG_CUDA_TRY(cudaFuncSetAttribute(reorth_check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)reorth_smem_bytes(kMaxRank)));
  NG_CUDA_TRY(cudaFuncSetAttribute(reorth_trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)trsm_smem_bytes(kMaxRank)));
  NG_CUDA_TRY(cudaFuncSetAttribute(apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(sizeof(float) * (kApplyRows * kMaxRank + kMaxRank * kApplyCols))));
  done = true;
  return NG_OK;
}

ng_status ngsgd_create_impl(int dim, int max_rows, const ngsgd_config* cfg, cudaStream_t st, ngsgd_ctx** out) {
  NG_REQUIRE(out != nullptr && cfg != nullptr, NG_EINVAL, "NULL argument");
  NG_REQUIRE(dim >= 1 && max_rows >= 1, NG_ESHAPE, "dim and max_rows must be >= 1");
  NG_REQUIRE(cfg->rank >= 0 && cfg->alpha >= 0.f && cfg->s_samples > 0.f && cfg->update_period >= 1 &&
                 cfg->always_update_first >= 0 && cfg->epsilon > 0.f &&
                 (cfg->precision == NG_FP32 || cfg->precision == NG_TF32 || cfg->precision == NG_FP32_SIMT),
             NG_EINVAL, "invalid ngsgd_config");
  NG_TRY(set_kernel_attrs());
  ngsgd_ctx* h = new ngsgd_ctx();
  h->dim = dim;
  h->cfg = *cfg;
  h->rank = std::max(0, std::min(cfg->rank, dim - 1));     // reading R29
  if (h->rank > kMaxRank) {
    delete h;
    set_error("ngsgd_create: rank > 112 is not supported");
    return NG_EINVAL;
  }
  h->ldw = (int)round_up(dim, 4);
  h->max_rows = max_rows;
  h->st = st;
  const int R = std::max(1, h->rank);
  h->h_splits = std::max(1, std::min(32, ceil_div(dim, 256)));
  h->h_splits = gemm_simt_splits(dim, h->h_splits);
  h->kl_splits = std::max(1, std::min(32, ceil_div(dim, 256)));
  h->kl_splits = gemm_simt_splits(dim, h->kl_splits);
  int l_splits = std::max(h->kl_splits, gemm_simt_splits(max_rows, std::max(1, max_rows / 128)));
  if (cfg->precision != NG_FP32_SIMT) {   // split-K capacities of the tensor-core path
    h->h_splits = std::max(h->h_splits, kTcMaxSplits);
    h->kl_splits = std::max(h->kl_splits, kTcMaxSplits);
    l_splits = std::max(l_splits, kTcMaxSplits);
  }
  h->ctiles = ceil_div(dim, 32);   // partial-norm slots for the narrowest column tiling
  ng_status s = NG_OK;
#define ALLOC(ptr, cnt) if (s == NG_OK) s = dalloc(&(ptr), (size_t)(cnt))
  ALLOC(h->W[0], (size_t)R * h->ldw);
  ALLOC(h->W[1], (size_t)R * h->ldw);
  ALLOC(h->dstate, 1 + 2 * R);
  ALLOC(h->Hpart, std::max((size_t)h->h_splits * max_rows * R, (size_t)kTcJSplits * R * h->ldw));
  ALLOC(h->H, (size_t)max_rows * R);
  ALLOC(h->J, (size_t)R * h->ldw);
  ALLOC(h->Kpart, (size_t)std::max(h->kl_splits, rr_chunks(dim)) * R * R);
  ALLOC(h->Lpart, (size_t)std::max(l_splits, rr_chunks(dim)) * R * R);
  ALLOC(h->KL, 2 * R * R);
  ALLOC(h->WWpart, (size_t)h->kl_splits * R * R);
  ALLOC(h->WW, R * R);
  ALLOC(h->Amat, R * R);
  ALLOC(h->Mmat, R * R);
  ALLOC(h->Cfac, R * R);
  ALLOC(h->trpart, max_rows);
  ALLOC(h->svec, R);
  ALLOC(h->xxpart, (size_t)h->ctiles * max_rows);
  ALLOC(h->ppart, (size_t)h->ctiles * max_rows);
  ALLOC(h->p, max_rows);
  ALLOC(h->sums, 4);   // [0] tr(XX^T) (apply), [1] sum p, [2] tr(XX^T) for the early refresh launch, [3] spare
  ALLOC(h->gamma, 1);
  ALLOC(h->flags, 8);
#undef ALLOC
  if (s == NG_OK && cudaMallocHost((void**)&h->h_scalar, 4 * sizeof(double)) != cudaSuccess) s = NG_ENOMEM;
  if (s == NG_OK && (cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, refresh_priority()) != cudaSuccess ||
                     cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
                     cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess ||
                     cudaEventCreateWithFlags(&h->ev_ab, cudaEventDisableTiming) != cudaSuccess)) {
    set_error("ngsgd_create: stream/event creation failed");
    s = NG_ECUDA;
  }
  if (s == NG_OK) {
    cudaMemsetAsync(h->W[0], 0, sizeof(float) * R * h->ldw, st);
    cudaMemsetAsync(h->W[1], 0, sizeof(float) * R * h->ldw, st);
    cudaMemsetAsync(h->J, 0, sizeof(float) * R * h->ldw, st);
    cudaMemsetAsync(h->flags, 0, sizeof(int) * 8, st);
    cudaMemsetAsync(h->dstate, 0, sizeof(double) * (1 + 2 * R), st);
    if (cudaGetLastError() != cudaSuccess) s = NG_ECUDA;
  }
  if (s != NG_OK) { ngsgd_destroy_impl(h); return s; }
  *out = h;
  return NG_OK;
}

void ngsgd_destroy_impl(ngsgd_ctx* h) {
  if (!h) return;
  float* fp[] = {h->W[0], h->W[1], h->Hpart, h->H, h->J, h->Kpart, h->Lpart, h->KL, h->WWpart, h->WW,
                 h->Amat, h->Mmat, h->svec, h->xxpart, h->ppart, h->p, h->gamma};
  for (float* p : fp) if (p) cudaFree(p);
  if (h->dstate) cudaFree(h->dstate);
  if (h->Cfac) cudaFree(h->Cfac);
  if (h->trpart) cudaFree(h->trpart);
  if (h->sums) cudaFree(h->sums);
  if (h->flags) cudaFree(h->flags);
  if (h->h_scalar) cudaFreeHost(h->h_scalar);
  if (h->side) { cudaStreamSynchronize(h->side); cudaStreamDestroy(h->side); }
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->ev_ab) cudaEventDestroy(h->ev_ab);
  delete h;
}

// One-time initialisation from the first non-zero minibatch (B.3.2).
static ng_status ngsgd_init(ngsgd_ctx* h, int n, const float* x, int64_t ld, double trXX) {
  const int D = h->dim, R = h->rank;
  cudaStream_t st = h->st;
  const bool gram = D > n;                    // N < D: eigenpairs of X X^T / N (Gram trick)
  const int ne = gram ? n : D;
  double *X64 = nullptr, *A = nullptr, *Vt = nullptr, *Vs = nullptr, *lam = nullptr, *R0 = nullptr, *wsd = nullptr;
  int* wsi = nullptr;
  ng_status s = NG_OK;
  s = dalloc(&X64, (size_t)n * D);
  if (s == NG_OK) s = dalloc(&A, (size_t)ne * ne);
  if (s == NG_OK) s = dalloc(&Vt, (size_t)ne * ne);
  if (s == NG_OK) s = dalloc(&Vs, (size_t)ne * ne);
  if (s == NG_OK) s = dalloc(&lam, ne);
  if (s == NG_OK) s = dalloc(&R0, (size_t)std::max(R, 1) * D);
  if (s == NG_OK) s = dalloc(&wsd, 3 * (ne / 2 + 1));
  if (s == NG_OK) s = dalloc(&wsi, 3 * (ne / 2 + 1) + ne + 2);
  if (s == NG_OK) {
    to_double_kernel<<<std::min(1024, ceil_div((int64_t)n * D, 256)), 256, 0, st>>>(n, D, x, ld, X64);
    s = check_launch("to_double_kernel");
  }
  if (s == NG_OK) {
    if (gram)   // A = X X^T / N  (N x N)
      s = gemm_simt<double, true, true>(st, n, n, D, X64, D, X64, D, EpiStore<double>{A, n, 1.0 / n});
    else        // A = S_0 = X^T X / N  (D x D)
      s = gemm_simt<double, false, false>(st, D, D, n, X64, D, X64, D, EpiStore<double>{A, D, 1.0 / n});
  }
  const int n_avail = std::min(ne, R);
  double* topw = nullptr;
  static const int use_jacobi = tune_int("NG_TUNE_INIT_JACOBI", 0);   // the round-1 solver (comparisons)
  const bool topr = !use_jacobi && ne <= kToprMaxN && n_avail <= kToprMaxR && n_avail >= 1;
  if (s == NG_OK && topr) {
    // Householder + multisection + inverse iteration for the top R only (eig_topr.cuh)
    s = dalloc(&topw, (size_t)3 * ne + (size_t)(1 + 3 * n_avail) * ne);
    if (s == NG_OK) {
      ToprWork w;
      w.A = A; w.V = Vt; w.tau = topw; w.d = topw + ne; w.e = topw + 2 * ne; w.X = Vs; w.lam = lam;
      w.scr = topw + 3 * ne;
      init_topr_kernel<<<1, 1024, 0, st>>>(ne, n_avail, w);
      s = check_launch("init_topr_kernel");
    }
  } else if (s == NG_OK) {
    init_eig_kernel<<<1, 1024, 0, st>>>(ne, A, Vt, Vs, lam, wsi, wsd);
    s = check_launch("init_eig_kernel");
  }
  if (s == NG_OK && R > 0) {
    if (gram)   // R0raw = Vs[:R] X  (rows X^T v_r)
      s = gemm_simt<double, true, false>(st, n_avail, D, n, Vs, n, X64, D, EpiStore<double>{R0, D, 1.0});
    else
      NG_CUDA_TRY(cudaMemcpyAsync(R0, Vs, sizeof(double) * (size_t)n_avail * D, cudaMemcpyDeviceToDevice, st));
  }
  if (s == NG_OK) {
    init_finalize_kernel<<<1, 512, 0, st>>>(R, D, n, n_avail, gram ? 1 : 0, trXX / n, h->cfg.alpha,
                                            h->cfg.epsilon, lam, R0, h->W[h->cur], h->ldw, h->dstate);
    s = check_launch("init_finalize_kernel");
  }
  if (s == NG_OK) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { set_error(std::string("ngsgd init: ") + cudaGetErrorString(e)); s = NG_ECUDA; }
  }
  cudaFree(X64); cudaFree(A); cudaFree(Vt); cudaFree(Vs); cudaFree(lam); cudaFree(R0); cudaFree(wsd); cudaFree(wsi);
  if (topw) cudaFree(topw);
  if (s == NG_OK) h->initialized = true;   // t is not reset (reading R7)
  return s;
}

// Make the handle's stream wait for the side-stream refresh of the previous update.
ng_status ngsgd_join_impl(ngsgd_ctx* h) {
  if (h->pending) {
    NG_CUDA_TRY(cudaStreamWaitEvent(h->st, h->ev_join, 0));
    h->pending = false;
  }
  return NG_OK;
}

// The R x R refresh (Z_t, eigendecomposition, rho', D', E', A_t), W_{t+1} = A_t B_t and
// the gated B.3.1 repair.  They only gate this state's NEXT call, so they run on the
// state's side stream, overlapping later work on the main stream (the other states'
// preconditioning, the weight update, the next forward/backward).  J holds J_t, KL holds
// K_t, L_t and sums[0] tr(X X^T) on entry (all written on the main stream before the fork).
// Profiling knob (never set in tests or bench): NG_PROFILE_SKIP_REFRESH=1 skips the side-stream
// refresh chain (the state then keeps W_t), to measure its share of the step.
static bool skip_refresh_knob() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("NG_PROFILE_SKIP_REFRESH"); v = (e && e[0] == '1') ? 1 : 0; }
  return v == 1;
}

static ng_status launch_refresh_chain(ngsgd_ctx* h, int n, double eta, const double* trx) {
  if (skip_refresh_knob()) return NG_OK;
  const int D = h->dim, R = h->rank;
  cudaStream_t st = h->st;
  float* W = h->W[h->cur];
  NG_CUDA_TRY(cudaEventRecord(h->ev_fork, st));
  NG_CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev_fork, 0));
  cudaStream_t ss = h->side;
  {
    // algorithmic work of a dense symmetric eigendecomposition with eigenvectors: ~9 R^3 flop
    ProfScope pe(NG_PROF_NG_EIG, ss, 9.0 * (double)R * R * R, 1.0);   // "bytes" = CTAs (one SM)
    const double a_ = (double)h->cfg.alpha, e_ = (double)h->cfg.epsilon;
    // FP64 eigensolve in both precision modes: with cond(C) > 1e6 (common) an
    // FP32 solve leaves R_{t+1} non-orthonormal beyond 1e-3 and B.3.1 repairs would fire on
    // most updates (measured on the config-3 network).
    static const int dbg = getenv("NG_PROFILE_JACOBI_MASK") ? atoi(getenv("NG_PROFILE_JACOBI_MASK")) : 0;
    // Solver choice: Householder + RRR/twisted eigenvectors (eig_tri.cuh, Jacobi fallback
    // inside) for 2 <= R <= kTriMax, the in-place Jacobi beyond.  NG_TUNE_EIG_MODE = 0
    // forces the Jacobi (comparisons only).
    static const int force = tune_int("NG_TUNE_EIG_MODE", -1);
    int mode = (R >= 2 && R <= kTriMax) ? REFRESH_TRI : REFRESH_INPLACE;
    if (force == REFRESH_INPLACE) mode = force;
    const RefreshSmem plan = refresh_plan(R, mode);
    if (mode == REFRESH_TRI) {
      refresh_kernel<REFRESH_TRI><<<1, kTriThreads, plan.total_bytes, ss>>>(R, D, n, eta, a_, e_, h->KL, h->dstate,
                                                                     trx, h->Amat, h->svec, h->flags, dbg);
    } else {
      refresh_kernel<REFRESH_INPLACE><<<1, 1024, plan.total_bytes, ss>>>(R, D, n, eta, a_, e_, h->KL, h->dstate,
                                                                         trx, h->Amat, h->svec, h->flags, dbg);
    }
    NG_TRY(check_launch("refresh_kernel"));
  }
  ProfScope ps(NG_PROF_NG_REFRESH, ss, 2.0 * (double)R * R * D + 2.0 * R * D, 4.0 * (4.0 * R * D));
  bscale_kernel<<<std::min(1024, ceil_div((int64_t)R * D, 256)), 256, 0, ss>>>(R, D, h->J, W, h->ldw, h->svec);
  NG_TRY(check_launch("bscale_kernel"));
  const int nxt = 1 - h->cur;
  float* Wn = h->W[nxt];
  // W_{t+1} = A_t B_t (eqn:wt1), FP32 in both modes (orthonormality of R_{t+1})
  NG_TRY((gemm_simt<float, true, false>(ss, R, D, R, h->Amat, R, h->J, h->ldw, EpiStore<float>{Wn, h->ldw, 1.f})));
  // B.3.1, gated on the device flag (no host synchronisation)
  const int ks = gemm_simt_splits(D, h->kl_splits);
  NG_TRY((gemm_simt<float, true, true>(ss, R, R, D, Wn, h->ldw, Wn, h->ldw,
                                       EpiStoreSplit<float>{h->WWpart, R, (int64_t)R * R}, ks, h->flags + 1)));
  reduce_splits_kernel<<<ceil_div(R * R, 256), 256, 0, ss>>>(h->WW, h->WWpart, R * R, ks, R * R, h->flags + 1);
  NG_TRY(check_launch("reduce_splits(WW)"));
  reorth_check_kernel<<<1, 1024, reorth_smem_bytes(R), ss>>>(R, h->WW, h->dstate, h->Cfac, h->flags);
  NG_TRY(check_launch("reorth_check_kernel"));
  reorth_trsm_kernel<<<ceil_div(D, kTrsmCols), kTrsmCols, trsm_smem_bytes(R), ss>>>(R, D, Wn, h->ldw, h->Cfac,
                                                                                   h->dstate, h->flags + 2);
  NG_TRY(check_launch("reorth_trsm_kernel"));
  NG_CUDA_TRY(cudaEventRecord(h->ev_join, ss));
  h->pending = true;
  h->cur = nxt;
  return NG_OK;
}

ng_status ngsgd_precondition_impl(ngsgd_ctx* h, int n, float* x, int64_t ld, float* gamma_out,
                                  float* p_out, int update, int* updated_out) {
  NG_REQUIRE(h != nullptr && x != nullptr, NG_EINVAL, "NULL argument");
  NG_REQUIRE(n >= 1 && n <= h->max_rows, NG_ESHAPE, "n must be in [1, max_rows]");
  NG_REQUIRE(ld >= h->dim, NG_ESHAPE, "ld < dim");
  const int D = h->dim, R = h->rank;
  cudaStream_t st = h->st;
  NG_TRY(ngsgd_join_impl(h));
  if (updated_out) *updated_out = 0;
  h->last_updated = 0;
  if (!h->initialized) {
    // Reading R7: defer initialisation to the first minibatch with tr(X^T X) > 0.
    sumsq_kernel<<<1, 1024, 0, st>>>(n, D, x, ld, h->sums);
    NG_TRY(check_launch("sumsq_kernel"));
    NG_CUDA_TRY(cudaMemcpyAsync(h->h_scalar, h->sums, sizeof(double), cudaMemcpyDeviceToHost, st));
    NG_CUDA_TRY(cudaStreamSynchronize(st));
    const double trXX = h->h_scalar[0];
    NG_REQUIRE(std::isfinite(trXX), NG_ENONFINITE, "non-finite input");
    if (trXX == 0.0) {
      // t still counts the minibatch: the update schedule is per minibatch
      h->t += 1;
      passthrough_kernel<<<1, 256, 0, st>>>(n, h->p, p_out, h->gamma, gamma_out);
      return check_launch("passthrough_kernel");
    }
    {
      ProfScope ps(NG_PROF_NG_INIT, st, 0.0, 0.0);
      NG_TRY(ngsgd_init(h, n, x, ld, trXX));
    }
  }
  const bool upd = (update < 0)
                       ? (h->t < h->cfg.always_update_first || (h->t % h->cfg.update_period) == 0)
                       : (update != 0);
  if (R == 0) {
    rownorm_part_kernel<<<n, 256, 0, st>>>(n, D, x, ld, h->xxpart, h->ppart);
    NG_TRY(check_launch("rownorm_part_kernel"));
    finalize_kernel<<<1, 512, 0, st>>>(n, 1, h->xxpart, h->ppart, h->max_rows, h->p, p_out, h->sums,
                                       h->gamma, gamma_out, h->flags);
    NG_TRY(check_launch("finalize_kernel"));
    h->t += 1;
    h->last_updated = upd;
    if (updated_out) *updated_out = upd;
    return NG_OK;
  }
  const double eta = 1.0 - exp(-(double)n / (double)h->cfg.s_samples);   // eqn:eta:ns
  float* W = h->W[h->cur];
  const double nRD = (double)n * R * D;
  // Tensor-core (TF32) projections when requested and the operands satisfy TMA alignment.
  const bool tc = h->cfg.precision != NG_FP32_SIMT && (ld % 4) == 0 && (R % 4) == 0 &&
                  (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  const int bnR = R <= 32 ? 32 : (R <= 64 ? 64 : 128);
  const int m_tiles = ceil_div(n, 128);
  // H = X W^T (eqn:ht), split over D, fixed-order reduction
  {
    ProfScope ps(NG_PROF_NG_PROJ, st, 2.0 * nRD, 4.0 * ((double)n * D + (double)R * D));
    int hs = 1;
    if (tc) {
      TcEpilogue e;
      e.kind = TC_EPI_PARTIAL; e.C = h->Hpart; e.ldc = R; e.zstride = (int64_t)n * R;
      const int want = std::min(kTcMaxSplits, std::max(1, 148 / (m_tiles * ceil_div(R, bnR))));
      NG_TRY(tc_gemm_tf32(st, n, R, D, x, ld, true, W, h->ldw, true, e, bnR, want, &hs, true));
    } else {
      NG_TRY((gemm_simt<float, true, true>(st, n, R, D, x, ld, W, h->ldw,
                                           EpiStoreSplit<float>{h->Hpart, R, (int64_t)n * R}, h->h_splits)));
      hs = gemm_simt_splits(D, h->h_splits);
    }
    reduce_splits_kernel<<<ceil_div((int64_t)n * R, 256), 256, 0, st>>>(h->H, h->Hpart, (int64_t)n * R, hs,
                                                                       (int64_t)n * R, nullptr);
    NG_TRY(check_launch("reduce_splits(H)"));
  }
  if (upd) {
    ProfScope ps(NG_PROF_NG_REFRESH, st, 2.0 * nRD + 4.0 * (double)R * R * D,
                 4.0 * ((double)n * D + 3.0 * R * D));
    if (tc) {
      // J = H^T X: A = H (MN-major), B = X (MN-major), split over N
      TcEpilogue e;
      e.kind = TC_EPI_PARTIAL; e.C = h->Hpart; e.ldc = h->ldw; e.zstride = (int64_t)R * h->ldw;
      int js = 1;
      NG_TRY(tc_gemm_tf32(st, R, D, n, h->H, R, false, x, ld, false, e, 128, kTcJSplits, &js, true));
      reduce_rows_kernel<<<std::min(1024, ceil_div((int64_t)R * D, 256)), 256, 0, st>>>(
          h->J, h->ldw, h->Hpart, (int64_t)R * h->ldw, js, R, D);
      NG_TRY(check_launch("reduce_rows(J)"));
      // K = J J^T and L = W J^T in 3xTF32 (FP32-grade): Z_t must equal Y_t Y_t^T for the
      // STORED J to FP32 accuracy, otherwise R_{t+1} = C^{-1/2} U^T Y_t loses orthonormality
      // at the TF32 level (1e-3) and B.3.1 repairs fire.  L = W J^T is used for every N
      // (it equals H^T H only when J = H^T X exactly).
      const int want = std::max(1, std::min(kTcMaxSplits, 64));
      int ks = 1, ls = 1;
      TcEpilogue ek;
      ek.kind = TC_EPI_PARTIAL; ek.C = h->Kpart; ek.ldc = R; ek.zstride = (int64_t)R * R;
      NG_TRY(tc_gemm_tf32(st, R, R, D, h->J, h->ldw, true, h->J, h->ldw, true, ek, 128, want, &ks, true));
      reduce_splits_kernel<<<ceil_div(R * R, 256), 256, 0, st>>>(h->KL, h->Kpart, R * R, ks, R * R, nullptr);
      NG_TRY(check_launch("reduce_splits(K)"));
      TcEpilogue el = ek;
      el.C = h->Lpart;
      NG_TRY(tc_gemm_tf32(st, R, R, D, W, h->ldw, true, h->J, h->ldw, true, el, 128, want, &ls, true));
      reduce_splits_kernel<<<ceil_div(R * R, 256), 256, 0, st>>>(h->KL + R * R, h->Lpart, R * R, ls, R * R, nullptr);
      NG_TRY(check_launch("reduce_splits(L)"));
    } else {
      // J = H^T X -- before X is overwritten
      NG_TRY((gemm_simt<float, false, false>(st, R, D, n, h->H, R, x, ld, EpiStore<float>{h->J, h->ldw, 1.f})));
      // K = J J^T
      const int ks = gemm_simt_splits(D, h->kl_splits);
      NG_TRY((gemm_simt<float, true, true>(st, R, R, D, h->J, h->ldw, h->J, h->ldw,
                                           EpiStoreSplit<float>{h->Kpart, R, (int64_t)R * R}, ks)));
      reduce_splits_kernel<<<ceil_div(R * R, 256), 256, 0, st>>>(h->KL, h->Kpart, R * R, ks, R * R, nullptr);
      NG_TRY(check_launch("reduce_splits(K)"));
      if (n > D) {   // L = W J^T
        NG_TRY((gemm_simt<float, true, true>(st, R, R, D, W, h->ldw, h->J, h->ldw,
                                             EpiStoreSplit<float>{h->Lpart, R, (int64_t)R * R}, ks)));
        reduce_splits_kernel<<<ceil_div(R * R, 256), 256, 0, st>>>(h->KL + R * R, h->Lpart, R * R, ks, R * R, nullptr);
      } else {       // L = H^T H
        const int ls = gemm_simt_splits(n, std::max(1, n / 128));
        NG_TRY((gemm_simt<float, false, false>(st, R, R, n, h->H, R, h->H, R,
                                               EpiStoreSplit<float>{h->Lpart, R, (int64_t)R * R}, ls)));
        reduce_splits_kernel<<<ceil_div(R * R, 256), 256, 0, st>>>(h->KL + R * R, h->Lpart, R * R, ls, R * R, nullptr);
      }
      NG_TRY(check_launch("reduce_splits(L)"));
    }
  }
  // X_hat = X - H W in place, with partial row norms
  {
    ProfScope ps(NG_PROF_NG_APPLY, st, 2.0 * nRD, 4.0 * (2.0 * n * D + (double)R * D));
    int tiles = ceil_div(D, kApplyCols);
    if (tc) {
      TcEpilogue e;
      e.kind = TC_EPI_NGAPPLY; e.C = x; e.ldc = ld; e.xx = h->xxpart; e.pp = h->ppart; e.part_ld = h->max_rows;
      NG_TRY(tc_gemm_tf32(st, n, D, R, h->H, R, true, W, h->ldw, false, e, apply_bn(), 1, nullptr, true));
      tiles = ceil_div(D, apply_bn());
    } else {
      dim3 grid(ceil_div(n, kApplyRows), ceil_div(D, kApplyCols));
      const size_t smem = sizeof(float) * (kApplyRows * R + R * kApplyCols);
      apply_kernel<<<grid, 256, smem, st>>>(n, D, R, x, ld, h->H, W, h->ldw, h->xxpart, h->ppart, h->max_rows);
      NG_TRY(check_launch("apply_kernel"));
    }
    finalize_kernel<<<1, 512, 0, st>>>(n, tiles, h->xxpart, h->ppart, h->max_rows, h->p, p_out, h->sums,
                                       h->gamma, gamma_out, h->flags);
    NG_TRY(check_launch("finalize_kernel"));
  }
  if (upd) NG_TRY(launch_refresh_chain(h, n, eta, h->sums));
  h->t += 1;
  h->last_updated = upd ? 1 : 0;
  if (updated_out) *updated_out = upd ? 1 : 0;
  return NG_OK;
}

// ------------------------------------------------------------------------------------
// grouped (multi-state) preconditioning: one launch per phase
// ------------------------------------------------------------------------------------

constexpr int kSegMax = 16;
struct SegReduce {            // out[i*ldo + j] = sum_z src[z*zstride + i*lds + j], i < rows, j < cols
  float* out[kSegMax];
  const float* src[kSegMax];
  int64_t ldo[kSegMax], lds[kSegMax], zstride[kSegMax];
  int rows[kSegMax], cols[kSegMax], splits[kSegMax], block_begin[kSegMax + 1];
  int count;
};

__global__ void __launch_bounds__(256) seg_reduce_kernel(const __grid_constant__ SegReduce sr) {
  pdl_trigger();
  pdl_wait();   // launched with launch_pdl
  int g = 0;
  while (g + 1 < sr.count && (int)blockIdx.x >= sr.block_begin[g + 1]) ++g;
  const int64_t total = (int64_t)sr.rows[g] * sr.cols[g];
  const int cols = sr.cols[g], sp = sr.splits[g];
  for (int64_t i = (int64_t)(blockIdx.x - sr.block_begin[g]) * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)(sr.block_begin[g + 1] - sr.block_begin[g]) * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    const float* src = sr.src[g] + r * sr.lds[g] + c;
    float a4[4] = {0.f, 0.f, 0.f, 0.f};   // independent loads in flight, fixed combination order
    int z = 0;
    for (; z + 4 <= sp; z += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) a4[u] += src[(int64_t)(z + u) * sr.zstride[g]];
    }
    for (; z < sp; ++z) a4[0] += src[(int64_t)z * sr.zstride[g]];
    sr.out[g][r * sr.ldo[g] + c] = (a4[0] + a4[1]) + (a4[2] + a4[3]);
  }
}

// tr(X X^T) of every updating state, computed before the apply so the refresh chains can
// be launched right after K_t, L_t (phase B): sums[2] = sum_i ||x_i||^2 in FP64; one CTA
// per row (row sums), then a fixed-order sum over the rows.
struct TraceGroup {
  const float* x[kSegMax];
  int64_t ld[kSegMax];
  int n[kSegMax], D[kSegMax];
  double* out[kSegMax];
  double* part[kSegMax];   // n row sums each
  int count;
};
__global__ void __launch_bounds__(128) trace_part_kernel(const __grid_constant__ TraceGroup tg) {
  __shared__ double sc[32];
  const int g = blockIdx.y, r = blockIdx.x;
  if (r >= tg.n[g]) return;
  const int D = tg.D[g];
  const float* xr = tg.x[g] + (int64_t)r * tg.ld[g];
  double acc = 0.0;
  if ((reinterpret_cast<uintptr_t>(xr) & 15) == 0) {
    const int d4 = D >> 2;
    for (int j = threadIdx.x; j < d4; j += blockDim.x) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(xr) + j);
      acc += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
    }
    for (int j = (d4 << 2) + threadIdx.x; j < D; j += blockDim.x) { const double v = xr[j]; acc += v * v; }
  } else {
    for (int j = threadIdx.x; j < D; j += blockDim.x) { const double v = xr[j]; acc += v * v; }
  }
  acc = block_sum(acc, sc);
  if (threadIdx.x == 0) tg.part[g][r] = acc;
}
__global__ void __launch_bounds__(256) trace_final_kernel(const __grid_constant__ TraceGroup tg) {
  __shared__ double sc[32];
  const int g = blockIdx.x;
  double acc = 0.0;
  for (int r = threadIdx.x; r < tg.n[g]; r += blockDim.x) acc += tg.part[g][r];
  acc = block_sum(acc, sc);
  if (threadIdx.x == 0) *tg.out[g] = acc;
}

struct FinalizeGroup {
  int n[kSegMax], tiles[kSegMax];
  const float* xxpart[kSegMax];
  const float* ppart[kSegMax];
  int64_t part_ld[kSegMax];
  float* p_int[kSegMax];
  float* p_out[kSegMax];
  double* sums[kSegMax];
  float* gamma_int[kSegMax];
  float* gamma_out[kSegMax];
  int* flags[kSegMax];
  int count;
};

// One CTA per state: identical arithmetic to finalize_kernel.
__global__ void __launch_bounds__(512) finalize_group_kernel(const __grid_constant__ FinalizeGroup fg) {
  pdl_trigger();
  pdl_wait();   // launched with launch_pdl
  const int g = blockIdx.x;
  __shared__ double sc[32];
  const int n = fg.n[g], tiles = fg.tiles[g];
  const int64_t pl = fg.part_ld[g];
  double sxx = 0.0, spp = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    // four interleaved partial sums (independent loads in flight), combined in a fixed
    // order; ||x||^2 and ||x_hat||^2 use the identical tree (R = 0 gives gamma = 1 exactly, R27)
    float xa[4] = {0.f, 0.f, 0.f, 0.f}, pa[4] = {0.f, 0.f, 0.f, 0.f};
    int t = 0;
    for (; t + 4 <= tiles; t += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        xa[u] += fg.xxpart[g][(int64_t)(t + u) * pl + i];
        pa[u] += fg.ppart[g][(int64_t)(t + u) * pl + i];
      }
    }
    for (; t < tiles; ++t) { xa[0] += fg.xxpart[g][(int64_t)t * pl + i]; pa[0] += fg.ppart[g][(int64_t)t * pl + i]; }
    const float xx = (xa[0] + xa[1]) + (xa[2] + xa[3]), pp = (pa[0] + pa[1]) + (pa[2] + pa[3]);
    fg.p_int[g][i] = pp;
    if (fg.p_out[g]) fg.p_out[g][i] = pp;
    sxx += (double)xx;
    spp += (double)pp;
  }
  sxx = block_sum(sxx, sc);
  spp = block_sum(spp, sc);
  if (threadIdx.x == 0) {
    fg.sums[g][0] = sxx;
    fg.sums[g][1] = spp;
    const float gm = (spp > 0.0) ? (float)sqrt(sxx / spp) : 1.0f;
    *fg.gamma_int[g] = gm;
    if (fg.gamma_out[g]) *fg.gamma_out[g] = gm;
    if (!isfinite(sxx) || !isfinite(spp)) atomicOr(reinterpret_cast<unsigned*>(fg.flags[g] + 3), kErrNonFinite);
  }
}

static ng_status launch_seg_reduce(cudaStream_t st, SegReduce& sr) {
  int blocks = 0;
  for (int g = 0; g < sr.count; ++g) {
    sr.block_begin[g] = blocks;
    blocks += std::max(1, std::min(64, ceil_div((int64_t)sr.rows[g] * sr.cols[g], 256)));
  }
  sr.block_begin[sr.count] = blocks;
  NG_CUDA_TRY(launch_pdl(seg_reduce_kernel, dim3(blocks), dim3(256), 0, st, sr));
  return check_launch("seg_reduce_kernel");
}

int rr_chunks(int D) { return ceil_div(D, 64); }   // split capacity of the K / L partial buffers

// The refresh chains of every updating state of a group as ONE chain of grouped launches on
// ONE side stream (the first state's): the R x R refresh (one CTA per state), B_t, W_{t+1} =
// A_t B_t and W_{t+1} W_{t+1}^T (3xTF32 tensor cores), the B.3.1 check and repair.  Every
// state's join event is recorded at its end; the main stream waits for it before that
// state's next call (the refresh only gates the next call).  Falls back to the
// per-state chains for ranks the one-CTA Householder/RRR solver does not take.
static ng_status launch_refresh_group(NgCall* calls, const std::vector<int>& grp, const std::vector<int>& ug,
                                      cudaStream_t st) {
  if (skip_refresh_knob() || ug.empty()) return NG_OK;
  static const int force = tune_int("NG_TUNE_EIG_MODE", -1);
  bool ok = force < 0 && (int)ug.size() <= kRefreshGroupMax;
  int maxR = 0;
  for (int g : ug) {
    const int R = calls[grp[g]].h->rank;
    ok = ok && R >= 2 && R <= kTriMax;
    maxR = std::max(maxR, R);
  }
  if (!ok) {
    for (int g : ug) {
      NgCall& c = calls[grp[g]];
      const double eta = 1.0 - exp(-(double)c.n / (double)c.h->cfg.s_samples);   // eqn:eta:ns
      NG_TRY(launch_refresh_chain(c.h, c.n, eta, c.h->sums + 2));
    }
    return NG_OK;
  }
  const int G = (int)ug.size();
  ngsgd_ctx* h0 = calls[grp[ug[0]]].h;
  cudaStream_t ss = h0->side;
  NG_CUDA_TRY(cudaEventRecord(h0->ev_fork, st));
  NG_CUDA_TRY(cudaStreamWaitEvent(ss, h0->ev_fork, 0));
  static const int dbg = getenv("NG_PROFILE_JACOBI_MASK") ? atoi(getenv("NG_PROFILE_JACOBI_MASK")) : 0;
  {
    RefreshGroup rg;
    std::memset(&rg, 0, sizeof(rg));
    rg.count = G;
    rg.dbg = dbg;
    double flops = 0.0;
    for (int u = 0; u < G; ++u) {
      NgCall& c = calls[grp[ug[u]]];
      ngsgd_ctx* h = c.h;
      RefreshJob& J = rg.j[u];
      J.R = h->rank; J.D = h->dim; J.N = c.n;
      J.eta = 1.0 - exp(-(double)c.n / (double)h->cfg.s_samples);   // eqn:eta:ns
      J.alpha = h->cfg.alpha; J.eps = h->cfg.epsilon;
      J.KL = h->KL; J.dstate = h->dstate; J.sums = h->sums + 2; J.Amat = h->Amat; J.svec = h->svec; J.flags = h->flags;
      flops += 9.0 * (double)J.R * J.R * J.R;
    }
    // ng_eig: algorithmic work ~9 R^3 per state; "bytes" carries the CTA (state) count so the
    // roofline is taken against that many SMs' FP64 rate
    ProfScope pe(NG_PROF_NG_EIG, ss, flops, (double)G);
    // NG_TUNE_REFRESH_SMEM_KB pads the refresh CTA's shared memory so that no main-stream
    // CTA can share its SM (measurement knob)
    static const size_t pad = (size_t)std::min(200, std::max(0, tune_int("NG_TUNE_REFRESH_SMEM_KB", 0))) * 1024;
    const size_t rsm = std::max(refresh_plan(maxR, REFRESH_TRI).total_bytes, pad);
    refresh_group_kernel<<<G, kTriThreads, rsm, ss>>>(rg);
    NG_TRY(check_launch("refresh_group_kernel"));
  }
  double flops = 0.0, bytes = 0.0;
  for (int g : ug) {
    const ngsgd_ctx* h = calls[grp[g]].h;
    flops += 4.0 * (double)h->rank * h->rank * h->dim;
    bytes += 4.0 * 4.0 * h->rank * h->dim;
  }
  ProfScope ps(NG_PROF_NG_REFRESH, ss, flops, bytes);
  {
    BscaleGroup bg;
    std::memset(&bg, 0, sizeof(bg));
    int64_t mx = 1;
    for (int u = 0; u < G; ++u) {
      ngsgd_ctx* h = calls[grp[ug[u]]].h;
      bg.J[u] = h->J; bg.W[u] = h->W[h->cur]; bg.s[u] = h->svec; bg.ldw[u] = h->ldw; bg.R[u] = h->rank;
      bg.D[u] = h->dim;
      mx = std::max<int64_t>(mx, (int64_t)h->rank * h->dim);
    }
    bscale_group_kernel<<<dim3(std::min(64, ceil_div(mx, 256)), G), 256, 0, ss>>>(bg);
    NG_TRY(check_launch("bscale_group_kernel"));
  }
  // W_{t+1} = A_t B_t (eqn:wt1): M = R, N = D, K = R; A_t K-major, B_t = J MN-major
  std::vector<TcGroupDesc> dw(G), dww(G);
  std::vector<int> spw(G);
  const int want = std::max(1, std::min(kTcMaxSplits, ceil_div(2 * 148, G)));
  for (int u = 0; u < G; ++u) {
    ngsgd_ctx* h = calls[grp[ug[u]]].h;
    const int R = h->rank, D = h->dim;
    float* Wn = h->W[1 - h->cur];
    TcGroupDesc& q = dw[u];
    std::memset(&q, 0, sizeof(q));
    q.M = R; q.N = D; q.K = R; q.splits = 1;
    q.A = h->Amat; q.lda = R; q.B = h->J; q.ldb = h->ldw;
    q.epi.kind = TC_EPI_STORE; q.epi.C = Wn; q.epi.ldc = h->ldw;
    TcGroupDesc& w = dww[u];
    std::memset(&w, 0, sizeof(w));
    w.M = R; w.N = R; w.K = D; w.splits = want;
    w.A = Wn; w.lda = h->ldw; w.B = Wn; w.ldb = h->ldw;
    w.epi.kind = TC_EPI_PARTIAL; w.epi.C = h->WWpart; w.epi.ldc = R; w.epi.zstride = (int64_t)R * R;
    w.splits_used = &spw[u];
  }
  NG_TRY(tc_gemm_tf32_grouped(ss, dw.data(), G, true, false, TC_EPI_STORE, 128, true));
  // B.3.1: W_{t+1} W_{t+1}^T (split over D, fixed-order reduction), check, repair
  NG_TRY(tc_gemm_tf32_grouped(ss, dww.data(), G, true, true, TC_EPI_PARTIAL, 128, true));
  {
    SegReduce sr;
    std::memset(&sr, 0, sizeof(sr));
    sr.count = G;
    for (int u = 0; u < G; ++u) {
      ngsgd_ctx* h = calls[grp[ug[u]]].h;
      const int R = h->rank;
      sr.out[u] = h->WW; sr.src[u] = h->WWpart; sr.ldo[u] = R; sr.lds[u] = R; sr.zstride[u] = (int64_t)R * R;
      sr.rows[u] = R; sr.cols[u] = R; sr.splits[u] = spw[u];
    }
    NG_TRY(launch_seg_reduce(ss, sr));
  }
  {
    ReorthGroup rg;
    std::memset(&rg, 0, sizeof(rg));
    rg.count = G;
    int blocks = 0;
    for (int u = 0; u < G; ++u) {
      ngsgd_ctx* h = calls[grp[ug[u]]].h;
      rg.WW[u] = h->WW; rg.dstate[u] = h->dstate; rg.Cfac[u] = h->Cfac; rg.flags[u] = h->flags;
      rg.W[u] = h->W[1 - h->cur]; rg.ldw[u] = h->ldw; rg.R[u] = h->rank; rg.D[u] = h->dim;
      rg.blk_begin[u] = blocks;
      blocks += ceil_div(h->dim, kTrsmCols);
    }
    rg.blk_begin[G] = blocks;
    reorth_check_group_kernel<<<G, 1024, reorth_smem_bytes(maxR), ss>>>(rg);
    NG_TRY(check_launch("reorth_check_group_kernel"));
    reorth_trsm_group_kernel<<<blocks, kTrsmCols, trsm_smem_bytes(maxR), ss>>>(rg);
    NG_TRY(check_launch("reorth_trsm_group_kernel"));
  }
  for (int g : ug) {
    ngsgd_ctx* h = calls[grp[g]].h;
    NG_CUDA_TRY(cudaEventRecord(h->ev_join, ss));
    h->pending = true;
    h->cur = 1 - h->cur;
  }
  return NG_OK;
}

ng_status ngsgd_precondition_group_impl(NgCall* calls, int count) {
  NG_REQUIRE(calls != nullptr && count >= 0, NG_EINVAL, "NULL argument");
  std::vector<int> grp;          // indices of tensor-core group members
  std::vector<char> upd(count, 0);
  cudaStream_t st = nullptr;
  for (int i = 0; i < count; ++i) {
    NgCall& c = calls[i];
    ngsgd_ctx* h = c.h;
    NG_REQUIRE(h != nullptr && c.x != nullptr, NG_EINVAL, "NULL argument");
    const bool eligible = h->initialized && h->rank > 0 && h->rank <= 128 && h->cfg.precision != NG_FP32_SIMT &&
                          (c.ld % 4) == 0 && (h->rank % 4) == 0 && (reinterpret_cast<uintptr_t>(c.x) & 15) == 0 &&
                          c.n >= 1 && c.n <= h->max_rows && c.ld >= h->dim && (int)grp.size() < kTcGroupMax &&
                          (grp.empty() || h->st == st);
    if (!eligible) {           // initialisation, FP32, odd shapes: the single-state path
      NG_TRY(ngsgd_precondition_impl(h, c.n, c.x, c.ld, c.gamma_out, c.p_out, c.update, c.updated_out));
      continue;
    }
    st = h->st;
    NG_TRY(ngsgd_join_impl(h));
    h->last_updated = 0;
    upd[i] = (c.update < 0) ? (h->t < h->cfg.always_update_first || (h->t % h->cfg.update_period) == 0)
                            : (c.update != 0);
    grp.push_back(i);
  }
  if (grp.empty()) return NG_OK;
  const int G = (int)grp.size();
  // phase C keeps using the pre-refresh W_t of every state
  std::vector<float*> Wold(G);
  for (int g = 0; g < G; ++g) Wold[g] = calls[grp[g]].h->W[calls[grp[g]].h->cur];
  // Phases A (H), B (J, K, L of the updating states), tr(X X^T) and the refresh launch for
  // the states `sub` (call indices) on stream sx; ev_ab (optional) is recorded on sx once H,
  // J and the trace are done, before the refresh chain is launched.
  auto phases_ab = [&](const std::vector<int>& sub, cudaStream_t sx, cudaEvent_t ev_ab) -> ng_status {
  const int S = (int)sub.size();
  if (S == 0) return NG_OK;
  // ---- phase A: H = X W^T for every state (split-K partials), one launch
  {
    double flops = 0, bytes = 0;
    int64_t total_kt = 0;
    for (int i : sub) total_kt += (int64_t)ceil_div(calls[i].n, 128) * ceil_div(calls[i].h->dim, 32);
    const int64_t target_kb = std::max<int64_t>(4, ceil_div(total_kt, 2 * 148));
    std::vector<TcGroupDesc> d(S);
    std::vector<int> sp(S);
    for (int g = 0; g < S; ++g) {
      NgCall& c = calls[sub[g]];
      ngsgd_ctx* h = c.h;
      const int R = h->rank, D = h->dim;
      flops += 2.0 * c.n * R * D;
      bytes += 4.0 * ((double)c.n * D + (double)R * D);
      TcGroupDesc& q = d[g];
      q.M = c.n; q.N = R; q.K = D;
      q.splits = (int)std::min<int64_t>(kTcMaxSplits, std::max<int64_t>(1, ceil_div(ceil_div(D, 32), target_kb)));
      q.A = c.x; q.lda = c.ld; q.B = h->W[h->cur]; q.ldb = h->ldw;
      q.epi.kind = TC_EPI_PARTIAL; q.epi.C = h->Hpart; q.epi.ldc = R; q.epi.zstride = (int64_t)c.n * R;
      q.splits_used = &sp[g];
    }
    ProfScope ps(NG_PROF_NG_PROJ, sx, flops, bytes);
    NG_TRY(tc_gemm_tf32_grouped(sx, d.data(), S, true, true, TC_EPI_PARTIAL, 128, true));
    SegReduce sr;
    std::memset(&sr, 0, sizeof(sr));
    sr.count = S;
    for (int g = 0; g < S; ++g) {
      NgCall& c = calls[sub[g]];
      const int R = c.h->rank;
      sr.out[g] = c.h->H; sr.src[g] = c.h->Hpart; sr.ldo[g] = R; sr.lds[g] = R;
      sr.zstride[g] = (int64_t)c.n * R; sr.rows[g] = c.n; sr.cols[g] = R; sr.splits[g] = sp[g];
    }
    NG_TRY(launch_seg_reduce(sx, sr));
  }
  // ---- phase B (update states): J = H^T X (one launch), K = J J^T, L = W J^T (FP32)
  std::vector<int> ug;
  for (int g = 0; g < S; ++g) if (upd[sub[g]]) ug.push_back(g);
  if (!ug.empty()) {
    double flops = 0, bytes = 0;
    std::vector<TcGroupDesc> d(ug.size());
    std::vector<int> sp(ug.size());
    for (size_t u = 0; u < ug.size(); ++u) {
      NgCall& c = calls[sub[ug[u]]];
      ngsgd_ctx* h = c.h;
      const int R = h->rank, D = h->dim;
      flops += 2.0 * c.n * R * D + 4.0 * (double)R * R * D;
      bytes += 4.0 * ((double)c.n * D + 3.0 * R * D);
      TcGroupDesc& q = d[u];
      q.M = R; q.N = D; q.K = c.n; q.splits = kTcJSplits;
      q.A = h->H; q.lda = R; q.B = c.x; q.ldb = c.ld;
      q.epi.kind = TC_EPI_PARTIAL; q.epi.C = h->Hpart; q.epi.ldc = h->ldw; q.epi.zstride = (int64_t)R * h->ldw;
      q.splits_used = &sp[u];
    }
    ProfScope ps(NG_PROF_NG_REFRESH, sx, flops, bytes);
    NG_TRY(tc_gemm_tf32_grouped(sx, d.data(), (int)ug.size(), false, false, TC_EPI_PARTIAL, 128, true));
    SegReduce sr;
    std::memset(&sr, 0, sizeof(sr));
    sr.count = (int)ug.size();
    for (size_t u = 0; u < ug.size(); ++u) {
      ngsgd_ctx* h = calls[sub[ug[u]]].h;
      sr.out[u] = h->J; sr.src[u] = h->Hpart; sr.ldo[u] = h->ldw; sr.lds[u] = h->ldw;
      sr.zstride[u] = (int64_t)h->rank * h->ldw; sr.rows[u] = h->rank; sr.cols[u] = h->dim; sr.splits[u] = sp[u];
    }
    NG_TRY(launch_seg_reduce(sx, sr));
    // K = J J^T and L = W J^T of every updating state: one grouped 3xTF32
    // tensor-core launch per 16 problems (FP32-grade: Z_t must equal Y_t Y_t^T for the
    // stored J to FP32 accuracy), split over D, then the fixed-order segmented reduction
    {
      std::vector<TcGroupDesc> d;
      std::vector<int> spk(2 * ug.size());
      const int nprob = 2 * (int)ug.size();
      const int want = std::max(1, std::min(kTcMaxSplits, ceil_div(2 * 148, nprob)));
      for (size_t u = 0; u < ug.size(); ++u) {
        ngsgd_ctx* h = calls[sub[ug[u]]].h;
        const int R = h->rank, D = h->dim;
        for (int w = 0; w < 2; ++w) {
          TcGroupDesc q;
          std::memset(&q, 0, sizeof(q));
          q.M = R; q.N = R; q.K = D; q.splits = want;
          q.A = w ? h->W[h->cur] : h->J; q.lda = h->ldw;
          q.B = h->J; q.ldb = h->ldw;
          q.epi.kind = TC_EPI_PARTIAL; q.epi.C = w ? h->Lpart : h->Kpart; q.epi.ldc = R;
          q.epi.zstride = (int64_t)R * R;
          q.splits_used = &spk[2 * u + w];
          d.push_back(q);
        }
      }
      for (size_t b = 0; b < d.size(); b += kTcGroupMax) {
        const int cnt = (int)std::min<size_t>(kTcGroupMax, d.size() - b);
        NG_TRY(tc_gemm_tf32_grouped(sx, d.data() + b, cnt, true, true, TC_EPI_PARTIAL, 128, true));
      }
      SegReduce kl;
      std::memset(&kl, 0, sizeof(kl));
      kl.count = 0;
      for (size_t u = 0; u < ug.size(); ++u) {
        ngsgd_ctx* h = calls[sub[ug[u]]].h;
        const int R = h->rank;
        for (int w = 0; w < 2; ++w) {
          if (kl.count == kSegMax) { NG_TRY(launch_seg_reduce(sx, kl)); kl.count = 0; }
          const int k = kl.count++;
          kl.out[k] = h->KL + w * R * R; kl.src[k] = w ? h->Lpart : h->Kpart; kl.ldo[k] = R; kl.lds[k] = R;
          kl.zstride[k] = (int64_t)R * R; kl.rows[k] = R; kl.cols[k] = R; kl.splits[k] = spk[2 * u + w];
        }
      }
      if (kl.count) NG_TRY(launch_seg_reduce(sx, kl));
    }
  }
  // ---- tr(X X^T) of the updating states, then their refresh chains start right away (they
  // need J, K, L and the trace only); phase C keeps using the pre-refresh W_t
  if (!ug.empty()) {
    TraceGroup tr;
    std::memset(&tr, 0, sizeof(tr));
    tr.count = (int)ug.size();
    for (size_t u = 0; u < ug.size(); ++u) {
      NgCall& c = calls[sub[ug[u]]];
      tr.x[u] = c.x; tr.ld[u] = c.ld; tr.n[u] = c.n; tr.D[u] = c.h->dim;
      tr.out[u] = c.h->sums + 2; tr.part[u] = c.h->trpart;
    }
    int nmax = 1;
    for (int u = 0; u < tr.count; ++u) nmax = std::max(nmax, tr.n[u]);
    trace_part_kernel<<<dim3(nmax, tr.count), 128, 0, sx>>>(tr);
    NG_TRY(check_launch("trace_part_kernel"));
    trace_final_kernel<<<tr.count, 256, 0, sx>>>(tr);
    NG_TRY(check_launch("trace_final_kernel"));
    if (ev_ab) NG_CUDA_TRY(cudaEventRecord(ev_ab, sx));   // H, J, trace done: phase C may go
    NG_TRY(launch_refresh_group(calls, sub, ug, sx));
  }
  if (ev_ab && ug.empty()) NG_CUDA_TRY(cudaEventRecord(ev_ab, sx));
  return NG_OK;
  };
  // On an update step the states with the largest refreshes (every updating state of the
  // largest rank; NG_TUNE_CRIT_FIRST=1: only the largest one, rank then dimension) get their
  // phases A/B on a side stream, concurrently with the other states' on the main stream, so
  // their refresh chains -- the ones the next step waits for -- start as soon as their own
  // J, K, L are formed instead of after everyone's (NG_TUNE_CRIT_FIRST=0: one group).
  static const int crit_first = tune_int("NG_TUNE_CRIT_FIRST", 2);
  int crit = -1, nupd = 0;
  for (int g = 0; g < G; ++g) {
    if (!upd[grp[g]]) continue;
    ++nupd;
    const ngsgd_ctx* h = calls[grp[g]].h;
    if (crit < 0 || h->rank > calls[grp[crit]].h->rank ||
        (h->rank == calls[grp[crit]].h->rank && h->dim > calls[grp[crit]].h->dim))
      crit = g;
  }
  if (crit_first && nupd >= 2 && crit >= 0) {
    std::vector<int> first, rest;
    const int rmax = calls[grp[crit]].h->rank;
    for (int g = 0; g < G; ++g) {
      const bool side = crit_first == 2 ? (upd[grp[g]] && calls[grp[g]].h->rank == rmax) : g == crit;
      (side ? first : rest).push_back(grp[g]);
    }
    if (rest.empty()) { first.assign(1, grp[crit]); rest.clear(); for (int g = 0; g < G; ++g) if (g != crit) rest.push_back(grp[g]); }
    ngsgd_ctx* hc = calls[first[0]].h;
    NG_CUDA_TRY(cudaEventRecord(hc->ev_fork, st));
    NG_CUDA_TRY(cudaStreamWaitEvent(hc->side, hc->ev_fork, 0));
    NG_TRY(phases_ab(first, hc->side, hc->ev_ab));
    NG_TRY(phases_ab(rest, st, nullptr));
    NG_CUDA_TRY(cudaStreamWaitEvent(st, hc->ev_ab, 0));
  } else {
    NG_TRY(phases_ab(grp, st, nullptr));
  }
  // ---- phase C: X_hat = X - H W with fused row norms (one launch), finalize (one launch)
  {
    double flops = 0, bytes = 0;
    std::vector<TcGroupDesc> d(G);
    FinalizeGroup fg;
    std::memset(&fg, 0, sizeof(fg));
    fg.count = G;
    for (int g = 0; g < G; ++g) {
      NgCall& c = calls[grp[g]];
      ngsgd_ctx* h = c.h;
      const int R = h->rank, D = h->dim;
      flops += 2.0 * c.n * R * D;
      bytes += 4.0 * (2.0 * c.n * D + (double)R * D);
      TcGroupDesc& q = d[g];
      q.M = c.n; q.N = D; q.K = R; q.splits = 1;
      q.A = h->H; q.lda = R; q.B = Wold[g]; q.ldb = h->ldw;
      q.epi.kind = TC_EPI_NGAPPLY; q.epi.C = c.x; q.epi.ldc = c.ld; q.epi.xx = h->xxpart; q.epi.pp = h->ppart;
      q.epi.part_ld = h->max_rows;
      q.splits_used = nullptr;
      fg.n[g] = c.n; fg.tiles[g] = ceil_div(D, apply_bn()); fg.xxpart[g] = h->xxpart; fg.ppart[g] = h->ppart;
      fg.part_ld[g] = h->max_rows; fg.p_int[g] = h->p; fg.p_out[g] = c.p_out; fg.sums[g] = h->sums;
      fg.gamma_int[g] = h->gamma; fg.gamma_out[g] = c.gamma_out; fg.flags[g] = h->flags;
    }
    ProfScope ps(NG_PROF_NG_APPLY, st, flops, bytes);
    NG_TRY(tc_gemm_tf32_grouped(st, d.data(), G, true, false, TC_EPI_NGAPPLY, apply_bn(), true));
    NG_CUDA_TRY(launch_pdl(finalize_group_kernel, dim3(G), dim3(512), 0, st, fg));
    NG_TRY(check_launch("finalize_group_kernel"));
  }
  // ---- phase D: refresh chains on the side streams; bookkeeping
  for (int g = 0; g < G; ++g) {
    NgCall& c = calls[grp[g]];
    ngsgd_ctx* h = c.h;
    h->t += 1;
    h->last_updated = upd[grp[g]] ? 1 : 0;
    if (c.updated_out) *c.updated_out = upd[grp[g]] ? 1 : 0;
  }
  return NG_OK;
}

}  // namespace ng

// ------------------------------------------------------------------------------------
// C ABI
// ------------------------------------------------------------------------------------
using namespace ng;

extern "C" {

const char* ng_last_error(void) { return ng::last_error(); }
const char* ng_version(void) { return "libngsgd 0.1 (sm_100a)"; }

void ngsgd_config_default(ngsgd_config* cfg, int32_t rank) {
  if (!cfg) return;
  cfg->rank = rank;
  cfg->alpha = 4.0f;
  cfg->s_samples = 2000.0f;
  cfg->update_period = 4;
  cfg->always_update_first = 10;
  cfg->epsilon = 1e-10f;
  cfg->precision = NG_FP32;
}

ng_status ng_profile_enable(uint32_t mask) {
  if (mask != 0 && g_ev0.empty()) {
    const int pool = 8192;
    g_ev0.resize(pool); g_ev1.resize(pool); g_ev_group.resize(pool);
    for (int i = 0; i < pool; ++i) {
      NG_CUDA_TRY(cudaEventCreate(&g_ev0[i]));
      NG_CUDA_TRY(cudaEventCreate(&g_ev1[i]));
    }
  }
  if (g_ev_used) prof_flush();
  std::memset(&g_prof, 0, sizeof(g_prof));
  g_prof_mask = mask;
  return NG_OK;
}

ng_status ng_profile_read(ng_profile_stats* out) {
  NG_REQUIRE(out != nullptr, NG_EINVAL, "NULL argument");
  prof_flush();
  *out = g_prof;
  return NG_OK;
}

int64_t ng_kernel_launches(void) { return g_launches.load(); }

ng_status ngsgd_create(int32_t dim, int32_t max_rows, const ngsgd_config* cfg, void* cuda_stream, ngsgd_t* out) {
  return ngsgd_create_impl(dim, max_rows, cfg, (cudaStream_t)cuda_stream, out);
}

ng_status ngsgd_join(ngsgd_t h) {
  NG_REQUIRE(h != nullptr, NG_EINVAL, "NULL argument");
  return ngsgd_join_impl(h);
}

ng_status ngsgd_destroy(ngsgd_t h) {
  if (!h) return NG_EINVAL;
  ngsgd_join_impl(h);
  cudaStreamSynchronize(h->st);
  ngsgd_destroy_impl(h);
  return NG_OK;
}

ng_status ngsgd_precondition(ngsgd_t h, int32_t n, float* x, int64_t ld, float* gamma_out, float* p_out,
                             int32_t update) {
  return ngsgd_precondition_impl(h, n, x, ld, gamma_out, p_out, update, nullptr);
}

ng_status ngsgd_get_state(ngsgd_t h, ngsgd_state_host* out) {
  NG_REQUIRE(h != nullptr && out != nullptr, NG_EINVAL, "NULL argument");
  NG_TRY(ngsgd_join_impl(h));
  NG_CUDA_TRY(cudaStreamSynchronize(h->st));
  const int R = h->rank, D = h->dim;
  out->dim = D;
  out->rank = R;
  out->t = h->t;
  out->initialized = h->initialized ? 1 : 0;
  int flags[8];
  NG_CUDA_TRY(cudaMemcpy(flags, h->flags, sizeof(flags), cudaMemcpyDeviceToHost));
  std::vector<double> ds(1 + 2 * std::max(R, 1));
  NG_CUDA_TRY(cudaMemcpy(ds.data(), h->dstate, sizeof(double) * ds.size(), cudaMemcpyDeviceToHost));
  out->rho = ds[0];
  if (out->d) for (int i = 0; i < R; ++i) out->d[i] = ds[1 + i];
  if (out->w && R > 0)
    NG_CUDA_TRY(cudaMemcpy2D(out->w, sizeof(float) * D, h->W[h->cur], sizeof(float) * h->ldw, sizeof(float) * D, R,
                             cudaMemcpyDeviceToHost));
  out->last_updated = h->last_updated;
  out->last_floored = h->last_updated ? flags[0] : 0;
  out->last_reorth_checked = h->last_updated ? flags[1] : 0;
  out->last_reorthogonalized = h->last_updated ? flags[2] : 0;
  out->last_jacobi_sweeps = h->last_updated ? flags[4] : 0;
  return status_from_flags((uint32_t)flags[3], "ngsgd_get_state");
}

ng_status ngsgd_set_state(ngsgd_t h, const ngsgd_state_host* in) {
  NG_REQUIRE(h != nullptr && in != nullptr, NG_EINVAL, "NULL argument");
  NG_REQUIRE(in->dim == h->dim && in->rank == h->rank, NG_ESHAPE, "state dim/rank mismatch");
  NG_REQUIRE(in->t >= 0, NG_EINVAL, "t < 0");
  const int R = h->rank, D = h->dim;
  NG_TRY(ngsgd_join_impl(h));
  NG_CUDA_TRY(cudaStreamSynchronize(h->st));
  if (R > 0) {
    NG_REQUIRE(in->d != nullptr && in->w != nullptr, NG_EINVAL, "d and w required");
    std::vector<double> ds(1 + 2 * R);
    ds[0] = in->rho;
    double sd = 0.0;
    for (int i = 0; i < R; ++i) { ds[1 + i] = in->d[i]; sd += in->d[i]; }
    const double beta = in->rho * (1.0 + h->cfg.alpha) + (h->cfg.alpha / D) * sd;
    for (int i = 0; i < R; ++i) ds[1 + R + i] = 1.0 / (beta / in->d[i] + 1.0);
    NG_CUDA_TRY(cudaMemcpy(h->dstate, ds.data(), sizeof(double) * ds.size(), cudaMemcpyHostToDevice));
    NG_CUDA_TRY(cudaMemset(h->W[0], 0, sizeof(float) * R * h->ldw));
    NG_CUDA_TRY(cudaMemcpy2D(h->W[0], sizeof(float) * h->ldw, in->w, sizeof(float) * D, sizeof(float) * D, R,
                             cudaMemcpyHostToDevice));
  } else {
    double rho = in->rho;
    NG_CUDA_TRY(cudaMemcpy(h->dstate, &rho, sizeof(double), cudaMemcpyHostToDevice));
  }
  NG_CUDA_TRY(cudaMemset(h->flags, 0, sizeof(int) * 8));
  h->cur = 0;
  h->t = in->t;
  h->initialized = in->initialized != 0;
  h->last_updated = 0;
  return NG_OK;
}

__global__ void __launch_bounds__(kTriThreads, 1) debug_eig_tri_kernel(const double* Z, int n, double* lam, double* vt, int* ok) {
  extern __shared__ __align__(16) unsigned char ng_smem[];
  double* sm = reinterpret_cast<double*>(ng_smem);
  const TriPlan tp = tri_plan(n);
  const long long t0 = clock64();
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) sm[tp.oA + (idx / n) * tp.lda + idx % n] = Z[idx];
  __syncthreads();
  const int r = eig_tri(tp, sm);
  const long long t1 = clock64();
  for (int i = threadIdx.x; i < n; i += blockDim.x) lam[i] = sm[tp.olam + i];
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) vt[idx] = sm[tp.oA + (idx / n) * tp.lda + idx % n];
  if (threadIdx.x == 0) {
    ok[0] = r;
    ok[1] = (int)min(t1 - t0, (long long)INT32_MAX);
    for (int k = 0; k < 4; ++k) ok[2 + k] = r || k < 2 ? (int)(g_tri_clk[k + 1] - g_tri_clk[k]) : 0;
    ok[5] = g_tri_maxit; g_tri_maxit = 0;
    ok[6] = (int)(g_tri_clk[6] - g_tri_clk[5]);   // multisection
    ok[7] = (int)(g_tri_clk[2] - g_tri_clk[6]);   // RQI + vectors + clusters
    if (ok[8] == 0x5eed) {                         // caller asked for the finer phase-2 stamps
      ok[8] = (int)(g_tri_dbg[0] - g_tri_clk[1]);   // split
      ok[9] = (int)(g_tri_dbg[1] - g_tri_dbg[0]);   // root representations
      ok[10] = (int)(g_tri_clk[5] - g_tri_dbg[1]);  // coarse negcounts
      ok[11] = (int)(g_tri_dbg[2] - g_tri_clk[6]);  // RQI + twisted vectors (all eigenvalues)
      ok[12] = (int)(g_tri_clk[2] - g_tri_dbg[2]);  // clusters
      ok[13] = (int)g_tri_rqimax;                    // slowest eigenvalue's RQI loop
      g_tri_rqimax = 0;
    }
  }
}

ng_status ng_debug_refresh_times(uint64_t* out, int32_t* count) {
  NG_REQUIRE(out && count, NG_EINVAL, "NULL argument");
  NG_CUDA_TRY(cudaDeviceSynchronize());
  unsigned int n = 0;
  NG_CUDA_TRY(cudaMemcpyFromSymbol(&n, g_ref_n, sizeof(n)));
  NG_CUDA_TRY(cudaMemcpyFromSymbol(out, g_ref_t, sizeof(unsigned long long) * 256 * 9));
  *count = (int32_t)n;
  return NG_OK;
}

ng_status ng_debug_tri_fail(double* z_host, int32_t* info_host) {
  NG_REQUIRE(z_host && info_host, NG_EINVAL, "NULL argument");
  NG_CUDA_TRY(cudaDeviceSynchronize());
  int v[5];
  NG_CUDA_TRY(cudaMemcpyFromSymbol(&v[3], g_tri_maxpos, sizeof(int)));
  NG_CUDA_TRY(cudaMemcpyFromSymbol(&v[4], g_tri_maxit, sizeof(int)));
  const int zero = 0;
  NG_CUDA_TRY(cudaMemcpyToSymbol(g_tri_maxpos, &zero, sizeof(int)));
  NG_CUDA_TRY(cudaMemcpyToSymbol(g_tri_maxit, &zero, sizeof(int)));
  NG_CUDA_TRY(cudaMemcpyFromSymbol(&v[0], g_tri_fail_n, sizeof(int)));
  NG_CUDA_TRY(cudaMemcpyFromSymbol(&v[1], g_tri_fail_count, sizeof(int)));
  NG_CUDA_TRY(cudaMemcpyFromSymbol(&v[2], g_tri_fail_why, sizeof(int)));
  NG_CUDA_TRY(cudaMemcpyFromSymbol(z_host, g_tri_fail_z, sizeof(double) * kTriMax * kTriMax));
  for (int i = 0; i < 5; ++i) info_host[i] = v[i];
  return NG_OK;
}

ng_status ng_debug_eig_tri(const double* z, int32_t n, double* lam, double* vt, int32_t* ok, void* stream) {
  NG_REQUIRE(z && lam && vt && ok, NG_EINVAL, "NULL argument");
  NG_REQUIRE(n >= 1 && n <= kTriMax, NG_ESHAPE, "n must be in [1, 80]");
  const size_t smem = tri_plan(n).total + 16;
  NG_TRY(set_kernel_attrs());   // (also the solver's tuning knobs)
  NG_CUDA_TRY(cudaFuncSetAttribute(debug_eig_tri_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  debug_eig_tri_kernel<<<1, kTriThreads, smem, (cudaStream_t)stream>>>(z, n, lam, vt, ok);
  return check_launch("debug_eig_tri_kernel");
}

}  // extern "C"
