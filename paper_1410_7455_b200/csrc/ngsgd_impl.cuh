// ngsgd_impl.cuh -- internal definition of the online NG-SGD handle (Appendix B),
// shared by ngsgd.cu (the preconditioner) and nnet.cu (which owns 2I of them).
#pragma once

#include <vector>

#include "ng_common.cuh"

struct ngsgd_ctx {
  int dim = 0, rank = 0, ldw = 0, max_rows = 0;
  ngsgd_config cfg{};
  cudaStream_t st = nullptr;
  int t = 0;
  bool initialized = false;
  int cur = 0;                 // which W buffer holds W_t
  int last_updated = 0;
  // ---- device state (B.5: rho_t, D_t, W_t)
  float* W[2] = {nullptr, nullptr};   // R x ldw each
  double* dstate = nullptr;           // [0] rho, [1..R] d (descending), [R+1..2R] e_{t+1}
  // ---- device workspace (sized at create time; the hot path never allocates)
  int h_splits = 1, kl_splits = 1, ctiles = 1;
  float* Hpart = nullptr;   // h_splits x max_rows x R
  float* H = nullptr;       // max_rows x R               (H_t = X W_t^T, eqn:ht)
  float* J = nullptr;       // R x ldw                    (J_t = H^T X)
  float* Kpart = nullptr;   // kl_splits x R x R
  float* Lpart = nullptr;   // max(kl_splits, n splits) x R x R
  float* KL = nullptr;      // 2 x R x R  (K_t then L_t)
  float* WWpart = nullptr;  // kl_splits x R x R (re-orthogonalisation, B.3.1)
  float* WW = nullptr;      // R x R
  float* Amat = nullptr;    // R x R  A_t; also M of B.3.1
  float* Mmat = nullptr;    // R x R (unused by the repair since the triangular-solve form)
  double* Cfac = nullptr;   // R x R lower Cholesky factor of O (B.3.1 repair)
  double* trpart = nullptr; // max_rows row sums of ||x_i||^2 (early tr(X X^T))
  float* svec = nullptr;    // R:  N(1-eta)/eta (d_i + rho)  (row scale of B_t)
  float* xxpart = nullptr;  // ctiles x max_rows: partial ||x_i||^2
  float* ppart = nullptr;   // ctiles x max_rows: partial ||x_hat_i||^2
  float* p = nullptr;       // max_rows
  double* sums = nullptr;   // [0] tr(X X^T)  [1] sum_i p_i
  float* gamma = nullptr;   // [1]
  int* flags = nullptr;     // [0] floored [1] reorth check [2] repaired [3] error bits [4] sweeps
  // pinned host mirror for the (one-time) initialisation sync
  double* h_scalar = nullptr;
  // side stream for the refresh (Z_t eigensolve, W_{t+1}); joined before the next use
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_ab = nullptr;   // critical state's phases A/B done on its side stream (group path)
  bool pending = false;
};

namespace ng {
// Precondition with explicit output buffers (used by nnet.cu).  gamma_out / p_out may be
// NULL (then the handle's internal buffers hold the results: h->gamma, h->p).
ng_status ngsgd_precondition_impl(ngsgd_ctx* h, int n, float* x, int64_t ld, float* gamma_out,
                                  float* p_out, int update, int* updated_out);
ng_status ngsgd_create_impl(int dim, int max_rows, const ngsgd_config* cfg, cudaStream_t st,
                            ngsgd_ctx** out);
void ngsgd_destroy_impl(ngsgd_ctx* h);
ng_status ngsgd_join_impl(ngsgd_ctx* h);

// One preconditioning call of a group (see ngsgd_precondition_group_impl).
struct NgCall {
  ngsgd_ctx* h;
  int n;
  float* x;
  int64_t ld;
  float* gamma_out;
  float* p_out;
  int update;          // -1 policy, 0/1 forced
  int* updated_out;    // optional
};
// Precondition several independent states on one stream with ONE launch per phase for
// all tensor-core-eligible states (H projections, their reduction, J, X_hat, finalize);
// other calls fall back to ngsgd_precondition_impl.  Results identical to calling
// ngsgd_precondition_impl on each call in turn.
ng_status ngsgd_precondition_group_impl(NgCall* calls, int count);
}  // namespace ng
