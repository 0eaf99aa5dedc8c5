// simple_ng_impl.cuh -- internal definition of the simple NG-SGD workspace (Appendix A),
// shared by simple_ng.cu and nnet.cu (precond = 2: 2I of them per network).
#pragma once

#include "ng_common.cuh"

struct ngsimple_ctx {
  int dim = 0, max_rows = 0;
  float alpha = 4.f;
  cudaStream_t st = nullptr;
  double* G = nullptr;        // min(dim, max_rows)^2: Gram / Cholesky factor
  double* Y = nullptr;        // dim x max_rows: solves
  double* DI = nullptr;       // inverses of the diagonal blocks of the Cholesky factor
  double* rowpart = nullptr;  // 2 x max_rows
  double* stats = nullptr;    // [0] tr X^T X [1] beta [2] sum ||x||^2 [3] sum ||x_hat||^2
  float* gamma = nullptr;
  float* p = nullptr;
  int* flags = nullptr;
};

namespace ng {
struct SimpleCall {
  ngsimple_ctx* h;
  int n;
  float* x;
  int64_t ld;
  float* gamma_out;   // may be NULL (then h->gamma)
  float* p_out;       // may be NULL (then h->p)
};
// All calls (sharing one stream) as one launch per phase: Gram, Cholesky, solves, rows, gamma.
ng_status ngsimple_precondition_group_impl(const SimpleCall* calls, int count);
}  // namespace ng

ng_status ngsimple_create_impl(int dim, int max_rows, float alpha, cudaStream_t st, ngsimple_ctx** out);
void ngsimple_destroy_impl(ngsimple_ctx* h);
