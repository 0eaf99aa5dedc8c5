// gemm_tc.cuh -- tcgen05/TMEM/TMA GEMMs for the BF16 path (sm_100a).  Interface used by
// nnet.cu; see gemm_tc.cu for the kernels.
#pragma once

#include <vector>

#include "ng_common.cuh"

struct EpiPnormBack;

namespace ng {

struct TcGemm {
  bool ready = false;
  ng_status init(const std::vector<int>& rows, const std::vector<int>& cols, const std::vector<int>& ldp, int max_n,
                 cudaStream_t st) {
    (void)rows; (void)cols; (void)ldp; (void)max_n; (void)st;
    set_error("BF16 tensor-core path is not built in this version (use precision = NG_FP32)");
    return NG_EINVAL;
  }
  template <class Epi>
  ng_status backward(int, int, const float*, const float*, const Epi&) { return NG_EINVAL; }
  ng_status forward(int, int, const float*, const float*, float*) { return NG_EINVAL; }
  ng_status update(int, int, const float*, const float*, float*, const float*) { return NG_EINVAL; }
  void release() {}
};

}  // namespace ng
