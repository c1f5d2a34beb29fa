// tcgen05 implicit-GEMM conv (sm_100a) -- placeholder until the tensor-core path lands;
// pmx_conv() falls back to the SIMT kernel (conv_simt.cu) for every shape.
#include "pmx_common.cuh"

namespace pmx {

pmx_status conv_tc_try(const pmx_conv_desc&, const void*, const void*, const float*, const float*, const float*,
                       const Outs&, uint32_t*, void*, size_t, cudaStream_t, bool* launched) {
  *launched = false;
  return PMX_OK;
}

size_t conv_tc_workspace(const pmx_conv_desc&) { return 0; }

const char* conv_tc_backend(int, int) { return "simt"; }

}  // namespace pmx
