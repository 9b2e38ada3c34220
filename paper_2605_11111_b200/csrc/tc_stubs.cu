// Placeholder tcgen05 entry points until conv_tc.cu / attn_tc.cu land:
// every configuration reports "not eligible", so AUTO picks the CUDA-core
// kernels and DP_ALGO_TC fails loudly.
#include "common.cuh"
namespace dp {
int conv_tc_eligible(const dp_conv_geom *, int, int) { return 0; }
int conv_fwd_tc_launch(const dp_conv_geom *, const void *, const void *, const void *, void *,
                       cudaStream_t) { return DP_ERR_UNSUPPORTED; }
int conv_dgrad_tc_launch(const dp_conv_geom *, const void *, const void *, void *, void *,
                         cudaStream_t) { return DP_ERR_UNSUPPORTED; }
int64_t conv_wgrad_tc_workspace(const dp_conv_geom *) { return -1; }
int conv_wgrad_tc_launch(const dp_conv_geom *, const void *, const void *, const void *, void *,
                         void *, int64_t, cudaStream_t) { return DP_ERR_UNSUPPORTED; }
int attn_tc_eligible(const dp_attn_geom *, int) { return 0; }
int attn_fwd_update_tc_launch(const dp_attn_geom *, const void *, const void *, const void *,
                              void *, void *, void *, cudaStream_t) { return DP_ERR_UNSUPPORTED; }
int attn_bwd_update_tc_launch(const dp_attn_geom *, const void *, const void *, const void *,
                              const void *, const void *, const void *, void *, void *, void *,
                              cudaStream_t) { return DP_ERR_UNSUPPORTED; }
}  // namespace dp
