// Placeholder tcgen05 attention entry points until attn_tc.cu lands: every
// configuration reports "not eligible", so AUTO picks the CUDA-core kernels
// and DP_ALGO_TC fails loudly.
#include "common.cuh"
namespace dp {
int attn_tc_eligible(const dp_attn_geom *, int) { return 0; }
int attn_fwd_update_tc_launch(const dp_attn_geom *, const void *, const void *, const void *,
                              void *, void *, void *, cudaStream_t) { return DP_ERR_UNSUPPORTED; }
int attn_bwd_update_tc_launch(const dp_attn_geom *, const void *, const void *, const void *,
                              const void *, const void *, const void *, void *, void *, void *,
                              cudaStream_t) { return DP_ERR_UNSUPPORTED; }
}  // namespace dp
