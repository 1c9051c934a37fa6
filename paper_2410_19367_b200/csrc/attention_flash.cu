// Flash attention (bf16 tensor cores) -- placeholder until the tiled kernel lands.
#include "common.cuh"

namespace bp {
bool opt_attn_exact();
bool attn_flash_supported(int dtype, int S, int Dh) { (void)dtype; (void)S; (void)Dh; return false; }
int attn_flash_fwd(int, int, int, int, int, float, const void*, void*, float*, cudaStream_t) {
  set_error("flash attention not built");
  return BP_ERR_UNSUPPORTED;
}
int attn_flash_bwd(int, int, int, int, int, float, const void*, const void*, const void*, const float*, void*, float*,
                   cudaStream_t) {
  set_error("flash attention not built");
  return BP_ERR_UNSUPPORTED;
}
}  // namespace bp
