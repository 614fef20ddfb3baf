// k_tc_gemm.cu — tcgen05/TMEM/TMA tensor-core engine (bring-up pending).
#include "internal.h"

namespace spk {

bool tc_supported(const ActorDims& d) {
  (void)d;
  return false;
}

int launch_lif_fwd_tc(const ActorDims& d, int l, int B, const uint32_t* bits_in,
                      const __nv_bfloat16* Wb16, uint32_t* bits_out, uint32_t* mask_out,
                      uint8_t* counts, cudaStream_t st) {
  (void)d; (void)l; (void)B; (void)bits_in; (void)Wb16; (void)bits_out; (void)mask_out;
  (void)counts; (void)st;
  set_error("tcgen05 engine not available");
  return SPIKERL_E_UNSUPPORTED;
}

}  // namespace spk
