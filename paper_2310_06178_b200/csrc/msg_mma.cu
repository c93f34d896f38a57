// K4 placeholder: dequantise-then-tcgen05.mma comparison kernel (see msg_mma_tc.cu when built).
#include "msg_common.cuh"

using namespace msg;

extern "C" int64_t msg_dequant_mma_workspace_bytes(int64_t m, int64_t k, int64_t b) {
  (void)m; (void)k; (void)b;
  return 0;
}

extern "C" int msg_dequant_mma(const uint8_t* packed, int64_t m, int64_t k, const double* values,
                               const void* x_f16, int64_t b, float* y, void* workspace,
                               int64_t workspace_bytes, void* stream) {
  (void)packed; (void)m; (void)k; (void)values; (void)x_f16; (void)b; (void)y;
  (void)workspace; (void)workspace_bytes; (void)stream;
  return fail(MSG_ERR_UNSUPPORTED, "dequant-MMA comparison kernel not built yet");
}
