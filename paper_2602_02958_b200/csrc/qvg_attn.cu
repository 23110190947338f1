// qvg_attn.cu — attention over the quantized cache (placeholder until the
// tcgen05 kernel lands; returns QVG_ERR_UNSUPPORTED).
#include "qvg_common.cuh"
#include "qvg_internal.h"

namespace qvg {
size_t attention_workspace_size(int64_t, int64_t, int64_t, int, int, const qvg_config *) { return 0; }
int run_attention(const uint16_t *, const uint8_t *, const uint8_t *, const uint16_t *,
                  const uint8_t *, const uint16_t *, const uint16_t *, const uint16_t *, int64_t,
                  int64_t, int64_t, int, int, const qvg_config *, float, uint16_t *, void *, size_t,
                  cudaStream_t) {
    return set_err(QVG_ERR_UNSUPPORTED, "attention kernel not built");
}
}  // namespace qvg
