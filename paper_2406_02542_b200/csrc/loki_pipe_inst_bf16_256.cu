// Instantiations of the pipe kernel for __nv_bfloat16 caches, head dim 256 (see loki_pipe.cu).
#include "loki_pipe_impl.cuh"

namespace loki {
LOKI_PIPE_SLICE(bf16_256, __nv_bfloat16, 256)
}  // namespace loki
