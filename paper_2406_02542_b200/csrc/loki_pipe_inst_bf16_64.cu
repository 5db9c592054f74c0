// Instantiations of the pipe kernel for __nv_bfloat16 caches, head dim 64 (see loki_pipe.cu).
#include "loki_pipe_impl.cuh"

namespace loki {
LOKI_PIPE_SLICE(bf16_64, __nv_bfloat16, 64)
}  // namespace loki
