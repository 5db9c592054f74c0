// Instantiations of the pipe kernel for __nv_bfloat16 caches, head dim 128 (see loki_pipe.cu).
#include "loki_pipe_impl.cuh"

namespace loki {
LOKI_PIPE_SLICE(bf16_128, __nv_bfloat16, 128)
}  // namespace loki
