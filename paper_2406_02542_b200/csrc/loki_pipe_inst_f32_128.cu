// Instantiations of the pipe kernel for float caches, head dim 128 (see loki_pipe.cu).
#include "loki_pipe_impl.cuh"

namespace loki {
LOKI_PIPE_SLICE(f32_128, float, 128)
}  // namespace loki
