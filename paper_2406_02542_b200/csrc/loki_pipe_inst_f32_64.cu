// Instantiations of the pipe kernel for float caches, head dim 64 (see loki_pipe.cu).
#include "loki_pipe_impl.cuh"

namespace loki {
LOKI_PIPE_SLICE(f32_64, float, 64)
}  // namespace loki
