// Backward kernels instantiated for float (bodies in gf_attn_bwd.cuh).
#include "gf_attn_bwd.cuh"

namespace gfb {
template int launch_bwd<float>(const DevGraph&, BwdArgs<float>, int, int, cudaStream_t);
}  // namespace gfb
