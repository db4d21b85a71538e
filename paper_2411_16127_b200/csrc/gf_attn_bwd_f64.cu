// Backward kernels instantiated for double (bodies in gf_attn_bwd.cuh).
#include "gf_attn_bwd.cuh"

namespace gfb {
template int launch_bwd<double>(const DevGraph&, BwdArgs<double>, int, int, cudaStream_t);
}  // namespace gfb
