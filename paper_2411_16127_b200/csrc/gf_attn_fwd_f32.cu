// Forward kernels instantiated for float (bodies in gf_attn_fwd.cuh).
#define GF_FWD_PRIMARY
#include "gf_attn_fwd.cuh"

namespace gfb {
template int launch_fwd<float>(const DevGraph&, const FwdArgs<float>&, int, cudaStream_t);
template int launch_fwd_mode<float>(const DevGraph&, const FwdArgs<float>&, int, int, cudaStream_t);
template int launch_materialize_p<float>(const DevGraph&, const FwdArgs<float>&, int, float*,
                                      cudaStream_t);
}  // namespace gfb
