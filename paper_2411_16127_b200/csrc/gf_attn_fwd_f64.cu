// Forward kernels instantiated for double (bodies in gf_attn_fwd.cuh).
#include "gf_attn_fwd.cuh"

namespace gfb {
template int launch_fwd<double>(const DevGraph&, const FwdArgs<double>&, int, cudaStream_t);
template int launch_fwd_mode<double>(const DevGraph&, const FwdArgs<double>&, int, int, cudaStream_t);
template int launch_materialize_p<double>(const DevGraph&, const FwdArgs<double>&, int, double*,
                                      cudaStream_t);
}  // namespace gfb
