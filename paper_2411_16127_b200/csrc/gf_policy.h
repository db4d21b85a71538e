// L2 cache-hint policy words shared by the host launchers and the kernels.
#pragma once

#include <cstdint>

namespace gfb {

// The word createpolicy.fractional.L2::evict_last 1.0 yields on sm_100a
// (ptxas folds the instruction to this constant; tests/test_gpu_state.py
// checks the two agree on the device).  The backward passes take it from their
// argument block (GF_POL_PARAM_BWD): a kernel-parameter word stays in a
// uniform register, where the in-kernel value is materialised into a register
// pair and copied back (2 x R2UR) before every gather — pass B 1.5 % faster
// on C4.  The forward keeps the in-kernel word: with the parameter its loop
// waits on a constant-bank load before its gathers and measured 12 % slower
// (profiles/r2/ab_r2_policy_param.txt).  Used only with GF_L2_EVICT_OP = 0:
// by default the gathers carry ld.L2::evict_last and need no policy word.
constexpr uint64_t kPolicyEvictLast = 0x14F0000000000000ull;

}  // namespace gfb

#ifndef GF_POL_PARAM_FWD
#define GF_POL_PARAM_FWD 0
#endif
#ifndef GF_POL_PARAM_BWD
#define GF_POL_PARAM_BWD 1
#endif
