// fp64 parity kernels.  Build flag -fmad=false: no FMA contraction, so each
// multiply/add rounds exactly like the reference's numba code (kernels.py,
// compiled without fastmath).
#define SL_UNIT_FP64 1
#include "sl_kernels_inst.cuh"
SL_DEFINE_LAUNCHERS(PREC_FP64, launch_fp64)
