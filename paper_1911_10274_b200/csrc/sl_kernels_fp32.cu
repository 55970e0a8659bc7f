// fp32 and mixed-precision kernels (tolerance modes, FMA allowed).
#include "sl_kernels_inst.cuh"
SL_DEFINE_LAUNCHERS(PREC_FP32, launch_fp32)
SL_DEFINE_LAUNCHERS(PREC_MIXED, launch_mixed)
