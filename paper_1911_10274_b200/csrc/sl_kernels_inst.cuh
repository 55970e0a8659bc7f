// sl_kernels_inst.cuh -- instantiate the launchers of one precision.
// Included by sl_kernels_fp64.cu (compiled with -fmad=false so the fp64
// operation order is the reference's strict IEEE order) and by
// sl_kernels_fp32.cu (FMA contraction allowed: tolerance modes).
#pragma once
#include "sl_device.cuh"

#define SL_DEFINE_LAUNCHERS(PREC, FN)                                        \
  namespace sl {                                                             \
  namespace {                                                                \
  void FN##_gather(const KState &S, const EnvP &E, const StepP &T,           \
                   cudaStream_t st) {                                        \
    if (S.m_n > 0) k_gather_step<PREC, false><<<blocks_for(S.m_n), 256, 0, st>>>(S, E, T); \
  }                                                                          \
  void FN##_tma(const KState &S, const EnvP &E, const StepP &T,             \
               const TmaCfg &C, int grid, cudaStream_t st) {                 \
    size_t sm = (size_t)C.warps * (2 * C.stage_bytes + 16);                  \
    k_gather_tma<PREC><<<grid, 32 * C.warps, sm, st>>>(S, E, T, C);          \
  }                                                                          \
  int FN##_tma_setup(int smem_bytes) {                                       \
    return (int)cudaFuncSetAttribute(k_gather_tma<PREC>,                     \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                     smem_bytes);                            \
  }                                                                          \
  void FN##_force(const KState &S, const EnvP &E, const StepP &T,            \
                  cudaStream_t st) {                                         \
    if (S.m_n > 0) k_gather_step<PREC, true><<<blocks_for(S.m_n), 256, 0, st>>>(S, E, T); \
  }                                                                          \
  void FN##_spring(const KState &S, const StepP &T, bool special,            \
                   cudaStream_t st) {                                        \
    if (S.s_n <= 0) return;                                                  \
    if (special)                                                             \
      k_spring_atomic<PREC, true><<<blocks_for(S.s_n), 256, 0, st>>>(S, T);  \
    else                                                                     \
      k_spring_atomic<PREC, false><<<blocks_for(S.s_n), 256, 0, st>>>(S, T); \
  }                                                                          \
  void FN##_mass(const KState &S, const EnvP &E, const StepP &T,             \
                 cudaStream_t st) {                                          \
    if (S.m_n > 0) k_mass<PREC><<<blocks_for(S.m_n), 256, 0, st>>>(S, E, T); \
  }                                                                          \
  }                                                                          \
  const Launch &FN() {                                                       \
    static const Launch L = {FN##_gather, FN##_tma, FN##_tma_setup,          \
                             FN##_force, FN##_spring, FN##_mass};           \
    return L;                                                                \
  }                                                                          \
  }
