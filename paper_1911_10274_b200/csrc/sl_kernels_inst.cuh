// sl_kernels_inst.cuh -- instantiate the launchers of one precision.
// Included by sl_kernels_fp64.cu (compiled with -fmad=false so the fp64
// operation order is the reference's strict IEEE order) and by
// sl_kernels_fp32.cu (FMA contraction allowed: tolerance modes).
#pragma once
#include "sl_device.cuh"
#include "sl_split.cuh"
#include "sl_window.cuh"
#include "sl_fused.cuh"


namespace sl {
// Launch a step kernel with programmatic dependent launch (the kernel
// waits with griddepcontrol.wait before touching the previous step's
// output); SL_PDL=0 launches it plainly.
template <class K, class... A>
inline void launch_pdl(K kern, int grid, int block, size_t smem,
                       cudaStream_t st, A... args) {
  static const bool on = [] {
    const char *ev = getenv("SL_PDL");
    return !(ev && ev[0] == '0');
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = on ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, args...);
}
// Opt a kernel into dynamic shared memory: always to the device maximum, so
// contexts of different layouts on one device (partition shards) never
// shrink the limit under one another's launch; `need` is only checked.
template <class K>
inline int smem_optin(K kern, size_t need) {
  int dev = 0, most = 0;
  cudaFuncAttributes fa;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&most, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                             dev) != cudaSuccess ||
      cudaFuncGetAttributes(&fa, kern) != cudaSuccess)
    return 1;
  most -= (int)fa.sharedSizeBytes;  // the kernel's static shared memory
  if (need > (size_t)most) return 1;
  return (int)cudaFuncSetAttribute(
      kern, cudaFuncAttributeMaxDynamicSharedMemorySize, most);
}
// split-layout launchers; the fp64 parity mode never uses the split layout
template <int P>
struct SplitLaunch {
  template <bool FO, bool ACT>
  static void step_k(const KState &S, const EnvP &E, const StepP &T,
                     const ActP &A, cudaStream_t st) {
    launch_pdl(k_split_step<P, FO, ACT>, (int)blocks_for(S.m_n), 256, 0, st, S, E, T, A);
  }
  static void atomic(const KState &S, const StepP &T, const ActP &A,
                     cudaStream_t st) {
    if (S.m_n <= 0) return;
    if (A.n > 1)
      launch_pdl(k_split_atomic<P, true>, (int)blocks_for(S.m_n), 256, 0, st,
                 S, T, A);
    else
      launch_pdl(k_split_atomic<P, false>, (int)blocks_for(S.m_n), 256, 0,
                 st, S, T, A);
  }
  static void step(const KState &S, const EnvP &E, const StepP &T,
                   const ActP &A, cudaStream_t st, bool force_only) {
    if (S.m_n <= 0) return;
    const bool act = A.n > 1;
    if (force_only)
      act ? step_k<true, true>(S, E, T, A, st)
          : step_k<true, false>(S, E, T, A, st);
    else
      act ? step_k<false, true>(S, E, T, A, st)
          : step_k<false, false>(S, E, T, A, st);
  }
  template <int U, bool ACT>
  static void tma_u(const KState &S, const EnvP &E, const StepP &T,
                    const SplitCfg &C, const ActP &A, int grid,
                    cudaStream_t st) {
    size_t sm = (size_t)C.warps * (2 * C.stage_bytes + 16);
    launch_pdl(k_split_tma<P, U, ACT>, grid, 32 * C.warps, sm, st, S, E, T, C, A);
  }
  static void tma(const KState &S, const EnvP &E, const StepP &T,
                  const SplitCfg &C, const ActP &A, int grid,
                  cudaStream_t st) {
    if (C.act) {  // actuated: more live registers per entry, U <= 8
      if (C.u == 4) tma_u<4, true>(S, E, T, C, A, grid, st);
      else tma_u<8, true>(S, E, T, C, A, grid, st);
      return;
    }
    switch (C.u) {
      case 4: tma_u<4, false>(S, E, T, C, A, grid, st); break;
      case 8: tma_u<8, false>(S, E, T, C, A, grid, st); break;
      default: tma_u<8, false>(S, E, T, C, A, grid, st);
    }
  }
  // tiled window kernel (fp32 and mixed)
  static void win(const KState &S, const EnvP &E, const StepP &T,
                  const WinCfg &C, int grid, cudaStream_t st) {
    {
      const size_t sm = win_smem(C);
      win_dispatch(C.tile_slices, [&](auto kern) {
        launch_pdl(kern, grid, (C.tile_slices + 1) * 32, sm, st, S, E, T, C);
      });
    }
  }
  static size_t win_smem(const WinCfg &C) {
    return (size_t)C.off_eff + WIN_MAXST * WIN_DMAX * 8 + 8 * 2 * WIN_MAXST;
  }
  // call f(kernel) for the instantiation of T
  template <class Fn>
  static void win_dispatch(int tt, Fn f) {
    if constexpr (P == PREC_MIXED) {  // fp64 windows: T = 16 or 12
      if (tt == 12)
        f(k_win_tma<P, 12>);
      else
        f(k_win_tma<P, 16>);
    } else {
      switch (tt) {
        case 4: f(k_win_tma<P, 4>); return;   // small meshes: more CTAs
        case 8: f(k_win_tma<P, 8>); return;
        case 10: f(k_win_tma<P, 10>); return;  // 3 ring stages (sweeps)
        case 12: f(k_win_tma<P, 12>); return;
        case 20: f(k_win_tma<P, 20>); return;
        case 24: f(k_win_tma<P, 24>); return;
        default: f(k_win_tma<P, 16>); return;
      }
    }
  }
  // multi-step fused small-body kernel (fp32 only); C.maxm = 512 (two
  // CTAs per SM) or 1024 (bodies of up to 1024 masses, one CTA per SM)
  static void fused(const KState &S, const EnvP &E, const FzCfg &C,
                    double dt, size_t smem, cudaStream_t st) {
    if constexpr (P == PREC_FP32) {
      if (C.maxm > FZ_MAXM)
        k_fused_small<P, FZ_MAXM_L>
            <<<(unsigned)C.n_groups, FZ_MAXM_L, smem, st>>>(S, E, C, dt);
      else
        k_fused_small<P, FZ_MAXM>
            <<<(unsigned)C.n_groups, FZ_MAXM, smem, st>>>(S, E, C, dt);
    }
  }
  static int fused_setup(size_t smem, int maxm) {
    if constexpr (P == PREC_FP32)
      return maxm > FZ_MAXM ? smem_optin(k_fused_small<P, FZ_MAXM_L>, smem)
                            : smem_optin(k_fused_small<P, FZ_MAXM>, smem);
    return 1;
  }
  static int win_setup(const WinCfg &C) {
    int rc = 1;
    win_dispatch(C.tile_slices, [&](auto kern) {
        rc = smem_optin(kern, win_smem(C));
      });
    return rc;
  }
  template <int U, bool ACT>
  static int setup_u(int smem_bytes) {
    return smem_optin(k_split_tma<P, U, ACT>, (size_t)smem_bytes);
  }
  static int setup(int smem_bytes, int u, int act) {
    if (act) return u == 4 ? setup_u<4, true>(smem_bytes)
                           : setup_u<8, true>(smem_bytes);
    switch (u) {
      case 4: return setup_u<4, false>(smem_bytes);
      case 8: return setup_u<8, false>(smem_bytes);
      default:
        return setup_u<8, false>(smem_bytes);
    }
  }
};
template <>
struct SplitLaunch<PREC_FP64> {
  static void atomic(const KState &, const StepP &, const ActP &,
                     cudaStream_t) {}
  static void step(const KState &, const EnvP &, const StepP &, const ActP &,
                   cudaStream_t, bool) {}
  static void tma(const KState &, const EnvP &, const StepP &,
                  const SplitCfg &, const ActP &, int, cudaStream_t) {}
  static int setup(int, int, int) { return 1; }
  // the window kernel over the exact layout (parity mode; this unit is
  // compiled with -fmad=false)
  static size_t win_smem(const WinCfg &C) {  // eff tables: double2 slots
    return (size_t)C.off_eff + WIN_MAXST * WIN_DMAX * 16 + 8 * 2 * WIN_MAXST;
  }
  // Only the -fmad=false unit instantiates the fp64 kernel: a copy
  // compiled with FMA contraction in another unit could be the one a launch
  // binds to (tests/test_abi.py checks each cubin's instantiations).
#ifdef SL_UNIT_FP64
  // T = SL_WIN64_T (12); 4-slice tiles for small meshes (more CTAs)
  static void win(const KState &S, const EnvP &E, const StepP &T,
                  const WinCfg &C, int grid, cudaStream_t st) {
    if (C.tile_slices == 4)
      launch_pdl(k_win_tma<PREC_FP64, 4>, grid, 5 * 32, win_smem(C), st, S,
                 E, T, C);
    else
      launch_pdl(k_win_tma<PREC_FP64, SL_WIN64_T>, grid,
                 (SL_WIN64_T + 1) * 32, win_smem(C), st, S, E, T, C);
  }
  static int win_setup(const WinCfg &C) {
    if (C.tile_slices == 4)
      return smem_optin(k_win_tma<PREC_FP64, 4>, win_smem(C));
    return smem_optin(k_win_tma<PREC_FP64, SL_WIN64_T>, win_smem(C));
  }
#else
  static void win(const KState &, const EnvP &, const StepP &,
                  const WinCfg &, int, cudaStream_t) {}
  static int win_setup(const WinCfg &) { return 1; }
#endif
  static void fused(const KState &, const EnvP &, const FzCfg &, double,
                    size_t, cudaStream_t) {}
  static int fused_setup(size_t, int) { return 1; }
};
}  // namespace sl

#define SL_DEFINE_LAUNCHERS(PREC, FN)                                        \
  namespace sl {                                                             \
  namespace {                                                                \
  void FN##_gather(const KState &S, const EnvP &E, const StepP &T,           \
                   cudaStream_t st) {                                        \
    if (S.m_n > 0) launch_pdl(k_gather_step<PREC, false>, (int)blocks_for(S.m_n), 256, 0, st, S, E, T); \
  }                                                                          \
  void FN##_tma(const KState &S, const EnvP &E, const StepP &T,             \
               const TmaCfg &C, int grid, cudaStream_t st) {                 \
    size_t sm = (size_t)C.warps * (2 * C.stage_bytes + 16);                  \
    launch_pdl(k_gather_tma<PREC>, grid, 32 * C.warps, sm, st, S, E, T, C);  \
  }                                                                          \
  int FN##_tma_setup(int smem_bytes) {                                       \
    return smem_optin(k_gather_tma<PREC>, (size_t)smem_bytes);               \
  }                                                                          \
  void FN##_force(const KState &S, const EnvP &E, const StepP &T,            \
                  cudaStream_t st) {                                         \
    if (S.m_n > 0) launch_pdl(k_gather_step<PREC, true>, (int)blocks_for(S.m_n), 256, 0, st, S, E, T); \
  }                                                                          \
  void FN##_spring(const KState &S, const StepP &T, bool special,            \
                   cudaStream_t st) {                                        \
    if (S.s_n <= 0) return;                                                  \
    if (special)                                                             \
      launch_pdl(k_spring_atomic<PREC, true>, (int)blocks_for(S.s_n), 256, 0, st, S, T); \
    else                                                                     \
      launch_pdl(k_spring_atomic<PREC, false>, (int)blocks_for(S.s_n), 256, 0, st, S, T); \
  }                                                                          \
  void FN##_mass(const KState &S, const EnvP &E, const StepP &T,             \
                 cudaStream_t st) {                                          \
    if (S.m_n > 0) launch_pdl(k_mass<PREC>, (int)blocks_for(S.m_n), 256, 0, st, S, E, T); \
  }                                                                          \
  void FN##_owner_atomic(const KState &S, const StepP &T, const ActP &A,    \
                         cudaStream_t st) {                                  \
    if (S.split)                                                             \
      SplitLaunch<PREC>::atomic(S, T, A, st);                                \
    else if (S.m_n > 0)                                                      \
      launch_pdl(k_gather_atomic<PREC>, (int)blocks_for(S.m_n), 256, 0, st,  \
                 S, T);                                                      \
  }                                                                          \
  void FN##_split(const KState &S, const EnvP &E, const StepP &T,           \
                  const ActP &A, cudaStream_t st) {                          \
    SplitLaunch<PREC>::step(S, E, T, A, st, false);                          \
  }                                                                          \
  void FN##_split_force(const KState &S, const EnvP &E, const StepP &T,     \
                        const ActP &A, cudaStream_t st) {                    \
    SplitLaunch<PREC>::step(S, E, T, A, st, true);                           \
  }                                                                          \
  void FN##_split_tma(const KState &S, const EnvP &E, const StepP &T,       \
                      const SplitCfg &C, const ActP &A, int grid,            \
                      cudaStream_t st) {                                     \
    SplitLaunch<PREC>::tma(S, E, T, C, A, grid, st);                         \
  }                                                                          \
  int FN##_split_setup(int smem_bytes, int u, int act) {                     \
    return SplitLaunch<PREC>::setup(smem_bytes, u, act);                     \
  }                                                                          \
  void FN##_win(const KState &S, const EnvP &E, const StepP &T,             \
                const WinCfg &C, int grid, cudaStream_t st) {                \
    SplitLaunch<PREC>::win(S, E, T, C, grid, st);                            \
  }                                                                          \
  int FN##_win_setup(const WinCfg &C) {                                      \
    return SplitLaunch<PREC>::win_setup(C);                                  \
  }                                                                          \
  void FN##_fused(const KState &S, const EnvP &E, const FzCfg &C, double dt, \
                  size_t smem, cudaStream_t st) {                            \
    SplitLaunch<PREC>::fused(S, E, C, dt, smem, st);                         \
  }                                                                          \
  int FN##_fused_setup(size_t smem, int maxm) {                              \
    return SplitLaunch<PREC>::fused_setup(smem, maxm);                       \
  }                                                                          \
  }                                                                          \
  const Launch &FN() {                                                       \
    static const Launch L = {FN##_gather, FN##_tma, FN##_tma_setup,          \
                             FN##_force, FN##_spring, FN##_mass,             \
                             FN##_owner_atomic,                              \
                             FN##_split, FN##_split_force, FN##_split_tma,   \
                             FN##_split_setup, FN##_win,                     \
                             FN##_win_setup, FN##_fused, FN##_fused_setup};  \
    return L;                                                                \
  }                                                                          \
  }
