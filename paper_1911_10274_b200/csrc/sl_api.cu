// sl_api.cu -- context, device buffers, incidence-layout build and the C ABI
// declared in include/softlat_cuda.h.
//
// Ownership mirrors the reference's engine cache (engine._StoreCache,
// engine.py:71-146): the context owns every device buffer of one store on one
// device and rebuilds the derived incidence layout when the spring topology
// changes (the reference rebuilds its slotted CSR the same way,
// engine.py:105-118) -- here the rebuild runs on the device (CUB radix sort),
// so a 12.7M-spring lattice re-indexes in milliseconds.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <cub/cub.cuh>
#include <nvtx3/nvToolsExt.h>

#include "../../include/softlat_cuda.h"
#include "sl_device.cuh"
#include "sl_split.cuh"
#include "sl_window.cuh"
#include "sl_fused.cuh"

namespace sl {
const Launch &launch_fp64();
const Launch &launch_fp32();
const Launch &launch_mixed();
const Launch &launchers(int prec) {
  if (prec == PREC_FP64) return launch_fp64();
  if (prec == PREC_FP32) return launch_fp32();
  return launch_mixed();
}
}  // namespace sl

using namespace sl;

namespace {

thread_local std::string g_err;

struct DevBuf {
  void *p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    if (want == 0) want = 16;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) {
      bytes = want;
      // debug: fill fresh buffers with a pattern (finds uninitialised reads)
      static const char *poison = getenv("SL_POISON");
      if (poison) e = cudaMemset(p, (int)strtol(poison, nullptr, 0), want);
    }
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T *as() const {
    return (T *)p;
  }
};

// NVTX ranges on the API entry points and the layout build: the host-side
// timeline in nsys / `ncu --nvtx` (near free when no tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define SL_RANGE(name) NvtxRange sl_nvtx_range_(name)

}  // namespace

struct sl_ctx {
  int device = 0;
  int prec = PREC_FP64;
  size_t rsz = 8, fsz = 8;  // sizeof(R), sizeof(F)
  cudaStream_t st = nullptr, side = nullptr;
  // k0 / k1 bracket the step kernels of the last sl_step call
  cudaEvent_t k0 = nullptr, k1 = nullptr;
  cudaEvent_t head_ev = nullptr, tail_ev = nullptr;  // sl_download_state
  cudaEvent_t extra_ev = nullptr;  // sl_download_state_ex: extra copies
  // sl_download_state_side: unpacked on the stream, copied on c->side
  cudaEvent_t side_ev = nullptr, side_done = nullptr;
  bool side_pending = false, stash_set = false;
  bool tail_pending = false;
  bool k_valid = false;
  cudaEvent_t t0 = nullptr, t1 = nullptr, snap_ev = nullptr,
              snap_done = nullptr;
  int64_t m_n = 0, s_n = 0;
  int cur = 0;
  bool masses_set = false, springs_set = false, env_set = false;
  bool layout_valid = false, validate_dirty = true, has_special = false;
  bool snap_pending = false;
  // mass SoA
  DevBuf pos[2], vel, acc, fext, load, m_gen, m_alive, xflags;
  DevBuf plo[2];  // fp32: position low parts (ly, lz); lx in pos[].w
  DevBuf pmass;   // fp32: masses (the position record's w holds lx)
  DevBuf lc_off, lc_kind, lc_vec;
  bool has_lc = false;
  // spring SoA
  DevBuf ends, kL0, s_alive, s_degen, mode, act, thr, custom, m1gen, m2gen;
  DevBuf damp;               // per-spring damping (sl_set_spring_damping)
  bool has_damping = false;  // some spring has c != 0
  // incidence layout
  DevBuf slice_ptr, ent_j, ent_kL0, ent_s, e1, e2;
  int64_t n_slices = 0, n_entries = 0, alive_springs = 0, layout_builds = 0;
  int64_t max_width = 0;     // widest slice (entries per mass, padded)
  int tma_warps = 0;         // warps per CTA of the TMA kernel (0 = off)
  int tma_grid = 0;
  TmaCfg tma;
  int sm_count = 0, smem_optin = 0;
  bool tma_enabled = true;
  // split layout (tolerance modes, sl_split.cuh)
  bool split_enabled = true;  // SL_DISABLE_SPLIT=1 forces the exact layout
  bool split = false;         // the current layout is split
  int sp_a = 0, sp_rows = 0;
  int64_t sp_wa = 0, sp_wb = 0;  // widest A / B sections
  DevBuf sp_j, sp_kl, sp_s, sp_w, sp_ekl, degB, sp_meta;
  SplitCfg scfg;
  int split_warps = 0, split_grid = 0;
  // tiled window kernel over the split layout (fp32, sl_window.cuh)
  bool win_enabled = true;  // SL_DISABLE_WIN=1 keeps the split kernel
  bool win = false;
  WinCfg wcfg;
  int win_grid = 0;
  DevBuf win_rec, win_dict, win_actb, win_zero, win_blk, win_fail;
  // multi-step fused small-body kernel (fp32, sl_fused.cuh)
  bool fz_enabled = true;  // SL_DISABLE_FUSED=1 keeps per-step kernels
  bool fz_ok = false;
  FzCfg fcfg;
  size_t fz_smem = 0;
  int64_t fz_launches = 0, fz_aborts = 0;
  DevBuf fz_gstart, fz_gcount, fz_ent, fz_code, fz_dict, fz_actb, fz_has,
      fz_zero, fz_gid, fz_fail, fz_times, fz_diff, vel2, fz_perm, fz_cnt,
      fz_epos, fz_cnt_a;
  DevBuf diag;  // diagnostics scratch (sl_energy / sl_spring_loads)
  bool auto_atomic = false;  // SL_ACC_AUTO resolved to the atomic variant
  bool atomic_owner = false;  // atomic accumulation: owner-aggregated kernel
  // grouped sine actuation of the split layout's fast path (ActP)
  ActP agrp;
  DevBuf s_grp, sp_actc, sp_acto;
  // partitioned runs
  DevBuf ghost;
  bool has_ghost = false;
  // in-library halo (sl_halo_*): device descriptor, per-mass send table,
  // the peers' counter words of this context, opened IPC mappings
  HaloDesc halo_host{};
  DevBuf halo_desc, halo_dst, halo_flags;
  bool halo_on = false;
  unsigned long long halo_step = 0;  // steps published so far
  std::vector<void *> halo_ipc;
  bool async_open = false;
  int64_t async_steps = 0;
  int async_cur0 = 0;
  // device copy of the kernel state block (KState::self)
  DevBuf kdev;
  KState khost;
  bool khost_valid = false;
  // scratch
  DevBuf stage, sort_tmp, keys[2], vals[2], deg, width, start;
  DevBuf stage2;  // sl_stash_state: the fp64 state at the last stash
  DevBuf inc_buf;  // insert_incremental: slots, touched tiles, fail flag
  // sl_checkpoint: device copy of the state a speculative run may undo
  DevBuf ck_pos, ck_plo, ck_vel, ck_acc, ck_fext, ck_view;
  int ck_cur = -1;
  cudaEvent_t ck_ev = nullptr, ck_done = nullptr;
  bool ck_pending = false;
  int64_t inc_edits = 0;  // record writes applied in place
  DevBuf status;
  unsigned long long *h_status = nullptr;
  DevBuf snap_dev;
  double *snap_host = nullptr;
  size_t snap_host_bytes = 0;
  int64_t snap_m = 0;
  EnvP env;
  int64_t launches = 0;
  std::string err;
};

namespace {

int fail(sl_ctx *c, int code, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c)
    c->err = buf;
  else
    g_err = buf;
  return code;
}

#define CK(call)                                                        \
  do {                                                                  \
    cudaError_t e_ = (call);                                            \
    if (e_ != cudaSuccess)                                              \
      return fail(c, SL_ECUDA, "%s failed: %s", #call,                  \
                  cudaGetErrorString(e_));                              \
  } while (0)

#define CKL()                                                           \
  do {                                                                  \
    cudaError_t e_ = cudaGetLastError();                                \
    if (e_ != cudaSuccess)                                              \
      return fail(c, SL_ECUDA, "kernel launch failed: %s",              \
                  cudaGetErrorString(e_));                              \
  } while (0)

// ------------------------------------------------------------- pack kernels
template <int P>
__global__ void k_pack_masses(int64_t n, const double *pos, const double *vel,
                              const double *acc, const double *fext,
                              const double *load, const double *mass,
                              const uint8_t *fixed, const uint8_t *alive,
                              const int64_t *slots, void *pos0, void *pos1,
                              void *plo0, void *plo1, float *pmass_o,
                              void *velo, void *acco, void *fexto,
                              void *loado, int64_t *gen_o, uint8_t *alive_o,
                              const int64_t *gen_in, const uint8_t *xflags) {
  using R = typename Tr<P>::R;
  using R4 = typename Tr<P>::R4;
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int64_t i = slots ? slots[r] : r;
  uint32_t fl = 0;
  if (alive[r]) fl |= MF_ALIVE;
  if (fixed[r]) fl |= MF_FIXED;
  const double *ld = load + 3 * r;
  if (__double_as_longlong(ld[0]) | __double_as_longlong(ld[1]) |
      __double_as_longlong(ld[2]))
    fl |= MF_LOAD;
  const double *fe = fext + 3 * r;
  if (__double_as_longlong(fe[0]) | __double_as_longlong(fe[1]) |
      __double_as_longlong(fe[2]))
    fl |= MF_FEXT;
  R4 p;
  p.x = (R)pos[3 * r];
  p.y = (R)pos[3 * r + 1];
  p.z = (R)pos[3 * r + 2];
  p.w = (R)mass[r];
  if constexpr (P == PREC_FP32) {  // compensated: the residuals x - hi
    p.w = (float)(pos[3 * r + 2] - (double)p.z);  // lz in the record
    const float2 l = make_float2((float)(pos[3 * r] - (double)p.x),
                                 (float)(pos[3 * r + 1] - (double)p.y));
    ((float2 *)plo0)[i] = l;
    ((float2 *)plo1)[i] = l;
    pmass_o[i] = (float)mass[r];
  }
  ((R4 *)pos0)[i] = p;
  ((R4 *)pos1)[i] = p;
  R4 v;
  v.x = (R)vel[3 * r];
  v.y = (R)vel[3 * r + 1];
  v.z = (R)vel[3 * r + 2];
  // keep an existing local-constraint flag (set by sl_set_local_constraints)
  if (slots) fl |= flags_of(((R4 *)velo)[i].w) & MF_LC;
  if (xflags && xflags[i]) fl |= MF_SPECIAL;  // layout-derived, still valid
  set_flags(v.w, fl);
  ((R4 *)velo)[i] = v;
  R *a = (R *)acco + 3 * i;
  a[0] = (R)acc[3 * r];
  a[1] = (R)acc[3 * r + 1];
  a[2] = (R)acc[3 * r + 2];
  R4 f;
  f.x = (R)fe[0];
  f.y = (R)fe[1];
  f.z = (R)fe[2];
  f.w = (R)0.0;
  ((R4 *)fexto)[i] = f;
  R *l = (R *)loado + 3 * i;
  l[0] = (R)ld[0];
  l[1] = (R)ld[1];
  l[2] = (R)ld[2];
  gen_o[i] = gen_in[r];
  alive_o[i] = alive[r];
}

// Positions / velocities (/ accelerations) of every mass from host fp64
// columns, the rest of the device state kept: velocity flags, the record's
// mass (fp64 / mixed), f_ext, load (sl_write_state).  Both position
// buffers are written (static masses are never rewritten by a step).
template <int P>
__global__ void k_write_state(int64_t n, const double *pos, const double *vel,
                              const double *acc, void *pos0, void *pos1,
                              void *plo0, void *plo1, void *velb,
                              void *accb) {
  using R = typename Tr<P>::R;
  using R4 = typename Tr<P>::R4;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (pos) {
    R4 p = ((const R4 *)pos0)[i];
    p.x = (R)pos[3 * i];
    p.y = (R)pos[3 * i + 1];
    p.z = (R)pos[3 * i + 2];
    if constexpr (P == PREC_FP32) {
      p.w = (float)(pos[3 * i + 2] - (double)p.z);
      const float2 l = make_float2((float)(pos[3 * i] - (double)p.x),
                                   (float)(pos[3 * i + 1] - (double)p.y));
      ((float2 *)plo0)[i] = l;
      ((float2 *)plo1)[i] = l;
    }
    ((R4 *)pos0)[i] = p;
    ((R4 *)pos1)[i] = p;
  }
  if (vel) {
    R4 v = ((const R4 *)velb)[i];
    v.x = (R)vel[3 * i];
    v.y = (R)vel[3 * i + 1];
    v.z = (R)vel[3 * i + 2];
    ((R4 *)velb)[i] = v;
  }
  if (acc) {
    R *a = (R *)accb + 3 * i;
    a[0] = (R)acc[3 * i];
    a[1] = (R)acc[3 * i + 1];
    a[2] = (R)acc[3 * i + 2];
  }
}

template <int P>
__global__ void k_unpack_masses(int64_t n, const void *posb, const void *plob,
                                const void *velb, const void *accb,
                                const void *fextb, double *pos, double *vel,
                                double *acc, double *fext) {
  using R = typename Tr<P>::R;
  using R4 = typename Tr<P>::R4;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (pos) {
    R4 p = ((const R4 *)posb)[i];
    double x = (double)p.x, y = (double)p.y, z = (double)p.z;
    if constexpr (P == PREC_FP32) {  // hi + lo, exact in fp64
      const float2 l = ((const float2 *)plob)[i];
      x += (double)l.x;
      y += (double)l.y;
      z += (double)p.w;
    }
    pos[3 * i] = x;
    pos[3 * i + 1] = y;
    pos[3 * i + 2] = z;
  }
  if (vel) {
    R4 v = ((const R4 *)velb)[i];
    vel[3 * i] = (double)v.x;
    vel[3 * i + 1] = (double)v.y;
    vel[3 * i + 2] = (double)v.z;
  }
  if (acc) {
    const R *a = (const R *)accb + 3 * i;
    acc[3 * i] = (double)a[0];
    acc[3 * i + 1] = (double)a[1];
    acc[3 * i + 2] = (double)a[2];
  }
  if (fext) {
    R4 f = ((const R4 *)fextb)[i];
    fext[3 * i] = (double)f.x;
    fext[3 * i + 1] = (double)f.y;
    fext[3 * i + 2] = (double)f.z;
  }
}

__global__ void k_set_lc_flags(int64_t n, const int64_t *lc_off, void *velb,
                               int is_double) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool has = lc_off && lc_off[i + 1] > lc_off[i];
  if (is_double) {
    double4 *v = (double4 *)velb + i;
    uint32_t fl = flags_of(v->w);
    set_flags(v->w, has ? (fl | MF_LC) : (fl & ~MF_LC));
  } else {
    float4 *v = (float4 *)velb + i;
    uint32_t fl = flags_of(v->w);
    set_flags(v->w, has ? (fl | MF_LC) : (fl & ~MF_LC));
  }
}

__global__ void k_clear_flag(int64_t n, void *velb, int is_double,
                             uint32_t bit) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (is_double) {
    double4 *v = (double4 *)velb + i;
    set_flags(v->w, flags_of(v->w) & ~bit);
  } else {
    float4 *v = (float4 *)velb + i;
    set_flags(v->w, flags_of(v->w) & ~bit);
  }
}

__global__ void k_set_fext_flags(int64_t n, void *velb, int is_double) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (is_double) {
    double4 *v = (double4 *)velb + i;
    set_flags(v->w, flags_of(v->w) | MF_FEXT);
  } else {
    float4 *v = (float4 *)velb + i;
    set_flags(v->w, flags_of(v->w) | MF_FEXT);
  }
}

// yield threshold exactly as kernels.py:78-81 evaluates it:
// area = ((0.25*pi)*d)*d ; break when |fmag| > y*area.
__device__ __forceinline__ double yield_threshold(double y, double d) {
  if (y == CUDART_INF) return CUDART_INF;
  double area = __dmul_rn(__dmul_rn(__dmul_rn(0.25, CUDART_PI), d), d);
  return __dmul_rn(y, area);
}

template <int P>
__global__ void k_pack_springs(int64_t n, const int64_t *slots,
                               const int64_t *m1, const int64_t *m2,
                               const int64_t *m1gen, const int64_t *m2gen,
                               const double *rest, const double *k,
                               const double *diam, const double *yield,
                               const int8_t *mode, const double *amp,
                               const double *freq, const double *off,
                               const double *per, const uint8_t *alive,
                               const uint8_t *degen, KState S,
                               int64_t *m1g_o, int64_t *m2g_o, int8_t *mode_o,
                               double4 *act_o, uint8_t *degen_o,
                               double *custom_o, int params_only,
                               int layout_valid, const uint8_t *grp_in,
                               uint8_t *grp_o) {
  using F = typename Tr<P>::F;
  using F2 = typename Tr<P>::F2;
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int64_t s = slots ? slots[r] : r;
  grp_o[s] = grp_in[r];
  F2 kl;
  kl.x = (F)k[r];
  kl.y = (F)rest[r];
  ((F2 *)S.kL0)[s] = kl;
  mode_o[s] = mode[r];
  act_o[s] = make_double4(amp[r], freq[r], off[r], per[r]);
  F th = (F)yield_threshold(yield[r], diam[r]);
  ((F *)S.thr)[s] = th;
  if (!params_only) {
    bool al = alive[r] != 0;
    S.ends[s] = al ? make_int2((int)m1[r], (int)m2[r]) : make_int2(-1, -1);
    S.s_alive[s] = alive[r];
    degen_o[s] = degen[r];
    m1g_o[s] = m1gen[r];
    m2g_o[s] = m2gen[r];
    custom_o[s] = 1.0;
  } else if (layout_valid) {
    // keep the incidence copies of (k, L0) and the special bit in sync;
    // the split layout runs grouped sine actuation in its fast path
    bool special = (mode[r] != 0 && !(S.split && grp_in[r] != 0)) ||
                   yield[r] != CUDART_INF || (S.damp && S.damp[s] != 0.0);
    int2 ab = S.ends[s];
    if (special && ab.x >= 0) {
      using R4 = typename Tr<P>::R4;
      S.xflags[ab.x] = 1;
      S.xflags[ab.y] = 1;
      or_flags((R4 *)S.vel + ab.x, MF_SPECIAL);
      or_flags((R4 *)S.vel + ab.y, MF_SPECIAL);
    }
    if (S.split) {
      if (ab.x >= 0 && S.e1[s] >= 0) {
        ((F2 *)S.sp_kl)[S.sp_ekl[s]] = kl;
        if (S.sp_actc) {
          S.sp_actc[S.sp_ekl[s]] = act_cell(off[r], freq[r], per[r], grp_in[r]);
          S.sp_acto[S.sp_ekl[s]] = off[r];
        }
      }
      return;
    }
    int64_t es[2] = {S.e1[s], S.e2[s]};
    for (int q = 0; q < 2; q++) {
      int64_t e = es[q];
      if (e < 0) continue;
      ((F2 *)S.ent_kL0)[e] = kl;
      uint32_t j = S.ent_j[e];
      S.ent_j[e] = special ? (j | EJ_SPECIAL) : (j & ~EJ_SPECIAL);
    }
  }
}

__global__ void k_kill_springs(int64_t n, const int64_t *slots, KState S,
                               int layout_valid) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int64_t s = slots[r];
  S.ends[s] = make_int2(-1, -1);
  S.s_alive[s] = 0;
  if (layout_valid) kill_entries(S, s);
}

__global__ void k_set_custom(int64_t n, const int64_t *slots,
                             const double *f, double *custom) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) custom[slots[r]] = f[r];
}

// Lazy endpoint invalidation, kernels.py:37-45: an alive spring whose
// endpoint is dead or was re-issued (generation mismatch) dies and counts as
// invalid.  Deletions only happen at pause points (store.py:221-224), so
// running this once before the first step after an edit is equivalent to the
// reference's per-step check.
__global__ void k_validate(KState S, const uint8_t *m_alive,
                           const int64_t *m_gen, const int64_t *m1gen,
                           const int64_t *m2gen, int layout_valid) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S.s_n) return;
  int2 ab = S.ends[s];
  if (ab.x < 0) return;
  if (m_alive[ab.x] && m_alive[ab.y] && m_gen[ab.x] == m1gen[s] &&
      m_gen[ab.y] == m2gen[s])
    return;
  count_spring(S, 1, s);
  S.ends[s] = make_int2(-1, -1);
  S.s_alive[s] = 0;
  if (layout_valid) kill_entries(S, s);
}

// ------------------------------------------------------- diagnostics
// position of mass i in fp64 (fp32 mode: hi + lo)
template <int P>
__device__ __forceinline__ double3 pos_f64(const KState &S, int cur,
                                           int64_t i) {
  using R4 = typename Tr<P>::R4;
  const R4 p = ((const R4 *)S.pos[cur])[i];
  double3 r = make_double3((double)p.x, (double)p.y, (double)p.z);
  if constexpr (P == PREC_FP32) {
    const float2 l = ((const float2 *)S.plo[cur])[i];
    r.x += (double)l.x;
    r.y += (double)l.y;
    r.z += (double)p.w;
  }
  return r;
}
// engine.mechanical_energy (engine.py:366-389) on the device: per-block
// partial sums of m |v|^2, m (x . g) and k (|d| - f L0)^2 in fp64 (fixed
// block tree order), finished on the host in block order -- deterministic.
constexpr int DIAG_BLOCKS = 592, DIAG_THREADS = 256;
template <int P>
__global__ void __launch_bounds__(DIAG_THREADS)
    k_energy(const KState S, int cur, double gx, double gy, double gz,
             double sim_t, double *part) {
  using R4 = typename Tr<P>::R4;
  using F2 = typename Tr<P>::F2;
  __shared__ double red[3][DIAG_THREADS];
  double ke = 0.0, gp = 0.0, sp = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t i = t0; i < S.m_n; i += stride) {
    const R4 v = ((const R4 *)S.vel)[i];
    if (!(flags_of(v.w) & MF_ALIVE)) continue;
    const double3 p = pos_f64<P>(S, cur, i);
    const double m = (double)mass_of<P>(S, ((const R4 *)S.pos[cur])[i], i);
    ke += m * ((double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z);
    gp += m * (p.x * gx + p.y * gy + p.z * gz);
  }
  for (int64_t s = t0; s < S.s_n; s += stride) {
    const int2 e = S.ends[s];
    if (e.x < 0) continue;
    const double3 a = pos_f64<P>(S, cur, e.x), b = pos_f64<P>(S, cur, e.y);
    const double dx = b.x - a.x, dy = b.y - a.y, dz = b.z - a.z;
    const double len = sqrt(dx * dx + dy * dy + dz * dz);
    const F2 kl = ((const F2 *)S.kL0)[s];
    const double f = S.mode[s] ? act_factor(S, s, sim_t) : 1.0;
    const double x = len - f * (double)kl.y;
    sp += (double)kl.x * (x * x);
  }
  red[0][threadIdx.x] = ke;
  red[1][threadIdx.x] = gp;
  red[2][threadIdx.x] = sp;
  __syncthreads();
  for (int h = DIAG_THREADS / 2; h; h >>= 1) {
    if ((int)threadIdx.x < h)
      for (int q = 0; q < 3; q++) red[q][threadIdx.x] += red[q][threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x < 3) part[3 * blockIdx.x + threadIdx.x] = red[threadIdx.x][0];
}

// engine.spring_loads (engine.py:392-412) minus the host-side stress: per
// slot the length and |k (|d| - f L0)| (NaN for dead slots)
template <int P>
__global__ void k_spring_loads(const KState S, int cur, double sim_t,
                               double *len_out, double *fmag_out) {
  using R4 = typename Tr<P>::R4;
  using F2 = typename Tr<P>::F2;
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S.s_n) return;
  const int2 e = S.ends[s];
  if (e.x < 0) {
    len_out[s] = fmag_out[s] = CUDART_NAN;
    return;
  }
  const double3 a = pos_f64<P>(S, cur, e.x), b = pos_f64<P>(S, cur, e.y);
  const double dx = b.x - a.x, dy = b.y - a.y, dz = b.z - a.z;
  const double len = sqrt(dx * dx + dy * dy + dz * dz);
  const F2 kl = ((const F2 *)S.kL0)[s];
  const double f = S.mode[s] ? act_factor(S, s, sim_t) : 1.0;
  len_out[s] = len;
  fmag_out[s] = fabs((double)kl.x * (len - f * (double)kl.y));
}

// ------------------------------------------------------- layout build kernels
// Two incidence records per alive spring: (owner m1, 2s) and (owner m2,
// 2s+1) -- the owner array of engine._refresh_slotted_layout.  A stable
// radix sort by owner leaves each mass's records in ascending slot order.
__global__ void k_make_keys(int64_t s_n, const int2 *ends, uint32_t m_n,
                            uint32_t *keys, uint32_t *vals, uint32_t *deg) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= s_n) return;
  int2 ab = ends[s];
  bool al = ab.x >= 0;
  keys[2 * s] = al ? (uint32_t)ab.x : m_n;
  keys[2 * s + 1] = al ? (uint32_t)ab.y : m_n;
  vals[2 * s] = (uint32_t)(2 * s);
  vals[2 * s + 1] = (uint32_t)(2 * s + 1);
  if (al) {
    atomicAdd(deg + ab.x, 1u);
    atomicAdd(deg + ab.y, 1u);
  }
}

// per-slice width = max degree of its 32 masses; entries = 32 * width
__global__ void k_slice_width(int64_t m_n, const uint32_t *deg,
                              int64_t n_slices, int64_t *slice_entries) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t w = i >> 5;
  if (w >= n_slices) return;
  uint32_t d = i < m_n ? deg[i] : 0u;
  for (int o = 16; o; o >>= 1) d = max(d, __shfl_xor_sync(0xffffffffu, d, o));
  if ((i & 31) == 0) slice_entries[w] = 32 * (int64_t)d;
}

// rank of each sorted record within its owner's run
__global__ void k_owner_start(int64_t n, const uint32_t *keys, uint32_t m_n,
                              int64_t *start) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  uint32_t k = keys[p];
  if (k >= m_n) return;
  if (p == 0 || keys[p - 1] != k) start[k] = p;
}

template <int P>
__global__ void k_fill_layout(int64_t n, const uint32_t *keys,
                              const uint32_t *vals, uint32_t m_n,
                              const int64_t *start, KState S,
                              uint32_t *ent_j, void *ent_kl, int32_t *ent_s,
                              int64_t *e1, int64_t *e2) {
  using F = typename Tr<P>::F;
  using F2 = typename Tr<P>::F2;
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  uint32_t i = keys[p];
  if (i >= m_n) return;
  uint32_t v = vals[p];
  int64_t s = v >> 1;
  int side = v & 1;
  int64_t rank = p - start[i];
  int64_t e = S.slice_ptr[i >> 5] + 32 * rank + (i & 31);
  int2 ab = S.ends[s];
  uint32_t other = side ? (uint32_t)ab.x : (uint32_t)ab.y;
  bool special = S.mode[s] != 0 ||
                 ((const F *)S.thr)[s] != (F)CUDART_INF ||
                 (S.damp && S.damp[s] != 0.0);
  ent_j[e] = other | (side ? EJ_M2 : 0u) | (special ? EJ_SPECIAL : 0u);
  if (special) {
    S.xflags[i] = 1;
    or_flags((typename Tr<P>::R4 *)S.vel + i, MF_SPECIAL);
  }
  ((F2 *)ent_kl)[e] = ((const F2 *)S.kL0)[s];
  ent_s[e] = (int32_t)s;
  (side ? e2 : e1)[s] = e;
}


// ------------------------------------------------ split layout build kernels
// Records: (key 2*m1, s) for the A entry, (key 2*m2+1, s) for the B entry;
// a stable radix sort by key groups each mass's A then B records, each in
// ascending spring slot; the rank within a group is the entry row.
__global__ void k_split_keys(int64_t s_n, const int2 *ends, uint32_t m_n,
                             uint32_t *keys, uint32_t *vals, uint32_t *deg_a,
                             uint32_t *deg_b) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= s_n) return;
  int2 ab = ends[s];
  bool al = ab.x >= 0;
  keys[2 * s] = al ? 2u * (uint32_t)ab.x : 2u * m_n;
  keys[2 * s + 1] = al ? 2u * (uint32_t)ab.y + 1u : 2u * m_n;
  vals[2 * s] = (uint32_t)s;
  vals[2 * s + 1] = (uint32_t)s;
  if (al) {
    atomicAdd(deg_a + ab.x, 1u);
    atomicAdd(deg_b + ab.y, 1u);
  }
}

// per-slice section widths; meta[0..1] = widest A / B, meta[2] = streamed
// entries (sum over slices of 32 * (wA + wB))
__global__ void k_split_widths(int64_t m_n, const uint32_t *deg_a,
                               const uint32_t *deg_b, int64_t n_slices,
                               uint32_t *sp_w, unsigned long long *meta) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t w = i >> 5;
  if (w >= n_slices) return;
  uint32_t da = i < m_n ? deg_a[i] : 0u, db = i < m_n ? deg_b[i] : 0u;
  for (int o = 16; o; o >>= 1) {
    da = max(da, __shfl_xor_sync(0xffffffffu, da, o));
    db = max(db, __shfl_xor_sync(0xffffffffu, db, o));
  }
  if ((i & 31) == 0) {
    sp_w[w] = min(da, 0xFFFFu) | (min(db, 0xFFFFu) << 16);
    atomicMax(meta + 0, (unsigned long long)da);
    atomicMax(meta + 1, (unsigned long long)db);
    atomicAdd(meta + 2, 32ull * (da + db));
  }
}

__global__ void k_split_init(int64_t n, int rows, int wa_stride,
                             uint32_t sent, uint32_t nul, uint32_t *sp_j) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  int row = (int)((e >> 5) % rows);
  sp_j[e] = row < wa_stride ? sent : nul;
}

template <int P>
__global__ void k_split_sentinel(void *pos0, void *pos1, int64_t m_pad) {
  using R = typename Tr<P>::R;
  using R4 = typename Tr<P>::R4;
  int q = threadIdx.x;
  R4 p;
  p.x = p.y = p.z = (R)SENTINEL_POS;
  p.w = (R)0.0;
  ((R4 *)pos0)[m_pad + q] = p;
  ((R4 *)pos1)[m_pad + q] = p;
}

template <int P>
__global__ void k_split_fill(int64_t n, const uint32_t *keys,
                             const uint32_t *vals, uint32_t kbound,
                             const int64_t *start, KState S, uint32_t *sp_j,
                             void *sp_kl, int32_t *sp_s, uint32_t *sp_ekl,
                             int64_t *e1, int64_t *e2, int pass,
                             float4 *sp_actc, double *sp_acto,
                             const uint8_t *grp) {
  using F = typename Tr<P>::F;
  using F2 = typename Tr<P>::F2;
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  uint32_t key = keys[p];
  if (key >= kbound || (int)(key & 1u) != pass) return;
  uint32_t owner = key >> 1;
  int64_t s = vals[p];
  int64_t r = p - start[key];
  int64_t sl = owner >> 5, lane = owner & 31;
  int2 ab = S.ends[s];
  if (pass == 0) {
    int64_t e = (sl * S.sp_rows + r) * 32 + lane;
    uint32_t kli = (uint32_t)((sl << (S.sp_a + 5)) | (r << 5) | lane);
    sp_j[e] = (uint32_t)ab.y;
    ((F2 *)sp_kl)[kli] = ((const F2 *)S.kL0)[s];
    if (sp_actc) {
      const double4 ac = S.act[s];
      sp_actc[kli] = act_cell(ac.z, ac.y, ac.w, grp[s]);
      sp_acto[kli] = ac.z;
    }
    sp_s[e] = (int32_t)s;
    sp_ekl[s] = kli;
    e1[s] = e;
  } else {
    int64_t e = (sl * S.sp_rows + ((int64_t)1 << S.sp_a) + r) * 32 + lane;
    sp_j[e] = sp_ekl[s];
    sp_s[e] = (int32_t)s;
    e2[s] = e;
  }
  bool special = (S.mode[s] != 0 && grp[s] == 0) ||
                 ((const F *)S.thr)[s] != (F)CUDART_INF ||
                 (S.damp && S.damp[s] != 0.0);
  if (special) {
    S.xflags[owner] = 1;
    or_flags((typename Tr<P>::R4 *)S.vel + owner, MF_SPECIAL);
  }
}

// O(edits) topology sync on a live split layout (sl_split.cuh): the
// written slots (created, re-used or re-wired springs -- DeviceMirror's
// journal replay) get their A / B cells in place, from the free rows of
// their endpoints' lanes (the device-side free list: a dead or padding cell
// is sent / nul), instead of a full re-index.  One warp, slots in order; a
// lane probes one row.  Cells of the slot's previous wiring are released;
// a slot whose endpoints did not change keeps its cells and gets the new
// (k, L0) (+ actuation cell).  The tiles of every touched slice are
// listed for the window layout's partial rebuild.  fail = 1: a lane has no
// free row within the layout's widths -- the caller re-indexes everything.
template <int P>
__global__ void k_split_insert(int64_t n, const int64_t *slots, KState S,
                               int cap_wa, int cap_wb, int tt,
                               float4 *sp_actc, double *sp_acto,
                               const uint8_t *grp, int32_t *tiles,
                               int *fail) {
  using F = typename Tr<P>::F;
  using F2 = typename Tr<P>::F2;
  const int lane = threadIdx.x;
  const int a = S.sp_a;
  const int64_t rows = S.sp_rows, wa_stride = (int64_t)1 << a;
  const uint32_t sent = S.sp_sent, nul = S.sp_null;
  // the layout arrays, writable here (KState carries them read-only)
  int64_t *E1 = (int64_t *)S.e1, *E2 = (int64_t *)S.e2;
  int32_t *SPS = (int32_t *)S.sp_s;
  uint32_t *SPW = (uint32_t *)S.sp_w, *EKL = (uint32_t *)S.sp_ekl;
  F2 *SKL = (F2 *)S.sp_kl;
  auto cell = [&](int64_t sl, int64_t r, int ln) {
    return (sl * rows + r) * 32 + ln;
  };
  auto kl_of = [&](int64_t e) {  // kl index of A cell e
    const int64_t sl = e / (rows * 32), rem = e - sl * rows * 32;
    return (uint32_t)((sl << (a + 5)) | rem);
  };
  // lowest row r in [r0, r0 + cap) of lane ln of slice sl holding `free_w`
  auto probe = [&](int64_t sl, int ln, int64_t r0, int cap,
                   uint32_t free_w) -> int {
    for (int base = 0; base < cap; base += 32) {
      const int r = base + lane;
      const bool ok = r < cap && S.sp_j[cell(sl, r0 + r, ln)] == free_w;
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      if (m) return base + __ffs(m) - 1;
    }
    return -1;
  };
  for (int64_t q = 0; q < n; q++) {
    const int64_t s = slots[q];
    const int2 ab = S.ends[s];
    const int64_t eA = S.e1[s], eB = S.e2[s];
    const bool ownA = eA >= 0 && S.sp_s[eA] == (int32_t)s && S.sp_j[eA] != sent;
    const bool ownB = eB >= 0 && S.sp_s[eB] == (int32_t)s && S.sp_j[eB] != nul;
    int32_t t0 = -1, t1 = -1, t2 = -1, t3 = -1;
    int32_t g0 = -1, g1 = -1, g2 = -1, g3 = -1;  // fused groups touched
    // mass of cell e: its slice's lane
    auto mass_of_cell = [&](int64_t e) {
      return (e / (rows * 32)) * 32 + (e & 31);
    };
    if (ownA) t0 = (int32_t)(eA / (rows * 32) / tt);
    if (ownB) t1 = (int32_t)(eB / (rows * 32) / tt);
    if (S.fz_gid) {
      if (ownA) g0 = S.fz_gid[mass_of_cell(eA)];
      if (ownB) g1 = S.fz_gid[mass_of_cell(eB)];
      if (ab.x >= 0 && S.fz_gid[ab.x] != S.fz_gid[ab.y]) {
        // the edit joins two fused groups: their packing changes
        if (lane == 0) *fail = 1;
        return;
      }
    }
    const bool same = ab.x >= 0 && ownA && ownB &&
                      (eA & 31) == (ab.x & 31) &&
                      eA / (rows * 32) == (ab.x >> 5) &&
                      S.sp_j[eA] == (uint32_t)ab.y &&
                      (eB & 31) == (ab.y & 31) &&
                      eB / (rows * 32) == (ab.y >> 5);
    int rA = -1, rB = -1;
    if (ab.x >= 0 && !same) {
      rA = probe(ab.x >> 5, ab.x & 31, 0, cap_wa, sent);
      rB = probe(ab.y >> 5, ab.y & 31, wa_stride, cap_wb, nul);
      if (rA < 0 || rB < 0) {
        if (lane == 0) *fail = 1;
        return;
      }
    }
    if (lane == 0) {
      if (!same) {  // release the previous wiring's cells
        if (ownA) {
          S.sp_j[eA] = sent;
          SKL[kl_of(eA)] = F2{};
          SPS[eA] = -1;
        }
        if (ownB) {
          S.sp_j[eB] = nul;
          SPS[eB] = -1;
        }
        E1[s] = -1;
        E2[s] = -1;
      }
      if (ab.x >= 0) {
        const int64_t sl1 = ab.x >> 5, sl2 = ab.y >> 5;
        int64_t ea = eA, eb = eB;
        if (!same) {
          ea = cell(sl1, rA, ab.x & 31);
          eb = cell(sl2, wa_stride + rB, ab.y & 31);
        }
        const uint32_t kli = kl_of(ea);
        SKL[kli] = ((const F2 *)S.kL0)[s];
        if (sp_actc) {
          const double4 ac = S.act[s];
          sp_actc[kli] = act_cell(ac.z, ac.y, ac.w, grp[s]);
          sp_acto[kli] = ac.z;
        }
        if (!same) {
          S.sp_j[ea] = (uint32_t)ab.y;
          SPS[ea] = (int32_t)s;
          S.sp_j[eb] = kli;
          SPS[eb] = (int32_t)s;
          EKL[s] = kli;
          E1[s] = ea;
          E2[s] = eb;
          uint32_t w1 = S.sp_w[sl1];
          if ((uint32_t)rA + 1 > (w1 & 0xFFFFu))
            w1 = (w1 & 0xFFFF0000u) | (uint32_t)(rA + 1);
          SPW[sl1] = w1;
          uint32_t w2 = S.sp_w[sl2];
          if ((uint32_t)rB + 1 > (w2 >> 16))
            w2 = (w2 & 0xFFFFu) | ((uint32_t)(rB + 1) << 16);
          SPW[sl2] = w2;
        }
        t2 = (int32_t)(sl1 / tt);
        t3 = (int32_t)(sl2 / tt);
        if (S.fz_gid) {
          g2 = S.fz_gid[ab.x];
          g3 = S.fz_gid[ab.y];
        }
        const bool special = (S.mode[s] != 0 && grp[s] == 0) ||
                             ((const F *)S.thr)[s] != (F)CUDART_INF ||
                             (S.damp && S.damp[s] != 0.0);
        if (special) {
          S.xflags[ab.x] = 1;
          S.xflags[ab.y] = 1;
          or_flags((typename Tr<P>::R4 *)S.vel + ab.x, MF_SPECIAL);
          or_flags((typename Tr<P>::R4 *)S.vel + ab.y, MF_SPECIAL);
        }
      }
      int32_t *tq = tiles + 8 * q;
      tq[0] = t0;
      tq[1] = t1;
      tq[2] = t2;
      tq[3] = t3;
      tq[4] = g0;
      tq[5] = g1;
      tq[6] = g2;
      tq[7] = g3;
    }
    __syncwarp();
  }
}

// O(edits) topology sync on the EXACT layout (fp64 parity mode): a mass's
// entries are kept in ascending spring slot (the reference's serial
// order), so an entry is inserted at its sorted row -- the live entries
// between it and the nearest free row (dead or padding) move over by one
// row, their springs' e1 / e2 following.  A written slot whose wiring is
// unchanged gets its (k, L0) / special bit refreshed in place; a re-wired
// or dead slot's entries become dead.  One warp, slots in order; the
// touched window tiles are listed (the fp64 window is re-derived for
// them).  fail = 1: a lane has no free row within its slice width.
template <int P>
__global__ void k_exact_insert(int64_t n, const int64_t *slots, KState S,
                               int tt, int32_t *tiles, int *fail) {
  using F = typename Tr<P>::F;
  using F2 = typename Tr<P>::F2;
  const int lane = threadIdx.x;
  int64_t *E1 = (int64_t *)S.e1, *E2 = (int64_t *)S.e2;
  int32_t *ES = (int32_t *)S.ent_s;
  F2 *EK = (F2 *)S.ent_kL0;
  auto mine = [&](int64_t e, int64_t s) {  // entry e is still s's
    return e >= 0 && ES[e] == (int32_t)s;
  };
  auto owned = [&](int64_t e, int64_t s) {  // ... and alive
    return mine(e, s) && !(S.ent_j[e] & EJ_DEAD);
  };
  // insert the entry of spring s at mass i (side 0: m1, 1: m2)
  auto insert = [&](int64_t s, int64_t i, uint32_t ej) -> int64_t {
    const int64_t sl = i >> 5, l = i & 31;
    const int64_t base = S.slice_ptr[sl];
    const int width = (int)((S.slice_ptr[sl + 1] - base) >> 5);
    // rows: live with slot < s (before), live with slot > s, free
    int p = width, f_after = -1, f_before = -1;
    for (int b = 0; b < width; b += 32) {
      const int r = b + lane;
      bool live = false, after = false;
      if (r < width) {
        const int64_t e = base + 32 * (int64_t)r + l;
        live = !(S.ent_j[e] & EJ_DEAD);
        after = live && ES[e] > (int32_t)s;
      }
      const unsigned ma = __ballot_sync(0xffffffffu, after);
      if (ma && p == width) p = b + __ffs(ma) - 1;
    }
    for (int b = 0; b < width; b += 32) {
      // first free row at or after p, last free row before p
      const int r = b + lane;
      const bool fr = r < width &&
                      (S.ent_j[base + 32 * (int64_t)r + l] & EJ_DEAD);
      const unsigned fa = __ballot_sync(0xffffffffu, fr && r >= p);
      const unsigned fb = __ballot_sync(0xffffffffu, fr && r < p);
      if (fa && f_after < 0) f_after = b + __ffs(fa) - 1;
      if (fb) f_before = b + 31 - __clz(fb);
    }
    if (f_after < 0 && f_before < 0) return -1;
    int64_t at;
    if (lane == 0) {
      auto mv = [&](int from, int to) {  // move a live entry one row
        const int64_t ef = base + 32 * (int64_t)from + l;
        const int64_t et = base + 32 * (int64_t)to + l;
        const uint32_t jr = S.ent_j[ef];
        const int32_t so = ES[ef];
        S.ent_j[et] = jr;
        EK[et] = EK[ef];
        ES[et] = so;
        ((jr & EJ_M2) ? E2 : E1)[so] = et;
      };
      if (f_after >= 0) {
        for (int r = f_after; r > p; r--) mv(r - 1, r);
        at = base + 32 * (int64_t)p + l;
      } else {
        for (int r = f_before; r < p - 1; r++) mv(r + 1, r);
        at = base + 32 * (int64_t)(p - 1) + l;
      }
      S.ent_j[at] = ej;
      EK[at] = ((const F2 *)S.kL0)[s];
      ES[at] = (int32_t)s;
    }
    return __shfl_sync(0xffffffffu, lane == 0 ? at : 0, 0);
  };
  for (int64_t q = 0; q < n; q++) {
    const int64_t s = slots[q];
    const int2 ab = S.ends[s];
    const int64_t eA = E1[s], eB = E2[s];
    const bool ownA = owned(eA, s), ownB = owned(eB, s);
    int32_t t[4] = {-1, -1, -1, -1};
    const bool special = ab.x >= 0 &&
                         (S.mode[s] != 0 ||
                          ((const F *)S.thr)[s] != (F)CUDART_INF ||
                          (S.damp && S.damp[s] != 0.0));
    // entry e sits in mass i's column: i's slice range, i's lane
    auto at_mass = [&](int64_t e, int64_t i) {
      return (e & 31) == (i & 31) && e >= S.slice_ptr[i >> 5] &&
             e < S.slice_ptr[(i >> 5) + 1];
    };
    const bool same = ab.x >= 0 && ownA && ownB &&
                      (S.ent_j[eA] & EJ_MASK) == (uint32_t)ab.y &&
                      (S.ent_j[eB] & EJ_MASK) == (uint32_t)ab.x &&
                      at_mass(eA, ab.x) && at_mass(eB, ab.y);
    if (same) {
      if (lane == 0) {
        const F2 kl = ((const F2 *)S.kL0)[s];
        EK[eA] = kl;
        EK[eB] = kl;
        const uint32_t sp = special ? EJ_SPECIAL : 0u;
        S.ent_j[eA] = (S.ent_j[eA] & ~EJ_SPECIAL) | sp;
        S.ent_j[eB] = (S.ent_j[eB] & ~EJ_SPECIAL) | sp;
      }
    } else {
      if (lane == 0) {
        // the previous wiring's entries (live, or killed since: their
        // partner fields still name the old endpoints, whose tiles the
        // window re-derives) become dead and unowned
        int2 old = make_int2(-1, -1);
        if (mine(eA, s)) {
          old.y = (int)(S.ent_j[eA] & EJ_MASK);
          S.ent_j[eA] |= EJ_DEAD;
          ES[eA] = -1;
        }
        if (mine(eB, s)) {
          old.x = (int)(S.ent_j[eB] & EJ_MASK);
          S.ent_j[eB] |= EJ_DEAD;
          ES[eB] = -1;
        }
        E1[s] = -1;
        E2[s] = -1;
        t[0] = old.x >= 0 ? (int32_t)((old.x >> 5) / tt) : -1;
        t[1] = old.y >= 0 ? (int32_t)((old.y >> 5) / tt) : -1;
      }
      __syncwarp();
      if (ab.x >= 0) {
        const uint32_t sp = special ? EJ_SPECIAL : 0u;
        const int64_t a1 = insert(s, ab.x, (uint32_t)ab.y | sp);
        __syncwarp();
        const int64_t a2 =
            a1 < 0 ? -1 : insert(s, ab.y, (uint32_t)ab.x | EJ_M2 | sp);
        if (a1 < 0 || a2 < 0) {
          if (lane == 0) *fail = 1;
          return;
        }
        if (lane == 0) {
          E1[s] = a1;
          E2[s] = a2;
        }
      }
    }
    if (lane == 0) {
      if (ab.x >= 0) {
        t[2] = (int32_t)((ab.x >> 5) / tt);
        t[3] = (int32_t)((ab.y >> 5) / tt);
        if (special) {
          S.xflags[ab.x] = 1;
          S.xflags[ab.y] = 1;
          or_flags((typename Tr<P>::R4 *)S.vel + ab.x, MF_SPECIAL);
          or_flags((typename Tr<P>::R4 *)S.vel + ab.y, MF_SPECIAL);
        }
      }
      int32_t *tq = tiles + 8 * q;
      for (int u = 0; u < 4; u++) tq[u] = t[u];
    }
    __syncwarp();
  }
}

KState make_state(sl_ctx *c) {
  KState S;
  memset(&S, 0, sizeof S);
  S.m_n = c->m_n;
  S.s_n = c->s_n;
  S.pos[0] = c->pos[0].p;
  S.pos[1] = c->pos[1].p;
  S.plo[0] = c->prec == PREC_FP32 ? c->plo[0].p : nullptr;
  S.plo[1] = c->prec == PREC_FP32 ? c->plo[1].p : nullptr;
  S.pmass = c->prec == PREC_FP32 ? c->pmass.as<float>() : nullptr;
  S.vel = c->vel.p;
  S.acc = c->acc.p;
  S.fext = c->fext.p;
  S.load = c->load.p;
  S.lc_off = c->has_lc ? c->lc_off.as<int64_t>() : nullptr;
  S.lc_kind = c->lc_kind.as<int8_t>();
  S.lc_vec = c->lc_vec.as<double>();
  S.ends = c->ends.as<int2>();
  S.kL0 = c->kL0.p;
  S.s_alive = c->s_alive.as<uint8_t>();
  S.s_degen = c->s_degen.as<uint8_t>();
  S.mode = c->mode.as<int8_t>();
  S.act = c->act.as<double4>();
  S.thr = c->thr.p;
  S.custom = c->custom.as<double>();
  S.damp = c->has_damping ? c->damp.as<double>() : nullptr;
  S.slice_ptr = c->slice_ptr.as<int64_t>();
  S.ent_j = c->ent_j.as<uint32_t>();
  S.ent_kL0 = c->ent_kL0.p;
  S.ent_s = c->ent_s.as<int32_t>();
  S.e1 = c->layout_valid ? c->e1.as<int64_t>() : nullptr;
  S.e2 = c->layout_valid ? c->e2.as<int64_t>() : nullptr;
  S.status = c->status.as<unsigned long long>();
  S.xflags = c->xflags.as<uint8_t>();
  S.fsz8 = c->fsz == 8;
  S.ghost = c->has_ghost ? c->ghost.as<uint8_t>() : nullptr;
  S.halo = c->halo_on ? c->halo_desc.as<HaloDesc>() : nullptr;
  S.self = c->kdev.as<KState>();
  S.split = c->layout_valid && c->split;
  if (c->split) {
    S.sp_a = c->sp_a;
    S.sp_rows = c->sp_rows;
    const int64_t m_pad = (c->m_n + 31) / 32 * 32;
    S.sp_sent = (uint32_t)m_pad;
    S.sp_null = (uint32_t)((m_pad / 32) << (c->sp_a + 5));
    S.sp_j = c->sp_j.as<uint32_t>();
    S.sp_kl = c->sp_kl.p;
    S.sp_s = c->sp_s.as<int32_t>();
    S.sp_w = c->sp_w.as<uint32_t>();
    S.sp_ekl = c->sp_ekl.as<uint32_t>();
    const bool act = c->agrp.n > 1;
    S.sp_actc = act ? c->sp_actc.as<float4>() : nullptr;
    S.sp_acto = act ? c->sp_acto.as<double>() : nullptr;
    if (c->fz_ok) {
      S.fz_code = c->fz_code.as<uint8_t>();
      S.fz_epos = c->fz_epos.as<uint16_t>();
      S.fz_gid = c->fz_gid.as<int32_t>();
      S.fz_gstart = c->fz_gstart.as<int32_t>();
      S.fz_zero = c->fz_zero.as<uint8_t>();
      S.fz_rows = c->fcfg.ra + c->fcfg.rb;
      S.fz_ra = c->fcfg.ra;
      S.fz_maxm = c->fcfg.maxm;
    }
    if (c->win) {
      S.win_blk = c->win_blk.as<unsigned char>();
      S.win_zero = c->win_zero.as<uint8_t>();
      S.win_sb = c->wcfg.bl.slice_bytes;
      S.win_tt = c->wcfg.tile_slices;
    }
  } else if (c->win && c->prec == PREC_FP64) {  // parity-mode window
    S.win_blk = c->win_blk.as<unsigned char>();
    S.win_sb = c->wcfg.bl.slice_bytes;
  }
  return S;
}

template <class T>
int stage_copy(sl_ctx *c, size_t &off, const T *host, int64_t count,
               const T **dev) {
  size_t bytes = sizeof(T) * (size_t)count;
  off = (off + 255) & ~(size_t)255;
  if (!host || count == 0) {
    *dev = nullptr;
    return SL_OK;
  }
  *dev = (const T *)((char *)c->stage.p + off);
  CK(cudaMemcpyAsync((void *)*dev, host, bytes, cudaMemcpyHostToDevice,
                     c->st));
  off += bytes;
  return SL_OK;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

int ensure_masses(sl_ctx *c, int64_t m_n) {
  size_t r4 = 4 * c->rsz;
  m_n = (m_n + 31) / 32 * 32;  // bulk copies move whole 32-mass slices
  // + one slice of sentinel records (split layout's dead / padding target)
  for (int b = 0; b < 2; b++) CK(c->pos[b].ensure(r4 * (m_n + 32)));
  if (c->prec == PREC_FP32)  // low parts; padding / sentinel rows stay 0
    for (int b = 0; b < 2; b++) {
      CK(c->plo[b].ensure(8 * (m_n + 32)));
      CK(cudaMemsetAsync(c->plo[b].p, 0, 8 * (m_n + 32), c->st));
      CK(c->pmass.ensure(4 * (m_n + 32)));
    }
  // padded to whole slices (+32): the window kernels bulk-copy whole slices
  // of velocity records; the padding reads as dead masses (flags 0)
  CK(c->vel.ensure(r4 * (m_n + 32)));
  CK(cudaMemsetAsync((char *)c->vel.p + r4 * m_n, 0, r4 * 32, c->st));
  CK(c->acc.ensure(3 * c->rsz * m_n));
  CK(c->fext.ensure(r4 * m_n));
  CK(c->load.ensure(3 * c->rsz * m_n));
  CK(c->m_gen.ensure(8 * m_n));
  CK(c->m_alive.ensure(m_n));
  CK(c->xflags.ensure(m_n + 1));
  return SL_OK;
}

int ensure_springs(sl_ctx *c, int64_t s_n) {
  CK(c->ends.ensure(8 * s_n));
  CK(c->kL0.ensure(2 * c->fsz * s_n));
  CK(c->s_alive.ensure(s_n));
  CK(c->s_degen.ensure(s_n));
  CK(c->mode.ensure(s_n));
  CK(c->act.ensure(32 * s_n));
  CK(c->thr.ensure(c->fsz * s_n));
  CK(c->custom.ensure(8 * s_n));
  CK(c->m1gen.ensure(8 * s_n));
  CK(c->m2gen.ensure(8 * s_n));
  CK(c->s_grp.ensure(s_n));
  return SL_OK;
}

// Size the per-warp shared-memory rings of the TMA kernel for the widest
// slice; one persistent CTA per SM with as many warps as fit.
void configure_tma(sl_ctx *c) {
  c->tma_warps = 0;
  if (!c->tma_enabled || c->n_slices == 0 || c->max_width == 0) return;
  const size_t f2 = 2 * c->fsz;
  // two 32-mass blocks (pos, vel) + entry words + (k, L0) pairs
  const size_t stage = 2 * 32 * 4 * c->rsz + (size_t)c->max_width * 32 * (4 + f2);
  const size_t per_warp = 2 * stage + 16;
  int warps = (int)std::min<size_t>(12, (size_t)c->smem_optin / per_warp);
  if (warps < 2) return;  // hub masses: fall back to the plain kernel
  c->tma.n_slices = c->n_slices;
  c->tma.cap_w = (int)c->max_width;
  c->tma.warps = warps;
  c->tma.stage_bytes = (uint32_t)stage;
  int64_t ctas = (c->n_slices + warps - 1) / warps;
  c->tma_grid = (int)std::min<int64_t>(ctas, c->sm_count);
  if (launchers(c->prec).tma_setup((int)(warps * per_warp)) != 0) return;
  c->tma_warps = warps;
}

int build_exact_layout(sl_ctx *c) {
  const int64_t m_n = c->m_n, s_n = c->s_n;
  if (m_n > (int64_t)EJ_MASK)
    return fail(c, SL_EUNSUPPORTED, "too many masses for one context (%lld)",
                (long long)m_n);
  if (2 * s_n >= (int64_t)0x7fffffff)
    return fail(c, SL_EUNSUPPORTED, "too many springs for one context");
  const int64_t n_slices = (m_n + 31) / 32;
  const int64_t n_rec = 2 * s_n;
  CK(c->deg.ensure(4 * (m_n + 1)));
  CK(c->width.ensure(8 * (n_slices + 1)));
  CK(c->slice_ptr.ensure(8 * (n_slices + 1)));
  CK(c->e1.ensure(8 * s_n));
  CK(c->e2.ensure(8 * s_n));
  CK(cudaMemsetAsync(c->deg.p, 0, 4 * (m_n + 1), c->st));
  CK(cudaMemsetAsync(c->e1.p, 0xFF, 8 * s_n, c->st));
  CK(cudaMemsetAsync(c->e2.p, 0xFF, 8 * s_n, c->st));
  for (int b = 0; b < 2; b++) {
    CK(c->keys[b].ensure(4 * n_rec));
    CK(c->vals[b].ensure(4 * n_rec));
  }
  if (s_n > 0) {
    k_make_keys<<<blocks_for(s_n), 256, 0, c->st>>>(
        s_n, c->ends.as<int2>(), (uint32_t)m_n, c->keys[0].as<uint32_t>(),
        c->vals[0].as<uint32_t>(), c->deg.as<uint32_t>());
    CKL();
  }
  // slice entry counts -> exclusive scan -> slice_ptr
  if (n_slices > 0) {
    k_slice_width<<<blocks_for(32 * n_slices), 256, 0, c->st>>>(
        m_n, c->deg.as<uint32_t>(), n_slices, c->width.as<int64_t>());
    CKL();
  }
  size_t tmp_bytes = 0, t2 = 0;
  int end_bit = 1;
  while (((uint64_t)1 << end_bit) <= (uint64_t)m_n) end_bit++;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, (int64_t *)nullptr,
                                (int64_t *)nullptr, (int)(n_slices + 1));
  if (n_rec > 0)
    cub::DeviceRadixSort::SortPairs(
        nullptr, t2, (uint32_t *)nullptr, (uint32_t *)nullptr,
        (uint32_t *)nullptr, (uint32_t *)nullptr, (int)n_rec, 0, end_bit);
  CK(c->sort_tmp.ensure(std::max(tmp_bytes, t2)));
  CK(cudaMemsetAsync(c->width.as<int64_t>() + n_slices, 0, 8, c->st));
  tmp_bytes = c->sort_tmp.bytes;
  CK(cub::DeviceScan::ExclusiveSum(c->sort_tmp.p, tmp_bytes,
                                   c->width.as<int64_t>(),
                                   c->slice_ptr.as<int64_t>(),
                                   (int)(n_slices + 1), c->st));
  int64_t n_ent = 0, max_ent = 0;
  CK(cudaMemcpyAsync(&n_ent, c->slice_ptr.as<int64_t>() + n_slices, 8,
                     cudaMemcpyDeviceToHost, c->st));
  if (n_slices > 0) {
    size_t rb = 0;
    cub::DeviceReduce::Max(nullptr, rb, (int64_t *)nullptr,
                           (int64_t *)nullptr, (int)n_slices);
    if (rb > c->sort_tmp.bytes) {
      CK(cudaStreamSynchronize(c->st));
      CK(c->sort_tmp.ensure(rb));
    }
    rb = c->sort_tmp.bytes;
    CK(cub::DeviceReduce::Max(c->sort_tmp.p, rb, c->width.as<int64_t>(),
                              c->width.as<int64_t>() + n_slices,
                              (int)n_slices, c->st));
    CK(cudaMemcpyAsync(&max_ent, c->width.as<int64_t>() + n_slices, 8,
                       cudaMemcpyDeviceToHost, c->st));
  }
  CK(cudaStreamSynchronize(c->st));
  CK(c->ent_j.ensure(4 * n_ent));
  CK(c->ent_kL0.ensure(2 * c->fsz * n_ent));
  CK(c->ent_s.ensure(4 * n_ent));
  CK(cudaMemsetAsync(c->ent_j.p, 0xFF, 4 * n_ent, c->st));
  CK(cudaMemsetAsync(c->xflags.p, 0, m_n + 1, c->st));
  if (m_n > 0) {
    k_clear_flag<<<blocks_for(m_n), 256, 0, c->st>>>(m_n, c->vel.p,
                                                      c->rsz == 8, MF_SPECIAL);
    CKL();
  }
  CK(cudaMemsetAsync(c->ent_s.p, 0xFF, 4 * n_ent, c->st));
  if (n_rec > 0) {
    tmp_bytes = c->sort_tmp.bytes;
    CK(cub::DeviceRadixSort::SortPairs(
        c->sort_tmp.p, tmp_bytes, c->keys[0].as<uint32_t>(),
        c->keys[1].as<uint32_t>(), c->vals[0].as<uint32_t>(),
        c->vals[1].as<uint32_t>(), (int)n_rec, 0, end_bit, c->st));
    DevBuf &start = c->start;
    CK(start.ensure(8 * (m_n + 1)));
    k_owner_start<<<blocks_for(n_rec), 256, 0, c->st>>>(
        n_rec, c->keys[1].as<uint32_t>(), (uint32_t)m_n,
        start.as<int64_t>());
    CKL();
    KState S = make_state(c);
    auto fill = c->prec == PREC_FP64   ? k_fill_layout<PREC_FP64>
                : c->prec == PREC_FP32 ? k_fill_layout<PREC_FP32>
                                       : k_fill_layout<PREC_MIXED>;
    fill<<<blocks_for(n_rec), 256, 0, c->st>>>(
        n_rec, c->keys[1].as<uint32_t>(), c->vals[1].as<uint32_t>(),
        (uint32_t)m_n, start.as<int64_t>(), S, c->ent_j.as<uint32_t>(),
        c->ent_kL0.p, c->ent_s.as<int32_t>(), c->e1.as<int64_t>(),
        c->e2.as<int64_t>());
    CKL();
  }
  CK(cudaStreamSynchronize(c->st));
  c->n_slices = n_slices;
  c->n_entries = n_ent;
  c->max_width = max_ent / 32;
  configure_tma(c);
  c->layout_valid = true;
  c->layout_builds++;
  c->launches += 5;
  return SL_OK;
}


// Size the per-warp rings of the split TMA kernel and pick its gather batch
// U: every section is processed in whole batches of U rows (the stage pads
// the tail with zero-force rows), so U trades padded rows against exposed
// gather latency (one L2 round trip per batch).  Cost model per slice:
// padded rows + 3 x batches.
void configure_split_tma(sl_ctx *c, const std::vector<uint32_t> &widths) {
  c->split_warps = 0;
  if (!c->tma_enabled || c->n_slices == 0) return;
  const bool act = c->agrp.n > 1;
  // fp64 state doubles the gather registers: batches of 4 (r1e sweep);
  // fp32 batches of 13 spill since the compensated positions (config B:
  // 140.7 us against 101.2 for 4 and 102.9 for 8, profiles/r3/
  // sweep_split_u_warps.txt)
  const int cands_fp32[] = {4, 8}, cands_act[] = {4, 8}, cands_mixed[] = {4};
  const int *cands = c->prec != PREC_FP32 ? cands_mixed
                     : act                ? cands_act
                                          : cands_fp32;
  const int n_cands = c->prec != PREC_FP32 ? 1 : 2;
  int best_u = 4;
  double best = 1e300;
  for (int q = 0; q < n_cands; q++) {
    const int u = cands[q];
    double cost = 0;
    for (uint32_t wd : widths) {
      const int wa = wd & 0xFFFF, wb = wd >> 16;
      const int ba = (wa + u - 1) / u, bb = (wb + u - 1) / u;
      cost += (double)(ba + bb) * u + 3.0 * (ba + bb);
    }
    if (cost < best) {
      best = cost;
      best_u = u;
    }
  }
  if (const char *ev = getenv("SL_SPLIT_U")) {  // tuning override
    const int f = atoi(ev);
    for (int q = 0; q < n_cands; q++)
      if (cands[q] == f) best_u = f;
  }
  const int u = best_u;
  const int64_t cap_a = (c->sp_wa + u - 1) / u * u;
  const int64_t cap_b = (c->sp_wb + u - 1) / u * u;
  const size_t stage = 2 * 32 * 4 * c->rsz + (size_t)(cap_a + cap_b) * 128 +
                       (size_t)cap_a * 32 * 2 * c->fsz +
                       (act ? (size_t)cap_a * 32 * 16 : 0);
  const size_t per_warp = 2 * stage + 16;
  int want = SPLIT_DEFAULT_WARPS;
  if (const char *ev = getenv("SL_SPLIT_WARPS"))  // tuning override
    want = std::max(2, std::min(SPLIT_MAX_WARPS, atoi(ev)));
  int warps = (int)std::min<size_t>((size_t)want,
                                    (size_t)c->smem_optin / per_warp);
  if (warps < 2) return;
  c->scfg.n_slices = c->n_slices;
  c->scfg.u = u;
  c->scfg.act = act;
  c->scfg.cap_a = (int)cap_a;
  c->scfg.cap_b = (int)cap_b;
  c->scfg.warps = warps;
  c->scfg.stage_bytes = (uint32_t)stage;
  int64_t ctas = (c->n_slices + warps - 1) / warps;
  c->split_grid = (int)std::min<int64_t>(ctas, c->sm_count);
  if (launchers(c->prec).split_setup((int)(warps * per_warp), u, act) !=
      0) {
    cudaGetLastError();
    return;
  }
  c->split_warps = warps;
}

// Tile/window geometry of the fp32 split layout (sl_window.cuh); c->win stays
// false when a tile does not fit (the split kernel then runs).
int build_window_tt(sl_ctx *c, int tt);
int build_window_layout(sl_ctx *c) {
  c->win = false;
  if (!c->win_enabled || !c->tma_enabled || c->prec == PREC_FP64 ||
      c->n_slices == 0 || c->sp_wa > 64 || c->sp_wb > 64)
    return SL_OK;
  // consumer warps per CTA: 16 (r1 sweeps: the more the better) unless the
  // mesh has too few slices to give every SM a tile -- small meshes are
  // latency-bound per tile, so 8-slice tiles spread them over more SMs
  // (10^3..30^3: 8.2 -> 6.2 us/step; 50^3 and up keep 16)
  int tt = c->n_slices <= (int64_t)8 * c->sm_count ? 8 : 16;
  if (c->prec == PREC_MIXED) tt = 16;  // mixed instantiations: 16, 12
  if (const char *ev = getenv("SL_WIN_T")) {
    const int v = atoi(ev);
    if (c->prec != PREC_MIXED)
      tt = v == 4 || v == 8 || v == 10 || v == 12 || v == 20 || v == 24
               ? v
               : 16;
    return build_window_tt(c, tt);
  }
  // fp32 with compensated positions (larger windows): 16-slice tiles fit 2
  // ring stages; measured against 12-slice tiles with 3 stages, 46.7 vs
  // 47.6 us/step (config B, profiles/r2/sweep_win2.txt); falls back to 12
  // when 16 does not fit at all
  if (int rc = build_window_tt(c, tt)) return rc;
  // (mixed: fp64 windows of 32 B records -- 16-slice tiles of 32-bit entry
  // words leave room for one stage only)
  if (tt == 16 && !c->win) return build_window_tt(c, 12);
  return SL_OK;
}

int build_window_tt(sl_ctx *c, int tt) {
  c->win = false;
  const int64_t n_tiles = (c->n_slices + tt - 1) / tt;
  WinCfg w{};
  w.n_tiles = n_tiles;
  w.tile_slices = tt;
  w.cap_a = (int)std::max<int64_t>(c->sp_wa, 1);
  w.cap_b = (int)std::max<int64_t>(c->sp_wb, 1);
  // slice block: entry words (sl_window.cuh ew_word), the slice's A rows
  // then its B rows, row pairs interleaved per lane; capacity wa + wb rows
  // (rounded up to even) of 32 lanes x 4 B
  const uint32_t cap_rows = (uint32_t)((w.cap_a + w.cap_b + 1) / 2 * 2);
  w.bl.off_acode = w.bl.off_b16 = w.bl.off_bcode = 0;
  w.bl.slice_bytes = cap_rows * 128u;
  CK(c->win_rec.ensure(sizeof(TileRec) * n_tiles));
  CK(c->win_dict.ensure(8 * WIN_DMAX * n_tiles));
  CK(c->win_actb.ensure((size_t)WIN_ACTB * n_tiles));
  CK(c->win_zero.ensure(n_tiles));
  CK(c->win_blk.ensure((size_t)w.bl.slice_bytes * n_tiles * tt));
  CK(c->win_fail.ensure(24));
  CK(cudaMemsetAsync(c->win_fail.p, 0, 24, c->st));
  const int64_t m_pad = c->n_slices * 32;
  k_win_build<<<(unsigned)n_tiles, 256, 0, c->st>>>(
      c->sp_j.as<uint32_t>(), c->sp_w.as<uint32_t>(), c->sp_kl.as<float2>(),
      c->n_slices, c->m_n, c->sp_a, c->sp_rows, (uint32_t)m_pad,
      (uint32_t)(c->n_slices << (c->sp_a + 5)), tt, w.bl, w.cap_a, w.cap_b,
      c->sp_s.as<int32_t>(), c->mode.as<int8_t>(), c->act.as<double4>(),
      c->s_grp.as<uint8_t>(), c->win_rec.as<TileRec>(),
      c->win_dict.as<float2>(), c->win_actb.as<unsigned char>(),
      c->win_zero.as<uint8_t>(), c->win_blk.as<unsigned char>(),
      c->prec == PREC_MIXED ? 1 : 0, c->win_fail.as<unsigned long long>());
  CKL();
  unsigned long long res[3] = {0, 0, 0};
  CK(cudaMemcpyAsync(res, c->win_fail.p, 24, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  c->launches++;
  if (res[0]) return SL_OK;
  // stage: record | material table | [actuation block] | windows (sized to
  // the widest tile) | tt slice blocks.  Without actuated tiles the
  // actuation block takes no space (config B: 3 stages of 16 slices fit
  // instead of 2)
  w.cap_rec = (uint32_t)((res[1] + 7) / 8 * 8);
  w.off_dict = sizeof(TileRec);
  w.off_act = w.off_dict + 8 * WIN_DMAX;
  w.off_win = w.off_act + (res[2] ? WIN_ACTB : 0);
  uint32_t win_end = w.off_win + (uint32_t)(4 * c->rsz) * w.cap_rec;
  if (c->prec == PREC_FP32) {  // the windows' position low parts, masses
    w.off_wlo = (win_end + 15) / 16 * 16;
    win_end = w.off_wlo + 8 * w.cap_rec;
    w.off_mass = (win_end + 15) / 16 * 16;
    win_end = w.off_mass + 4 * 32 * tt;
    w.pmass = c->pmass.as<float>();
  }
  w.off_slice = (win_end + 127) / 128 * 128;
  w.stage_bytes = w.off_slice + (uint32_t)tt * w.bl.slice_bytes;
  const int64_t bar = 8 * 2 * WIN_MAXST + 8 * WIN_MAXST * WIN_DMAX;
  // stage the tile's velocities with the windows when 2 stages still fit
  // (SL_WIN_VSTAGE=0: keep the consumers' register prefetch)
  {
    const uint32_t vb = (uint32_t)(32 * 4 * c->rsz) * (uint32_t)tt;
    const char *ev = getenv("SL_WIN_VSTAGE");
    const bool want = ev ? atoi(ev) != 0 : c->prec == PREC_MIXED;
    if (want && ((int64_t)c->smem_optin - bar) / (w.stage_bytes + vb) >= 2) {
      w.off_vel = w.stage_bytes;
      w.stage_bytes += vb;
    }
  }
  int nst = (int)std::min<int64_t>(
      WIN_MAXST, ((int64_t)c->smem_optin - bar) / w.stage_bytes);
  if (const char *ev = getenv("SL_WIN_STAGES"))  // tuning override
    nst = std::min(nst, std::max(2, atoi(ev)));
  if (nst < 2) return SL_OK;
  w.nst = nst;
  w.off_eff = (uint32_t)nst * w.stage_bytes;
  if (const char *ev = getenv("SL_WIN_DBG")) w.dbg_nocompute = atoi(ev);
  if (getenv("SL_WIN_INFO"))
    fprintf(stderr,
            "[softlat] window layout: %lld tiles of %d slices, cap_rec %u, "
            "slice %u B, stage %u B (windows %u B), %d stages of %lld B "
            "opt-in\n",
            (long long)n_tiles, tt, w.cap_rec, w.bl.slice_bytes,
            w.stage_bytes, w.off_slice - w.off_win, nst,
            (long long)c->smem_optin);
  w.rec = c->win_rec.as<TileRec>();
  w.dict = c->win_dict.as<float2>();
  w.actb = c->win_actb.as<unsigned char>();
  w.blk = c->win_blk.as<unsigned char>();
  if (launchers(c->prec).win_setup(w) != 0) {
    cudaGetLastError();
    return SL_OK;
  }
  c->wcfg = w;
  c->win_grid = (int)std::min<int64_t>(n_tiles, c->sm_count);
  c->win = true;
  return SL_OK;
}

// The window layout over the exact layout (fp64 parity mode): T = 12
// tiles, fp64 windows, exact (k, L0) tables, entries in ascending slot
// order (k_win64_build).  c->win stays false when a tile does not fit.
int build_window_exact(sl_ctx *c) {
  c->win = false;
  if (!c->win_enabled || !c->tma_enabled || c->prec != PREC_FP64 ||
      c->n_slices == 0 || c->max_width == 0 || c->max_width > 64)
    return SL_OK;
  // 4-slice tiles for meshes of at most one slice per SM (10^3: 9.8 ->
  // 8.4 us/step; at 30^3 the 12-slice tiles are faster, 10.3 vs 14.6)
  int tt = c->n_slices <= (int64_t)c->sm_count ? 4 : SL_WIN64_T;
  if (const char *ev = getenv("SL_WIN64_T"))
    tt = atoi(ev) == 4 ? 4 : SL_WIN64_T;
  const int64_t n_tiles = (c->n_slices + tt - 1) / tt;
  WinCfg w{};
  w.n_tiles = n_tiles;
  w.tile_slices = tt;
  w.cap_a = (int)((c->max_width + 1) / 2 * 2);  // entry-word row pairs
  w.cap_b = 0;
  // slice block: entry words (sl_window.cuh ew_word64), row pairs per lane
  w.bl.off_acode = w.bl.off_b16 = w.bl.off_bcode = 0;
  w.bl.slice_bytes = (uint32_t)w.cap_a * 128u;
  CK(c->win_rec.ensure(sizeof(TileRec) * n_tiles));
  CK(c->win_dict.ensure(16 * WIN_DMAX * n_tiles));
  CK(c->win_blk.ensure((size_t)w.bl.slice_bytes * n_tiles * tt));
  CK(c->win_fail.ensure(16));
  CK(cudaMemsetAsync(c->win_fail.p, 0, 16, c->st));
  const int64_t m_pad = c->n_slices * 32;
  KState S = make_state(c);
  k_win64_build<<<(unsigned)n_tiles, 256, 0, c->st>>>(
      S.slice_ptr, c->ent_j.as<uint32_t>(), c->ent_kL0.as<double2>(),
      c->n_slices, c->m_n, (uint32_t)m_pad, tt, w.bl, w.cap_a,
      c->win_rec.as<TileRec>(), c->win_dict.as<double2>(),
      c->win_blk.as<unsigned char>(), c->win_fail.as<unsigned long long>());
  CKL();
  unsigned long long res[2] = {0, 0};
  CK(cudaMemcpyAsync(res, c->win_fail.p, 16, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  c->launches++;
  if (res[0]) return SL_OK;
  w.cap_rec = (uint32_t)((res[1] + 7) / 8 * 8);
  w.off_dict = sizeof(TileRec);
  w.off_act = w.off_dict + 16 * WIN_DMAX;
  w.off_win = w.off_act;  // no actuation block in parity mode
  w.off_slice = (w.off_win + 32 * w.cap_rec + 127) / 128 * 128;
  w.stage_bytes = w.off_slice + (uint32_t)tt * w.bl.slice_bytes;
  const int64_t bar = 8 * 2 * WIN_MAXST + 16 * WIN_MAXST * WIN_DMAX;
  // the tile's velocities staged by the producer (frees the consumers'
  // register prefetch, which spilled at 128 registers) when 2 stages fit
  w.off_vel = w.stage_bytes;  // (the fp64 kernel always stages them)
  w.stage_bytes += 32 * 32 * tt;
  int nst = (int)std::min<int64_t>(
      WIN_MAXST, ((int64_t)c->smem_optin - bar) / w.stage_bytes);
  if (nst < 2) return SL_OK;
  w.nst = nst;
  w.off_eff = (uint32_t)nst * w.stage_bytes;
  w.rec = c->win_rec.as<TileRec>();
  w.dict = c->win_dict.as<float2>();  // double2 entries (parity mode)
  w.blk = c->win_blk.as<unsigned char>();
  if (launchers(c->prec).win_setup(w) != 0) {
    cudaGetLastError();
    return SL_OK;
  }
  c->wcfg = w;
  c->win_grid = (int)std::min<int64_t>(n_tiles, c->sm_count);
  c->win = true;
  return SL_OK;
}

// Groups of whole connected components for the multi-step fused kernel
// (sl_fused.cuh); c->fz_ok stays false when the context is not eligible.
int build_fused_groups(sl_ctx *c) {
  c->fz_ok = false;
  const int64_t m_n = c->m_n, s_n = c->s_n;
  if (!c->fz_enabled || c->prec != PREC_FP32 || !c->split || c->has_ghost ||
      m_n == 0 || c->sp_wa + c->sp_wb > FZ_MAXR)
    return SL_OK;
  // component boundaries: no alive spring spans (b - 1, b)
  CK(c->fz_diff.ensure(4 * (m_n + 1)));
  CK(cudaMemsetAsync(c->fz_diff.p, 0, 4 * (m_n + 1), c->st));
  if (s_n > 0) {
    k_fused_cover<<<blocks_for(s_n), 256, 0, c->st>>>(
        s_n, c->ends.as<int2>(), c->fz_diff.as<int32_t>());
    CKL();
  }
  std::vector<int32_t> diff(m_n + 1);
  CK(cudaMemcpyAsync(diff.data(), c->fz_diff.p, 4 * (m_n + 1),
                     cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  // group capacity: 512 masses (two CTAs per SM) unless a component needs
  // up to 1024 (one 1024-thread CTA per SM)
  int maxm = FZ_MAXM;
  {
    int64_t cov = 0, c0 = 0;
    for (int64_t b = 1; b <= m_n; b++) {
      cov += diff[b];
      if (b < m_n && cov != 0) continue;
      if (b - c0 > FZ_MAXM_L) return SL_OK;  // a body too large for a CTA
      if (b - c0 > FZ_MAXM) maxm = FZ_MAXM_L;
      c0 = b;
    }
  }
  // pack consecutive components into groups of <= maxm masses
  std::vector<int32_t> gs, gc;
  int64_t cover = 0, comp0 = 0, g0 = 0;
  for (int64_t b = 1; b <= m_n; b++) {
    cover += diff[b];
    if (b < m_n && cover != 0) continue;  // (b - 1, b) is spanned
    const int64_t len = b - comp0;        // component [comp0, b)
    if (len > maxm) return SL_OK;         // (checked above)
    if (b - g0 > maxm) {                  // close the group before comp0
      gs.push_back((int32_t)g0);
      gc.push_back((int32_t)(comp0 - g0));
      g0 = comp0;
    }
    comp0 = b;
  }
  gs.push_back((int32_t)g0);
  gc.push_back((int32_t)(m_n - g0));
  const int64_t ng = (int64_t)gs.size();
  const int ra = (int)c->sp_wa, rb = (int)c->sp_wb;
  const int rows = std::max(1, ra + rb);
  CK(c->fz_gstart.ensure(4 * ng));
  CK(c->fz_gcount.ensure(4 * ng));
  CK(c->fz_ent.ensure((size_t)2 * ng * rows * maxm));
  CK(c->fz_code.ensure((size_t)ng * rows * maxm));
  CK(c->fz_epos.ensure((size_t)2 * ng * rows * maxm));
  CK(c->fz_perm.ensure((size_t)2 * ng * maxm));
  CK(c->fz_cnt.ensure((size_t)ng * maxm));
  CK(c->fz_cnt_a.ensure((size_t)ng * maxm));
  CK(c->fz_dict.ensure((size_t)8 * WIN_DMAX * ng));
  CK(c->fz_actb.ensure((size_t)WIN_ACTB * ng));
  CK(c->fz_has.ensure(ng));
  CK(c->fz_zero.ensure(ng));
  CK(c->fz_gid.ensure(4 * m_n));
  CK(c->fz_fail.ensure(8));
  CK(cudaMemcpyAsync(c->fz_gstart.p, gs.data(), 4 * ng,
                     cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(c->fz_gcount.p, gc.data(), 4 * ng,
                     cudaMemcpyHostToDevice, c->st));
  CK(cudaMemsetAsync(c->fz_fail.p, 0, 8, c->st));
  const int64_t m_pad = c->n_slices * 32;
  auto build = maxm > FZ_MAXM ? k_fused_build<FZ_MAXM_L>
                              : k_fused_build<FZ_MAXM>;
  build<<<(unsigned)ng, maxm, 0, c->st>>>(
      c->sp_j.as<uint32_t>(), c->sp_w.as<uint32_t>(), c->sp_kl.as<float2>(),
      c->sp_s.as<int32_t>(), c->mode.as<int8_t>(), c->act.as<double4>(),
      c->s_grp.as<uint8_t>(), c->vel.as<float4>(), c->sp_a, c->sp_rows,
      (uint32_t)m_pad, (uint32_t)(c->n_slices << (c->sp_a + 5)),
      c->fz_gstart.as<int32_t>(), c->fz_gcount.as<int32_t>(), ra, rb,
      c->fz_ent.as<uint16_t>(), c->fz_code.as<uint8_t>(),
      c->fz_perm.as<uint16_t>(), c->fz_cnt.as<uint8_t>(),
      c->fz_cnt_a.as<uint8_t>(), c->fz_epos.as<uint16_t>(),
      c->fz_dict.as<float2>(), c->fz_actb.as<unsigned char>(),
      c->fz_has.as<uint8_t>(), c->fz_zero.as<uint8_t>(),
      c->fz_gid.as<int32_t>(), c->fz_fail.as<unsigned long long>(), nullptr);
  CKL();
  unsigned long long failed = 0;
  CK(cudaMemcpyAsync(&failed, c->fz_fail.p, 8, cudaMemcpyDeviceToHost,
                     c->st));
  CK(cudaStreamSynchronize(c->st));
  c->launches += 2;
  if (failed) return SL_OK;
  FzCfg f{};
  f.n_groups = ng;
  f.gstart = c->fz_gstart.as<int32_t>();
  f.gcount = c->fz_gcount.as<int32_t>();
  f.ent = c->fz_ent.as<uint16_t>();
  f.code = c->fz_code.as<uint8_t>();
  f.perm = c->fz_perm.as<uint16_t>();
  f.cnt = c->fz_cnt.as<uint8_t>();
  f.cnt_a = c->fz_cnt_a.as<uint8_t>();
  f.dict = c->fz_dict.as<float2>();
  f.actb = c->fz_actb.as<unsigned char>();
  f.has_act = c->fz_has.as<uint8_t>();
  f.ra = ra;
  f.rb = rb;
  const size_t smem = 32 * WIN_DMAX + 24 * 2 * (maxm + 1) +
                      8 * 4 * WIN_DMAX + (size_t)4 * rows * maxm + WIN_DMAX;
  f.maxm = maxm;
  if (launchers(c->prec).fused_setup(smem, maxm) != 0) {
    cudaGetLastError();
    return SL_OK;
  }
  c->fcfg = f;
  c->fz_smem = smem;
  c->fz_ok = true;
  return SL_OK;
}

// One fused launch of n steps (sl_fused.cuh).  *aborted: the launch hit
// something only the per-step kernels represent and committed nothing.
int run_fused(sl_ctx *c, const KState &S, int64_t n, const double *times,
              double dt, bool *aborted) {
  *aborted = false;
  CK(c->fz_times.ensure(8 * n));
  CK(cudaMemcpyAsync(c->fz_times.p, times, 8 * n, cudaMemcpyHostToDevice,
                     c->st));
  CK(c->vel2.ensure(c->vel.bytes));
  CK(cudaMemsetAsync((char *)c->vel2.p + 16 * c->m_n, 0, 16 * 32,
                     c->st));  // the padding records (window bulk copies)
  FzCfg f = c->fcfg;
  f.vel_out = c->vel2.p;
  f.times = c->fz_times.as<double>();
  f.n_steps = n;
  f.cur = c->cur;
  f.write_acc = 1;
  CK(cudaEventRecord(c->k0, c->st));
  launchers(c->prec).fused(S, c->env, f, dt, c->fz_smem, c->st);
  CKL();
  CK(cudaEventRecord(c->k1, c->st));
  c->k_valid = true;
  c->launches++;
  c->fz_launches++;
  CK(cudaMemcpyAsync(c->h_status, c->status.p, 8 * 8, cudaMemcpyDeviceToHost,
                     c->st));
  CK(cudaStreamSynchronize(c->st));
  if (c->h_status[5]) {
    *aborted = true;
    c->fz_aborts++;
    // keep the counters already in status (prepare's invalid-endpoint
    // kills, kernels.py:37-45): the per-step re-run adds to them
    CK(cudaMemsetAsync(c->status.as<unsigned long long>() + 5, 0, 2 * 8,
                       c->st));
    return SL_OK;
  }
  std::swap(c->vel, c->vel2);  // committed: the new velocities
  c->cur ^= 1;                  // final positions in pos[cur ^ 1]
  if (c->h_status[6]) {
    k_fused_clear_fext<<<blocks_for(c->m_n), 256, 0, c->st>>>(
        c->m_n, c->vel2.as<float4>(), c->fext.as<float4>());
    CKL();
    c->launches++;
  }
  return SL_OK;
}

// Device build of the split layout (sl_split.cuh).  *used = false when the
// mesh does not fit its index encoding (the caller falls back to the exact
// layout).
int build_split_layout(sl_ctx *c, bool *used) {
  *used = false;
  const int64_t m_n = c->m_n, s_n = c->s_n;
  const int64_t n_slices = (m_n + 31) / 32;
  const int64_t m_pad = n_slices * 32;
  if (m_pad + 32 >= (int64_t)0xFFFFFFFF || 2 * m_n + 1 >= (int64_t)0xFFFFFFFF ||
      2 * s_n >= (int64_t)0x7fffffff)
    return SL_OK;
  const int64_t n_rec = 2 * s_n;
  CK(c->deg.ensure(4 * (m_n + 1)));
  CK(c->degB.ensure(4 * (m_n + 1)));
  CK(c->sp_w.ensure(4 * (n_slices + 1)));
  CK(c->sp_meta.ensure(8 * 4));
  CK(cudaMemsetAsync(c->deg.p, 0, 4 * (m_n + 1), c->st));
  CK(cudaMemsetAsync(c->degB.p, 0, 4 * (m_n + 1), c->st));
  CK(cudaMemsetAsync(c->sp_meta.p, 0, 8 * 4, c->st));
  CK(cudaMemsetAsync(c->sp_w.p, 0, 4 * (n_slices + 1), c->st));
  for (int b = 0; b < 2; b++) {
    CK(c->keys[b].ensure(4 * n_rec));
    CK(c->vals[b].ensure(4 * n_rec));
  }
  if (s_n > 0) {
    k_split_keys<<<blocks_for(s_n), 256, 0, c->st>>>(
        s_n, c->ends.as<int2>(), (uint32_t)m_n, c->keys[0].as<uint32_t>(),
        c->vals[0].as<uint32_t>(), c->deg.as<uint32_t>(),
        c->degB.as<uint32_t>());
    CKL();
  }
  if (n_slices > 0) {
    k_split_widths<<<blocks_for(32 * n_slices), 256, 0, c->st>>>(
        m_n, c->deg.as<uint32_t>(), c->degB.as<uint32_t>(), n_slices,
        c->sp_w.as<uint32_t>(), c->sp_meta.as<unsigned long long>());
    CKL();
  }
  unsigned long long meta[3] = {0, 0, 0};
  CK(cudaMemcpyAsync(meta, c->sp_meta.p, sizeof meta, cudaMemcpyDeviceToHost,
                     c->st));
  CK(cudaStreamSynchronize(c->st));
  const int64_t wa = (int64_t)meta[0], wb = (int64_t)meta[1];
  int a = 0;
  while (((int64_t)1 << a) < std::max<int64_t>(wa, 1)) a++;
  const int64_t rows = ((int64_t)1 << a) + wb;
  // encodings: 16-bit widths, 32-bit kl indices (incl. the zero slice)
  if (wa > 0xFFFF || wb > 0xFFFF || a > 16 ||
      ((n_slices + 1) << (a + 5)) >= ((int64_t)1 << 32) ||
      n_slices * rows * 32 >= ((int64_t)1 << 32) ||
      // footprint guard for hub masses: stride padding must not explode
      n_slices * rows * 32 > 4 * (int64_t)meta[2] + (1 << 20))
    return SL_OK;
  c->split = true;
  c->sp_a = a;
  c->sp_rows = (int)rows;
  c->sp_wa = wa;
  c->sp_wb = wb;
  const int64_t n_j = n_slices * rows * 32;
  const int64_t n_kl = (n_slices + 1) << (a + 5);
  const size_t f2 = 2 * c->fsz;
  CK(c->sp_j.ensure(4 * n_j));
  CK(c->sp_s.ensure(4 * n_j));
  CK(c->sp_kl.ensure(f2 * n_kl));
  CK(c->sp_ekl.ensure(4 * std::max<int64_t>(s_n, 1)));
  CK(c->e1.ensure(8 * s_n));
  CK(c->e2.ensure(8 * s_n));
  CK(cudaMemsetAsync(c->e1.p, 0xFF, 8 * s_n, c->st));
  CK(cudaMemsetAsync(c->e2.p, 0xFF, 8 * s_n, c->st));
  CK(cudaMemsetAsync(c->sp_kl.p, 0, f2 * n_kl, c->st));
  const bool act = c->agrp.n > 1;
  if (act) {
    CK(c->sp_actc.ensure(16 * n_kl));
    CK(c->sp_acto.ensure(8 * n_kl));
    // zero cells = group 0 (factor exactly 1: amp 0)
    CK(cudaMemsetAsync(c->sp_actc.p, 0, 16 * n_kl, c->st));
    CK(cudaMemsetAsync(c->sp_acto.p, 0, 8 * n_kl, c->st));
  }
  CK(cudaMemsetAsync(c->sp_s.p, 0xFF, 4 * n_j, c->st));
  CK(cudaMemsetAsync(c->xflags.p, 0, m_n + 1, c->st));
  if (n_j > 0) {
    k_split_init<<<blocks_for(n_j), 256, 0, c->st>>>(
        n_j, (int)rows, 1 << a, (uint32_t)m_pad,
        (uint32_t)(n_slices << (a + 5)), c->sp_j.as<uint32_t>());
    CKL();
  }
  if (m_n > 0) {
    k_clear_flag<<<blocks_for(m_n), 256, 0, c->st>>>(m_n, c->vel.p,
                                                      c->rsz == 8, MF_SPECIAL);
    CKL();
  }
  auto sent = c->prec == PREC_FP32 ? k_split_sentinel<PREC_FP32>
                                   : k_split_sentinel<PREC_MIXED>;
  sent<<<1, 32, 0, c->st>>>(c->pos[0].p, c->pos[1].p, m_pad);
  CKL();
  if (n_rec > 0) {
    int end_bit = 1;
    while (((uint64_t)1 << end_bit) <= (uint64_t)(2 * m_n)) end_bit++;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(
        nullptr, tb, (uint32_t *)nullptr, (uint32_t *)nullptr,
        (uint32_t *)nullptr, (uint32_t *)nullptr, (int)n_rec, 0, end_bit);
    CK(c->sort_tmp.ensure(tb));
    tb = c->sort_tmp.bytes;
    CK(cub::DeviceRadixSort::SortPairs(
        c->sort_tmp.p, tb, c->keys[0].as<uint32_t>(),
        c->keys[1].as<uint32_t>(), c->vals[0].as<uint32_t>(),
        c->vals[1].as<uint32_t>(), (int)n_rec, 0, end_bit, c->st));
    CK(c->start.ensure(8 * (2 * m_n + 1)));
    k_owner_start<<<blocks_for(n_rec), 256, 0, c->st>>>(
        n_rec, c->keys[1].as<uint32_t>(), (uint32_t)(2 * m_n),
        c->start.as<int64_t>());
    CKL();
    KState S = make_state(c);
    auto fill = c->prec == PREC_FP32 ? k_split_fill<PREC_FP32>
                                     : k_split_fill<PREC_MIXED>;
    for (int pass = 0; pass < 2; pass++) {
      fill<<<blocks_for(n_rec), 256, 0, c->st>>>(
          n_rec, c->keys[1].as<uint32_t>(), c->vals[1].as<uint32_t>(),
          (uint32_t)(2 * m_n), c->start.as<int64_t>(), S,
          c->sp_j.as<uint32_t>(), c->sp_kl.p, c->sp_s.as<int32_t>(),
          c->sp_ekl.as<uint32_t>(), c->e1.as<int64_t>(), c->e2.as<int64_t>(),
          pass, act ? c->sp_actc.as<float4>() : nullptr,
          c->sp_acto.as<double>(), c->s_grp.as<uint8_t>());
      CKL();
    }
  }
  std::vector<uint32_t> widths(n_slices);
  if (n_slices > 0)
    CK(cudaMemcpyAsync(widths.data(), c->sp_w.p, 4 * n_slices,
                       cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  c->n_slices = n_slices;
  c->n_entries = (int64_t)meta[2];
  c->max_width = 0;
  c->tma_warps = 0;
  configure_split_tma(c, widths);
  if (int rc = build_window_layout(c)) return rc;
  if (int rc = build_fused_groups(c)) return rc;
  c->layout_valid = true;
  c->layout_builds++;
  c->launches += 8;
  *used = true;
  return SL_OK;
}

// Accumulation variant per mesh (tools/hub_sweep.py, profiles/hub_sweep_r2.txt:
// gather vs atomic step time on lattices and on hub meshes of degree D).
// The gather's slice-ELL pads a 32-mass slice to its widest list, so a hub
// makes its whole slice D wide; the per-spring atomic kernel's cost does
// not depend on D.  Measured crossover (B200): fp32 / mixed between D = 64
// (gather 131 us vs atomic 205 us) and 128 (970 vs 203); fp64 between 8
// (208 vs 297) and 16 (359 vs 278).  A mesh is a "hub mesh" when its
// widest list exceeds the threshold AND padding more than doubles the
// stored entries -- uniform meshes (a lattice: 26 entries every mass)
// never qualify, whatever their width.
int64_t hub_threshold(const sl_ctx *c) {
  if (const char *ev = getenv("SL_HUB_ENTRIES")) return atoll(ev);
  return c->prec == PREC_FP64 ? 12 : 96;
}
int resolve_accumulation(sl_ctx *c, int acc) {
  const int64_t widest = c->split ? c->sp_wa + c->sp_wb : c->max_width;
  const bool hubs = c->layout_valid && widest > hub_threshold(c) &&
                    c->n_entries > 4 * c->s_n;
  // atomic accumulation: the owner-aggregated kernel (one thread per mass,
  // its m1 springs) on regular meshes; on hub meshes one thread per spring
  // with warp-aggregated reductions (the hub's thread would serialise)
  c->atomic_owner = c->layout_valid && !hubs;
  if (const char *ev = getenv("SL_ATOMIC_KERNEL"))  // tuning / sweeps
    c->atomic_owner = c->layout_valid && strcmp(ev, "spring") != 0;
  if (acc != SL_ACC_AUTO) return acc;
  c->auto_atomic = hubs;
  return c->auto_atomic ? SL_ACC_ATOMIC : SL_ACC_GATHER;
}

int build_layout(sl_ctx *c) {
  SL_RANGE("build_layout");
  c->split = false;
  if (c->prec != PREC_FP64 && c->split_enabled) {
    bool used = false;
    int rc = build_split_layout(c, &used);
    if (rc || used) return rc;
    c->split = false;
  }
  c->win = false;
  if (int rc = build_exact_layout(c)) return rc;
  return build_window_exact(c);
}

int prepare(sl_ctx *c, bool need_layout, bool reset_status = true) {
  if (!c->masses_set || !c->springs_set)
    return fail(c, SL_ESTATE, "masses and springs must be uploaded first");
  if (!c->env_set)
    return fail(c, SL_ESTATE, "environment not set (sl_set_environment)");
  if (reset_status) CK(cudaMemsetAsync(c->status.p, 0, 8 * 8, c->st));
  if (c->validate_dirty && c->s_n > 0) {
    KState S = make_state(c);
    k_validate<<<blocks_for(c->s_n), 256, 0, c->st>>>(
        S, c->m_alive.as<uint8_t>(), c->m_gen.as<int64_t>(),
        c->m1gen.as<int64_t>(), c->m2gen.as<int64_t>(), c->layout_valid);
    CKL();
    c->launches++;
  }
  c->validate_dirty = false;
  if (need_layout && !c->layout_valid) {
    int rc = build_layout(c);
    if (rc) return rc;
  }
  return SL_OK;
}

// Refresh the device copy of S (read by out-of-line rare paths) when it
// changed since the last upload.
int upload_state(sl_ctx *c, const KState &S) {
  if (c->khost_valid && memcmp(&c->khost, &S, sizeof S) == 0) return SL_OK;
  c->khost = S;
  CK(cudaMemcpyAsync(c->kdev.p, &c->khost, sizeof S, cudaMemcpyHostToDevice,
                     c->st));
  c->khost_valid = true;
  return SL_OK;
}

int finish_status(sl_ctx *c, int64_t *counters, int64_t *err_slot) {
  CK(cudaMemcpyAsync(c->h_status, c->status.p, 8 * 8, cudaMemcpyDeviceToHost,
                     c->st));
  CK(cudaStreamSynchronize(c->st));
  if (counters)
    for (int q = 0; q < 3; q++) counters[q] += (int64_t)c->h_status[q];
  if (err_slot) *err_slot = (int64_t)c->h_status[3];
  return SL_OK;
}

}  // namespace

// ============================================================== C ABI
extern "C" {

int sl_abi_version(void) { return 1; }

int sl_device_count(int *count) {
  sl_ctx *c = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *count = 0;
    return fail(c, SL_ECUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  }
  *count = n;
  return SL_OK;
}

int sl_host_alloc(size_t bytes, void **out) {
  sl_ctx *c = nullptr;
  if (!out) return fail(c, SL_EINVAL, "out is NULL");
  *out = nullptr;
  cudaError_t e = cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    *out = nullptr;
    return fail(c, SL_ECUDA, "cudaHostAlloc(%zu): %s", bytes,
                cudaGetErrorString(e));
  }
  return SL_OK;
}

int sl_host_free(void *p) {
  sl_ctx *c = nullptr;
  if (!p) return SL_OK;
  cudaError_t e = cudaFreeHost(p);
  if (e != cudaSuccess)
    return fail(c, SL_ECUDA, "cudaFreeHost: %s", cudaGetErrorString(e));
  return SL_OK;
}

const char *sl_last_error(const sl_ctx *ctx) {
  return ctx ? ctx->err.c_str() : g_err.c_str();
}

int sl_create(int device, int precision, sl_ctx **out) {
  sl_ctx *c = nullptr;
  if (!out) return fail(c, SL_EINVAL, "out is NULL");
  *out = nullptr;
  if (precision < 0 || precision > 2)
    return fail(c, SL_EINVAL, "unknown precision %d", precision);
  CK(cudaSetDevice(device));
  c = new sl_ctx();
  c->device = device;
  c->prec = precision;
  c->rsz = precision == PREC_FP32 ? 4 : 8;
  c->fsz = precision == PREC_FP64 ? 8 : 4;
  if (const char *ev = getenv("SL_DISABLE_TMA")) c->tma_enabled = ev[0] == '0';
  if (const char *ev = getenv("SL_DISABLE_WIN")) c->win_enabled = ev[0] == '0';
  if (const char *ev = getenv("SL_DISABLE_FUSED"))
    c->fz_enabled = ev[0] == '0';
  if (const char *ev = getenv("SL_DISABLE_SPLIT"))
    c->split_enabled = ev[0] == '0';
  memset(&c->env, 0, sizeof c->env);
  cudaError_t e = cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking);
  if (e == cudaSuccess)
    e = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&c->t0);
  if (e == cudaSuccess) e = cudaEventCreate(&c->t1);
  if (e == cudaSuccess) e = cudaEventCreate(&c->k0);
  if (e == cudaSuccess) e = cudaEventCreate(&c->k1);
  if (e == cudaSuccess)
    e = cudaEventCreateWithFlags(&c->head_ev, cudaEventDisableTiming);
  if (e == cudaSuccess)
    e = cudaEventCreateWithFlags(&c->tail_ev, cudaEventDisableTiming);
  if (e == cudaSuccess)
    e = cudaEventCreateWithFlags(&c->extra_ev, cudaEventDisableTiming);
  if (e == cudaSuccess)
    e = cudaEventCreateWithFlags(&c->side_ev, cudaEventDisableTiming);
  if (e == cudaSuccess)
    e = cudaEventCreateWithFlags(&c->ck_ev, cudaEventDisableTiming);
  if (e == cudaSuccess)
    e = cudaEventCreateWithFlags(&c->ck_done, cudaEventDisableTiming);
  if (e == cudaSuccess)
    e = cudaEventCreateWithFlags(&c->side_done, cudaEventDisableTiming);
  if (e == cudaSuccess)
    e = cudaEventCreateWithFlags(&c->snap_ev, cudaEventDisableTiming);
  if (e == cudaSuccess)
    e = cudaEventCreateWithFlags(&c->snap_done, cudaEventDisableTiming);
  if (e == cudaSuccess)
    e = cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount,
                               device);
  if (e == cudaSuccess)
    e = cudaDeviceGetAttribute(&c->smem_optin,
                               cudaDevAttrMaxSharedMemoryPerBlockOptin,
                               device);
  if (e == cudaSuccess) e = c->status.ensure(8 * 8);
  if (e == cudaSuccess) e = c->kdev.ensure(sizeof(KState));
  if (e == cudaSuccess) memset(&c->khost, 0, sizeof c->khost);
  if (e == cudaSuccess)
    e = cudaMallocHost((void **)&c->h_status, 8 * 8);
  if (e != cudaSuccess) {
    int rc = fail(nullptr, SL_ECUDA, "context init failed: %s",
                  cudaGetErrorString(e));
    sl_destroy(c);
    return rc;
  }
  *out = c;
  return SL_OK;
}

int sl_destroy(sl_ctx *c) {
  if (!c) return SL_OK;
  cudaSetDevice(c->device);
  if (c->st) cudaStreamSynchronize(c->st);
  if (c->side) cudaStreamSynchronize(c->side);
  DevBuf *bufs[] = {&c->pos[0], &c->pos[1], &c->plo[0], &c->plo[1], &c->pmass, &c->vel, &c->acc, &c->fext,
                    &c->load, &c->m_gen, &c->m_alive, &c->xflags, &c->lc_off,
                    &c->lc_kind, &c->lc_vec, &c->ends, &c->kL0, &c->s_alive,
                    &c->s_degen, &c->mode, &c->act, &c->thr, &c->custom,
                    &c->m1gen, &c->m2gen, &c->slice_ptr, &c->ent_j,
                    &c->ent_kL0, &c->ent_s, &c->e1, &c->e2, &c->stage,
                    &c->sort_tmp, &c->keys[0], &c->keys[1], &c->vals[0],
                    &c->vals[1], &c->deg, &c->width, &c->start, &c->status,
                    &c->snap_dev, &c->sp_j, &c->sp_kl, &c->sp_s, &c->sp_w,
                    &c->sp_ekl, &c->degB, &c->sp_meta, &c->kdev,
                    &c->ghost, &c->s_grp, &c->sp_actc, &c->sp_acto, &c->win_rec, &c->win_dict, &c->win_actb, &c->win_zero, &c->win_blk,
                    &c->fz_gstart, &c->fz_gcount, &c->fz_ent, &c->fz_code,
                    &c->fz_dict, &c->fz_actb, &c->fz_has, &c->fz_fail,
                    &c->fz_times, &c->fz_diff, &c->vel2, &c->fz_zero,
                    &c->fz_gid, &c->diag, &c->fz_perm, &c->fz_cnt,
                    &c->fz_epos, &c->fz_cnt_a,
                    &c->win_fail, &c->stage2, &c->inc_buf, &c->ck_pos, &c->ck_plo, &c->ck_vel, &c->ck_acc, &c->ck_fext, &c->ck_view};
  for (void *p : c->halo_ipc) cudaIpcCloseMemHandle(p);
  c->halo_desc.release();
  c->halo_dst.release();
  c->halo_flags.release();
  for (DevBuf *b : bufs) b->release();
  if (c->h_status) cudaFreeHost(c->h_status);
  if (c->snap_host) cudaFreeHost(c->snap_host);
  if (c->t0) cudaEventDestroy(c->t0);
  if (c->t1) cudaEventDestroy(c->t1);
  if (c->k0) cudaEventDestroy(c->k0);
  if (c->k1) cudaEventDestroy(c->k1);
  if (c->head_ev) cudaEventDestroy(c->head_ev);
  if (c->tail_ev) cudaEventDestroy(c->tail_ev);
  if (c->extra_ev) cudaEventDestroy(c->extra_ev);
  if (c->side_ev) cudaEventDestroy(c->side_ev);
  if (c->ck_ev) cudaEventDestroy(c->ck_ev);
  if (c->ck_done) cudaEventDestroy(c->ck_done);
  if (c->side_done) cudaEventDestroy(c->side_done);
  if (c->snap_ev) cudaEventDestroy(c->snap_ev);
  if (c->snap_done) cudaEventDestroy(c->snap_done);
  if (c->st) cudaStreamDestroy(c->st);
  if (c->side) cudaStreamDestroy(c->side);
  delete c;
  return SL_OK;
}

int sl_get_stats(sl_ctx *c, sl_stats *o) {
  if (!c || !o) return fail(c, SL_EINVAL, "NULL argument");
  memset(o, 0, sizeof *o);
  o->masses = c->m_n;
  o->springs = c->s_n;
  o->entries = c->n_entries;
  o->slices = c->n_slices;
  o->layout_builds = c->layout_builds;
  o->kernel_launches = c->launches;
  o->precision = c->prec;
  o->device = c->device;
  o->step_path = !c->layout_valid ? SL_PATH_NONE
                 : c->split       ? (c->win           ? SL_PATH_WINDOW_TMA
                                     : c->split_warps ? SL_PATH_SPLIT_TMA
                                                      : SL_PATH_SPLIT)
                 : c->win         ? SL_PATH_EXACT_WINDOW
                 : (c->tma_warps ? SL_PATH_EXACT_TMA : SL_PATH_EXACT);
  o->split_batch = c->split && c->split_warps ? c->scfg.u : 0;
  o->fused_groups = c->fz_ok ? c->fcfg.n_groups : 0;
  o->fused_launches = c->fz_launches;
  o->fused_aborts = c->fz_aborts;
  o->win_tile_slices = c->win ? c->wcfg.tile_slices : 0;
  o->win_stages = c->win ? c->wcfg.nst : 0;
  o->inplace_edits = c->inc_edits;
  const DevBuf *bufs[] = {&c->pos[0], &c->pos[1], &c->plo[0], &c->plo[1], &c->pmass, &c->vel, &c->acc,
                          &c->fext, &c->load, &c->m_gen, &c->m_alive,
                          &c->ends, &c->kL0, &c->s_alive, &c->s_degen,
                          &c->mode, &c->act, &c->thr, &c->custom, &c->m1gen,
                          &c->m2gen, &c->slice_ptr, &c->ent_j, &c->ent_kL0,
                          &c->ent_s, &c->e1, &c->e2, &c->stage, &c->sort_tmp,
                          &c->keys[0], &c->keys[1], &c->vals[0], &c->vals[1],
                          &c->deg, &c->width, &c->sp_j, &c->sp_kl, &c->sp_s,
                          &c->sp_w, &c->sp_ekl, &c->degB, &c->stage2};
  for (const DevBuf *b : bufs) o->device_bytes += (int64_t)b->bytes;
  if (c->springs_set) {
    std::vector<uint8_t> al(c->s_n);
    if (c->s_n) {
      CK(cudaMemcpyAsync(al.data(), c->s_alive.p, c->s_n,
                         cudaMemcpyDeviceToHost, c->st));
      CK(cudaStreamSynchronize(c->st));
    }
    for (uint8_t a : al) o->alive_springs += a;
  }
  return SL_OK;
}

int sl_upload_masses(sl_ctx *c, int64_t m_n, const double *pos,
                     const double *vel, const double *acc, const double *fext,
                     const double *load, const double *mass,
                     const uint8_t *fixed, const uint8_t *alive,
                     const int64_t *gen) {
  SL_RANGE("sl_upload_masses");
  if (!c) return fail(c, SL_EINVAL, "NULL context");
  if (m_n < 0 || (m_n > 0 && (!pos || !vel || !mass || !fixed || !alive ||
                              !gen)))
    return fail(c, SL_EINVAL, "sl_upload_masses: bad arguments");
  CK(cudaSetDevice(c->device));
  if (m_n != c->m_n) {
    c->layout_valid = false;  // slices follow mass count
    c->has_ghost = false;
  }
  if (c->async_open)
    return fail(c, SL_ESTATE, "asynchronous run open (sl_step_finish)");
  int rc = ensure_masses(c, m_n);
  if (rc) return rc;
  std::vector<double> zeros;
  if (!acc || !fext || !load) zeros.assign(3 * (size_t)m_n, 0.0);
  size_t need = 0;
  need += align256(24 * m_n) * 5 + align256(8 * m_n) * 2 +
          align256(m_n) * 2 + 1024;
  CK(c->stage.ensure(need));
  size_t off = 0;
  const double *dp, *dv, *da, *df, *dl, *dm;
  const uint8_t *dfx, *dal;
  const int64_t *dg;
  if ((rc = stage_copy(c, off, pos, 3 * m_n, &dp))) return rc;
  if ((rc = stage_copy(c, off, vel, 3 * m_n, &dv))) return rc;
  if ((rc = stage_copy(c, off, acc ? acc : zeros.data(), 3 * m_n, &da)))
    return rc;
  if ((rc = stage_copy(c, off, fext ? fext : zeros.data(), 3 * m_n, &df)))
    return rc;
  if ((rc = stage_copy(c, off, load ? load : zeros.data(), 3 * m_n, &dl)))
    return rc;
  if ((rc = stage_copy(c, off, mass, m_n, &dm))) return rc;
  if ((rc = stage_copy(c, off, fixed, m_n, &dfx))) return rc;
  if ((rc = stage_copy(c, off, alive, m_n, &dal))) return rc;
  if ((rc = stage_copy(c, off, gen, m_n, &dg))) return rc;
  if (m_n > 0) {
    auto k = c->prec == PREC_FP64   ? k_pack_masses<PREC_FP64>
             : c->prec == PREC_FP32 ? k_pack_masses<PREC_FP32>
                                    : k_pack_masses<PREC_MIXED>;
    k<<<blocks_for(m_n), 256, 0, c->st>>>(
        m_n, dp, dv, da, df, dl, dm, dfx, dal, nullptr, c->pos[0].p,
        c->pos[1].p, c->plo[0].p, c->plo[1].p, c->pmass.as<float>(), c->vel.p,
        c->acc.p, c->fext.p, c->load.p,
        c->m_gen.as<int64_t>(), c->m_alive.as<uint8_t>(), dg,
        (c->layout_valid && m_n == c->m_n) ? c->xflags.as<uint8_t>()
                                           : nullptr);
    CKL();
    c->launches++;
    if (c->has_lc && m_n == c->m_n) {
      k_set_lc_flags<<<blocks_for(m_n), 256, 0, c->st>>>(
          m_n, c->lc_off.as<int64_t>(), c->vel.p, c->rsz == 8);
      CKL();
    } else if (c->has_lc) {
      // the constraint table was built for the old mass count (reading it
      // for the new one ran past its end -- compute-sanitizer memcheck on
      // tests/test_gpu_fuzz_edits.py): dropped until the host re-sends it
      // (sl_set_local_constraints, which the engine does on a count change)
      c->has_lc = false;
    }
  }
  CK(cudaStreamSynchronize(c->st));  // staging is reused by the next call
  c->m_n = m_n;
  c->cur = 0;
  c->masses_set = true;
  c->validate_dirty = true;
  return SL_OK;
}

static int upload_springs_impl(sl_ctx *c, int64_t n, const int64_t *slots,
                               const int64_t *m1, const int64_t *m2,
                               const int64_t *m1gen, const int64_t *m2gen,
                               const double *rest, const double *k,
                               const double *diam, const double *yield,
                               const int8_t *mode, const double *amp,
                               const double *freq, const double *off_,
                               const double *per, const uint8_t *alive,
                               const uint8_t *degen, bool params_only) {
  CK(cudaSetDevice(c->device));
  // host-side validation of the pieces the device trusts
  for (int64_t r = 0; r < n; r++) {
    if (!params_only && alive[r] &&
        (m1[r] < 0 || m2[r] < 0 || m1[r] >= c->m_n || m2[r] >= c->m_n))
      return fail(c, SL_EINVAL, "spring %lld endpoint out of range",
                  (long long)(slots ? slots[r] : r));
    if (mode[r] != 0 || yield[r] != INFINITY) c->has_special = true;
  }
  // group sine actuation (modes 1, 2) by (mode, amp, freq, per) for the
  // split fast path of the fp32 mode; group 0 = not actuated, 0 also when
  // the table is full (the spring then takes the exact path).  The mixed
  // mode keeps actuated springs on the exact path: its fp64 sin holds the
  // 1e-9 split-vs-exact bar that the fast path's fp32 sin cannot.
  if (!params_only && !slots) {  // a full upload: groups from scratch
    memset(&c->agrp, 0, sizeof c->agrp);
    c->agrp.n = 1;
    c->agrp.per[0] = 1.0;
    c->agrp.inv_per[0] = 1.0;
  }
  const int groups_before = c->agrp.n;
  std::vector<uint8_t> grp(n, 0);
  for (int64_t r = 0; r < n; r++) {
    if ((mode[r] != 1 && mode[r] != 2) || c->prec != PREC_FP32) continue;
    if (!(per[r] > 0.0) || !std::isfinite(per[r]) || !std::isfinite(freq[r]))
      continue;
    int g = 1;
    for (; g < c->agrp.n; g++)
      if (c->agrp.mode[g] == mode[r] && c->agrp.amp[g] == (float)amp[r] &&
          c->agrp.freq[g] == freq[r] && c->agrp.per[g] == per[r])
        break;
    if (g == c->agrp.n) {
      if (g >= MAX_ACT_GROUPS) continue;
      c->agrp.mode[g] = mode[r];
      c->agrp.amp[g] = (float)amp[r];
      c->agrp.freq[g] = freq[r];
      c->agrp.per[g] = per[r];
      c->agrp.inv_per[g] = 1.0 / per[r];
      c->agrp.n++;
    }
    grp[r] = (uint8_t)g;
  }
  // first actuated group on a live split layout: re-layout with act cells
  if (params_only && groups_before <= 1 && c->agrp.n > 1 && c->split)
    c->layout_valid = false;
  // the window / fused layouts' material tables hold (k, L0) by value:
  // rebuild
  if (params_only && (c->win || c->fz_ok)) c->layout_valid = false;
  size_t need = align256(8 * n) * 16 + align256(n) * 5 + 2048;
  CK(c->stage.ensure(need));
  size_t off = 0;
  const int64_t *dsl = nullptr, *d1 = nullptr, *d2 = nullptr, *dg1 = nullptr,
                *dg2 = nullptr;
  const double *dr, *dk, *dd, *dy, *da, *df, *doff, *dper;
  const int8_t *dmo;
  const uint8_t *dal = nullptr, *dde = nullptr;
  int rc;
  if ((rc = stage_copy(c, off, slots, slots ? n : 0, &dsl))) return rc;
  if (!params_only) {
    if ((rc = stage_copy(c, off, m1, n, &d1))) return rc;
    if ((rc = stage_copy(c, off, m2, n, &d2))) return rc;
    if ((rc = stage_copy(c, off, m1gen, n, &dg1))) return rc;
    if ((rc = stage_copy(c, off, m2gen, n, &dg2))) return rc;
    if ((rc = stage_copy(c, off, alive, n, &dal))) return rc;
    if ((rc = stage_copy(c, off, degen, n, &dde))) return rc;
  }
  if ((rc = stage_copy(c, off, rest, n, &dr))) return rc;
  if ((rc = stage_copy(c, off, k, n, &dk))) return rc;
  if ((rc = stage_copy(c, off, diam, n, &dd))) return rc;
  if ((rc = stage_copy(c, off, yield, n, &dy))) return rc;
  if ((rc = stage_copy(c, off, mode, n, &dmo))) return rc;
  if ((rc = stage_copy(c, off, amp, n, &da))) return rc;
  if ((rc = stage_copy(c, off, freq, n, &df))) return rc;
  if ((rc = stage_copy(c, off, off_, n, &doff))) return rc;
  if ((rc = stage_copy(c, off, per, n, &dper))) return rc;
  const uint8_t *dgrp;
  if ((rc = stage_copy(c, off, grp.data(), n, &dgrp))) return rc;
  if (n > 0) {
    KState S = make_state(c);
    auto kk = c->prec == PREC_FP64   ? k_pack_springs<PREC_FP64>
              : c->prec == PREC_FP32 ? k_pack_springs<PREC_FP32>
                                     : k_pack_springs<PREC_MIXED>;
    kk<<<blocks_for(n), 256, 0, c->st>>>(
        n, dsl, d1, d2, dg1, dg2, dr, dk, dd, dy, dmo, da, df, doff, dper,
        dal, dde, S, c->m1gen.as<int64_t>(), c->m2gen.as<int64_t>(),
        c->mode.as<int8_t>(), c->act.as<double4>(),
        c->s_degen.as<uint8_t>(), c->custom.as<double>(), params_only,
        c->layout_valid, dgrp, c->s_grp.as<uint8_t>());
    CKL();
    c->launches++;
  }
  CK(cudaStreamSynchronize(c->st));
  return SL_OK;
}

int sl_upload_springs(sl_ctx *c, int64_t s_n, const int64_t *m1,
                      const int64_t *m2, const int64_t *m1gen,
                      const int64_t *m2gen, const double *rest,
                      const double *k, const double *diam,
                      const double *yield, const int8_t *mode,
                      const double *amp, const double *freq,
                      const double *off, const double *per,
                      const uint8_t *alive, const uint8_t *degen) {
  SL_RANGE("sl_upload_springs");
  if (!c) return fail(c, SL_EINVAL, "NULL context");
  if (!c->masses_set)
    return fail(c, SL_ESTATE, "upload masses before springs");
  if (s_n < 0 || (s_n > 0 && (!m1 || !m2 || !m1gen || !m2gen || !rest ||
                              !k || !diam || !yield || !mode || !amp ||
                              !freq || !off || !per || !alive || !degen)))
    return fail(c, SL_EINVAL, "sl_upload_springs: bad arguments");
  CK(cudaSetDevice(c->device));
  int rc = ensure_springs(c, s_n);
  if (rc) return rc;
  c->has_special = false;
  c->has_damping = false;  // a full upload clears the dampers (re-sent)
  c->s_n = s_n;
  c->layout_valid = false;
  rc = upload_springs_impl(c, s_n, nullptr, m1, m2, m1gen, m2gen, rest, k,
                           diam, yield, mode, amp, freq, off, per, alive,
                           degen, false);
  if (rc) return rc;
  c->springs_set = true;
  c->validate_dirty = true;
  return SL_OK;
}

// O(edits) re-wiring of a live split + window layout after a record write
// of n slots (k_split_insert, then k_win_build on the touched tiles only).
// Leaves c->layout_valid false -- the full device re-index at the next
// step -- whenever the edit does not fit in place.
static int insert_incremental(sl_ctx *c, int64_t n, const int64_t *slots) {
  const WinCfg &w = c->wcfg;
  const int tt = c->win ? w.tile_slices : 1 << 30;
  CK(c->inc_buf.ensure(align256(8 * n) + align256(32 * n) + 256));
  int64_t *dsl = c->inc_buf.as<int64_t>();
  int32_t *dtiles = (int32_t *)((char *)c->inc_buf.p + align256(8 * n));
  int *dfail = (int *)((char *)dtiles + align256(32 * n));
  CK(cudaMemcpyAsync(dsl, slots, 8 * n, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemsetAsync(dfail, 0, sizeof(int), c->st));
  CK(cudaMemsetAsync(dtiles, 0xFF, 32 * n, c->st));
  KState S = make_state(c);
  S.split = true;
  const bool act = c->agrp.n > 1;
  auto k = c->prec == PREC_FP32 ? k_split_insert<PREC_FP32>
                                : k_split_insert<PREC_MIXED>;
  k<<<1, 32, 0, c->st>>>(n, dsl, S, (int)c->sp_wa, (int)c->sp_wb, tt,
                         act ? c->sp_actc.as<float4>() : nullptr,
                         c->sp_acto.as<double>(), c->s_grp.as<uint8_t>(),
                         dtiles, dfail);
  CKL();
  c->launches++;
  int failed = 0;
  std::vector<int32_t> out(8 * n);
  CK(cudaMemcpyAsync(&failed, dfail, sizeof(int), cudaMemcpyDeviceToHost,
                     c->st));
  CK(cudaMemcpyAsync(out.data(), dtiles, 32 * n, cudaMemcpyDeviceToHost,
                     c->st));
  CK(cudaStreamSynchronize(c->st));
  if (failed) {
    c->layout_valid = false;
    return SL_OK;
  }
  // touched window tiles and fused groups, each once
  std::vector<int32_t> tiles, groups;
  for (int64_t q = 0; q < n; q++)
    for (int u = 0; u < 4; u++) {
      if (out[8 * q + u] >= 0) tiles.push_back(out[8 * q + u]);
      if (out[8 * q + 4 + u] >= 0) groups.push_back(out[8 * q + 4 + u]);
    }
  auto uniq = [](std::vector<int32_t> &v) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  };
  uniq(tiles);
  uniq(groups);
  if (c->win && !tiles.empty()) {
    CK(cudaMemcpyAsync(dtiles, tiles.data(), 4 * tiles.size(),
                       cudaMemcpyHostToDevice, c->st));
    CK(cudaMemsetAsync(c->win_fail.p, 0, 24, c->st));
    const int64_t m_pad = c->n_slices * 32;
    k_win_build<<<(unsigned)tiles.size(), 256, 0, c->st>>>(
        c->sp_j.as<uint32_t>(), c->sp_w.as<uint32_t>(), c->sp_kl.as<float2>(),
        c->n_slices, c->m_n, c->sp_a, c->sp_rows, (uint32_t)m_pad,
        (uint32_t)(c->n_slices << (c->sp_a + 5)), tt, w.bl, w.cap_a, w.cap_b,
        c->sp_s.as<int32_t>(), c->mode.as<int8_t>(), c->act.as<double4>(),
        c->s_grp.as<uint8_t>(), c->win_rec.as<TileRec>(),
        c->win_dict.as<float2>(), c->win_actb.as<unsigned char>(),
        c->win_zero.as<uint8_t>(), c->win_blk.as<unsigned char>(),
        c->prec == PREC_MIXED ? 1 : 0, c->win_fail.as<unsigned long long>(),
        dtiles);
    CKL();
    c->launches++;
    unsigned long long res[3] = {0, 0, 0};
    CK(cudaMemcpyAsync(res, c->win_fail.p, 24, cudaMemcpyDeviceToHost,
                       c->st));
    CK(cudaStreamSynchronize(c->st));
    const bool act_block = w.off_win > w.off_act;
    if (res[0] || res[1] > w.cap_rec || (res[2] && !act_block)) {
      c->layout_valid = false;  // a tile outgrew the stage: full re-index
      return SL_OK;
    }
  }
  if (c->fz_ok && !groups.empty()) {
    // the fused small-body layout: the touched groups re-derived from the
    // split layout (their packing is unchanged: the edit stays inside)
    CK(cudaMemcpyAsync(dtiles, groups.data(), 4 * groups.size(),
                       cudaMemcpyHostToDevice, c->st));
    CK(cudaMemsetAsync(c->fz_fail.p, 0, 8, c->st));
    const int64_t m_pad = c->n_slices * 32;
    const FzCfg &f = c->fcfg;
    auto build = f.maxm > FZ_MAXM ? k_fused_build<FZ_MAXM_L>
                                  : k_fused_build<FZ_MAXM>;
    build<<<(unsigned)groups.size(), f.maxm, 0, c->st>>>(
        c->sp_j.as<uint32_t>(), c->sp_w.as<uint32_t>(), c->sp_kl.as<float2>(),
        c->sp_s.as<int32_t>(), c->mode.as<int8_t>(), c->act.as<double4>(),
        c->s_grp.as<uint8_t>(), c->vel.as<float4>(), c->sp_a, c->sp_rows,
        (uint32_t)m_pad, (uint32_t)(c->n_slices << (c->sp_a + 5)),
        c->fz_gstart.as<int32_t>(), c->fz_gcount.as<int32_t>(), f.ra, f.rb,
        c->fz_ent.as<uint16_t>(), c->fz_code.as<uint8_t>(),
        c->fz_perm.as<uint16_t>(), c->fz_cnt.as<uint8_t>(),
        c->fz_cnt_a.as<uint8_t>(), c->fz_epos.as<uint16_t>(),
        c->fz_dict.as<float2>(), c->fz_actb.as<unsigned char>(),
        c->fz_has.as<uint8_t>(), c->fz_zero.as<uint8_t>(),
        c->fz_gid.as<int32_t>(), c->fz_fail.as<unsigned long long>(),
        dtiles);
    CKL();
    c->launches++;
    unsigned long long ffail = 0;
    CK(cudaMemcpyAsync(&ffail, c->fz_fail.p, 8, cudaMemcpyDeviceToHost,
                       c->st));
    CK(cudaStreamSynchronize(c->st));
    if (ffail) {
      c->layout_valid = false;
      return SL_OK;
    }
  }
  c->inc_edits++;
  return SL_OK;
}

// The same on the EXACT layout (fp64 parity mode): k_exact_insert keeps
// each mass's entries in ascending slot order, then the fp64 window layout
// is re-derived for the touched tiles (k_win64_build over a tile list).
static int insert_incremental_exact(sl_ctx *c, int64_t n,
                                    const int64_t *slots) {
  const WinCfg &w = c->wcfg;
  const int tt = c->win ? w.tile_slices : 1 << 30;
  CK(c->inc_buf.ensure(align256(8 * n) + align256(32 * n) + 256));
  int64_t *dsl = c->inc_buf.as<int64_t>();
  int32_t *dtiles = (int32_t *)((char *)c->inc_buf.p + align256(8 * n));
  int *dfail = (int *)((char *)dtiles + align256(32 * n));
  CK(cudaMemcpyAsync(dsl, slots, 8 * n, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemsetAsync(dfail, 0, sizeof(int), c->st));
  CK(cudaMemsetAsync(dtiles, 0xFF, 32 * n, c->st));
  KState S = make_state(c);
  auto k = c->prec == PREC_FP64   ? k_exact_insert<PREC_FP64>
           : c->prec == PREC_FP32 ? k_exact_insert<PREC_FP32>
                                  : k_exact_insert<PREC_MIXED>;
  k<<<1, 32, 0, c->st>>>(n, dsl, S, tt, dtiles, dfail);
  CKL();
  c->launches++;
  int failed = 0;
  std::vector<int32_t> out(8 * n);
  CK(cudaMemcpyAsync(&failed, dfail, sizeof(int), cudaMemcpyDeviceToHost,
                     c->st));
  CK(cudaMemcpyAsync(out.data(), dtiles, 32 * n, cudaMemcpyDeviceToHost,
                     c->st));
  CK(cudaStreamSynchronize(c->st));
  if (failed) {
    c->layout_valid = false;
    return SL_OK;
  }
  std::vector<int32_t> tiles;
  for (int64_t q = 0; q < n; q++)
    for (int u = 0; u < 4; u++)
      if (out[8 * q + u] >= 0) tiles.push_back(out[8 * q + u]);
  std::sort(tiles.begin(), tiles.end());
  tiles.erase(std::unique(tiles.begin(), tiles.end()), tiles.end());
  if (c->win && !tiles.empty()) {
    CK(cudaMemcpyAsync(dtiles, tiles.data(), 4 * tiles.size(),
                       cudaMemcpyHostToDevice, c->st));
    CK(cudaMemsetAsync(c->win_fail.p, 0, 16, c->st));
    const int64_t m_pad = c->n_slices * 32;
    k_win64_build<<<(unsigned)tiles.size(), 256, 0, c->st>>>(
        S.slice_ptr, c->ent_j.as<uint32_t>(), c->ent_kL0.as<double2>(),
        c->n_slices, c->m_n, (uint32_t)m_pad, tt, w.bl, w.cap_a,
        c->win_rec.as<TileRec>(), c->win_dict.as<double2>(),
        c->win_blk.as<unsigned char>(), c->win_fail.as<unsigned long long>(),
        dtiles);
    CKL();
    c->launches++;
    unsigned long long res[2] = {0, 0};
    CK(cudaMemcpyAsync(res, c->win_fail.p, 16, cudaMemcpyDeviceToHost,
                       c->st));
    CK(cudaStreamSynchronize(c->st));
    if (res[0] || res[1] > w.cap_rec) {
      c->layout_valid = false;  // a tile outgrew the stage: full re-index
      return SL_OK;
    }
  }
  c->inc_edits++;
  return SL_OK;
}

int sl_write_springs(sl_ctx *c, int64_t n, const int64_t *slots,
                     const int64_t *m1, const int64_t *m2,
                     const int64_t *m1gen, const int64_t *m2gen,
                     const double *rest, const double *k, const double *diam,
                     const double *yield, const int8_t *mode,
                     const double *amp, const double *freq, const double *off,
                     const double *per, const uint8_t *alive,
                     const uint8_t *degen) {
  SL_RANGE("sl_write_springs");
  if (!c || !c->springs_set) return fail(c, SL_ESTATE, "no springs");
  if (n < 0 || (n > 0 && (!slots || !m1 || !m2 || !m1gen || !m2gen ||
                          !rest || !k || !diam || !yield || !mode || !amp ||
                          !freq || !off || !per || !alive || !degen)))
    return fail(c, SL_EINVAL, "sl_write_springs: bad arguments");
  for (int64_t r = 0; r < n; r++)
    if (slots[r] < 0 || slots[r] >= c->s_n)
      return fail(c, SL_EINVAL, "spring slot %lld out of range",
                  (long long)slots[r]);
  if (n == 0) return SL_OK;
  CK(cudaSetDevice(c->device));
  // in place when the live layout is the split + window one (the fp32 /
  // mixed production path) and the edit is small; else re-indexed on the
  // device at the next step
  static const bool no_inc = getenv("SL_NO_INCREMENTAL") != nullptr;
  const bool inc = !no_inc && c->layout_valid && c->split &&
                   (c->win || c->fz_ok) && n <= 256;  // (serial insert:
                                                      // above, the
                                                      // re-index is faster)
  const bool inc_exact = !no_inc && c->layout_valid && !c->split &&
                         n <= 256;
  const int groups_before = c->agrp.n;
  c->layout_valid = false;
  int rc = upload_springs_impl(c, n, slots, m1, m2, m1gen, m2gen, rest, k,
                               diam, yield, mode, amp, freq, off, per, alive,
                               degen, false);
  if (rc) return rc;
  if (inc_exact) {
    c->layout_valid = true;
    return insert_incremental_exact(c, n, slots);
  }
  if (!inc || c->agrp.n != groups_before) return rc;
  c->layout_valid = true;
  return insert_incremental(c, n, slots);
}

int sl_write_spring_params(sl_ctx *c, int64_t n, const int64_t *slots,
                           const double *rest, const double *k,
                           const double *diam, const double *yield,
                           const int8_t *mode, const double *amp,
                           const double *freq, const double *off,
                           const double *per) {
  if (!c || !c->springs_set) return fail(c, SL_ESTATE, "no springs");
  if (n < 0 || (n > 0 && (!slots || !rest || !k || !diam || !yield ||
                          !mode || !amp || !freq || !off || !per)))
    return fail(c, SL_EINVAL, "sl_write_spring_params: bad arguments");
  for (int64_t r = 0; r < n; r++)
    if (slots[r] < 0 || slots[r] >= c->s_n)
      return fail(c, SL_EINVAL, "spring slot %lld out of range",
                  (long long)slots[r]);
  // the window layout's material tables hold (k, L0) by value: refreshed
  // for the touched tiles in place (insert_incremental keeps a slot's
  // cells when its endpoints are unchanged), else a full re-index
  static const bool no_inc = getenv("SL_NO_INCREMENTAL") != nullptr;
  const bool inc = !no_inc && c->layout_valid && c->split &&
                   (c->win || c->fz_ok) && n <= 256;  // (serial insert:
                                                      // above, the
                                                      // re-index is faster)
  const bool inc_exact = !no_inc && c->layout_valid && !c->split &&
                         c->win && n <= 256;
  const int groups_before = c->agrp.n;
  int rc = upload_springs_impl(c, n, slots, nullptr, nullptr, nullptr,
                               nullptr, rest, k, diam, yield, mode, amp, freq,
                               off, per, nullptr, nullptr, true);
  if (rc) return rc;
  if (inc_exact) {  // (k, L0) refreshed in place; the tiles' tables
    c->layout_valid = true;
    return insert_incremental_exact(c, n, slots);
  }
  if (!inc || c->agrp.n != groups_before) return rc;
  c->layout_valid = true;
  return insert_incremental(c, n, slots);
}

int sl_kill_springs(sl_ctx *c, int64_t n, const int64_t *slots) {
  SL_RANGE("sl_kill_springs");
  if (!c || !c->springs_set) return fail(c, SL_ESTATE, "no springs");
  if (n <= 0) return SL_OK;
  for (int64_t r = 0; r < n; r++)
    if (slots[r] < 0 || slots[r] >= c->s_n)
      return fail(c, SL_EINVAL, "spring slot %lld out of range",
                  (long long)slots[r]);
  CK(cudaSetDevice(c->device));
  CK(c->stage.ensure(8 * n + 256));
  size_t off = 0;
  const int64_t *ds;
  int rc = stage_copy(c, off, slots, n, &ds);
  if (rc) return rc;
  KState S = make_state(c);
  k_kill_springs<<<blocks_for(n), 256, 0, c->st>>>(n, ds, S, c->layout_valid);
  CKL();
  c->launches++;
  // (the parity-mode window: kill_entries sets the entry words' skip bit;
  // the tiles' windows and tables stay a valid superset)
  CK(cudaStreamSynchronize(c->st));
  return SL_OK;
}

static int write_state_impl(sl_ctx *c, int64_t m_n, const double *pos,
                            const double *vel, const double *acc, bool wait);
int sl_write_state(sl_ctx *c, int64_t m_n, const double *pos,
                   const double *vel, const double *acc) {
  return write_state_impl(c, m_n, pos, vel, acc, true);
}
int sl_write_state_async(sl_ctx *c, int64_t m_n, const double *pos,
                         const double *vel, const double *acc) {
  return write_state_impl(c, m_n, pos, vel, acc, false);
}
static int write_state_impl(sl_ctx *c, int64_t m_n, const double *pos,
                            const double *vel, const double *acc, bool wait) {
  if (!c || !c->masses_set) return fail(c, SL_ESTATE, "no masses");
  if (m_n != c->m_n)
    return fail(c, SL_EINVAL, "sl_write_state: %lld masses, context has %lld",
                (long long)m_n, (long long)c->m_n);
  if (c->async_open)
    return fail(c, SL_ESTATE, "asynchronous run open (sl_step_finish)");
  if (m_n == 0 || (!pos && !vel && !acc)) return SL_OK;
  CK(cudaSetDevice(c->device));
  CK(c->stage.ensure(3 * align256(24 * m_n) + 1024));
  size_t off = 0;
  const double *dp, *dv, *da;
  int rc;
  if ((rc = stage_copy(c, off, pos, 3 * m_n, &dp))) return rc;
  if ((rc = stage_copy(c, off, vel, 3 * m_n, &dv))) return rc;
  if ((rc = stage_copy(c, off, acc, 3 * m_n, &da))) return rc;
  auto k = c->prec == PREC_FP64   ? k_write_state<PREC_FP64>
           : c->prec == PREC_FP32 ? k_write_state<PREC_FP32>
                                  : k_write_state<PREC_MIXED>;
  k<<<blocks_for(m_n), 256, 0, c->st>>>(m_n, dp, dv, da, c->pos[0].p,
                                        c->pos[1].p, c->plo[0].p, c->plo[1].p,
                                        c->vel.p, c->acc.p);
  CKL();
  c->launches++;
  // staging is reused by the next call (which is stream-ordered after this
  // one); the synchronous form also releases the caller's host arrays
  if (wait) CK(cudaStreamSynchronize(c->st));
  return SL_OK;
}

int sl_write_masses(sl_ctx *c, int64_t n, const int64_t *slots,
                    const double *pos, const double *vel, const double *acc,
                    const double *fext, const double *load,
                    const double *mass, const uint8_t *fixed,
                    const uint8_t *alive, const int64_t *gen) {
  if (!c || !c->masses_set) return fail(c, SL_ESTATE, "no masses");
  if (n < 0 || (n > 0 && (!slots || !pos || !vel || !acc || !fext || !load ||
                          !mass || !fixed || !alive || !gen)))
    return fail(c, SL_EINVAL, "sl_write_masses: bad arguments");
  if (n == 0) return SL_OK;
  for (int64_t r = 0; r < n; r++)
    if (slots[r] < 0 || slots[r] >= c->m_n)
      return fail(c, SL_EINVAL, "mass slot %lld out of range",
                  (long long)slots[r]);
  CK(cudaSetDevice(c->device));
  CK(c->stage.ensure(align256(24 * n) * 5 + align256(8 * n) * 3 +
                     align256(n) * 2 + 1024));
  size_t off = 0;
  const double *dp, *dv, *da, *df, *dl, *dm;
  const uint8_t *dfx, *dal;
  const int64_t *dg, *ds;
  int rc;
  if ((rc = stage_copy(c, off, slots, n, &ds))) return rc;
  if ((rc = stage_copy(c, off, pos, 3 * n, &dp))) return rc;
  if ((rc = stage_copy(c, off, vel, 3 * n, &dv))) return rc;
  if ((rc = stage_copy(c, off, acc, 3 * n, &da))) return rc;
  if ((rc = stage_copy(c, off, fext, 3 * n, &df))) return rc;
  if ((rc = stage_copy(c, off, load, 3 * n, &dl))) return rc;
  if ((rc = stage_copy(c, off, mass, n, &dm))) return rc;
  if ((rc = stage_copy(c, off, fixed, n, &dfx))) return rc;
  if ((rc = stage_copy(c, off, alive, n, &dal))) return rc;
  if ((rc = stage_copy(c, off, gen, n, &dg))) return rc;
  auto k = c->prec == PREC_FP64   ? k_pack_masses<PREC_FP64>
           : c->prec == PREC_FP32 ? k_pack_masses<PREC_FP32>
                                  : k_pack_masses<PREC_MIXED>;
  // write the current buffer and its partner (static masses are never
  // rewritten by the step kernels, so both halves must agree)
  k<<<blocks_for(n), 256, 0, c->st>>>(
      n, dp, dv, da, df, dl, dm, dfx, dal, ds, c->pos[0].p, c->pos[1].p,
      c->plo[0].p, c->plo[1].p, c->pmass.as<float>(), c->vel.p, c->acc.p,
      c->fext.p, c->load.p, c->m_gen.as<int64_t>(),
      c->m_alive.as<uint8_t>(), dg,
      c->layout_valid ? c->xflags.as<uint8_t>() : nullptr);
  CKL();
  c->launches++;
  CK(cudaStreamSynchronize(c->st));
  c->validate_dirty = true;
  return SL_OK;
}

int sl_set_environment(sl_ctx *c, const double *gravity, double drag,
                       const double *planes, int64_t n_planes,
                       const double *balls, int64_t n_balls,
                       const int8_t *gc_kind, const double *gc_vec,
                       int64_t n_gc, double v_stick) {
  if (!c) return fail(c, SL_EINVAL, "NULL context");
  if (!gravity) return fail(c, SL_EINVAL, "gravity is NULL");
  if (n_planes < 0 || n_planes > MAXP || n_balls < 0 || n_balls > MAXB ||
      n_gc < 0 || n_gc > MAXG)
    return fail(c, SL_EUNSUPPORTED,
                "environment too large (planes<=%d balls<=%d global<=%d)",
                MAXP, MAXB, MAXG);
  EnvP &E = c->env;
  memset(&E, 0, sizeof E);
  for (int q = 0; q < 3; q++) E.g[q] = gravity[q];
  E.drag = drag;
  E.v_stick = v_stick;
  E.np = (int)n_planes;
  E.nb = (int)n_balls;
  E.ngc = (int)n_gc;
  for (int p = 0; p < n_planes; p++)
    for (int q = 0; q < 7; q++) E.pl[p][q] = planes[7 * p + q];
  for (int b = 0; b < n_balls; b++)
    for (int q = 0; q < 5; q++) E.bl[b][q] = balls[5 * b + q];
  for (int g = 0; g < n_gc; g++) {
    E.gck[g] = gc_kind[g];
    for (int q = 0; q < 3; q++) E.gcv[g][q] = gc_vec[3 * g + q];
  }
  auto f32 = [](double x) {  // (float) x, denormals flushed as under -ftz
    const float f = (float)x;
    return std::fpclassify(f) == FP_SUBNORMAL ? std::copysign(0.0f, f) : f;
  };
  for (int q = 0; q < 3; q++) E.gf[q] = f32(E.g[q]);
  E.dragf = f32(drag);
  E.v_stickf = f32(v_stick);
  for (int p = 0; p < n_planes; p++)
    for (int q = 0; q < 7; q++) E.plf[p][q] = f32(E.pl[p][q]);
  c->env_set = true;
  return SL_OK;
}

int sl_set_local_constraints(sl_ctx *c, int64_t m_n, const int64_t *lc_off,
                             const int8_t *lc_kind, const double *lc_vec,
                             int64_t n_lc) {
  if (!c || !c->masses_set) return fail(c, SL_ESTATE, "upload masses first");
  if (m_n != c->m_n) return fail(c, SL_EINVAL, "lc_off must have m_n+1 rows");
  CK(cudaSetDevice(c->device));
  if (n_lc <= 0 || !lc_off) {
    c->has_lc = false;
    if (m_n > 0) {
      k_set_lc_flags<<<blocks_for(m_n), 256, 0, c->st>>>(m_n, nullptr,
                                                         c->vel.p, c->rsz == 8);
      CKL();
    }
    CK(cudaStreamSynchronize(c->st));
    return SL_OK;
  }
  CK(c->lc_off.ensure(8 * (m_n + 1)));
  CK(c->lc_kind.ensure(n_lc));
  CK(c->lc_vec.ensure(24 * n_lc));
  CK(cudaMemcpyAsync(c->lc_off.p, lc_off, 8 * (m_n + 1),
                     cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(c->lc_kind.p, lc_kind, n_lc, cudaMemcpyHostToDevice,
                     c->st));
  CK(cudaMemcpyAsync(c->lc_vec.p, lc_vec, 24 * n_lc, cudaMemcpyHostToDevice,
                     c->st));
  c->has_lc = true;
  if (m_n > 0) {
    k_set_lc_flags<<<blocks_for(m_n), 256, 0, c->st>>>(
        m_n, c->lc_off.as<int64_t>(), c->vel.p, c->rsz == 8);
    CKL();
  }
  CK(cudaStreamSynchronize(c->st));
  return SL_OK;
}

int sl_set_spring_damping(sl_ctx *c, int64_t n, const double *damping) {
  if (!c || !c->springs_set) return fail(c, SL_ESTATE, "no springs");
  if (n != c->s_n || (n > 0 && !damping))
    return fail(c, SL_EINVAL, "sl_set_spring_damping: need s_n values");
  bool any = false;
  for (int64_t r = 0; r < n; r++) {
    if (!(damping[r] >= 0.0) || !std::isfinite(damping[r]))
      return fail(c, SL_EINVAL, "damping of spring %lld must be finite and "
                  ">= 0, got %g", (long long)r, damping[r]);
    any |= damping[r] != 0.0;
  }
  CK(cudaSetDevice(c->device));
  if (any) {
    CK(c->damp.ensure(8 * n));
    CK(cudaMemcpyAsync(c->damp.p, damping, 8 * n, cudaMemcpyHostToDevice,
                       c->st));
    CK(cudaStreamSynchronize(c->st));
  }
  // damped springs take the exact per-entry path: the special flags of the
  // incidence layouts change, so the layout is rebuilt at the next step
  if (any || c->has_damping) c->layout_valid = false;
  c->has_damping = any;
  c->has_special |= any;
  return SL_OK;
}

int sl_set_custom_factors(sl_ctx *c, int64_t n, const int64_t *slots,
                          const double *factors) {
  if (!c || !c->springs_set) return fail(c, SL_ESTATE, "no springs");
  if (n <= 0) return SL_OK;
  CK(cudaSetDevice(c->device));
  CK(c->stage.ensure(align256(8 * n) * 2 + 512));
  size_t off = 0;
  const int64_t *ds;
  const double *df;
  int rc;
  if ((rc = stage_copy(c, off, slots, n, &ds))) return rc;
  if ((rc = stage_copy(c, off, factors, n, &df))) return rc;
  k_set_custom<<<blocks_for(n), 256, 0, c->st>>>(n, ds, df,
                                                 c->custom.as<double>());
  CKL();
  c->launches++;
  CK(cudaStreamSynchronize(c->st));
  return SL_OK;
}

// Halo step boundary: publish "my step k's ghost stores are done" to every
// peer (system-scope fence + release store of k into the peer's counter
// word for me), then wait until every peer has published k.  One block;
// thread t serves peer t.  Never triggers dependents early: the next step
// kernel starts after the wait.
__global__ void k_halo_sync(const HaloDesc *H, unsigned long long k) {
  const int t = threadIdx.x;
  if (t < H->n_peers) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(H->flag_out[t]),
                 "l"(k)
                 : "memory");
    unsigned long long v = 0;
    do {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];"
                   : "=l"(v)
                   : "l"(H->flag_in + t)
                   : "memory");
      if (v < k) __nanosleep(100);
    } while (v < k);
  }
  __syncthreads();
}

static void halo_sync(sl_ctx *c) {
  c->halo_step++;
  k_halo_sync<<<1, 32, 0, c->st>>>(c->halo_desc.as<HaloDesc>(), c->halo_step);
  c->launches++;
}

int sl_step(sl_ctx *c, int64_t n_steps, const double *sim_times, double dt,
            int accumulation, int64_t *counters, int64_t *err_slot,
            int64_t *steps_done) {
  SL_RANGE("sl_step");
  if (!c) return fail(c, SL_EINVAL, "NULL context");
  if (n_steps < 0 || (n_steps > 0 && !sim_times))
    return fail(c, SL_EINVAL, "sl_step: bad arguments");
  if (!(dt > 0) || !std::isfinite(dt))
    return fail(c, SL_EINVAL, "dt must be positive, got %g", dt);
  if (accumulation != SL_ACC_GATHER && accumulation != SL_ACC_ATOMIC &&
      accumulation != SL_ACC_AUTO)
    return fail(c, SL_EINVAL, "unknown accumulation %d", accumulation);
  if (err_slot) *err_slot = 0;
  if (steps_done) *steps_done = 0;
  if (c->async_open)
    return fail(c, SL_ESTATE, "asynchronous run open (sl_step_finish)");
  CK(cudaSetDevice(c->device));
  int rc = prepare(c, true);  // gather and owner-atomic use the layout
  if (rc) return rc;
  accumulation = resolve_accumulation(c, accumulation);
  const Launch &L = launchers(c->prec);
  KState S = make_state(c);
  if ((rc = upload_state(c, S))) return rc;
  if (accumulation == SL_ACC_GATHER && c->fz_ok && !c->has_ghost &&
      !c->has_damping && n_steps >= 2) {
    // small bodies: all n steps in one launch, state on chip
    bool aborted = false;
    if ((rc = run_fused(c, S, n_steps, sim_times, dt, &aborted))) return rc;
    if (!aborted) {
      // no spring events / errors inside the fused launch (eligibility);
      // the counters are prepare's invalid-endpoint kills of this call
      if (counters)
        for (int q = 0; q < 3; q++) counters[q] += (int64_t)c->h_status[q];
      if (steps_done) *steps_done = n_steps;
      return SL_OK;
    }
  }
  c->k_valid = false;
  // diagnostic (SL_FIRST_STEP_MS=1): the first step's device time apart
  static cudaEvent_t first_ev = [] {
    cudaEvent_t e = nullptr;
    if (getenv("SL_FIRST_STEP_MS")) cudaEventCreate(&e);
    return e;
  }();
  CK(cudaEventRecord(c->k0, c->st));
  for (int64_t n = 0; n < n_steps; n++) {
    StepP T;
    T.sim_t = sim_times[n];
    T.dt = dt;
    T.step = n;
    T.cur = (int)((c->cur + n) & 1);
    // accelerations are stored on the last step of a batch -- and on every
    // step in fp64 parity mode, so a numerical abort at any step leaves the
    // aborting step's accelerations, as the reference's mass pass does
    // (kernels.py:368-376)
    T.write_acc = n == n_steps - 1 || c->prec == PREC_FP64;
    T.early = n > 0;
    if (accumulation == SL_ACC_GATHER && c->has_damping) {
      // dampers read neighbour velocities: the force pass (into f_ext) and
      // the mass pass as two kernels, gather order kept
      if (c->split)
        L.split_force(S, c->env, T, c->agrp, c->st);
      else
        L.force_only(S, c->env, T, c->st);
      L.mass(S, c->env, T, c->st);
      c->launches += 2;
    } else if (accumulation == SL_ACC_GATHER) {
      if (c->split) {
        if (c->win)
          L.win(S, c->env, T, c->wcfg, c->win_grid, c->st);
        else if (c->split_warps)
          L.split_tma(S, c->env, T, c->scfg, c->agrp, c->split_grid, c->st);
        else
          L.split(S, c->env, T, c->agrp, c->st);
      } else if (c->win) {
        L.win(S, c->env, T, c->wcfg, c->win_grid, c->st);
      } else if (c->tma_warps) {
        L.gather_tma(S, c->env, T, c->tma, c->tma_grid, c->st);
      } else {
        L.gather(S, c->env, T, c->st);
      }
      c->launches++;
    } else {
      if (c->atomic_owner)
        L.owner_atomic(S, T, c->agrp, c->st);
      else
        L.spring_atomic(S, T, c->has_special, c->st);
      L.mass(S, c->env, T, c->st);
      c->launches += 2;
    }
    if (c->halo_on) halo_sync(c);
    if (n == 0 && first_ev) CK(cudaEventRecord(first_ev, c->st));
  }
  CKL();
  CK(cudaEventRecord(c->k1, c->st));
  c->k_valid = true;
  int64_t err = 0;
  if ((rc = finish_status(c, counters, &err))) return rc;
  if (first_ev && n_steps > 1) {  // SL_FIRST_STEP_MS: diagnostic split
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, c->k0, first_ev);
    cudaEventElapsedTime(&b, first_ev, c->k1);
    fprintf(stderr, "sl_step: first step %.2f us, later steps %.2f us each\n",
            1e3 * a, 1e3 * b / (double)(n_steps - 1));
  }
  int64_t done = n_steps;
  if (c->h_status[4]) done = (int64_t)c->h_status[4];
  c->cur = (int)((c->cur + done) & 1);
  if (steps_done) *steps_done = done;
  if (err_slot) *err_slot = err;
  if (err) return fail(c, SL_ENUMERIC, "non-finite state on mass slot %lld",
                       (long long)(err - 1));
  return SL_OK;
}

int sl_spring_pass(sl_ctx *c, double sim_t, int accumulation,
                   int64_t *counters) {
  if (!c) return fail(c, SL_EINVAL, "NULL context");
  CK(cudaSetDevice(c->device));
  int rc = prepare(c, accumulation != SL_ACC_ATOMIC);
  if (rc) return rc;
  accumulation = resolve_accumulation(c, accumulation);
  const Launch &L = launchers(c->prec);
  KState S = make_state(c);
  if ((rc = upload_state(c, S))) return rc;
  StepP T;
  T.sim_t = sim_t;
  T.dt = 0.0;
  T.step = 0;
  T.cur = c->cur;
  T.write_acc = 0;
  T.early = 0;
  if (accumulation == SL_ACC_GATHER) {
    if (c->split)
      L.split_force(S, c->env, T, c->agrp, c->st);
    else
      L.force_only(S, c->env, T, c->st);
    c->launches++;
  } else {
    L.spring_atomic(S, T, c->has_special, c->st);
    if (c->m_n > 0)
      k_set_fext_flags<<<blocks_for(c->m_n), 256, 0, c->st>>>(c->m_n, c->vel.p,
                                                            c->rsz == 8);
    c->launches += 2;
  }
  CKL();
  return finish_status(c, counters, nullptr);
}

int sl_mass_pass(sl_ctx *c, double dt, int64_t *err_slot) {
  if (!c) return fail(c, SL_EINVAL, "NULL context");
  if (!(dt > 0)) return fail(c, SL_EINVAL, "dt must be positive");
  CK(cudaSetDevice(c->device));
  int rc = prepare(c, false);
  if (rc) return rc;
  KState S = make_state(c);
  StepP T;
  T.sim_t = 0.0;
  T.dt = dt;
  T.step = 0;
  T.cur = c->cur;
  T.write_acc = 1;
  T.early = 0;
  launchers(c->prec).mass(S, c->env, T, c->st);
  c->launches++;
  CKL();
  int64_t err = 0;
  if ((rc = finish_status(c, nullptr, &err))) return rc;
  c->cur ^= 1;
  if (err_slot) *err_slot = err;
  if (err) return fail(c, SL_ENUMERIC, "non-finite state on mass slot %lld",
                       (long long)(err - 1));
  return SL_OK;
}

int sl_energy(sl_ctx *c, double sim_t, const double *gravity,
              double *out) {
  SL_RANGE("sl_energy");
  if (!c || !gravity || !out) return fail(c, SL_EINVAL, "sl_energy: NULL");
  if (!c->masses_set || !c->springs_set)
    return fail(c, SL_ESTATE, "masses and springs must be uploaded first");
  CK(cudaSetDevice(c->device));
  CK(c->diag.ensure(8 * 3 * DIAG_BLOCKS));
  KState S = make_state(c);
  auto k = c->prec == PREC_FP64   ? k_energy<PREC_FP64>
           : c->prec == PREC_FP32 ? k_energy<PREC_FP32>
                                  : k_energy<PREC_MIXED>;
  k<<<DIAG_BLOCKS, DIAG_THREADS, 0, c->st>>>(S, c->cur, gravity[0],
                                             gravity[1], gravity[2], sim_t,
                                             c->diag.as<double>());
  CKL();
  c->launches++;
  std::vector<double> part(3 * DIAG_BLOCKS);
  CK(cudaMemcpyAsync(part.data(), c->diag.p, 8 * 3 * DIAG_BLOCKS,
                     cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  double ke = 0.0, gp = 0.0, sp = 0.0;
  for (int b = 0; b < DIAG_BLOCKS; b++) {
    ke += part[3 * b];
    gp += part[3 * b + 1];
    sp += part[3 * b + 2];
  }
  out[0] = 0.5 * ke;  // kinetic
  out[1] = 0.5 * sp;  // spring potential
  out[2] = -gp;       // gravitational potential (origin reference)
  return SL_OK;
}

int sl_spring_loads(sl_ctx *c, double sim_t, double *lengths,
                    double *force_magnitudes) {
  SL_RANGE("sl_spring_loads");
  if (!c || !lengths || !force_magnitudes)
    return fail(c, SL_EINVAL, "sl_spring_loads: NULL");
  if (!c->masses_set || !c->springs_set)
    return fail(c, SL_ESTATE, "masses and springs must be uploaded first");
  const int64_t n = c->s_n;
  if (n == 0) return SL_OK;
  CK(cudaSetDevice(c->device));
  CK(c->diag.ensure(16 * n));
  KState S = make_state(c);
  auto k = c->prec == PREC_FP64   ? k_spring_loads<PREC_FP64>
           : c->prec == PREC_FP32 ? k_spring_loads<PREC_FP32>
                                  : k_spring_loads<PREC_MIXED>;
  double *d = c->diag.as<double>();
  k<<<blocks_for(n), 256, 0, c->st>>>(S, c->cur, sim_t, d, d + n);
  CKL();
  c->launches++;
  CK(cudaMemcpyAsync(lengths, d, 8 * n, cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(force_magnitudes, d + n, 8 * n, cudaMemcpyDeviceToHost,
                     c->st));
  CK(cudaStreamSynchronize(c->st));
  return SL_OK;
}

int sl_download_masses(sl_ctx *c, double *pos, double *vel, double *acc,
                       double *fext) {
  SL_RANGE("sl_download_masses");
  if (!c || !c->masses_set) return fail(c, SL_ESTATE, "no masses");
  const int64_t m = c->m_n;
  if (m == 0) return SL_OK;
  CK(cudaSetDevice(c->device));
  size_t vb = align256(24 * m);
  CK(c->stage.ensure(4 * vb));
  double *dp = pos ? (double *)c->stage.p : nullptr;
  double *dv = vel ? (double *)((char *)c->stage.p + vb) : nullptr;
  double *da = acc ? (double *)((char *)c->stage.p + 2 * vb) : nullptr;
  double *df = fext ? (double *)((char *)c->stage.p + 3 * vb) : nullptr;
  auto k = c->prec == PREC_FP64   ? k_unpack_masses<PREC_FP64>
           : c->prec == PREC_FP32 ? k_unpack_masses<PREC_FP32>
                                  : k_unpack_masses<PREC_MIXED>;
  k<<<blocks_for(m), 256, 0, c->st>>>(m, c->pos[c->cur].p,
                                      c->plo[c->cur].p, c->vel.p, c->acc.p,
                                      c->fext.p, dp, dv, da, df);
  CKL();
  c->launches++;
  if (pos) CK(cudaMemcpyAsync(pos, dp, 24 * m, cudaMemcpyDeviceToHost, c->st));
  if (vel) CK(cudaMemcpyAsync(vel, dv, 24 * m, cudaMemcpyDeviceToHost, c->st));
  if (acc) CK(cudaMemcpyAsync(acc, da, 24 * m, cudaMemcpyDeviceToHost, c->st));
  if (fext)
    CK(cudaMemcpyAsync(fext, df, 24 * m, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  return SL_OK;
}

int sl_download_state(sl_ctx *c, double *pos, double *vel, double *acc,
                      double *fext) {
  if (!c || !c->masses_set) return fail(c, SL_ESTATE, "no masses");
  const int64_t m = c->m_n;
  if (m == 0) return SL_OK;
  CK(cudaSetDevice(c->device));
  size_t vb = align256(24 * m);
  CK(c->stage.ensure(4 * vb));
  double *dp = pos ? (double *)c->stage.p : nullptr;
  double *dv = vel ? (double *)((char *)c->stage.p + vb) : nullptr;
  double *da = acc ? (double *)((char *)c->stage.p + 2 * vb) : nullptr;
  double *df = fext ? (double *)((char *)c->stage.p + 3 * vb) : nullptr;
  auto k = c->prec == PREC_FP64   ? k_unpack_masses<PREC_FP64>
           : c->prec == PREC_FP32 ? k_unpack_masses<PREC_FP32>
                                  : k_unpack_masses<PREC_MIXED>;
  k<<<blocks_for(m), 256, 0, c->st>>>(m, c->pos[c->cur].p,
                                      c->plo[c->cur].p, c->vel.p, c->acc.p,
                                      c->fext.p, dp, dv, da, df);
  CKL();
  c->launches++;
  if (pos) CK(cudaMemcpyAsync(pos, dp, 24 * m, cudaMemcpyDeviceToHost, c->st));
  if (vel) CK(cudaMemcpyAsync(vel, dv, 24 * m, cudaMemcpyDeviceToHost, c->st));
  CK(cudaEventRecord(c->head_ev, c->st));
  if (acc) CK(cudaMemcpyAsync(acc, da, 24 * m, cudaMemcpyDeviceToHost, c->st));
  if (fext)
    CK(cudaMemcpyAsync(fext, df, 24 * m, cudaMemcpyDeviceToHost, c->st));
  CK(cudaEventRecord(c->tail_ev, c->st));
  c->tail_pending = acc || fext;
  CK(cudaEventSynchronize(c->head_ev));  // positions / velocities landed
  return SL_OK;
}

int sl_download_state_ex(sl_ctx *c, double *pos, double *vel, double *acc,
                         double *fext, double *pos2, double *vel2,
                         int wait_head) {
  SL_RANGE("sl_download_state_ex");
  if (!c || !c->masses_set) return fail(c, SL_ESTATE, "no masses");
  const int64_t m = c->m_n;
  if (m == 0) return SL_OK;
  if (c->tail_pending) CK(cudaEventSynchronize(c->tail_ev));
  c->tail_pending = false;
  CK(cudaSetDevice(c->device));
  size_t vb = align256(24 * m);
  CK(c->stage.ensure(4 * vb));
  const bool want_p = pos || pos2, want_v = vel || vel2;
  double *dp = want_p ? (double *)c->stage.p : nullptr;
  double *dv = want_v ? (double *)((char *)c->stage.p + vb) : nullptr;
  double *da = acc ? (double *)((char *)c->stage.p + 2 * vb) : nullptr;
  double *df = fext ? (double *)((char *)c->stage.p + 3 * vb) : nullptr;
  auto k = c->prec == PREC_FP64   ? k_unpack_masses<PREC_FP64>
           : c->prec == PREC_FP32 ? k_unpack_masses<PREC_FP32>
                                  : k_unpack_masses<PREC_MIXED>;
  k<<<blocks_for(m), 256, 0, c->st>>>(m, c->pos[c->cur].p,
                                      c->plo[c->cur].p, c->vel.p, c->acc.p,
                                      c->fext.p, dp, dv, da, df);
  CKL();
  c->launches++;
  // the extra destinations first (a snapshot waits for them alone), then
  // the primary positions / velocities, then accelerations and f_ext
  if (pos2) CK(cudaMemcpyAsync(pos2, dp, 24 * m, cudaMemcpyDeviceToHost, c->st));
  if (vel2) CK(cudaMemcpyAsync(vel2, dv, 24 * m, cudaMemcpyDeviceToHost, c->st));
  CK(cudaEventRecord(c->extra_ev, c->st));
  if (pos) CK(cudaMemcpyAsync(pos, dp, 24 * m, cudaMemcpyDeviceToHost, c->st));
  if (vel) CK(cudaMemcpyAsync(vel, dv, 24 * m, cudaMemcpyDeviceToHost, c->st));
  CK(cudaEventRecord(c->head_ev, c->st));
  if (acc) CK(cudaMemcpyAsync(acc, da, 24 * m, cudaMemcpyDeviceToHost, c->st));
  if (fext)
    CK(cudaMemcpyAsync(fext, df, 24 * m, cudaMemcpyDeviceToHost, c->st));
  CK(cudaEventRecord(c->tail_ev, c->st));
  c->tail_pending = true;
  if (wait_head) CK(cudaEventSynchronize(c->head_ev));
  return SL_OK;
}

int sl_stash_state(sl_ctx *c) {
  if (!c || !c->masses_set) return fail(c, SL_ESTATE, "no masses");
  const int64_t m = c->m_n;
  if (m == 0) return SL_OK;
  CK(cudaSetDevice(c->device));
  const size_t vb = align256(24 * m);
  // a previous stash may still be read by sl_download_stash (side stream)
  if (c->side_pending) CK(cudaEventSynchronize(c->side_done));
  c->side_pending = false;
  CK(c->stage2.ensure(4 * vb));
  char *b = (char *)c->stage2.p;
  auto k = c->prec == PREC_FP64   ? k_unpack_masses<PREC_FP64>
           : c->prec == PREC_FP32 ? k_unpack_masses<PREC_FP32>
                                  : k_unpack_masses<PREC_MIXED>;
  k<<<blocks_for(m), 256, 0, c->st>>>(
      m, c->pos[c->cur].p, c->plo[c->cur].p, c->vel.p, c->acc.p, c->fext.p,
      (double *)b, (double *)(b + vb), (double *)(b + 2 * vb),
      (double *)(b + 3 * vb));
  CKL();
  c->launches++;
  CK(cudaEventRecord(c->side_ev, c->st));
  c->stash_set = true;
  return SL_OK;
}

int sl_checkpoint(sl_ctx *c, double *view_pos, double *view_vel) {
  SL_RANGE("sl_checkpoint");
  if (!c || !c->masses_set) return fail(c, SL_ESTATE, "no masses");
  if (c->async_open)
    return fail(c, SL_ESTATE, "asynchronous run open (sl_step_finish)");
  const int64_t m = c->m_n;
  CK(cudaSetDevice(c->device));
  const int64_t mp = (m + 31) / 32 * 32 + 32;
  const size_t r4 = 4 * c->rsz;
  CK(c->ck_pos.ensure(r4 * mp));
  CK(c->ck_vel.ensure(r4 * (m + 32)));
  CK(c->ck_acc.ensure(3 * c->rsz * m + 16));
  CK(c->ck_fext.ensure(r4 * m + 16));
  auto d2d = [&](DevBuf &dst, const void *src, size_t bytes) -> int {
    if (bytes)
      CK(cudaMemcpyAsync(dst.p, src, bytes, cudaMemcpyDeviceToDevice, c->st));
    return SL_OK;
  };
  int rc;
  if ((rc = d2d(c->ck_pos, c->pos[c->cur].p, r4 * mp))) return rc;
  if (c->prec == PREC_FP32) {
    CK(c->ck_plo.ensure(8 * mp));
    if ((rc = d2d(c->ck_plo, c->plo[c->cur].p, 8 * mp))) return rc;
  }
  if ((rc = d2d(c->ck_vel, c->vel.p, r4 * (m + 32)))) return rc;
  if ((rc = d2d(c->ck_acc, c->acc.p, 3 * c->rsz * m))) return rc;
  if ((rc = d2d(c->ck_fext, c->fext.p, r4 * m))) return rc;
  c->ck_cur = c->cur;
  if (m && (view_pos || view_vel)) {  // the predicate's view, side stream
    if (c->ck_pending) CK(cudaEventSynchronize(c->ck_done));
    const size_t vb = align256(24 * m);
    CK(c->ck_view.ensure(2 * vb));
    char *b = (char *)c->ck_view.p;
    auto k = c->prec == PREC_FP64   ? k_unpack_masses<PREC_FP64>
             : c->prec == PREC_FP32 ? k_unpack_masses<PREC_FP32>
                                    : k_unpack_masses<PREC_MIXED>;
    k<<<blocks_for(m), 256, 0, c->st>>>(
        m, c->pos[c->cur].p, c->plo[c->cur].p, c->vel.p, nullptr, nullptr,
        view_pos ? (double *)b : nullptr,
        view_vel ? (double *)(b + vb) : nullptr, nullptr, nullptr);
    CKL();
    c->launches++;
    CK(cudaEventRecord(c->ck_ev, c->st));
    CK(cudaStreamWaitEvent(c->side, c->ck_ev, 0));
    if (view_pos)
      CK(cudaMemcpyAsync(view_pos, b, 24 * m, cudaMemcpyDeviceToHost,
                         c->side));
    if (view_vel)
      CK(cudaMemcpyAsync(view_vel, b + vb, 24 * m, cudaMemcpyDeviceToHost,
                         c->side));
    CK(cudaEventRecord(c->ck_done, c->side));
    c->ck_pending = true;
  }
  return SL_OK;
}

int sl_checkpoint_view_wait(sl_ctx *c) {
  if (!c) return fail(c, SL_EINVAL, "NULL context");
  if (!c->ck_pending) return SL_OK;
  CK(cudaSetDevice(c->device));
  CK(cudaEventSynchronize(c->ck_done));
  c->ck_pending = false;
  return SL_OK;
}

int sl_restore(sl_ctx *c) {
  SL_RANGE("sl_restore");
  if (!c || c->ck_cur < 0) return fail(c, SL_ESTATE, "no checkpoint");
  if (c->async_open)
    return fail(c, SL_ESTATE, "asynchronous run open (sl_step_finish)");
  CK(cudaSetDevice(c->device));
  const int64_t m = c->m_n;
  const int64_t mp = (m + 31) / 32 * 32 + 32;
  const size_t r4 = 4 * c->rsz;
  const int b = c->ck_cur;
  CK(cudaMemcpyAsync(c->pos[b].p, c->ck_pos.p, r4 * mp,
                     cudaMemcpyDeviceToDevice, c->st));
  if (c->prec == PREC_FP32)
    CK(cudaMemcpyAsync(c->plo[b].p, c->ck_plo.p, 8 * mp,
                       cudaMemcpyDeviceToDevice, c->st));
  CK(cudaMemcpyAsync(c->vel.p, c->ck_vel.p, r4 * (m + 32),
                     cudaMemcpyDeviceToDevice, c->st));
  if (m) {
    CK(cudaMemcpyAsync(c->acc.p, c->ck_acc.p, 3 * c->rsz * m,
                       cudaMemcpyDeviceToDevice, c->st));
    CK(cudaMemcpyAsync(c->fext.p, c->ck_fext.p, r4 * m,
                       cudaMemcpyDeviceToDevice, c->st));
  }
  c->cur = b;
  CK(cudaStreamSynchronize(c->st));
  return SL_OK;
}

int sl_download_stash(sl_ctx *c, double *pos, double *vel, double *acc,
                      double *fext) {
  if (!c || !c->stash_set) return fail(c, SL_ESTATE, "no stashed state");
  const int64_t m = c->m_n;
  if (m == 0) return SL_OK;
  CK(cudaSetDevice(c->device));
  const size_t vb = align256(24 * m);
  const char *b = (const char *)c->stage2.p;
  CK(cudaStreamWaitEvent(c->side, c->side_ev, 0));
  double *dst[4] = {pos, vel, acc, fext};
  for (int q = 0; q < 4; q++)
    if (dst[q])
      CK(cudaMemcpyAsync(dst[q], b + q * vb, 24 * m, cudaMemcpyDeviceToHost,
                         c->side));
  CK(cudaEventRecord(c->side_done, c->side));
  CK(cudaEventSynchronize(c->side_done));
  return SL_OK;
}

int sl_download_wait_extra(sl_ctx *c) {
  if (!c) return fail(c, SL_EINVAL, "NULL context");
  CK(cudaSetDevice(c->device));
  CK(cudaEventSynchronize(c->extra_ev));
  return SL_OK;
}

int sl_download_wait(sl_ctx *c) {
  if (!c) return fail(c, SL_EINVAL, "NULL context");
  if (!c->tail_pending) return SL_OK;
  CK(cudaSetDevice(c->device));
  CK(cudaEventSynchronize(c->tail_ev));
  c->tail_pending = false;
  return SL_OK;
}

int sl_download_springs(sl_ctx *c, uint8_t *alive, uint8_t *degen) {
  if (!c || !c->springs_set) return fail(c, SL_ESTATE, "no springs");
  if (c->s_n == 0) return SL_OK;
  CK(cudaSetDevice(c->device));
  if (alive)
    CK(cudaMemcpyAsync(alive, c->s_alive.p, c->s_n, cudaMemcpyDeviceToHost,
                       c->st));
  if (degen)
    CK(cudaMemcpyAsync(degen, c->s_degen.p, c->s_n, cudaMemcpyDeviceToHost,
                       c->st));
  CK(cudaStreamSynchronize(c->st));
  return SL_OK;
}

int sl_snapshot_begin(sl_ctx *c) {
  SL_RANGE("sl_snapshot_begin");
  if (!c || !c->masses_set) return fail(c, SL_ESTATE, "no masses");
  const int64_t m = c->m_n;
  CK(cudaSetDevice(c->device));
  if (c->snap_pending) CK(cudaEventSynchronize(c->snap_done));
  size_t bytes = 48 * (size_t)m + 16;
  CK(c->snap_dev.ensure(bytes));
  if (c->snap_host_bytes < bytes) {
    if (c->snap_host) cudaFreeHost(c->snap_host);
    c->snap_host = nullptr;
    c->snap_host_bytes = 0;
    CK(cudaMallocHost((void **)&c->snap_host, bytes));
    c->snap_host_bytes = bytes;
  }
  if (m > 0) {
    auto k = c->prec == PREC_FP64   ? k_unpack_masses<PREC_FP64>
             : c->prec == PREC_FP32 ? k_unpack_masses<PREC_FP32>
                                    : k_unpack_masses<PREC_MIXED>;
    double *dp = (double *)c->snap_dev.p;
    k<<<blocks_for(m), 256, 0, c->st>>>(m, c->pos[c->cur].p,
                                        c->plo[c->cur].p, c->vel.p, nullptr,
                                        nullptr, dp, dp + 3 * m, nullptr,
                                        nullptr);
    CKL();
    c->launches++;
  }
  CK(cudaEventRecord(c->snap_ev, c->st));
  CK(cudaStreamWaitEvent(c->side, c->snap_ev, 0));
  if (m > 0)
    CK(cudaMemcpyAsync(c->snap_host, c->snap_dev.p, 48 * m,
                       cudaMemcpyDeviceToHost, c->side));
  CK(cudaEventRecord(c->snap_done, c->side));
  c->snap_m = m;
  c->snap_pending = true;
  return SL_OK;
}

int sl_snapshot_ready(sl_ctx *c, int *ready) {
  if (!c || !ready) return fail(c, SL_EINVAL, "NULL argument");
  if (!c->snap_pending) return fail(c, SL_ESTATE, "no snapshot in flight");
  cudaError_t e = cudaEventQuery(c->snap_done);
  if (e == cudaErrorNotReady) {
    *ready = 0;
    return SL_OK;
  }
  CK(e);
  *ready = 1;
  return SL_OK;
}

int sl_snapshot_wait(sl_ctx *c, double *pos, double *vel) {
  if (!c) return fail(c, SL_EINVAL, "NULL context");
  if (!c->snap_pending) return fail(c, SL_ESTATE, "no snapshot in flight");
  CK(cudaEventSynchronize(c->snap_done));
  const int64_t m = c->snap_m;
  if (pos) memcpy(pos, c->snap_host, 24 * m);
  if (vel) memcpy(vel, c->snap_host + 3 * m, 24 * m);
  c->snap_pending = false;
  return SL_OK;
}

// Enqueue the launches of n steps starting at run-relative step index base
// (the loop of sl_step without the final synchronisation).
static int enqueue_steps(sl_ctx *c, const KState &S, int64_t n_steps,
                         const double *sim_times, double dt,
                         int accumulation, int64_t base, int cur0) {
  const Launch &L = launchers(c->prec);
  for (int64_t n = 0; n < n_steps; n++) {
    StepP T;
    T.sim_t = sim_times[n];
    T.dt = dt;
    T.step = base + n;
    T.cur = (int)((cur0 + n) & 1);
    T.write_acc = 1;
    T.early = n > 0;  // a foreign launch (halo) may precede this chunk
    if (accumulation == SL_ACC_GATHER && c->has_damping) {
      // dampers read neighbour velocities: the force pass (into f_ext) and
      // the mass pass as two kernels, gather order kept
      if (c->split)
        L.split_force(S, c->env, T, c->agrp, c->st);
      else
        L.force_only(S, c->env, T, c->st);
      L.mass(S, c->env, T, c->st);
      c->launches += 2;
    } else if (accumulation == SL_ACC_GATHER) {
      if (c->split) {
        if (c->win)
          L.win(S, c->env, T, c->wcfg, c->win_grid, c->st);
        else if (c->split_warps)
          L.split_tma(S, c->env, T, c->scfg, c->agrp, c->split_grid, c->st);
        else
          L.split(S, c->env, T, c->agrp, c->st);
      } else if (c->win) {
        L.win(S, c->env, T, c->wcfg, c->win_grid, c->st);
      } else if (c->tma_warps) {
        L.gather_tma(S, c->env, T, c->tma, c->tma_grid, c->st);
      } else {
        L.gather(S, c->env, T, c->st);
      }
      c->launches++;
    } else {
      if (c->atomic_owner)
        L.owner_atomic(S, T, c->agrp, c->st);
      else
        L.spring_atomic(S, T, c->has_special, c->st);
      L.mass(S, c->env, T, c->st);
      c->launches += 2;
    }
    if (c->halo_on) halo_sync(c);
  }
  CKL();
  return SL_OK;
}

int sl_step_async(sl_ctx *c, int64_t n_steps, const double *sim_times,
                  double dt, int accumulation) {
  SL_RANGE("sl_step_async");
  if (!c) return fail(c, SL_EINVAL, "NULL context");
  if (n_steps < 0 || (n_steps > 0 && !sim_times))
    return fail(c, SL_EINVAL, "sl_step_async: bad arguments");
  if (!(dt > 0) || !std::isfinite(dt))
    return fail(c, SL_EINVAL, "dt must be positive, got %g", dt);
  if (accumulation != SL_ACC_GATHER && accumulation != SL_ACC_ATOMIC &&
      accumulation != SL_ACC_AUTO)
    return fail(c, SL_EINVAL, "unknown accumulation %d", accumulation);
  CK(cudaSetDevice(c->device));
  int rc = prepare(c, true, !c->async_open);
  if (rc) return rc;
  accumulation = resolve_accumulation(c, accumulation);
  if (!c->async_open) {
    c->async_open = true;
    c->async_steps = 0;
    c->async_cur0 = c->cur;
  }
  KState S = make_state(c);
  if ((rc = upload_state(c, S))) return rc;
  rc = enqueue_steps(c, S, n_steps, sim_times, dt, accumulation,
                     c->async_steps, c->cur);
  if (rc) return rc;
  c->async_steps += n_steps;
  c->cur = (int)((c->cur + n_steps) & 1);
  return SL_OK;
}

int sl_step_finish(sl_ctx *c, int64_t *counters, int64_t *err_slot,
                   int64_t *steps_done) {
  if (!c) return fail(c, SL_EINVAL, "NULL context");
  if (err_slot) *err_slot = 0;
  if (steps_done) *steps_done = 0;
  if (!c->async_open) return SL_OK;
  CK(cudaSetDevice(c->device));
  c->async_open = false;
  int64_t err = 0;
  int rc = finish_status(c, counters, &err);
  if (rc) return rc;
  int64_t done = c->async_steps;
  if (c->h_status[4]) done = (int64_t)c->h_status[4];
  c->cur = (int)((c->async_cur0 + done) & 1);
  if (steps_done) *steps_done = done;
  if (err_slot) *err_slot = err;
  if (err) return fail(c, SL_ENUMERIC, "non-finite state on mass slot %lld",
                       (long long)(err - 1));
  return SL_OK;
}

__global__ void k_set_ghosts(int64_t n, const int64_t *slots, uint8_t *g) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) g[slots[r]] = 1;
}

int sl_mark_ghosts(sl_ctx *c, int64_t n, const int64_t *slots) {
  if (!c || !c->masses_set) return fail(c, SL_ESTATE, "no masses");
  if (n < 0 || (n > 0 && !slots))
    return fail(c, SL_EINVAL, "sl_mark_ghosts: bad arguments");
  for (int64_t r = 0; r < n; r++)
    if (slots[r] < 0 || slots[r] >= c->m_n)
      return fail(c, SL_EINVAL, "mass slot %lld out of range",
                  (long long)slots[r]);
  CK(cudaSetDevice(c->device));
  CK(c->ghost.ensure(c->m_n + 1));
  CK(cudaMemsetAsync(c->ghost.p, 0, c->m_n + 1, c->st));
  if (n > 0) {
    CK(c->stage.ensure(8 * n + 256));
    size_t off = 0;
    const int64_t *ds;
    int rc = stage_copy(c, off, slots, n, &ds);
    if (rc) return rc;
    k_set_ghosts<<<blocks_for(n), 256, 0, c->st>>>(n, ds,
                                                   c->ghost.as<uint8_t>());
    CKL();
    c->launches++;
  }
  CK(cudaStreamSynchronize(c->st));
  c->has_ghost = n > 0;
  return SL_OK;
}

// ------------------------------------------------ in-library halo (config E)
int sl_halo_init(sl_ctx *c, int n_peers, const int32_t *dst) {
  if (!c || !c->masses_set) return fail(c, SL_ESTATE, "no masses");
  if (n_peers < 0 || n_peers > HALO_MAXP || (c->m_n > 0 && !dst))
    return fail(c, SL_EINVAL, "sl_halo_init: 0..%d peers", HALO_MAXP);
  for (int64_t r = 0; r < 2 * c->m_n; r++)
    if (dst[r] >= 0 && (dst[r] & 7) >= n_peers)
      return fail(c, SL_EINVAL, "halo destination %lld: peer out of range",
                  (long long)r);
  CK(cudaSetDevice(c->device));
  CK(c->halo_flags.ensure(8 * HALO_MAXP));
  CK(cudaMemset(c->halo_flags.p, 0, 8 * HALO_MAXP));
  CK(c->halo_dst.ensure(8 * std::max<int64_t>(c->m_n, 1)));
  if (c->m_n > 0)
    CK(cudaMemcpy(c->halo_dst.p, dst, 8 * c->m_n, cudaMemcpyHostToDevice));
  CK(c->halo_desc.ensure(sizeof(HaloDesc)));
  memset(&c->halo_host, 0, sizeof c->halo_host);
  c->halo_host.n_peers = n_peers;
  c->halo_host.flag_in = c->halo_flags.as<unsigned long long>();
  c->halo_host.dst = c->halo_dst.as<int2>();
  c->halo_on = false;
  c->halo_step = 0;
  return SL_OK;
}

int sl_halo_local(sl_ctx *c, void **ptrs) {
  if (!c || !c->masses_set || !c->halo_flags.p)
    return fail(c, SL_ESTATE, "sl_halo_init first");
  ptrs[0] = c->pos[0].p;
  ptrs[1] = c->pos[1].p;
  ptrs[2] = c->prec == PREC_FP32 ? c->plo[0].p : nullptr;
  ptrs[3] = c->prec == PREC_FP32 ? c->plo[1].p : nullptr;
  ptrs[4] = c->halo_flags.p;
  return SL_OK;
}

int sl_halo_ipc_handles(sl_ctx *c, void *out) {
  void *p[5];
  int rc = sl_halo_local(c, p);
  if (rc) return rc;
  CK(cudaSetDevice(c->device));
  unsigned char *o = (unsigned char *)out;
  memset(o, 0, 5 * SL_IPC_HANDLE_BYTES);
  for (int q = 0; q < 5; q++) {
    if (!p[q]) continue;
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, p[q]));
    memcpy(o + q * SL_IPC_HANDLE_BYTES, &h, sizeof h);
  }
  return SL_OK;
}

int sl_halo_ipc_open(sl_ctx *c, const void *handles, void **ptrs) {
  if (!c || !handles || !ptrs) return fail(c, SL_EINVAL, "NULL argument");
  CK(cudaSetDevice(c->device));
  const unsigned char *in = (const unsigned char *)handles;
  static const unsigned char zero[SL_IPC_HANDLE_BYTES] = {0};
  for (int q = 0; q < 5; q++) {
    ptrs[q] = nullptr;
    if (!memcmp(in + q * SL_IPC_HANDLE_BYTES, zero, SL_IPC_HANDLE_BYTES))
      continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, in + q * SL_IPC_HANDLE_BYTES, sizeof h);
    CK(cudaIpcOpenMemHandle(&ptrs[q], h, cudaIpcMemLazyEnablePeerAccess));
    c->halo_ipc.push_back(ptrs[q]);
  }
  return SL_OK;
}

int sl_halo_set_peer(sl_ctx *c, int peer, void *const *ptrs, int slot) {
  if (!c || !ptrs || peer < 0 || peer >= c->halo_host.n_peers || slot < 0 ||
      slot >= HALO_MAXP)
    return fail(c, SL_EINVAL, "sl_halo_set_peer: bad arguments");
  if (!ptrs[0] || !ptrs[1] || !ptrs[4] ||
      (c->prec == PREC_FP32 && (!ptrs[2] || !ptrs[3])))
    return fail(c, SL_EINVAL, "sl_halo_set_peer: missing peer buffers");
  HaloDesc &h = c->halo_host;
  h.pos[peer][0] = ptrs[0];
  h.pos[peer][1] = ptrs[1];
  h.lo[peer][0] = ptrs[2];
  h.lo[peer][1] = ptrs[3];
  h.flag_out[peer] = (unsigned long long *)ptrs[4] + slot;
  return SL_OK;
}

int sl_halo_commit(sl_ctx *c) {
  if (!c || !c->halo_desc.p) return fail(c, SL_ESTATE, "sl_halo_init first");
  const HaloDesc &h = c->halo_host;
  for (int q = 0; q < h.n_peers; q++)
    if (!h.pos[q][0] || !h.flag_out[q])
      return fail(c, SL_ESTATE, "halo peer %d not set", q);
  if (c->has_damping)
    return fail(c, SL_EUNSUPPORTED,
                "damped springs read ghost velocities, which the halo does "
                "not carry");
  CK(cudaSetDevice(c->device));
  CK(cudaMemcpy(c->halo_desc.p, &h, sizeof h, cudaMemcpyHostToDevice));
  c->halo_on = h.n_peers > 0;
  c->halo_step = 0;
  return SL_OK;
}

int sl_state_pointers(sl_ctx *c, void **pos_read, int64_t *rows,
                      int32_t *record_bytes) {
  if (!c || !c->masses_set) return fail(c, SL_ESTATE, "no masses");
  if (pos_read) *pos_read = c->pos[c->cur].p;
  if (rows) *rows = (int64_t)(c->pos[c->cur].bytes / (4 * c->rsz));
  if (record_bytes) *record_bytes = (int32_t)(4 * c->rsz);
  return SL_OK;
}

int sl_state_lo(sl_ctx *c, void **lo_read) {
  if (!c || !c->masses_set) return fail(c, SL_ESTATE, "no masses");
  if (lo_read) *lo_read = c->prec == PREC_FP32 ? c->plo[c->cur].p : nullptr;
  return SL_OK;
}

int sl_get_stream(sl_ctx *c, void **stream) {
  if (!c || !stream) return fail(c, SL_EINVAL, "NULL argument");
  *stream = (void *)c->st;
  return SL_OK;
}

int sl_timer_start(sl_ctx *c) {
  if (!c) return fail(c, SL_EINVAL, "NULL context");
  CK(cudaEventRecord(c->t0, c->st));
  return SL_OK;
}

int sl_timer_stop(sl_ctx *c, float *ms) {
  if (!c || !ms) return fail(c, SL_EINVAL, "NULL argument");
  CK(cudaEventRecord(c->t1, c->st));
  CK(cudaEventSynchronize(c->t1));
  CK(cudaEventElapsedTime(ms, c->t0, c->t1));
  return SL_OK;
}

int sl_last_step_ms(sl_ctx *c, float *ms) {
  if (!c || !ms) return fail(c, SL_EINVAL, "NULL argument");
  if (!c->k_valid) return fail(c, SL_ESTATE, "no sl_step call timed yet");
  CK(cudaEventSynchronize(c->k1));
  CK(cudaEventElapsedTime(ms, c->k0, c->k1));
  return SL_OK;
}

int sl_sync(sl_ctx *c) {
  if (!c) return fail(c, SL_EINVAL, "NULL context");
  CK(cudaStreamSynchronize(c->st));
  return SL_OK;
}

}  // extern "C"
