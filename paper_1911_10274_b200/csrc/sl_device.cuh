// sl_device.cuh -- device-side types and kernel templates for the
// spring-mass step (sm_100a).
//
// Semantics follow the reference kernels (/root/reference/pkg/src/softlat/
// kernels.py); the code is a B200-first re-design, not a translation:
//
//   * Mass state is resident in HBM as 16/32-byte records:
//       pos[2][M] = (x, y, z, m)        -- ping-pong: step n reads buffer
//                                          (cur+n)&1, writes the other, so
//                                          the barrier invariant of
//                                          engine.py:5-7 holds inside one
//                                          fused kernel
//       vel[M]    = (vx, vy, vz, flags)  -- flags packed in the spare lane
//   * Deterministic accumulation ("gather", == reference slotted/serial
//     order, engine.py:105-118) uses a per-mass incidence list in a sliced
//     ELL layout: slice = 32 consecutive masses = one warp; entry t of lane l
//     lives at slice_ptr[w] + 32*t + l so every warp-wide load of the list is
//     one contiguous 128/256-byte transaction.  Entries of a mass appear in
//     ascending spring slot, so the per-mass sum has exactly the serial
//     operation order (bit-exact in fp64).  Each entry carries the other
//     endpoint and a copy of (k, L0); the spring force is recomputed at both
//     endpoints (identical inputs -> identical bits), which removes the
//     scatter, the atomics and the f_ext round trip entirely: one kernel per
//     step does spring pass + mass pass.
//   * "atomic" accumulation (reference linearizable) = one thread per
//     spring, red.global vector atomics into f_ext, then a mass kernel.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cooperative_groups.h>
#include <cooperative_groups/reduce.h>
#include <math_constants.h>

namespace sl {

enum : int { PREC_FP64 = 0, PREC_FP32 = 1, PREC_MIXED = 2 };

// mass flag bits (packed into vel[i].w)
enum : uint32_t {
  MF_ALIVE = 1u,
  MF_FIXED = 2u,
  MF_LC = 4u,     // has local constraints (CSR lookup needed)
  MF_LOAD = 8u,   // persistent load has non-zero bits
  MF_FEXT = 16u,  // f_ext accumulator has non-zero bits at step start
  MF_SPECIAL = 32u,  // has actuated / breakable springs (exact entry path)
};

// incidence entry word: low 29 bits other endpoint
enum : uint32_t {
  EJ_MASK = 0x1FFFFFFFu,
  EJ_SPECIAL = 1u << 29,  // actuated or finite yield: per-slot lookup
  EJ_M2 = 1u << 30,       // this mass is endpoint m2: subtract the force
  EJ_DEAD = 1u << 31,     // dead spring or padding
};
constexpr uint32_t EJ_PAD = 0xFFFFFFFFu;

constexpr int MAXP = 8;  // contact planes
constexpr int MAXB = 8;  // contact balls
constexpr int MAXG = 4;  // global constraints

struct EnvP {
  double g[3];
  double drag;
  double v_stick;
  int np, nb, ngc, pad_;
  double pl[MAXP][7];
  double bl[MAXB][5];
  double gcv[MAXG][3];
  int gck[MAXG];
  // fp32 copies (rounded once on the host, denormals flushed as the -ftz
  // fp32 unit would): the per-mass update reads them directly instead of
  // converting the fp64 parameters for every mass
  float gf[3], dragf, v_stickf;
  float plf[MAXP][7];
};
// environment parameter in the mass update's arithmetic type
template <class R>
__device__ __forceinline__ R env_g(const EnvP &E, int q) {
  if constexpr (sizeof(R) == 4) return E.gf[q]; else return (R)E.g[q];
}
template <class R>
__device__ __forceinline__ R env_pl(const EnvP &E, int p, int q) {
  if constexpr (sizeof(R) == 4) return E.plf[p][q]; else return (R)E.pl[p][q];
}

// Halo of a mass-range partition (config E): the owning
// rank's step kernel, as it stores an owned boundary mass's new position,
// also stores it straight into the ghost row of every peer that needs it --
// the peers' position buffers are mapped into this process (CUDA IPC over
// NVLink, or plain pointers between contexts of one process), so the
// exchange rides on the mass update itself, tile by tile.  After each step
// a one-block kernel (k_halo_sync, sl_api.cu) publishes a per-peer step
// counter with a system-scope release and waits for the peers' counters:
// the next step reads complete ghost rows.
constexpr int HALO_MAXP = 8;
struct HaloDesc {
  int n_peers;
  void *pos[HALO_MAXP][2];  // peer's position record buffers (mapped)
  void *lo[HALO_MAXP][2];   // peer's fp32 low parts (mapped) or null
  unsigned long long *flag_out[HALO_MAXP];  // our counter word at the peer
  unsigned long long *flag_in;  // [HALO_MAXP] the peers' counters (local)
  const int2 *dst;  // per local mass: up to two (row << 3 | peer), -1 none
};

// All device pointers of one context (type-erased; kernels cast).
struct KState {
  int64_t m_n, s_n;
  void *pos[2];
  void *plo[2];  // fp32: position low parts (ly, lz) float2 per mass (the
                 // record's w holds lx, see lo_at); null in fp64 / mixed
  const float *pmass;  // fp32: masses (the record's w is lx); else null
  void *vel;
  void *acc;   // R[3*m_n]
  void *fext;  // R4[m_n]
  const void *load;  // R[3*m_n]
  const int64_t *lc_off;
  const int8_t *lc_kind;
  const double *lc_vec;
  // spring SoA by slot
  int2 *ends;          // (m1, m2); x < 0 => dead
  const void *kL0;     // F2 (k, rest)
  uint8_t *s_alive;
  uint8_t *s_degen;
  const int8_t *mode;
  const double4 *act;  // (amp, freq, off, per)
  const void *thr;     // F: yield * area, +inf if no yield
  const double *custom;
  // per-spring damping c (N s / m) of the opt-in damper along the spring
  // (north_star "Hooke plus damping"; no reference counterpart,
  // kernels.py:66 is Hooke only); null when every spring has c = 0.
  // Damped springs are special (exact per-entry path) and a damped context
  // steps force pass + mass pass as two kernels (no in-place velocity race)
  const double *damp;
  // incidence layout
  const int64_t *slice_ptr;
  uint32_t *ent_j;
  const void *ent_kL0;  // F2
  const int32_t *ent_s;
  const int64_t *e1, *e2;
  uint8_t *xflags;  // per-mass layout-derived flag bits (MF_SPECIAL)
  // ghost masses of a partitioned run (partition.py): spring side effects
  // are counted only where the m1 endpoint is owned; null when no ghosts
  const uint8_t *ghost;
  const HaloDesc *halo;  // partitioned run with the in-library halo
  // split layout (tolerance modes, sl_split.cuh); split == 0 => exact layout
  const KState *self;  // device-memory copy of this struct (rare paths)
  int split;
  int fsz8;        // sizeof(F) == 8 (fp64 spring parameters)
  int sp_a;        // log2 of the A-section row stride
  int sp_rows;     // rows per slice block (A stride + widest B section)
  uint32_t sp_sent;  // sentinel mass index (dead / padding A entries)
  uint32_t sp_null;  // zero (k, L0) cell (dead / padding B entries)
  uint32_t *sp_j;
  const void *sp_kl;
  const int32_t *sp_s;
  const uint32_t *sp_w;
  const uint32_t *sp_ekl;  // per spring: kl index of its A cell
  float4 *sp_actc;         // act cell per kl cell (null: no groups)
  double *sp_acto;         // exact fp64 act offset per kl cell
  // tiled window layout (sl_window.cuh; null when not built): the slice
  // blocks (A / B code rows at win_oac / win_obc) and each tile's zero code
  unsigned char *win_blk;
  const uint8_t *win_zero;
  uint32_t win_sb;  // split-window slice block bytes (entry words)
  int win_tt;
  // multi-step fused groups (sl_fused.cuh; null when not built): material
  // codes [group][rows][maxm], group of every mass, group starts / zero codes
  uint8_t *fz_code;
  const uint16_t *fz_epos;  // split row of a mass -> compacted row, thread
  const int32_t *fz_gid, *fz_gstart;
  const uint8_t *fz_zero;
  int fz_rows, fz_ra, fz_maxm;
  // status: [0..2] counters, [3] err_slot (max slot+1), [4] err step+1
  unsigned long long *status;
};

struct StepP {
  double sim_t;
  double dt;
  int64_t step;   // index within the current sl_step call
  int cur;        // pos buffer read this step
  int write_acc;  // store acceleration (final step of a launch)
  // the previous launch on the stream is a step kernel of this same call
  // on the same layout (host-set): the window kernel may then request its
  // first tile's layout data before the grid-dependency wait
  int early;
};

// fp64 / mixed state: a position is its R4 record alone
struct NoLo {};
template <int P>
struct Tr;
template <>
struct Tr<PREC_FP64> {
  using L = NoLo;
  using R = double;
  using F = double;
  using R4 = double4;
  using F2 = double2;
  using M = double;  // force arithmetic
  static constexpr int U = 4;
  static constexpr int UP = 4;  // gather batch (registers: 4 x 52 B)
};
template <>
struct Tr<PREC_FP32> {
  using L = float3;  // compensated positions: x = hi + lo
  using R = float;
  using F = float;
  using R4 = float4;
  using F2 = float2;
  using M = float;
  static constexpr int U = 8;
  static constexpr int UP = 11;  // pipelined batch (2 in flight)
};
template <>
struct Tr<PREC_MIXED> {
  using L = NoLo;
  using R = double;
  using F = float;
  using R4 = double4;
  using F2 = float2;
  using M = double;  // fp32 storage of (k, L0), fp64 force arithmetic
  static constexpr int U = 6;
  static constexpr int UP = 6;
};

// read-only 16/32-byte loads through the non-coherent path
__device__ __forceinline__ float4 ldg4(const float4 *p) { return __ldg(p); }
__device__ __forceinline__ double4 ldg4(const double4 *p) {
  const double2 a = __ldg((const double2 *)p);
  const double2 b = __ldg((const double2 *)p + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

__device__ __forceinline__ uint32_t flags_of(float w) {
  return __float_as_uint(w);
}
__device__ __forceinline__ uint32_t flags_of(double w) {
  return (uint32_t)__double_as_longlong(w);
}
__device__ __forceinline__ void set_flags(float &w, uint32_t f) {
  w = __uint_as_float(f);
}
__device__ __forceinline__ void set_flags(double &w, uint32_t f) {
  w = __longlong_as_double((long long)f);
}
// atomically OR flag bits into vel[i].w (flags live in the low 32 bits)
__device__ __forceinline__ void or_flags(float4 *v, uint32_t f) {
  atomicOr((unsigned int *)&v->w, f);
}
__device__ __forceinline__ void or_flags(double4 *v, uint32_t f) {
  atomicOr((unsigned int *)&v->w, f);
}

// ---------------------------------------------------------------------------
// fp32 mode: compensated positions.  A position is hi + lo, hi the fp32
// coordinates and lo their rounding residuals, all fp32:
//   pos[b][i] = (x_hi, y_hi, z_hi, lz)   plo[b][i] = (lx, ly)
// (the mass lives in pmass).  Spring vectors are formed as
// (o_hi - me_hi) + (o_lo - me_lo): the first difference is exact for
// neighbouring masses (Sterbenz), so |d| carries ~2^-48 of |x| instead of
// fp32's 2^-24 -- the spurious strain of a rounded position (ulp 6e-8 m at
// |x| ~ 1 m, 1.2e-4 m at |x| ~ 1 km, times k) no longer exists, which is
// what holds fp32 velocities to 1e-4 of the fp64 reference.
// The position update is a two-sum (integrate_vals).
// lo of mass j whose record is o (fp32; an empty value otherwise)
template <int P>
__device__ __forceinline__ typename Tr<P>::L lo_at(
    const typename Tr<P>::R4 &o, const void *plo, int64_t j) {
  if constexpr (P == PREC_FP32) {
    const float2 b = __ldg((const float2 *)plo + j);
    return make_float3(b.x, b.y, o.w);
  } else {
    return {};
  }
}
// mass of mass i (fp32: pmass; else the record's w)
template <int P>
__device__ __forceinline__ typename Tr<P>::R mass_of(
    const KState &S, const typename Tr<P>::R4 &me, int64_t i) {
  if constexpr (P == PREC_FP32)
    return __ldg(S.pmass + i);
  else
    return me.w;
}
// d = (o + o_lo) - (me + me_lo), in the force arithmetic type M
template <int P, class M>
__device__ __forceinline__ void pdiff(const typename Tr<P>::R4 &me,
                                      const typename Tr<P>::L &ml,
                                      const typename Tr<P>::R4 &o,
                                      const typename Tr<P>::L &ol, M &dx,
                                      M &dy, M &dz) {
  if constexpr (P == PREC_FP32) {
    dx = (o.x - me.x) + (ol.x - ml.x);
    dy = (o.y - me.y) + (ol.y - ml.y);
    dz = (o.z - me.z) + (ol.z - ml.z);
  } else {
    dx = (M)(o.x - me.x);
    dy = (M)(o.y - me.y);
    dz = (M)(o.z - me.z);
  }
}
// exact sum hi + t as (s, e), s = fl(hi + t) (Knuth's two-sum)
__device__ __forceinline__ float two_sum(float a, float b, float &e) {
  const float s = __fadd_rn(a, b);
  const float bb = __fsub_rn(s, a);
  e = __fadd_rn(__fsub_rn(a, __fsub_rn(s, bb)), __fsub_rn(b, bb));
  return s;
}

// Python float % (CPython float_rem, which numba follows; kernels.py:58).
__device__ __forceinline__ double py_mod(double a, double b) {
  double r = fmod(a, b);
  if (r != 0.0) {
    if ((r < 0.0) != (b < 0.0)) r += b;
  } else {
    r = copysign(0.0, b);
  }
  return r;
}

// kernels.py:55-65 (fp64 always: the phase wraps sim time of arbitrary size)
__device__ __forceinline__ double act_factor(const KState &S, int64_t s,
                                             double sim_t) {
  int m = S.mode[s];
  if (m == 1 || m == 2) {
    double4 a = S.act[s];  // amp, freq, off, per
    if (m == 2 && !(sim_t >= a.z)) return 1.0;
    double t = py_mod(sim_t - a.z, a.w);
    return 1.0 + a.x * sin(a.y * t);
  }
  if (m == 3) return S.custom[s];
  return 1.0;
}

__device__ __forceinline__ bool stopped(const KState &S, int64_t step) {
  // a strictly earlier step of this launch went non-finite: do nothing
  // (written only by earlier launches -- every caller reads it after
  // griddepcontrol.wait -- so the read-only path sees it, and every warp
  // after an SM's first hits L1, instead of a volatile system-scope
  // LDG.STRONG.SYS per thread to one L2 line)
  const unsigned long long e =
      __ldg((const unsigned long long *)(S.status + 4));
  return e != 0ull && (int64_t)e - 1 < step;
}

__device__ __forceinline__ void count(const KState &S, int which) {
  atomicAdd(S.status + which, 1ull);
}
// count a spring event unless the spring's m1 endpoint is a ghost (the
// owning rank counts it); m1 = ends[s].x, read before a kill clears it
__device__ __forceinline__ void count_spring(const KState &S, int which,
                                             int64_t s) {
  if (!S.ghost || !S.ghost[S.ends[s].x]) atomicAdd(S.status + which, 1ull);
}

__device__ __forceinline__ void mark_nonfinite(const KState &S, int64_t i,
                                               int64_t step) {
  atomicMax(S.status + 3, (unsigned long long)(i + 1));
  *(volatile unsigned long long *)(S.status + 4) =
      (unsigned long long)(step + 1);
}

// vector atomics into f_ext (sm_90+: red.global.add.v4.f32)
__device__ __forceinline__ void red_add(float4 *p, float x, float y,
                                        float z) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p),
               "f"(x), "f"(y), "f"(z), "f"(0.0f)
               : "memory");
}
__device__ __forceinline__ void red_add(double4 *p, double x, double y,
                                        double z) {
  atomicAdd(&p->x, x);
  atomicAdd(&p->y, y);
  atomicAdd(&p->z, z);
}

// Warp-aggregated reduction into f_ext[target]: the converged lanes of the
// warp are partitioned by target mass (match-any); each partition sums its
// contributions with shuffles and its first lane issues ONE vector RED.
// Hub meshes (a star's spokes: consecutive slots, one shared endpoint) turn
// 32 same-address atomics into one; without duplicates (lattices in slot
// order: consecutive springs have distinct endpoints) the warp takes the
// plain RED after a single vote.
template <class R4, class R>
__device__ __forceinline__ void red_add_agg(R4 *fe, uint32_t target, R x,
                                            R y, R z) {
  namespace cg = cooperative_groups;
  const cg::coalesced_group g = cg::coalesced_threads();
  const cg::coalesced_group part = cg::labeled_partition(g, target);
  if (g.all(part.size() == 1)) {  // no shared target in this warp
    red_add(fe + target, x, y, z);
    return;
  }
  const R sx = cg::reduce(part, x, cg::plus<R>());
  const R sy = cg::reduce(part, y, cg::plus<R>());
  const R sz = cg::reduce(part, z, cg::plus<R>());
  if (part.thread_rank() == 0) red_add(fe + target, sx, sy, sz);
}

// ---------------------------------------------------------------------------
// Mass pass body (kernels.py:271-376), shared by the fused gather step and
// the standalone mass kernel.  (fx, fy, fz) enters as the accumulated f_ext.
// Writes pos_next / vel / acc; returns false on non-finite state.
// integrate_vals: the new position (xyz, mass in w), velocity (xyz) and
// acceleration of mass i, nothing stored; integrate(): the same plus the
// stores and the non-finite check of the per-step kernels.
template <int P>
__device__ __forceinline__ void integrate_vals(
    const KState &S, const EnvP &E, double dt_, int64_t i,
    typename Tr<P>::R4 me, typename Tr<P>::L lo, typename Tr<P>::R mm,
    typename Tr<P>::R4 v, uint32_t fl, typename Tr<P>::R fx,
    typename Tr<P>::R fy, typename Tr<P>::R fz, typename Tr<P>::R4 &np4,
    typename Tr<P>::L &nlo, typename Tr<P>::R4 &nv, typename Tr<P>::R &ax,
    typename Tr<P>::R &ay, typename Tr<P>::R &az) {
  using R = typename Tr<P>::R;
  R px = me.x, py = me.y, pz = me.z;
  R vx = v.x, vy = v.y, vz = v.z;
  // F = ((f_ext + load) + m*g) - drag*v; an all-zero load adds +0.0, which
  // keeps the sign-of-zero behaviour of the reference's addition.
  if (fl & MF_LOAD) {
    const R *ld = (const R *)S.load + 3 * i;
    fx = fx + ld[0];
    fy = fy + ld[1];
    fz = fz + ld[2];
  } else {
    fx = fx + (R)0.0;
    fy = fy + (R)0.0;
    fz = fz + (R)0.0;
  }
  fx = fx + mm * env_g<R>(E, 0);
  fy = fy + mm * env_g<R>(E, 1);
  fz = fz + mm * env_g<R>(E, 2);
  const R drag = sizeof(R) == 4 ? (R)E.dragf : (R)E.drag;
  fx = fx - drag * vx;
  fy = fy - drag * vy;
  fz = fz - drag * vz;
  // contact planes with Coulomb friction on the running force
  for (int p = 0; p < E.np; p++) {
    const R nx = env_pl<R>(E, p, 0), ny = env_pl<R>(E, p, 1),
            nz = env_pl<R>(E, p, 2);
    R depth = env_pl<R>(E, p, 3) - (px * nx + py * ny + pz * nz);
    if constexpr (P == PREC_FP32)
      depth = depth - (lo.x * nx + lo.y * ny + lo.z * nz);
    if (depth > (R)0.0) {
      const R nmag = env_pl<R>(E, p, 4) * depth;
      fx += nmag * nx;
      fy += nmag * ny;
      fz += nmag * nz;
      const R vn = vx * nx + vy * ny + vz * nz;
      const R tvx = vx - vn * nx, tvy = vy - vn * ny, tvz = vz - vn * nz;
      const R tv = sqrt(tvx * tvx + tvy * tvy + tvz * tvz);
      const R fn = fx * nx + fy * ny + fz * nz;
      const R tfx = fx - fn * nx, tfy = fy - fn * ny, tfz = fz - fn * nz;
      const R tf = sqrt(tfx * tfx + tfy * tfy + tfz * tfz);
      const R vs = sizeof(R) == 4 ? (R)E.v_stickf : (R)E.v_stick;
      if (tv < vs && tf <= env_pl<R>(E, p, 5) * nmag) {
        fx -= tfx;
        fy -= tfy;
        fz -= tfz;
      } else if (tv >= vs) {
        const R sc = env_pl<R>(E, p, 6) * nmag / tv;
        fx -= sc * tvx;
        fy -= sc * tvy;
        fz -= sc * tvz;
      } else if (tf > (R)0.0) {
        const R sc = env_pl<R>(E, p, 6) * nmag / tf;
        fx -= sc * tfx;
        fy -= sc * tfy;
        fz -= sc * tfz;
      }
    }
  }
  for (int b = 0; b < E.nb; b++) {
    R ddx = px - (R)E.bl[b][0], ddy = py - (R)E.bl[b][1],
      ddz = pz - (R)E.bl[b][2];
    if constexpr (P == PREC_FP32) {
      ddx = ddx + lo.x;
      ddy = ddy + lo.y;
      ddz = ddz + lo.z;
    }
    const R dist = sqrt(ddx * ddx + ddy * ddy + ddz * ddz);
    const R depth = (R)E.bl[b][3] - dist;
    if (depth > (R)0.0 && dist > (R)0.0) {
      const R sc = (R)E.bl[b][4] * depth / dist;
      fx += sc * ddx;
      fy += sc * ddy;
      fz += sc * ddz;
    }
  }
  if constexpr (P == PREC_FP64) {  // parity: three true divisions
    ax = fx / mm;
    ay = fy / mm;
    az = fz / mm;
  } else if constexpr (P == PREC_FP32) {
    // tolerance mode: the MUFU reciprocal (~1 ulp: far inside the 1e-4
    // contract) instead of the IEEE division sequence
    R im;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(im) : "f"(mm));
    ax = fx * im;
    ay = fy * im;
    az = fz * im;
  } else {  // mixed: one correctly rounded reciprocal
    const R im = (R)1.0 / mm;
    ax = fx * im;
    ay = fy * im;
    az = fz * im;
  }
  const R dt = (R)dt_;
  vx += ax * dt;
  vy += ay * dt;
  vz += az * dt;
  for (int g = 0; g < E.ngc; g++) {
    const R cx = (R)E.gcv[g][0], cy = (R)E.gcv[g][1], cz = (R)E.gcv[g][2];
    const R vd = vx * cx + vy * cy + vz * cz;
    if (E.gck[g] == 1) {
      vx = vd * cx;
      vy = vd * cy;
      vz = vd * cz;
    } else {
      vx -= vd * cx;
      vy -= vd * cy;
      vz -= vd * cz;
    }
  }
  if (fl & MF_LC) {
    for (int64_t kk = S.lc_off[i]; kk < S.lc_off[i + 1]; kk++) {
      const R cx = (R)S.lc_vec[3 * kk], cy = (R)S.lc_vec[3 * kk + 1],
              cz = (R)S.lc_vec[3 * kk + 2];
      const R vd = vx * cx + vy * cy + vz * cz;
      if (S.lc_kind[kk] == 1) {
        vx = vd * cx;
        vy = vd * cy;
        vz = vd * cz;
      } else {
        vx -= vd * cx;
        vy -= vd * cy;
        vz -= vd * cz;
      }
    }
  }
  if constexpr (P == PREC_FP32) {
    // (hi, lo) + v dt: lo absorbs the increment, a two-sum renormalises
    float ex, ey, ez;
    px = two_sum(px, fmaf(vx, dt, lo.x), ex);
    py = two_sum(py, fmaf(vy, dt, lo.y), ey);
    pz = two_sum(pz, fmaf(vz, dt, lo.z), ez);
    nlo = make_float3(ex, ey, ez);
  } else {
    px += vx * dt;
    py += vy * dt;
    pz += vz * dt;
  }
  np4.x = px;
  np4.y = py;
  np4.z = pz;
  if constexpr (P == PREC_FP32)
    np4.w = nlo.z;  // the record carries lz
  else
    np4.w = mm;
  nv.x = vx;
  nv.y = vy;
  nv.z = vz;
  set_flags(nv.w, fl & ~MF_FEXT);
}

template <int P>
__device__ __forceinline__ void integrate(
    const KState &S, const EnvP &E, const StepP &T, int64_t i,
    typename Tr<P>::R4 me, typename Tr<P>::L lo, typename Tr<P>::R mm,
    typename Tr<P>::R4 v, uint32_t fl, typename Tr<P>::R fx,
    typename Tr<P>::R fy, typename Tr<P>::R fz) {
  using R = typename Tr<P>::R;
  using R4 = typename Tr<P>::R4;
  R4 np4, nv;
  typename Tr<P>::L nlo;
  R ax, ay, az;
  integrate_vals<P>(S, E, T.dt, i, me, lo, mm, v, fl, fx, fy, fz, np4, nlo,
                    nv, ax, ay, az);
  if constexpr (P == PREC_FP32)
    ((float2 *)S.plo[T.cur ^ 1])[i] = make_float2(nlo.x, nlo.y);
  if (S.halo) {  // owned boundary mass: its ghost rows at the peers
    const int2 d = __ldg(&S.halo->dst[i]);
    const int dd[2] = {d.x, d.y};
#pragma unroll
    for (int q = 0; q < 2; q++) {
      if (dd[q] < 0) continue;
      const int p = dd[q] & 7;
      const int64_t row = dd[q] >> 3;
      ((R4 *)S.halo->pos[p][T.cur ^ 1])[row] = np4;
      if constexpr (P == PREC_FP32)
        ((float2 *)S.halo->lo[p][T.cur ^ 1])[row] =
            make_float2(nlo.x, nlo.y);
    }
    if (d.x >= 0) __threadfence_system();
  }
  const R px = np4.x, py = np4.y, pz = np4.z, vx = nv.x, vy = nv.y,
          vz = nv.z;
  ((R4 *)S.pos[T.cur ^ 1])[i] = np4;
  ((R4 *)S.vel)[i] = nv;
  if (T.write_acc) {
    R *a = (R *)S.acc + 3 * i;
    a[0] = ax;
    a[1] = ay;
    a[2] = az;
  }
  // x * 0 is 0 for finite x and NaN for +-inf / NaN
  const R z0 = px * (R)0.0 + py * (R)0.0 + pz * (R)0.0 + vx * (R)0.0 +
               vy * (R)0.0 + vz * (R)0.0;
  if (!(z0 == (R)0.0)) mark_nonfinite(S, i, T.step);
}

template <int P>
__device__ __forceinline__ void fixed_mass(const KState &S, const StepP &T,
                                           int64_t i, typename Tr<P>::R4 v,
                                           uint32_t fl) {
  using R = typename Tr<P>::R;
  using R4 = typename Tr<P>::R4;
  // kernels.py:260-270: vel = acc = f_ext = 0, pos and load untouched
  R4 nv;
  nv.x = (R)0.0;
  nv.y = (R)0.0;
  nv.z = (R)0.0;
  set_flags(nv.w, fl & ~MF_FEXT);
  ((R4 *)S.vel)[i] = nv;
  if (T.write_acc) {
    R *a = (R *)S.acc + 3 * i;
    a[0] = a[1] = a[2] = (R)0.0;
  }
  if (fl & MF_FEXT) {
    R4 z;
    z.x = z.y = z.z = z.w = (R)0.0;
    ((R4 *)S.fext)[i] = z;
  }
}

// Damper term of spring s as a multiple of d = pos[m2] - pos[m1]:
// c ((v2 - v1) . d) / |d|^2, i.e. c ((v2 - v1) . d^) d^ on m1 (equal and
// opposite on m2; both endpoints form the same bits).  0 for c = 0.
template <int P, class F>
__device__ __forceinline__ F damper_scale(const KState &S, int64_t s, F dx,
                                          F dy, F dz, F len2) {
  using R4 = typename Tr<P>::R4;
  const double c = S.damp[s];
  if (c == 0.0) return (F)0;
  const int2 ab = S.ends[s];
  const R4 v1 = ((const R4 *)S.vel)[ab.x], v2 = ((const R4 *)S.vel)[ab.y];
  const F vr = (F)(v2.x - v1.x) * dx + (F)(v2.y - v1.y) * dy +
               (F)(v2.z - v1.z) * dz;
  return (F)c * vr / len2;
}

// ---------------------------------------------------------------------------
// One incidence entry: spring force between this mass and `other`, in the
// reference's operation order (kernels.py:46-83).  Returns false if the
// entry contributes nothing.  Side effects (yield break, zero-length flag,
// counters) are performed exactly once per spring, by its m1 endpoint; the
// m2 endpoint reaches the same decision from the same bits and only kills
// its own entry.
template <int P>
__device__ __forceinline__ bool entry_force(
    const KState &S, int64_t e, uint32_t jr, typename Tr<P>::R4 me,
    typename Tr<P>::L ml, typename Tr<P>::R4 other, typename Tr<P>::L ol,
    typename Tr<P>::F2 kl, double sim_t, typename Tr<P>::R &fx,
    typename Tr<P>::R &fy, typename Tr<P>::R &fz) {
  using R = typename Tr<P>::R;
  using F = typename Tr<P>::M;
  const bool is_m2 = (jr & EJ_M2) != 0;
  // d = pos[m2] - pos[m1]
  F dx, dy, dz;
  if (is_m2)
    pdiff<P>(other, ol, me, ml, dx, dy, dz);
  else
    pdiff<P>(me, ml, other, ol, dx, dy, dz);
  const F len2 = dx * dx + dy * dy + dz * dz;
  if (len2 == (F)0.0) {  // <=> sqrt(len2) == 0, kernels.py:50
    if (!is_m2) {
      const int32_t s = S.ent_s[e];
      if (!S.s_degen[s]) {
        S.s_degen[s] = 1;
        count_spring(S, 2, s);
      }
    }
    return false;
  }
  F factor = (F)1.0;
  if (jr & EJ_SPECIAL) factor = (F)act_factor(S, S.ent_s[e], sim_t);
  F len, inv;  // |d| and the factor turning fmag into fmag/|d|
  if constexpr (P == PREC_FP64) {
    // parity mode: IEEE sqrt and a true division, as the reference
    len = sqrt(len2);
  } else if constexpr (P == PREC_FP32) {
    // tolerance mode: one MUFU.RSQ replaces sqrt + divide
    inv = rsqrtf(len2);
    len = len2 * inv;
  } else {
    // mixed: float rsqrt seed + one fp64 Newton step (~1e-14 relative)
    double r = (double)rsqrtf((float)len2);
    r = r * (1.5 - 0.5 * len2 * r * r);
    inv = r;
    len = len2 * r;
  }
  const F fmag = (F)kl.x * (len - factor * (F)kl.y);
  F scale;
  if constexpr (P == PREC_FP64)
    scale = fmag / len;
  else
    scale = fmag * inv;
  if ((jr & EJ_SPECIAL) && S.damp)
    scale += damper_scale<P, F>(S, S.ent_s[e], dx, dy, dz, len2);
  if (is_m2) scale = -scale;  // -(s*d) == (-s)*d exactly; f - g == f + (-g)
  fx += (R)(scale * dx);
  fy += (R)(scale * dy);
  fz += (R)(scale * dz);
  if (jr & EJ_SPECIAL) {
    const int32_t s = S.ent_s[e];
    const F thr = (F)((const typename Tr<P>::F *)S.thr)[s];
    const F mag = fmag >= (F)0.0 ? fmag : -fmag;
    if (mag > thr) {
      S.ent_j[e] = jr | EJ_DEAD;
      if (!is_m2) {
        count_spring(S, 0, s);
        S.s_alive[s] = 0;
        S.ends[s] = make_int2(-1, -1);
      }
    }
  }
  return true;
}

// Spring forces of one mass from its incidence list.  ej / ekl point at the
// mass's first entry (lane-strided by 32: global memory or a shared-memory
// stage); ebase is the global index of that entry (for side effects).
// Batches of U entries: every independent load of a batch is issued before
// any is consumed (U neighbour gathers in flight per thread), accumulation
// then runs in ascending entry (= spring slot) order -- the serial order.
// This exact path serves fp64 parity mode.
template <int P, bool GLOBAL_SRC>
__device__ __forceinline__ void gather_forces_exact(
    const KState &S, const typename Tr<P>::R4 *pos, const void *plo,
    const uint32_t *ej, const typename Tr<P>::F2 *ekl, int width,
    int64_t ebase, typename Tr<P>::R4 me, typename Tr<P>::L ml, double sim_t,
    typename Tr<P>::R &fx, typename Tr<P>::R &fy, typename Tr<P>::R &fz) {
  using R4 = typename Tr<P>::R4;
  using F2 = typename Tr<P>::F2;
  using L = typename Tr<P>::L;
  // fp64 parity mode runs everything here; in the tolerance modes only
  // masses with actuated / breakable springs do -- keep it register-light
  constexpr int U = P == PREC_FP64 ? Tr<P>::U : 2;
  for (int t0 = 0; t0 < width; t0 += U) {
    uint32_t jr[U];
    F2 kl[U];
    R4 o[U];
    L ol[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (t0 + u < width)
        jr[u] = GLOBAL_SRC ? __ldg(ej + 32 * (t0 + u)) : ej[32 * (t0 + u)];
      else
        jr[u] = EJ_PAD;
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (!(jr[u] & EJ_DEAD)) {
        kl[u] = GLOBAL_SRC ? __ldg(ekl + 32 * (t0 + u)) : ekl[32 * (t0 + u)];
        o[u] = pos[jr[u] & EJ_MASK];
        ol[u] = lo_at<P>(o[u], plo, jr[u] & EJ_MASK);
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (!(jr[u] & EJ_DEAD))
        entry_force<P>(S, ebase + 32 * (int64_t)(t0 + u), jr[u], me, ml,
                       o[u], ol[u], kl[u], sim_t, fx, fy, fz);
    }
  }
}

// Tolerance modes (fp32 / mixed), masses without actuated / breakable
// springs: branch-free loop.  The endpoint orientation cancels -- the force
// on this mass is k(|d| - L0)/|d| * (p_other - p_me) for either endpoint --
// so no sign logic is needed.  Dead / padding entries gather this mass's own
// position (|d| = 0) and are zeroed by a select; an alive zero-length spring
// (also |d| = 0, force 0) only needs its flag side effect, detected as
// "|d| == 0 xor dead" and replayed afterwards.  Accumulation order is fixed
// (deterministic run to run).  Returns true if a zero-length spring was seen.
template <int P, bool GLOBAL_SRC>
__device__ __forceinline__ bool gather_forces_fast(
    const typename Tr<P>::R4 *pos, const void *plo, const uint32_t *ej,
    const typename Tr<P>::F2 *ekl, int width, uint32_t self,
    typename Tr<P>::R4 me, typename Tr<P>::L ml, typename Tr<P>::R &fx,
    typename Tr<P>::R &fy, typename Tr<P>::R &fz) {
  using R = typename Tr<P>::R;
  using M = typename Tr<P>::M;
  using R4 = typename Tr<P>::R4;
  using F2 = typename Tr<P>::F2;
  constexpr int U = Tr<P>::U;
  bool odd = false;
  auto body = [&](uint32_t jr, F2 kl, R4 o) {
    const uint32_t j = (jr & EJ_DEAD) ? self : (jr & EJ_MASK);
    M dx, dy, dz;
    pdiff<P>(me, ml, o, lo_at<P>(o, plo, j), dx, dy, dz);
    const M len2 = dx * dx + dy * dy + dz * dz;
    M r;
    if constexpr (P == PREC_FP32) {
      r = rsqrtf(len2);  // +inf at 0: the select below discards it
    } else {
      r = (double)rsqrtf((float)len2);
      r = r * (1.5 - 0.5 * len2 * r * r);  // one Newton step, ~1e-14
    }
    const M sc = (M)kl.x * (len2 * r - (M)kl.y) * r;
    const bool zero = len2 == (M)0;
    odd |= zero != ((jr & EJ_DEAD) != 0);
    const M s = zero ? (M)0 : sc;
    fx += (R)(s * dx);
    fy += (R)(s * dy);
    fz += (R)(s * dz);
  };
  auto ld_j = [&](const uint32_t *p) { return GLOBAL_SRC ? __ldg(p) : *p; };
  auto ld_k = [&](const F2 *p) { return GLOBAL_SRC ? __ldg(p) : *p; };
  auto nbr = [&](uint32_t jr) {
    return pos[(jr & EJ_DEAD) ? self : (jr & EJ_MASK)];
  };
  int t = 0;
  for (; t + U <= width; t += U, ej += 32 * U, ekl += 32 * U) {
    uint32_t jr[U];
    F2 kl[U];
    R4 o[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      jr[u] = ld_j(ej + 32 * u);
      kl[u] = ld_k(ekl + 32 * u);
    }
#pragma unroll
    for (int u = 0; u < U; u++) o[u] = nbr(jr[u]);
#pragma unroll
    for (int u = 0; u < U; u++) body(jr[u], kl[u], o[u]);
  }
  for (; t < width; t++, ej += 32, ekl += 32) {
    const uint32_t jr = ld_j(ej);
    body(jr, ld_k(ekl), nbr(jr));
  }
  return odd;
}

// Same contract as gather_forces_fast, software-pipelined across batches:
// the neighbour gathers of batch b+1 are issued before batch b is reduced,
// so 2*U gathers are in flight per thread.  Used by the TMA kernel, which
// runs few warps per SM and can afford the registers.
template <int P, int U>
__device__ __forceinline__ bool gather_forces_pipe(
    const typename Tr<P>::R4 *pos, const void *plo, const uint32_t *ej,
    const typename Tr<P>::F2 *ekl, int width, uint32_t self,
    typename Tr<P>::R4 me, typename Tr<P>::L ml, typename Tr<P>::R &fx,
    typename Tr<P>::R &fy, typename Tr<P>::R &fz) {
  using R = typename Tr<P>::R;
  using M = typename Tr<P>::M;
  using R4 = typename Tr<P>::R4;
  using F2 = typename Tr<P>::F2;
  bool odd = false;
  auto body = [&](uint32_t jr, F2 kl, R4 o) {
    const uint32_t j = (jr & EJ_DEAD) ? self : (jr & EJ_MASK);
    M dx, dy, dz;
    pdiff<P>(me, ml, o, lo_at<P>(o, plo, j), dx, dy, dz);
    const M len2 = dx * dx + dy * dy + dz * dz;
    M r;
    if constexpr (P == PREC_FP32) {
      r = rsqrtf(len2);
    } else {
      r = (double)rsqrtf((float)len2);
      r = r * (1.5 - 0.5 * len2 * r * r);
    }
    const M sc = (M)kl.x * (len2 * r - (M)kl.y) * r;
    const bool zero = len2 == (M)0;
    odd |= zero != ((jr & EJ_DEAD) != 0);
    const M s = zero ? (M)0 : sc;
    fx += (R)(s * dx);
    fy += (R)(s * dy);
    fz += (R)(s * dz);
  };
  auto nbr = [&](uint32_t jr) {
    return pos[(jr & EJ_DEAD) ? self : (jr & EJ_MASK)];
  };
  // only the gathered positions live in registers; entry words and (k, L0)
  // are re-read from the shared-memory stage when the batch is reduced
  struct Batch {
    R4 o[U];
  };
  auto load = [&](Batch &B, int t) {
#pragma unroll
    for (int u = 0; u < U; u++) B.o[u] = nbr(ej[32 * (t + u)]);
  };
  auto reduce_at = [&](const Batch &B, int t) {
#pragma unroll
    for (int u = 0; u < U; u++)
      body(ej[32 * (t + u)], ekl[32 * (t + u)], B.o[u]);
  };
  const int nb = width / U;
  Batch A, B;
  if (nb > 0) load(A, 0);
  for (int b = 0; b < nb; b += 2) {
    if (b + 1 < nb) load(B, (b + 1) * U);
    reduce_at(A, b * U);
    if (b + 1 >= nb) break;
    if (b + 2 < nb) load(A, (b + 2) * U);
    reduce_at(B, (b + 1) * U);
  }
  for (int t = nb * U; t < width; t++) {
    const uint32_t jr = ej[32 * t];
    body(jr, ekl[32 * t], nbr(jr));
  }
  return odd;
}

// Side effects of alive zero-length springs (kernels.py:50-54) for a mass
// that went through the fast loop.
template <int P, bool GLOBAL_SRC>
__device__ __noinline__ void degenerate_flags(
    const int32_t *ent_s, uint8_t *s_degen, unsigned long long *status,
    const uint8_t *ghost, int64_t self, const typename Tr<P>::R4 *pos,
    const void *plo, const uint32_t *ej, int width, int64_t ebase,
    typename Tr<P>::R4 me, typename Tr<P>::L ml) {
  for (int t = 0; t < width; t++) {
    const uint32_t jr = GLOBAL_SRC ? __ldg(ej + 32 * t) : ej[32 * t];
    if (jr & (EJ_DEAD | EJ_M2)) continue;
    const typename Tr<P>::R4 o = pos[jr & EJ_MASK];
    typename Tr<P>::M dx, dy, dz;
    pdiff<P>(me, ml, o, lo_at<P>(o, plo, jr & EJ_MASK), dx, dy, dz);
    if (dx == 0 && dy == 0 && dz == 0) {
      const int32_t s = ent_s[ebase + 32 * (int64_t)t];
      if (!s_degen[s]) {
        s_degen[s] = 1;
        if (!ghost || !ghost[self]) atomicAdd(status + 2, 1ull);  // self = m1
      }
    }
  }
}

template <int P, bool GLOBAL_SRC>
__device__ __forceinline__ void gather_forces(
    const KState &S, const typename Tr<P>::R4 *pos, const void *plo,
    const uint32_t *ej, const typename Tr<P>::F2 *ekl, int width,
    int64_t ebase, int64_t self, uint32_t fl, typename Tr<P>::R4 me,
    typename Tr<P>::L ml, double sim_t, typename Tr<P>::R &fx,
    typename Tr<P>::R &fy, typename Tr<P>::R &fz) {
  if constexpr (P == PREC_FP64) {
    gather_forces_exact<P, GLOBAL_SRC>(S, pos, plo, ej, ekl, width, ebase, me,
                                       ml, sim_t, fx, fy, fz);
  } else {
    if (fl & MF_SPECIAL)
      gather_forces_exact<P, GLOBAL_SRC>(S, pos, plo, ej, ekl, width, ebase,
                                         me, ml, sim_t, fx, fy, fz);
    else if (gather_forces_fast<P, GLOBAL_SRC>(pos, plo, ej, ekl, width,
                                                 (uint32_t)self, me, ml, fx,
                                                 fy, fz))
      degenerate_flags<P, GLOBAL_SRC>(S.ent_s, S.s_degen, S.status, S.ghost,
                                      self, pos, plo, ej, width, ebase, me,
                                      ml);
  }
}

// Tail of a mass update after its spring forces are known.
template <int P, bool FORCE_ONLY>
__device__ __forceinline__ void finish_mass(
    const KState &S, const EnvP &E, const StepP &T, int64_t i,
    typename Tr<P>::R4 me, typename Tr<P>::L ml, typename Tr<P>::R mm,
    typename Tr<P>::R4 v, uint32_t fl, typename Tr<P>::R fx,
    typename Tr<P>::R fy, typename Tr<P>::R fz) {
  using R = typename Tr<P>::R;
  using R4 = typename Tr<P>::R4;
  if (FORCE_ONLY) {
    R4 f;
    f.x = fx;
    f.y = fy;
    f.z = fz;
    f.w = (R)0.0;
    ((R4 *)S.fext)[i] = f;
    R4 nv = v;
    set_flags(nv.w, fl | MF_FEXT);
    ((R4 *)S.vel)[i] = nv;
    return;
  }
  if (fl & MF_FIXED) {
    fixed_mass<P>(S, T, i, v, fl);
    return;
  }
  if (fl & MF_FEXT) {
    R4 z;
    z.x = z.y = z.z = z.w = (R)0.0;
    ((R4 *)S.fext)[i] = z;
  }
  integrate<P>(S, E, T, i, me, ml, mm, v, fl, fx, fy, fz);
}

template <int P>
__device__ __forceinline__ void initial_force(const KState &S, int64_t i,
                                              uint32_t fl, bool force_only,
                                              typename Tr<P>::R &fx,
                                              typename Tr<P>::R &fy,
                                              typename Tr<P>::R &fz) {
  using R = typename Tr<P>::R;
  using R4 = typename Tr<P>::R4;
  fx = fy = fz = (R)0.0;
  if (force_only || (fl & MF_FEXT)) {
    const R4 f0 = ((const R4 *)S.fext)[i];
    fx = f0.x;
    fy = f0.y;
    fz = f0.z;
  }
}

// Fused step, plain variant: one thread per mass, entries read straight
// from global memory.  Used for spring_pass (FORCE_ONLY), for tiny bodies
// and for layouts with very wide slices (hub masses).
// Programmatic dependent launch: let the next step kernel launch now and
// wait here for the previous one's completion (and memory) before reading
// anything it wrote.  A no-op for ordinary launches.
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <int P, bool FORCE_ONLY>
static __global__ void __launch_bounds__(256)
    k_gather_step(const KState S, const EnvP E, const StepP T) {
  pdl_wait();
  using R = typename Tr<P>::R;
  using R4 = typename Tr<P>::R4;
  using F2 = typename Tr<P>::F2;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S.m_n) return;
  if (!FORCE_ONLY && stopped(S, T.step)) return;
  const R4 *pos = (const R4 *)S.pos[T.cur];
  const R4 v = ((const R4 *)S.vel)[i];
  const uint32_t fl = flags_of(v.w);
  if (!(fl & MF_ALIVE)) return;
  const R4 me = pos[i];
  const void *plo = S.plo[T.cur];
  const typename Tr<P>::L ml = lo_at<P>(me, plo, i);
  R fx, fy, fz;
  initial_force<P>(S, i, fl, FORCE_ONLY, fx, fy, fz);
  const int64_t w = i >> 5;
  const int64_t ebase = S.slice_ptr[w] + (i & 31);
  const int width = (int)((S.slice_ptr[w + 1] - S.slice_ptr[w]) >> 5);
  gather_forces<P, true>(S, pos, plo, S.ent_j + ebase,
                         (const F2 *)S.ent_kL0 + ebase, width, ebase, i, fl,
                         me, ml, T.sim_t, fx, fy, fz);
  finish_mass<P, FORCE_ONLY>(S, E, T, i, me, ml, mass_of<P>(S, me, i), v,
                             fl, fx, fy, fz);
}

// ---------------------------------------------------------------------------
// TMA-pipelined fused step (the production path).
//
// Persistent CTAs; every warp owns a strided sequence of 32-mass slices and
// a private 2-stage shared-memory ring.  Lane 0 streams the NEXT slice's
// incidence list (entry words + (k, L0)) from HBM into the free stage with
// two 1-D bulk async copies (cp.async.bulk -> UBLKCP, completion counted on
// an mbarrier) while the warp computes the current slice out of the other
// stage.  The HBM stream is thereby decoupled from the dependent neighbour
// gathers (which hit L2), and the bytes in flight per SM are bounded only by
// the ring size, not by registers.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile(
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src,
                                         uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Warp-collective issue of one stage: every lane calls with the same
// (warp-uniform) operands, elect.sync picks one lane for the expect_tx
// arrival and up to five bulk copies (zero-byte copies are skipped).  With
// uniform operands ptxas keeps them in uniform registers instead of
// serialising the copies through a per-lane loop.
__device__ __forceinline__ void bulk_stage_elect(
    uint64_t *bar, uint32_t tx, void *d0, const void *s0, uint32_t n0,
    void *d1, const void *s1, uint32_t n1, void *d2, const void *s2,
    uint32_t n2, void *d3, const void *s3, uint32_t n3, void *d4,
    const void *s4, uint32_t n4, void *d5 = nullptr,
    const void *s5 = nullptr, uint32_t n5 = 0) {
  asm volatile(
      "{\n"
      ".reg .pred E, Q;\n"
      "elect.sync _|E, 0xffffffff;\n"
      "@E mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
      "setp.ne.and.u32 Q, %4, 0, E;\n"
      "@Q cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%2], [%3], %4, [%0];\n"
      "setp.ne.and.u32 Q, %7, 0, E;\n"
      "@Q cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%5], [%6], %7, [%0];\n"
      "setp.ne.and.u32 Q, %10, 0, E;\n"
      "@Q cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%8], [%9], %10, [%0];\n"
      "setp.ne.and.u32 Q, %13, 0, E;\n"
      "@Q cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%11], [%12], %13, [%0];\n"
      "setp.ne.and.u32 Q, %16, 0, E;\n"
      "@Q cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%14], [%15], %16, [%0];\n"
      "setp.ne.and.u32 Q, %19, 0, E;\n"
      "@Q cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%17], [%18], %19, [%0];\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(tx), "r"(smem_u32(d0)), "l"(s0), "r"(n0), "r"(smem_u32(d1)),
      "l"(s1), "r"(n1), "r"(smem_u32(d2)), "l"(s2), "r"(n2),
      "r"(smem_u32(d3)), "l"(s3), "r"(n3), "r"(smem_u32(d4)), "l"(s4),
      "r"(n4), "r"(smem_u32(d5 ? d5 : d4)), "l"(s5 ? s5 : s4), "r"(n5)
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

struct TmaCfg {
  int64_t n_slices;
  int cap_w;             // max slice width the stages hold
  int warps;             // warps per CTA
  uint32_t stage_bytes;  // one stage: 32 pos + 32 vel records, j, (k, L0)
};

// Stage layout: [pos of the slice's 32 masses][their vel][cap_w*32 entry
// words][cap_w*32 (k, L0) pairs].  Everything a warp needs for one slice
// arrives through four bulk copies on one mbarrier, so the only exposed
// latency left in the loop is the L2 gather of neighbour positions.
template <int P>
static __global__ void __launch_bounds__(384)
    k_gather_tma(const KState S, const EnvP E, const StepP T,
                 const TmaCfg C) {
  pdl_wait();
  using R = typename Tr<P>::R;
  using R4 = typename Tr<P>::R4;
  using F2 = typename Tr<P>::F2;
  extern __shared__ __align__(128) unsigned char smem[];
  if (stopped(S, T.step)) return;  // uniform across the grid
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *ring = smem + (size_t)warp * 2 * C.stage_bytes;
  uint64_t *bars =
      (uint64_t *)(smem + (size_t)C.warps * 2 * C.stage_bytes) + 2 * warp;
  constexpr uint32_t MB = 32 * sizeof(R4);  // mass block bytes
  const uint32_t j_off = 2 * MB;
  const uint32_t k_off = j_off + (uint32_t)C.cap_w * 128u;
  if (lane == 0) {
    mbar_init(bars + 0, 1);
    mbar_init(bars + 1, 1);
    fence_proxy_async();
  }
  __syncwarp();
  const R4 *pos = (const R4 *)S.pos[T.cur];
  const int64_t stride = (int64_t)gridDim.x * C.warps;
  int64_t s = (int64_t)blockIdx.x * C.warps + warp;
  // lane 0 holds slice_ptr of the current and the next slice
  int64_t cur0 = 0, cur1 = 0, nxt0 = 0, nxt1 = 0;
  auto issue = [&](int64_t sl, int64_t e0, int64_t e1, int stage) {
    const uint32_t n = (uint32_t)(e1 - e0);
    unsigned char *dst = ring + (size_t)stage * C.stage_bytes;
    mbar_expect_tx(bars + stage, 2 * MB + n * (uint32_t)(4 + sizeof(F2)));
    bulk_g2s(dst, pos + sl * 32, MB, bars + stage);
    bulk_g2s(dst + MB, (const R4 *)S.vel + sl * 32, MB, bars + stage);
    if (n) {
      bulk_g2s(dst + j_off, S.ent_j + e0, n * 4u, bars + stage);
      bulk_g2s(dst + k_off, (const F2 *)S.ent_kL0 + e0,
               n * (uint32_t)sizeof(F2), bars + stage);
    }
  };
  if (lane == 0 && s < C.n_slices) {
    cur0 = S.slice_ptr[s];
    cur1 = S.slice_ptr[s + 1];
    issue(s, cur0, cur1, 0);
    if (s + stride < C.n_slices) {
      nxt0 = S.slice_ptr[s + stride];
      nxt1 = S.slice_ptr[s + stride + 1];
    }
  }
  for (int k = 0; s < C.n_slices; s += stride, k++) {
    const int stage = k & 1;
    const int64_t e0 = __shfl_sync(0xffffffffu, cur0, 0);
    const int width = (int)((__shfl_sync(0xffffffffu, cur1, 0) - e0) >> 5);
    if (lane == 0 && s + stride < C.n_slices) {
      fence_proxy_async();  // generic reads of that stage finished (syncwarp)
      issue(s + stride, nxt0, nxt1, stage ^ 1);
      cur0 = nxt0;
      cur1 = nxt1;
      const int64_t s2 = s + 2 * stride;
      if (s2 < C.n_slices) {  // metadata one slice further ahead
        nxt0 = S.slice_ptr[s2];
        nxt1 = S.slice_ptr[s2 + 1];
      }
    }
    const int64_t i = s * 32 + lane;
    const unsigned char *st = ring + (size_t)stage * C.stage_bytes;
    mbar_wait(bars + stage, (uint32_t)((k >> 1) & 1));
    if (i < S.m_n) {
      const R4 v = ((const R4 *)(st + MB))[lane];
      const uint32_t fl = flags_of(v.w);
      if (fl & MF_ALIVE) {
        const R4 me = ((const R4 *)st)[lane];
        const void *plo = S.plo[T.cur];
        const typename Tr<P>::L ml = lo_at<P>(me, plo, i);
        R fx, fy, fz;
        initial_force<P>(S, i, fl, false, fx, fy, fz);
        const uint32_t *ej = (const uint32_t *)(st + j_off) + lane;
        const F2 *ekl = (const F2 *)(st + k_off) + lane;
        if constexpr (P == PREC_FP64) {
          gather_forces_exact<P, false>(S, pos, plo, ej, ekl, width,
                                        e0 + lane, me, ml, T.sim_t, fx, fy,
                                        fz);
        } else {
          if (fl & MF_SPECIAL)
            gather_forces_exact<P, false>(S, pos, plo, ej, ekl, width,
                                          e0 + lane, me, ml, T.sim_t, fx, fy,
                                          fz);
          else if (gather_forces_pipe<P, Tr<P>::UP>(pos, plo, ej, ekl, width,
                                                     (uint32_t)i, me, ml, fx,
                                                     fy, fz))
            degenerate_flags<P, false>(S.ent_s, S.s_degen, S.status, S.ghost,
                                       i, pos, plo, ej, width, e0 + lane, me,
                                       ml);
        }
        finish_mass<P, false>(S, E, T, i, me, ml, mass_of<P>(S, me, i), v, fl,
                              fx, fy, fz);
      }
    }
    __syncwarp();
  }
}

// Mark both incidence entries of spring s dead (host-time kills and the
// atomic variant's yield breaks; no fused step is running concurrently, so
// the split layout's (k, L0) cell can be zeroed as well).
__device__ __forceinline__ void kill_entries(const KState &S, int64_t s) {
  if (S.split) {
    // cells another spring took over since this one died (in-place topology
    // sync, k_split_insert) are not this spring's to kill
    const int64_t e1 = S.e1[s] >= 0 && S.sp_s[S.e1[s]] == (int32_t)s ? S.e1[s]
                                                                       : -1;
    const int64_t e2 = S.e2[s] >= 0 && S.sp_s[S.e2[s]] == (int32_t)s ? S.e2[s]
                                                                       : -1;
    if (e1 < 0 && e2 < 0) return;
    if (e1 >= 0) {
      S.sp_j[e1] = S.sp_sent;
      if (S.fsz8)
        ((double2 *)S.sp_kl)[S.sp_ekl[s]] = make_double2(0.0, 0.0);
      else
        ((float2 *)S.sp_kl)[S.sp_ekl[s]] = make_float2(0.f, 0.f);
    }
    if (e2 >= 0) S.sp_j[e2] = S.sp_null;
    if (S.fz_code) {  // fused groups: both entries get the zero code
      const int64_t per = (int64_t)S.sp_rows * 32;
      const int64_t es[2] = {e1, e2};
      for (int q = 0; q < 2; q++) {
        if (es[q] < 0) continue;
        const int64_t sl = es[q] / per;
        const int rem = (int)(es[q] - sl * per);
        const int64_t i = sl * 32 + (rem & 31);
        const int row = q == 0 ? rem >> 5 : S.fz_ra + (rem >> 5) - (1 << S.sp_a);
        const int32_t g = S.fz_gid[i];
        const int mm = S.fz_maxm;
        const uint32_t qt =
            S.fz_epos[((int64_t)g * S.fz_rows + row) * mm +
                      (i - S.fz_gstart[g])];
        S.fz_code[((int64_t)g * S.fz_rows + qt / mm) * mm + qt % mm] =
            S.fz_zero[g];
      }
    }
    if (S.win_blk) {  // window layout: both entries get the zero code
      // (entry word: sl_window.cuh ew_word; merged rows A then B)
      const int a = S.sp_a;
      auto zero_code = [&](int64_t sl, int row, int lane) {
        uint32_t *wp = (uint32_t *)(S.win_blk + sl * S.win_sb +
                                    (row >> 1) * 256 + lane * 8 + (row & 1) * 4);
        *wp = (*wp & ((1u << 26) - 1u)) |
              ((uint32_t)S.win_zero[sl / S.win_tt] << 26);
      };
      if (e1 >= 0) {
        const uint32_t kli = S.sp_ekl[s];
        const int64_t sl = kli >> (a + 5);
        zero_code(sl, (int)((kli >> 5) & ((1u << a) - 1)), (int)(kli & 31));
      }
      if (e2 >= 0) {
        const int64_t per = (int64_t)S.sp_rows * 32, e = e2;
        const int64_t sl = e / per;
        const int rem = (int)(e - sl * per);
        const int rb = (rem >> 5) - (1 << a);
        zero_code(sl, (int)(S.sp_w[sl] & 0xFFFF) + rb, rem & 31);
      }
    }
    return;
  }
  // (only entries still this spring's: in-place insertion re-uses rows)
  const int64_t es[2] = {S.e1[s], S.e2[s]};
  for (int q = 0; q < 2; q++) {
    const int64_t e = es[q];
    if (e < 0 || S.ent_s[e] != (int32_t)s) continue;
    S.ent_j[e] |= EJ_DEAD;
    if (S.win_blk) {  // parity-mode window: the entry word's skip bit
      // (k_win64_build: entry e = slice_ptr[w] + 32 row + lane <-> word
      // ew_off(row, lane) of slice w's block)
      int64_t lo = 0, hi = (S.m_n + 31) >> 5;  // slice_ptr[lo] <= e < [hi]
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (S.slice_ptr[mid] <= e) lo = mid; else hi = mid;
      }
      const int rel = (int)(e - S.slice_ptr[lo]);
      *(uint32_t *)(S.win_blk + lo * S.win_sb +
                    (uint32_t)((rel >> 6) * 256 + (rel & 31) * 8 +
                               ((rel >> 5) & 1) * 4)) |= 1u;
    }
  }
}

// Owner-aggregated atomic accumulation on the EXACT layout (fp64 and the
// exact-layout tolerance contexts): one thread per mass walks the entries
// it is m1 of (ascending slot), sums their forces in registers, pushes -f
// to each m2 and its own sum with one reduction each (see k_split_atomic,
// sl_split.cuh).  Each spring is evaluated once, with entry_force's
// arithmetic and side effects; a yield break kills both entries.
template <int P>
static __global__ void __launch_bounds__(256)
    k_gather_atomic(const KState S, const StepP T) {
  pdl_wait();
  using R = typename Tr<P>::R;
  using R4 = typename Tr<P>::R4;
  using F2 = typename Tr<P>::F2;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S.m_n) return;
  if (stopped(S, T.step)) return;
  const uint32_t fl = flags_of(((const R4 *)S.vel)[i].w);
  if (!(fl & MF_ALIVE)) return;
  const R4 *pos = (const R4 *)S.pos[T.cur];
  const void *plo = S.plo[T.cur];
  const R4 me = pos[i];
  const typename Tr<P>::L ml = lo_at<P>(me, plo, i);
  const int64_t w = i >> 5;
  const int64_t ebase = S.slice_ptr[w] + (i & 31);
  const int width = (int)((S.slice_ptr[w + 1] - S.slice_ptr[w]) >> 5);
  R4 *fe = (R4 *)S.fext;
  R ox = 0, oy = 0, oz = 0;
  // four entries' words, partners and (k, L0) requested together, then
  // evaluated one by one in slot order (the r3 ncu: one dependent
  // entry -> partner round trip per entry, long-scoreboard 26 per issue)
  constexpr int U = 4;
  for (int t0 = 0; t0 < width; t0 += U) {
    uint32_t jr[U];
    R4 o[U];
    F2 kl[U];
#pragma unroll
    for (int u = 0; u < U; u++)
      jr[u] = t0 + u < width ? __ldg(S.ent_j + ebase + 32 * (int64_t)(t0 + u))
                             : EJ_PAD;
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (jr[u] & (EJ_DEAD | EJ_M2)) continue;  // dead, padding, m2 side
      o[u] = pos[jr[u] & EJ_MASK];
      kl[u] = ((const F2 *)S.ent_kL0)[ebase + 32 * (int64_t)(t0 + u)];
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (jr[u] & (EJ_DEAD | EJ_M2)) continue;
      const int64_t e = ebase + 32 * (int64_t)(t0 + u);
      const uint32_t j = jr[u] & EJ_MASK;
      // entry_force on a zeroed accumulator: the m1-side force itself
      R gx = 0, gy = 0, gz = 0;
      // a yield break (special entries only) kills both entries
      const bool sp = (jr[u] & EJ_SPECIAL) != 0;
      const int32_t s = sp ? S.ent_s[e] : 0;
      const bool was_alive = sp && S.s_alive[s] != 0;
      if (!entry_force<P>(S, e, jr[u], me, ml, o[u], lo_at<P>(o[u], plo, j),
                          kl[u], T.sim_t, gx, gy, gz))
        continue;
      if (was_alive && !S.s_alive[s]) kill_entries(S, s);
      ox += gx;
      oy += gy;
      oz += gz;
      red_add(fe + j, -gx, -gy, -gz);
    }
  }
  red_add(fe + i, ox, oy, oz);
}

// Atomic variant, spring side: one thread per spring slot (kernels.py:36-83
// with the accumulation of the paper's GPU design).
template <int P, bool SPECIAL>
static __global__ void __launch_bounds__(256)
    k_spring_atomic(const KState S, const StepP T) {
  pdl_wait();
  using R = typename Tr<P>::R;
  using F = typename Tr<P>::M;
  using FS = typename Tr<P>::F;
  using R4 = typename Tr<P>::R4;
  using F2 = typename Tr<P>::F2;
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S.s_n) return;
  if (stopped(S, T.step)) return;
  const int2 ab = S.ends[s];
  if (ab.x < 0) return;
  const R4 *pos = (const R4 *)S.pos[T.cur];
  const R4 pa = pos[ab.x], pb = pos[ab.y];
  const F2 kl = ((const F2 *)S.kL0)[s];
  F dx, dy, dz;
  pdiff<P>(pa, lo_at<P>(pa, S.plo[T.cur], ab.x), pb,
           lo_at<P>(pb, S.plo[T.cur], ab.y), dx, dy, dz);
  const F len = sqrt(dx * dx + dy * dy + dz * dz);
  if (len == (F)0.0) {
    if (!S.s_degen[s]) {
      S.s_degen[s] = 1;
      count_spring(S, 2, s);
    }
    return;
  }
  F factor = (F)1.0;
  bool special = false;
  if (SPECIAL) {
    special = S.mode[s] != 0 || ((const FS *)S.thr)[s] != (FS)CUDART_INF;
    if (S.mode[s] != 0) factor = (F)act_factor(S, s, T.sim_t);
  }
  const F fmag = (F)kl.x * (len - factor * (F)kl.y);
  F scale = fmag / len;
  if (SPECIAL && S.damp)
    scale += damper_scale<P, F>(S, s, dx, dy, dz, dx * dx + dy * dy + dz * dz);
  const F gx = scale * dx, gy = scale * dy, gz = scale * dz;
  R4 *fe = (R4 *)S.fext;
  red_add_agg(fe, (uint32_t)ab.x, (R)gx, (R)gy, (R)gz);
  red_add_agg(fe, (uint32_t)ab.y, -(R)gx, -(R)gy, -(R)gz);
  if (SPECIAL && special) {
    const F thr = (F)((const FS *)S.thr)[s];
    const F mag = fmag >= (F)0.0 ? fmag : -fmag;
    if (mag > thr) {
      count_spring(S, 0, s);
      S.s_alive[s] = 0;
      S.ends[s] = make_int2(-1, -1);
      if (S.e1) kill_entries(S, s);  // incidence layout present: keep it
                                     // consistent
    }
  }
}

// Standalone mass pass (engine.mass_pass; second half of the atomic step).
template <int P>
static __global__ void __launch_bounds__(256)
    k_mass(const KState S, const EnvP E, const StepP T) {
  pdl_wait();
  using R = typename Tr<P>::R;
  using R4 = typename Tr<P>::R4;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S.m_n) return;
  // every load of the mass issued up front (one round trip, not a chain
  // of flag -> f_ext -> position; the r3 ncu: long-scoreboard 149 per issue)
  const bool stop = stopped(S, T.step);
  const R4 v = ((const R4 *)S.vel)[i];
  R4 *fe = (R4 *)S.fext + i;
  const R4 f0 = *fe;
  const R4 me = ((const R4 *)S.pos[T.cur])[i];
  const auto ml = lo_at<P>(me, S.plo[T.cur], i);
  const R mass = mass_of<P>(S, me, i);
  if (stop) return;
  const uint32_t fl = flags_of(v.w);
  if (!(fl & MF_ALIVE)) return;
  if (fl & MF_FIXED) {
    fixed_mass<P>(S, T, i, v, fl | MF_FEXT);
    return;
  }
  integrate<P>(S, E, T, i, me, ml, mass, v, fl, f0.x, f0.y, f0.z);
  // f_ext cleared after the update's stores: a constant store issued while
  // the load of the same line is still in flight (the compiler hoisted it
  // there) held the SM's later memory instructions behind that miss --
  // 57 us instead of ~21 on config B (tools/probe/kmass_probe.cu)
  R4 z;
  z.x = z.y = z.z = z.w = (R)0.0;
  *fe = z;
}

inline unsigned blocks_for(int64_t n) { return (unsigned)((n + 255) / 256); }

// Host-side launchers, one set per precision (defined in sl_kernels_*.cu).
struct Launch {
  void (*gather)(const KState &, const EnvP &, const StepP &, cudaStream_t);
  void (*gather_tma)(const KState &, const EnvP &, const StepP &,
                     const TmaCfg &, int grid, cudaStream_t);
  int (*tma_setup)(int smem_bytes);  // opt into large dynamic smem
  void (*force_only)(const KState &, const EnvP &, const StepP &,
                     cudaStream_t);
  void (*spring_atomic)(const KState &, const StepP &, bool special,
                        cudaStream_t);
  void (*mass)(const KState &, const EnvP &, const StepP &, cudaStream_t);
  // owner-aggregated atomic force pass (split or exact layout)
  void (*owner_atomic)(const KState &, const StepP &, const struct ActP &,
                       cudaStream_t);
  // split layout (tolerance modes; no-ops for fp64)
  void (*split)(const KState &, const EnvP &, const StepP &,
                const struct ActP &, cudaStream_t);
  void (*split_force)(const KState &, const EnvP &, const StepP &,
                      const struct ActP &, cudaStream_t);
  void (*split_tma)(const KState &, const EnvP &, const StepP &,
                    const struct SplitCfg &, const struct ActP &, int grid,
                    cudaStream_t);
  int (*split_setup)(int smem_bytes, int u, int act);
  // tiled window kernel (fp32 split layout, sl_window.cuh)
  void (*win)(const KState &, const EnvP &, const StepP &,
              const struct WinCfg &, int grid, cudaStream_t);
  int (*win_setup)(const struct WinCfg &);
  // multi-step fused small-body kernel (fp32, sl_fused.cuh)
  void (*fused)(const KState &, const EnvP &, const struct FzCfg &,
                double dt, size_t smem, cudaStream_t);
  int (*fused_setup)(size_t smem, int maxm);
};

const Launch &launchers(int prec);

}  // namespace sl
