// sl_split.cuh -- the "split" (half-duplex) incidence layout and its fused
// step kernels, used by the tolerance modes (fp32 / mixed).
//
// Why: the exact layout of sl_device.cuh stores every spring twice -- once
// in the incidence list of each endpoint, each copy carrying (k, L0) -- so a
// step streams 2 x (4 + 8) = 24 B per spring from HBM against the 16 B of
// algorithmic spring data (i, j, k, L0).  Here each spring
// keeps (k, L0) once, in the list of its m1 endpoint (section A); the m2
// endpoint's entry (section B) is a single 32-bit word holding the index of
// that (k, L0) cell, from which the partner mass is also decoded.  HBM bytes
// per spring: A word 4 + (k, L0) 8 + B word 4 = 16 -- the algorithmic
// figure.  The (k, L0) read of a B entry is a gather that hits L2 (the cell
// was streamed recently by the partner's slice, and the lattice's row-major
// ordering keeps partners within a few thousand masses).
//
// Layout (m_pad = m_n rounded up to 32, n_slices = m_pad / 32, WA = 2^a >=
// widest A section, WB = widest B section, rows = WA + WB):
//   sp_j [slice][rows][32] u32  rows [0, WA): A entries = partner mass index
//                               (sentinel m_pad if dead / padding)
//                               rows [WA, rows): B entries = kl index of the
//                               spring's A cell (sp_null if dead / padding)
//   sp_kl[slice][WA][32] F2     (k, L0) of A entries; kl index of (slice, r,
//                               lane) = slice << (a+5) | r << 5 | lane, so a
//                               B word decodes its partner with two ops:
//                               j = ((w >> a) & ~31) | (w & 31)
//   sp_s [slice][rows][32] i32  spring slot of every entry (special path)
//   sp_w [slice] u32            wA | wB << 16 (this slice's section widths;
//                               only these rows are streamed)
// Slice n_slices of sp_kl is all zero (sp_null points into it) and mass
// records [m_pad, m_pad + 32) hold a far-away sentinel position, so dead and
// padding entries contribute exactly 0 force (k = 0 at a finite distance)
// without a branch.
//
// Fast path (masses without actuated / breakable springs): branch-free
// k (|d| - L0) / |d| * d with one MUFU.RSQ.  A zero-length alive spring
// makes the sum non-finite (0 * inf); such a mass -- like a genuinely
// non-finite one -- is recomputed through the special path, which owns all
// side effects (zero-length flag, yield break, counters: kernels.py:50-54,
// 77-86).  Accumulation order is fixed by the layout (deterministic run to
// run), not the reference's slot order: tolerance modes only.
#pragma once
#include "sl_device.cuh"

namespace sl {

constexpr int SPLIT_MAX_WARPS = 12;  // warps per CTA (register budget)
constexpr int SPLIT_DEFAULT_WARPS = 12;
constexpr double SENTINEL_POS = 1.0e15;  // |d| finite, k = 0 => force 0

struct SplitCfg {
  int64_t n_slices;
  int u;                 // gather batch (rows per batch; stage rows padded)
  int act;               // actuated fast path (ActP groups in use)
  int cap_a, cap_b;      // stage capacity, rows (widest sections padded to u)
  int warps;             // warps per CTA
  uint32_t stage_bytes;  // pos + vel + A words + B words + A (k, L0)
};

__device__ __forceinline__ uint32_t split_partner(uint32_t w, int a) {
  return ((w >> a) & ~31u) | (w & 31u);
}

// Force on this mass from one entry, fast form (see header comment);
// `factor` scales the rest length (actuation, 1 otherwise).
template <int P, bool ACT>
__device__ __forceinline__ void split_body(typename Tr<P>::R4 me,
                                           typename Tr<P>::L ml,
                                           typename Tr<P>::R4 o,
                                           typename Tr<P>::L ol,
                                           typename Tr<P>::F2 kl,
                                           float factor,
                                           typename Tr<P>::R &fx,
                                           typename Tr<P>::R &fy,
                                           typename Tr<P>::R &fz) {
  using R = typename Tr<P>::R;
  using M = typename Tr<P>::M;
  M dx, dy, dz;
  pdiff<P>(me, ml, o, ol, dx, dy, dz);
  const M len2 = dx * dx + dy * dy + dz * dz;
  M r;
  if constexpr (P == PREC_FP32) {
    r = rsqrtf(len2);
  } else {
    r = (double)rsqrtf((float)len2);
    r = r * (1.5 - 0.5 * len2 * r * r);  // one Newton step, ~1e-14
  }
  M l0 = (M)kl.y;
  if constexpr (ACT) l0 = (M)factor * l0;
  const M sc = (M)kl.x * (len2 * r - l0) * r;
  fx += (R)(sc * dx);
  fy += (R)(sc * dy);
  fz += (R)(sc * dz);
}

// ---------------------------------------------------------------------------
// Sine actuation in the fast path of the fp32 mode (reference
// kernels.py:55-65 modes 1 and 2, actuation.py:57-69):
// factor = 1 + amp sin(freq t), t = (T - off) mod per (Python floor-mod),
// mode 2 only once T >= off.  Springs are grouped by (mode, amp, freq, per)
// -- a swarm of worm robots has one group -- and each (k, L0) cell gets a
// companion 16-byte act cell (o, sin B, cos B, group) with o = off mod per
// and B = freq o, computed once in fp64 when the layout is built.  Per step
// every CTA computes each group's phase P = T mod per and the angles
// A = freq P, A' = freq (P + per) in fp64, as (sin, cos) pairs in shared
// memory.  Per entry t = P - o (+ per when negative), and
//   sin(freq t) = sin(A - B) = sin A cos B - cos A sin B   (A' if wrapped),
// two FMAs instead of a range reduction and a polynomial.
//
// The waveform is discontinuous at every wrap (freq per is not a multiple
// of 2 pi), so the wrap DECISION must be the reference's: an entry whose
// fp32 t lies within eps = 1e-6 per of 0 or per (the fp32 path's error is
// < 3e-7 per), and every mode-2 entry, is recomputed from the spring's exact
// fp64 offset (sp_acto) with the reference's own arithmetic: d = T - off,
// then a floor-mod whose quotient is corrected to the exact one.  Group 0 is
// "not actuated" (amp 0: factor exactly 1).  Both endpoints evaluate the
// same factor from the same bits.  Callable waveforms stay on the exact
// per-entry path.
constexpr int MAX_ACT_GROUPS = 64;
struct ActP {
  int n;  // groups in use (incl. group 0)
  int8_t mode[MAX_ACT_GROUPS];
  float amp[MAX_ACT_GROUPS];
  double freq[MAX_ACT_GROUPS], per[MAX_ACT_GROUPS], inv_per[MAX_ACT_GROUPS];
};
struct ActG {  // one group, shared-memory copy for the current step
  float sa, ca, saw, caw;  // sin/cos of A = freq P and A' = freq (P + per)
  float phase, per, eps, amp;
  uint32_t quiescent, pad_;  // mode 2: factor 1 while T < off (slow path)
  double freqd, perd, inv_per;
};

// act cell of one spring (device: py_mod lives in sl_device.cuh)
__device__ __forceinline__ float4 act_cell(double off, double freq,
                                           double per, uint32_t grp) {
  if (grp == 0) return make_float4(0.f, 0.f, 1.f, 0.f);
  const double o = py_mod(off, per);
  double sb, cb;
  sincos(freq * o, &sb, &cb);
  return make_float4((float)o, (float)sb, (float)cb, __uint_as_float(grp));
}

// block-wide: the group table for step time sim_t into shared memory
__device__ __forceinline__ void act_table(const ActP &A, double sim_t,
                                          ActG *tab) {
  for (int g = threadIdx.x; g < A.n; g += blockDim.x) {
    const double p = py_mod(sim_t, A.per[g]);
    double sa, ca, saw, caw;
    sincos(A.freq[g] * p, &sa, &ca);
    sincos(A.freq[g] * (p + A.per[g]), &saw, &caw);
    const float per = (float)A.per[g];
    tab[g] = ActG{(float)sa, (float)ca, (float)saw, (float)caw, (float)p,
                  per, per * 1e-6f, A.amp[g], A.mode[g] == 2 ? 1u : 0u, 0u,
                  A.freq[g], A.per[g], A.inv_per[g]};
  }
  __syncthreads();
}

// Exact-phase factor (rare: near a wrap, or mode 2).  floor-mod: r = d -
// q per for q = floor(d / per) exactly; the estimate is off by at most one
// and corrected by the sign of the exact residual (fma rounds once, never
// across zero), so r is the correctly rounded d - q per -- the value
// Python's fmod-then-add produces (kernels.py:58, SURVEY.md 7 hard part 2).
static __device__ __noinline__ float act_slow(const ActG *G, double off,
                                              double sim_t) {
  if (G->quiescent && !(sim_t >= off)) return 1.0f;  // kernels.py:61
  const double d = sim_t - off;
  const double per = G->perd;
  const double q = floor(d * G->inv_per);
  double r = fma(-q, per, d);
  if (r < 0.0) {
    r = fma(-(q - 1.0), per, d);
  } else {
    const double r2 = fma(-(q + 1.0), per, d);
    r = r2 >= 0.0 ? r2 : r;
  }
  return (float)(1.0 + (double)G->amp * sin(G->freqd * r));
}

// factor of act cell c; kli() yields its kl index (slow path only)
template <class K>
__device__ __forceinline__ float act_fast(const ActG *tab, float4 c,
                                          const double *acto, K kli,
                                          double sim_t) {
  const ActG *G = tab + __float_as_uint(c.w);
  const float4 sc = *(const float4 *)G;  // sa, ca, saw, caw
  const float4 pp = *(const float4 *)&G->phase;  // phase, per, eps, amp
  const float d = pp.x - c.x;
  const bool wrap = d < 0.f;
  const float t = wrap ? d + pp.y : d;
  if ((t < pp.z) | (t > pp.y - pp.z) | (G->quiescent != 0u))
    return act_slow(G, acto[kli()], sim_t);
  const float sa = wrap ? sc.z : sc.x, ca = wrap ? sc.w : sc.y;
  return fmaf(pp.w, fmaf(sa, c.z, -ca * c.y), 1.0f);
}

// Fast spring forces of one mass.  ja / jb / kla (/ kaa) point at the lane's
// first A word, B word, A (k, L0) (and A act key), lane-strided by 32
// (shared-memory stage or global memory); wa / wb are the slice's section
// widths; tab is the block's actuation table (ACT only).
template <int P, int U, bool PADDED, bool ACT>
__device__ __forceinline__ void split_fast(const KState &S,
                                           const typename Tr<P>::R4 *pos,
                                           const void *plo,
                                           const uint32_t *ja,
                                           const uint32_t *jb,
                                           const typename Tr<P>::F2 *kla,
                                           const float4 *kaa,
                                           uint32_t kc0, const ActG *tab,
                                           double sim_t,
                                           int wa, int wb,
                                           typename Tr<P>::R4 me,
                                           typename Tr<P>::L ml,
                                           typename Tr<P>::R &fx,
                                           typename Tr<P>::R &fy,
                                           typename Tr<P>::R &fz) {
  using R = typename Tr<P>::R;
  using R4 = typename Tr<P>::R4;
  using F2 = typename Tr<P>::F2;
  using L = typename Tr<P>::L;
  const F2 *gkl = (const F2 *)S.sp_kl;
  const float4 *gact = S.sp_actc;
  const double *acto = S.sp_acto;
  const int a = S.sp_a;
  auto fa = [&](int row) {
    return ACT ? act_fast(tab, kaa[32 * row], acto,
                          [&] { return kc0 + 32u * row; }, sim_t)
               : 1.0f;
  };
  if constexpr (PADDED) {
    // stage rows are padded to whole batches: batch t of section A and
    // batch t of section B issue all their gathers together (one exposed L2
    // round trip per pair), then reduce A then B
    // B sums into its own accumulators: two independent FFMA chains
    R bx = 0, by = 0, bz = 0;
    for (int t = 0; t < wa || t < wb; t += U) {
      R4 oa[U], ob[U];
      L la[U], lb[U];
      F2 kb[U];
      float4 ab[U];
      const bool has_a = t < wa, has_b = t < wb;  // warp-uniform
      if (has_a) {
#pragma unroll
        for (int u = 0; u < U; u++) {
          const uint32_t j = ja[32 * (t + u)];
          oa[u] = ldg4(pos + j);
          la[u] = lo_at<P>(oa[u], plo, j);
        }
      }
      if (has_b) {
#pragma unroll
        for (int u = 0; u < U; u++) {
          const uint32_t w = jb[32 * (t + u)];
          kb[u] = __ldg(gkl + w);
          if constexpr (ACT) ab[u] = __ldg(gact + w);
          ob[u] = ldg4(pos + split_partner(w, a));
          lb[u] = lo_at<P>(ob[u], plo, split_partner(w, a));
        }
      }
      if (has_a) {
#pragma unroll
        for (int u = 0; u < U; u++)
          split_body<P, ACT>(me, ml, oa[u], la[u], kla[32 * (t + u)],
                             fa(t + u), fx, fy, fz);
      }
      if (has_b) {
#pragma unroll
        for (int u = 0; u < U; u++)
          split_body<P, ACT>(me, ml, ob[u], lb[u], kb[u],
                             ACT ? act_fast(tab, ab[u], acto,
                                            [&] { return jb[32 * (t + u)]; },
                                            sim_t)
                                 : 1.0f,
                             bx, by, bz);
      }
    }
    fx += bx;
    fy += by;
    fz += bz;
    return;
  }
  // section A: partner index + (k, L0) from the source rows
  for (int t = 0; t < wa; t += U) {
    R4 o[U];
    L lo[U];
#pragma unroll
    for (int u = 0; u < U; u++)
      if (t + u < wa) {
        const uint32_t j = ja[32 * (t + u)];
        o[u] = ldg4(pos + j);
        lo[u] = lo_at<P>(o[u], plo, j);
      }
#pragma unroll
    for (int u = 0; u < U; u++)
      if (t + u < wa)
        split_body<P, ACT>(me, ml, o[u], lo[u], kla[32 * (t + u)], fa(t + u),
                           fx, fy, fz);
  }
  // section B: (k, L0) gathered from the partner's A cell (L2)
  for (int t = 0; t < wb; t += U) {
    R4 o[U];
    L lo[U];
    F2 kl[U];
    float4 ab[U];
#pragma unroll
    for (int u = 0; u < U; u++)
      if (t + u < wb) {
        const uint32_t w = jb[32 * (t + u)];
        kl[u] = __ldg(gkl + w);
        if constexpr (ACT) ab[u] = __ldg(gact + w);
        o[u] = ldg4(pos + split_partner(w, a));
        lo[u] = lo_at<P>(o[u], plo, split_partner(w, a));
      }
#pragma unroll
    for (int u = 0; u < U; u++)
      if (t + u < wb)
        split_body<P, ACT>(me, ml, o[u], lo[u], kl[u],
                           ACT ? act_fast(tab, ab[u], acto,
                                          [&] { return jb[32 * (t + u)]; },
                                          sim_t)
                               : 1.0f,
                           fx, fy, fz);
  }
}

// One entry through the full reference semantics (kernels.py:46-83):
// actuation factor, zero-length flag, yield break.  Side effects on the
// spring (alive flag, counters, zero-length flag) are made once, by the m1
// endpoint (section A); each endpoint marks only its own entry dead, both
// reaching the same decision from bit-identical inputs (d and -d square to
// the same bits).
template <int P>
__device__ __forceinline__ void split_entry_exact(
    const KState *S, int64_t e, bool side_b, typename Tr<P>::R4 me,
    typename Tr<P>::L ml, typename Tr<P>::R4 other, typename Tr<P>::L ol,
    typename Tr<P>::F2 kl, double sim_t, typename Tr<P>::R &fx,
    typename Tr<P>::R &fy, typename Tr<P>::R &fz) {
  using R = typename Tr<P>::R;
  using F = typename Tr<P>::M;
  using FS = typename Tr<P>::F;
  F dx, dy, dz;
  pdiff<P>(me, ml, other, ol, dx, dy, dz);
  const F len2 = dx * dx + dy * dy + dz * dz;
  const int32_t s = S->sp_s[e];
  if (len2 == (F)0.0) {
    if (!side_b && !S->s_degen[s]) {
      S->s_degen[s] = 1;
      count_spring(*S, 2, s);
    }
    return;
  }
  const int mode = S->mode[s];
  F factor = (F)1.0;
  if (mode != 0) factor = (F)act_factor(*S, s, sim_t);
  const F len = sqrt(len2);
  const F fmag = (F)kl.x * (len - factor * (F)kl.y);
  F scale = fmag / len;
  if (S->damp) {
    // damper on d = other - me: c ((v_other - v_me) . d) / |d|^2, the same
    // bits at both endpoints (both vectors negate)
    const double c = S->damp[s];
    if (c != 0.0) {
      const int2 ab = S->ends[s];
      using R4 = typename Tr<P>::R4;
      const R4 vm = ((const R4 *)S->vel)[side_b ? ab.y : ab.x];
      const R4 vo = ((const R4 *)S->vel)[side_b ? ab.x : ab.y];
      const F vr = (F)(vo.x - vm.x) * dx + (F)(vo.y - vm.y) * dy +
                   (F)(vo.z - vm.z) * dz;
      scale += (F)c * vr / len2;
    }
  }
  fx += (R)(scale * dx);
  fy += (R)(scale * dy);
  fz += (R)(scale * dz);
  const F thr = (F)((const FS *)S->thr)[s];
  const F mag = fmag >= (F)0.0 ? fmag : -fmag;
  if (mag > thr) {
    S->sp_j[e] = side_b ? S->sp_null : S->sp_sent;
    if (!side_b) {
      count_spring(*S, 0, s);
      S->s_alive[s] = 0;
      S->ends[s] = make_int2(-1, -1);
    }
  }
}

// Rare path, kept out of line; it reads the context state through the
// device-memory copy (S.self) so the kernel never spills its parameter block
// to the stack.
template <class R>
struct Vec3R {
  R x, y, z;
};

template <int P>
__device__ __noinline__ Vec3R<typename Tr<P>::R> split_special(
    const KState *S, const typename Tr<P>::R4 *pos, const void *plo,
    const uint32_t *ja, const uint32_t *jb, const typename Tr<P>::F2 *kla,
    int wa, int wb, int64_t ea, int64_t eb, typename Tr<P>::R4 me,
    typename Tr<P>::L ml, double sim_t, typename Tr<P>::R fx,
    typename Tr<P>::R fy, typename Tr<P>::R fz) {
  using F2 = typename Tr<P>::F2;
  const F2 *gkl = (const F2 *)S->sp_kl;
  const uint32_t sent = S->sp_sent, nul = S->sp_null;
  const int a = S->sp_a;
  for (int t = 0; t < wa; t++) {
    const uint32_t j = ja[32 * t];
    if (j == sent) continue;
    split_entry_exact<P>(S, ea + 32 * (int64_t)t, false, me, ml, pos[j],
                         lo_at<P>(pos[j], plo, j), kla[32 * t], sim_t, fx, fy,
                         fz);
  }
  for (int t = 0; t < wb; t++) {
    const uint32_t w = jb[32 * t];
    if (w == nul) continue;
    const uint32_t j = split_partner(w, a);
    split_entry_exact<P>(S, eb + 32 * (int64_t)t, true, me, ml, pos[j],
                         lo_at<P>(pos[j], plo, j), gkl[w], sim_t, fx, fy, fz);
  }
  return {fx, fy, fz};
}

template <int P, int U, bool PADDED, bool ACT>
__device__ __forceinline__ void split_forces(
    const KState &S, const typename Tr<P>::R4 *pos, const void *plo,
    const uint32_t *ja, const uint32_t *jb, const typename Tr<P>::F2 *kla,
    const float4 *kaa, uint32_t kc0, const ActG *tab, int wa, int wb,
    int64_t ea, int64_t eb, uint32_t fl, typename Tr<P>::R4 me,
    typename Tr<P>::L ml, double sim_t, typename Tr<P>::R &fx,
    typename Tr<P>::R &fy, typename Tr<P>::R &fz) {
  using R = typename Tr<P>::R;
  if (!(fl & MF_SPECIAL)) {
    R gx = fx, gy = fy, gz = fz;
    split_fast<P, U, PADDED, ACT>(S, pos, plo, ja, jb, kla, kaa, kc0, tab,
                                  sim_t, wa, wb, me, ml, gx, gy, gz);
    if (isfinite(gx + gy + gz)) {
      fx = gx;
      fy = gy;
      fz = gz;
      return;
    }
  }
  const Vec3R<R> f = split_special<P>(S.self, pos, plo, ja, jb, kla, wa, wb,
                                      ea, eb, me, ml, sim_t, fx, fy, fz);
  fx = f.x;
  fy = f.y;
  fz = f.z;
}

// ---------------------------------------------------------------------------
// Owner-aggregated ATOMIC accumulation on the split layout (the paper's
// atomic design; reference linearizable accumulation,
// kernels.py:28-86 -- order-free, tolerance only): one thread per mass
// walks its A section (the springs it is m1 of), sums their forces in
// registers and pushes -f to each m2 with a vector RED, then adds its own
// sum with one RED -- 14 reductions per lattice mass instead of the 26 of
// one thread per spring.  Every spring is evaluated exactly once.
// Special masses (callable waveforms, yield, dampers) take the reference
// semantics per entry (split_atomic_exact); a yield break kills both of the
// spring's entries.

// one A entry through the full reference semantics; returns the force on
// m1 (this mass) in g, false if it contributes nothing
template <int P>
__device__ __noinline__ bool split_atomic_exact(
    const KState *S, int64_t e, typename Tr<P>::R4 me, typename Tr<P>::L ml,
    typename Tr<P>::R4 other, typename Tr<P>::L ol, typename Tr<P>::F2 kl,
    double sim_t, typename Tr<P>::M *g) {
  using F = typename Tr<P>::M;
  using FS = typename Tr<P>::F;
  F dx, dy, dz;
  pdiff<P>(me, ml, other, ol, dx, dy, dz);
  const F len2 = dx * dx + dy * dy + dz * dz;
  const int32_t s = S->sp_s[e];
  if (len2 == (F)0.0) {  // kernels.py:50-54
    if (!S->s_degen[s]) {
      S->s_degen[s] = 1;
      count_spring(*S, 2, s);
    }
    return false;
  }
  F factor = (F)1.0;
  if (S->mode[s] != 0) factor = (F)act_factor(*S, s, sim_t);
  const F len = sqrt(len2);
  const F fmag = (F)kl.x * (len - factor * (F)kl.y);
  F scale = fmag / len;
  if (S->damp) scale += damper_scale<P, F>(*S, s, dx, dy, dz, len2);
  g[0] = scale * dx;
  g[1] = scale * dy;
  g[2] = scale * dz;
  const F thr = (F)((const FS *)S->thr)[s];
  const F mag = fmag >= (F)0.0 ? fmag : -fmag;
  if (mag > thr) {  // breaks after applying its force (kernels.py:77-83)
    count_spring(*S, 0, s);
    S->s_alive[s] = 0;
    S->ends[s] = make_int2(-1, -1);
    kill_entries(*S, s);
  }
  return true;
}

template <int P, bool ACT>
static __global__ void __launch_bounds__(256)
    k_split_atomic(const KState S, const StepP T, const ActP A) {
  pdl_wait();
  using R = typename Tr<P>::R;
  using R4 = typename Tr<P>::R4;
  using F2 = typename Tr<P>::F2;
  using M = typename Tr<P>::M;
  __shared__ ActG tab[ACT ? MAX_ACT_GROUPS : 1];
  if (stopped(S, T.step)) return;  // uniform
  if constexpr (ACT) act_table(A, T.sim_t, tab);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S.m_n) return;
  const uint32_t fl = flags_of(((const R4 *)S.vel)[i].w);
  if (!(fl & MF_ALIVE)) return;
  const R4 *pos = (const R4 *)S.pos[T.cur];
  const void *plo = S.plo[T.cur];
  const R4 me = pos[i];
  const typename Tr<P>::L ml = lo_at<P>(me, plo, i);
  const int64_t w = i >> 5;
  const int wa = (int)(__ldg(S.sp_w + w) & 0xFFFF);
  const int64_t ea = w * S.sp_rows * 32 + (i & 31);
  const int64_t kc = (w << (S.sp_a + 5)) | (i & 31);
  const F2 *kla = (const F2 *)S.sp_kl + kc;
  const uint32_t sent = S.sp_sent;
  R4 *fe = (R4 *)S.fext;
  M ox = 0, oy = 0, oz = 0;
  if (fl & MF_SPECIAL) {
    for (int t = 0; t < wa; t++) {
      const uint32_t j = __ldg(S.sp_j + ea + 32 * t);
      if (j == sent) continue;
      const R4 o = ldg4(pos + j);
      M g[3];
      if (!split_atomic_exact<P>(S.self, ea + 32 * t, me, ml, o,
                                 lo_at<P>(o, plo, j), kla[32 * t], T.sim_t,
                                 g))
        continue;
      ox += g[0];
      oy += g[1];
      oz += g[2];
      red_add(fe + j, -(R)g[0], -(R)g[1], -(R)g[2]);
    }
    red_add(fe + i, (R)ox, (R)oy, (R)oz);
    return;
  }
  // fast path, U entries per batch: every load of a batch is issued before
  // any is consumed (the kernel is latency-bound on the dependent partner
  // gathers, profiles/ncu_k_split_atomic_r2.txt)
  constexpr int U = 4;
  for (int t0 = 0; t0 < wa; t0 += U) {
    uint32_t j[U];
    R4 o[U];
    typename Tr<P>::L ol[U];
    F2 kl[U];
#pragma unroll
    for (int u = 0; u < U; u++)
      j[u] = t0 + u < wa ? __ldg(S.sp_j + ea + 32 * (t0 + u)) : sent;
#pragma unroll
    for (int u = 0; u < U; u++) {
      o[u] = ldg4(pos + j[u]);  // sentinel rows for padding / dead entries
      ol[u] = lo_at<P>(o[u], plo, j[u]);
      kl[u] = t0 + u < wa ? kla[32 * (t0 + u)] : F2{};
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (j[u] == sent) continue;
      M dx, dy, dz;
      pdiff<P>(me, ml, o[u], ol[u], dx, dy, dz);
      const M len2 = dx * dx + dy * dy + dz * dz;
      if (len2 == (M)0) {  // zero length: flag it, no force
        const int32_t s = S.sp_s[ea + 32 * (t0 + u)];
        if (!S.s_degen[s]) {
          S.s_degen[s] = 1;
          count_spring(S, 2, s);
        }
        continue;
      }
      M r;
      if constexpr (P == PREC_FP32) {
        r = rsqrtf(len2);
      } else {
        r = (double)rsqrtf((float)len2);
        r = r * (1.5 - 0.5 * len2 * r * r);
      }
      M l0 = (M)kl[u].y;
      if constexpr (ACT)
        l0 = (M)act_fast(tab, S.sp_actc[kc + 32 * (t0 + u)], S.sp_acto,
                         [&] { return (uint32_t)(kc + 32 * (t0 + u)); },
                         T.sim_t) *
             l0;
      const M sc = (M)kl[u].x * (len2 * r - l0) * r;
      const M gx = sc * dx, gy = sc * dy, gz = sc * dz;
      ox += gx;
      oy += gy;
      oz += gz;
      red_add(fe + j[u], -(R)gx, -(R)gy, -(R)gz);
    }
  }
  red_add(fe + i, (R)ox, (R)oy, (R)oz);
}

// Plain variant: one thread per mass, entries read from global memory.
// Serves spring_pass (FORCE_ONLY) and layouts too wide for the TMA stages.
template <int P, bool FORCE_ONLY, bool ACT>
static __global__ void __launch_bounds__(256)
    k_split_step(const KState S, const EnvP E, const StepP T, const ActP A) {
  pdl_wait();
  using R = typename Tr<P>::R;
  using R4 = typename Tr<P>::R4;
  using F2 = typename Tr<P>::F2;
  __shared__ ActG tab[ACT ? MAX_ACT_GROUPS : 1];
  if (!FORCE_ONLY && stopped(S, T.step)) return;  // uniform
  if constexpr (ACT) act_table(A, T.sim_t, tab);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S.m_n) return;
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
  const uint32_t wd = __ldg(S.sp_w + w);
  const int64_t ea = w * S.sp_rows * 32 + (i & 31);
  const int64_t eb = ea + ((int64_t)32 << S.sp_a);
  const int64_t kc = (w << (S.sp_a + 5)) | (i & 31);
  split_forces<P, 4, false, ACT>(S, pos, plo, S.sp_j + ea, S.sp_j + eb,
                                 (const F2 *)S.sp_kl + kc,
                                 ACT ? S.sp_actc + kc : nullptr,
                                 (uint32_t)kc, tab,
                                 wd & 0xFFFF, wd >> 16, ea, eb, fl, me, ml,
                                 T.sim_t, fx, fy, fz);
  finish_mass<P, FORCE_ONLY>(S, E, T, i, me, ml, mass_of<P>(S, me, i), v,
                             fl, fx, fy, fz);
}

// TMA-pipelined fused step on the split layout (production path of the
// tolerance modes).  Same skeleton as k_gather_tma: persistent CTAs, each
// warp owns a strided sequence of 32-mass slices and a private 2-stage
// shared-memory ring; lane 0 streams the next slice (pos, vel, A words,
// B words, A (k, L0): five bulk async copies on one mbarrier) while the warp
// computes the current one.
template <int P, int U, bool ACT>
static __global__ void __launch_bounds__(SPLIT_MAX_WARPS * 32)
    k_split_tma(const KState S, const EnvP E, const StepP T,
                const SplitCfg C, const ActP A) {
  pdl_wait();
  using R = typename Tr<P>::R;
  using R4 = typename Tr<P>::R4;
  using F2 = typename Tr<P>::F2;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ ActG tab[ACT ? MAX_ACT_GROUPS : 1];
  if (stopped(S, T.step)) return;  // uniform across the grid
  if constexpr (ACT) act_table(A, T.sim_t, tab);
  // warp index broadcast from lane 0: provably warp-uniform for ptxas, so
  // the stage addresses below live in uniform registers
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  unsigned char *ring = smem + (size_t)warp * 2 * C.stage_bytes;
  uint64_t *bars =
      (uint64_t *)(smem + (size_t)C.warps * 2 * C.stage_bytes) + 2 * warp;
  constexpr uint32_t MB = 32 * sizeof(R4);
  const uint32_t ja_off = 2 * MB;
  const uint32_t jb_off = ja_off + (uint32_t)C.cap_a * 128u;
  const uint32_t kl_off = jb_off + (uint32_t)C.cap_b * 128u;
  const uint32_t ac_off = kl_off + (uint32_t)C.cap_a * 32u * sizeof(F2);
  if (lane == 0) {
    mbar_init(bars + 0, 1);
    mbar_init(bars + 1, 1);
    fence_proxy_async();
  }
  __syncwarp();
  const R4 *pos = (const R4 *)S.pos[T.cur];
  const int a = S.sp_a;
  const int64_t rows32 = (int64_t)S.sp_rows * 32;
  const int64_t stride = (int64_t)gridDim.x * C.warps;
  int64_t s = (int64_t)blockIdx.x * C.warps + warp;
  // whole warp: issue the five bulk copies of slice sl into a stage
  // 32-bit element offsets (the layout build guarantees they fit)
  const uint32_t rows32u = (uint32_t)rows32;
  const uint32_t jb_rel = 32u << a;
  auto issue = [&](int64_t sl, uint32_t wd, int stage) {
    const uint32_t su = (uint32_t)sl;
    const uint32_t wa = wd & 0xFFFF, wb = wd >> 16;
    unsigned char *dst = ring + (stage ? C.stage_bytes : 0u);
    const uint32_t *jsl = S.sp_j + su * rows32u;
    const uint32_t kb = wa * 32u * (uint32_t)sizeof(F2);
    const uint32_t ab = ACT ? wa * 32u * 16u : 0u;
    bulk_stage_elect(bars + stage, 2 * MB + (wa + wb) * 128u + kb + ab, dst,
                     pos + su * 32u, MB, dst + MB,
                     (const R4 *)S.vel + su * 32u, MB, dst + ja_off, jsl,
                     wa * 128u, dst + kl_off,
                     (const F2 *)S.sp_kl + (su << (a + 5)), kb, dst + jb_off,
                     jsl + jb_rel, wb * 128u, dst + ac_off,
                     S.sp_actc + (su << (a + 5)), ab);
  };
  // slice widths, loaded by every lane (one transaction) and broadcast
  auto widths = [&](int64_t sl) {
    const uint32_t w = sl < C.n_slices ? __ldg(S.sp_w + sl) : 0u;
    return __shfl_sync(0xffffffffu, w, 0);
  };
  uint32_t wcur = widths(s), wnxt = widths(s + stride);
  uint32_t wraw = s + 2 * stride < C.n_slices ? __ldg(S.sp_w + s + 2 * stride)
                                               : 0u;  // one more in flight
  if (s < C.n_slices) issue(s, wcur, 0);
  for (int k = 0; s < C.n_slices; s += stride, k++) {
    const int stage = k & 1;
    const uint32_t wd = wcur;
    if (s + stride < C.n_slices) {
      fence_proxy_async();  // generic reads of that stage finished (syncwarp)
      issue(s + stride, wnxt, stage ^ 1);
    }
    wcur = wnxt;
    wnxt = __shfl_sync(0xffffffffu, wraw, 0);
    wraw = s + 3 * stride < C.n_slices ? __ldg(S.sp_w + s + 3 * stride) : 0u;
    const int64_t i = s * 32 + lane;
    const unsigned char *st = ring + (size_t)stage * C.stage_bytes;
    {
      // rows between the section widths and the next multiple of U are not
      // TMA destinations: fill them with zero-force padding so the batches
      // run without guards
      const int wa = wd & 0xFFFF, wb = wd >> 16;
      uint32_t *sja = (uint32_t *)(ring + (size_t)stage * C.stage_bytes +
                                   ja_off) + lane;
      F2 *skl = (F2 *)(ring + (size_t)stage * C.stage_bytes + kl_off) + lane;
      float4 *sac = (float4 *)(ring + (size_t)stage * C.stage_bytes +
                                 ac_off) + lane;
      F2 zero;
      zero.x = zero.y = 0;
      for (int r = wa; r < (wa + U - 1) / U * U; r++) {
        sja[32 * r] = S.sp_sent;
        skl[32 * r] = zero;
        if (ACT) sac[32 * r] = make_float4(0.f, 0.f, 1.f, 0.f);
      }
      uint32_t *sjb = (uint32_t *)(ring + (size_t)stage * C.stage_bytes +
                                   jb_off) + lane;
      for (int r = wb; r < (wb + U - 1) / U * U; r++) sjb[32 * r] = S.sp_null;
    }
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
        const int64_t ea = s * rows32 + lane;
        const int64_t eb = ea + ((int64_t)32 << a);
        split_forces<P, U, true, ACT>(
            S, pos, plo, (const uint32_t *)(st + ja_off) + lane,
            (const uint32_t *)(st + jb_off) + lane,
            (const F2 *)(st + kl_off) + lane,
            (const float4 *)(st + ac_off) + lane,
            ((uint32_t)s << (a + 5)) | (uint32_t)lane, tab, wd & 0xFFFF,
            wd >> 16,
            ea, eb, fl, me, ml, T.sim_t, fx, fy, fz);
        finish_mass<P, false>(S, E, T, i, me, ml, mass_of<P>(S, me, i), v, fl,
                              fx, fy, fz);
      }
    }
    __syncwarp();
  }
}

}  // namespace sl
