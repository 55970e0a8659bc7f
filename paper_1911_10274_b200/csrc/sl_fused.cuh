// sl_fused.cuh -- several steps per launch for small bodies (fp32):
// north_star "optional fusion of several steps per launch using
// shared-memory staging for small bodies"; SURVEY.md 7 build step 9.
//
// Config D (an RL batch of thousands of 5^3 robots) is a swarm of small
// disconnected bodies.  Bodies are packed into GROUPS of whole connected
// components (<= 512 masses, or <= 1024 with 1024-thread CTAs when a body
// needs it; the host finds component boundaries from
// the springs), one CTA per group, one thread per mass.  The group's
// positions (double-buffered), its incidence entries (16-bit local partner
// + 8-bit material code, A section then B section per mass, the split
// layout's order) and its material table live in shared memory for the
// whole launch; velocities and flags live in registers.  A launch runs all
// n steps of an sl_step call with one __syncthreads per step and touches
// HBM only to load the state at the start and store it at the end.
//
// Per-step semantics are the window kernel's (same entry arithmetic,
// win_body; same mass update, integrate_vals; actuation through the
// per-group table, factor in fp64 once per material per step).  A context
// is eligible only without special masses (breakable / custom-waveform
// springs), ghosts or oversized components.  Anything the fast path cannot
// represent -- a zero-length spring, a non-finite state -- aborts the whole
// launch: nothing is committed (final positions go to the other ping-pong
// buffer, velocities to a second buffer, swapped only on success) and the
// host re-runs the same steps through the per-step kernels, which own the
// reference's exact event semantics.
#pragma once
#include "sl_window.cuh"

namespace sl {

constexpr int FZ_MAXM = 512;    // masses per group = threads per CTA
constexpr int FZ_MAXM_L = 1024;  // large groups (bodies of 513..1024 masses,
                                 // e.g. the 10^3 cube of config A): 1 CTA/SM
constexpr int FZ_MAXR = 32;   // entry rows per mass (A + B)

struct FzCfg {
  int64_t n_groups;
  const int32_t *gstart;  // [g] first mass of the group
  const int32_t *gcount;  // [g] masses
  const uint16_t *ent;    // [g][ra + rb][maxm] local partner of the
                          // q-th entry of thread t (maxm: sentinel)
  const uint8_t *code;    // [g][ra + rb][maxm] material code
  const uint16_t *perm;   // [g][maxm] thread t -> local mass
  const uint8_t *cnt;     // [g][maxm] entries of thread t
  const uint8_t *cnt_a;   // [g][maxm] of which A-section entries
  const float2 *dict;     // [g][WIN_DMAX] (k, k L0)
  const unsigned char *actb;  // [g][WIN_ACTB] actuation block (window fmt)
  const uint8_t *has_act;     // [g]
  int ra, rb;                 // A / B rows per mass
  int maxm;                   // group capacity (threads per CTA): 512 / 1024
  void *vel_out;              // final velocities (swapped in on success)
  const double *times;        // [n_steps] step times (device)
  int64_t n_steps;
  int cur;        // position buffer read at step 0; final -> cur ^ 1
  int write_acc;  // store the last step's accelerations
};

// Group build: one CTA per group, one thread per mass.  fail[0] |= 1 when
// the group does not fit (partner outside the group, too many materials,
// special mass, hash collision).
template <int M>
static __global__ void __launch_bounds__(M)
    k_fused_build(const uint32_t *sp_j, const uint32_t *sp_w,
                  const float2 *sp_kl, const int32_t *sp_s, const int8_t *mode,
                  const double4 *act, const uint8_t *grp, const float4 *vel,
                  int a, int rows, uint32_t sent, uint32_t nul,
                  const int32_t *gstart, const int32_t *gcount, int ra, int rb,
                  uint16_t *ent, uint8_t *code, uint16_t *perm, uint8_t *cnt,
                  uint8_t *cnt_a, uint16_t *epos, float2 *dict,
                  unsigned char *actb,
                  uint8_t *has_act, uint8_t *zero, int32_t *gid,
                  unsigned long long *fail,
                  const int32_t *group_list = nullptr) {
  __shared__ int16_t scnt[M];
  __shared__ unsigned long long dkey[WIN_DMAX];
  __shared__ float2 dkl[WIN_DMAX];
  __shared__ double4 dact[WIN_DMAX];
  __shared__ int8_t dmode[WIN_DMAX];
  __shared__ int ok;
  // every group, or (O(edits) topology sync) the listed ones
  const int64_t g = group_list ? group_list[blockIdx.x] : blockIdx.x;
  const int li = threadIdx.x;
  const int32_t g0 = gstart[g], gn = gcount[g];
  const int64_t i = (int64_t)g0 + li;
  const bool mine = li < gn;
  if (li < WIN_DMAX) dkey[li] = WIN_EMPTY;
  if (li == 0) ok = 1;
  __syncthreads();
  MatTable tab{dkey, dkl, dact, dmode};
  const Mat zero_m = mat_zero();
  const unsigned long long zero_key = mat_hash(zero_m);
  if (li == 0 && tab.find(zero_key, true, &zero_m) < 0) ok = 0;
  if (mine && (flags_of(vel[i].w) & MF_SPECIAL)) ok = 0;
  __syncthreads();
  const int64_t sl = i >> 5;
  const int lane = (int)(i & 31);
  const uint32_t wd = mine ? sp_w[sl] : 0u;
  const int wa = (int)(wd & 0xFFFF), wb = (int)(wd >> 16);
  // entry q of this mass: (partner, kl index, spring slot) or none
  auto entry = [&](int q, uint32_t *kli, uint32_t *s) -> uint32_t {
    if (!mine) return 0xFFFFFFFFu;
    if (q < ra) {
      if (q >= wa) return 0xFFFFFFFFu;
      const int64_t e = (sl * rows + q) * 32 + lane;
      const uint32_t w = sp_j[e];
      if (w == sent) return 0xFFFFFFFFu;
      *kli = (uint32_t)((sl << (a + 5)) | (q << 5) | lane);
      *s = (uint32_t)sp_s[e];
      return w;
    }
    const int r = q - ra;
    if (r >= wb) return 0xFFFFFFFFu;
    const int64_t e = (sl * rows + (1 << a) + r) * 32 + lane;
    const uint32_t w = sp_j[e];
    if (w == nul) return 0xFFFFFFFFu;
    *kli = w;
    *s = (uint32_t)sp_s[e];
    return split_partner(w, a);
  };
  int n_mine = 0, n_a = 0;
  for (int q = 0; q < ra + rb; q++) {
    uint32_t kli = 0, s = 0;
    const uint32_t j = entry(q, &kli, &s);
    if (j == 0xFFFFFFFFu) continue;
    n_mine++;
    n_a += q < ra;
    if ((int64_t)j < g0 || (int64_t)j >= (int64_t)g0 + gn) ok = 0;
    const Mat x = mat_of_spring(sp_kl, mode, act, grp, kli, s);
    if (tab.find(mat_hash(x), true, &x) < 0) ok = 0;
  }
  // sort key: entry count, then A-section count (both loops warp-uniform)
  scnt[li] = (int16_t)(mine ? n_mine * 64 + n_a : -1);
  __syncthreads();
  // thread slot of this mass: masses sorted by entry count, descending
  // (stable), so a warp's 32 masses have similar counts and its loop runs
  // to about their own count instead of the group's maximum row count
  int t = 0;
  for (int j = 0; j < M; j++) {
    const int cj = scnt[j];
    t += cj > scnt[li] || (cj == scnt[li] && j < li);
  }
  perm[g * M + t] = (uint16_t)li;
  cnt[g * M + t] = (uint8_t)(mine ? n_mine : 0);
  cnt_a[g * M + t] = (uint8_t)(mine ? n_a : 0);
  const int zc = tab.find(zero_key, false, nullptr);
  if (mine) gid[i] = (int32_t)g;
  if (li == 0) zero[g] = (uint8_t)(zc < 0 ? 0 : zc);
  int qq = 0;  // compacted row: valid entries in (A rows, B rows) order
  for (int q = 0; q < ra + rb; q++) {
    uint32_t kli = 0, s = 0;
    const uint32_t j = entry(q, &kli, &s);
    if (j == 0xFFFFFFFFu) continue;
    const Mat x = mat_of_spring(sp_kl, mode, act, grp, kli, s);
    const int c = tab.find(mat_hash(x), false, nullptr);
    if (!tab.same(c, x)) ok = 0;
    const int64_t o = (g * (ra + rb) + qq) * M + t;
    ent[o] = (uint16_t)(j - (uint32_t)g0);
    code[o] = (uint8_t)(c < 0 ? 0 : c);
    // split row q of mass li -> (compacted row, thread): device kills
    epos[(g * (ra + rb) + q) * M + li] = (uint16_t)(qq * M + t);
    qq++;
  }
  for (; qq < ra + rb; qq++) {  // padding (never read: the loop stops at cnt)
    const int64_t o = (g * (ra + rb) + qq) * M + t;
    ent[o] = M;
    code[o] = (uint8_t)(zc < 0 ? 0 : zc);
  }
  __syncthreads();
  if (!ok) {
    if (li == 0) atomicOr(fail, 1ull);
    return;
  }
  if (li < WIN_DMAX) {  // table + actuation block, the window formats
    const bool used = dkey[li] != WIN_EMPTY;
    const float2 kl = used ? dkl[li] : make_float2(0.f, 0.f);
    dict[g * WIN_DMAX + li] = make_float2(kl.x, kl.x * kl.y);
    unsigned char *ab = actb + g * WIN_ACTB;
    ((double4 *)ab)[li] = used ? dact[li] : make_double4(0.0, 0.0, 0.0, 0.0);
    ((float2 *)(ab + 32 * WIN_DMAX))[li] = kl;
    ((int8_t *)(ab + 40 * WIN_DMAX))[li] = used ? dmode[li] : (int8_t)0;
  }
  if (li == 0) {
    int any = 0;
    for (int q = 0; q < WIN_DMAX; q++)
      if (dkey[q] != WIN_EMPTY && (dmode[q] == 1 || dmode[q] == 2)) any = 1;
    has_act[g] = (uint8_t)any;
  }
}

// The fused multi-step kernel (fp32).  Dynamic shared memory:
//   act (WIN_DMAX double4) | pos [2][M + 1] (x, y, z, lx) | low parts
//   [2][M + 1] (ly, lz) | tables [2] + static table (3 x WIN_DMAX float2) |
//   raw (k, L0) (WIN_DMAX float2) | entries (rows x M u32: partner |
//   code << 16) | modes
// (the global fp32 layout: compensated positions, sl_device.cuh lo_at)
template <int P, int M>
static __global__ void __launch_bounds__(M, M <= 512 ? 2 : 1)
    k_fused_small(const KState S, const EnvP E, const FzCfg C, double dt) {
  using R = typename Tr<P>::R;
  using R4 = typename Tr<P>::R4;
  using F2 = typename Tr<P>::F2;
  extern __shared__ __align__(16) unsigned char smem[];
  const int rows = C.ra + C.rb;
  double4 *sact = (double4 *)smem;
  // positions: record (x, y, z, lx) + (ly, lz), one 16 B and one 8 B
  // shared load per entry
  float4 *sp4 = (float4 *)(sact + WIN_DMAX);  // [2][M + 1]
  float2 *sl2 = (float2 *)(sp4 + 2 * (M + 1));  // [2][M + 1]
  F2 *stab = (F2 *)(sl2 + 2 * (M + 1));  // [3][..]
  F2 *skl = stab + 3 * WIN_DMAX;
  // entries packed as partner | code << 16: one shared load per entry
  uint32_t *sen = (uint32_t *)(skl + WIN_DMAX);
  int8_t *smode = (int8_t *)(sen + rows * M);
  __shared__ int sbad;
  const int64_t g = blockIdx.x;
  const int t = threadIdx.x;  // thread slot (masses sorted by entry count)
  const int32_t g0 = C.gstart[g], gn = C.gcount[g];
  const bool mine = t < gn;
  const int li = mine ? (int)C.perm[g * M + t] : t;  // local mass
  const int n_ent = mine ? (int)C.cnt[g * M + t] : 0;
  const int n_a = mine ? (int)C.cnt_a[g * M + t] : 0;
  const int64_t i = (int64_t)g0 + li;
  const bool act = C.has_act[g] != 0;
  // ---- load the group
  R4 me, v;
  float3 ml = make_float3(0.f, 0.f, 0.f);
  R mm = (R)1;
  uint32_t fl = 0;
  if (mine) {
    me = ((const R4 *)S.pos[C.cur])[i];
    ml = lo_at<P>(me, S.plo[C.cur], i);
    mm = mass_of<P>(S, me, i);
    v = ((const R4 *)S.vel)[i];
    fl = flags_of(v.w);
  } else {
    me.x = me.y = me.z = (R)SENTINEL_POS;
    me.w = (R)0;
    v.x = v.y = v.z = v.w = (R)0;
  }
  sp4[li] = me;
  sl2[li] = make_float2(ml.x, ml.y);
  if (li == 0) {
    R4 far;
    far.x = far.y = far.z = (R)SENTINEL_POS;
    far.w = (R)0;
    sp4[M] = sp4[2 * M + 1] = far;
    sl2[M] = sl2[2 * M + 1] = make_float2(0.f, 0.f);
    sbad = 0;
  }
  for (int q = 0; q < rows; q++) {
    const int64_t x = (g * rows + q) * M + t;
    sen[q * M + t] = (uint32_t)C.ent[x] | ((uint32_t)C.code[x] << 16);
  }
  if (t < WIN_DMAX) {
    stab[2 * WIN_DMAX + t] = C.dict[g * WIN_DMAX + t];
    if (act) {
      const unsigned char *ab = C.actb + g * WIN_ACTB;
      sact[t] = ((const double4 *)ab)[t];
      skl[t] = ((const float2 *)(ab + 32 * WIN_DMAX))[t];
      smode[t] = ((const int8_t *)(ab + 40 * WIN_DMAX))[t];
    }
  }
  // f_ext at the first step (loads / spring_pass results), then cleared
  R f0x = 0, f0y = 0, f0z = 0;
  const bool had_fext = mine && (fl & MF_FEXT);
  if (had_fext) {
    const R4 f = ((const R4 *)S.fext)[i];
    f0x = f.x;
    f0y = f.y;
    f0z = f.z;
  }
  const bool live = mine && (fl & MF_ALIVE);
  R ax = 0, ay = 0, az = 0;
  // step k's effective table (k, k L0 factor(T_k)) into buffer k & 1
  // (kernels.py:55-62), by the first WIN_DMAX threads; computed one step
  // ahead so each step needs one barrier
  auto eff_table = [&](int64_t k) {
    if (!act || t >= WIN_DMAX || k >= C.n_steps) return;
    const double T = __ldg(C.times + k);
    const double4 A = sact[t];
    const int m = smode[t];
    float f = 1.0f;
    if ((m == 1 || m == 2) && !(m == 2 && !(T >= A.z)))
      f = (float)(1.0 + A.x * sin(A.y * py_mod(T - A.z, A.w)));
    F2 e;
    e.x = skl[t].x;
    e.y = skl[t].x * (f * skl[t].y);
    stab[(k & 1) * WIN_DMAX + t] = e;
  };
  eff_table(0);
  __syncthreads();
  // ---- the steps
  int64_t k = 0;
  for (; k < C.n_steps; k++) {
    const int b = (int)(k & 1);
    const F2 *tab = act ? stab + b * WIN_DMAX : stab + 2 * WIN_DMAX;
    const float4 *pp = sp4 + b * (M + 1);
    const float2 *pl = sl2 + b * (M + 1);
    R4 np = me;
    if (live) {
      if (fl & MF_FIXED) {  // kernels.py:260-270
        v.x = v.y = v.z = (R)0;
        ax = ay = az = (R)0;
      } else {
        float2 gxy = make_float2(0.f, 0.f), bxy = gxy;
        R gz = 0, bz = 0;
        const float2 mlxy = make_float2(ml.x, ml.y);
        const uint32_t *e = sen + t;
        // this mass's own entries only (compacted at build), A and B
        // sections summed separately as the window / split kernels do
#pragma unroll 4
        for (int q = 0; q < n_a; q++) {
          const uint32_t w = e[q * M];
          win_body(me, mlxy, ml.z, pp[w & 0xFFFFu], pl[w & 0xFFFFu],
                   tab[w >> 16], gxy, gz);
        }
#pragma unroll 4
        for (int q = n_a; q < n_ent; q++) {
          const uint32_t w = e[q * M];
          win_body(me, mlxy, ml.z, pp[w & 0xFFFFu], pl[w & 0xFFFFu],
                   tab[w >> 16], bxy, bz);
        }
        const R fx = f0x + (gxy.x + bxy.x), fy = f0y + (gxy.y + bxy.y),
                fz = f0z + (gz + bz);
        f0x = f0y = f0z = (R)0;
        R4 nv;
        float3 nl;
        integrate_vals<P>(S, E, dt, i, me, ml, mm, v, fl, fx, fy, fz, np, nl,
                          nv, ax, ay, az);
        ml = nl;
        v = nv;
        const R z0 = np.x * (R)0 + np.y * (R)0 + np.z * (R)0 + v.x * (R)0 +
                     v.y * (R)0 + v.z * (R)0;
        if (!(z0 == (R)0)) sbad = 1;  // zero-length spring or blow-up
      }
    }
    sp4[(b ^ 1) * (M + 1) + li] = np;
    sl2[(b ^ 1) * (M + 1) + li] = make_float2(ml.x, ml.y);
    me = np;
    eff_table(k + 1);  // the other buffer: nobody reads it this step
    __syncthreads();
    if (sbad) break;
  }
  if (sbad) {  // nothing committed; the host re-runs the steps
    if (li == 0) atomicOr(S.status + 5, 1ull);
    return;
  }
  if (!mine) return;
  ((R4 *)S.pos[C.cur ^ 1])[i] = me;
  ((float2 *)S.plo[C.cur ^ 1])[i] = make_float2(ml.x, ml.y);
  R4 vo = v;
  set_flags(vo.w, fl & ~MF_FEXT);
  ((R4 *)C.vel_out)[i] = vo;
  if (C.write_acc && live) {
    R *a = (R *)S.acc + 3 * i;
    a[0] = ax;
    a[1] = ay;
    a[2] = az;
  }
  if (had_fext) atomicAdd(S.status + 6, 1ull);  // f_ext rows to clear
}

// f_ext rows of masses whose (pre-launch) flags had MF_FEXT are zeroed after
// a committed fused launch (kernels.py:372: the accumulator is cleared)
static __global__ void k_fused_clear_fext(int64_t m_n, const float4 *vel_old,
                                          float4 *fext) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m_n && (flags_of(vel_old[i].w) & MF_FEXT))
    fext[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// component boundaries: cover[b] = springs spanning (b - 1, b)
static __global__ void k_fused_cover(int64_t s_n, const int2 *ends,
                                     int32_t *diff) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= s_n) return;
  const int2 e = ends[s];
  if (e.x < 0) return;
  const int lo = e.x < e.y ? e.x : e.y, hi = e.x < e.y ? e.y : e.x;
  if (lo == hi) return;
  atomicAdd(diff + lo + 1, 1);
  atomicAdd(diff + hi + 1, -1);
}

}  // namespace sl
