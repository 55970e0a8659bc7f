/*
 * softlat_oracle.c -- CPU restatement of the reference spring-mass step.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path in paper_1911_10274_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The
 * product path never links or calls it.
 *
 * It restates, in plain C with strict IEEE double arithmetic (compile with
 * -ffp-contract=off, no -ffast-math), the numba kernels of the reference:
 *
 *   orc_spring_serial   <- /root/reference/pkg/src/softlat/kernels.py:28-86
 *   orc_spring_slotted  <- kernels.py:166-232
 *   orc_reduce_slots    <- kernels.py:235-247
 *   orc_build_slots     <- engine.py:105-118 (stable argsort by owner)
 *   orc_mass_pass       <- kernels.py:250-376
 *
 * The reference compiles the same bodies with numba/LLVM without FMA
 * contraction (probe), so with -ffp-contract=off this oracle is
 * bit-identical to the reference serial backend; tests/golden pins that.
 * OpenMP variants (slotted spring + reduce + mass pass) are bit-identical to
 * serial by construction (each output element is written by one thread in
 * the same operation order), exactly like the reference's slotted backend.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_API __attribute__((visibility("default")))

/* Python float modulo (numba follows CPython float_rem): result takes the
 * sign of the divisor; an exact zero becomes copysign(0, b).
 * Used by the actuation phase, kernels.py:58, actuation.py:57-59. */
static inline double py_mod(double a, double b) {
    double r = fmod(a, b);
    if (r != 0.0) {
        if ((r < 0.0) != (b < 0.0)) r += b;
    } else {
        r = copysign(0.0, b);
    }
    return r;
}

/* Rest-length factor, kernels.py:55-65. */
static inline double act_factor(int8_t mode, double sim_t, double amp,
                                double freq, double off, double per,
                                double custom) {
    if (mode == 1) {
        double t = py_mod(sim_t - off, per);
        return 1.0 + amp * sin(freq * t);
    } else if (mode == 2) {
        if (sim_t >= off) {
            double t = py_mod(sim_t - off, per);
            return 1.0 + amp * sin(freq * t);
        }
        return 1.0;
    } else if (mode == 3) {
        return custom;
    }
    return 1.0;
}

typedef struct {
    int64_t s_n;
    uint8_t *s_alive;
    const int64_t *s_m1, *s_m2, *s_m1gen, *s_m2gen;
    const uint8_t *m_alive;
    const int64_t *m_gen;
    const double *pos; /* [M,3] */
    const double *rest, *k, *diam, *yield;
    const int8_t *mode;
    const double *amp, *freq, *off, *per, *custom;
    uint8_t *s_degen;
    double sim_t;
} orc_springs;

/* Per-spring work shared by the serial and slotted passes.  Returns
 * 0 = no force (dead / invalid / degenerate), 1 = force in *f.
 * Side effects and counter increments follow kernels.py:37-83. */
static inline int spring_eval(const orc_springs *S, int64_t s, double f[3],
                              int64_t *broken, int64_t *invalid,
                              int64_t *degen_new) {
    if (!S->s_alive[s]) return 0;
    int64_t i = S->s_m1[s], j = S->s_m2[s];
    if (!S->m_alive[i] || !S->m_alive[j] || S->m_gen[i] != S->s_m1gen[s] ||
        S->m_gen[j] != S->s_m2gen[s]) {
        S->s_alive[s] = 0;
        (*invalid)++;
        return 0;
    }
    double dx = S->pos[3 * j + 0] - S->pos[3 * i + 0];
    double dy = S->pos[3 * j + 1] - S->pos[3 * i + 1];
    double dz = S->pos[3 * j + 2] - S->pos[3 * i + 2];
    double length = sqrt(dx * dx + dy * dy + dz * dz);
    if (length == 0.0) {
        if (!S->s_degen[s]) {
            S->s_degen[s] = 1;
            (*degen_new)++;
        }
        return 0;
    }
    double factor = act_factor(S->mode[s], S->sim_t, S->amp[s], S->freq[s],
                               S->off[s], S->per[s],
                               S->custom ? S->custom[s] : 1.0);
    double fmag = S->k[s] * (length - factor * S->rest[s]);
    double scale = fmag / length;
    f[0] = scale * dx;
    f[1] = scale * dy;
    f[2] = scale * dz;
    double y = S->yield[s];
    if (y != INFINITY) {
        double area = 0.25 * M_PI * S->diam[s] * S->diam[s];
        double mag = fmag >= 0.0 ? fmag : -fmag;
        if (mag > y * area) {
            S->s_alive[s] = 0;
            (*broken)++;
        }
    }
    return 1;
}

#define SPRING_ARGS                                                         \
    int64_t s_n, uint8_t *s_alive, const int64_t *s_m1, const int64_t *s_m2, \
        const int64_t *s_m1gen, const int64_t *s_m2gen,                      \
        const uint8_t *m_alive, const int64_t *m_gen, const double *pos

#define SPRING_TAIL                                                          \
    const double *rest, const double *k, const double *diam,                 \
        const double *yield, const int8_t *mode, const double *amp,          \
        const double *freq, const double *off, const double *per,            \
        const double *custom, uint8_t *s_degen, double sim_t,                \
        int64_t *counters

#define FILL_SPRINGS(S)                                                      \
    orc_springs S = {s_n,  s_alive, s_m1, s_m2, s_m1gen, s_m2gen, m_alive, \
                     m_gen, pos,    rest, k,    diam, yield,   mode,        \
                     amp,  freq,    off,  per,  custom, s_degen, sim_t}

/* kernels.py:28-86 -- default linearizable serial path: fext += / -= in
 * ascending slot order. */
ORC_API void orc_spring_serial(SPRING_ARGS, double *fext, SPRING_TAIL) {
    FILL_SPRINGS(S);
    int64_t broken = 0, invalid = 0, degen_new = 0;
    for (int64_t s = 0; s < s_n; s++) {
        double f[3];
        if (!spring_eval(&S, s, f, &broken, &invalid, &degen_new)) continue;
        int64_t i = s_m1[s], j = s_m2[s];
        fext[3 * i + 0] += f[0];
        fext[3 * i + 1] += f[1];
        fext[3 * i + 2] += f[2];
        fext[3 * j + 0] -= f[0];
        fext[3 * j + 1] -= f[1];
        fext[3 * j + 2] -= f[2];
    }
    counters[0] += broken;
    counters[1] += invalid;
    counters[2] += degen_new;
}

/* kernels.py:166-232 -- each spring writes +f to slot 2s, -f to slot 2s+1. */
ORC_API void orc_spring_slotted(SPRING_ARGS, double *slot_force, SPRING_TAIL,
                                int nthreads) {
    FILL_SPRINGS(S);
    int64_t broken = 0, invalid = 0, degen_new = 0;
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for num_threads(nthreads) schedule(static) \
    reduction(+ : broken, invalid, degen_new)
#endif
    for (int64_t s = 0; s < s_n; s++) {
        double *a = slot_force + 6 * s, *b = a + 3;
        a[0] = a[1] = a[2] = 0.0;
        b[0] = b[1] = b[2] = 0.0;
        double f[3];
        if (!spring_eval(&S, s, f, &broken, &invalid, &degen_new)) continue;
        a[0] = f[0];
        a[1] = f[1];
        a[2] = f[2];
        b[0] = -f[0];
        b[1] = -f[1];
        b[2] = -f[2];
    }
    (void)nthreads;
    counters[0] += broken;
    counters[1] += invalid;
    counters[2] += degen_new;
}

/* kernels.py:235-247 */
ORC_API void orc_reduce_slots(int64_t m_n, double *fext,
                              const double *slot_force, const int64_t *red_off,
                              const int64_t *red_idx, int nthreads) {
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for num_threads(nthreads) schedule(static)
#endif
    for (int64_t i = 0; i < m_n; i++) {
        double ax = 0.0, ay = 0.0, az = 0.0;
        for (int64_t kk = red_off[i]; kk < red_off[i + 1]; kk++) {
            const double *sf = slot_force + 3 * red_idx[kk];
            ax += sf[0];
            ay += sf[1];
            az += sf[2];
        }
        fext[3 * i + 0] += ax;
        fext[3 * i + 1] += ay;
        fext[3 * i + 2] += az;
    }
    (void)nthreads;
}

/* engine.py:105-118: owner[2s]=m1[s], owner[2s+1]=m2[s]; stable argsort by
 * owner, CSR offsets per mass.  A stable counting sort gives the identical
 * permutation. */
ORC_API void orc_build_slots(int64_t s_n, int64_t m_n, const int64_t *m1,
                             const int64_t *m2, int64_t *red_off,
                             int64_t *red_idx) {
    memset(red_off, 0, sizeof(int64_t) * (size_t)(m_n + 1));
    for (int64_t s = 0; s < s_n; s++) {
        red_off[m1[s] + 1]++;
        red_off[m2[s] + 1]++;
    }
    for (int64_t i = 0; i < m_n; i++) red_off[i + 1] += red_off[i];
    int64_t *cursor = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m_n + 1));
    memcpy(cursor, red_off, sizeof(int64_t) * (size_t)(m_n + 1));
    for (int64_t s = 0; s < s_n; s++) {
        red_idx[cursor[m1[s]]++] = 2 * s;
        red_idx[cursor[m2[s]]++] = 2 * s + 1;
    }
    free(cursor);
}

/* kernels.py:250-376 -- semi-implicit Euler with contacts and constraints.
 * planes [P,7] = (nx,ny,nz,offset,k,mu_s,mu_k); balls [B,5] = (cx,cy,cz,r,k);
 * gc_kind/gc_vec global constraints; lc_off/lc_kind/lc_vec per-mass CSR.
 * err_slot[0] = highest non-finite slot + 1 (the serial loop's last write). */
ORC_API void orc_mass_pass(int64_t m_n, const uint8_t *m_alive,
                           const uint8_t *m_fixed, double *pos, double *vel,
                           double *acc, double *fext, const double *load,
                           const double *m_arr, double gx, double gy,
                           double gz, double drag, const double *planes,
                           int64_t n_planes, const double *balls,
                           int64_t n_balls, const int8_t *gc_kind,
                           const double *gc_vec, int64_t n_gc,
                           const int64_t *lc_off, const int8_t *lc_kind,
                           const double *lc_vec, double dt, double v_stick,
                           int64_t *err_slot, int nthreads) {
    int64_t err = err_slot[0];
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for num_threads(nthreads) schedule(static) \
    reduction(max : err)
#endif
    for (int64_t i = 0; i < m_n; i++) {
        if (!m_alive[i]) continue;
        double *P = pos + 3 * i, *V = vel + 3 * i, *A = acc + 3 * i,
               *F = fext + 3 * i;
        if (m_fixed[i]) {
            V[0] = V[1] = V[2] = 0.0;
            A[0] = A[1] = A[2] = 0.0;
            F[0] = F[1] = F[2] = 0.0;
            continue;
        }
        double mm = m_arr[i];
        double px = P[0], py = P[1], pz = P[2];
        double vx = V[0], vy = V[1], vz = V[2];
        double fx = F[0] + load[3 * i + 0] + mm * gx - drag * vx;
        double fy = F[1] + load[3 * i + 1] + mm * gy - drag * vy;
        double fz = F[2] + load[3 * i + 2] + mm * gz - drag * vz;
        for (int64_t p = 0; p < n_planes; p++) {
            const double *pl = planes + 7 * p;
            double nx = pl[0], ny = pl[1], nz = pl[2];
            double depth = pl[3] - (px * nx + py * ny + pz * nz);
            if (depth > 0.0) {
                double nmag = pl[4] * depth;
                fx += nmag * nx;
                fy += nmag * ny;
                fz += nmag * nz;
                double vn = vx * nx + vy * ny + vz * nz;
                double tvx = vx - vn * nx, tvy = vy - vn * ny,
                       tvz = vz - vn * nz;
                double tv = sqrt(tvx * tvx + tvy * tvy + tvz * tvz);
                double fn = fx * nx + fy * ny + fz * nz;
                double tfx = fx - fn * nx, tfy = fy - fn * ny,
                       tfz = fz - fn * nz;
                double tf = sqrt(tfx * tfx + tfy * tfy + tfz * tfz);
                if (tv < v_stick && tf <= pl[5] * nmag) {
                    fx -= tfx;
                    fy -= tfy;
                    fz -= tfz;
                } else if (tv >= v_stick) {
                    double sc = pl[6] * nmag / tv;
                    fx -= sc * tvx;
                    fy -= sc * tvy;
                    fz -= sc * tvz;
                } else if (tf > 0.0) {
                    double sc = pl[6] * nmag / tf;
                    fx -= sc * tfx;
                    fy -= sc * tfy;
                    fz -= sc * tfz;
                }
            }
        }
        for (int64_t b = 0; b < n_balls; b++) {
            const double *bl = balls + 5 * b;
            double ddx = px - bl[0], ddy = py - bl[1], ddz = pz - bl[2];
            double dist = sqrt(ddx * ddx + ddy * ddy + ddz * ddz);
            double depth = bl[3] - dist;
            if (depth > 0.0 && dist > 0.0) {
                double sc = bl[4] * depth / dist;
                fx += sc * ddx;
                fy += sc * ddy;
                fz += sc * ddz;
            }
        }
        double ax = fx / mm, ay = fy / mm, az = fz / mm;
        vx += ax * dt;
        vy += ay * dt;
        vz += az * dt;
        for (int64_t g = 0; g < n_gc; g++) {
            double cx = gc_vec[3 * g], cy = gc_vec[3 * g + 1],
                   cz = gc_vec[3 * g + 2];
            double vdot = vx * cx + vy * cy + vz * cz;
            if (gc_kind[g] == 1) {
                vx = vdot * cx;
                vy = vdot * cy;
                vz = vdot * cz;
            } else {
                vx -= vdot * cx;
                vy -= vdot * cy;
                vz -= vdot * cz;
            }
        }
        for (int64_t kk = lc_off[i]; kk < lc_off[i + 1]; kk++) {
            double cx = lc_vec[3 * kk], cy = lc_vec[3 * kk + 1],
                   cz = lc_vec[3 * kk + 2];
            double vdot = vx * cx + vy * cy + vz * cz;
            if (lc_kind[kk] == 1) {
                vx = vdot * cx;
                vy = vdot * cy;
                vz = vdot * cz;
            } else {
                vx -= vdot * cx;
                vy -= vdot * cy;
                vz -= vdot * cz;
            }
        }
        px += vx * dt;
        py += vy * dt;
        pz += vz * dt;
        P[0] = px;
        P[1] = py;
        P[2] = pz;
        V[0] = vx;
        V[1] = vy;
        V[2] = vz;
        A[0] = ax;
        A[1] = ay;
        A[2] = az;
        F[0] = F[1] = F[2] = 0.0;
        if (!(isfinite(px) && isfinite(py) && isfinite(pz) && isfinite(vx) &&
              isfinite(vy) && isfinite(vz))) {
            if (i + 1 > err) err = i + 1;
        }
    }
    (void)nthreads;
    err_slot[0] = err;
}

ORC_API int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
