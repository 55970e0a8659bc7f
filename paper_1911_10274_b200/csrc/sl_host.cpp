// sl_io.cpp -- host-side snapshot formatting.
//
// The reference writes snapshots as CSV, header "id,x,y,z,vx,vy,vz", one
// row per alive mass, every double printed with Python's "{:.17g}" so it
// round-trips bit-exactly (io.py:19-32).  The Python loop costs ~2 us per
// row; this formats rows with the C library's correctly rounded "%.17g"
// (the same digits) on several threads.  Non-finite values follow Python:
// "inf", "-inf", "nan" (never "-nan").
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "softlat_cuda.h"

namespace {

constexpr const char kHeader[] = "id,x,y,z,vx,vy,vz\n";

inline int put_double(char *p, double v) {
  if (std::isnan(v)) {
    std::memcpy(p, "nan", 3);
    return 3;
  }
  if (std::isinf(v)) {
    if (v < 0) {
      std::memcpy(p, "-inf", 4);
      return 4;
    }
    std::memcpy(p, "inf", 3);
    return 3;
  }
  return std::snprintf(p, SL_SNAPSHOT_ROW_MAX, "%.17g", v);
}

// one row into p (room for SL_SNAPSHOT_ROW_MAX bytes); returns its length
inline size_t put_row(char *p, int64_t id, const double *x, const double *v) {
  char *q = p;
  q += std::snprintf(q, 24, "%lld", (long long)id);
  for (int c = 0; c < 3; c++) {
    *q++ = ',';
    q += put_double(q, x[c]);
  }
  for (int c = 0; c < 3; c++) {
    *q++ = ',';
    q += put_double(q, v[c]);
  }
  *q++ = '\n';
  return (size_t)(q - p);
}

}  // namespace

extern "C" int sl_format_snapshot(int64_t n, const int64_t *ids,
                                  const double *pos, const double *vel,
                                  int threads, char *out, size_t cap,
                                  size_t *len) {
  if (n < 0 || !out || !len || (n > 0 && (!ids || !pos || !vel)))
    return SL_EINVAL;
  const size_t hdr = sizeof(kHeader) - 1;
  if (cap < hdr + (size_t)n * SL_SNAPSHOT_ROW_MAX) return SL_EINVAL;
  std::memcpy(out, kHeader, hdr);
  if (threads < 1) threads = 1;
  const int64_t min_rows = 4096;  // per thread
  int64_t nt = (n + min_rows - 1) / min_rows;
  if (nt > threads) nt = threads;
  if (nt < 1) nt = 1;
  // each chunk formats into its own region of `out` (sized for the worst
  // case), then the chunks are packed in order
  std::vector<size_t> used((size_t)nt, 0);
  std::vector<int64_t> lo((size_t)nt + 1);
  for (int64_t t = 0; t <= nt; t++) lo[(size_t)t] = n * t / nt;
  auto work = [&](int64_t t) {
    char *p = out + hdr + (size_t)lo[(size_t)t] * SL_SNAPSHOT_ROW_MAX;
    size_t u = 0;
    for (int64_t i = lo[(size_t)t]; i < lo[(size_t)t + 1]; i++)
      u += put_row(p + u, ids[i], pos + 3 * i, vel + 3 * i);
    used[(size_t)t] = u;
  };
  if (nt == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int64_t t = 0; t < nt; t++) pool.emplace_back(work, t);
    for (auto &th : pool) th.join();
  }
  size_t at = hdr;
  for (int64_t t = 0; t < nt; t++) {
    const char *src = out + hdr + (size_t)lo[(size_t)t] * SL_SNAPSHOT_ROW_MAX;
    if (src != out + at) std::memmove(out + at, src, used[(size_t)t]);
    at += used[(size_t)t];
  }
  *len = at;
  return SL_OK;
}

// ---------------------------------------------------------------------------
// Parallel fill: first touch of fresh store capacity on several threads (the
// page faults dominate np.full at store sizes: ~1 GB/s on one thread).
namespace {
template <class Fn>
void parallel_for(int64_t n, int threads, int64_t grain, Fn fn) {
  if (threads < 1) threads = 1;
  int64_t nt = (n + grain - 1) / grain;
  if (nt > threads) nt = threads;
  if (nt <= 1) {
    if (n > 0) fn((int64_t)0, n);
    return;
  }
  std::vector<std::thread> pool;
  for (int64_t t = 0; t < nt; t++)
    pool.emplace_back(fn, n * t / nt, n * (t + 1) / nt);
  for (auto &th : pool) th.join();
}
}  // namespace

extern "C" int sl_host_fill(void *dst, const void *value, size_t elem_bytes,
                            int64_t count, int threads) {
  if (count < 0 || (count > 0 && (!dst || !value)) || elem_bytes == 0 ||
      elem_bytes > 64)
    return SL_EINVAL;
  unsigned char *d = (unsigned char *)dst;
  unsigned char pat[64];
  std::memcpy(pat, value, elem_bytes);
  bool uniform = true;
  for (size_t i = 1; i < elem_bytes; i++) uniform &= pat[i] == pat[0];
  parallel_for(count, threads, (int64_t)(1 << 20) / (int64_t)elem_bytes + 1,
               [&](int64_t lo, int64_t hi) {
                 unsigned char *p = d + (size_t)lo * elem_bytes;
                 if (uniform) {
                   std::memset(p, pat[0], (size_t)(hi - lo) * elem_bytes);
                   return;
                 }
                 for (int64_t i = lo; i < hi; i++, p += elem_bytes)
                   std::memcpy(p, pat, elem_bytes);
               });
  return SL_OK;
}

// ---------------------------------------------------------------------------
// Lattice generation (builder.py:112-186 as restated by builder.py here):
// row-major node ids (i*ny + j)*nz + k, positions corner + spacing*index,
// springs grouped by the 13 cell offsets in the reference order, each group
// row-major over its lower node; rest = sqrt((dx*dx + dy*dy) + dz*dz) of the
// build-time positions, k = (E*area)/rest, node mass = the half-bar masses
// ((0.5*rho)*area)*rest added in numpy's np.add.at order (all a-side
// contributions in spring order, then all b-side ones).  Every operation is
// the numpy expression's, rounded the same way (this unit: no contraction).
namespace {
const int kOff[13][3] = {{1, 0, 0},  {0, 1, 0},  {0, 0, 1},   {1, 1, 0},
                         {1, -1, 0}, {1, 0, 1},  {1, 0, -1},  {0, 1, 1},
                         {0, 1, -1}, {1, 1, 1},  {1, 1, -1},  {1, -1, 1},
                         {1, -1, -1}};
struct Grid {
  int64_t n[3];
  int64_t lo[13][3], hi[13][3], start[14];
};
Grid make_grid(int64_t nx, int64_t ny, int64_t nz) {
  Grid g;
  g.n[0] = nx;
  g.n[1] = ny;
  g.n[2] = nz;
  g.start[0] = 0;
  for (int o = 0; o < 13; o++) {
    int64_t cnt = 1;
    for (int c = 0; c < 3; c++) {
      g.lo[o][c] = kOff[o][c] < 0 ? -kOff[o][c] : 0;
      g.hi[o][c] = g.n[c] - (kOff[o][c] > 0 ? kOff[o][c] : 0);
      const int64_t e = g.hi[o][c] - g.lo[o][c];
      cnt *= e > 0 ? e : 0;
    }
    g.start[o + 1] = g.start[o] + cnt;
  }
  return g;
}
}  // namespace

extern "C" int sl_lattice_counts(int64_t nx, int64_t ny, int64_t nz,
                                 int64_t *n_masses, int64_t *n_springs) {
  if (nx < 1 || ny < 1 || nz < 1 || !n_masses || !n_springs) return SL_EINVAL;
  const Grid g = make_grid(nx, ny, nz);
  *n_masses = nx * ny * nz;
  *n_springs = g.start[13];
  return SL_OK;
}

extern "C" int sl_build_lattice(int64_t nx, int64_t ny, int64_t nz,
                                const double *corner, double spacing,
                                double elastic_modulus, double density,
                                double diameter, int threads, double *pos,
                                double *node_mass, int64_t *a, int64_t *b,
                                double *rest, double *stiff) {
  if (nx < 1 || ny < 1 || nz < 1 || !corner || !pos || !node_mass)
    return SL_EINVAL;
  const Grid g = make_grid(nx, ny, nz);
  const int64_t nm = nx * ny * nz, ns = g.start[13];
  if (ns > 0 && (!a || !b || !rest || !stiff)) return SL_EINVAL;
  const double half_d = diameter * 0.5;
  const double area = 3.141592653589793 * (half_d * half_d);
  const double ka = elastic_modulus * area;
  const double half_rho_area = (0.5 * density) * area;
  auto p_of = [&](int64_t i, int64_t j, int64_t k, double *out) {
    out[0] = corner[0] + spacing * (double)i;
    out[1] = corner[1] + spacing * (double)j;
    out[2] = corner[2] + spacing * (double)k;
  };
  auto rest_of = [&](int64_t i, int64_t j, int64_t k, int o) {
    double pa[3], pb[3];
    p_of(i, j, k, pa);
    p_of(i + kOff[o][0], j + kOff[o][1], k + kOff[o][2], pb);
    const double dx = pb[0] - pa[0], dy = pb[1] - pa[1], dz = pb[2] - pa[2];
    return std::sqrt(dx * dx + dy * dy + dz * dz);
  };
  // masses: positions and accumulated half-bar masses, node-parallel
  parallel_for(nm, threads, 1 << 14, [&](int64_t lo, int64_t hi) {
    for (int64_t id = lo; id < hi; id++) {
      const int64_t i = id / (ny * nz), j = (id / nz) % ny, k = id % nz;
      p_of(i, j, k, pos + 3 * id);
      double m = 0.0;
      for (int side = 0; side < 2; side++) {  // a-side first, then b-side
        for (int o = 0; o < 13; o++) {
          // the spring's lower node: this node (a) or this node - offset (b)
          const int64_t li = side ? i - kOff[o][0] : i;
          const int64_t lj = side ? j - kOff[o][1] : j;
          const int64_t lk = side ? k - kOff[o][2] : k;
          if (li < g.lo[o][0] || li >= g.hi[o][0] || lj < g.lo[o][1] ||
              lj >= g.hi[o][1] || lk < g.lo[o][2] || lk >= g.hi[o][2])
            continue;
          m += half_rho_area * rest_of(li, lj, lk, o);
        }
      }
      node_mass[id] = m;
    }
  });
  // springs, spring-parallel within each offset group
  for (int o = 0; o < 13; o++) {
    const int64_t e0 = g.hi[o][0] - g.lo[o][0], e1 = g.hi[o][1] - g.lo[o][1],
                  e2 = g.hi[o][2] - g.lo[o][2];
    const int64_t cnt = g.start[o + 1] - g.start[o];
    if (cnt <= 0) continue;
    const int64_t base = g.start[o];
    parallel_for(cnt, threads, 1 << 15, [&](int64_t lo, int64_t hi) {
      for (int64_t q = lo; q < hi; q++) {
        const int64_t i = g.lo[o][0] + q / (e1 * e2);
        const int64_t j = g.lo[o][1] + (q / e2) % e1;
        const int64_t k = g.lo[o][2] + q % e2;
        const int64_t s = base + q;
        a[s] = (i * ny + j) * nz + k;
        b[s] = ((i + kOff[o][0]) * ny + (j + kOff[o][1])) * nz +
               (k + kOff[o][2]);
        const double r = rest_of(i, j, k, o);
        rest[s] = r;
        stiff[s] = ka / r;
      }
    });
    (void)e0;
  }
  return SL_OK;
}

// Copy on several threads (fresh destination pages fault in parallel):
// snapshot copies of the store's mass columns (control.snapshot).
extern "C" int sl_host_copy(void *dst, const void *src, size_t bytes,
                            int threads) {
  if (bytes && (!dst || !src)) return SL_EINVAL;
  unsigned char *d = (unsigned char *)dst;
  const unsigned char *s = (const unsigned char *)src;
  parallel_for((int64_t)bytes, threads, (int64_t)1 << 20,
               [&](int64_t lo, int64_t hi) {
                 std::memcpy(d + lo, s + lo, (size_t)(hi - lo));
               });
  return SL_OK;
}

// *out = 1 when ids[i] == i for all i < n (a snapshot of every slot in
// order: io.apply_snapshot then copies whole columns), else 0.
extern "C" int sl_host_is_iota(const int64_t *ids, int64_t n, int threads,
                               int *out) {
  if (n < 0 || !out || (n > 0 && !ids)) return SL_EINVAL;
  std::atomic<int> bad{0};
  parallel_for(n, threads, (int64_t)1 << 20, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; i++)
      if (ids[i] != i) {
        bad.store(1, std::memory_order_relaxed);
        return;
      }
  });
  *out = bad.load() ? 0 : 1;
  return SL_OK;
}

// min and max of v[i] over mask[i] != 0 (mask NULL: all), NaN-propagating
// like numpy's masked np.min / np.max; empty selection: +inf / -inf.
// check_stability's k_max / m_min over 12.7 M springs (engine.py:274-296).
extern "C" int sl_host_masked_extrema(const double *v, const uint8_t *mask,
                                      int64_t n, int threads, double *out_min,
                                      double *out_max) {
  if (n < 0 || !out_min || !out_max || (n > 0 && !v)) return SL_EINVAL;
  int64_t nt = threads < 1 ? 1 : threads;
  if (nt > n / (1 << 16) + 1) nt = n / (1 << 16) + 1;
  std::vector<double> mn((size_t)nt), mx((size_t)nt);
  std::vector<int> nan((size_t)nt);
  auto chunk = [&](int64_t t) {
    double a = INFINITY, b = -INFINITY;
    int bad = 0;
    for (int64_t i = n * t / nt; i < n * (t + 1) / nt; i++) {
      if (mask && !mask[i]) continue;
      const double x = v[i];
      bad |= x != x;
      a = x < a ? x : a;
      b = x > b ? x : b;
    }
    mn[(size_t)t] = a;
    mx[(size_t)t] = b;
    nan[(size_t)t] = bad;
  };
  if (nt == 1) {
    chunk(0);
  } else {
    std::vector<std::thread> pool;
    for (int64_t t = 0; t < nt; t++) pool.emplace_back(chunk, t);
    for (auto &th : pool) th.join();
  }
  double a = INFINITY, b = -INFINITY;
  int bad = 0;
  for (int64_t t = 0; t < nt; t++) {
    a = mn[(size_t)t] < a ? mn[(size_t)t] : a;
    b = mx[(size_t)t] > b ? mx[(size_t)t] : b;
    bad |= nan[(size_t)t];
  }
  *out_min = bad ? NAN : a;
  *out_max = bad ? NAN : b;
  return SL_OK;
}
