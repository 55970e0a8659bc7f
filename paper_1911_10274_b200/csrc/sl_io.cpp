// sl_io.cpp -- host-side snapshot formatting.
//
// The reference writes snapshots as CSV, header "id,x,y,z,vx,vy,vz", one
// row per alive mass, every double printed with Python's "{:.17g}" so it
// round-trips bit-exactly (io.py:19-32).  The Python loop costs ~2 us per
// row; this formats rows with the C library's correctly rounded "%.17g"
// (the same digits) on several threads.  Non-finite values follow Python:
// "inf", "-inf", "nan" (never "-nan").
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
