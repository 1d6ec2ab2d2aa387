// sa_host.cpp -- host-side writers of the reference CLI's CSV outputs for
// CPI-scale maps (cli.py:74-116 _write_csv, cli.py:184-191 the
// ambiguity surface rows).  The reference formats every float with Python's
// repr() through csv.writer, one Python call per row: ~10 s for a 4096 x 2048
// map.  Here the rows are formatted in parallel host threads with the shortest
// round-trip digits (std::to_chars) laid out exactly as repr() does, so the file
// is byte-identical to the reference's.
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/signadd_b200.h"

namespace {

// Python float repr (float_repr_style 'short'): shortest round-trip digits
// d1..dn with x = 0.d1..dn x 10^decpt; exponential iff decpt > 16 or decpt < -3.
int py_repr(double x, char *out) {
  char *p = out;
  if (std::isnan(x)) return (int)(std::memcpy(out, "nan", 3), 3);
  if (std::isinf(x)) {
    if (x < 0) *p++ = '-';
    std::memcpy(p, "inf", 3);
    return (int)(p - out) + 3;
  }
  if (std::signbit(x)) *p++ = '-', x = -x;
  if (x == 0.0) return (int)(std::memcpy(p, "0.0", 3), p - out + 3);
  char sci[64];
  auto r = std::to_chars(sci, sci + sizeof(sci), x, std::chars_format::scientific);
  char *end = r.ptr;
  *end = 0;
  // sci = "d[.ddd]e[+-]XX"
  char digits[32] = {};
  int nd = 0;
  char *q = sci;
  for (; q < end && *q != 'e'; ++q)
    if (*q != '.') digits[nd++] = *q;
  const int e10 = std::atoi(q + 1);  // x = d1.d2.. x 10^e10
  const int decpt = e10 + 1;
  if (decpt > 16 || decpt < -3) {
    *p++ = digits[0];
    if (nd > 1) {
      *p++ = '.';
      std::memcpy(p, digits + 1, nd - 1);
      p += nd - 1;
    }
    *p++ = 'e';
    int ee = e10;
    *p++ = ee < 0 ? '-' : '+';
    if (ee < 0) ee = -ee;
    char eb[8];
    int ne = 0;
    do eb[ne++] = (char)('0' + ee % 10), ee /= 10;
    while (ee);
    if (ne < 2) eb[ne++] = '0';
    while (ne) *p++ = eb[--ne];
  } else if (decpt <= 0) {
    *p++ = '0';
    *p++ = '.';
    for (int i = 0; i < -decpt; ++i) *p++ = '0';
    std::memcpy(p, digits, nd);
    p += nd;
  } else if (decpt >= nd) {
    std::memcpy(p, digits, nd);
    p += nd;
    for (int i = nd; i < decpt; ++i) *p++ = '0';
    *p++ = '.';
    *p++ = '0';
  } else {
    std::memcpy(p, digits, decpt);
    p += decpt;
    *p++ = '.';
    std::memcpy(p, digits + decpt, nd - decpt);
    p += nd - decpt;
  }
  return (int)(p - out);
}

int put_int(int64_t v, char *out) {
  auto r = std::to_chars(out, out + 24, v);
  return (int)(r.ptr - out);
}

}  // namespace

extern "C" int sa_format_float_repr(double x, char *out, int cap) {
  if (!out || cap < 32) return SA_ERR_ARG;
  const int n = py_repr(x, out);
  out[n] = 0;
  return n;
}

// "# manifest=<name>\nl,p,magnitude_db\n" + one "l,p,repr(db[l][p])" row per cell,
// row-major, '\n' line ends -- cli.py:184-191 through _write_csv (cli.py:83-90).
extern "C" int sa_format_surface_csv(const double *db, int64_t rows, int64_t cols, const char *manifest,
                                     char **out, int64_t *out_len, int nthreads) {
  if (!db || !out || !out_len || !manifest || rows < 0 || cols < 0) return SA_ERR_ARG;
  const int64_t cells = rows * cols;
  int nt = nthreads > 0 ? nthreads : (int)std::thread::hardware_concurrency();
  if (nt < 1) nt = 1;
  if (cells < 65536) nt = 1;
  std::vector<std::string> parts(nt);
  auto work = [&](int t) {
    const int64_t c0 = cells * t / nt, c1 = cells * (t + 1) / nt;
    std::string &s = parts[t];
    s.resize((size_t)(c1 - c0) * 48);
    char *p = s.data();
    for (int64_t c = c0; c < c1; ++c) {
      p += put_int(c / cols, p);
      *p++ = ',';
      p += put_int(c % cols, p);
      *p++ = ',';
      p += py_repr(db[c], p);
      *p++ = '\n';
    }
    s.resize((size_t)(p - s.data()));
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
  work(0);
  for (auto &x : th) x.join();
  std::string head = std::string("# manifest=") + manifest + "\nl,p,magnitude_db\n";
  size_t total = head.size();
  for (auto &s : parts) total += s.size();
  char *buf = (char *)std::malloc(total + 1);
  if (!buf) return SA_ERR_ARG;
  char *p = buf;
  std::memcpy(p, head.data(), head.size());
  p += head.size();
  for (auto &s : parts) {
    std::memcpy(p, s.data(), s.size());
    p += s.size();
  }
  *p = 0;
  *out = buf;
  *out_len = (int64_t)total;
  return SA_OK;
}

extern "C" void sa_free_host(void *p) { std::free(p); }
