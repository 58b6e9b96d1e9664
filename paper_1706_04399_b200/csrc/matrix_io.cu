// Plain-text cost-matrix files (graph.py:123-143: save_cost_matrix /
// load_cost_matrix), host code behind the C ABI.
//
// Format: a header line "n", then n lines of n numbers, each written as
// Python's repr(float(x)) and separated by single spaces.  The writer
// reproduces repr byte for byte (shortest round-trip digits, fixed notation
// for decimal exponents -4 < e <= 16, else "d.ddde+XX"), so a matrix written
// here is the reference's file.  The reader splits on whitespace and parses
// every token like Python's int() / float() (signs, inf/nan, digit-group
// underscores), with the reference's error messages, straight into the
// caller's (pinned) row-major buffer.
#include <errno.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include <charconv>
#include <cmath>
#include <algorithm>
#include <string>
#include <mutex>
#include <thread>
#include <vector>

#include "dpso_internal.cuh"

namespace {

int fail(int code, const char* msg) { return dpso::api_fail(code, msg); }

// repr(float(x)) (Objects/floatobject.c float_repr -> 'r' format with
// Py_DTSF_ADD_DOT_0)
size_t py_repr(double x, char* out) {
  char* p = out;
  if (std::isnan(x)) {
    memcpy(p, "nan", 3);
    return 3;
  }
  if (std::signbit(x)) *p++ = '-';
  const double a = std::fabs(x);
  if (std::isinf(a)) {
    memcpy(p, "inf", 3);
    return (size_t)(p - out) + 3;
  }
  if (a == 0.0) {
    memcpy(p, "0.0", 3);
    return (size_t)(p - out) + 3;
  }
  char sci[40];
  auto r = std::to_chars(sci, sci + sizeof sci - 1, a,
                         std::chars_format::scientific);
  // sci = d[.ddd]e(+|-)XX
  char digits[32];
  int k = 0;
  const char* q = sci;
  while (*q != 'e' && q < r.ptr) {
    if (*q != '.') digits[k++] = *q;
    ++q;
  }
  *r.ptr = 0;
  const int e10 = atoi(q + 1);
  const int decpt = e10 + 1;  // value = 0.d1d2... x 10^decpt
  if (decpt <= -4 || decpt > 16) {
    *p++ = digits[0];
    if (k > 1) {
      *p++ = '.';
      memcpy(p, digits + 1, k - 1);
      p += k - 1;
    }
    const int ex = decpt - 1;
    p += sprintf(p, "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
  } else if (decpt <= 0) {
    *p++ = '0';
    *p++ = '.';
    for (int i = 0; i < -decpt; ++i) *p++ = '0';
    memcpy(p, digits, k);
    p += k;
  } else if (decpt < k) {
    memcpy(p, digits, decpt);
    p += decpt;
    *p++ = '.';
    memcpy(p, digits + decpt, k - decpt);
    p += k - decpt;
  } else {
    memcpy(p, digits, k);
    p += k;
    for (int i = k; i < decpt; ++i) *p++ = '0';
    *p++ = '.';
    *p++ = '0';
  }
  return (size_t)(p - out);
}

bool is_space(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\f' ||
         c == '\v' || c == '\x1c' || c == '\x1d' || c == '\x1e' ||
         c == '\x1f';
}

// Python's digit-group underscores: single '_' between two digits
bool strip_underscores(const char* b, const char* e, std::string* out) {
  out->clear();
  for (const char* c = b; c < e; ++c) {
    if (*c == '_') {
      if (c == b || c + 1 == e || !isdigit((unsigned char)c[-1]) ||
          !isdigit((unsigned char)c[1]))
        return false;
      continue;
    }
    out->push_back(*c);
  }
  return true;
}

bool ieq(const char* b, const char* e, const char* lit) {
  const size_t n = strlen(lit);
  if ((size_t)(e - b) != n) return false;
  for (size_t i = 0; i < n; ++i)
    if (tolower((unsigned char)b[i]) != lit[i]) return false;
  return true;
}

// float(token) for a whitespace-free token
bool py_float(const char* b, const char* e, double* v) {
  std::string tmp;
  if (memchr(b, '_', e - b)) {
    if (!strip_underscores(b, e, &tmp)) return false;
    b = tmp.data();
    e = b + tmp.size();
  }
  bool neg = false;
  const char* s = b;
  if (s < e && (*s == '+' || *s == '-')) {
    neg = *s == '-';
    ++s;
  }
  if (s == e) return false;
  if (ieq(s, e, "inf") || ieq(s, e, "infinity")) {
    *v = neg ? -HUGE_VAL : HUGE_VAL;
    return true;
  }
  if (ieq(s, e, "nan")) {
    *v = neg ? -NAN : NAN;
    return true;
  }
  if (!(isdigit((unsigned char)*s) || *s == '.')) return false;
  double x = 0.0;
  auto r = std::from_chars(s, e, x, std::chars_format::general);
  if (r.ptr != e) return false;
  if (r.ec == std::errc::result_out_of_range) {
    // Python rounds out-of-range literals to inf or 0 like strtod
    std::string t(s, e);
    x = strtod(t.c_str(), nullptr);
  } else if (r.ec != std::errc()) {
    return false;
  }
  *v = neg ? -x : x;
  return true;
}

// int(token, 10)
bool py_int(const char* b, const char* e, long long* v) {
  std::string tmp;
  if (memchr(b, '_', e - b)) {
    if (!strip_underscores(b, e, &tmp)) return false;
    b = tmp.data();
    e = b + tmp.size();
  }
  bool neg = false;
  if (b < e && (*b == '+' || *b == '-')) {
    neg = *b == '-';
    ++b;
  }
  if (b == e) return false;
  long long x = 0;
  for (const char* c = b; c < e; ++c) {
    if (!isdigit((unsigned char)*c)) return false;
    x = x * 10 + (*c - '0');
    if (x > (1ll << 40)) return false;
  }
  *v = neg ? -x : x;
  return true;
}

// the whole file (or its first `limit` bytes) in one read
bool read_file(const char* path, std::string* buf, size_t limit = SIZE_MAX) {
  FILE* f = fopen(path, "rb");
  if (!f) return false;
  size_t size = 0;
  if (fseek(f, 0, SEEK_END) == 0) {
    const long e = ftell(f);
    if (e > 0) size = (size_t)e;
    fseek(f, 0, SEEK_SET);
  }
  if (size > limit) size = limit;
  buf->resize(size);
  size_t got = size ? fread(&(*buf)[0], 1, size, f) : 0;
  buf->resize(got);
  if (got == size && size < limit) {  // not seekable / grew: read the rest
    char chunk[1 << 16];
    size_t k;
    while (buf->size() < limit &&
           (k = fread(chunk, 1, sizeof chunk, f)) > 0)
      buf->append(chunk, k);
  }
  fclose(f);
  return true;
}

int bad_token(const char* kind, const char* b, const char* e) {
  std::string msg = kind;
  msg += " '";
  msg.append(b, e);
  msg += "'";
  return fail(DPSO_EINVAL, msg.c_str());
}

}  // namespace

extern "C" {

int dpso_write_matrix_text(const char* path, const double* host, int64_t ld,
                           int32_t n) {
  if (!path || (n > 0 && !host) || n < 0 || ld < n)
    return fail(DPSO_EINVAL, "bad arguments");
  FILE* f = fopen(path, "wb");
  if (!f) return fail(DPSO_EINVAL, (std::string("cannot open ") + path).c_str());
  std::string line;
  line.reserve((size_t)n * 24 + 2);
  fprintf(f, "%d\n", n);
  char tok[48];
  for (int32_t r = 0; r < n; ++r) {
    line.clear();
    for (int32_t c = 0; c < n; ++c) {
      if (c) line.push_back(' ');
      line.append(tok, py_repr(host[(size_t)r * ld + c], tok));
    }
    line.push_back('\n');
    if (fwrite(line.data(), 1, line.size(), f) != line.size()) {
      fclose(f);
      return fail(DPSO_EINVAL, "write failed");
    }
  }
  if (fclose(f) != 0) return fail(DPSO_EINVAL, "write failed");
  return DPSO_OK;
}

int dpso_read_matrix_text(const char* path, double* out, int64_t ld,
                          int32_t cap_n, int32_t* n_out) {
  if (!path || !n_out) return fail(DPSO_EINVAL, "bad arguments");
  std::string buf;
  // header only: the first token (a dimension) is within the first 4 KiB
  // unless the file starts with a long run of whitespace
  if (!read_file(path, &buf, out ? SIZE_MAX : 4096))
    return fail(DPSO_EINVAL, (std::string("cannot open ") + path).c_str());
  if (!out) {
    size_t i = 0;
    while (i < buf.size() && is_space(buf[i])) ++i;
    size_t j = i;
    while (j < buf.size() && !is_space(buf[j])) ++j;
    if (j == buf.size() && buf.size() == 4096 &&
        !read_file(path, &buf))  // token not complete in 4 KiB
      return fail(DPSO_EINVAL, (std::string("cannot open ") + path).c_str());
  }
  const char* p = buf.data();
  const char* end = p + buf.size();
  auto next_token = [&](const char** b, const char** e) -> bool {
    while (p < end && is_space(*p)) ++p;
    if (p == end) return false;
    *b = p;
    while (p < end && !is_space(*p)) ++p;
    *e = p;
    return true;
  };
  const char *tb, *te;
  if (!next_token(&tb, &te)) {
    std::string m = std::string("empty cost matrix file ") + path;
    return fail(DPSO_EINVAL, m.c_str());
  }
  long long n = 0;
  if (!py_int(tb, te, &n))
    return bad_token("invalid literal for int() with base 10:", tb, te);
  if (n < 0 || n > 2000000000ll / (n > 0 ? n : 1))
    return fail(DPSO_EINVAL, "matrix dimension out of range");
  *n_out = (int32_t)n;
  if (!out) return DPSO_OK;  // header only: the caller sizes the buffer
  if (n > cap_n || ld < n) return fail(DPSO_EINVAL, "output buffer too small");
  const long long want = n * n;
  // Parallel parse: chunks cut at whitespace; pass 1 counts each chunk's
  // tokens, pass 2 parses them into their global positions.  The first bad
  // token in file order is reported, as Python's list comprehension would.
  const size_t body = (size_t)(p - buf.data());
  const size_t len = buf.size() - body;
  long hw = sysconf(_SC_NPROCESSORS_ONLN);
  int nt = (int)std::max(1L, std::min(hw > 0 ? hw : 1L, 32L));
  if (len < (1u << 20)) nt = 1;
  if (const char* e = getenv("DPSO_IO_THREADS")) nt = std::max(1, atoi(e));
  std::vector<size_t> cut(nt + 1);
  cut[0] = body;
  cut[nt] = buf.size();
  for (int t = 1; t < nt; ++t) {
    size_t c = std::max(cut[t - 1], body + len * t / nt);
    while (c < buf.size() && !is_space(buf[c])) ++c;
    cut[t] = c;
  }
  std::vector<long long> cnt(nt, 0), bad_at(nt, -1);
  std::vector<const char*> bad_b(nt, nullptr), bad_e(nt, nullptr);
  auto scan = [&](int t, bool parse, long long base) {
    const char* q = buf.data() + cut[t];
    const char* qe = buf.data() + cut[t + 1];
    long long k = 0;
    while (true) {
      while (q < qe && is_space(*q)) ++q;
      if (q == qe) break;
      const char* b = q;
      while (q < qe && !is_space(*q)) ++q;
      if (parse) {
        double v;
        if (!py_float(b, q, &v)) {
          bad_at[t] = k;
          bad_b[t] = b;
          bad_e[t] = q;
          return;
        }
        const long long g = base + k;
        if (g < want) out[(size_t)(g / n) * ld + (size_t)(g % n)] = v;
      }
      ++k;
    }
    if (!parse) cnt[t] = k;
  };
  auto run = [&](bool parse, const std::vector<long long>& base) {
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) th.emplace_back(scan, t, parse, base[t]);
    scan(0, parse, base[0]);
    for (auto& x : th) x.join();
  };
  std::vector<long long> base(nt, 0);
  run(false, base);
  long long got = 0;
  for (int t = 0; t < nt; ++t) {
    base[t] = got;
    got += cnt[t];
  }
  run(true, base);
  for (int t = 0; t < nt; ++t)
    if (bad_at[t] >= 0)
      return bad_token("could not convert string to float:", bad_b[t],
                       bad_e[t]);
  if (got != want) {
    char m[512];
    snprintf(m, sizeof m, "cost matrix %s: expected %lld entries, got %lld",
             path, want, got);
    return fail(DPSO_EINVAL, m);
  }
  return DPSO_OK;
}

// Python repr of one double (testing the writer without a file)
int dpso_py_repr(double x, char* out, int32_t cap) {
  char tok[48];
  const size_t k = py_repr(x, tok);
  if (!out || (size_t)cap < k + 1) return fail(DPSO_EINVAL, "buffer too small");
  memcpy(out, tok, k);
  out[k] = 0;
  return DPSO_OK;
}

}  // extern "C"

// ---- host -> device matrix upload ------------------------------------------
// A pageable cudaMemcpy stages through the driver's own small pinned buffers
// on one thread (~11 GB/s measured for the 800 MB C5 matrix).  Here: a ring
// of two pinned chunks, each filled by several host threads (memcpy of row
// slices) while the other chunk's DMA runs on the caller's stream.
namespace {
// (the pinned chunks are kept for the process: page-locking 64 MB costs
// more than an upload of it)
struct PinnedRing {
  std::mutex mu;
  unsigned char* buf[2] = {nullptr, nullptr};
};
PinnedRing& pinned_ring() {
  static PinnedRing r;
  return r;
}
constexpr size_t kUploadChunk = 32u << 20;   // bytes per pinned chunk
constexpr size_t kUploadDirect = 16u << 20;  // below: one pageable copy
}  // namespace

extern "C" int dpso_upload_matrix(const double* host, int64_t host_ld,
                                  int32_t rows, int32_t cols, double* dev,
                                  int64_t dev_ld, void* cuda_stream) {
  if (!host || !dev || rows < 0 || cols < 0 || host_ld < cols ||
      dev_ld < cols)
    return fail(DPSO_EINVAL, "bad arguments");
  if (rows == 0 || cols == 0) return DPSO_OK;
  cudaStream_t s = (cudaStream_t)cuda_stream;
  const size_t row_b = (size_t)cols * 8;
  const size_t total = row_b * (size_t)rows;
  cudaError_t e;
  if (total <= kUploadDirect || row_b > kUploadChunk) {
    e = cudaMemcpy2DAsync(dev, (size_t)dev_ld * 8, host, (size_t)host_ld * 8,
                          row_b, rows, cudaMemcpyHostToDevice, s);
    if (!e) e = cudaStreamSynchronize(s);
    return e ? fail(DPSO_ECUDA, cudaGetErrorString(e)) : DPSO_OK;
  }
  PinnedRing& R = pinned_ring();
  std::lock_guard<std::mutex> lock(R.mu);
  if (!R.buf[0]) {
    for (int b = 0; b < 2; ++b) {
      e = cudaHostAlloc((void**)&R.buf[b], kUploadChunk,
                        cudaHostAllocPortable);
      if (e) return fail(DPSO_ECUDA, cudaGetErrorString(e));
    }
  }
  // events of the stream's device (the caller may upload to several GPUs)
  struct Events {
    cudaEvent_t ev[2] = {nullptr, nullptr};
    ~Events() {
      for (auto x : ev)
        if (x) cudaEventDestroy(x);
    }
  } E;
  for (int b = 0; b < 2; ++b)
    if ((e = cudaEventCreateWithFlags(&E.ev[b], cudaEventDisableTiming)))
      return fail(DPSO_ECUDA, cudaGetErrorString(e));
  const int per_chunk = (int)(kUploadChunk / row_b);
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int nthr = (int)std::min<unsigned>(8, hw);
  bool used[2] = {false, false};
  int chunk = 0;
  for (int r0 = 0; r0 < rows; r0 += per_chunk, ++chunk) {
    const int nr = std::min(per_chunk, rows - r0);
    const int b = chunk & 1;
    // the DMA that last read this chunk is done
    // (on an error, drain the stream: no DMA may still read a chunk the
    // next call refills)
    auto bail = [&](cudaError_t err) {
      cudaStreamSynchronize(s);
      return fail(DPSO_ECUDA, cudaGetErrorString(err));
    };
    if (used[b] && (e = cudaEventSynchronize(E.ev[b]))) return bail(e);
    unsigned char* dst = R.buf[b];
    auto fill = [&](int t) {
      const int a = r0 + (int)((int64_t)nr * t / nthr);
      const int z = r0 + (int)((int64_t)nr * (t + 1) / nthr);
      if (host_ld == cols) {
        memcpy(dst + (size_t)(a - r0) * row_b, host + (size_t)a * host_ld,
               row_b * (size_t)(z - a));
      } else {
        for (int r = a; r < z; ++r)
          memcpy(dst + (size_t)(r - r0) * row_b, host + (size_t)r * host_ld,
                 row_b);
      }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nthr; ++t) th.emplace_back(fill, t);
    fill(0);
    for (auto& x : th) x.join();
    e = cudaMemcpy2DAsync(dev + (size_t)r0 * dev_ld, (size_t)dev_ld * 8, dst,
                          row_b, row_b, nr, cudaMemcpyHostToDevice, s);
    if (!e) e = cudaEventRecord(E.ev[b], s);
    if (e) return bail(e);
    used[b] = true;
  }
  e = cudaStreamSynchronize(s);
  return e ? fail(DPSO_ECUDA, cudaGetErrorString(e)) : DPSO_OK;
}
