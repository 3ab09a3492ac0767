// tns.cu — FROSTT .tns ingestion / output and tensor statistics (host code; SURVEY.md §8(f)
// NEXT-3; the paper's datasets come as .tns files; format SPEC.md:41-49,
// statistics of Table I).
//
// The reader maps the text to memory, splits it at line boundaries into one chunk per host
// thread, parses the chunks in parallel (std::from_chars: exact, locale-free) and
// concatenates them in file order, so nonzeros — duplicates included — keep their order.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "ctx.hpp"

struct splatt_tensor {
  int32_t N = 0;
  uint64_t nnz = 0;
  uint64_t dims[SPLATT_MAX_NMODES] = {0};
  std::vector<uint32_t> ind[SPLATT_MAX_NMODES];
  std::vector<double> vals;
};

namespace {

thread_local std::string g_tns_err;

struct Chunk {
  const char* b;
  const char* e;
  uint64_t lines = 0;        // newline-terminated lines in the chunk
  uint64_t err_line = 0;     // 1-based line within the chunk of the first error (0 = none)
  std::string err;
  std::vector<uint32_t> ind[SPLATT_MAX_NMODES];
  std::vector<double> vals;
  uint32_t maxi[SPLATT_MAX_NMODES] = {0};
};

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// Fields of one line [p, q): returns the count (up to cap + 1) and their spans.
int split_fields(const char* p, const char* q, const char** fb, const char** fe, int cap) {
  int n = 0;
  while (p < q) {
    while (p < q && is_space(*p)) ++p;
    if (p >= q) break;
    const char* s = p;
    while (p < q && !is_space(*p)) ++p;
    if (n < cap) { fb[n] = s; fe[n] = p; }
    ++n;
    if (n > cap) break;
  }
  return n;
}

// Number of fields of the first data line (0 if none).
int first_width(const char* b, const char* e) {
  const char* fb[SPLATT_MAX_NMODES + 2];
  const char* fe[SPLATT_MAX_NMODES + 2];
  while (b < e) {
    const char* nl = static_cast<const char*>(memchr(b, '\n', e - b));
    const char* q = nl ? nl : e;
    const char* s = b;
    while (s < q && is_space(*s)) ++s;
    if (s < q && *s != '#') return split_fields(s, q, fb, fe, SPLATT_MAX_NMODES + 1);
    b = nl ? nl + 1 : e;
  }
  return 0;
}

void parse_chunk(Chunk& c, int N) {
  const char* fb[SPLATT_MAX_NMODES + 2];
  const char* fe[SPLATT_MAX_NMODES + 2];
  const char* b = c.b;
  uint64_t line = 0;
  while (b < c.e) {
    const char* nl = static_cast<const char*>(memchr(b, '\n', c.e - b));
    const char* q = nl ? nl : c.e;
    ++line;
    const char* s = b;
    b = nl ? nl + 1 : c.e;
    while (s < q && is_space(*s)) ++s;
    if (s >= q || *s == '#') continue;
    if (c.err_line) continue;  // keep counting lines, stop parsing after the first error
    const int nf = split_fields(s, q, fb, fe, N + 1);
    if (nf != N + 1) {
      c.err_line = line;
      c.err = "expected " + std::to_string(N + 1) + " fields";
      continue;
    }
    uint32_t idx[SPLATT_MAX_NMODES];
    bool ok = true;
    for (int m = 0; m < N && ok; ++m) {
      uint64_t v = 0;
      const auto r = std::from_chars(fb[m], fe[m], v);
      if (r.ec != std::errc() || r.ptr != fe[m]) { c.err = "non-integer index"; ok = false; }
      else if (v < 1) { c.err = "index < 1"; ok = false; }
      else if (v > 0xffffffffull) { c.err = "index >= 2^32"; ok = false; }
      else idx[m] = (uint32_t)(v - 1);
    }
    double val = 0.0;
    if (ok) {
      const auto r = std::from_chars(fb[N], fe[N], val);
      if (r.ec != std::errc() || r.ptr != fe[N]) { c.err = "non-numeric value"; ok = false; }
    }
    if (!ok) {
      c.err_line = line;
      continue;
    }
    for (int m = 0; m < N; ++m) {
      c.ind[m].push_back(idx[m]);
      c.maxi[m] = std::max(c.maxi[m], idx[m] + 1);
    }
    c.vals.push_back(val);
  }
  c.lines = line;
}

int host_threads() {
  const unsigned h = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(h, 64u));
}

}  // namespace

extern "C" {

const char* splatt_tensor_error(void) { return g_tns_err.c_str(); }

splatt_status splatt_tns_read(const char* path, splatt_tensor** out) {
  g_tns_err.clear();
  if (!path || !out) return SPLATT_ERR_BADINPUT;
  try {
    FILE* f = fopen(path, "rb");
    if (!f) {
      g_tns_err = std::string("cannot open ") + path;
      return SPLATT_ERR_BADINPUT;
    }
    fseek(f, 0, SEEK_END);
    const long sz = ftell(f);
    fseek(f, 0, SEEK_SET);
    std::vector<char> text((size_t)std::max<long>(sz, 0));
    const size_t got = sz > 0 ? fread(text.data(), 1, (size_t)sz, f) : 0;
    fclose(f);
    text.resize(got);
    const char* b = text.data();
    const char* e = b + text.size();
    const int width = first_width(b, e);
    if (width == 0) {
      g_tns_err = "no nonzeros";
      return SPLATT_ERR_BADINPUT;
    }
    const int N = width - 1;
    if (N < 1 || N > SPLATT_MAX_NMODES) {
      g_tns_err = "line width gives " + std::to_string(N) + " modes (supported: 1..8)";
      return SPLATT_ERR_BADINPUT;
    }
    // chunks at line boundaries
    const int T = (int)std::max<size_t>(1, std::min<size_t>(host_threads(), text.size() >> 20));
    std::vector<Chunk> ch(T);
    const char* p = b;
    for (int t = 0; t < T; ++t) {
      ch[t].b = p;
      const char* target = (t == T - 1) ? e : b + (text.size() * (t + 1)) / T;
      if (target < p) target = p;
      const char* nl = (target < e) ? static_cast<const char*>(memchr(target, '\n', e - target)) : nullptr;
      p = (t == T - 1 || !nl) ? e : nl + 1;
      ch[t].e = p;
    }
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(parse_chunk, std::ref(ch[t]), N);
    parse_chunk(ch[0], N);
    for (auto& x : th) x.join();
    uint64_t line0 = 0, nnz = 0;
    for (int t = 0; t < T; ++t) {
      if (ch[t].err_line) {
        g_tns_err = "line " + std::to_string(line0 + ch[t].err_line) + ": " + ch[t].err;
        return SPLATT_ERR_BADINPUT;
      }
      line0 += ch[t].lines;
      nnz += ch[t].vals.size();
    }
    if (nnz == 0) {
      g_tns_err = "no nonzeros";
      return SPLATT_ERR_BADINPUT;
    }
    auto* tt = new splatt_tensor();
    tt->N = N;
    tt->nnz = nnz;
    for (int m = 0; m < N; ++m) {
      tt->ind[m].resize(nnz);
      uint32_t mx = 0;
      for (int t = 0; t < T; ++t) mx = std::max(mx, ch[t].maxi[m]);
      tt->dims[m] = mx;
    }
    tt->vals.resize(nnz);
    uint64_t off = 0;
    for (int t = 0; t < T; ++t) {
      const size_t n = ch[t].vals.size();
      for (int m = 0; m < N; ++m)
        std::memcpy(tt->ind[m].data() + off, ch[t].ind[m].data(), n * 4);
      std::memcpy(tt->vals.data() + off, ch[t].vals.data(), n * 8);
      off += n;
    }
    *out = tt;
    return SPLATT_OK;
  } catch (const std::bad_alloc&) {
    g_tns_err = "host allocation failed";
    return SPLATT_ERR_NOMEM;
  } catch (const std::exception& ex) {
    g_tns_err = ex.what();
    return SPLATT_ERR_BADINPUT;
  }
}

splatt_status splatt_tensor_coo(const splatt_tensor* t, splatt_coo* view) {
  if (!t || !view) return SPLATT_ERR_BADINPUT;
  std::memset(view, 0, sizeof(*view));
  view->nmodes = t->N;
  view->nnz = t->nnz;
  for (int m = 0; m < t->N; ++m) {
    view->dims[m] = t->dims[m];
    view->ind[m] = t->ind[m].data();
  }
  view->vals = t->vals.data();
  return SPLATT_OK;
}

void splatt_tensor_free(splatt_tensor* t) { delete t; }

splatt_status splatt_tns_write(const char* path, const splatt_coo* coo) {
  g_tns_err.clear();
  if (!path || !coo || coo->nmodes < 1 || coo->nmodes > SPLATT_MAX_NMODES || !coo->vals)
    return SPLATT_ERR_BADINPUT;
  for (int m = 0; m < coo->nmodes; ++m)
    if (!coo->ind[m]) return SPLATT_ERR_BADINPUT;
  try {
    const int N = coo->nmodes;
    const uint64_t nnz = coo->nnz;
    const int T = (int)std::max<uint64_t>(1, std::min<uint64_t>(host_threads(), nnz >> 16));
    std::vector<std::string> buf(T);
    std::vector<std::thread> th;
    auto work = [&](int t) {
      const uint64_t lo = nnz * t / T, hi = nnz * (t + 1) / T;
      std::string& s = buf[t];
      s.reserve((hi - lo) * (N * 8 + 26));
      char tmp[64];
      for (uint64_t p = lo; p < hi; ++p) {
        for (int m = 0; m < N; ++m) {
          const auto r = std::to_chars(tmp, tmp + sizeof(tmp), (uint64_t)coo->ind[m][p] + 1);
          s.append(tmp, r.ptr);
          s.push_back(' ');
        }
        const auto r = std::to_chars(tmp, tmp + sizeof(tmp), coo->vals[p]);  // shortest round trip
        s.append(tmp, r.ptr);
        s.push_back('\n');
      }
    };
    for (int t = 1; t < T; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    FILE* f = fopen(path, "wb");
    if (!f) {
      g_tns_err = std::string("cannot open ") + path;
      return SPLATT_ERR_BADINPUT;
    }
    bool ok = true;
    for (auto& s : buf) ok = ok && fwrite(s.data(), 1, s.size(), f) == s.size();
    ok = (fclose(f) == 0) && ok;
    if (!ok) {
      g_tns_err = std::string("write failed: ") + path;
      return SPLATT_ERR_BADINPUT;
    }
    return SPLATT_OK;
  } catch (const std::bad_alloc&) {
    return SPLATT_ERR_NOMEM;
  }
}

splatt_status splatt_coo_stats(const splatt_coo* coo, splatt_tensor_stats* out) {
  if (!coo || !out || coo->nmodes < 1 || coo->nmodes > SPLATT_MAX_NMODES) return SPLATT_ERR_BADINPUT;
  for (int m = 0; m < coo->nmodes; ++m)
    if (!coo->ind[m] || coo->dims[m] < 1) return SPLATT_ERR_BADINPUT;
  try {
    std::memset(out, 0, sizeof(*out));
    out->nmodes = coo->nmodes;
    out->nnz = coo->nnz;
    double cells = 1.0;
    for (int m = 0; m < coo->nmodes; ++m) {
      out->dims[m] = coo->dims[m];
      cells *= (double)coo->dims[m];
    }
    out->density = (double)coo->nnz / cells;
    for (int m = 0; m < coo->nmodes; ++m) {
      std::vector<uint64_t> cnt(coo->dims[m], 0);
      for (uint64_t p = 0; p < coo->nnz; ++p) {
        const uint32_t i = coo->ind[m][p];
        if (i >= coo->dims[m]) return SPLATT_ERR_BADINPUT;
        ++cnt[i];
      }
      uint64_t ne = 0, mx = 0;
      for (uint64_t c : cnt) {
        ne += (c > 0);
        mx = std::max(mx, c);
      }
      out->nonempty_slices[m] = ne;
      out->max_slice_nnz[m] = mx;
    }
    return SPLATT_OK;
  } catch (const std::bad_alloc&) {
    return SPLATT_ERR_NOMEM;
  }
}

}  // extern "C"
