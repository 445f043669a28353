// nnm_csv.cpp -- native CSV ingestion for the NNM drop-in.
//
// Restates parclust.dataio.load_dataset (dataio.py:49-116) so a 2M-row input parses in
// well under a second instead of minutes of Python:
//   * lines: str.splitlines() boundaries (\n, \r\n, \r, \v, \f, \x1c-\x1e, U+0085,
//     U+2028, U+2029); blank lines (str.strip() empty) are skipped; line numbers are
//     1-based physical lines;
//   * fields: line.split(delimiter), each field str.strip()'d;
//   * header: the first kept line is a header if any field fails float();
//   * id column by header name or 0-based index; remaining fields parse with Python's
//     float() grammar (sign, digits with single underscores between digits, fraction,
//     exponent, inf / infinity / nan, case-insensitive), correctly rounded (strtod);
//   * the same ValidationError messages, reporting the first offending line.
// Rows are parsed by std::thread workers over contiguous line ranges.
#include <errno.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

namespace {

struct Line {
  int64_t begin, end;  // byte range (without the terminator)
  int64_t no;          // 1-based physical line number
};

// Python str.isspace for the code points we can meet in UTF-8 text (ASCII + the
// common Unicode spaces); returns the byte length of a whitespace char at p, or 0.
int ws_len(const unsigned char* p, const unsigned char* e) {
  const unsigned char c = p[0];
  if (c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f)) return 1;
  if (c == 0xc2 && p + 1 < e && (p[1] == 0x85 || p[1] == 0xa0)) return 2;
  if (c == 0xe1 && p + 2 < e && p[1] == 0x9a && p[2] == 0x80) return 3;  // U+1680
  if (c == 0xe2 && p + 2 < e && p[1] == 0x80 &&
      ((p[2] >= 0x80 && p[2] <= 0x8a) || p[2] == 0xa8 || p[2] == 0xa9 || p[2] == 0xaf))
    return 3;  // U+2000-200A, U+2028/2029, U+202F
  if (c == 0xe2 && p + 2 < e && p[1] == 0x81 && p[2] == 0x9f) return 3;  // U+205F
  if (c == 0xe3 && p + 2 < e && p[1] == 0x80 && p[2] == 0x80) return 3;  // U+3000
  return 0;
}

// length of the trailing whitespace char ending at e (or 0)
int ws_len_back(const unsigned char* b, const unsigned char* e) {
  for (int k = 1; k <= 3 && e - k >= b; ++k)
    if (ws_len(e - k, e) == k) return k;
  return 0;
}

void strip(const unsigned char*& b, const unsigned char*& e) {
  int k;
  while (b < e && (k = ws_len(b, e)) > 0) b += k;
  while (e > b && (k = ws_len_back(b, e)) > 0) e -= k;
}

// Python float() on an already stripped token; false if it would raise ValueError.
bool py_float(const unsigned char* b, const unsigned char* e, double& out) {
  if (b == e) return false;
  const unsigned char* p = b;
  std::string buf;
  buf.reserve(e - b);
  if (*p == '+' || *p == '-') buf.push_back((char)*p++);
  // inf / infinity / nan (case-insensitive)
  auto word = [&](const char* w) {
    const size_t L = strlen(w);
    if ((size_t)(e - p) != L) return false;
    for (size_t k = 0; k < L; ++k)
      if (tolower(p[k]) != w[k]) return false;
    return true;
  };
  if (word("inf") || word("infinity")) {
    out = (buf == "-") ? -INFINITY : INFINITY;
    return true;
  }
  if (word("nan")) {
    out = NAN;
    return true;
  }
  // digits with single underscores strictly between digits
  auto digits = [&](bool& any) {
    any = false;
    bool prev_digit = false;
    while (p < e) {
      if (*p >= '0' && *p <= '9') {
        buf.push_back((char)*p++);
        any = prev_digit = true;
      } else if (*p == '_' && prev_digit && p + 1 < e && p[1] >= '0' && p[1] <= '9') {
        ++p;
        prev_digit = false;
      } else {
        break;
      }
    }
  };
  bool int_digits = false, frac_digits = false;
  digits(int_digits);
  if (p < e && *p == '.') {
    buf.push_back('.');
    ++p;
    digits(frac_digits);
  }
  if (!int_digits && !frac_digits) return false;
  if (p < e && (*p == 'e' || *p == 'E')) {
    buf.push_back('e');
    ++p;
    if (p < e && (*p == '+' || *p == '-')) buf.push_back((char)*p++);
    bool exp_digits = false;
    digits(exp_digits);
    if (!exp_digits) return false;
  }
  if (p != e) return false;
  char* endp = nullptr;
  out = strtod(buf.c_str(), &endp);  // correctly rounded, as CPython's dtoa
  return endp && *endp == '\0';
}

std::string py_repr(const unsigned char* b, const unsigned char* e) {
  // repr() of a str: single quotes unless the text contains ' and no "
  std::string s((const char*)b, e - b);
  const bool sq = s.find('\'') != std::string::npos, dq = s.find('"') != std::string::npos;
  const char q = (sq && !dq) ? '"' : '\'';
  std::string r(1, q);
  for (unsigned char c : s) {
    if (c == (unsigned char)q || c == '\\') {
      r.push_back('\\');
      r.push_back((char)c);
    } else if (c == '\t') {
      r += "\\t";
    } else if (c < 0x20 || c == 0x7f) {
      char t[8];
      snprintf(t, sizeof t, "\\x%02x", c);
      r += t;
    } else {
      r.push_back((char)c);
    }
  }
  r.push_back(q);
  return r;
}

struct Fields {
  std::vector<std::pair<const unsigned char*, const unsigned char*>> f;
};

void split(const unsigned char* b, const unsigned char* e, char delim, Fields& out) {
  out.f.clear();
  const unsigned char* s = b;
  for (const unsigned char* p = b; p <= e; ++p) {
    if (p == e || *p == (unsigned char)delim) {
      const unsigned char *fb = s, *fe = p;
      strip(fb, fe);
      out.f.emplace_back(fb, fe);
      s = p + 1;
    }
  }
}

}  // namespace

struct nnm_csv {
  std::string path;
  std::vector<unsigned char> text;
  int64_t n = 0, d = 0;
  std::vector<double> values;
  std::vector<std::string> ids;
  bool has_ids = false;
};

// errors: message into *err (caller frees with nnm_csv_free) -- see nnm_api.cu wrappers
int nnm_csv_parse_impl(const char* path, char delim, const char* id_column, int threads,
                       nnm_csv** out, std::string& err) {
  auto* c = new nnm_csv();
  c->path = path;
  FILE* fh = fopen(path, "rb");
  if (!fh) {
    err = std::string("cannot read ") + path + ": " + strerror(errno);
    delete c;
    return -1;
  }
  fseek(fh, 0, SEEK_END);
  const long sz = ftell(fh);
  fseek(fh, 0, SEEK_SET);
  c->text.resize(sz > 0 ? (size_t)sz : 0);
  if (sz > 0 && fread(c->text.data(), 1, (size_t)sz, fh) != (size_t)sz) {
    fclose(fh);
    err = std::string("cannot read ") + path;
    delete c;
    return -1;
  }
  fclose(fh);
  const unsigned char* T = c->text.data();
  const int64_t N = (int64_t)c->text.size();
  // str.splitlines() boundaries; keep non-blank lines with their 1-based numbers
  std::vector<Line> lines;
  int64_t s = 0, no = 1;
  auto push = [&](int64_t b, int64_t e) {
    const unsigned char *pb = T + b, *pe = T + e;
    strip(pb, pe);
    if (pb < pe) lines.push_back({b, e, no});
    ++no;
  };
  for (int64_t i = 0; i < N;) {
    const unsigned char ch = T[i];
    int brk = 0;
    if (ch == '\n' || ch == '\v' || ch == '\f' || ch == 0x1c || ch == 0x1d || ch == 0x1e) brk = 1;
    else if (ch == '\r') brk = (i + 1 < N && T[i + 1] == '\n') ? 2 : 1;
    else if (ch == 0xc2 && i + 1 < N && T[i + 1] == 0x85) brk = 2;
    else if (ch == 0xe2 && i + 2 < N && T[i + 1] == 0x80 && (T[i + 2] == 0xa8 || T[i + 2] == 0xa9)) brk = 3;
    if (brk) {
      push(s, i);
      i += brk;
      s = i;
    } else {
      ++i;
    }
  }
  if (s < N) push(s, N);
  if (lines.empty()) {
    err = c->path + ": empty input";
    delete c;
    return -1;
  }
  Fields first;
  split(T + lines[0].begin, T + lines[0].end, delim, first);
  const int64_t ncols = (int64_t)first.f.size();
  bool header = false;
  for (auto& f : first.f) {
    double v;
    if (!py_float(f.first, f.second, v)) header = true;
  }
  size_t l0 = header ? 1 : 0;
  if (header && lines.size() == 1) {
    err = c->path + ": no data rows after header";
    delete c;
    return -1;
  }
  int64_t id_idx = -1;
  if (id_column) {
    const std::string want(id_column);
    bool found = false;
    if (header)
      for (int64_t j = 0; j < ncols; ++j)
        if (std::string((const char*)first.f[j].first, first.f[j].second - first.f[j].first) == want) {
          id_idx = j;
          found = true;
          break;
        }
    if (!found) {
      // int(id_column): optional sign, digits (underscores allowed), surrounding spaces
      const unsigned char *b = (const unsigned char*)id_column, *e = b + want.size();
      strip(b, e);
      std::string dg;
      bool neg = false, ok = b < e;
      const unsigned char* p = b;
      if (ok && (*p == '+' || *p == '-')) neg = *p++ == '-';
      bool prev = false;
      for (; ok && p < e; ++p) {
        if (*p >= '0' && *p <= '9') {
          dg.push_back((char)*p);
          prev = true;
        } else if (*p == '_' && prev && p + 1 < e && p[1] >= '0' && p[1] <= '9') {
          prev = false;
        } else {
          ok = false;
        }
      }
      if (!ok || dg.empty()) {
        err = "id column " + py_repr((const unsigned char*)id_column,
                                     (const unsigned char*)id_column + want.size()) +
              " not found in header and not an index";
        delete c;
        return -1;
      }
      const size_t nz = std::min(dg.find_first_not_of('0'), dg.size() - 1);
      dg = dg.substr(nz);  // int() drops leading zeros
      long long v = dg.size() > 18 ? (1LL << 62) : atoll(dg.c_str());
      if (neg) v = -v;
      if (!(v >= 0 && v < ncols)) {
        err = "id column index " + std::string(neg && dg != "0" ? "-" : "") + dg +
              " out of range for " + std::to_string(ncols) + " columns";
        delete c;
        return -1;
      }
      id_idx = v;
    }
  }
  c->has_ids = id_idx >= 0;
  c->d = ncols - (c->has_ids ? 1 : 0);
  const int64_t nrows = (int64_t)(lines.size() - l0);
  c->n = nrows;
  c->values.resize((size_t)nrows * (size_t)c->d);
  if (c->has_ids) c->ids.resize(nrows);
  // parallel row parse; each worker remembers its first error (lowest line)
  int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = (int)std::min<int64_t>(nt, std::max<int64_t>(1, nrows / 4096));
  std::vector<std::string> errs(nt);
  std::vector<int64_t> err_line(nt, INT64_MAX);
  auto work = [&](int t) {
    const int64_t r0 = nrows * t / nt, r1 = nrows * (t + 1) / nt;
    Fields fl;
    for (int64_t r = r0; r < r1; ++r) {
      const Line& L = lines[l0 + r];
      split(T + L.begin, T + L.end, delim, fl);
      if ((int64_t)fl.f.size() != ncols) {
        errs[t] = "line " + std::to_string(L.no) + ": expected " + std::to_string(ncols) +
                  " columns, got " + std::to_string(fl.f.size());
        err_line[t] = L.no;
        return;
      }
      int64_t col = 0;
      for (int64_t j = 0; j < ncols; ++j) {
        const auto& f = fl.f[j];
        if (j == id_idx) {
          c->ids[r].assign((const char*)f.first, f.second - f.first);
          continue;
        }
        double v;
        if (!py_float(f.first, f.second, v)) {
          errs[t] = "line " + std::to_string(L.no) + ": non-numeric value " + py_repr(f.first, f.second);
          err_line[t] = L.no;
          return;
        }
        if (!std::isfinite(v)) {
          errs[t] = "line " + std::to_string(L.no) + ": non-finite feature value " +
                    py_repr(f.first, f.second);
          err_line[t] = L.no;
          return;
        }
        c->values[(size_t)r * c->d + col++] = v;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  int best = -1;
  for (int t = 0; t < nt; ++t)
    if (err_line[t] != INT64_MAX && (best < 0 || err_line[t] < err_line[best])) best = t;
  if (best >= 0) {
    err = errs[best];
    delete c;
    return -1;
  }
  if (c->has_ids) {
    std::unordered_set<std::string> seen;
    seen.reserve(c->ids.size() * 2);
    for (auto& v : c->ids)
      if (!seen.insert(v).second) {
        err = c->path + ": duplicate id " + py_repr((const unsigned char*)v.data(),
                                                    (const unsigned char*)v.data() + v.size());
        delete c;
        return -1;
      }
  }
  c->text.clear();
  c->text.shrink_to_fit();
  *out = c;
  return 0;
}

// ---------------------------------------------------------------- C ABI helpers
// (the error plumbing lives in nnm_api.cu: nnm_csv_load wraps nnm_csv_parse_impl)
int64_t nnm_csv_rows(const nnm_csv* c) { return c->n; }
int64_t nnm_csv_cols(const nnm_csv* c) { return c->d; }
bool nnm_csv_has_ids(const nnm_csv* c) { return c->has_ids; }
void nnm_csv_copy_values(const nnm_csv* c, double* out) {
  if (!c->values.empty()) memcpy(out, c->values.data(), c->values.size() * sizeof(double));
}
int64_t nnm_csv_id_bytes(const nnm_csv* c) {
  int64_t t = 0;
  for (auto& v : c->ids) t += (int64_t)v.size();
  return t;
}
void nnm_csv_copy_ids(const nnm_csv* c, char* buf, int64_t* offsets) {
  int64_t o = 0;
  for (size_t i = 0; i < c->ids.size(); ++i) {
    offsets[i] = o;
    memcpy(buf + o, c->ids[i].data(), c->ids[i].size());
    o += (int64_t)c->ids[i].size();
  }
  offsets[c->ids.size()] = o;
}
void nnm_csv_destroy(nnm_csv* c) { delete c; }

// ---------------------------------------------------------------- Dataset validation
// First non-finite element of a row-major float64 matrix (-1 if none): the
// model.Dataset check (model.py:29-76, "non-finite feature value in row r"),
// split over threads so a 2M x 25 matrix (400 MB) takes milliseconds.
int64_t nnm_first_nonfinite_impl(const double* x, int64_t count, int threads) {
  int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  const int64_t min_chunk = 1 << 20;
  nt = (int)std::max<int64_t>(1, std::min<int64_t>(nt, (count + min_chunk - 1) / min_chunk));
  std::vector<int64_t> first(nt, -1);
  auto work = [&](int t) {
    const int64_t lo = count * t / nt, hi = count * (t + 1) / nt;
    const int64_t B = 4096;
    for (int64_t b = lo; b < hi; b += B) {
      const int64_t e = std::min(hi, b + B);
      bool bad = false;
      for (int64_t i = b; i < e; ++i) bad |= !std::isfinite(x[i]);
      if (bad) {
        for (int64_t i = b; i < e; ++i)
          if (!std::isfinite(x[i])) { first[t] = i; return; }
      }
    }
  };
  if (nt == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
  }
  for (int t = 0; t < nt; ++t)
    if (first[t] >= 0) return first[t];
  return -1;
}
