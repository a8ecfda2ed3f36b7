// Native parser of the multi-label dataset text format (datasets.py:81-167),
// SURVEY.md section 8(f) rank 2.  Host code: one pass over the UTF-8 buffer,
// CSR arrays out.  The accept/reject decisions follow the reference loader
// token by token (Python str.splitlines / str.split / int() / float()
// grammars, checks in the same order); on a rejection the parser reports the
// error kind, the 1-based line and the offending token's byte span, and the
// Python wrapper renders the reference's exact message from them.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/fastpi_b200.h"

namespace {

struct Parsed {
  int64_t m = 0, n = 0, L = 0;
  std::vector<int64_t> fptr, fidx, lptr, lidx;
  std::vector<double> fval;
};

// Python str.splitlines() boundaries (ASCII set plus U+0085, U+2028, U+2029 in UTF-8).
// Returns the length of the line break starting at p (0 if none).
inline int line_break(const unsigned char* p, const unsigned char* end) {
  const unsigned c = p[0];
  if (c == '\r') return (p + 1 < end && p[1] == '\n') ? 2 : 1;
  if (c == '\n' || c == 0x0b || c == 0x0c || c == 0x1c || c == 0x1d || c == 0x1e) return 1;
  if (c == 0xc2 && p + 1 < end && p[1] == 0x85) return 2;
  if (c == 0xe2 && p + 2 < end && p[1] == 0x80 && (p[2] == 0xa8 || p[2] == 0xa9)) return 3;
  return 0;
}

// ASCII whitespace of Python's str.split() / int() / float() stripping
inline bool py_space(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == 0x0b || c == 0x0c || (c >= 0x1c && c <= 0x1f);
}
inline bool is_digit(unsigned char c) { return c >= '0' && c <= '9'; }

// digitpart: digit (["_"] digit)*   -- returns end or nullptr
const char* digitpart(const char* p, const char* e) {
  if (p >= e || !is_digit(*p)) return nullptr;
  ++p;
  while (p < e) {
    if (is_digit(*p)) {
      ++p;
    } else if (*p == '_' && p + 1 < e && is_digit(p[1])) {
      p += 2;
    } else {
      break;
    }
  }
  return p;
}

// Python int(s, 10): optional surrounding whitespace, sign, digitpart.  ovf: exceeds int64.
bool py_int(const char* b, const char* e, int64_t& out, bool& ovf) {
  while (b < e && py_space((unsigned char)*b)) ++b;
  while (e > b && py_space((unsigned char)e[-1])) --e;
  bool neg = false;
  if (b < e && (*b == '+' || *b == '-')) neg = *b++ == '-';
  const char* d = digitpart(b, e);
  if (!d || d != e) return false;
  unsigned long long v = 0;
  ovf = false;
  for (const char* p = b; p < e; ++p) {
    if (*p == '_') continue;
    const unsigned dig = (unsigned)(*p - '0');
    if (v > (0x7fffffffffffffffULL - dig) / 10) ovf = true;
    if (!ovf) v = v * 10 + dig;
  }
  out = neg ? -(int64_t)v : (int64_t)v;
  return true;
}

bool ieq(const char* b, const char* e, const char* lit) {
  const size_t n = strlen(lit);
  if ((size_t)(e - b) != n) return false;
  for (size_t i = 0; i < n; ++i)
    if ((b[i] | 0x20) != lit[i]) return false;
  return true;
}

// Python float(s): whitespace, sign, (inf | infinity | nan | numeric with '_' grouping).
bool py_float(const char* b, const char* e, double& out) {
  while (b < e && py_space((unsigned char)*b)) ++b;
  while (e > b && py_space((unsigned char)e[-1])) --e;
  const char* s = b;
  bool neg = false;
  if (s < e && (*s == '+' || *s == '-')) neg = *s++ == '-';
  if (ieq(s, e, "inf") || ieq(s, e, "infinity")) {
    out = neg ? -INFINITY : INFINITY;
    return true;
  }
  if (ieq(s, e, "nan")) {
    out = NAN;
    return true;
  }
  const char* p = s;
  bool mant = false;
  if (const char* d = digitpart(p, e)) {
    p = d;
    mant = true;
  }
  if (p < e && *p == '.') {
    ++p;
    if (const char* d = digitpart(p, e)) {
      p = d;
      mant = true;
    }
  }
  if (!mant) return false;
  if (p < e && (*p == 'e' || *p == 'E')) {
    ++p;
    if (p < e && (*p == '+' || *p == '-')) ++p;
    const char* d = digitpart(p, e);
    if (!d) return false;
    p = d;
  }
  if (p != e) return false;
  std::string clean;
  clean.reserve((size_t)(e - b));
  for (const char* q = b; q < e; ++q)
    if (*q != '_') clean.push_back(*q);
  errno = 0;
  out = strtod(clean.c_str(), nullptr);  // correctly rounded; overflow -> inf, underflow -> 0 as in Python
  return true;
}

struct Fail {
  int32_t kind;
  int64_t line;
  const char *t0, *t1, *u0, *u1;
};

int fail(fpi_dataset_info* info, const char* base, const Fail& f) {
  info->err_kind = f.kind;
  info->err_line = f.line;
  info->tok_begin = f.t0 ? f.t0 - base : -1;
  info->tok_end = f.t1 ? f.t1 - base : -1;
  info->tok2_begin = f.u0 ? f.u0 - base : -1;
  info->tok2_end = f.u1 ? f.u1 - base : -1;
  return FPI_EDOMAIN;
}

}  // namespace

extern "C" int fpi_dataset_parse(const char* buf, int64_t len, void** h_out, fpi_dataset_info* info) {
  if (!info || !h_out || (!buf && len)) return FPI_EDOMAIN;
  *info = fpi_dataset_info{};
  *h_out = nullptr;
  // split into lines (Python splitlines: a trailing break does not open a new line)
  std::vector<std::pair<const char*, const char*>> lines;
  {
    const unsigned char* p = (const unsigned char*)buf;
    const unsigned char* end = p + len;
    const unsigned char* start = p;
    while (p < end) {
      const int lb = line_break(p, end);
      if (lb) {
        lines.emplace_back((const char*)start, (const char*)p);
        p += lb;
        start = p;
      } else {
        ++p;
      }
    }
    if (start < end) lines.emplace_back((const char*)start, (const char*)end);
  }
  info->n_lines = (int64_t)lines.size();
  if (lines.empty()) return fail(info, buf, {FPI_DS_EMPTY, 1, nullptr, nullptr, nullptr, nullptr});
  // header: exactly three whitespace-separated integers
  const char* hb = lines[0].first;
  const char* he = lines[0].second;
  std::vector<std::pair<const char*, const char*>> parts;
  for (const char* p = hb; p < he;) {
    while (p < he && py_space((unsigned char)*p)) ++p;
    const char* q = p;
    while (q < he && !py_space((unsigned char)*q)) ++q;
    if (q > p) parts.emplace_back(p, q);
    p = q;
  }
  if (parts.size() != 3) return fail(info, buf, {FPI_DS_HEADER_SHAPE, 1, hb, he, nullptr, nullptr});
  int64_t hv[3];
  for (int i = 0; i < 3; ++i) {
    bool ovf = false;
    if (!py_int(parts[i].first, parts[i].second, hv[i], ovf) || ovf)
      return fail(info, buf, {ovf ? FPI_DS_HEADER_RANGE : FPI_DS_HEADER_INT, 1, hb, he, nullptr, nullptr});
  }
  if (hv[0] < 0 || hv[1] < 0 || hv[2] < 0) return fail(info, buf, {FPI_DS_HEADER_NEG, 1, hb, he, nullptr, nullptr});
  const int64_t m = hv[0], n = hv[1], L = hv[2];
  info->m = m;
  info->n = n;
  info->L = L;
  if ((int64_t)lines.size() - 1 != m)
    return fail(info, buf, {FPI_DS_LINE_COUNT, (int64_t)lines.size(), nullptr, nullptr, nullptr, nullptr});

  Parsed* P = new (std::nothrow) Parsed();
  if (!P) return FPI_ECAPACITY;
  P->m = m;
  P->n = n;
  P->L = L;
  P->fptr.assign((size_t)m + 1, 0);
  P->lptr.assign((size_t)m + 1, 0);
  std::vector<int64_t> row_labels;
  std::vector<std::pair<const char*, const char*>> toks;
  for (int64_t row = 0; row < m; ++row) {
    const int64_t lineno = row + 2;
    const char* b = lines[(size_t)row + 1].first;
    const char* e = lines[(size_t)row + 1].second;
    const char* cut = (const char*)memchr(b, ' ', (size_t)(e - b));
    const char *lb = b, *le = cut ? cut : e;
    toks.clear();
    if (cut) {  // rest.split()
      for (const char* p = cut + 1; p < e;) {
        while (p < e && py_space((unsigned char)*p)) ++p;
        const char* q = p;
        while (q < e && !py_space((unsigned char)*q)) ++q;
        if (q > p) toks.emplace_back(p, q);
        p = q;
      }
    }
    if (memchr(lb, ':', (size_t)(le - lb))) {  // a label field holding a colon is a feature token
      toks.insert(toks.begin(), {lb, le});
      le = lb;
    }
    row_labels.clear();
    if (le > lb) {
      for (const char* p = lb;;) {  // label_field.split(",")
        const char* q = (const char*)memchr(p, ',', (size_t)(le - p));
        const char* te = q ? q : le;
        int64_t lab;
        bool ovf = false;
        if (!py_int(p, te, lab, ovf)) {
          delete P;
          return fail(info, buf, {FPI_DS_BAD_LABEL, lineno, p, te, nullptr, nullptr});
        }
        if (ovf || lab < 0 || lab >= L) {
          delete P;
          return fail(info, buf, {FPI_DS_LABEL_RANGE, lineno, p, te, nullptr, nullptr});
        }
        for (int64_t x : row_labels)
          if (x == lab) {
            delete P;
            return fail(info, buf, {FPI_DS_LABEL_DUP, lineno, p, te, nullptr, nullptr});
          }
        row_labels.push_back(lab);
        if (!q) break;
        p = q + 1;
      }
    }
    std::sort(row_labels.begin(), row_labels.end());
    P->lidx.insert(P->lidx.end(), row_labels.begin(), row_labels.end());
    P->lptr[(size_t)row + 1] = (int64_t)P->lidx.size();

    int64_t prev = -1;
    const char *pb = nullptr, *pe = nullptr;
    for (auto& t : toks) {
      const char* colon = (const char*)memchr(t.first, ':', (size_t)(t.second - t.first));
      if (!colon || colon + 1 == t.second) {
        delete P;
        return fail(info, buf, {FPI_DS_FEAT_TOKEN, lineno, t.first, t.second, nullptr, nullptr});
      }
      int64_t idx;
      double val;
      bool ovf = false;
      if (!py_int(t.first, colon, idx, ovf) || !py_float(colon + 1, t.second, val)) {
        delete P;
        return fail(info, buf, {FPI_DS_FEAT_PARSE, lineno, t.first, t.second, nullptr, nullptr});
      }
      if (ovf || idx < 0 || idx >= n) {
        delete P;
        return fail(info, buf, {FPI_DS_FEAT_RANGE, lineno, t.first, colon, nullptr, nullptr});
      }
      if (idx == prev) {
        delete P;
        return fail(info, buf, {FPI_DS_FEAT_DUP, lineno, t.first, colon, nullptr, nullptr});
      }
      if (idx < prev) {
        delete P;
        return fail(info, buf, {FPI_DS_FEAT_ORDER, lineno, t.first, colon, pb, pe});
      }
      if (!std::isfinite(val)) {
        delete P;
        return fail(info, buf, {FPI_DS_FEAT_NONFINITE, lineno, colon + 1, t.second, nullptr, nullptr});
      }
      if (val == 0.0) {
        delete P;
        return fail(info, buf, {FPI_DS_FEAT_ZERO, lineno, t.first, colon, nullptr, nullptr});
      }
      prev = idx;
      pb = t.first;
      pe = colon;
      P->fidx.push_back(idx);
      P->fval.push_back(val);
    }
    P->fptr[(size_t)row + 1] = (int64_t)P->fidx.size();
  }
  info->nnz_feat = (int64_t)P->fidx.size();
  info->nnz_lab = (int64_t)P->lidx.size();
  *h_out = P;
  return FPI_OK;
}

extern "C" int fpi_dataset_fetch(void* h, int64_t* feat_ptr, int64_t* feat_idx, double* feat_val, int64_t* lab_ptr,
                                 int64_t* lab_idx) {
  if (!h) return FPI_EDOMAIN;
  const Parsed* P = static_cast<const Parsed*>(h);
  auto cp = [](auto* dst, const auto& v) {
    if (dst && !v.empty()) memcpy(dst, v.data(), v.size() * sizeof(v[0]));
  };
  cp(feat_ptr, P->fptr);
  cp(feat_idx, P->fidx);
  cp(feat_val, P->fval);
  cp(lab_ptr, P->lptr);
  cp(lab_idx, P->lidx);
  return FPI_OK;
}

extern "C" int fpi_dataset_free(void* h) {
  delete static_cast<Parsed*>(h);
  return FPI_OK;
}
