// trace.cpp — trace ingestion for the window path, host side.
//
// Parses the reference's trace files into the structure-of-arrays the window
// scheduler consumes, with the reference's semantics and error reporting
// (workload.py:343-437):
//   CSV   (`_load_csv`, :343-381): csv.reader rows (excel dialect: ',' delimiter,
//         '"' quoting with "" escapes, quoted fields may span lines), blank rows
//         skipped, a row whose first field is "arrival_s" skipped (optional
//         header), exactly 4 fields, arrival = float(), input / output = int()
//         (output may be empty -> None), class online|offline (case-insensitive,
//         stripped), input >= 1, output >= 1.
//   JSONL (`_load_jsonl`, :384-419): one JSON object per non-blank line, known keys
//         only, arrival_s / input_tokens / class required, type checks as the
//         reference (bools are not numbers, input / output must be JSON integers).
// Ids follow file order; records are then stable-sorted by arrival time
// (`load_trace`, :422-431).  The first malformed record stops the parse with the
// reference's TraceFormatError text ("line N: ...", errors.py:8-13).
//
// Lines are split across threads (std::thread): every thread parses whole records
// of its byte range, the earliest error in file order wins, and the per-thread
// record lists are concatenated in order before the stable sort.  Text is taken as
// UTF-8 bytes; numbers follow CPython's float() / int() on ASCII text (whitespace,
// sign, '_' between digits, inf / nan); integers must fit in 64 bits.
//
// The binary SoA format (.bst) stores the parsed arrays (and optionally a token
// store) for direct loads into pinned memory: a 64-byte header then the arrays,
// each padded to 64 bytes.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "bucketserve.h"

namespace {

struct Rec {
  double arrival;
  int64_t input;
  int64_t output;  // -1: missing (None)
  uint8_t cls;     // 0 online, 1 offline
};

struct Err {
  int64_t line = -1;  // 1-based; -1 = none
  std::string msg;
};

// ---- CPython-compatible scalar parsing ------------------------------------------------
inline bool is_space(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f';
}

std::string strip(const std::string& s) {
  size_t a = 0, b = s.size();
  while (a < b && is_space((unsigned char)s[a])) ++a;
  while (b > a && is_space((unsigned char)s[b - 1])) --b;
  return s.substr(a, b - a);
}

// digits with single underscores between digits (PEP 515); returns the digits
bool take_digits(const std::string& s, size_t& i, std::string& out) {
  const size_t start = i;
  while (i < s.size()) {
    if (s[i] >= '0' && s[i] <= '9') {
      out.push_back(s[i++]);
    } else if (s[i] == '_' && i > start && i + 1 < s.size() && s[i - 1] != '_' &&
               s[i + 1] >= '0' && s[i + 1] <= '9') {
      ++i;
    } else {
      break;
    }
  }
  return i > start;
}

// int(text) for base-10 text
bool py_int(const std::string& text, int64_t& v) {
  const std::string s = strip(text);
  size_t i = 0;
  bool neg = false;
  if (i < s.size() && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
  std::string d;
  if (!take_digits(s, i, d) || i != s.size()) return false;
  errno = 0;
  char* end = nullptr;
  const unsigned long long u = strtoull(d.c_str(), &end, 10);
  if (errno == ERANGE || u > (unsigned long long)INT64_MAX) return false;  // beyond int64
  v = neg ? -(int64_t)u : (int64_t)u;
  return true;
}

// float(text)
bool py_float(const std::string& text, double& v) {
  const std::string s = strip(text);
  size_t i = 0;
  std::string t;
  if (i < s.size() && (s[i] == '+' || s[i] == '-')) t.push_back(s[i++]);
  std::string rest = s.substr(i);
  std::string low;
  for (char c : rest) low.push_back((char)tolower((unsigned char)c));
  if (low == "inf" || low == "infinity") {
    v = (t == "-") ? -INFINITY : INFINITY;
    return true;
  }
  if (low == "nan") {
    v = NAN;
    return true;
  }
  bool any = take_digits(s, i, t);
  if (i < s.size() && s[i] == '.') {
    t.push_back(s[i++]);
    if (i < s.size() && s[i] >= '0' && s[i] <= '9') any = take_digits(s, i, t) || any;
  }
  if (!any) return false;
  if (i < s.size() && (s[i] == 'e' || s[i] == 'E')) {
    t.push_back('e');
    ++i;
    if (i < s.size() && (s[i] == '+' || s[i] == '-')) t.push_back(s[i++]);
    if (!take_digits(s, i, t)) return false;
  }
  if (i != s.size()) return false;
  v = strtod(t.c_str(), nullptr);  // correctly rounded, as CPython
  return true;
}

// repr() of a str (ASCII escapes as CPython; other bytes kept)
std::string py_repr(const std::string& s) {
  const bool has_sq = s.find('\'') != std::string::npos;
  const bool has_dq = s.find('"') != std::string::npos;
  const char q = (has_sq && !has_dq) ? '"' : '\'';
  std::string o(1, q);
  for (unsigned char c : s) {
    if (c == (unsigned char)q || c == '\\') { o.push_back('\\'); o.push_back((char)c); }
    else if (c == '\t') o += "\\t";
    else if (c == '\n') o += "\\n";
    else if (c == '\r') o += "\\r";
    else if (c < 0x20 || c == 0x7f) {
      char b[8];
      snprintf(b, sizeof b, "\\x%02x", c);
      o += b;
    } else {
      o.push_back((char)c);
    }
  }
  o.push_back(q);
  return o;
}

bool parse_class(const std::string& text, uint8_t& c) {
  std::string t = strip(text);
  for (auto& ch : t) ch = (char)tolower((unsigned char)ch);
  if (t == "online") { c = 0; return true; }
  if (t == "offline") { c = 1; return true; }
  return false;
}

// ---- CSV (csv.reader, excel dialect) ------------------------------------------------------
// Reads one record starting at p; advances p and the physical line counter.
// Returns false at end of input.
bool csv_record(const char*& p, const char* end, int64_t& line, std::vector<std::string>& row) {
  row.clear();
  if (p >= end) return false;
  ++line;
  std::string field;
  bool in_q = false, was_q = false, any = false;
  while (p < end) {
    const char c = *p;
    if (in_q) {
      ++p;
      if (c == '"') {
        if (p < end && *p == '"') { field.push_back('"'); ++p; }
        else in_q = false;
      } else {
        if (c == '\n') ++line;
        field.push_back(c);
      }
      continue;
    }
    if (c == '\n' || c == '\r') {
      ++p;
      if (c == '\r' && p < end && *p == '\n') ++p;
      break;
    }
    ++p;
    any = true;
    if (c == ',') {
      row.push_back(field);
      field.clear();
      was_q = false;
    } else if (c == '"' && field.empty() && !was_q) {
      in_q = was_q = true;
    } else {
      field.push_back(c);
    }
  }
  if (any || !field.empty() || was_q) row.push_back(field);
  return true;
}

bool csv_row_to_rec(const std::vector<std::string>& row, int64_t line, Rec& r, Err& err,
                    bool& skip) {
  skip = false;
  bool blank = true;
  for (const auto& c : row) if (!strip(c).empty()) { blank = false; break; }
  if (row.empty() || blank) { skip = true; return true; }
  if (strip(row[0]) == "arrival_s") { skip = true; return true; }
  auto fail = [&](const std::string& m) { err.line = line; err.msg = m; return false; };
  if (row.size() != 4) return fail("expected 4 fields, got " + std::to_string(row.size()));
  if (!py_float(row[0], r.arrival)) return fail("arrival_s is not a number: " + py_repr(row[0]));
  if (!py_int(row[1], r.input)) return fail("input_tokens is not an integer: " + py_repr(row[1]));
  const std::string out = strip(row[2]);
  if (!out.empty()) {
    if (!py_int(out, r.output)) return fail("output_tokens is not an integer: " + py_repr(row[2]));
  } else {
    r.output = -1;
  }
  if (!parse_class(row[3], r.cls))
    return fail("class must be online or offline, got " + py_repr(row[3]));
  if (r.input < 1) return fail("input_tokens must be >= 1, got " + std::to_string(r.input));
  if (r.output != -1 && r.output < 1)
    return fail("output_tokens must be >= 1, got " + std::to_string(r.output));
  return true;
}

// ---- JSON (json.loads) --------------------------------------------------------------------
enum JType { J_NONE, J_NULL, J_BOOL, J_INT, J_FLOAT, J_STR, J_ARR, J_OBJ };

struct JVal {
  JType t = J_NONE;
  int64_t i = 0;
  double d = 0;
  bool big = false;  // integer beyond int64
  std::string s;
};

struct JParser {
  const char* b;
  const char* p;
  const char* e;
  std::string err;
  int64_t pos() const { return p - b; }
  void ws() { while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p; }
  bool fail(const std::string& m) { if (err.empty()) err = m; return false; }
  bool lit(const char* w) {
    const size_t n = strlen(w);
    if ((size_t)(e - p) >= n && memcmp(p, w, n) == 0) { p += n; return true; }
    return false;
  }
  bool string(std::string& out) {  // p at the opening quote
    const char* start = p;
    ++p;
    while (p < e) {
      const char c = *p++;
      if (c == '"') return true;
      if (c == '\\') {
        if (p >= e) break;
        const char x = *p++;
        switch (x) {
          case '"': out.push_back('"'); break;
          case '\\': out.push_back('\\'); break;
          case '/': out.push_back('/'); break;
          case 'b': out.push_back('\b'); break;
          case 'f': out.push_back('\f'); break;
          case 'n': out.push_back('\n'); break;
          case 'r': out.push_back('\r'); break;
          case 't': out.push_back('\t'); break;
          case 'u': {
            if (e - p < 4) { p = start; return fail("Invalid \\uXXXX escape"); }
            unsigned cp = 0;
            for (int k = 0; k < 4; ++k) {
              const char h = *p++;
              cp <<= 4;
              if (h >= '0' && h <= '9') cp |= h - '0';
              else if (h >= 'a' && h <= 'f') cp |= h - 'a' + 10;
              else if (h >= 'A' && h <= 'F') cp |= h - 'A' + 10;
              else { p = start; return fail("Invalid \\uXXXX escape"); }
            }
            if (cp < 0x80) out.push_back((char)cp);
            else if (cp < 0x800) { out.push_back((char)(0xc0 | (cp >> 6))); out.push_back((char)(0x80 | (cp & 63))); }
            else { out.push_back((char)(0xe0 | (cp >> 12))); out.push_back((char)(0x80 | ((cp >> 6) & 63))); out.push_back((char)(0x80 | (cp & 63))); }
            break;
          }
          default: p = start; return fail("Invalid \\escape");
        }
      } else if ((unsigned char)c < 0x20) {
        p = start;
        return fail("Invalid control character at");
      } else {
        out.push_back(c);
      }
    }
    p = start;
    return fail("Unterminated string starting at");
  }
  bool number(JVal& v) {
    const char* s = p;
    if (p < e && *p == '-') ++p;
    if (p < e && *p == '0') ++p;
    else if (p < e && *p >= '1' && *p <= '9') { while (p < e && *p >= '0' && *p <= '9') ++p; }
    else { p = s; return fail("Expecting value"); }
    bool flt = false;
    if (p + 1 < e && *p == '.' && p[1] >= '0' && p[1] <= '9') {
      flt = true;
      p += 2;
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    if (p < e && (*p == 'e' || *p == 'E')) {
      const char* q = p + 1;
      if (q < e && (*q == '+' || *q == '-')) ++q;
      if (q < e && *q >= '0' && *q <= '9') {
        flt = true;
        p = q;
        while (p < e && *p >= '0' && *p <= '9') ++p;
      }
    }
    const std::string t(s, p);
    v.d = strtod(t.c_str(), nullptr);
    if (flt) {
      v.t = J_FLOAT;
    } else {
      v.t = J_INT;
      errno = 0;
      v.i = strtoll(t.c_str(), nullptr, 10);
      v.big = errno == ERANGE;
    }
    return true;
  }
  bool value(JVal& v, int depth) {
    ws();
    if (p >= e) return fail("Expecting value");
    const char c = *p;
    if (c == '"') { v.t = J_STR; return string(v.s); }
    if (c == '{') return object(nullptr, depth + 1, &v);
    if (c == '[') {
      ++p;
      v.t = J_ARR;
      ws();
      if (p < e && *p == ']') { ++p; return true; }
      for (;;) {
        JVal x;
        if (!value(x, depth + 1)) return false;
        ws();
        if (p < e && *p == ',') { ++p; continue; }
        if (p < e && *p == ']') { ++p; return true; }
        return fail("Expecting ',' delimiter");
      }
    }
    if (c == 'n' && lit("null")) { v.t = J_NULL; return true; }
    if (c == 't' && lit("true")) { v.t = J_BOOL; return true; }
    if (c == 'f' && lit("false")) { v.t = J_BOOL; return true; }
    if (c == 'N' && lit("NaN")) { v.t = J_FLOAT; v.d = NAN; return true; }
    if (c == 'I' && lit("Infinity")) { v.t = J_FLOAT; v.d = INFINITY; return true; }
    if (c == '-' && lit("-Infinity")) { v.t = J_FLOAT; v.d = -INFINITY; return true; }
    return number(v);
  }
  // object at p ('{'); the top-level call collects the members into `keys`
  bool object(std::vector<std::pair<std::string, JVal>>* keys, int depth, JVal* self) {
    if (self) self->t = J_OBJ;
    ++p;
    ws();
    if (p < e && *p == '}') { ++p; return true; }
    for (;;) {
      ws();
      if (p >= e || *p != '"') return fail("Expecting property name enclosed in double quotes");
      std::string k;
      if (!string(k)) return false;
      ws();
      if (p >= e || *p != ':') return fail("Expecting ':' delimiter");
      ++p;
      JVal v;
      if (!value(v, depth)) return false;
      if (keys) {
        bool found = false;
        for (auto& kv : *keys) if (kv.first == k) { kv.second = v; found = true; }  // last wins
        if (!found) keys->emplace_back(k, v);
      }
      ws();
      if (p < e && *p == ',') {
        ++p;
        ws();
        if (p >= e || *p != '"') return fail("Expecting property name enclosed in double quotes");
        continue;
      }
      if (p < e && *p == '}') { ++p; return true; }
      return fail("Expecting ',' delimiter");
    }
  }
};

bool jsonl_line_to_rec(const char* b, const char* e, int64_t line, Rec& r, Err& err, bool& skip) {
  skip = false;
  {
    const char* q = b;
    while (q < e && is_space((unsigned char)*q)) ++q;
    if (q == e) { skip = true; return true; }
  }
  auto fail = [&](const std::string& m) { err.line = line; err.msg = m; return false; };
  JParser jp{b, b, e, {}};
  jp.ws();
  std::vector<std::pair<std::string, JVal>> keys;
  JVal top;
  bool ok;
  bool is_obj = jp.p < e && *jp.p == '{';
  if (is_obj) ok = jp.object(&keys, 1, &top);
  else ok = jp.value(top, 0);
  if (ok) {
    jp.ws();
    if (jp.p != e) { jp.err = "Extra data"; ok = false; }
  }
  if (!ok) return fail("invalid JSON: " + jp.err);
  if (!is_obj) return fail("each line must be a JSON object");
  std::vector<std::string> unknown;
  for (auto& kv : keys)
    if (kv.first != "arrival_s" && kv.first != "input_tokens" && kv.first != "output_tokens" &&
        kv.first != "class")
      unknown.push_back(kv.first);
  if (!unknown.empty()) {
    std::sort(unknown.begin(), unknown.end());
    return fail("unknown key " + py_repr(unknown[0]));
  }
  auto get = [&](const char* k) -> const JVal* {
    for (auto& kv : keys) if (kv.first == k) return &kv.second;
    return nullptr;
  };
  for (const char* k : {"arrival_s", "input_tokens", "class"})
    if (!get(k)) return fail(std::string("missing key '") + k + "'");
  const JVal* a = get("arrival_s");
  if (a->t != J_INT && a->t != J_FLOAT) return fail("arrival_s must be a number");
  r.arrival = a->d;  // float(int) for integers (exact below 2^53, correctly rounded above)
  const JVal* in = get("input_tokens");
  if (in->t != J_INT) return fail("input_tokens must be an integer");
  if (in->big) return fail("input_tokens must fit in 64 bits");
  r.input = in->i;
  const JVal* out = get("output_tokens");
  r.output = -1;
  if (out && out->t != J_NULL) {
    if (out->t != J_INT) return fail("output_tokens must be an integer");
    if (out->big) return fail("output_tokens must fit in 64 bits");
    r.output = out->i;
  }
  const JVal* c = get("class");
  if (c->t != J_STR) return fail("class must be a string");
  if (!parse_class(c->s, r.cls)) return fail("class must be online or offline, got " + py_repr(c->s));
  if (r.input < 1) return fail("input_tokens must be >= 1, got " + std::to_string(r.input));
  if (r.output != -1 && r.output < 1)
    return fail("output_tokens must be >= 1, got " + std::to_string(r.output));
  return true;
}

// ---- chunked parallel parse -----------------------------------------------------------------
struct Chunk {
  const char* b;
  const char* e;
  int64_t first_line;  // physical line number of the chunk's first line
  std::vector<Rec> recs;
  Err err;
};

int64_t count_lines(const char* b, const char* e) {
  int64_t n = 0;
  for (const char* q = b; q < e; ++q) n += *q == '\n';
  return n;
}

// ---- CSV fast path ---------------------------------------------------------------------------
// A line of plain fields — digits / '.' / 'e' / sign only in the numbers, a bare class
// word, no quotes, whitespace or underscores — is parsed in place; anything else (and
// every error) goes through the exact CPython-semantics path above.
inline bool fast_uint(const char* b, const char* e, int64_t& v) {
  if (b >= e || e - b > 18) return false;
  int64_t x = 0;
  for (const char* q = b; q < e; ++q) {
    if (*q < '0' || *q > '9') return false;
    x = x * 10 + (*q - '0');
  }
  v = x;
  return true;
}

inline bool fast_float(const char* b, const char* e, double& v) {
  if (b >= e || e - b > 40) return false;
  char buf[48];
  for (const char* q = b; q < e; ++q) {
    const char c = *q;
    if (!((c >= '0' && c <= '9') || c == '.' || c == 'e' || c == 'E' || c == '-' || c == '+'))
      return false;
  }
  const size_t n = (size_t)(e - b);
  memcpy(buf, b, n);
  buf[n] = 0;
  char* end = nullptr;
  v = strtod(buf, &end);
  return end == buf + n;
}

// returns 1 parsed, 0 not a fast line (caller falls back); p advanced past the line
inline int csv_fast_line(const char*& p, const char* e, Rec& r) {
  const char* le = (const char*)memchr(p, '\n', (size_t)(e - p));
  const char* end = le ? le : e;
  const char* stop = end;
  if (stop > p && stop[-1] == '\r') --stop;
  const char* f[5];
  int nf = 0;
  f[nf++] = p;
  for (const char* q = p; q < stop; ++q) {
    const char c = *q;
    if (c == '"') return 0;
    if (c == ',') {
      if (nf == 4) return 0;
      f[nf++] = q + 1;
    }
  }
  if (nf != 4) return 0;
  const char* fe[4] = {f[1] - 1, f[2] - 1, f[3] - 1, stop};
  if (!fast_float(f[0], fe[0], r.arrival)) return 0;
  if (!fast_uint(f[1], fe[1], r.input) || r.input < 1) return 0;
  if (f[2] == fe[2]) r.output = -1;
  else if (!fast_uint(f[2], fe[2], r.output) || r.output < 1) return 0;
  const size_t cl = (size_t)(fe[3] - f[3]);
  if (cl == 6 && memcmp(f[3], "online", 6) == 0) r.cls = 0;
  else if (cl == 7 && memcmp(f[3], "offline", 7) == 0) r.cls = 1;
  else return 0;
  p = le ? le + 1 : e;
  return 1;
}

void parse_chunk(Chunk& c, int fmt) {
  if (fmt == 0) {
    const char* p = c.b;
    int64_t line = c.first_line - 1;
    std::vector<std::string> row;
    while (p < c.e) {
      Rec r{};
      if (csv_fast_line(p, c.e, r)) {
        ++line;
        c.recs.push_back(r);
        continue;
      }
      if (!csv_record(p, c.e, line, row)) break;
      bool skip;
      // errors cite csv.reader.line_num: the record's last physical line
      if (!csv_row_to_rec(row, line, r, c.err, skip)) return;
      if (!skip) c.recs.push_back(r);
    }
  } else {
    const char* p = c.b;
    int64_t line = c.first_line;
    while (p < c.e) {
      const char* q = (const char*)memchr(p, '\n', (size_t)(c.e - p));
      const char* le = q ? q + 1 : c.e;  // json.loads sees the line with its newline
      Rec r{};
      bool skip;
      if (!jsonl_line_to_rec(p, le, line, r, c.err, skip)) return;
      if (!skip) c.recs.push_back(r);
      ++line;
      p = q ? q + 1 : c.e;
    }
  }
}

// CSV quotes may hide newlines: a chunk boundary is only safe where the number of
// quote characters before it is even (fields open and close their quotes).
std::vector<const char*> split_points(const char* b, const char* e, int parts, int fmt) {
  std::vector<const char*> cut{b};
  const int64_t len = e - b;
  for (int k = 1; k < parts; ++k) {
    const char* t = b + len * k / parts;
    if (t <= cut.back()) continue;
    const char* q = (const char*)memchr(t, '\n', (size_t)(e - t));
    if (!q) break;
    cut.push_back(q + 1);
  }
  cut.push_back(e);
  if (fmt == 0) {  // drop cuts inside quoted fields
    std::vector<const char*> ok{b};
    int64_t quotes = 0;
    const char* scan = b;
    for (size_t k = 1; k + 1 < cut.size(); ++k) {
      for (; scan < cut[k]; ++scan) quotes += *scan == '"';
      if ((quotes & 1) == 0) ok.push_back(cut[k]);
    }
    ok.push_back(e);
    cut.swap(ok);
  }
  return cut;
}

}  // namespace

extern "C" {

int bs_trace_parse(const char* text, int64_t len, int32_t format, int32_t threads,
                   bs_trace* out) {
  if (!out) return BS_ERR_INVALID_ARG;
  memset(out, 0, sizeof(*out));
  out->err_line = -1;
  if ((!text && len > 0) || len < 0 || (format != BS_TRACE_CSV && format != BS_TRACE_JSONL))
    return BS_ERR_INVALID_ARG;
  const char* b = text;
  const char* e = text + len;
  int parts = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  if (parts < 1) parts = 1;
  if (len < ((int64_t)1 << 20)) parts = 1;
  const auto cuts = split_points(b, e, parts, format);
  std::vector<Chunk> chunks(cuts.size() - 1);
  int64_t line = 1;
  for (size_t k = 0; k < chunks.size(); ++k) {
    chunks[k].b = cuts[k];
    chunks[k].e = cuts[k + 1];
    chunks[k].first_line = line;
    line += count_lines(cuts[k], cuts[k + 1]);
  }
  if (chunks.size() == 1) {
    parse_chunk(chunks[0], format);
  } else {
    std::vector<std::thread> pool;
    for (auto& c : chunks) pool.emplace_back(parse_chunk, std::ref(c), (int)format);
    for (auto& t : pool) t.join();
  }
  for (auto& c : chunks) {
    if (c.err.line >= 0) {  // the first malformed record in file order
      out->err_line = c.err.line;
      snprintf(out->err_msg, sizeof out->err_msg, "line %lld: %s", (long long)c.err.line,
               c.err.msg.c_str());
      return BS_ERR_CONFIG;
    }
  }
  int64_t n = 0;
  for (auto& c : chunks) n += (int64_t)c.recs.size();
  std::vector<Rec> all;
  all.reserve((size_t)n);
  for (auto& c : chunks) all.insert(all.end(), c.recs.begin(), c.recs.end());
  // ids follow file order; stable sort by arrival (load_trace, workload.py:426)
  std::vector<int64_t> order((size_t)n);
  std::iota(order.begin(), order.end(), 0);
  bool sorted = true;  // traces are usually written in arrival order: skip the sort then
  for (int64_t i = 1; i < n && sorted; ++i) sorted = !(all[(size_t)i].arrival < all[(size_t)i - 1].arrival);
  if (!sorted)
    std::stable_sort(order.begin(), order.end(),
                     [&](int64_t x, int64_t y) { return all[x].arrival < all[y].arrival; });
  out->n = n;
  const size_t nn = (size_t)(n > 0 ? n : 1);
  out->id = (int64_t*)malloc(sizeof(int64_t) * nn);
  out->arrival = (double*)malloc(sizeof(double) * nn);
  out->input_len = (int64_t*)malloc(sizeof(int64_t) * nn);
  out->output_len = (int64_t*)malloc(sizeof(int64_t) * nn);
  out->cls = (uint8_t*)malloc(nn);
  if (!out->id || !out->arrival || !out->input_len || !out->output_len || !out->cls) {
    bs_trace_free(out);
    return BS_ERR_CAPACITY;
  }
  for (int64_t i = 0; i < n; ++i) {
    const Rec& r = all[(size_t)order[(size_t)i]];
    out->id[i] = order[(size_t)i];
    out->arrival[i] = r.arrival;
    out->input_len[i] = r.input;
    out->output_len[i] = r.output;
    out->cls[i] = r.cls;
  }
  return BS_OK;
}

void bs_trace_free(bs_trace* t) {
  if (!t) return;
  free(t->id);
  free(t->arrival);
  free(t->input_len);
  free(t->output_len);
  free(t->cls);
  t->id = nullptr;
  t->arrival = nullptr;
  t->input_len = t->output_len = nullptr;
  t->cls = nullptr;
  t->n = 0;
}

static const char kBstMagic[8] = {'B', 'S', 'T', 'R', 'A', 'C', 'E', '1'};

int bs_trace_write_bst(const char* path, const bs_trace* t) {
  if (!path || !t || t->n < 0) return BS_ERR_INVALID_ARG;
  FILE* f = fopen(path, "wb");
  if (!f) return BS_ERR_INVALID_ARG;
  unsigned char hdr[64] = {0};
  memcpy(hdr, kBstMagic, 8);
  memcpy(hdr + 8, &t->n, 8);
  bool ok = fwrite(hdr, 1, 64, f) == 64;
  const unsigned char zero[64] = {0};
  auto put = [&](const void* p, size_t bytes) {
    if (bytes && fwrite(p, 1, bytes, f) != bytes) ok = false;
    const size_t pad = (64 - bytes % 64) % 64;
    if (pad && fwrite(zero, 1, pad, f) != pad) ok = false;
  };
  const size_t n = (size_t)t->n;
  put(t->id, 8 * n);
  put(t->arrival, 8 * n);
  put(t->input_len, 8 * n);
  put(t->output_len, 8 * n);
  put(t->cls, n);
  ok = (fclose(f) == 0) && ok;
  return ok ? BS_OK : BS_ERR_INVALID_ARG;
}

int bs_trace_read_bst(const char* path, bs_trace* out) {
  if (!path || !out) return BS_ERR_INVALID_ARG;
  memset(out, 0, sizeof(*out));
  out->err_line = -1;
  FILE* f = fopen(path, "rb");
  if (!f) return BS_ERR_INVALID_ARG;
  unsigned char hdr[64];
  int64_t n = -1;
  if (fread(hdr, 1, 64, f) != 64 || memcmp(hdr, kBstMagic, 8) != 0) { fclose(f); return BS_ERR_CONFIG; }
  memcpy(&n, hdr + 8, 8);
  if (n < 0) { fclose(f); return BS_ERR_CONFIG; }
  const size_t nn = (size_t)(n > 0 ? n : 1);
  out->id = (int64_t*)malloc(8 * nn);
  out->arrival = (double*)malloc(8 * nn);
  out->input_len = (int64_t*)malloc(8 * nn);
  out->output_len = (int64_t*)malloc(8 * nn);
  out->cls = (uint8_t*)malloc(nn);
  bool ok = out->id && out->arrival && out->input_len && out->output_len && out->cls;
  auto get = [&](void* p, size_t bytes) {
    if (ok && bytes && fread(p, 1, bytes, f) != bytes) ok = false;
    const size_t pad = (64 - bytes % 64) % 64;
    if (ok && pad && fseek(f, (long)pad, SEEK_CUR) != 0) ok = false;
  };
  get(out->id, 8 * (size_t)n);
  get(out->arrival, 8 * (size_t)n);
  get(out->input_len, 8 * (size_t)n);
  get(out->output_len, 8 * (size_t)n);
  get(out->cls, (size_t)n);
  fclose(f);
  if (!ok) { bs_trace_free(out); return BS_ERR_CONFIG; }
  out->n = n;
  return BS_OK;
}

}  // extern "C"
