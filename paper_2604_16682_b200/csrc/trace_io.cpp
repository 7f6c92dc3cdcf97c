/*
 * trace_io.cpp — native JSON-lines trace reader: file -> CSR arrays.
 *
 * Format (/root/reference/pkg/src/agentsim/workload.py:11-16, 217-276):
 *   {"agent_id": "a000001", "arrival_time": 12.5, "turns": [[400, 150, 2.0], ...]}
 * one agent per line; unknown fields are ignored; blank lines are skipped.
 *
 * This is the fast path of `load_trace_arrays` (workload.py here).  It
 * accepts the canonical shape that `save_trace` writes and plain JSON
 * variations of it (whitespace, field order, unknown fields with scalar /
 * array / object values, integral token counts written as 400 or 400.0).
 * Anything else — invalid JSON, a missing field, a non-numeric value, a
 * duplicate agent_id, a value the reference's TurnRecord / AgentTrace
 * would reject — is reported with its line number and the Python loader
 * (the reference's exact semantics and error messages) handles the file.
 *
 * Numbers must follow the JSON grammar exactly (RFC 8259 §6: optional '-',
 * no leading zeros, digits on both sides of '.', digits after the exponent;
 * json.loads rejects "1.", ".5", "0400", "+1") and are then converted with
 * std::from_chars, correctly rounded like Python's float(); token counts
 * must be integral and fit in int32 (the engine's layout).
 *
 * The file is read ONCE into a parsed handle; the caller sizes its buffers
 * from the handle's counts and copies out of it, so a file that changes
 * between the two calls cannot overrun anything.
 *
 * C ABI (ctypes, paper_2604_16682_b200/workload.py):
 *   int asb_trace_parse(const char* path, void** handle, int64_t* n_agents,
 *                       int64_t* n_turns, int64_t* id_bytes, int64_t* bad_line);
 *   int asb_trace_copy(const void* handle, double* arrival, int64_t* turn_off,
 *                      int32_t* prefill, int32_t* decode, double* tool,
 *                      char* ids, int64_t* id_off);
 *   void asb_trace_free(void* handle);
 * parse returns 0 ok (handle set), 1 = needs the Python loader (bad_line =
 * 1-based line), -1 I/O; copy returns 0 (or -1 for a NULL handle).
 */
#include <errno.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <charconv>
#include <string>
#include <system_error>
#include <unordered_set>
#include <vector>

namespace {

struct Cursor {
  const char* p;
  const char* end;
  void ws() {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n')) p++;
  }
  bool eat(char c) {
    ws();
    if (p < end && *p == c) {
      p++;
      return true;
    }
    return false;
  }
};

/* JSON string without escapes other than the simple ones; returns false on
 * anything unusual (unicode escapes are left to the Python loader) */
bool parse_string(Cursor& c, std::string* out) {
  c.ws();
  if (c.p >= c.end || *c.p != '"') return false;
  c.p++;
  std::string s;
  while (c.p < c.end && *c.p != '"') {
    char ch = *c.p++;
    if (ch == '\\') {
      if (c.p >= c.end) return false;
      char e = *c.p++;
      switch (e) {
        case '"': ch = '"'; break;
        case '\\': ch = '\\'; break;
        case '/': ch = '/'; break;
        case 'b': ch = '\b'; break;
        case 'f': ch = '\f'; break;
        case 'n': ch = '\n'; break;
        case 'r': ch = '\r'; break;
        case 't': ch = '\t'; break;
        default: return false; /* \uXXXX: Python loader */
      }
    } else if ((unsigned char)ch < 0x20) {
      return false;
    }
    s.push_back(ch);
  }
  if (c.p >= c.end) return false;
  c.p++;
  if (out) *out = s;
  return true;
}

/* JSON number (RFC 8259 §6): -? (0 | [1-9][0-9]*) (. [0-9]+)? ([eE] [+-]? [0-9]+)? */
const char* json_number_end(const char* s, const char* end) {
  if (s < end && *s == '-') s++;
  if (s >= end || *s < '0' || *s > '9') return nullptr;
  if (*s == '0') {
    s++;
  } else {
    while (s < end && *s >= '0' && *s <= '9') s++;
  }
  if (s < end && *s == '.') {
    s++;
    if (s >= end || *s < '0' || *s > '9') return nullptr;
    while (s < end && *s >= '0' && *s <= '9') s++;
  }
  if (s < end && (*s == 'e' || *s == 'E')) {
    s++;
    if (s < end && (*s == '+' || *s == '-')) s++;
    if (s >= end || *s < '0' || *s > '9') return nullptr;
    while (s < end && *s >= '0' && *s <= '9') s++;
  }
  /* "0400" parses as "0" followed by "400": the next token check rejects it */
  if (s < end && ((*s >= '0' && *s <= '9') || *s == '.' || *s == 'e' || *s == 'E' || *s == '+' || *s == '-'))
    return nullptr;
  return s;
}

bool parse_number(Cursor& c, double* v, bool* integral) {
  c.ws();
  const char* s = json_number_end(c.p, c.end);
  if (!s) return false;
  bool frac = false;
  for (const char* q = c.p; q < s; q++)
    if (*q == '.' || *q == 'e' || *q == 'E') frac = true;
  /* correctly rounded (like Python's float()) */
  double x = 0.0;
  const std::from_chars_result r = std::from_chars(c.p, s, x);
  if (r.ptr != s || r.ec != std::errc() || !isfinite(x)) return false;
  if (!frac && x == 0) x = 0.0; /* "-0" is the int 0 in json.loads, float(0) == +0.0 */
  *v = x;
  *integral = !frac;
  c.p = s;
  return true;
}

/* skip any JSON value (for unknown fields) */
bool skip_value(Cursor& c, int depth = 0) {
  if (depth > 64) return false;
  c.ws();
  if (c.p >= c.end) return false;
  char ch = *c.p;
  if (ch == '"') return parse_string(c, nullptr);
  if (ch == '{' || ch == '[') {
    const char close = ch == '{' ? '}' : ']';
    c.p++;
    if (c.eat(close)) return true;
    for (;;) {
      if (ch == '{') {
        if (!parse_string(c, nullptr) || !c.eat(':')) return false;
      }
      if (!skip_value(c, depth + 1)) return false;
      if (c.eat(',')) continue;
      return c.eat(close);
    }
  }
  static const char* lits[] = {"true", "false", "null"};
  for (const char* l : lits) {
    size_t n = strlen(l);
    if ((size_t)(c.end - c.p) >= n && !strncmp(c.p, l, n)) {
      c.p += n;
      return true;
    }
  }
  double v;
  bool integral;
  return parse_number(c, &v, &integral);
}

struct Agent {
  std::string id;
  double arrival;
  std::vector<int32_t> pre, dec;
  std::vector<double> tool;
};

/* one line -> agent; false = not the fast-path shape or a value the
 * reference rejects (the Python loader then reports it) */
bool parse_line(const char* b, const char* e, Agent* a) {
  Cursor c{b, e};
  if (!c.eat('{')) return false;
  bool has_id = false, has_arr = false, has_turns = false;
  a->pre.clear();
  a->dec.clear();
  a->tool.clear();
  if (!c.eat('}')) {
    for (;;) {
      std::string key;
      if (!parse_string(c, &key) || !c.eat(':')) return false;
      if (key == "agent_id") {
        if (!parse_string(c, &a->id)) return false;
        has_id = true;
      } else if (key == "arrival_time") {
        bool integral;
        if (!parse_number(c, &a->arrival, &integral)) return false;
        has_arr = true;
      } else if (key == "turns") {
        a->pre.clear(); /* a repeated key keeps the last value, like json.loads */
        a->dec.clear();
        a->tool.clear();
        if (!c.eat('[')) return false;
        if (!c.eat(']')) {
          for (;;) {
            double v[3];
            bool integral[3];
            if (!c.eat('[')) return false;
            for (int k = 0; k < 3; k++) {
              if (k && !c.eat(',')) return false;
              if (!parse_number(c, &v[k], &integral[k])) return false;
            }
            if (!c.eat(']')) return false;
            /* TurnRecord(int(p), int(d), float(t)): counts integral, >= 1, int32 */
            for (int k = 0; k < 2; k++)
              if (v[k] != floor(v[k]) || v[k] < 1 || v[k] > 2147483647.0) return false;
            if (!(v[2] >= 0)) return false;
            a->pre.push_back((int32_t)v[0]);
            a->dec.push_back((int32_t)v[1]);
            a->tool.push_back(v[2]);
            if (c.eat(',')) continue;
            if (!c.eat(']')) return false;
            break;
          }
        }
        has_turns = true;
      } else {
        if (!skip_value(c)) return false;
      }
      if (c.eat(',')) continue;
      if (!c.eat('}')) return false;
      break;
    }
  }
  c.ws();
  if (c.p != c.end) return false;
  /* AgentTrace: non-empty id, arrival >= 0, at least one turn */
  return has_id && has_arr && has_turns && !a->id.empty() && a->arrival >= 0 && !a->pre.empty();
}

struct File {
  std::vector<char> buf;
  bool read(const char* path) {
    FILE* f = fopen(path, "rb");
    if (!f) return false;
    fseek(f, 0, SEEK_END);
    long n = ftell(f);
    fseek(f, 0, SEEK_SET);
    buf.resize((n > 0 ? (size_t)n : 0) + 1);
    size_t got = n > 0 ? fread(buf.data(), 1, (size_t)n, f) : 0;
    fclose(f);
    buf[got] = 0; /* strtod may look one past a number at the very end */
    return got == buf.size() - 1;
  }
};

/* walk the file line by line; fn(agent_index, agent) for every agent */
template <class Fn>
int walk(const char* path, int64_t* bad_line, Fn fn) {
  File f;
  if (!f.read(path)) return -1;
  const char* p = f.buf.data();
  const char* end = p + f.buf.size() - 1;
  int64_t lineno = 0, idx = 0;
  Agent a;
  std::unordered_set<std::string> seen;
  while (p < end) {
    const char* nl = (const char*)memchr(p, '\n', (size_t)(end - p));
    const char* le = nl ? nl : end;
    lineno++;
    const char* b = p;
    while (b < le && (*b == ' ' || *b == '\t' || *b == '\r')) b++;
    const char* e = le;
    while (e > b && (e[-1] == ' ' || e[-1] == '\t' || e[-1] == '\r')) e--;
    if (b < e) {
      if (!parse_line(b, e, &a) || !seen.insert(a.id).second) {
        *bad_line = lineno;
        return 1;
      }
      fn(idx++, a);
    }
    p = nl ? nl + 1 : end;
  }
  return 0;
}

/* the whole file, parsed once */
struct Parsed {
  std::vector<double> arrival, tool;
  std::vector<int64_t> turn_off, id_off;
  std::vector<int32_t> pre, dec;
  std::string ids;
};

}  // namespace

extern "C" {

int asb_trace_parse(const char* path, void** handle, int64_t* n_agents, int64_t* n_turns, int64_t* id_bytes,
                    int64_t* bad_line) {
  *handle = nullptr;
  *bad_line = 0;
  Parsed* P = new Parsed();
  P->turn_off.push_back(0);
  P->id_off.push_back(0);
  const int rc = walk(path, bad_line, [&](int64_t, const Agent& a) {
    P->arrival.push_back(a.arrival);
    P->pre.insert(P->pre.end(), a.pre.begin(), a.pre.end());
    P->dec.insert(P->dec.end(), a.dec.begin(), a.dec.end());
    P->tool.insert(P->tool.end(), a.tool.begin(), a.tool.end());
    P->turn_off.push_back((int64_t)P->pre.size());
    P->ids += a.id;
    P->id_off.push_back((int64_t)P->ids.size());
  });
  if (rc != 0) {
    delete P;
    return rc;
  }
  *n_agents = (int64_t)P->arrival.size();
  *n_turns = (int64_t)P->pre.size();
  *id_bytes = (int64_t)P->ids.size();
  *handle = P;
  return 0;
}

int asb_trace_copy(const void* handle, double* arrival, int64_t* turn_off, int32_t* prefill, int32_t* decode,
                   double* tool, char* ids, int64_t* id_off) {
  const Parsed* P = static_cast<const Parsed*>(handle);
  if (!P) return -1;
  const size_t na = P->arrival.size(), nt = P->pre.size();
  memcpy(arrival, P->arrival.data(), na * 8);
  memcpy(turn_off, P->turn_off.data(), (na + 1) * 8);
  memcpy(prefill, P->pre.data(), nt * 4);
  memcpy(decode, P->dec.data(), nt * 4);
  memcpy(tool, P->tool.data(), nt * 8);
  memcpy(ids, P->ids.data(), P->ids.size());
  memcpy(id_off, P->id_off.data(), (na + 1) * 8);
  return 0;
}

void asb_trace_free(void* handle) { delete static_cast<Parsed*>(handle); }

}  // extern "C"
