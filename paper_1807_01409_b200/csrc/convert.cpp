// N-Triples -> TripleID conversion on the host cores:
// the reference's cmd_convert (cli.py:64-114) = nt.parse_stream (nt.py:196-224)
// + Dictionary.encode in first-occurrence order (dictionary.py:71-80)
// + write_tid (store.py:97-104) + write_id_files (dictionary.py:98-107).
//
// String work stays on the host (north star); this is its native, parallel
// form.  Output files are byte-identical to the reference's:
//   1. the input is read into memory by T threads (pread);
//   2. it is cut at line boundaries into T chunks; each thread parses its
//      lines exactly as nt.parse_line/_parse_term (UTF-8 validated as Python's
//      strict decoder, language tags scanned with Python's str.isalnum table)
//      and encodes terms into a chunk-local dictionary in local
//      first-occurrence order;
//   3. one sequential merge walks the chunks in order and assigns global IDs
//      to terms not seen in earlier chunks, in each chunk's local order —
//      which is the global first-occurrence order the reference assigns;
//   4. threads remap the local triples to global IDs and format the three
//      role files (ascending ID, "<id>\t<term>\n").
// Lenient mode skips malformed lines and reports them; strict mode stops at
// the first malformed line in stream order and writes nothing.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cerrno>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "internal.cuh"
#include "unicode_tables.h"

namespace tidq {
namespace convert {

// ---- Python semantics helpers ----------------------------------------------------

static bool in_ranges(const uint32_t (*r)[2], int n, uint32_t cp) {
  int lo = 0, hi = n - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) / 2;
    if (cp < r[mid][0]) hi = mid - 1;
    else if (cp > r[mid][1]) lo = mid + 1;
    else return true;
  }
  return false;
}

static bool py_isalnum(uint32_t cp) {
  if (cp < 0x80) return (cp >= '0' && cp <= '9') || (cp >= 'a' && cp <= 'z') || (cp >= 'A' && cp <= 'Z');
  return in_ranges(kIsAlnum, kIsAlnum_n, cp);
}

static bool py_isprintable(uint32_t cp) {
  if (cp < 0x80) return cp >= 0x20 && cp < 0x7F;
  return in_ranges(kIsPrintable, kIsPrintable_n, cp);
}

// Decode the code point at p (valid UTF-8 guaranteed by the line check).
static uint32_t decode_cp(const unsigned char* p, int* len) {
  const uint32_t c = p[0];
  if (c < 0x80) { *len = 1; return c; }
  if (c < 0xE0) { *len = 2; return ((c & 0x1F) << 6) | (p[1] & 0x3F); }
  if (c < 0xF0) { *len = 3; return ((c & 0x0F) << 12) | ((p[1] & 0x3F) << 6) | (p[2] & 0x3F); }
  *len = 4;
  return ((c & 0x07) << 18) | ((p[1] & 0x3F) << 12) | ((p[2] & 0x3F) << 6) | (p[3] & 0x3F);
}

static void append_utf8(std::string& s, uint32_t cp) {
  if (cp < 0x80) s += char(cp);
  else if (cp < 0x800) { s += char(0xC0 | (cp >> 6)); s += char(0x80 | (cp & 0x3F)); }
  else if (cp < 0x10000) {
    s += char(0xE0 | (cp >> 12)); s += char(0x80 | ((cp >> 6) & 0x3F)); s += char(0x80 | (cp & 0x3F));
  } else {
    s += char(0xF0 | (cp >> 18)); s += char(0x80 | ((cp >> 12) & 0x3F));
    s += char(0x80 | ((cp >> 6) & 0x3F)); s += char(0x80 | (cp & 0x3F));
  }
}

// repr() of a one-character str (the {c!r} of nt.py:142).
static std::string py_repr_char(uint32_t cp) {
  const bool dq = cp == '\'';
  std::string s(1, dq ? '"' : '\'');
  char buf[16];
  if (cp == '\\') s += "\\\\";
  else if (cp == '\t') s += "\\t";
  else if (cp == '\n') s += "\\n";
  else if (cp == '\r') s += "\\r";
  else if (py_isprintable(cp)) append_utf8(s, cp);
  else if (cp < 0x100) { snprintf(buf, sizeof buf, "\\x%02x", cp); s += buf; }
  else if (cp < 0x10000) { snprintf(buf, sizeof buf, "\\u%04x", cp); s += buf; }
  else { snprintf(buf, sizeof buf, "\\U%08x", cp); s += buf; }
  s += dq ? '"' : '\'';
  return s;
}

// CPython's strict UTF-8 decoder (Objects/stringlib/codecs.h): returns -1 if
// valid, else the byte index of the failing sequence and its reason.
static int64_t utf8_check(const unsigned char* s, size_t n, const char** reason) {
  size_t i = 0;
  auto cont = [](unsigned char b) { return (b & 0xC0) == 0x80; };
  while (i < n) {
    const unsigned char c = s[i];
    if (c < 0x80) { ++i; continue; }
    if (c < 0xC2 || c > 0xF4) { *reason = "invalid start byte"; return int64_t(i); }
    const size_t need = c < 0xE0 ? 2 : (c < 0xF0 ? 3 : 4);
    const size_t have = std::min(need, n - i);
    for (size_t k = 1; k < have; ++k) {
      const unsigned char b = s[i + k];
      bool ok = cont(b);
      if (ok && k == 1) {
        if (c == 0xE0) ok = b >= 0xA0;
        else if (c == 0xED) ok = b < 0xA0;
        else if (c == 0xF0) ok = b >= 0x90;
        else if (c == 0xF4) ok = b < 0x90;
      }
      if (!ok) { *reason = "invalid continuation byte"; return int64_t(i); }
    }
    if (have < need) { *reason = "unexpected end of data"; return int64_t(i); }
    i += need;
  }
  return -1;
}

// ---- parsing (nt.py:96-193) ------------------------------------------------------

enum Kind : uint8_t { kIri = 0, kLiteral = 1, kBlank = 2 };

struct Tok {
  uint32_t off;  // byte offset within the line
  uint32_t len;
  Kind kind;
};

struct LineError {
  uint64_t line;    // chunk-local line number (0-based), globalised later
  uint64_t offset;  // byte offset
  std::string msg;
};

static inline bool ws(unsigned char c) { return c == ' ' || c == '\t'; }

// nt.py:_parse_term.  Returns false and fills err on a parse error.
static bool parse_term(const unsigned char* L, size_t n, size_t i, Tok* tok, size_t* next, LineError* err) {
  const unsigned char c = L[i];
  if (c == '<') {
    const void* e = memchr(L + i + 1, '>', n - i - 1);
    if (!e) { err->offset = i; err->msg = "unterminated IRI"; return false; }
    const size_t end = size_t(static_cast<const unsigned char*>(e) - L);
    *tok = {uint32_t(i), uint32_t(end + 1 - i), kIri};
    *next = end + 1;
    return true;
  }
  if (c == '"') {
    size_t j = i + 1;
    while (j < n) {
      const unsigned char ch = L[j];
      if (ch == '\\') { j += 2; continue; }
      if (ch == '"') break;
      ++j;
    }
    if (j >= n) { err->offset = i; err->msg = "unterminated literal"; return false; }
    size_t end = j + 1;
    if (end + 3 <= n && L[end] == '^' && L[end + 1] == '^' && L[end + 2] == '<') {
      const void* e = end + 3 < n ? memchr(L + end + 3, '>', n - end - 3) : nullptr;
      if (!e) { err->offset = end; err->msg = "unterminated datatype IRI"; return false; }
      end = size_t(static_cast<const unsigned char*>(e) - L) + 1;
    } else if (end < n && L[end] == '@') {
      size_t k = end + 1;
      while (k < n) {
        int len;
        const uint32_t cp = decode_cp(L + k, &len);
        if (!(py_isalnum(cp) || cp == '-')) break;
        k += len;
      }
      if (k == end + 1) { err->offset = end; err->msg = "empty language tag"; return false; }
      end = k;
    }
    *tok = {uint32_t(i), uint32_t(end - i), kLiteral};
    *next = end;
    return true;
  }
  if (c == '_') {
    if (i + 1 >= n || L[i + 1] != ':') { err->offset = i; err->msg = "malformed blank node"; return false; }
    size_t j = i + 2;
    while (j < n && L[j] != ' ' && L[j] != '\t' && L[j] != '.') ++j;
    if (j == i + 2) { err->offset = i; err->msg = "empty blank node label"; return false; }
    *tok = {uint32_t(i), uint32_t(j - i), kBlank};
    *next = j;
    return true;
  }
  int len;
  err->offset = i;
  err->msg = "unexpected character " + py_repr_char(decode_cp(L + i, &len));
  return false;
}

// nt.py:parse_line: 0 = blank/comment, 1 = statement (toks[0..2]), -1 = error.
static int parse_line(const unsigned char* L, size_t n, Tok toks[4], LineError* err) {
  size_t i = 0;
  while (i < n && ws(L[i])) ++i;
  if (i == n || L[i] == '#') return 0;
  int nt = 0;
  while (true) {
    if (i == n) { err->offset = i; err->msg = "missing terminal '.'"; return -1; }
    if (L[i] == '.') { ++i; break; }
    if (nt == 4) { err->offset = i; err->msg = "too many terms"; return -1; }
    size_t next;
    if (!parse_term(L, n, i, &toks[nt], &next, err)) return -1;
    ++nt;
    i = next;
    while (i < n && ws(L[i])) ++i;
  }
  while (i < n && ws(L[i])) ++i;
  if (i < n && L[i] != '#') { err->offset = i; err->msg = "trailing content after '.'"; return -1; }
  if (nt < 3) { err->offset = 0; err->msg = "expected 3 terms, found " + std::to_string(nt); return -1; }
  if (toks[1].kind != kIri) { err->offset = 0; err->msg = "predicate must be an IRI"; return -1; }
  if (toks[0].kind == kLiteral) { err->offset = 0; err->msg = "subject must not be a literal"; return -1; }
  if (nt == 4 && toks[3].kind == kLiteral) {
    err->offset = 0;
    err->msg = "context term must not be a literal";
    return -1;
  }
  return 1;
}

// ---- term tables -------------------------------------------------------------------

static inline uint64_t hash_bytes(const unsigned char* p, size_t n) {
  uint64_t h = 0x9E3779B97F4A7C15ull ^ (uint64_t(n) * 0xC2B2AE3D27D4EB4Full);
  while (n >= 8) {
    uint64_t v;
    memcpy(&v, p, 8);
    h = (h ^ v) * 0xFF51AFD7ED558CCDull;
    h ^= h >> 32;
    p += 8;
    n -= 8;
  }
  uint64_t v = 0;
  memcpy(&v, p, n);
  h = (h ^ v) * 0xC4CEB9FE1A85EC53ull;
  h ^= h >> 29;
  return h * 0x9E3779B97F4A7C15ull;
}

struct Term {
  const unsigned char* p;
  uint32_t len;
  uint64_t h;
};

// Open addressing (linear probing) from term bytes to a dense index.  A slot
// holds the hash's high 32 bits next to index + 1 (0 = empty), so a probe
// touches the term bytes only on a 32-bit hash match.
struct TermTable {
  std::vector<uint64_t> slot;
  uint64_t mask = 0;
  std::vector<Term> terms;

  static constexpr uint64_t kHi = 0xFFFFFFFF00000000ull;
  void reserve(size_t n) {
    size_t cap = 1024;
    while (cap < 2 * n) cap <<= 1;
    slot.assign(cap, 0);
    mask = cap - 1;
    terms.reserve(n);
  }
  void grow() {
    std::vector<uint64_t> old;
    old.swap(slot);
    slot.assign(old.size() * 2, 0);
    mask = slot.size() - 1;
    for (uint64_t v : old)
      if (v) {
        uint64_t s = terms[uint32_t(v) - 1].h & mask;
        while (slot[s]) s = (s + 1) & mask;
        slot[s] = v;
      }
  }
  // index of the term, inserting it (returns true in *fresh) if new
  uint32_t intern(const unsigned char* p, uint32_t len, uint64_t h, bool* fresh) {
    uint64_t s = h & mask;
    while (const uint64_t v = slot[s]) {
      if (((v ^ h) & kHi) == 0) {
        const Term& t = terms[uint32_t(v) - 1];
        if (t.len == len && memcmp(t.p, p, len) == 0) {
          *fresh = false;
          return uint32_t(v) - 1;
        }
      }
      s = (s + 1) & mask;
    }
    *fresh = true;
    terms.push_back({p, len, h});
    slot[s] = (h & kHi) | uint64_t(terms.size());
    if (terms.size() * 2 > slot.size()) grow();
    return uint32_t(terms.size() - 1);
  }
};

struct Chunk {
  size_t lo = 0, hi = 0;  // byte range of whole lines
  uint64_t lines = 0;     // physical lines in the chunk
  uint64_t skipped = 0;
  TermTable dict;                 // local first-occurrence order
  std::vector<uint8_t> roles;     // role bits per local term
  std::vector<uint32_t> triples;  // local ids, 3 per statement
  std::vector<LineError> errors;  // in line order
  std::vector<uint32_t> remap;    // local -> global id
};

static void parse_chunk(const unsigned char* buf, Chunk& ck, bool strict) {
  ck.dict.reserve(std::max<size_t>(1024, (ck.hi - ck.lo) / 256));
  size_t pos = ck.lo;
  uint64_t ln = 0;
  Tok toks[4];
  while (pos < ck.hi) {
    const void* nl = memchr(buf + pos, '\n', ck.hi - pos);
    const size_t end = nl ? size_t(static_cast<const unsigned char*>(nl) - buf) : ck.hi;
    size_t le = end;
    if (le > pos && buf[le - 1] == '\r') --le;
    const unsigned char* L = buf + pos;
    const size_t n = le - pos;
    LineError err;
    const char* reason = nullptr;
    const int64_t bad = utf8_check(L, n, &reason);
    int r;
    if (bad >= 0) {
      err.offset = uint64_t(bad);
      err.msg = std::string("invalid UTF-8: ") + reason;
      r = -1;
    } else {
      r = parse_line(L, n, toks, &err);
    }
    if (r < 0) {
      err.line = ln;
      ck.errors.push_back(std::move(err));
      if (strict) {
        ck.lines = ln + 1;
        return;  // nothing after the first error of this chunk matters
      }
    } else if (r == 0) {
      ++ck.skipped;
    } else {
      for (int k = 0; k < 3; ++k) {
        const unsigned char* p = L + toks[k].off;
        bool fresh;
        const uint32_t id = ck.dict.intern(p, toks[k].len, hash_bytes(p, toks[k].len), &fresh);
        if (fresh) ck.roles.push_back(0);
        ck.roles[id] |= uint8_t(1u << k);
        ck.triples.push_back(id);
      }
    }
    ++ln;
    pos = end + 1;
  }
  ck.lines = ln;
}

// TIDQ_CONVERT_TRACE=1: per-phase wall times on stderr
struct Trace {
  bool on = getenv("TIDQ_CONVERT_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void operator()(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[convert] %-10s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

template <class F>
static void parallel_for(int T, F&& f) {
  std::vector<std::thread> th;
  for (int t = 1; t < T; ++t) th.emplace_back(f, t);
  f(0);
  for (auto& x : th) x.join();
}

static void io_fail(tidq_convert_report* rep, const std::string& path, int e) {
  rep->io_errno = e;
  snprintf(rep->io_path, sizeof rep->io_path, "%s", path.c_str());
  throw Error(TIDQ_E_IO, path + ": " + strerror(e));
}

static void write_all(int fd, const void* data, size_t n, tidq_convert_report* rep, const std::string& path) {
  const char* p = static_cast<const char*>(data);
  while (n) {
    const ssize_t w = write(fd, p, n);
    if (w < 0) {
      if (errno == EINTR) continue;
      io_fail(rep, path, errno);
    }
    p += w;
    n -= size_t(w);
  }
}

static size_t n_digits(uint32_t v) {
  size_t d = 1;
  while (v >= 10) { v /= 10; ++d; }
  return d;
}

}  // namespace convert
}  // namespace tidq

using namespace tidq;
using namespace tidq::convert;

extern "C" int tidq_convert_nt(const char* input, const char* out_prefix, int strict, int threads,
                               tidq_convert_report* rep, char** errors_tsv) {
  return guarded([&] {
    TIDQ_REQUIRE(input && out_prefix && rep, TIDQ_E_INVALID, "null argument");
    memset(rep, 0, sizeof *rep);
    if (errors_tsv) *errors_tsv = nullptr;
    int T = threads > 0 ? threads : int(std::max(1u, std::thread::hardware_concurrency()));
    Trace trace;
    // ---- read
    const int fd = open(input, O_RDONLY);
    if (fd < 0) io_fail(rep, input, errno);
    struct Fd { int fd; ~Fd() { close(fd); } } fdg{fd};
    struct stat sb;
    if (fstat(fd, &sb) != 0) io_fail(rep, input, errno);
    const size_t size = size_t(sb.st_size);
    std::vector<unsigned char> buf(size + 8);
    {
      std::atomic<int> fail{0};
      const size_t per = (size + T - 1) / std::max(T, 1);
      parallel_for(T, [&](int t) {
        size_t a = size_t(t) * per, b = std::min(size, a + per);
        while (a < b) {
          const ssize_t r = pread(fd, buf.data() + a, b - a, off_t(a));
          if (r <= 0) { fail = r < 0 ? errno : EIO; return; }
          a += size_t(r);
        }
      });
      if (fail) io_fail(rep, input, fail);
    }
    trace("read");
    const unsigned char* B = buf.data();
    // ---- chunks at line boundaries
    if (size < (size_t(1) << 20)) T = 1;
    std::vector<Chunk> ck(T);
    {
      std::vector<size_t> start(T + 1, size);
      start[0] = 0;
      for (int t = 1; t < T; ++t) {
        size_t a = size * size_t(t) / size_t(T);
        const void* nl = memchr(B + a, '\n', size - a);
        start[t] = nl ? size_t(static_cast<const unsigned char*>(nl) - B) + 1 : size;
        start[t] = std::max(start[t], start[t - 1]);
      }
      for (int t = 0; t < T; ++t) {
        ck[t].lo = start[t];
        ck[t].hi = start[t + 1];
      }
    }
    parallel_for(T, [&](int t) { parse_chunk(B, ck[t], strict != 0); });
    trace("parse");
    // ---- line numbers, errors
    std::string errs;
    uint64_t line0 = 1;  // 1-based number of the chunk's first line
    for (int t = 0; t < T; ++t) {
      for (const LineError& e : ck[t].errors) {
        const uint64_t ln = line0 + e.line;
        if (strict) {
          rep->first_error_line = ln;
          rep->first_error_offset = e.offset;
          throw Error(TIDQ_E_PARSE, "line " + std::to_string(ln) + ", byte " + std::to_string(e.offset) + ": " +
                                        e.msg);
        }
        ++rep->parse_errors;
        if (errors_tsv)
          errs += std::to_string(ln) + "\t" + std::to_string(e.offset) + "\t" + e.msg + "\n";
      }
      rep->skipped_lines += ck[t].skipped;
      line0 += ck[t].lines;
    }
    // ---- global dictionary, first-occurrence order (dictionary.py:71-80)
    size_t total_local = 0;
    for (auto& c : ck) total_local += c.dict.terms.size();
    TermTable g;
    g.reserve(std::max<size_t>(total_local / 2, 1024));
    std::vector<uint8_t> groles;
    for (auto& c : ck) {
      c.remap.resize(c.dict.terms.size());
      for (size_t k = 0; k < c.dict.terms.size(); ++k) {
        const Term& tm = c.dict.terms[k];
        bool fresh;
        const uint32_t id = g.intern(tm.p, tm.len, tm.h, &fresh);
        if (fresh) groles.push_back(0);
        groles[id] |= c.roles[k];
        c.remap[k] = id + 1;  // IDs start at 1; 0 is the wildcard
      }
      TIDQ_REQUIRE(g.terms.size() <= 0xFFFFFFFFull, TIDQ_E_INVALID, "cannot assign ID beyond 4294967295");
    }
    const uint64_t n_terms = g.terms.size();
    trace("merge");
    rep->terms = n_terms;
    for (uint64_t k = 0; k < n_terms; ++k)
      for (int r = 0; r < 3; ++r) rep->distinct[r] += (groles[k] >> r) & 1u;
    // ---- .tid (store.py:97-104)
    std::vector<uint64_t> tri0(T + 1, 0);
    for (int t = 0; t < T; ++t) tri0[t + 1] = tri0[t] + ck[t].triples.size() / 3;
    const uint64_t n_tri = tri0[T];
    rep->triples = n_tri;
    std::vector<uint32_t> ids(size_t(n_tri) * 3 + 4);
    memcpy(ids.data(), "TID1", 4);
    ids[1] = 1;
    memcpy(&ids[2], &n_tri, 8);
    parallel_for(T, [&](int t) {
      uint32_t* dst = ids.data() + 4 + tri0[t] * 3;
      const auto& src = ck[t].triples;
      const auto& rm = ck[t].remap;
      for (size_t k = 0; k < src.size(); ++k) dst[k] = rm[src[k]];
      std::vector<uint32_t>().swap(ck[t].triples);
    });
    trace("remap");
    const std::string prefix(out_prefix);
    {
      const std::string path = prefix + ".tid.tmp";
      const int o = open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
      if (o < 0) io_fail(rep, path, errno);
      write_all(o, ids.data(), ids.size() * 4, rep, path);
      close(o);
      rep->file_bytes[0] = ids.size() * 4;
    }
    // ---- role files (dictionary.py:98-107): ascending ID, "<id>\t<term>\n"
    static const char* kSuffix[3] = {".sid", ".pid", ".oid"};
    for (int r = 0; r < 3; ++r) {
      std::vector<size_t> part(T + 1, 0);
      parallel_for(T, [&](int t) {
        const uint64_t a = n_terms * t / T, b = n_terms * (t + 1) / T;
        size_t s = 0;
        for (uint64_t k = a; k < b; ++k)
          if ((groles[k] >> r) & 1u) s += n_digits(uint32_t(k + 1)) + 2 + g.terms[k].len;
        part[t + 1] = s;
      });
      for (int t = 0; t < T; ++t) part[t + 1] += part[t];
      std::vector<char> out(part[T]);
      parallel_for(T, [&](int t) {
        const uint64_t a = n_terms * t / T, b = n_terms * (t + 1) / T;
        char* p = out.data() + part[t];
        for (uint64_t k = a; k < b; ++k) {
          if (!((groles[k] >> r) & 1u)) continue;
          uint32_t v = uint32_t(k + 1);
          const size_t d = n_digits(v);
          for (size_t q = d; q-- > 0; v /= 10) p[q] = char('0' + v % 10);
          p += d;
          *p++ = '\t';
          memcpy(p, g.terms[k].p, g.terms[k].len);
          p += g.terms[k].len;
          *p++ = '\n';
        }
      });
      const std::string path = prefix + ".tmp" + kSuffix[r];
      const int o = open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
      if (o < 0) io_fail(rep, path, errno);
      write_all(o, out.data(), out.size(), rep, path);
      close(o);
      rep->file_bytes[1 + r] = out.size();
    }
    trace("write");
    if (errors_tsv && !errs.empty()) {
      *errors_tsv = static_cast<char*>(malloc(errs.size() + 1));
      memcpy(*errors_tsv, errs.c_str(), errs.size() + 1);
    }
  });
}

extern "C" int tidq_convert_free(char* p) {
  free(p);
  return TIDQ_OK;
}
