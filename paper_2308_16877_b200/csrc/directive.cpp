// directive.cpp — the approximation directive language (docs/directives.md)
// on the host: parse_directive / unparse (directive.hpp:522-554) with the
// reference's diagnostics (ParseErrorCode + byte offset, directive.hpp:86-100)
// and canonical form. Extension: perfo(random:p).
//
// The C-ABI carries the flattened spec plus the canonical text (which keeps
// the array sections); hpac_unparse renders specs built without sections.
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <string>
#include <string_view>
#include <vector>

#include "hpac_offload.h"

#define HPAC_API extern "C" __attribute__((visibility("default")))

namespace {

enum Code : int32_t {
  kEmptyDirective = 0,
  kUnknownClause,
  kUnexpectedChar,
  kArityMismatch,
  kNonNumeric,
  kDuplicateClause,
  kBadMemoKind,
  kBadPerfoKind,
  kBadLevel,
  kBadSection,
  kOutOfRange,
  kMissingInput,
  kMissingOutput,
};

const char* code_name(int32_t c) {
  static const char* names[] = {"empty-directive", "unknown-clause", "unexpected-char",
                                "arity-mismatch",  "non-numeric",    "duplicate-clause",
                                "bad-memo-kind",   "bad-perfo-kind", "bad-level",
                                "bad-section",     "out-of-range",   "missing-input",
                                "missing-output"};
  return c >= 0 && c <= kMissingOutput ? names[c] : "?";
}

struct Failure {
  int32_t code;
  size_t offset;
  std::string message;
};

// A length/stride: positive literal or host symbol (directive.hpp:31-41).
struct Dim {
  long long value = 1;
  std::string symbol;
};

// base[a*i+b : length : stride] (directive.hpp:43-56)
struct Section {
  std::string base;
  long long coef = 0, offset = 0;
  Dim length, stride;
};

struct Parsed {
  hpac_spec_t spec{};
  std::vector<Section> ins, outs;
};

// Shortest round-trip decimal (fmtnum.hpp:13-19).
std::string fmt_double(double v) {
  if (std::isnan(v)) return "nan";
  if (std::isinf(v)) return v > 0 ? "inf" : "-inf";
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  return std::string(buf, r.ptr);
}

// parse_double (fmtnum.hpp:23-41): inf/infinity any case, optional f/F suffix.
bool read_double(std::string_view text, double& out) {
  if (text.empty()) return false;
  std::string low(text);
  for (char& c : low) c = (char)std::tolower((unsigned char)c);
  std::string_view body = low;
  bool neg = false;
  if (body.front() == '+' || body.front() == '-') {
    neg = body.front() == '-';
    body.remove_prefix(1);
  }
  if (body == "inf" || body == "infinity") {
    out = neg ? -std::numeric_limits<double>::infinity() : std::numeric_limits<double>::infinity();
    return true;
  }
  if (text.back() == 'f' || text.back() == 'F') text.remove_suffix(1);
  if (text.empty()) return false;
  auto r = std::from_chars(text.data(), text.data() + text.size(), out);
  return r.ec == std::errc{} && r.ptr == text.data() + text.size();
}

class Scanner {
 public:
  explicit Scanner(std::string_view t) : s_(t) {}

  Parsed run() {
    ws();
    if (end()) die(kEmptyDirective, at_, "directive is empty");
    if (word_here() == "approx") take_word();
    for (ws(); !end(); ws()) clause();
    if (!have_tech_) die(kUnknownClause, 0, "directive has no memo or perfo clause");
    const int32_t t = out_.spec.technique;
    if (t == HPAC_TECH_IACT && out_.ins.empty())
      die(kMissingInput, tech_at_, "memo(in:...) requires an in(...) clause");
    if ((t == HPAC_TECH_IACT || t == HPAC_TECH_TAF) && out_.outs.empty())
      die(kMissingOutput, tech_at_, "memoization requires an out(...) clause");
    out_.spec.n_input_sections = (int32_t)out_.ins.size();
    out_.spec.n_output_sections = (int32_t)out_.outs.size();
    return out_;
  }

 private:
  [[noreturn]] void die(int32_t code, size_t off, const std::string& msg) {
    throw Failure{code, off, msg};
  }
  bool end() const { return at_ >= s_.size(); }
  char ch() const { return s_[at_]; }
  static bool wordch(char c) { return std::isalnum((unsigned char)c) || c == '_'; }
  void ws() {
    while (!end() && std::isspace((unsigned char)ch())) ++at_;
  }
  bool eat(char c) {
    ws();
    if (!end() && ch() == c) {
      ++at_;
      return true;
    }
    return false;
  }
  void need(char c) {
    ws();
    if (end() || ch() != c) die(kUnexpectedChar, at_, std::string("expected '") + c + "'");
    ++at_;
  }
  // separators inside a technique tuple: ')' for ':' is an arity error
  void colon(const char* what) {
    ws();
    if (!end() && ch() == ':') {
      ++at_;
      return;
    }
    if (!end() && ch() == ')') die(kArityMismatch, at_, std::string(what) + " has too few arguments");
    die(kUnexpectedChar, at_, "expected ':'");
  }
  void close(const char* what) {
    ws();
    if (!end() && ch() == ')') {
      ++at_;
      return;
    }
    if (!end() && ch() == ':') die(kArityMismatch, at_, std::string(what) + " has too many arguments");
    die(kUnexpectedChar, at_, "expected ')'");
  }
  std::string word_here() const {
    size_t p = at_;
    while (p < s_.size() && wordch(s_[p])) ++p;
    return std::string(s_.substr(at_, p - at_));
  }
  std::string take_word() {
    ws();
    size_t start = at_;
    std::string w = word_here();
    if (w.empty() || std::isdigit((unsigned char)s_[at_]))
      die(kUnexpectedChar, start, "expected identifier");
    at_ += w.size();
    return w;
  }
  long long whole(const std::string& what) {
    ws();
    size_t start = at_;
    bool neg = eat('-');
    if (end() || !std::isdigit((unsigned char)ch())) die(kNonNumeric, start, what + " must be an integer");
    long long v = 0;
    while (!end() && std::isdigit((unsigned char)ch())) v = v * 10 + (s_[at_++] - '0');
    return neg ? -v : v;
  }
  double number(const std::string& what) {
    ws();
    size_t start = at_, stop = at_;
    while (stop < s_.size() &&
           (std::isalnum((unsigned char)s_[stop]) || s_[stop] == '.' || s_[stop] == '+' ||
            s_[stop] == '-' || s_[stop] == '_'))
      ++stop;
    double v;
    if (stop == at_ || !read_double(s_.substr(at_, stop - at_), v))
      die(kNonNumeric, start, what + " must be numeric");
    at_ = stop;
    return v;
  }
  int32_t at_least(long long v, long long lo, size_t off, const std::string& what) {
    if (v < lo) die(kOutOfRange, off, what + " must be >= " + std::to_string(lo));
    return (int32_t)v;
  }
  double nonneg(double v, size_t off, const std::string& what) {
    if (!(v >= 0.0)) die(kOutOfRange, off, what + " must be >= 0");
    return v;
  }

  void clause() {
    ws();
    size_t start = at_;
    std::string name = take_word();
    if (name == "memo") return memo(start);
    if (name == "perfo") return perfo(start);
    if (name == "level") return level(start);
    if (name == "in") return sections(out_.ins);
    if (name == "out") return sections(out_.outs);
    die(kUnknownClause, start, "unknown clause '" + name + "'");
  }

  void technique_once(size_t start) {
    if (have_tech_) die(kDuplicateClause, start, "directive already has a technique clause");
    have_tech_ = true;
    tech_at_ = start;
  }

  void memo(size_t start) {
    technique_once(start);
    need('(');
    size_t kat = at_;
    std::string kind = take_word();
    hpac_spec_t& sp = out_.spec;
    if (kind == "in") {
      colon("memo(in)");
      sp.iact_table_size = at_least(whole("table size"), 1, kat, "table size");
      colon("memo(in)");
      sp.iact_threshold = nonneg(number("distance threshold"), kat, "distance threshold");
      if (eat(':')) sp.iact_tables_per_warp = at_least(whole("tables per warp"), 1, kat, "tables per warp");
      close("memo(in)");
      sp.technique = HPAC_TECH_IACT;
    } else if (kind == "out") {
      colon("memo(out)");
      sp.taf_h_size = at_least(whole("history size"), 1, kat, "history size");
      colon("memo(out)");
      sp.taf_p_size = at_least(whole("prediction size"), 1, kat, "prediction size");
      colon("memo(out)");
      sp.taf_threshold = nonneg(number("RSD threshold"), kat, "RSD threshold");
      close("memo(out)");
      sp.technique = HPAC_TECH_TAF;
    } else {
      die(kBadMemoKind, kat, "memo kind must be 'in' or 'out', got '" + kind + "'");
    }
  }

  void perfo(size_t start) {
    technique_once(start);
    need('(');
    size_t kat = at_;
    std::string kind = take_word();
    static const struct {
      const char* name;
      int32_t id;
    } kinds[] = {{"small", HPAC_PERFO_SMALL},
                 {"large", HPAC_PERFO_LARGE},
                 {"ini", HPAC_PERFO_INI},
                 {"fini", HPAC_PERFO_FINI},
                 {"herded_small", HPAC_PERFO_HERDED_SMALL},
                 {"herded_large", HPAC_PERFO_HERDED_LARGE},
                 {"random", HPAC_PERFO_RANDOM}};
    int32_t id = -1;
    for (auto& k : kinds)
      if (kind == k.name) id = k.id;
    if (id < 0) die(kBadPerfoKind, kat, "unknown perforation kind '" + kind + "'");
    colon("perfo");
    hpac_spec_t& sp = out_.spec;
    sp.perfo_kind = id;
    bool modulus = id == HPAC_PERFO_SMALL || id == HPAC_PERFO_LARGE ||
                   id == HPAC_PERFO_HERDED_SMALL || id == HPAC_PERFO_HERDED_LARGE;
    if (modulus) {
      sp.perfo_modulus = at_least(whole("skip modulus"), 2, kat, "skip modulus");
    } else {
      long long p = whole("skip percent");
      if (p < 1 || p > 99) die(kOutOfRange, kat, "skip percent must be in [1, 99]");
      sp.perfo_skip_percent = (int32_t)p;
    }
    close("perfo");
    sp.technique = HPAC_TECH_PERFO;
  }

  void level(size_t start) {
    if (have_level_) die(kDuplicateClause, start, "duplicate level clause");
    have_level_ = true;
    need('(');
    size_t lat = at_;
    std::string name = take_word();
    if (name == "thread")
      out_.spec.level = HPAC_LEVEL_THREAD;
    else if (name == "warp")
      out_.spec.level = HPAC_LEVEL_WARP;
    else if (name == "team" || name == "block")
      out_.spec.level = HPAC_LEVEL_TEAM;
    else
      die(kBadLevel, lat, "level must be thread, warp, or team; got '" + name + "'");
    need(')');
  }

  void sections(std::vector<Section>& into) {
    need('(');
    do into.push_back(section());
    while (eat(','));
    need(')');
  }

  Section section() {
    ws();
    size_t sat = at_;
    Section s;
    s.base = take_word();
    need('[');
    affine(sat, s);
    if (eat(':')) {
      s.length = dim("section length", sat);
      if (eat(':')) s.stride = dim("section stride", sat);
    }
    need(']');
    if (s.length.symbol.empty() && s.length.value < 1)
      die(kOutOfRange, sat, "section length must be >= 1");
    if (s.stride.symbol.empty() && s.stride.value < 1)
      die(kOutOfRange, sat, "section stride must be >= 1");
    return s;
  }

  // a*i + b, integer a and b, loop variable spelled i
  void affine(size_t sat, Section& s) {
    for (bool first = true;; first = false) {
      ws();
      long long sign = 1;
      if (eat('+'))
        sign = 1;
      else if (eat('-'))
        sign = -1;
      else if (!first)
        break;
      ws();
      if (end()) die(kBadSection, sat, "unterminated index expression");
      if (std::isdigit((unsigned char)ch())) {
        long long v = whole("index term");
        if (eat('*')) {
          if (take_word() != "i") die(kBadSection, sat, "index must be affine in i");
          s.coef += sign * v;
        } else {
          s.offset += sign * v;
        }
      } else {
        if (take_word() != "i") die(kBadSection, sat, "index must be affine in i");
        if (eat('*')) {
          ws();
          if (end() || !std::isdigit((unsigned char)ch()))
            die(kBadSection, sat, "index must be affine in i");
          s.coef += sign * whole("index coefficient");
        } else {
          s.coef += sign;
        }
      }
      ws();
      if (end() || (ch() != '+' && ch() != '-')) break;
    }
  }

  Dim dim(const std::string& what, size_t sat) {
    ws();
    Dim d;
    if (!end() && std::isdigit((unsigned char)ch())) {
      d.value = whole(what);
      return d;
    }
    std::string w = word_here();
    if (w.empty()) die(kBadSection, sat, what + " must be an integer or symbol");
    if (w == "i") die(kBadSection, sat, what + " cannot be the loop variable");
    at_ += w.size();
    d.symbol = w;
    d.value = 0;
    return d;
  }

  std::string_view s_;
  size_t at_ = 0;
  Parsed out_;
  bool have_tech_ = false, have_level_ = false;
  size_t tech_at_ = 0;
};

std::string render_dim(const Dim& d) { return d.symbol.empty() ? std::to_string(d.value) : d.symbol; }

std::string render_section(const Section& s) {
  std::string idx;
  if (s.coef == 0) {
    idx = std::to_string(s.offset);
  } else {
    idx = s.coef == 1 ? "i" : "i*" + std::to_string(s.coef);
    if (s.offset > 0) idx += "+" + std::to_string(s.offset);
    if (s.offset < 0) idx += std::to_string(s.offset);
  }
  std::string out = s.base + "[" + idx;
  bool len1 = s.length.symbol.empty() && s.length.value == 1;
  bool str1 = s.stride.symbol.empty() && s.stride.value == 1;
  if (!len1 || !str1) {
    out += ":" + render_dim(s.length);
    if (!str1) out += ":" + render_dim(s.stride);
  }
  return out + "]";
}

const char* perfo_name(int32_t k) {
  switch (k) {
    case HPAC_PERFO_SMALL: return "small";
    case HPAC_PERFO_LARGE: return "large";
    case HPAC_PERFO_INI: return "ini";
    case HPAC_PERFO_FINI: return "fini";
    case HPAC_PERFO_HERDED_SMALL: return "herded_small";
    case HPAC_PERFO_HERDED_LARGE: return "herded_large";
    case HPAC_PERFO_RANDOM: return "random";
  }
  return "?";
}

// unparse (directive.hpp:528-554): technique, non-default level, sections.
std::string canonical(const hpac_spec_t& sp, const std::vector<Section>* ins,
                      const std::vector<Section>* outs) {
  std::string o;
  switch (sp.technique) {
    case HPAC_TECH_TAF:
      o = "memo(out:" + std::to_string(sp.taf_h_size) + ":" + std::to_string(sp.taf_p_size) + ":" +
          fmt_double(sp.taf_threshold) + ")";
      break;
    case HPAC_TECH_IACT:
      o = "memo(in:" + std::to_string(sp.iact_table_size) + ":" + fmt_double(sp.iact_threshold);
      if (sp.iact_tables_per_warp > 0) o += ":" + std::to_string(sp.iact_tables_per_warp);
      o += ")";
      break;
    default: {
      bool modulus = sp.perfo_kind == HPAC_PERFO_SMALL || sp.perfo_kind == HPAC_PERFO_LARGE ||
                     sp.perfo_kind == HPAC_PERFO_HERDED_SMALL ||
                     sp.perfo_kind == HPAC_PERFO_HERDED_LARGE;
      o = std::string("perfo(") + perfo_name(sp.perfo_kind) + ":" +
          std::to_string(modulus ? sp.perfo_modulus : sp.perfo_skip_percent) + ")";
    }
  }
  if (sp.level == HPAC_LEVEL_WARP) o += " level(warp)";
  if (sp.level == HPAC_LEVEL_TEAM) o += " level(team)";
  auto join = [](const std::vector<Section>& v) {
    std::string r;
    for (size_t i = 0; i < v.size(); ++i) r += (i ? "," : "") + render_section(v[i]);
    return r;
  };
  if (ins && !ins->empty()) o += " in(" + join(*ins) + ")";
  if (outs && !outs->empty()) o += " out(" + join(*outs) + ")";
  return o;
}

void put(char* buf, size_t len, const std::string& s) {
  if (!buf || !len) return;
  size_t n = s.size() < len - 1 ? s.size() : len - 1;
  std::memcpy(buf, s.data(), n);
  buf[n] = 0;
}

}  // namespace

// On success `err` receives the canonical text (unparse) of the directive.
HPAC_API int hpac_parse_directive(const char* text, hpac_spec_t* out, int32_t* err_code,
                                  int64_t* err_offset, char* err, size_t errlen) {
  if (!text || !out) return HPAC_ERR_CONFIG;
  try {
    Parsed p = Scanner(text).run();
    *out = p.spec;
    put(err, errlen, canonical(p.spec, &p.ins, &p.outs));
    if (err_code) *err_code = -1;
    if (err_offset) *err_offset = -1;
    return HPAC_OK;
  } catch (const Failure& f) {
    if (err_code) *err_code = f.code;
    if (err_offset) *err_offset = (int64_t)f.offset;
    put(err, errlen,
        "directive error at byte " + std::to_string(f.offset) + " [" + code_name(f.code) +
            "]: " + f.message);
    return HPAC_ERR_DIRECTIVE;
  }
}

HPAC_API int hpac_unparse(const hpac_spec_t* spec, char* buf, size_t len) {
  if (!spec) return HPAC_ERR_CONFIG;
  if (spec->technique < HPAC_TECH_TAF || spec->technique > HPAC_TECH_PERFO) return HPAC_ERR_CONFIG;
  put(buf, len, canonical(*spec, nullptr, nullptr));
  return HPAC_OK;
}
