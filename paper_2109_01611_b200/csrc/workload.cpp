// SPEC-format inputs of the native scheduler: the profile CSV
// (SPEC S:130 + sm_count), the interference coefficients JSON and the
// workload JSON, with the C4 post-processing the scheduler consumes
// (SURVEY §8(c) C4): the min-envelope (C4.1), the SLO rule / Table constants
// (C4.2), the B200 rate scaling and the scenarios (C4.3-C4.4,
// P:787-806, DESIGN R23).  Pure host code; the CUDA path is not involved, so
// these run (and are parity-tested against oracle/profiles.py and
// oracle/workload.py) on a CPU-only host.
//
// Exactness: decimal latencies are converted by a decimal shift (no binary
// rounding) and rounded up to whole µs; utilisations, coefficients and the
// multiplier x are parsed with std::from_chars (correctly rounded, as Python's
// float()); the rate expression is evaluated in IEEE double in the documented
// order (this TU is compiled with -ffp-contract=off).
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/gpulet.h"

namespace gl {
gl_status set_error(gl_status s, const char* m);
}

namespace {

constexpr int kM = 6, kB = 32, kP = 6;
constexpr int kGrid[kP] = {20, 40, 50, 60, 80, 100};
constexpr int kStatB[6] = {1, 2, 4, 8, 16, 32};
constexpr int kSmDefault[kP] = {30, 60, 74, 88, 118, 148};
const char* const kNames[kM] = {"lenet5", "googlenet", "resnet50", "ssd_mobilenet_v1", "vgg16", "bert_base"};
// Table tab:ml-models, ms; BERT-base is not in the paper: 95 ms (ResNet-50's), DESIGN R2/R17.
constexpr int64_t kPaperSloMs[kM] = {5, 44, 95, 136, 130, 95};

gl_status err(gl_status s, const std::string& m) { return gl::set_error(s, m.c_str()); }

int model_index(const std::string& n) {
  for (int i = 0; i < kM; ++i)
    if (n == kNames[i]) return i;
  return -1;
}
int grid_index(int p) {
  for (int i = 0; i < kP; ++i)
    if (kGrid[i] == p) return i;
  return -1;
}
int stat_index(int b) {
  for (int i = 0; i < 6; ++i)
    if (kStatB[i] == b) return i;
  return -1;
}

std::string trim(const std::string& s) {
  size_t a = 0, b = s.size();
  while (a < b && (s[a] == ' ' || s[a] == '\t' || s[a] == '\r')) ++a;
  while (b > a && (s[b - 1] == ' ' || s[b - 1] == '\t' || s[b - 1] == '\r')) --b;
  return s.substr(a, b - a);
}

bool read_file(const char* path, std::string& out) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return false;
  std::ostringstream ss;
  ss << f.rdbuf();
  out = ss.str();
  return true;
}

// Exact ceil(value * 10^shift) of a plain decimal string [+]digits[.digits][e[+-]digits]
// (non-negative); false if malformed or out of range.
bool decimal_ceil_scaled(const std::string& s, int shift, int64_t& out) {
  size_t i = 0;
  if (i < s.size() && s[i] == '+') ++i;
  std::string digits;
  int exp10 = 0;
  bool any = false, dot = false;
  for (; i < s.size(); ++i) {
    const char c = s[i];
    if (c >= '0' && c <= '9') {
      digits += c;
      any = true;
      if (dot) --exp10;
    } else if (c == '.' && !dot) {
      dot = true;
    } else {
      break;
    }
  }
  if (!any) return false;
  if (i < s.size()) {
    if (s[i] != 'e' && s[i] != 'E') return false;
    ++i;
    int e = 0;
    auto r = std::from_chars(s.data() + i, s.data() + s.size(), e);
    if (r.ec != std::errc() || r.ptr != s.data() + s.size()) return false;
    exp10 += e;
  }
  exp10 += shift;
  // strip leading zeros; value = digits * 10^exp10
  size_t nz = digits.find_first_not_of('0');
  if (nz == std::string::npos) {
    out = 0;
    return true;
  }
  digits = digits.substr(nz);
  // drop trailing fractional digits beyond the integer part, remembering whether any is non-zero
  bool frac = false;
  while (exp10 < 0) {
    if (digits.empty()) break;
    if (digits.back() != '0') frac = true;
    digits.pop_back();
    ++exp10;
  }
  if (digits.empty()) digits = "0";
  if (digits.size() + (size_t)std::max(exp10, 0) > 17) return false;
  int64_t v = 0;
  for (char c : digits) v = v * 10 + (c - '0');
  for (int k = 0; k < exp10; ++k) v *= 10;
  out = v + (frac ? 1 : 0);
  return true;
}

bool parse_double(const std::string& s, double& v) {
  const std::string t = trim(s);
  if (t.empty()) return false;
  const char* b = t.data();
  if (*b == '+') ++b;
  auto r = std::from_chars(b, t.data() + t.size(), v);
  return r.ec == std::errc() && r.ptr == t.data() + t.size() && std::isfinite(v);
}

bool parse_int(const std::string& s, int64_t& v) {
  const std::string t = trim(s);
  if (t.empty()) return false;
  auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  return r.ec == std::errc() && r.ptr == t.data() + t.size();
}

std::vector<std::string> split_csv(const std::string& line) {
  std::vector<std::string> f;
  std::string cur;
  for (char c : line) {
    if (c == ',') {
      f.push_back(trim(cur));
      cur.clear();
    } else {
      cur += c;
    }
  }
  f.push_back(trim(cur));
  return f;
}

struct Table {
  std::vector<int32_t> lat;   // [m][b-1][gi]
  std::vector<double> l2, mem;  // [m][si][gi]
  int32_t sm[kP];
};

gl_status load_profile(const char* path, bool strict, Table& T) {
  std::string text;
  if (!read_file(path, text)) return err(GL_E_PARSE, std::string("profile: cannot read ") + path);
  T.lat.assign(kM * kB * kP, 0);
  T.l2.assign(kM * 6 * kP, 0.0);
  T.mem.assign(kM * 6 * kP, 0.0);
  for (int i = 0; i < kP; ++i) T.sm[i] = 0;
  std::vector<char> seen(kM * kB * kP, 0);
  std::istringstream in(text);
  std::string line;
  int lineno = 0;
  int c_model = -1, c_batch = -1, c_p = -1, c_us = -1, c_ms = -1, c_sm = -1, c_l2 = -1, c_mem = -1;
  size_t ncols = 0;
  bool header = false;
  while (std::getline(in, line)) {
    ++lineno;
    if (trim(line).empty()) continue;
    std::vector<std::string> f = split_csv(line);
    const std::string where = "profile line " + std::to_string(lineno) + ": ";
    if (!header) {
      for (size_t k = 0; k < f.size(); ++k) {
        const std::string& h = f[k];
        if (h == "model") c_model = (int)k;
        else if (h == "batch") c_batch = (int)k;
        else if (h == "partition_pct") c_p = (int)k;
        else if (h == "latency_us") c_us = (int)k;
        else if (h == "latency_ms") c_ms = (int)k;
        else if (h == "sm_count") c_sm = (int)k;
        else if (h == "l2_util") c_l2 = (int)k;
        else if (h == "mem_bw_util") c_mem = (int)k;
      }
      if (c_model < 0 || c_batch < 0 || c_p < 0 || (c_us < 0 && c_ms < 0))
        return err(GL_E_PARSE, where + "header needs model,batch,partition_pct,latency_us|latency_ms");
      ncols = f.size();
      header = true;
      continue;
    }
    if (f.size() != ncols) return err(GL_E_PARSE, where + "expected " + std::to_string(ncols) + " fields");
    const int m = model_index(f[c_model]);
    if (m < 0) return err(GL_E_DATA, where + "unknown model '" + f[c_model] + "'");
    int64_t b, p;
    if (!parse_int(f[c_batch], b) || !parse_int(f[c_p], p)) return err(GL_E_PARSE, where + "batch / partition_pct");
    if (b < 1 || b > kB) return err(GL_E_DATA, where + "batch outside 1..32");
    const int gi = grid_index((int)p);
    if (gi < 0) return err(GL_E_DATA, where + "partition_pct off the grid {20,40,50,60,80,100}");
    int64_t us;
    const bool ok_lat = c_us >= 0 ? decimal_ceil_scaled(f[c_us], 0, us) : decimal_ceil_scaled(f[c_ms], 3, us);
    if (!ok_lat) return err(GL_E_PARSE, where + "latency");
    if (us <= 0 || us > INT32_MAX) return err(GL_E_DATA, where + "latency must be positive");
    const size_t idx = ((size_t)m * kB + (b - 1)) * kP + gi;
    if (seen[idx]) return err(GL_E_DATA, where + "duplicate row");
    seen[idx] = 1;
    T.lat[idx] = (int32_t)us;
    if (c_sm >= 0 && !f[c_sm].empty()) {
      int64_t n;
      if (!parse_int(f[c_sm], n)) return err(GL_E_PARSE, where + "sm_count");
      if (n < 1) return err(GL_E_DATA, where + "sm_count must be positive");
      if (T.sm[gi] && T.sm[gi] != n) return err(GL_E_DATA, where + "sm_count differs from an earlier row");
      T.sm[gi] = (int32_t)n;
    }
    const int si = stat_index((int)b);
    if (si >= 0) {
      for (int which = 0; which < 2; ++which) {
        const int c = which ? c_mem : c_l2;
        if (c < 0 || f[c].empty()) continue;
        double v;
        if (!parse_double(f[c], v)) return err(GL_E_PARSE, where + (which ? "mem_bw_util" : "l2_util"));
        if (v < 0.0 || v > 1.0) return err(GL_E_DATA, where + "utilisation outside [0,1]");
        (which ? T.mem : T.l2)[((size_t)m * 6 + si) * kP + gi] = v;
      }
    }
  }
  if (!header) return err(GL_E_PARSE, "profile: empty file");
  for (int m = 0; m < kM; ++m)
    for (int b = 1; b <= kB; ++b)
      for (int g = 0; g < kP; ++g)
        if (!seen[((size_t)m * kB + (b - 1)) * kP + g])
          return err(GL_E_DATA, std::string("profile: missing row (") + kNames[m] + ", " + std::to_string(b) + ", " +
                                    std::to_string(kGrid[g]) + ")");
  for (int g = 0; g < kP; ++g)
    if (!T.sm[g]) T.sm[g] = kSmDefault[g];
  auto L = [&](int m, int b, int g) -> int32_t& { return T.lat[((size_t)m * kB + (b - 1)) * kP + g]; };
  if (strict) {
    // non-decreasing in b, non-increasing in p
    for (int m = 0; m < kM; ++m)
      for (int b = 1; b <= kB; ++b)
        for (int g = 0; g < kP; ++g) {
          const bool bad_b = b > 1 && L(m, b, g) < L(m, b - 1, g);
          const bool bad_p = g > 0 && L(m, b, g) > L(m, b, g - 1);
          if (bad_b || bad_p)
            return err(GL_E_DATA, std::string("profile: monotonicity violated at (") + kNames[m] + ", " +
                                      std::to_string(b) + ", " + std::to_string(kGrid[g]) + ")" +
                                      (bad_b ? " in batch" : " in partition"));
        }
  } else {
    // C4.1 min-envelope over (b' >= b, p' <= p)
    for (int m = 0; m < kM; ++m)
      for (int b = kB; b >= 1; --b)
        for (int g = 0; g < kP; ++g) {
          int32_t v = L(m, b, g);
          if (b < kB) v = std::min(v, L(m, b + 1, g));
          if (g > 0) v = std::min(v, L(m, b, g - 1));
          L(m, b, g) = v;
        }
  }
  return GL_OK;
}

// ---- a small JSON reader (objects, arrays, strings, numbers kept as text, literals) ----
struct JVal {
  enum Kind { NUL, BOOL, NUM, STR, ARR, OBJ } kind = NUL;
  bool b = false;
  std::string s;  // NUM: the literal text; STR: the string
  std::vector<JVal> a;
  std::vector<std::pair<std::string, JVal>> o;
  const JVal* get(const char* k) const {
    for (auto& kv : o)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

struct JParser {
  const std::string& t;
  size_t i = 0;
  std::string why;
  explicit JParser(const std::string& t) : t(t) {}
  void ws() {
    while (i < t.size() && (t[i] == ' ' || t[i] == '\n' || t[i] == '\r' || t[i] == '\t')) ++i;
  }
  bool fail(const char* w) {
    if (why.empty()) why = std::string(w) + " at offset " + std::to_string(i);
    return false;
  }
  bool str(std::string& out) {
    if (i >= t.size() || t[i] != '"') return fail("expected string");
    ++i;
    out.clear();
    while (i < t.size() && t[i] != '"') {
      char c = t[i++];
      if (c == '\\') {
        if (i >= t.size()) return fail("bad escape");
        const char e = t[i++];
        switch (e) {
          case '"': c = '"'; break;
          case '\\': c = '\\'; break;
          case '/': c = '/'; break;
          case 'n': c = '\n'; break;
          case 't': c = '\t'; break;
          case 'r': c = '\r'; break;
          case 'b': c = '\b'; break;
          case 'f': c = '\f'; break;
          default: return fail("unsupported escape");
        }
      }
      out += c;
    }
    if (i >= t.size()) return fail("unterminated string");
    ++i;
    return true;
  }
  bool val(JVal& v, int depth = 0) {
    if (depth > 32) return fail("nesting too deep");
    ws();
    if (i >= t.size()) return fail("unexpected end");
    const char c = t[i];
    if (c == '{') {
      v.kind = JVal::OBJ;
      ++i;
      ws();
      if (i < t.size() && t[i] == '}') {
        ++i;
        return true;
      }
      for (;;) {
        ws();
        std::string k;
        if (!str(k)) return false;
        ws();
        if (i >= t.size() || t[i] != ':') return fail("expected ':'");
        ++i;
        JVal x;
        if (!val(x, depth + 1)) return false;
        v.o.emplace_back(k, std::move(x));
        ws();
        if (i < t.size() && t[i] == ',') {
          ++i;
          continue;
        }
        if (i < t.size() && t[i] == '}') {
          ++i;
          return true;
        }
        return fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.kind = JVal::ARR;
      ++i;
      ws();
      if (i < t.size() && t[i] == ']') {
        ++i;
        return true;
      }
      for (;;) {
        JVal x;
        if (!val(x, depth + 1)) return false;
        v.a.push_back(std::move(x));
        ws();
        if (i < t.size() && t[i] == ',') {
          ++i;
          continue;
        }
        if (i < t.size() && t[i] == ']') {
          ++i;
          return true;
        }
        return fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = JVal::STR;
      return str(v.s);
    }
    if (t.compare(i, 4, "true") == 0) {
      v.kind = JVal::BOOL;
      v.b = true;
      i += 4;
      return true;
    }
    if (t.compare(i, 5, "false") == 0) {
      v.kind = JVal::BOOL;
      i += 5;
      return true;
    }
    if (t.compare(i, 4, "null") == 0) {
      v.kind = JVal::NUL;
      i += 4;
      return true;
    }
    const size_t s0 = i;
    while (i < t.size() && (std::isdigit((unsigned char)t[i]) || t[i] == '-' || t[i] == '+' || t[i] == '.' ||
                            t[i] == 'e' || t[i] == 'E'))
      ++i;
    if (i == s0) return fail("unexpected character");
    v.kind = JVal::NUM;
    v.s = t.substr(s0, i - s0);
    return true;
  }
};

gl_status parse_json_arg(const char* arg, const char* what, JVal& v) {
  std::string text;
  const char* p = arg;
  while (*p == ' ' || *p == '\n' || *p == '\t' || *p == '\r') ++p;
  if (*p == '{') {
    text = arg;
  } else if (!read_file(arg, text)) {
    return err(GL_E_PARSE, std::string(what) + ": cannot read " + arg);
  }
  JParser P(text);
  if (!P.val(v)) return err(GL_E_PARSE, std::string(what) + ": " + P.why);
  P.ws();
  if (P.i != text.size()) return err(GL_E_PARSE, std::string(what) + ": trailing text at offset " + std::to_string(P.i));
  if (v.kind != JVal::OBJ) return err(GL_E_PARSE, std::string(what) + ": not a JSON object");
  return GL_OK;
}

bool jnum_double(const JVal* v, double& d) { return v && v->kind == JVal::NUM && parse_double(v->s, d); }
bool jnum_int(const JVal* v, int64_t& n) { return v && v->kind == JVal::NUM && parse_int(v->s, n); }

int scenario_base(const std::string& name, int64_t base[kM], int& app_ref) {
  static const struct {
    const char* n;
    int64_t r[kM];
    int app;
  } S[] = {{"equal", {50, 50, 50, 50, 50, 50}, -1},
           {"mix6", {50, 50, 50, 50, 50, 50}, -1},
           {"long-only", {0, 0, 100, 100, 100, 100}, -1},
           {"short-skew", {100, 100, 100, 50, 50, 50}, -1},
           {"game", {600, 0, 100, 0, 0, 0}, 2},      // 6 LeNet + 1 ResNet-50 per app request
           {"traffic", {0, 100, 0, 100, 100, 0}, 3}};  // SSD -> GoogLeNet + VGG-16
  for (auto& s : S)
    if (name == s.n) {
      for (int m = 0; m < kM; ++m) base[m] = s.r[m];
      app_ref = s.app;
      return 1;
    }
  return 0;
}

void slos(const int32_t* lat, int slo_mode, int32_t* slo) {
  for (int m = 0; m < kM; ++m)
    slo[m] = slo_mode == 0 ? 2 * lat[((size_t)m * kB + (kB - 1)) * kP + (kP - 1)] : (int32_t)(kPaperSloMs[m] * 1000);
}

// C4.3: paper rates (req/s on the 2080 Ti) -> B200 rates at multiplier x on num_gpus GPUs
gl_status scale_rates(const int32_t* slo, const int64_t* base, int app, double x, int num_gpus, int64_t* rates) {
  if (!(x >= 0.0) || !std::isfinite(x)) return err(GL_E_ARG, "x must be finite and >= 0");
  for (int m = 0; m < kM; ++m) {
    // per-model time compression; BERT-base (not in the paper) reuses ResNet-50's (C4.3);
    // an application keeps its composition with its app-SLO model's scale (R23)
    const int ref = app >= 0 ? app : (m == 5 ? 2 : m);
    const double num = (double)(base[m] * kPaperSloMs[ref] * 1000);
    const double v = num * x / (double)slo[ref];
    rates[m] = (int64_t)std::floor(v) * num_gpus;
  }
  return GL_OK;
}

gl_status rates_of(const int32_t* slo, const std::string& scen, double x, int num_gpus, int64_t* rates,
                   int64_t* base_out) {
  int64_t base[kM];
  int app = -1;
  if (!scenario_base(scen, base, app)) return err(GL_E_ARG, "unknown scenario '" + scen + "'");
  if (base_out)
    for (int m = 0; m < kM; ++m) base_out[m] = base[m];
  return scale_rates(slo, base, app, x, num_gpus, rates);
}

// F3 `traffic` as a two-stage chain (DESIGN R28): application SLO = 2 x the longest
// member's L*(32, 100 %) (136 ms in table mode); the detector's budget is
// its share of the two stages' solo latencies, s1 = floor(s_app L_ssd / (L_ssd +
// max(L_goo, L_vgg))); the recognisers get s_app - s1 - handoff from their spawn;
// rates floor((100 * 136 ms * x) / s_app) * num_gpus for SSD, GoogLeNet, VGG-16.
constexpr int kSsd = 3, kGoo = 1, kVgg = 4;
constexpr int64_t kPaperTrafficSloMs = 136;
gl_status chain_workload(const int32_t* lat, int slo_mode, double x, int num_gpus, int64_t handoff, int32_t* slo,
                         int64_t* rates, int64_t* s_app_out) {
  if (!(x >= 0.0) || !std::isfinite(x)) return err(GL_E_ARG, "x must be finite and >= 0");
  auto L = [&](int m) { return (int64_t)lat[((size_t)m * kB + (kB - 1)) * kP + (kP - 1)]; };
  const int64_t l1 = L(kSsd), l2 = std::max(L(kGoo), L(kVgg));
  const int64_t s_app = slo_mode == 0 ? 2 * std::max(l1, l2) : kPaperTrafficSloMs * 1000;
  const int64_t s1 = (s_app * l1) / (l1 + l2);
  if (handoff < 0 || s_app - s1 - handoff <= 0) return err(GL_E_ARG, "traffic-chain: handoff_us");
  slos(lat, slo_mode, slo);
  for (int m = 0; m < kM; ++m) rates[m] = 0;
  for (int m : {kGoo, kSsd, kVgg}) {
    slo[m] = (int32_t)(m == kSsd ? s1 : s_app - s1 - handoff);
    rates[m] = (int64_t)std::floor((double)(100 * kPaperTrafficSloMs * 1000) * x / (double)s_app) * num_gpus;
  }
  *s_app_out = s_app;
  return GL_OK;
}

std::string ints_json(const int64_t* v, int n) {
  std::string s = "[";
  for (int i = 0; i < n; ++i) s += (i ? "," : "") + std::to_string(v[i]);
  return s + "]";
}

}  // namespace

extern "C" gl_status gl_profile_load(const char* profile_csv, int32_t flags, int32_t* lat_us, double* l2, double* mem,
                                     int32_t* sm_count) {
  if (!profile_csv) return err(GL_E_ARG, "gl_profile_load: NULL path");
  Table T;
  gl_status rc = load_profile(profile_csv, (flags & 1) != 0, T);
  if (rc) return rc;
  if (lat_us) std::memcpy(lat_us, T.lat.data(), T.lat.size() * sizeof(int32_t));
  if (l2) std::memcpy(l2, T.l2.data(), T.l2.size() * sizeof(double));
  if (mem) std::memcpy(mem, T.mem.data(), T.mem.size() * sizeof(double));
  if (sm_count) std::memcpy(sm_count, T.sm, sizeof T.sm);
  return GL_OK;
}

extern "C" gl_status gl_workload_rates(const int32_t* lat_us, int32_t slo_mode, const char* scenario, double x,
                                       int32_t num_gpus, int32_t* slo_us, int32_t* rates) {
  if (!lat_us || !scenario || !slo_us || !rates || num_gpus < 1 || slo_mode < 0 || slo_mode > 1)
    return err(GL_E_ARG, "gl_workload_rates: bad argument");
  int32_t slo[kM];
  slos(lat_us, slo_mode, slo);
  int64_t r[kM];
  int64_t s_app = 0;
  gl_status rc = std::string(scenario) == "traffic-chain"
                     ? chain_workload(lat_us, slo_mode, x, num_gpus, 0, slo, r, &s_app)
                     : rates_of(slo, scenario, x, num_gpus, r, nullptr);
  if (rc) return rc;
  for (int m = 0; m < kM; ++m) {
    if (r[m] > INT32_MAX) return err(GL_E_ARG, "gl_workload_rates: rate overflows int32");
    slo_us[m] = slo[m];
    rates[m] = (int32_t)r[m];
  }
  return GL_OK;
}

extern "C" gl_status gl_schedule_files(const char* profile_csv, const char* coeffs_json, const char* workload_json,
                                       char* plan_buf, size_t cap, size_t* len, int32_t* verdict) {
  if (!profile_csv || !workload_json || !plan_buf || !len || !verdict)
    return err(GL_E_ARG, "gl_schedule_files: NULL argument");
  JVal W;
  gl_status rc = parse_json_arg(workload_json, "workload", W);
  if (rc) return rc;
  bool strict = false;
  if (const JVal* e = W.get("envelope")) {
    if (e->kind != JVal::BOOL) return err(GL_E_ARG, "workload: envelope must be true/false");
    strict = !e->b;
  }
  Table T;
  rc = load_profile(profile_csv, strict, T);
  if (rc) return rc;
  int64_t num_gpus = 1;
  if (const JVal* v = W.get("num_gpus"))
    if (!jnum_int(v, num_gpus) || num_gpus < 1 || num_gpus > 64) return err(GL_E_ARG, "workload: num_gpus");
  std::string mode = "gpulet";
  if (const JVal* v = W.get("mode")) {
    if (v->kind != JVal::STR) return err(GL_E_ARG, "workload: mode");
    mode = v->s;
  }
  int imode;
  if (mode == "gpulet") imode = 0;
  else if (mode == "gpulet+int") imode = 1;
  else if (mode == "sbp") imode = 2;
  else if (mode == "ideal") imode = 3;
  else if (mode == "sbp50") imode = 4;
  else return err(GL_E_ARG, "workload: unknown mode '" + mode + "'");
  std::string slo_mode = "rule";
  if (const JVal* v = W.get("slo_mode")) {
    if (v->kind != JVal::STR || (v->s != "rule" && v->s != "table")) return err(GL_E_ARG, "workload: slo_mode");
    slo_mode = v->s;
  }
  int32_t slo[kM];
  slos(T.lat.data(), slo_mode == "rule" ? 0 : 1, slo);
  int64_t rates[kM] = {0, 0, 0, 0, 0, 0};
  int truncated = -1;
  const JVal* scen = W.get("scenario");
  const JVal* rts = W.get("rates");
  const JVal* mods = W.get("models");
  const JVal* brts = W.get("base_rates");
  if ((scen != nullptr) + (rts != nullptr) + (mods != nullptr) + (brts != nullptr) != 1)
    return err(GL_E_ARG, "workload: give exactly one of scenario, base_rates, rates, models");
  int64_t app_slo = -1;
  if (scen && scen->kind == JVal::STR && scen->s == "traffic-chain") {
    double x = 1.0;
    if (const JVal* v = W.get("x"))
      if (!jnum_double(v, x)) return err(GL_E_ARG, "workload: x");
    int64_t handoff = 0;
    if (const JVal* v = W.get("handoff_us"))
      if (!jnum_int(v, handoff)) return err(GL_E_ARG, "workload: handoff_us");
    rc = chain_workload(T.lat.data(), slo_mode == "rule" ? 0 : 1, x, (int)num_gpus, handoff, slo, rates, &app_slo);
    if (rc) return rc;
    for (int m : {kGoo, kSsd, kVgg})   // canonical order: the first model whose rate truncated
      if (rates[m] == 0 && truncated < 0) truncated = m;
  } else if (scen || brts) {
    if (scen && scen->kind != JVal::STR) return err(GL_E_ARG, "workload: scenario");
    double x = 1.0;
    if (const JVal* v = W.get("x"))
      if (!jnum_double(v, x)) return err(GL_E_ARG, "workload: x");
    int64_t base[kM];
    if (scen) {
      rc = rates_of(slo, scen->s, x, (int)num_gpus, rates, base);
    } else {
      if (brts->kind != JVal::ARR || brts->a.size() != kM) return err(GL_E_ARG, "workload: base_rates must list 6 ints");
      int64_t b6[kM];
      for (int m = 0; m < kM; ++m)
        if (!jnum_int(&brts->a[m], b6[m]) || b6[m] < 0 || b6[m] > 1000000) return err(GL_E_ARG, "workload: base_rates");
      rc = scale_rates(slo, b6, -1, x, (int)num_gpus, rates);
      for (int m = 0; m < kM; ++m) base[m] = b6[m];
    }
    if (rc) return rc;
    for (int m = 0; m < kM && truncated < 0; ++m)
      if (base[m] > 0 && rates[m] == 0) truncated = m;
  } else if (rts) {
    if (rts->kind != JVal::ARR || rts->a.size() != kM) return err(GL_E_ARG, "workload: rates must list 6 ints");
    for (int m = 0; m < kM; ++m)
      if (!jnum_int(&rts->a[m], rates[m]) || rates[m] < 0) return err(GL_E_ARG, "workload: rates");
  } else {
    if (mods->kind != JVal::ARR) return err(GL_E_ARG, "workload: models must be a list");
    for (const JVal& e : mods->a) {
      const JVal* n = e.get("name");
      if (e.kind != JVal::OBJ || !n || n->kind != JVal::STR) return err(GL_E_ARG, "workload: models[].name");
      const int m = model_index(n->s);
      if (m < 0) return err(GL_E_ARG, "workload: unknown model '" + n->s + "'");
      if (!jnum_int(e.get("rate"), rates[m]) || rates[m] < 0) return err(GL_E_ARG, "workload: models[].rate");
      if (const JVal* s = e.get("slo_ms")) {
        int64_t us;
        if (s->kind != JVal::NUM || !decimal_ceil_scaled(s->s, 3, us) || us <= 0 || us > INT32_MAX)
          return err(GL_E_ARG, "workload: models[].slo_ms");
        slo[m] = (int32_t)us;
      }
    }
  }
  for (int m = 0; m < kM; ++m)
    if (rates[m] > INT32_MAX) return err(GL_E_ARG, "workload: rate overflows int32");
  double coeffs[5] = {0, 0, 0, 0, 0};
  if (coeffs_json) {
    JVal C;
    rc = parse_json_arg(coeffs_json, "coeffs", C);
    if (rc) return rc;
    const JVal* c = C.get("coeffs");
    if (!c || c->kind != JVal::ARR || c->a.size() != 5) return err(GL_E_PARSE, "coeffs: need \"coeffs\": [c1..c5]");
    for (int k = 0; k < 5; ++k)
      if (!jnum_double(&c->a[k], coeffs[k])) return err(GL_E_PARSE, "coeffs: c" + std::to_string(k + 1));
  } else if (imode == 1) {
    return err(GL_E_ARG, "gl_schedule_files: mode gpulet+int needs coeffs_json");
  }
  int64_t slo64[kM];
  for (int m = 0; m < kM; ++m) slo64[m] = slo[m];
  std::string head = "{\"slo_us\":" + ints_json(slo64, kM) + ",\"rates\":" + ints_json(rates, kM) +
                     ",\"num_gpus\":" + std::to_string(num_gpus) + ",\"mode\":\"" + mode + "\",\"slo_mode\":\"" +
                     slo_mode + "\"" + (app_slo >= 0 ? ",\"app_slo_us\":" + std::to_string(app_slo) : std::string()) +
                     "}\n";
  std::string out;
  int32_t ok = 0;
  if (truncated >= 0) {
    out = head + "{\"verdict\":\"NotSchedulable\",\"failed_model\":\"" + kNames[truncated] +
          "\",\"reason\":\"rate_truncated\"}\n";
  } else {
    int32_t r32[kM];
    for (int m = 0; m < kM; ++m) r32[m] = (int32_t)rates[m];
    gl_sched_input in{};
    in.n_models = kM;
    in.names = kNames;
    in.lat_us = T.lat.data();
    in.l2 = T.l2.data();
    in.mem = T.mem.data();
    in.slo_us = slo;
    in.rates = r32;
    for (int k = 0; k < 5; ++k) in.coeffs[k] = coeffs[k];
    in.num_gpus = (int32_t)num_gpus;
    in.mode = imode;
    in.sm_count = T.sm;
    std::vector<char> buf(1 << 20);
    size_t n = 0;
    rc = gl_schedule(&in, buf.data(), buf.size(), &n, &ok);
    if (rc) return err(rc, "gl_schedule_files: scheduler failed");
    out = head + std::string(buf.data(), n);
  }
  if (out.size() + 1 > cap) return err(GL_E_BUDGET, "gl_schedule_files: plan buffer too small");
  std::memcpy(plan_buf, out.c_str(), out.size() + 1);
  *len = out.size();
  *verdict = ok;
  return GL_OK;
}
