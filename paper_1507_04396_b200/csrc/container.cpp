// container.cpp — the factorization container:
// save_factorization / load_factorization of the reference
// (serialize.hpp:25-181) without a JSON library.  Same schema, key names and
// version ("pmmf-factorization", 1), keys in the order nlohmann::json writes
// them (sorted), doubles in shortest round-trip form (std::to_chars), so a
// file written here loads in the reference and vice versa, and a
// save -> load round trip reproduces every value bit for bit.
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "result.cuh"

namespace pmmf_b200 {

namespace {

constexpr const char* kFormat = "pmmf-factorization";  // serialize.hpp:23
constexpr int kVersion = 1;                             // serialize.hpp:24

// ------------------------------------------------------------ writer
struct Out {
  std::string b;
  void raw(const char* s) { b += s; }
  void num(double v) {
    if (!std::isfinite(v)) {  // nlohmann::json writes non-finite numbers as null
      b += "null";
      return;
    }
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof buf, v);
    b.append(buf, r.ptr);
  }
  void num(int64_t v) {
    char buf[32];
    auto r = std::to_chars(buf, buf + sizeof buf, v);
    b.append(buf, r.ptr);
  }
  void num(uint64_t v) {
    char buf[32];
    auto r = std::to_chars(buf, buf + sizeof buf, v);
    b.append(buf, r.ptr);
  }
  void key(const char* k) {
    b += '"';
    b += k;
    b += "\":";
  }
  template <typename T>
  void arr(const T* p, size_t n) {
    b += '[';
    for (size_t i = 0; i < n; ++i) {
      if (i) b += ',';
      num(p[i]);
    }
    b += ']';
  }
};

// ------------------------------------------------------------ reader
// A small DOM; arrays of numbers keep their tokens' integer and double
// readings (indices and seeds are integers, values doubles).
struct JVal {
  enum Type { Null, Bool, Num, Str, Arr, Obj } t = Null;
  bool b = false;
  double d = 0.0;
  bool is_int = false;
  bool neg = false;
  uint64_t u = 0;  // |integer| when is_int
  std::string s;
  std::vector<JVal> a;
  std::vector<std::pair<std::string, JVal>> o;

  const JVal& at(const char* k) const {
    if (t != Obj) fail(PMMF_DATA, std::string("factorization file: expected an object around '") + k + "'");
    for (const auto& kv : o)
      if (kv.first == k) return kv.second;
    fail(PMMF_DATA, std::string("factorization file: missing key '") + k + "'");
  }
  const JVal* find(const char* k) const {
    if (t != Obj) return nullptr;
    for (const auto& kv : o)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
  double as_double() const {
    if (t == Null) return std::nan("");
    if (t != Num) fail(PMMF_DATA, "factorization file: expected a number");
    return d;
  }
  int64_t as_int() const {
    if (t != Num || !is_int) fail(PMMF_DATA, "factorization file: expected an integer");
    return neg ? -static_cast<int64_t>(u) : static_cast<int64_t>(u);
  }
  uint64_t as_u64() const {
    if (t != Num || !is_int || neg) fail(PMMF_DATA, "factorization file: expected an unsigned integer");
    return u;
  }
  bool as_bool() const {
    if (t != Bool) fail(PMMF_DATA, "factorization file: expected a boolean");
    return b;
  }
  const std::vector<JVal>& arr() const {
    if (t != Arr) fail(PMMF_DATA, "factorization file: expected an array");
    return a;
  }
};

struct Parser {
  const char* p;
  const char* e;
  [[noreturn]] void bad(const char* what) {
    fail(PMMF_DATA, std::string("factorization file: ") + what + " at byte " +
                        std::to_string(static_cast<long long>(p - start)));
  }
  const char* start;
  void ws() {
    while (p < e && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
  }
  void lit(const char* w) {
    const size_t n = std::strlen(w);
    if (static_cast<size_t>(e - p) < n || std::memcmp(p, w, n) != 0) bad("invalid literal");
    p += n;
  }
  std::string str() {
    if (p >= e || *p != '"') bad("expected a string");
    ++p;
    std::string r;
    while (p < e && *p != '"') {
      if (*p == '\\') {
        ++p;
        if (p >= e) bad("bad escape");
        const char c = *p;
        if (c == 'n') r += '\n';
        else if (c == 't') r += '\t';
        else if (c == 'r') r += '\r';
        else if (c == 'b') r += '\b';
        else if (c == 'f') r += '\f';
        else if (c == 'u') bad("unicode escapes are not used by the container");
        else r += c;
        ++p;
      } else {
        r += *p++;
      }
    }
    if (p >= e) bad("unterminated string");
    ++p;
    return r;
  }
  void number(JVal& v) {
    const char* b = p;
    if (p < e && (*p == '-' || *p == '+')) ++p;
    bool integral = true;
    while (p < e && ((*p >= '0' && *p <= '9') || *p == '.' || *p == 'e' || *p == 'E' || *p == '-' || *p == '+')) {
      if (*p == '.' || *p == 'e' || *p == 'E') integral = false;
      ++p;
    }
    if (p == b) bad("expected a value");
    v.t = JVal::Num;
    auto rd = std::from_chars(b, p, v.d);
    if (rd.ec != std::errc() || rd.ptr != p) bad("bad number");
    if (integral) {
      const char* q = b;
      v.neg = *q == '-';
      if (*q == '-' || *q == '+') ++q;
      auto ri = std::from_chars(q, p, v.u);
      v.is_int = ri.ec == std::errc() && ri.ptr == p;
    }
  }
  void value(JVal& v, int depth) {
    if (depth > 64) bad("nesting too deep");
    ws();
    if (p >= e) bad("unexpected end");
    switch (*p) {
      case '{': {
        ++p;
        v.t = JVal::Obj;
        ws();
        if (p < e && *p == '}') {
          ++p;
          return;
        }
        for (;;) {
          ws();
          std::string k = str();
          ws();
          if (p >= e || *p != ':') bad("expected ':'");
          ++p;
          v.o.emplace_back(std::move(k), JVal());
          value(v.o.back().second, depth + 1);
          ws();
          if (p < e && *p == ',') {
            ++p;
            continue;
          }
          if (p < e && *p == '}') {
            ++p;
            return;
          }
          bad("expected ',' or '}'");
        }
      }
      case '[': {
        ++p;
        v.t = JVal::Arr;
        ws();
        if (p < e && *p == ']') {
          ++p;
          return;
        }
        for (;;) {
          v.a.emplace_back();
          value(v.a.back(), depth + 1);
          ws();
          if (p < e && *p == ',') {
            ++p;
            continue;
          }
          if (p < e && *p == ']') {
            ++p;
            return;
          }
          bad("expected ',' or ']'");
        }
      }
      case '"':
        v.t = JVal::Str;
        v.s = str();
        return;
      case 't':
        lit("true");
        v.t = JVal::Bool;
        v.b = true;
        return;
      case 'f':
        lit("false");
        v.t = JVal::Bool;
        v.b = false;
        return;
      case 'n':
        lit("null");
        v.t = JVal::Null;
        return;
      default:
        number(v);
    }
  }
};

std::vector<int64_t> ints(const JVal& v) {
  std::vector<int64_t> r;
  r.reserve(v.arr().size());
  for (const JVal& x : v.arr()) r.push_back(x.as_int());
  return r;
}

}  // namespace

std::string factorization_to_json(const Result& r) {  // serialize.hpp:61-110
  Out o;
  const pmmf_b200_params& p = r.params;
  o.raw("{");
  o.key("active_history");
  o.arr(r.hist.data(), r.hist.size());
  o.raw(",");
  o.key("core");
  o.raw("{");
  o.key("dense");
  o.arr(r.core.data(), r.core.size());
  o.raw(",");
  o.key("indices");
  o.arr(r.core_idx.data(), r.core_idx.size());
  o.raw("},\n");
  o.key("diagonal");
  o.raw("[");
  for (size_t i = 0; i < r.diag.size(); ++i) {
    o.raw(i ? ",{" : "{");
    o.key("d");
    o.num(r.diag[i].second);
    o.raw(",");
    o.key("i");
    o.num(static_cast<int64_t>(r.diag[i].first));
    o.raw("}");
  }
  o.raw("],\n");
  o.key("format");
  o.raw("\"");
  o.raw(kFormat);
  o.raw("\",");
  o.key("n");
  o.num(static_cast<int64_t>(r.n));
  o.raw(",");
  o.key("params");  // serialize.hpp:25-42
  o.raw("{");
  o.key("cluster");
  o.raw("{");
  o.key("bypass");
  o.raw(p.bypass_enabled ? "true" : "false");
  o.raw(",");
  o.key("c_max");
  o.num(static_cast<int64_t>(p.c_max));
  o.raw(",");
  o.key("c_min");
  o.num(static_cast<int64_t>(p.c_min));
  o.raw(",");
  o.key("d_max");
  o.num(static_cast<int64_t>(p.d_max));
  o.raw(",");
  o.key("m_target");
  o.num(static_cast<int64_t>(p.m_target));
  o.raw(",");
  o.key("seed");
  o.num(static_cast<uint64_t>(p.cluster_seed));
  o.raw("},");
  o.key("core_cap");
  o.num(static_cast<int64_t>(p.core_cap));
  o.raw(",");
  o.key("core_min");
  o.num(static_cast<int64_t>(p.core_min));
  o.raw(",");
  o.key("eta");
  o.num(p.eta);
  o.raw(",");
  o.key("k");
  o.num(static_cast<int64_t>(p.k));
  o.raw(",");
  o.key("n_stages");
  o.num(static_cast<int64_t>(p.n_stages));
  o.raw(",");
  o.key("seed");
  o.num(static_cast<uint64_t>(p.seed));
  o.raw("},\n");
  o.key("residual_sq");
  o.num(r.residual_sq);
  o.raw(",\n");
  o.key("stages");
  o.raw("[");
  const int k = r.k;
  for (size_t si = 0; si < r.stages.size(); ++si) {
    const Result::Stage& st = r.stages[si];
    o.raw(si ? ",\n{" : "\n{");
    o.key("bypassed");
    o.arr(st.bypassed.data(), st.bypassed.size());
    o.raw(",\n");
    o.key("eliminated");
    o.raw("[");
    for (size_t i = 0; i < st.elim_idx.size(); ++i) {
      o.raw(i ? ",{" : "{");
      o.key("d");
      o.num(st.elim_diag[i]);
      o.raw(",");
      o.key("i");
      o.num(static_cast<int64_t>(st.elim_idx[i]));
      o.raw(",");
      o.key("m");
      o.num(st.elim_mass[i]);
      o.raw("}");
    }
    o.raw("],\n");
    o.key("partition");
    o.raw("[");
    for (size_t u = 0; u + 1 < st.off.size(); ++u) {
      if (u) o.raw(",");
      o.arr(st.members.data() + st.off[u], static_cast<size_t>(st.off[u + 1] - st.off[u]));
    }
    o.raw("],\n");
    o.key("rotations");
    o.raw("[");
    const size_t nr = k ? st.rot_idx.size() / static_cast<size_t>(k) : 0;
    for (size_t t = 0; t < nr; ++t) {
      o.raw(t ? ",{" : "{");
      o.key("i");
      o.arr(st.rot_idx.data() + t * k, static_cast<size_t>(k));
      o.raw(",");
      o.key("q");
      o.arr(st.rot_q.data() + t * k * k, static_cast<size_t>(k) * k);
      o.raw("}");
    }
    o.raw("]}");
  }
  o.raw("],\n");
  o.key("version");
  o.num(static_cast<int64_t>(kVersion));
  o.raw("}\n");
  return std::move(o.b);
}

// A loaded factorization drives device kernels that index arrays by these
// values (operator.cu): reject anything out of range as PMMF_DATA instead
// of corrupting memory.  k bounds the operator's per-rotation registers
// (kMaxK = 8, factorizer.hpp:44-46 allows k >= 2).
void validate_result(const Result& r) {
  auto bad = [](const char* what) { fail(PMMF_DATA, std::string("factorization file: ") + what); };
  if (r.n < 0) bad("negative n");
  if (r.k < 2 || r.k > 8) bad("params.k outside [2, 8]");
  auto in_range = [&](int64_t i) { return i >= 0 && i < r.n; };
  for (const Result::Stage& st : r.stages) {
    if (st.off.empty() || st.off.front() != 0 || st.off.back() != static_cast<int64_t>(st.members.size()))
      bad("inconsistent partition offsets");
    for (size_t u = 0; u + 1 < st.off.size(); ++u)
      if (st.off[u + 1] < st.off[u]) bad("inconsistent partition offsets");
    for (int64_t m : st.members)
      if (!in_range(m)) bad("partition member out of range");
    for (int64_t b : st.bypassed)
      if (!in_range(b)) bad("bypassed index out of range");
    for (int64_t i : st.rot_idx)
      if (!in_range(i)) bad("rotation index out of range");
    for (int64_t i : st.elim_idx)
      if (!in_range(i)) bad("eliminated index out of range");
    if (st.rot_q.size() != st.rot_idx.size() * static_cast<size_t>(r.k)) bad("rotation matrix size mismatch");
  }
  for (int64_t i : r.core_idx)
    if (!in_range(i)) bad("core index out of range");
  for (const auto& d : r.diag)
    if (!in_range(d.first)) bad("diagonal index out of range");
  if (r.hist.size() > 0)
    for (int64_t h : r.hist)
      if (h < 0 || h > r.n) bad("active history out of range");
}

std::unique_ptr<Result> factorization_from_json(const char* text, size_t len) {  // serialize.hpp:112-165
  JVal j;
  Parser ps{text, text + len, text};
  ps.value(j, 0);
  ps.ws();
  if (ps.p != ps.e) ps.bad("trailing characters");
  const JVal* fmt = j.find("format");
  if (!fmt || fmt->t != JVal::Str || fmt->s != kFormat) fail(PMMF_DATA, "factorization file: unknown format");
  const JVal* ver = j.find("version");
  if (!ver || ver->t != JVal::Num || !ver->is_int || ver->as_int() != kVersion)
    fail(PMMF_DATA, "factorization file: unsupported version");
  auto r = std::make_unique<Result>();
  r->n = j.at("n").as_int();
  r->residual_sq = j.at("residual_sq").as_double();
  r->hist = ints(j.at("active_history"));
  {  // serialize.hpp:44-59
    const JVal& pj = j.at("params");
    pmmf_b200_params& p = r->params;
    p.k = static_cast<int32_t>(pj.at("k").as_int());
    p.n_stages = static_cast<int32_t>(pj.at("n_stages").as_int());
    p.eta = pj.at("eta").as_double();
    p.core_min = pj.at("core_min").as_int();
    p.core_cap = pj.at("core_cap").as_int();
    p.seed = pj.at("seed").as_u64();
    const JVal& c = pj.at("cluster");
    p.m_target = c.at("m_target").as_int();
    p.c_min = c.at("c_min").as_int();
    p.c_max = c.at("c_max").as_int();
    p.d_max = static_cast<int32_t>(c.at("d_max").as_int());
    p.bypass_enabled = c.at("bypass").as_bool() ? 1 : 0;
    p.cluster_seed = c.at("seed").as_u64();
    r->k = p.k;
    if (r->k < 2 || r->k > 8) fail(PMMF_DATA, "factorization file: params.k outside [2, 8]");
    if (r->n < 0) fail(PMMF_DATA, "factorization file: negative n");
  }
  int k = r->k;
  for (const JVal& js : j.at("stages").arr()) {
    Result::Stage st;
    st.off.push_back(0);
    for (const JVal& jc : js.at("partition").arr()) {
      for (const JVal& x : jc.arr()) st.members.push_back(x.as_int());
      st.off.push_back(static_cast<int64_t>(st.members.size()));
    }
    st.bypassed = ints(js.at("bypassed"));
    for (const JVal& jr : js.at("rotations").arr()) {
      const std::vector<int64_t> idx = ints(jr.at("i"));
      const std::vector<JVal>& q = jr.at("q").arr();
      if (static_cast<int>(idx.size()) != k) {
        // the reference allows any order per rotation; this container keeps
        // one k per factorization (FactorizeParams::k)
        fail(PMMF_DATA, "factorization file: rotation order differs from params.k");
      }
      if (q.size() != static_cast<size_t>(k) * k) fail(PMMF_DATA, "factorization file: rotation matrix size mismatch");
      st.rot_idx.insert(st.rot_idx.end(), idx.begin(), idx.end());
      for (const JVal& x : q) st.rot_q.push_back(x.as_double());
    }
    for (const JVal& je : js.at("eliminated").arr()) {
      st.elim_idx.push_back(je.at("i").as_int());
      st.elim_diag.push_back(je.at("d").as_double());
      st.elim_mass.push_back(je.at("m").as_double());
    }
    r->stages.push_back(std::move(st));
  }
  r->core_idx = ints(j.at("core").at("indices"));
  {
    const std::vector<JVal>& cv = j.at("core").at("dense").arr();
    const size_t g = r->core_idx.size();
    if (cv.size() != g * g) fail(PMMF_DATA, "factorization file: core size mismatch");
    r->core.reserve(cv.size());
    for (const JVal& x : cv) r->core.push_back(x.as_double());
  }
  for (const JVal& jd : j.at("diagonal").arr()) r->diag.emplace_back(jd.at("i").as_int(), jd.at("d").as_double());
  r->trivial = r->stages.empty();
  validate_result(*r);
  return r;
}

void save_factorization(const Result& r, const std::string& path) {  // serialize.hpp:167-171
  std::ofstream out(path, std::ios::binary);
  if (!out) fail(PMMF_DATA, "cannot open '" + path + "' for writing");
  const std::string s = factorization_to_json(r);
  out.write(s.data(), static_cast<std::streamsize>(s.size()));
  if (!out) fail(PMMF_DATA, "cannot write '" + path + "'");
}

std::unique_ptr<Result> load_factorization(const std::string& path) {  // serialize.hpp:173-183
  std::ifstream in(path, std::ios::binary);
  if (!in) fail(PMMF_DATA, "cannot open '" + path + "'");
  std::ostringstream ss;
  ss << in.rdbuf();
  const std::string s = ss.str();
  return factorization_from_json(s.data(), s.size());
}

}  // namespace pmmf_b200
