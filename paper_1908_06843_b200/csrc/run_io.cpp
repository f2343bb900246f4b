// Run I/O and the training driver around the GPU engines (see run_io.hpp).
//
// Written from the formats, not from the reference's sources:
//   * PRSPAR01 arrays (array_io.hpp:25-28): 8 magic bytes, rows and cols as
//     little-endian u64, then rows·cols little-endian f64 in row-major order;
//   * datasets: PRSPAR01 when the magic matches, else headerless comma-separated
//     numbers, one data point per non-empty line;
//   * SHA-256: FIPS 180-4 (section 6.2);
//   * the run directory a prsp run leaves (free_energy.csv, checkpoint_* /
//     final_* / abort_* arrays, a prsp-manifest-1 JSON manifest) and the EM
//     driver contract of prsp::run (em.cpp): T and weight-noise schedules read at
//     the iteration's position in the budget, the tolerance stop on inert
//     iterations, and params_to_arrays naming (model.cpp:77-130).
#include "run_io.hpp"

#include <algorithm>
#include <array>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <memory>
#include <sstream>

#include "bsc_engine.hpp"
#include "mca_engine.hpp"
#include "rng_stream.hpp"

namespace bscgpu {

namespace fs = std::filesystem;

namespace {

// ====================================================================== bytes
std::vector<char> read_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary | std::ios::ate);
  if (!f) throw Error(kData, "cannot open file: " + path);
  const std::streamoff size = f.tellg();
  std::vector<char> buf(static_cast<size_t>(std::max<std::streamoff>(size, 0)));
  f.seekg(0);
  if (!buf.empty() && !f.read(buf.data(), static_cast<std::streamsize>(buf.size())))
    throw Error(kData, "read failed: " + path);
  return buf;
}

void write_file(const std::string& path, const std::vector<std::pair<const void*, size_t>>& parts) {
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw Error(kData, "cannot write file: " + path);
  for (const auto& [p, n] : parts) f.write(static_cast<const char*>(p), static_cast<std::streamsize>(n));
  if (!f) throw Error(kData, "write failed: " + path);
}

// ================================================================= PRSPAR01
constexpr std::array<char, 8> kPrsparMagic{'P', 'R', 'S', 'P', 'A', 'R', '0', '1'};
constexpr size_t kPrsparHeader = 8 + 2 * sizeof(uint64_t);

uint64_t get_le64(const char* p) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | static_cast<unsigned char>(p[i]);
  return v;
}
void put_le64(char* p, uint64_t v) {
  for (int i = 0; i < 8; ++i) p[i] = static_cast<char>((v >> (8 * i)) & 0xff);
}
bool has_magic(const std::vector<char>& b, size_t n) {
  return b.size() >= n && std::equal(kPrsparMagic.begin(), kPrsparMagic.begin() + n, b.begin());
}

Array decode_prspar(const std::vector<char>& b, const std::string& path) {
  if (!has_magic(b, 8)) throw Error(kData, path + ": bad PRSPAR01 magic");
  if (b.size() < kPrsparHeader) throw Error(kData, path + ": PRSPAR01 header cut short");
  Array a;
  a.rows = get_le64(b.data() + 8);
  a.cols = get_le64(b.data() + 16);
  uint64_t count = 0, bytes = 0;
  // shapes whose payload could not exist on any file system (or overflow) are refused
  if (__builtin_mul_overflow(a.rows, a.cols, &count) || __builtin_mul_overflow(count, 8ull, &bytes) ||
      bytes > (1ull << 51))
    throw Error(kData, path + ": PRSPAR01 shape " + std::to_string(a.rows) + "x" + std::to_string(a.cols) +
                           " is not plausible");
  if (b.size() - kPrsparHeader < bytes)
    throw Error(kData, path + ": PRSPAR01 payload has " + std::to_string(b.size() - kPrsparHeader) +
                           " bytes, the header needs " + std::to_string(bytes));
  a.data.resize(count);
  if (bytes) std::memcpy(a.data.data(), b.data() + kPrsparHeader, bytes);  // little-endian hosts
  return a;
}

// ===================================================================== CSV
// Fields are numbers (std::from_chars: correctly rounded) with optional spaces
// on either side; lines may end in CR LF; blank lines carry no data point.
Array decode_csv(const std::vector<char>& b, const std::string& path) {
  Array a;
  const char* p = b.data();
  const char* const end = p + b.size();
  for (size_t line = 1; p < end; ++line) {
    const char* eol = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
    const char* stop = eol ? eol : end;
    const char* next = eol ? eol + 1 : end;
    if (stop > p && stop[-1] == '\r') --stop;
    if (stop == p) {  // blank line
      p = next;
      continue;
    }
    auto where = [&] { return path + ": line " + std::to_string(line) + ": "; };
    uint64_t fields = 0;
    for (const char* q = p;;) {
      while (q < stop && *q == ' ') ++q;
      double v;
      const auto r = std::from_chars(q, stop, v);
      if (r.ec != std::errc()) throw Error(kData, where() + "field " + std::to_string(fields + 1) + " is not a number");
      a.data.push_back(v);
      ++fields;
      q = r.ptr;
      while (q < stop && *q == ' ') ++q;
      if (q == stop) break;
      if (*q++ != ',') throw Error(kData, where() + "fields must be separated by ','");
    }
    if (a.rows == 0) a.cols = fields;
    if (fields != a.cols)
      throw Error(kData, where() + std::to_string(fields) + " fields where the first data line has " +
                             std::to_string(a.cols));
    ++a.rows;
    p = next;
  }
  if (a.rows == 0) throw Error(kData, path + ": no data points");
  return a;
}

// ================================================================= SHA-256
// FIPS 180-4 §6.2: 64-byte blocks, a 16-word rolling message schedule.
constexpr uint32_t kShaK[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

struct ShaState {
  std::array<uint32_t, 8> h{0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                            0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
  uint64_t length = 0;  // bytes absorbed

  static uint32_t ror(uint32_t x, unsigned r) { return (x >> r) | (x << (32u - r)); }

  void compress(const unsigned char* m) {
    uint32_t w[16];
    for (int t = 0; t < 16; ++t)
      w[t] = (uint32_t{m[4 * t]} << 24) | (uint32_t{m[4 * t + 1]} << 16) | (uint32_t{m[4 * t + 2]} << 8) |
             uint32_t{m[4 * t + 3]};
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], k = h[7];
    for (int t = 0; t < 64; ++t) {
      if (t >= 16) {  // W_t from the 16 previous words, kept in a ring
        const uint32_t x = w[(t + 1) & 15], y = w[(t + 14) & 15];
        w[t & 15] += (ror(x, 7) ^ ror(x, 18) ^ (x >> 3)) + w[(t + 9) & 15] + (ror(y, 17) ^ ror(y, 19) ^ (y >> 10));
      }
      const uint32_t s1 = ror(e, 6) ^ ror(e, 11) ^ ror(e, 25), ch = (e & f) ^ (~e & g);
      const uint32_t s0 = ror(a, 2) ^ ror(a, 13) ^ ror(a, 22), maj = (a & b) ^ (a & c) ^ (b & c);
      const uint32_t t1 = k + s1 + ch + kShaK[t] + w[t & 15], t2 = s0 + maj;
      k = g;
      g = f;
      f = e;
      e = d + t1;
      d = c;
      c = b;
      b = a;
      a = t1 + t2;
    }
    h[0] += a, h[1] += b, h[2] += c, h[3] += d, h[4] += e, h[5] += f, h[6] += g, h[7] += k;
  }

  // absorb whole blocks; returns the bytes left over (< 64)
  size_t absorb(const unsigned char* p, size_t n) {
    const size_t full = n / 64 * 64;
    for (size_t o = 0; o < full; o += 64) compress(p + o);
    length += full;
    return n - full;
  }

  // the final block(s): tail, 0x80, zeros, the message length in bits (big-endian)
  std::string finish(const unsigned char* tail, size_t n) {
    unsigned char last[128] = {};
    std::memcpy(last, tail, n);
    last[n] = 0x80;
    const size_t blocks = n + 1 + 8 <= 64 ? 1 : 2;
    const uint64_t bits = (length + n) * 8;
    for (int i = 0; i < 8; ++i) last[64 * blocks - 1 - i] = static_cast<unsigned char>(bits >> (8 * i));
    for (size_t i = 0; i < blocks; ++i) compress(last + 64 * i);
    std::string hex;
    hex.reserve(64);
    for (uint32_t v : h) {
      char buf[9];
      std::snprintf(buf, sizeof buf, "%08x", v);
      hex += buf;
    }
    return hex;
  }
};

// ==================================================================== JSON
// A small JSON tree: written by the manifest writer, read back by load_run.
struct JsonValue {
  enum class T { Null, Bool, Num, Int, Str, Arr, Obj } t = T::Null;
  bool b = false;
  double num = 0.0;
  uint64_t i = 0;
  std::string s;
  std::vector<JsonValue> a;
  std::vector<std::pair<std::string, JsonValue>> o;

  static JsonValue integer(uint64_t v) {
    JsonValue j;
    j.t = T::Int;
    j.i = v;
    j.num = static_cast<double>(v);
    return j;
  }
  static JsonValue number(double v) {
    JsonValue j;
    j.t = T::Num;
    j.num = v;
    return j;
  }
  static JsonValue string(std::string v) {
    JsonValue j;
    j.t = T::Str;
    j.s = std::move(v);
    return j;
  }
  static JsonValue array(std::vector<JsonValue> v = {}) {
    JsonValue j;
    j.t = T::Arr;
    j.a = std::move(v);
    return j;
  }
  static JsonValue object() {
    JsonValue j;
    j.t = T::Obj;
    return j;
  }
  JsonValue& set(const std::string& k, JsonValue v) {
    o.emplace_back(k, std::move(v));
    return *this;
  }
  const JsonValue* find(const std::string& k) const {
    auto it = std::find_if(o.begin(), o.end(), [&](const auto& kv) { return kv.first == k; });
    return it == o.end() ? nullptr : &it->second;
  }
  double as_num() const { return num; }
};

void json_quote(std::string& out, const std::string& s) {
  out += '"';
  for (unsigned char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\t': out += "\\t"; break;
      case '\r': out += "\\r"; break;
      default:
        if (c < 0x20) {
          char u[8];
          std::snprintf(u, sizeof u, "\\u%04x", c);
          out += u;
        } else {
          out += static_cast<char>(c);
        }
    }
  }
  out += '"';
}

// 2-space indentation, one element per line; doubles shortest round-trip with
// a ".0" on integral values so readers keep them floating point
void json_write(std::string& out, const JsonValue& v, int depth) {
  const std::string pad(2 * (depth + 1), ' '), close(2 * depth, ' ');
  switch (v.t) {
    case JsonValue::T::Null: out += "null"; return;
    case JsonValue::T::Bool: out += v.b ? "true" : "false"; return;
    case JsonValue::T::Int: out += std::to_string(v.i); return;
    case JsonValue::T::Num: {
      std::string s = format_double(v.num);
      if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
      out += s;
      return;
    }
    case JsonValue::T::Str: json_quote(out, v.s); return;
    case JsonValue::T::Arr:
      if (v.a.empty()) {
        out += "[]";
        return;
      }
      out += "[\n";
      for (size_t k = 0; k < v.a.size(); ++k) {
        out += pad;
        json_write(out, v.a[k], depth + 1);
        out += k + 1 < v.a.size() ? ",\n" : "\n";
      }
      out += close + "]";
      return;
    case JsonValue::T::Obj:
      out += "{\n";
      for (size_t k = 0; k < v.o.size(); ++k) {
        out += pad;
        json_quote(out, v.o[k].first);
        out += ": ";
        json_write(out, v.o[k].second, depth + 1);
        out += k + 1 < v.o.size() ? ",\n" : "\n";
      }
      out += close + "}";
      return;
  }
}

class JsonReader {
 public:
  JsonReader(const std::string& text, std::string where) : p_(text.data()), end_(p_ + text.size()), w_(std::move(where)) {}
  JsonValue document() {
    JsonValue v = value();
    skip();
    if (p_ != end_) bad("unexpected text after the top-level value");
    return v;
  }

 private:
  [[noreturn]] void bad(const std::string& why) { throw Error(kData, w_ + ": malformed manifest: " + why); }
  void skip() {
    while (p_ < end_ && (*p_ == ' ' || *p_ == '\t' || *p_ == '\n' || *p_ == '\r')) ++p_;
  }
  bool eat(char c) {
    skip();
    if (p_ < end_ && *p_ == c) {
      ++p_;
      return true;
    }
    return false;
  }
  bool word(const char* w) {
    const size_t n = std::strlen(w);
    if (static_cast<size_t>(end_ - p_) >= n && std::memcmp(p_, w, n) == 0) {
      p_ += n;
      return true;
    }
    return false;
  }
  std::string text() {
    if (!eat('"')) bad("a string was expected");
    std::string s;
    while (p_ < end_ && *p_ != '"') {
      char c = *p_++;
      if (c == '\\') {
        if (p_ >= end_) break;
        const char e = *p_++;
        c = e == 'n' ? '\n' : e == 't' ? '\t' : e == 'r' ? '\r' : e == 'b' ? '\b' : e == 'f' ? '\f' : e;
        if (e == 'u') {  // \uXXXX below 0x80 (all this writer emits)
          if (end_ - p_ < 4) bad("short \\u escape");
          c = static_cast<char>(std::stoi(std::string(p_, 4), nullptr, 16));
          p_ += 4;
        }
      }
      s += c;
    }
    if (p_ >= end_) bad("a string is not terminated");
    ++p_;
    return s;
  }
  JsonValue value() {
    skip();
    if (p_ >= end_) bad("the document ends early");
    JsonValue v;
    if (*p_ == '{') {
      ++p_;
      v = JsonValue::object();
      if (eat('}')) return v;
      do {
        std::string k = text();
        if (!eat(':')) bad("':' expected after a key");
        v.o.emplace_back(std::move(k), value());
      } while (eat(','));
      if (!eat('}')) bad("'}' expected");
      return v;
    }
    if (*p_ == '[') {
      ++p_;
      v = JsonValue::array();
      if (eat(']')) return v;
      do v.a.push_back(value());
      while (eat(','));
      if (!eat(']')) bad("']' expected");
      return v;
    }
    if (*p_ == '"') return JsonValue::string(text());
    if (word("null")) return v;
    if (word("true") || word("false")) {
      v.t = JsonValue::T::Bool;
      v.b = p_[-1] == 'e' && p_[-2] == 'u';
      return v;
    }
    v.t = JsonValue::T::Num;
    const auto r = std::from_chars(p_, end_, v.num);
    if (r.ec != std::errc()) bad("a value was expected");
    p_ = r.ptr;
    return v;
  }
  const char* p_;
  const char* end_;
  std::string w_;
};

// ======================================================== model parameters
// The host copy of a model's parameters, named as params_to_arrays names them.
struct HostParams {
  std::vector<double> w;
  double pi = 0.0, sigma2 = 1.0;
  std::vector<double> values, probs;  // dsc

  std::vector<NamedArray> named(uint32_t d, uint32_t h) const {
    std::vector<NamedArray> out{{"W", Array{d, h, w}}, {"sigma2", Array{1, 1, {sigma2}}}};
    if (values.empty()) {
      out.push_back({"pi", Array{1, 1, {pi}}});
    } else {
      out.push_back({"values", Array{1, values.size(), values}});
      out.push_back({"probs", Array{1, probs.size(), probs}});
    }
    return out;
  }
};

bool is_linear_family(const std::string& m) { return m == "bsc" || m == "tsc" || m == "dsc"; }
bool is_max_family(const std::string& m) { return m == "mca" || m == "mmca"; }

// The model families on the GPU path, each behind its engine.
class Engine {
 public:
  Engine(const RunConfig& c, uint32_t d) : c_(c), d_(d) {
    if (c.model != "dsc" && !c.values.empty())
      throw Error(kConfig, "model " + c.model + " does not take a value alphabet");
    const uint32_t hp = c.hprime ? c.hprime : c.latents, g = c.gamma ? c.gamma : hp;
    if (is_linear_family(c.model)) {
      const int fam = c.model == "bsc" ? kBsc : c.model == "tsc" ? kTsc : kDsc;
      lin_ = std::make_unique<BscEngine>(fam, d, c.latents, hp, g, 1000000, c.values.empty() ? nullptr : c.values.data(),
                                         static_cast<uint32_t>(c.values.size()), c.device);
    } else if (is_max_family(c.model)) {
      max_ = std::make_unique<McaEngine>(c.model == "mca" ? 0 : 1, c.soft_winner_rho, d, c.latents, hp, g, 1000000,
                                         c.device);
    } else {
      throw Error(kConfig, "gpu: model '" + c.model + "' is not on the GPU path (bsc, tsc, dsc, mca, mmca)");
    }
  }

  void load(const double* y, uint64_t n) { lin_ ? lin_->load_data(y, n, false) : max_->load_data(y, n); }

  void put(const HostParams& p) {
    if (lin_)
      lin_->set_params_ex(p.w.data(), p.pi, p.sigma2, p.probs.empty() ? nullptr : p.probs.data(),
                          static_cast<uint32_t>(p.probs.size()));
    else
      max_->set_params(p.w.data(), p.pi, p.sigma2);
  }

  HostParams take() {
    HostParams p;
    p.w.assign(static_cast<size_t>(d_) * c_.latents, 0.0);
    if (max_) {
      max_->get_params(p.w.data(), &p.pi, &p.sigma2);
      return p;
    }
    if (c_.model == "dsc") {
      p.values = lin_->alphabet();
      p.probs.assign(p.values.size(), 0.0);
    }
    lin_->get_params_ex(p.w.data(), &p.pi, &p.sigma2, p.probs.empty() ? nullptr : p.probs.data());
    return p;
  }

  double step(double temperature) { return lin_ ? lin_->step(temperature) : max_->step(temperature); }

  void inference(double* ms, double* mm, double* ex) {
    lin_ ? lin_->inference(ms, mm, ex) : max_->inference(ms, mm, ex);
  }

  const std::vector<double>& alphabet() const { return lin_->alphabet(); }

 private:
  RunConfig c_;
  uint32_t d_;
  std::unique_ptr<BscEngine> lin_;
  std::unique_ptr<McaEngine> max_;
};

// Model::standard_init of the families (linear_discrete.cpp:129-148,
// max_causes.cpp:121-130): W = column mean + sqrt(data variance / H)·N(0,1)
// (mca: |·| floored at 1e-8), σ² = the mean data variance, π = H'/(2H); dsc puts
// H'/(2H) of the mass on the non-zero values evenly.
HostParams initial_params(const RunConfig& c, const Engine& eng, const double* y, uint64_t n, uint32_t d,
                          Stream& rng) {
  if (n < 2) throw Error(kData, "standard_init requires at least two data points");
  std::vector<double> mean(d, 0.0);
  for (uint64_t r = 0; r < n; ++r)
    for (uint32_t j = 0; j < d; ++j) mean[j] += y[r * d + j];
  for (double& m : mean) m /= static_cast<double>(n);
  double ss = 0.0;
  for (uint64_t r = 0; r < n; ++r)
    for (uint32_t j = 0; j < d; ++j) ss += (y[r * d + j] - mean[j]) * (y[r * d + j] - mean[j]);
  const double var = ss / static_cast<double>(n * d);
  const uint32_t h = c.latents;
  const double spread = var > 0.0 ? std::sqrt(var / h) : 0.0;
  HostParams p;
  p.w.resize(static_cast<size_t>(d) * h);
  for (uint32_t j = 0; j < d; ++j)
    for (uint32_t k = 0; k < h; ++k) {
      const double v = mean[j] + spread * rng.normal();
      p.w[static_cast<size_t>(j) * h + k] = c.model == "mca" ? std::max(std::abs(v), 1e-8) : v;
    }
  p.sigma2 = std::max(var, 1e-12);
  const double hp = static_cast<double>(std::min(c.hprime ? c.hprime : h, h)), hh = static_cast<double>(h);
  const double frac = hp / (2.0 * hh);
  if (c.model == "dsc") {
    p.values = eng.alphabet();
    const double k = static_cast<double>(p.values.size());
    for (double v : p.values) p.probs.push_back(v == 0.0 ? 1.0 - frac * (1.0 - 1.0 / k) : hp / (2.0 * hh * k));
  } else {
    p.pi = frac;
  }
  return p;
}

// Weight noise of a step (perturb_weights, linear_discrete.cpp:510-514 and
// max_causes.cpp:476-484): every column gets N(0, (std·rms(column))²) noise,
// then mca floors W at 1e-8.
void add_weight_noise(HostParams& p, const RunConfig& c, uint32_t d, double std_dev, Stream& rng) {
  const uint32_t h = c.latents;
  std::vector<double> rms(h, 0.0);
  for (uint32_t j = 0; j < d; ++j)
    for (uint32_t k = 0; k < h; ++k) rms[k] += p.w[static_cast<size_t>(j) * h + k] * p.w[static_cast<size_t>(j) * h + k];
  for (double& r : rms) r = std::sqrt(r / d);
  for (uint32_t j = 0; j < d; ++j)
    for (uint32_t k = 0; k < h; ++k) p.w[static_cast<size_t>(j) * h + k] += std_dev * rms[k] * rng.normal();
  if (c.model == "mca")
    for (double& v : p.w) v = std::max(v, 1e-8);
}

// ============================================================ run directory
class RunDirectory {
 public:
  explicit RunDirectory(std::string dir) : dir_(std::move(dir)) {
    if (dir_.empty()) return;
    fs::create_directories(dir_);
    trace_.open(fs::path(dir_) / "free_energy.csv", std::ios::trunc);
    if (!trace_) throw Error(kData, "cannot write trace in " + dir_);
    trace_ << "iteration,free_energy,seconds\n" << std::flush;
  }
  bool active() const { return !dir_.empty(); }

  void record(size_t iteration, double f, double seconds, const std::vector<NamedArray>& params) {
    if (!active()) return;
    trace_ << iteration << ',' << format_double(f) << ',' << format_double(seconds) << '\n' << std::flush;
    size_t floats = 0;
    for (const auto& p : params) floats += p.a.data.size();
    if (iteration % (floats < 1000000 ? 1 : 10) == 0) save("checkpoint", params);  // checkpoint cadence
  }

  std::vector<std::string> save(const std::string& prefix, const std::vector<NamedArray>& params) const {
    std::vector<std::string> names;
    if (!active()) return names;
    for (const auto& p : params) {
      names.push_back(prefix + "_" + p.name + ".prsp");
      save_array((fs::path(dir_) / names.back()).string(), p.a.data.data(), p.a.rows, p.a.cols);
    }
    return names;
  }

  const std::string& path() const { return dir_; }

 private:
  std::string dir_;
  std::ofstream trace_;
};

const Array& param_named(const std::vector<NamedArray>& v, const char* name) {
  for (const auto& p : v)
    if (p.name == name) return p.a;
  throw Error(kData, std::string("run: missing parameter array ") + name);
}

}  // namespace

// ======================================================================== API
void save_array(const std::string& path, const double* data, uint64_t rows, uint64_t cols) {
  char head[kPrsparHeader];
  std::copy(kPrsparMagic.begin(), kPrsparMagic.end(), head);
  put_le64(head + 8, rows);
  put_le64(head + 16, cols);
  write_file(path, {{head, sizeof head}, {data, static_cast<size_t>(rows * cols * sizeof(double))}});
}

Array load_array(const std::string& path) { return decode_prspar(read_file(path), path); }

Array load_csv(const std::string& path) { return decode_csv(read_file(path), path); }

Array load_dataset(const std::string& path) {
  const std::vector<char> b = read_file(path);
  if (has_magic(b, 8)) return decode_prspar(b, path);
  if (has_magic(b, 4)) throw Error(kData, path + ": starts like PRSPAR01 but is not one");
  return decode_csv(b, path);
}

std::string format_double(double v) {
  std::array<char, 32> buf;
  const auto r = std::to_chars(buf.data(), buf.data() + buf.size(), v);  // shortest round-trip form
  if (r.ec != std::errc()) throw Error(kInternal, "format_double failed");
  return std::string(buf.data(), r.ptr);
}

std::string sha256_hex(const void* data, size_t n) {
  ShaState st;
  const auto* p = static_cast<const unsigned char*>(data);
  const size_t rest = st.absorb(p, n);
  return st.finish(p + (n - rest), rest);
}

std::string sha256_hex_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw Error(kData, "cannot open file: " + path);
  ShaState st;
  std::vector<unsigned char> buf((1u << 20) + 64);
  size_t held = 0;  // bytes carried over from the previous read (< 64)
  for (;;) {
    f.read(reinterpret_cast<char*>(buf.data()) + held, static_cast<std::streamsize>(buf.size() - held));
    const size_t got = held + static_cast<size_t>(f.gcount());
    const size_t rest = st.absorb(buf.data(), got);
    std::memmove(buf.data(), buf.data() + (got - rest), rest);
    held = rest;
    if (!f) break;
  }
  return st.finish(buf.data(), held);
}

// Piecewise-linear over the anchors, constant beyond the first and last.
void Schedule::validate() const {
  if (anchors.empty()) throw Error(kConfig, "schedule: at least one anchor required");
  double last = -1.0;
  for (const auto& [pos, val] : anchors) {
    if (!std::isfinite(pos) || !std::isfinite(val)) throw Error(kConfig, "schedule: anchors must be finite");
    if (pos < 0.0 || pos > 1.0) throw Error(kConfig, "schedule: anchor positions must lie in [0,1]");
    if (pos <= last) throw Error(kConfig, "schedule: anchor positions must be strictly increasing");
    last = pos;
  }
}

double Schedule::value_at(double position) const {
  if (position <= anchors.front().first) return anchors.front().second;
  if (position >= anchors.back().first) return anchors.back().second;
  // the segment (x0, x1] holding the position
  const auto hi = std::lower_bound(anchors.begin(), anchors.end(), position,
                                   [](const std::pair<double, double>& a, double x) { return a.first < x; });
  const auto& [x0, y0] = *(hi - 1);
  const auto& [x1, y1] = *hi;
  return y0 + (position - x0) / (x1 - x0) * (y1 - y0);
}

void write_manifest(const std::string& path, const RunConfig& c, const std::vector<std::string>& files) {
  auto sched = [](const Schedule& s) {
    JsonValue a = JsonValue::array();
    for (const auto& [pos, val] : s.anchors) a.a.push_back(JsonValue::array({JsonValue::number(pos), JsonValue::number(val)}));
    return a;
  };
  JsonValue m = JsonValue::object();
  m.set("format", JsonValue::string("prsp-manifest-1"))
      .set("library", JsonValue::string("0.1.0"))  // core.hpp kVersion of the reference build it mirrors
      .set("rng", JsonValue::string("mt19937_64/box-muller"))
      .set("model", JsonValue::string(c.model))
      .set("dim", JsonValue::integer(c.dim))
      .set("latents", JsonValue::integer(c.latents));
  if (c.model != "gmm" && c.model != "pmm") m.set("hprime", JsonValue::integer(c.hprime)).set("gamma", JsonValue::integer(c.gamma));
  if (c.model == "dsc") {
    JsonValue v = JsonValue::array();
    for (double x : c.values) v.a.push_back(JsonValue::number(x));
    m.set("values", v);
  }
  m.set("iterations", JsonValue::integer(c.iterations))
      .set("seed", JsonValue::integer(c.seed))
      .set("workers", JsonValue::integer(c.workers))
      .set("shards", JsonValue::integer(c.shards))
      .set("tolerance", c.tolerance ? JsonValue::number(*c.tolerance) : JsonValue())
      .set("temperature", sched(c.temperature))
      .set("w_noise", sched(c.w_noise));
  JsonValue data = JsonValue::object();
  data.set("file", JsonValue::string(c.data_file))
      .set("sha256", JsonValue::string(c.data_sha256))
      .set("rows", JsonValue::integer(c.data_rows))
      .set("cols", JsonValue::integer(c.data_cols));
  m.set("data", data);
  JsonValue params = JsonValue::array();
  for (const auto& f : files) params.a.push_back(JsonValue::string(f));
  m.set("parameters", params);
  std::string text;
  json_write(text, m, 0);
  text += '\n';
  write_file(path, {{text.data(), text.size()}});
}

RunConfig read_manifest(const std::string& path) {
  const std::vector<char> raw = read_file(path);
  const JsonValue j = JsonReader(std::string(raw.begin(), raw.end()), path).document();
  auto field = [&](const JsonValue& o, const char* k) -> const JsonValue& {
    const JsonValue* v = o.find(k);
    if (!v) throw Error(kData, path + ": malformed manifest: missing '" + k + "'");
    return *v;
  };
  const JsonValue* fmt = j.find("format");
  if (!fmt || fmt->s != "prsp-manifest-1") throw Error(kData, path + ": unknown manifest format");
  auto u64 = [&](const JsonValue& o, const char* k) { return static_cast<uint64_t>(field(o, k).as_num()); };
  auto sched = [&](const char* k) {
    Schedule s;
    for (const auto& pair : field(j, k).a) {
      if (pair.a.size() != 2) throw Error(kData, path + ": malformed manifest: schedule anchors are [position, value]");
      s.anchors.emplace_back(pair.a[0].as_num(), pair.a[1].as_num());
    }
    return s;
  };
  RunConfig c;
  c.model = field(j, "model").s;
  c.dim = static_cast<uint32_t>(u64(j, "dim"));
  c.latents = static_cast<uint32_t>(u64(j, "latents"));
  c.hprime = j.find("hprime") ? static_cast<uint32_t>(u64(j, "hprime")) : c.latents;
  c.gamma = j.find("gamma") ? static_cast<uint32_t>(u64(j, "gamma")) : c.hprime;
  if (const JsonValue* v = j.find("values"))
    for (const auto& x : v->a) c.values.push_back(x.as_num());
  c.iterations = u64(j, "iterations");
  c.seed = u64(j, "seed");
  c.workers = static_cast<uint32_t>(u64(j, "workers"));
  c.shards = static_cast<uint32_t>(u64(j, "shards"));
  if (field(j, "tolerance").t != JsonValue::T::Null) c.tolerance = field(j, "tolerance").as_num();
  c.temperature = sched("temperature");
  c.w_noise = sched("w_noise");
  const JsonValue& d = field(j, "data");
  c.data_file = field(d, "file").s;
  c.data_sha256 = field(d, "sha256").s;
  c.data_rows = u64(d, "rows");
  c.data_cols = u64(d, "cols");
  return c;
}

// The EM driver (prsp::run semantics, em.cpp): iteration t = 1..T sits at
// position t/T of the budget, where the temperature (≥ 1) and the weight-noise
// level (≥ 0) are read; one GPU step per iteration; weight noise, when on, is
// applied to the new parameters; a non-finite F aborts (abort_* arrays); with a
// tolerance, an inert iteration (T = 1, no noise) whose F moved by at most
// tol·(1 + |F|) ends the run.
TrainResult train_run(RunConfig& cfg, const double* y, uint64_t n, uint64_t d, const std::string& data_file,
                      const std::string& out_dir) {
  if (n == 0) throw Error(kData, "run: empty dataset");
  if (cfg.iterations == 0) throw Error(kConfig, "annealing: max_iterations must be >= 1");
  cfg.temperature.validate();
  cfg.w_noise.validate();
  if (cfg.tolerance && !(*cfg.tolerance >= 0.0)) throw Error(kConfig, "run: convergence tolerance must be >= 0");
  if (cfg.shards == 0 || cfg.workers == 0) throw Error(kConfig, "shard plan: shards and workers must be >= 1");
  cfg.dim = static_cast<uint32_t>(d);
  if (!cfg.hprime) cfg.hprime = cfg.latents;
  if (!cfg.gamma) cfg.gamma = cfg.hprime;
  cfg.data_rows = n;
  cfg.data_cols = d;
  cfg.data_file = data_file.empty() ? "(memory)" : data_file;
  cfg.data_sha256 = data_file.empty() ? sha256_hex(y, n * d * sizeof(double)) : sha256_hex_file(data_file);

  Engine eng(cfg, cfg.dim);
  Stream init_rng = Stream::derived(cfg.seed, 0x696e6974ULL);   // "init"
  Stream noise_rng = Stream::derived(cfg.seed, 0x6e6f6973ULL);  // "nois"
  HostParams params = initial_params(cfg, eng, y, n, cfg.dim, init_rng);
  if (cfg.model == "dsc") cfg.values = params.values;  // the sorted alphabet the model holds
  eng.load(y, n);
  eng.put(params);

  RunDirectory run(out_dir);
  TrainResult res;
  auto converged = [&](double f, bool inert) {
    return cfg.tolerance && inert && !res.trace.empty() &&
           std::abs(f - res.trace.back()) <= *cfg.tolerance * (1.0 + std::abs(f));
  };
  for (uint64_t t = 1; t <= cfg.iterations; ++t) {
    const double at = static_cast<double>(t) / static_cast<double>(cfg.iterations);
    const double temperature = std::max(1.0, cfg.temperature.value_at(at));
    const double noise = std::max(0.0, cfg.w_noise.value_at(at));
    const auto t0 = std::chrono::steady_clock::now();
    const double f = eng.step(temperature);
    params = eng.take();
    if (noise > 0.0) {
      add_weight_noise(params, cfg, cfg.dim, noise, noise_rng);
      eng.put(params);
    }
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const auto arrays = params.named(cfg.dim, cfg.latents);
    const bool stop = converged(f, temperature == 1.0 && noise == 0.0);
    run.record(res.trace.size(), f, secs, arrays);
    res.trace.push_back(f);
    res.seconds.push_back(secs);
    if (!std::isfinite(f)) {
      run.save("abort", arrays);
      throw Error(kNumeric, "run: non-finite free energy at iteration " + std::to_string(res.trace.size() - 1));
    }
    if (stop) break;
  }
  res.params = params.named(cfg.dim, cfg.latents);
  if (run.active()) write_manifest((fs::path(out_dir) / "manifest.json").string(), cfg, run.save("final", res.params));
  return res;
}

TrainedRun load_run(const std::string& dir) {
  const std::string mpath = (fs::path(dir) / "manifest.json").string();
  TrainedRun run;
  run.config = read_manifest(mpath);
  const std::vector<char> raw = read_file(mpath);
  const JsonValue j = JsonReader(std::string(raw.begin(), raw.end()), mpath).document();
  const JsonValue* files = j.find("parameters");
  if (!files) throw Error(kData, mpath + ": malformed manifest: missing 'parameters'");
  for (const auto& f : files->a) {
    const std::string& file = f.s;
    constexpr std::string_view pre = "final_", post = ".prsp";
    if (file.size() <= pre.size() + post.size() || file.rfind(pre, 0) != 0 ||
        file.compare(file.size() - post.size(), post.size(), post) != 0)
      throw Error(kData, dir + ": unexpected parameter file name " + file);
    run.params.push_back({file.substr(pre.size(), file.size() - pre.size() - post.size()),
                          load_array((fs::path(dir) / file).string())});
  }
  return run;
}

void infer_run(const TrainedRun& run, const double* y, uint64_t n, uint64_t d, double* map_states, double* map_mass,
               double* expected, int device) {
  RunConfig c = run.config;
  c.device = device;
  if (d != c.dim) throw Error(kData, c.model + ": data dimension mismatch");
  const Array& w = param_named(run.params, "W");
  if (w.rows != c.dim || w.cols != c.latents) throw Error(kConfig, c.model + ": dictionary shape mismatch");
  HostParams p;
  p.w = w.data;
  p.sigma2 = param_named(run.params, "sigma2").data.at(0);
  if (c.model == "dsc") {
    p.values = param_named(run.params, "values").data;
    p.probs = param_named(run.params, "probs").data;
    c.values = p.values;
  } else {
    p.pi = param_named(run.params, "pi").data.at(0);
  }
  Engine eng(c, static_cast<uint32_t>(d));
  eng.load(y, n);
  eng.put(p);
  std::vector<double> scratch(expected ? 0 : n * c.latents);
  eng.inference(map_states, map_mass, expected ? expected : scratch.data());
}

}  // namespace bscgpu
