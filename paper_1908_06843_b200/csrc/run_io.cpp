// Run I/O and the training driver around the GPU engines (see run_io.hpp).
#include "run_io.hpp"

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <memory>
#include <sstream>

#include "bsc_engine.hpp"
#include "mca_engine.hpp"
#include "rng_stream.hpp"

namespace bscgpu {

namespace fs = std::filesystem;

namespace {

constexpr char kMagic[8] = {'P', 'R', 'S', 'P', 'A', 'R', '0', '1'};  // array_io.hpp:28
constexpr const char* kLibraryVersion = "0.1.0";                     // core.hpp:29
constexpr const char* kRngAlgorithm = "mt19937_64/box-muller";       // core.hpp:131

// ---------------------------------------------------------------- SHA-256
// FIPS 180-4. The round and initial constants are derived at first use from
// their definition (fractional parts of the cube / square roots of the first
// primes) rather than tabulated.
struct ShaConsts {
  uint32_t k[64], h0[8];
  ShaConsts() {
    int primes[64], np = 0;
    for (int c = 2; np < 64; ++c) {
      bool p = true;
      for (int i = 0; i < np && primes[i] * primes[i] <= c; ++i)
        if (c % primes[i] == 0) p = false;
      if (p) primes[np++] = c;
    }
    for (int i = 0; i < 64; ++i) {
      const long double r = std::cbrt(static_cast<long double>(primes[i]));
      k[i] = static_cast<uint32_t>((r - std::floor(r)) * 4294967296.0L);
    }
    for (int i = 0; i < 8; ++i) {
      const long double r = std::sqrt(static_cast<long double>(primes[i]));
      h0[i] = static_cast<uint32_t>((r - std::floor(r)) * 4294967296.0L);
    }
  }
};

const ShaConsts& sha_consts() {
  static const ShaConsts c;
  return c;
}

class Sha256 {
 public:
  Sha256() { std::memcpy(h_, sha_consts().h0, sizeof h_); }
  void update(const uint8_t* p, size_t n) {
    total_ += n;
    while (n > 0) {
      const size_t take = std::min(n, 64 - fill_);
      std::memcpy(buf_ + fill_, p, take);
      fill_ += take;
      p += take;
      n -= take;
      if (fill_ == 64) {
        block(buf_);
        fill_ = 0;
      }
    }
  }
  std::string hex() {
    const uint64_t bits = total_ * 8;
    const uint8_t one = 0x80, zero = 0;
    update(&one, 1);
    while (fill_ != 56) update(&zero, 1);
    uint8_t len[8];
    for (int i = 0; i < 8; ++i) len[i] = static_cast<uint8_t>(bits >> (56 - 8 * i));
    update(len, 8);
    static const char* digits = "0123456789abcdef";
    std::string out;
    for (uint32_t v : h_)
      for (int s = 28; s >= 0; s -= 4) out.push_back(digits[(v >> s) & 0xf]);
    return out;
  }

 private:
  static uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }
  void block(const uint8_t* p) {
    const uint32_t* k = sha_consts().k;
    uint32_t w[64];
    for (int i = 0; i < 16; ++i)
      w[i] = (uint32_t(p[4 * i]) << 24) | (uint32_t(p[4 * i + 1]) << 16) | (uint32_t(p[4 * i + 2]) << 8) | p[4 * i + 3];
    for (int i = 16; i < 64; ++i)
      w[i] = w[i - 16] + (rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3)) + w[i - 7] +
             (rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10));
    uint32_t v[8];
    std::memcpy(v, h_, sizeof v);
    for (int i = 0; i < 64; ++i) {
      const uint32_t e = v[4], a = v[0];
      const uint32_t t1 = v[7] + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & v[5]) ^ (~e & v[6])) + k[i] + w[i];
      const uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & v[1]) ^ (a & v[2]) ^ (v[1] & v[2]));
      for (int j = 7; j > 0; --j) v[j] = v[j - 1];
      v[4] += t1;
      v[0] = t1 + t2;
    }
    for (int i = 0; i < 8; ++i) h_[i] += v[i];
  }
  uint32_t h_[8];
  uint8_t buf_[64];
  size_t fill_ = 0;
  uint64_t total_ = 0;
};

// ------------------------------------------------------------ tiny JSON
// Enough JSON to read a prsp-manifest-1 file back (objects, arrays,
// strings, numbers, booleans, null).
struct Json {
  enum Kind { kNull, kBool, kNum, kStr, kArr, kObj } kind = kNull;
  double num = 0.0;
  bool b = false;
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;
  const Json* get(const std::string& k) const {
    for (const auto& [key, v] : obj)
      if (key == k) return &v;
    return nullptr;
  }
};

class JsonParser {
 public:
  JsonParser(const std::string& s, const std::string& where) : s_(s), where_(where) {}
  Json parse() {
    Json v = value();
    ws();
    if (i_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const std::string& m) { throw Error(kData, where_ + ": malformed manifest: " + m); }
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\n' || s_[i_] == '\r' || s_[i_] == '\t')) ++i_;
  }
  Json value() {
    ws();
    if (i_ >= s_.size()) fail("unexpected end");
    const char c = s_[i_];
    Json v;
    if (c == '{') {
      v.kind = Json::kObj;
      ++i_;
      ws();
      if (i_ < s_.size() && s_[i_] == '}') {
        ++i_;
        return v;
      }
      for (;;) {
        ws();
        std::string k = string();
        ws();
        if (i_ >= s_.size() || s_[i_] != ':') fail("expected ':'");
        ++i_;
        v.obj.emplace_back(k, value());
        ws();
        if (i_ < s_.size() && s_[i_] == ',') {
          ++i_;
          continue;
        }
        if (i_ < s_.size() && s_[i_] == '}') {
          ++i_;
          return v;
        }
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.kind = Json::kArr;
      ++i_;
      ws();
      if (i_ < s_.size() && s_[i_] == ']') {
        ++i_;
        return v;
      }
      for (;;) {
        v.arr.push_back(value());
        ws();
        if (i_ < s_.size() && s_[i_] == ',') {
          ++i_;
          continue;
        }
        if (i_ < s_.size() && s_[i_] == ']') {
          ++i_;
          return v;
        }
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = Json::kStr;
      v.str = string();
      return v;
    }
    if (s_.compare(i_, 4, "null") == 0) {
      i_ += 4;
      return v;
    }
    if (s_.compare(i_, 4, "true") == 0) {
      i_ += 4;
      v.kind = Json::kBool;
      v.b = true;
      return v;
    }
    if (s_.compare(i_, 5, "false") == 0) {
      i_ += 5;
      v.kind = Json::kBool;
      return v;
    }
    v.kind = Json::kNum;
    const char* b = s_.data() + i_;
    const auto [end, ec] = std::from_chars(b, s_.data() + s_.size(), v.num);
    if (ec != std::errc()) fail("bad number");
    i_ += static_cast<size_t>(end - b);
    return v;
  }
  std::string string() {
    if (i_ >= s_.size() || s_[i_] != '"') fail("expected a string");
    ++i_;
    std::string out;
    while (i_ < s_.size() && s_[i_] != '"') {
      char c = s_[i_++];
      if (c == '\\' && i_ < s_.size()) {
        const char e = s_[i_++];
        c = e == 'n' ? '\n' : e == 't' ? '\t' : e == 'r' ? '\r' : e;
      }
      out.push_back(c);
    }
    if (i_ >= s_.size()) fail("unterminated string");
    ++i_;
    return out;
  }
  const std::string& s_;
  std::string where_;
  size_t i_ = 0;
};

std::string json_str(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o.push_back('\\');
    o.push_back(c);
  }
  return o + "\"";
}

std::string json_num(double v) {
  // JSON numbers: shortest round-trip, integral doubles keep a ".0"
  std::string s = format_double(v);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

std::string json_schedule(const Schedule& s, const std::string& ind) {
  std::string o = "[";
  for (size_t i = 0; i < s.anchors.size(); ++i) {
    o += (i ? ",\n" : "\n") + ind + "  [\n" + ind + "    " + json_num(s.anchors[i].first) + ",\n" + ind + "    " +
         json_num(s.anchors[i].second) + "\n" + ind + "  ]";
  }
  return o + "\n" + ind + "]";
}

bool uses_truncation(const std::string& m) { return m != "gmm" && m != "pmm"; }

// detail::add_column_scaled_noise (model.cpp:222-232).
void add_column_scaled_noise(std::vector<double>& w, uint32_t d, uint32_t h, double noise_std, Stream& rng) {
  std::vector<double> rms(h, 0.0);
  for (uint32_t i = 0; i < d; ++i)
    for (uint32_t j = 0; j < h; ++j) rms[j] += w[(size_t)i * h + j] * w[(size_t)i * h + j];
  for (uint32_t j = 0; j < h; ++j) rms[j] = std::sqrt(rms[j] / static_cast<double>(d));
  for (uint32_t i = 0; i < d; ++i)
    for (uint32_t j = 0; j < h; ++j) w[(size_t)i * h + j] += noise_std * rms[j] * rng.normal();
}

// data_column_means / data_mean_variance (model.cpp:187-199).
void column_stats(const double* y, uint64_t n, uint64_t d, std::vector<double>& means, double& var) {
  means.assign(d, 0.0);
  for (uint64_t i = 0; i < n; ++i)
    for (uint64_t j = 0; j < d; ++j) means[j] += y[i * d + j];
  for (auto& m : means) m /= static_cast<double>(n);
  double acc = 0.0;
  for (uint64_t i = 0; i < n; ++i)
    for (uint64_t j = 0; j < d; ++j) {
      const double c = y[i * d + j] - means[j];
      acc += c * c;
    }
  var = acc / static_cast<double>(n * d);
}

Array scalar_array(double v) { return Array{1, 1, {v}}; }

// The model's parameters on the host, in params_to_arrays order (model.cpp:77-130).
struct HostParams {
  std::vector<double> w;
  double pi = 0.0, sigma2 = 1.0;
  std::vector<double> values, probs;  // dsc
  std::vector<NamedArray> arrays(uint32_t d, uint32_t h) const {
    std::vector<NamedArray> out;
    out.push_back({"W", Array{d, h, w}});
    out.push_back({"sigma2", scalar_array(sigma2)});
    if (values.empty()) {
      out.push_back({"pi", scalar_array(pi)});
    } else {
      out.push_back({"values", Array{1, values.size(), values}});
      out.push_back({"probs", Array{1, probs.size(), probs}});
    }
    return out;
  }
};

// One engine behind the model families the GPU path implements.
class GpuModel {
 public:
  GpuModel(const RunConfig& c, uint32_t d) : cfg_(c), d_(d) {
    if (c.model != "dsc" && !c.values.empty())
      throw Error(kConfig, "model " + c.model + " does not take a value alphabet");
    const TruncationLike t = trunc(c);
    if (c.model == "bsc" || c.model == "tsc" || c.model == "dsc") {
      const int fam = c.model == "bsc" ? kBsc : c.model == "tsc" ? kTsc : kDsc;
      ld_ = std::make_unique<BscEngine>(fam, d, c.latents, t.hprime, t.gamma, 1000000,
                                        c.values.empty() ? nullptr : c.values.data(),
                                        static_cast<uint32_t>(c.values.size()), c.device);
    } else if (c.model == "mca" || c.model == "mmca") {
      mca_ = std::make_unique<McaEngine>(c.model == "mca" ? 0 : 1, c.soft_winner_rho, d, c.latents, t.hprime, t.gamma,
                                         1000000, c.device);
    } else {
      throw Error(kConfig, "gpu: model '" + c.model + "' is not on the GPU path (bsc, tsc, dsc, mca, mmca)");
    }
  }
  struct TruncationLike {
    uint32_t hprime, gamma;
  };
  static TruncationLike trunc(const RunConfig& c) {
    const uint32_t hp = c.hprime ? c.hprime : c.latents;
    return {hp, c.gamma ? c.gamma : hp};
  }
  void load(const double* y, uint64_t n) {
    if (ld_) ld_->load_data(y, n, false);
    else mca_->load_data(y, n);
  }
  void set(const HostParams& p) {
    if (ld_) ld_->set_params_ex(p.w.data(), p.pi, p.sigma2, p.probs.empty() ? nullptr : p.probs.data(),
                                static_cast<uint32_t>(p.probs.size()));
    else mca_->set_params(p.w.data(), p.pi, p.sigma2);
  }
  HostParams get() {
    HostParams p;
    p.w.resize((size_t)d_ * cfg_.latents);
    if (ld_) {
      if (cfg_.model == "dsc") {
        p.values = ld_->alphabet();
        p.probs.resize(p.values.size());
      }
      ld_->get_params_ex(p.w.data(), &p.pi, &p.sigma2, p.probs.empty() ? nullptr : p.probs.data());
    } else {
      mca_->get_params(p.w.data(), &p.pi, &p.sigma2);
    }
    return p;
  }
  double step(double temperature) { return ld_ ? ld_->step(temperature) : mca_->step(temperature); }
  // standard_init (linear_discrete.cpp:129-148, max_causes.cpp:121-130) with
  // detail::init_weights (model.cpp:201-220).
  HostParams standard_init(const double* y, uint64_t n, Stream& rng) const {
    if (n < 2) throw Error(kData, "standard_init requires at least two data points");
    std::vector<double> means;
    double var = 0.0;
    column_stats(y, n, d_, means, var);
    const uint32_t h = cfg_.latents;
    const double sd = var > 0.0 ? std::sqrt(var / h) : 0.0;
    const bool take_abs = cfg_.model == "mca";
    HostParams p;
    p.w.resize((size_t)d_ * h);
    for (uint32_t i = 0; i < d_; ++i)
      for (uint32_t j = 0; j < h; ++j) {
        double v = means[i] + sd * rng.normal();
        if (take_abs) v = std::max(std::abs(v), 1e-8);
        p.w[(size_t)i * h + j] = v;
      }
    p.sigma2 = std::max(var, 1e-12);
    const double hh = static_cast<double>(h);
    const double hp = static_cast<double>(std::min(trunc(cfg_).hprime, h));
    if (cfg_.model == "dsc") {
      p.values = ld_->alphabet();
      const double k = static_cast<double>(p.values.size());
      const double nonzero = hp / (2.0 * hh * k);
      p.probs.assign(p.values.size(), nonzero);
      for (size_t i = 0; i < p.values.size(); ++i)
        if (p.values[i] == 0.0) p.probs[i] = 1.0 - hp / (2.0 * hh) * (1.0 - 1.0 / k);
    } else {
      p.pi = hp / (2.0 * hh);
    }
    return p;
  }
  // perturb_weights (linear_discrete.cpp:510-514, max_causes.cpp:476-484)
  void perturb(HostParams& p, double noise_std, Stream& rng) const {
    add_column_scaled_noise(p.w, d_, cfg_.latents, noise_std, rng);
    if (cfg_.model == "mca")
      for (double& v : p.w) v = std::max(v, 1e-8);
  }
  void inference(double* ms, double* mm, double* ex) {
    if (ld_) ld_->inference(ms, mm, ex);
    else mca_->inference(ms, mm, ex);
  }

 private:
  RunConfig cfg_;
  uint32_t d_;
  std::unique_ptr<BscEngine> ld_;
  std::unique_ptr<McaEngine> mca_;
};

size_t float_count(const std::vector<NamedArray>& a) {
  size_t n = 0;
  for (const auto& x : a) n += x.a.data.size();
  return n;
}

std::vector<std::string> write_params(const std::string& dir, const std::string& prefix,
                                      const std::vector<NamedArray>& arrays) {
  std::vector<std::string> files;
  for (const auto& [name, a] : arrays) {
    const std::string file = prefix + "_" + name + ".prsp";
    save_array((fs::path(dir) / file).string(), a.data.data(), a.rows, a.cols);
    files.push_back(file);
  }
  return files;
}

}  // namespace

// ------------------------------------------------------------- arrays
void save_array(const std::string& path, const double* data, uint64_t rows, uint64_t cols) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw Error(kData, "cannot write file: " + path);
  out.write(kMagic, 8);
  out.write(reinterpret_cast<const char*>(&rows), 8);  // little-endian hosts (x86-64 / aarch64)
  out.write(reinterpret_cast<const char*>(&cols), 8);
  out.write(reinterpret_cast<const char*>(data), static_cast<std::streamsize>(rows * cols * sizeof(double)));
  if (!out) throw Error(kData, "write failed: " + path);
}

Array load_array(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Error(kData, "cannot open file: " + path);
  char magic[8];
  in.read(magic, 8);
  if (in.gcount() != 8 || std::memcmp(magic, kMagic, 8) != 0) throw Error(kData, path + ": not a PRSPAR01 file");
  Array a;
  in.read(reinterpret_cast<char*>(&a.rows), 8);
  in.read(reinterpret_cast<char*>(&a.cols), 8);
  if (!in) throw Error(kData, path + ": truncated header");
  if (a.rows != 0 && a.cols > (1ull << 48) / a.rows) throw Error(kData, path + ": implausible array shape");
  a.data.resize(a.rows * a.cols);
  in.read(reinterpret_cast<char*>(a.data.data()), static_cast<std::streamsize>(a.data.size() * sizeof(double)));
  if (static_cast<size_t>(in.gcount()) != a.data.size() * sizeof(double))
    throw Error(kData, path + ": payload shorter than header promises");
  return a;
}

Array load_csv(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw Error(kData, "cannot open file: " + path);
  Array a;
  std::string line;
  size_t line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    size_t row_cols = 0;
    const char* p = line.data();
    const char* end = p + line.size();
    for (;;) {
      while (p < end && *p == ' ') ++p;
      double v = 0.0;
      const auto [next, ec] = std::from_chars(p, end, v);
      if (ec != std::errc()) throw Error(kData, path + ": line " + std::to_string(line_no) + ": malformed number");
      a.data.push_back(v);
      ++row_cols;
      p = next;
      while (p < end && *p == ' ') ++p;
      if (p == end) break;
      if (*p != ',') throw Error(kData, path + ": line " + std::to_string(line_no) + ": expected ','");
      ++p;
    }
    if (a.cols == 0) {
      a.cols = row_cols;
    } else if (row_cols != a.cols) {
      throw Error(kData, path + ": line " + std::to_string(line_no) + ": expected " + std::to_string(a.cols) +
                             " columns, found " + std::to_string(row_cols));
    }
    ++a.rows;
  }
  if (a.rows == 0) throw Error(kData, path + ": empty dataset");
  return a;
}

Array load_dataset(const std::string& path) {
  std::ifstream probe(path, std::ios::binary);
  if (!probe) throw Error(kData, "cannot open file: " + path);
  char head[8] = {};
  probe.read(head, 8);
  const size_t got = static_cast<size_t>(probe.gcount());
  probe.close();
  if (got == 8 && std::memcmp(head, kMagic, 8) == 0) return load_array(path);
  if (got >= 4 && std::memcmp(head, kMagic, 4) == 0) throw Error(kData, path + ": not a PRSPAR01 file");
  return load_csv(path);
}

std::string format_double(double v) {
  char buf[32];
  const auto [end, ec] = std::to_chars(buf, buf + sizeof(buf), v);
  if (ec != std::errc()) throw Error(kInternal, "format_double failed");
  return std::string(buf, end);
}

std::string sha256_hex(const void* data, size_t n) {
  Sha256 s;
  s.update(static_cast<const uint8_t*>(data), n);
  return s.hex();
}

std::string sha256_hex_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Error(kData, "cannot open file: " + path);
  Sha256 s;
  std::vector<char> buf(1 << 20);
  while (in) {
    in.read(buf.data(), static_cast<std::streamsize>(buf.size()));
    s.update(reinterpret_cast<const uint8_t*>(buf.data()), static_cast<size_t>(in.gcount()));
  }
  return s.hex();
}

// ------------------------------------------------------------ schedules
void Schedule::validate() const {
  if (anchors.empty()) throw Error(kConfig, "schedule: at least one anchor required");
  for (size_t i = 0; i < anchors.size(); ++i) {
    if (!std::isfinite(anchors[i].first) || !std::isfinite(anchors[i].second))
      throw Error(kConfig, "schedule: anchors must be finite");
    if (anchors[i].first < 0.0 || anchors[i].first > 1.0)
      throw Error(kConfig, "schedule: anchor positions must lie in [0,1]");
    if (i > 0 && anchors[i].first <= anchors[i - 1].first)
      throw Error(kConfig, "schedule: anchor positions must be strictly increasing");
  }
}

double Schedule::value_at(double position) const {
  if (position <= anchors.front().first) return anchors.front().second;
  if (position >= anchors.back().first) return anchors.back().second;
  for (size_t i = 1; i < anchors.size(); ++i)
    if (position <= anchors[i].first) {
      const auto [p0, v0] = anchors[i - 1];
      const auto [p1, v1] = anchors[i];
      const double t = (position - p0) / (p1 - p0);
      return v0 + t * (v1 - v0);
    }
  return anchors.back().second;
}

// ------------------------------------------------------------- manifest
void write_manifest(const std::string& path, const RunConfig& c, const std::vector<std::string>& files) {
  std::ostringstream o;
  o << "{\n";
  o << "  \"format\": \"prsp-manifest-1\",\n";
  o << "  \"library\": " << json_str(kLibraryVersion) << ",\n";
  o << "  \"rng\": " << json_str(kRngAlgorithm) << ",\n";
  o << "  \"model\": " << json_str(c.model) << ",\n";
  o << "  \"dim\": " << c.dim << ",\n";
  o << "  \"latents\": " << c.latents << ",\n";
  if (uses_truncation(c.model)) {
    o << "  \"hprime\": " << c.hprime << ",\n";
    o << "  \"gamma\": " << c.gamma << ",\n";
  }
  if (c.model == "dsc") {
    o << "  \"values\": [";
    for (size_t i = 0; i < c.values.size(); ++i) o << (i ? ",\n    " : "\n    ") << json_num(c.values[i]);
    o << "\n  ],\n";
  }
  o << "  \"iterations\": " << c.iterations << ",\n";
  o << "  \"seed\": " << c.seed << ",\n";
  o << "  \"workers\": " << c.workers << ",\n";
  o << "  \"shards\": " << c.shards << ",\n";
  o << "  \"tolerance\": " << (c.tolerance ? json_num(*c.tolerance) : std::string("null")) << ",\n";
  o << "  \"temperature\": " << json_schedule(c.temperature, "  ") << ",\n";
  o << "  \"w_noise\": " << json_schedule(c.w_noise, "  ") << ",\n";
  o << "  \"data\": {\n    \"file\": " << json_str(c.data_file) << ",\n    \"sha256\": " << json_str(c.data_sha256)
    << ",\n    \"rows\": " << c.data_rows << ",\n    \"cols\": " << c.data_cols << "\n  },\n";
  o << "  \"parameters\": [";
  for (size_t i = 0; i < files.size(); ++i) o << (i ? ",\n    " : "\n    ") << json_str(files[i]);
  o << (files.empty() ? "]\n" : "\n  ]\n");
  o << "}\n";
  std::ofstream out(path, std::ios::trunc);
  if (!out) throw Error(kData, "cannot write file: " + path);
  out << o.str();
  if (!out) throw Error(kData, "write failed: " + path);
}

RunConfig read_manifest(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw Error(kData, "cannot open manifest: " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  const std::string text = ss.str();
  const Json j = JsonParser(text, path).parse();
  auto need = [&](const Json& o, const char* k) -> const Json& {
    const Json* v = o.get(k);
    if (!v) throw Error(kData, path + ": malformed manifest: missing '" + k + "'");
    return *v;
  };
  const Json* fmt = j.get("format");
  if (!fmt || fmt->kind != Json::kStr || fmt->str != "prsp-manifest-1")
    throw Error(kData, path + ": unknown manifest format");
  RunConfig c;
  c.model = need(j, "model").str;
  c.dim = static_cast<uint32_t>(need(j, "dim").num);
  c.latents = static_cast<uint32_t>(need(j, "latents").num);
  c.hprime = j.get("hprime") ? static_cast<uint32_t>(j.get("hprime")->num) : c.latents;
  c.gamma = j.get("gamma") ? static_cast<uint32_t>(j.get("gamma")->num) : c.hprime;
  if (const Json* v = j.get("values"))
    for (const auto& x : v->arr) c.values.push_back(x.num);
  c.iterations = static_cast<uint64_t>(need(j, "iterations").num);
  c.seed = static_cast<uint64_t>(need(j, "seed").num);
  c.workers = static_cast<uint32_t>(need(j, "workers").num);
  c.shards = static_cast<uint32_t>(need(j, "shards").num);
  if (need(j, "tolerance").kind != Json::kNull) c.tolerance = need(j, "tolerance").num;
  auto sched = [&](const Json& a) {
    Schedule s;
    for (const auto& p : a.arr) s.anchors.emplace_back(p.arr.at(0).num, p.arr.at(1).num);
    return s;
  };
  c.temperature = sched(need(j, "temperature"));
  c.w_noise = sched(need(j, "w_noise"));
  const Json& d = need(j, "data");
  c.data_file = need(d, "file").str;
  c.data_sha256 = need(d, "sha256").str;
  c.data_rows = static_cast<uint64_t>(need(d, "rows").num);
  c.data_cols = static_cast<uint64_t>(need(d, "cols").num);
  return c;
}

// ------------------------------------------------------------- training
// train_run (run_io.cpp:196-230) + run (em.cpp:27-77) + DirectoryLogger
// (run_io.cpp:131-161): init from RngStream::derived(seed, "init"), the
// annealing schedules, weight noise from RngStream::derived(seed, "nois"),
// one GPU step per iteration, trace / checkpoints / final arrays / manifest.
TrainResult train_run(RunConfig& cfg, const double* y, uint64_t n, uint64_t d, const std::string& data_file,
                      const std::string& out_dir) {
  if (n == 0) throw Error(kData, "run: empty dataset");
  if (cfg.iterations == 0) throw Error(kConfig, "annealing: max_iterations must be >= 1");
  cfg.temperature.validate();
  cfg.w_noise.validate();
  if (cfg.tolerance && !(*cfg.tolerance >= 0.0)) throw Error(kConfig, "run: convergence tolerance must be >= 0");
  if (cfg.shards == 0 || cfg.workers == 0) throw Error(kConfig, "shard plan: shards and workers must be >= 1");
  cfg.dim = static_cast<uint32_t>(d);
  const auto t = GpuModel::trunc(cfg);
  cfg.hprime = t.hprime;
  cfg.gamma = t.gamma;
  cfg.data_rows = n;
  cfg.data_cols = d;
  if (!data_file.empty()) {
    cfg.data_file = data_file;
    cfg.data_sha256 = sha256_hex_file(data_file);
  } else {
    cfg.data_file = "(memory)";
    cfg.data_sha256 = sha256_hex(y, n * d * sizeof(double));
  }
  GpuModel model(cfg, static_cast<uint32_t>(d));
  Stream init_rng = Stream::derived(cfg.seed, 0x696e6974ULL);
  HostParams params = model.standard_init(y, n, init_rng);
  if (cfg.model == "dsc") cfg.values = params.values;  // the sorted alphabet, as the model holds it
  model.load(y, n);
  model.set(params);

  std::ofstream trace;
  if (!out_dir.empty()) {
    fs::create_directories(out_dir);
    trace.open(fs::path(out_dir) / "free_energy.csv", std::ios::trunc);
    if (!trace) throw Error(kData, "cannot write trace in " + out_dir);
    trace << "iteration,free_energy,seconds\n";
    trace.flush();
  }
  Stream noise_rng = Stream::derived(cfg.seed, 0x6e6f6973ULL);
  TrainResult res;
  double prev_f = std::nan("");
  for (uint64_t it = 1; it <= cfg.iterations; ++it) {
    const double pos = static_cast<double>(it) / static_cast<double>(cfg.iterations);
    const double temp = std::max(1.0, cfg.temperature.value_at(pos));  // annealing.cpp:59-63
    const double noise = std::max(0.0, cfg.w_noise.value_at(pos));
    const auto t0 = std::chrono::steady_clock::now();
    const double f = model.step(temp);
    params = model.get();
    if (noise > 0.0) {
      model.perturb(params, noise, noise_rng);
      model.set(params);
    }
    const double seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const size_t iteration = res.trace.size();
    res.trace.push_back(f);
    res.seconds.push_back(seconds);
    const auto arrays = params.arrays(cfg.dim, cfg.latents);
    if (!out_dir.empty()) {
      trace << iteration << ',' << format_double(f) << ',' << format_double(seconds) << '\n';
      trace.flush();
      const size_t cadence = float_count(arrays) < 1000000 ? 1 : 10;
      if (iteration % cadence == 0) write_params(out_dir, "checkpoint", arrays);
    }
    if (!std::isfinite(f)) {
      if (!out_dir.empty()) write_params(out_dir, "abort", arrays);
      throw Error(kNumeric, "run: non-finite free energy at iteration " + std::to_string(iteration));
    }
    const bool inert = temp == 1.0 && noise == 0.0;
    if (cfg.tolerance && inert && !std::isnan(prev_f) &&
        std::abs(f - prev_f) <= *cfg.tolerance * (1.0 + std::abs(f)))
      break;
    prev_f = f;
  }
  res.params = params.arrays(cfg.dim, cfg.latents);
  if (!out_dir.empty()) {
    const auto files = write_params(out_dir, "final", res.params);
    write_manifest((fs::path(out_dir) / "manifest.json").string(), cfg, files);
  }
  return res;
}

TrainedRun load_run(const std::string& dir) {
  const std::string mpath = (fs::path(dir) / "manifest.json").string();
  std::ifstream in(mpath);
  if (!in) throw Error(kData, "cannot open manifest: " + mpath);
  std::stringstream ss;
  ss << in.rdbuf();
  const std::string text = ss.str();
  const Json j = JsonParser(text, mpath).parse();
  TrainedRun run;
  run.config = read_manifest(mpath);
  const Json* files = j.get("parameters");
  if (!files) throw Error(kData, mpath + ": malformed manifest: missing 'parameters'");
  for (const auto& f : files->arr) {
    const std::string& file = f.str;
    const std::string prefix = "final_", suffix = ".prsp";
    if (file.size() <= prefix.size() + suffix.size() || file.compare(0, prefix.size(), prefix) != 0)
      throw Error(kData, dir + ": unexpected parameter file name " + file);
    run.params.push_back({file.substr(prefix.size(), file.size() - prefix.size() - suffix.size()),
                          load_array((fs::path(dir) / file).string())});
  }
  return run;
}

void infer_run(const TrainedRun& run, const double* y, uint64_t n, uint64_t d, double* map_states, double* map_mass,
               double* expected, int device) {
  RunConfig c = run.config;
  c.device = device;
  if (d != c.dim) throw Error(kData, c.model + ": data dimension mismatch");
  auto arr = [&](const char* name) -> const Array& {
    for (const auto& p : run.params)
      if (p.name == name) return p.a;
    throw Error(kData, std::string("run: missing parameter array ") + name);
  };
  HostParams p;
  p.w = arr("W").data;
  if (arr("W").rows != c.dim || arr("W").cols != c.latents) throw Error(kConfig, c.model + ": dictionary shape mismatch");
  p.sigma2 = arr("sigma2").data.at(0);
  if (c.model == "dsc") {
    p.values = arr("values").data;
    p.probs = arr("probs").data;
    c.values = p.values;
  } else {
    p.pi = arr("pi").data.at(0);
  }
  GpuModel model(c, static_cast<uint32_t>(d));
  model.load(y, n);
  model.set(p);
  std::vector<double> ex(expected ? 0 : n * c.latents);
  model.inference(map_states, map_mass, expected ? expected : ex.data());
}

}  // namespace bscgpu
