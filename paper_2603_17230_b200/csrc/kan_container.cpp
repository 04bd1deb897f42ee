// kan_container.cpp -- the reference's .kant model container, host side.
//
// Replaces save_container / load_container (proj/include/kantize/io.hpp:99-350):
//   "KANT" magic, u32 LE version (1), u32 LE metadata length, UTF-8 JSON
//   metadata, payload (f32 LE coefficient matrices and u8 table blobs in
//   declared order), u32 LE CRC-32 of the payload (io.hpp:31-45).
// The metadata is written byte-for-byte as the reference's nlohmann
// ordered_json::dump() does (insertion-ordered keys, compact separators,
// shortest round-trip doubles with nlohmann's fixed/exponent layout), so a
// container saved here is identical to the reference's for the same model
// (the frozen 275-byte layout of test_io.cpp:145-165 included).
//
// Errors keep the reference's classes and messages: io_error -> KAN_ERR_IO,
// format_error -> KAN_ERR_FORMAT (bad magic, unsupported version named in the
// message, truncation before checksum), checksum_error -> KAN_ERR_CHECKSUM.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <memory>
#include <string>
#include <vector>

#include "../../include/kan_b200.h"
#include "kan_json.hpp"

struct kan_container {
  std::string err;
  std::string descriptor;  // the model in the reference's descriptor schema
  std::vector<std::vector<double>> coeffs;  // per KAN layer, [n_in*(G+P), n_out]
  std::vector<uint8_t> lut;
  int lut_degree = 0, lut_k = 0, lut_h = 0;
  struct Table {
    std::vector<uint8_t> values;
    int n_in = 0, n_out = 0, bits_a = 0, h = 0;
    double qd[2] = {0, 0};
    int64_t qi[4] = {0, 0, 0, 0};
  };
  std::vector<Table> tables;
};

namespace kan {
namespace {

struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ChecksumError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Unsupported : std::runtime_error {
  using std::runtime_error::runtime_error;
};

uint32_t crc32(const uint8_t* data, size_t len) {  // io.hpp:31-45 (reflected 0xEDB88320)
  static uint32_t table[256];
  static bool init = false;
  if (!init) {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int b = 0; b < 8; ++b) c = (c >> 1) ^ ((c & 1) ? 0xEDB88320u : 0u);
      table[i] = c;
    }
    init = true;
  }
  uint32_t c = ~0u;
  for (size_t i = 0; i < len; ++i) c = table[(c ^ data[i]) & 0xFF] ^ (c >> 8);
  return ~c;
}

void put_u32(std::vector<uint8_t>& out, uint32_t v) {
  for (int b = 0; b < 4; ++b) out.push_back(static_cast<uint8_t>((v >> (8 * b)) & 0xFF));
}
uint32_t get_u32(const uint8_t* p) {
  return static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8) | (static_cast<uint32_t>(p[2]) << 16) |
         (static_cast<uint32_t>(p[3]) << 24);
}

// nlohmann::json's double layout: shortest round-trip digits d1..dk with
// decimal exponent, then fixed notation for -4 < n <= 15 (n = k + exponent,
// ".0" appended to integers) and d.ddde+XX otherwise (exponent >= 2 digits).
std::string json_double(double v) {
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  std::string sign = v < 0 ? "-" : "";
  const double a = std::fabs(v);
  char buf[64];
  int prec = 1;
  for (; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof(buf), "%.*e", prec - 1, a);
    if (std::strtod(buf, nullptr) == a) break;
  }
  // buf = d.ddddde[+-]XX
  std::string s(buf);
  const size_t epos = s.find('e');
  const int e10 = std::atoi(s.c_str() + epos + 1);
  std::string digits;
  for (size_t i = 0; i < epos; ++i)
    if (s[i] != '.') digits.push_back(s[i]);
  while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
  const int k = static_cast<int>(digits.size());
  const int n = e10 + 1;  // decimal point position after n digits
  std::string out;
  if (k <= n && n <= 15) {
    out = digits + std::string(static_cast<size_t>(n - k), '0') + ".0";
  } else if (0 < n && n <= 15) {
    out = digits.substr(0, static_cast<size_t>(n)) + "." + digits.substr(static_cast<size_t>(n));
  } else if (-4 < n && n <= 0) {
    out = "0." + std::string(static_cast<size_t>(-n), '0') + digits;
  } else {
    out = digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    const int e = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof(eb), "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
    out += eb;
  }
  return sign + out;
}

std::string json_str(const std::string& s) { return "\"" + s + "\""; }  // plain ASCII keys / names

struct Grid4 {
  int G = 0, P = 0;
  double lo = -1.0, hi = 1.0;
};

std::string grid_json(const Grid4& g) {
  return "{\"intervals\":" + std::to_string(g.G) + ",\"degree\":" + std::to_string(g.P) + ",\"lo\":" +
         json_double(g.lo) + ",\"hi\":" + json_double(g.hi) + "}";
}

std::string quant_json(double scale, int64_t zp, int bits) {
  return "{\"scale\":" + json_double(scale) + ",\"zero_point\":" + std::to_string(zp) + ",\"bits\":" +
         std::to_string(bits) + "}";
}

std::vector<uint8_t> read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("load_container: cannot open " + path);
  return std::vector<uint8_t>((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}

// load_container (io.hpp:217-350) into the host-side container
void load(kan_container* c, const std::string& path) {
  const std::vector<uint8_t> file = read_file(path);
  if (file.size() < 12 || std::memcmp(file.data(), "KANT", 4) != 0)
    throw FormatError("load_container: bad magic bytes");
  const uint32_t version = get_u32(file.data() + 4);
  if (version != 1) throw FormatError("load_container: unsupported version " + std::to_string(version));
  const uint32_t meta_len = get_u32(file.data() + 8);
  if (file.size() < 12ull + meta_len + 4) throw FormatError("load_container: truncated file");
  Json meta;
  try {
    meta = Json::parse(std::string(file.begin() + 12, file.begin() + 12 + meta_len));
  } catch (const FormatError& e) {
    throw FormatError(std::string("load_container: bad metadata: ") + e.what());
  }
  const uint8_t* payload = file.data() + 12 + meta_len;
  const size_t payload_len = file.size() - 12 - meta_len - 4;

  struct Ref {
    std::string name, dtype;
    size_t offset = 0, bytes = 0;
    const Json* j = nullptr;
  };
  std::vector<Ref> tensors;
  size_t declared = 0;
  for (const auto& t : meta.at("tensors").arr) {
    Ref r;
    r.name = t.at("name").string();
    r.dtype = t.at("dtype").string();
    r.offset = static_cast<size_t>(t.at("offset").number());
    r.bytes = static_cast<size_t>(t.at("bytes").number());
    r.j = &t;
    declared = std::max(declared, r.offset + r.bytes);
    tensors.push_back(r);
  }
  // length first (truncation is a format problem), checksum second
  if (payload_len < declared)
    throw FormatError("load_container: truncated file (payload has " + std::to_string(payload_len) + " of " +
                      std::to_string(declared) + " bytes)");
  if (crc32(payload, payload_len) != get_u32(payload + payload_len))
    throw ChecksumError("load_container: payload checksum mismatch");
  auto find = [&](const std::string& name) -> const Ref* {
    for (const auto& r : tensors)
      if (r.name == name) return &r;
    return nullptr;
  };

  // descriptor: one grid per model (Model::grid, layers.hpp:225-231)
  bool have_grid = false;
  Grid4 grid;
  std::string layers_json;
  int idx = 0;
  for (const auto& jl : meta.at("layers").arr) {
    const std::string type = jl.at("type").string();
    std::string lj;
    if (type == "kan_linear" || type == "kan_conv") {
      const Json& jg = jl.at("grid");
      Grid4 g{jg.at("intervals").integer(), jg.at("degree").integer(), jg.at("lo").number(), jg.at("hi").number()};
      if (!have_grid) {
        grid = g;
        have_grid = true;
      } else if (g.G != grid.G || g.P != grid.P || g.lo != grid.lo || g.hi != grid.hi) {
        throw Unsupported("load_container: layers with different grids (the engine runs one grid per model)");
      }
      int64_t rows, cols;
      if (type == "kan_linear") {
        const int n_in = jl.at("n_in").integer(), n_out = jl.at("n_out").integer();
        lj = "{\"type\":\"linear\",\"n_in\":" + std::to_string(n_in) + ",\"n_out\":" + std::to_string(n_out) + "}";
        rows = static_cast<int64_t>(n_in) * (g.G + g.P);
        cols = n_out;
      } else {
        const int ci = jl.at("c_in").integer(), co = jl.at("c_out").integer(), k = jl.at("kernel").integer();
        const int st = jl.at("stride").integer(), pd = jl.at("padding").integer();
        lj = "{\"type\":\"conv\",\"c_in\":" + std::to_string(ci) + ",\"c_out\":" + std::to_string(co) +
             ",\"kernel\":" + std::to_string(k) + ",\"stride\":" + std::to_string(st) + ",\"padding\":" +
             std::to_string(pd) + "}";
        rows = static_cast<int64_t>(ci) * k * k * (g.G + g.P);
        cols = co;
      }
      const std::string name = "layer" + std::to_string(idx) + ".coeffs";
      const Ref* r = find(name);
      if (!r) throw FormatError("load_container: missing tensor '" + name + "'");
      if (r->bytes != static_cast<size_t>(rows * cols) * 4)
        throw FormatError("load_container: tensor '" + name + "' has unexpected size");
      std::vector<double> w(static_cast<size_t>(rows * cols));
      for (size_t i = 0; i < w.size(); ++i) {
        const uint32_t u = get_u32(payload + r->offset + i * 4);
        float f;
        std::memcpy(&f, &u, 4);
        w[i] = static_cast<double>(f);
      }
      c->coeffs.push_back(std::move(w));
    } else if (type == "maxpool") {
      lj = "{\"type\":\"maxpool\",\"window\":" + std::to_string(jl.value_int("window", 2)) + "}";
    } else if (type == "flatten") {
      lj = "{\"type\":\"flatten\"}";
    } else {
      throw FormatError("load_container: unknown layer type '" + type + "'");
    }
    layers_json += (layers_json.empty() ? "" : ",") + lj;
    ++idx;
  }
  if (!have_grid) throw FormatError("Model::grid: model has no KAN layers");
  std::string input;
  for (const auto& d : meta.at("input_shape").arr) input += (input.empty() ? "" : ",") + std::to_string(d.integer());
  c->descriptor = "{\"name\":\"kant\",\"grid\":{\"intervals\":" + std::to_string(grid.G) + ",\"degree\":" +
                  std::to_string(grid.P) + "},\"domain\":[" + json_double(grid.lo) + "," + json_double(grid.hi) +
                  "],\"input\":[" + input + "],\"layers\":[" + layers_json + "]}";

  for (const auto& r : tensors) {
    if (r.dtype != "u8") continue;
    const Json& t = *r.j;
    const Json& attrs = t.at("attrs");
    const std::string kind = attrs.at("kind").string();
    std::vector<uint8_t> data(payload + r.offset, payload + r.offset + r.bytes);
    if (kind == "bspline_lut") {
      c->lut = std::move(data);
      c->lut_degree = attrs.at("degree").integer();
      c->lut_k = attrs.at("bits_per_interval").integer();
      c->lut_h = attrs.at("value_bits").integer();
    } else if (kind == "spline_tables") {
      kan_container::Table tb;
      tb.n_in = attrs.at("n_in").integer();
      tb.n_out = attrs.at("n_out").integer();
      tb.bits_a = attrs.at("bits_a").integer();
      tb.h = attrs.at("value_bits").integer();
      const Json& iq = attrs.at("in_quant");
      const Json& oq = t.at("quant");
      tb.qd[0] = iq.at("scale").number();
      tb.qd[1] = oq.at("scale").number();
      tb.qi[0] = static_cast<int64_t>(iq.at("zero_point").number());
      const int ib = iq.at("bits").integer(), ob = oq.at("bits").integer();
      tb.qi[1] = ib >= 1 && ib <= 8 ? (int64_t{1} << ib) - 1 : 0;  // quant_from_json, io.hpp:86-94
      tb.qi[2] = static_cast<int64_t>(oq.at("zero_point").number());
      tb.qi[3] = ob >= 1 && ob <= 8 ? (int64_t{1} << ob) - 1 : 0;
      tb.values = std::move(data);
      c->tables.push_back(std::move(tb));
    }
  }
}

// save_container (io.hpp:108-211) from a descriptor + coefficients (+ tables)
void save(const std::string& path, const std::string& descriptor, const double* const* coeffs, const uint8_t* lut,
          int64_t lut_n, int lut_k, int lut_h, const uint8_t* const* st_values, int st_bits_a, int st_h,
          const double* st_qd, const int64_t* st_qi) {
  const Json j = Json::parse(descriptor);
  Grid4 g;
  g.G = j.at("grid").at("intervals").integer();
  g.P = j.at("grid").at("degree").integer();
  if (j.has("domain")) {
    g.lo = j.at("domain").at(0).number();
    g.hi = j.at("domain").at(1).number();
  }
  const int nb = g.G + g.P;
  std::vector<uint8_t> payload;
  std::string tensors, layers;
  std::vector<std::pair<int64_t, int64_t>> kan_shapes;  // (n_in, n_out) per KAN layer
  auto add_sep = [](std::string& s) {
    if (!s.empty()) s += ",";
  };
  int idx = 0, kan = 0;
  for (const auto& jl : j.at("layers").arr) {
    for (const char* ext : {"id", "input_from", "residual"})
      if (jl.has(ext)) throw Unsupported("save_container: descriptor extension '" + std::string(ext) + "' has no container form");
    const std::string type = jl.at("type").string();
    std::string lj;
    if (type == "linear" || type == "conv") {
      int64_t rows, cols, n_in;
      if (type == "linear") {
        n_in = jl.at("n_in").integer();
        cols = jl.at("n_out").integer();
        lj = "{\"type\":\"kan_linear\",\"n_in\":" + std::to_string(n_in) + ",\"n_out\":" + std::to_string(cols) +
             ",\"grid\":" + grid_json(g) + "}";
      } else {
        const int ci = jl.at("c_in").integer(), k = jl.at("kernel").integer();
        cols = jl.at("c_out").integer();
        n_in = static_cast<int64_t>(ci) * k * k;
        lj = "{\"type\":\"kan_conv\",\"c_in\":" + std::to_string(ci) + ",\"c_out\":" + std::to_string(cols) +
             ",\"kernel\":" + std::to_string(k) + ",\"stride\":" + std::to_string(jl.value_int("stride", 1)) +
             ",\"padding\":" + std::to_string(jl.value_int("padding", 0)) + ",\"grid\":" + grid_json(g) + "}";
      }
      rows = n_in * nb;
      kan_shapes.emplace_back(n_in, cols);
      add_sep(tensors);
      tensors += "{\"name\":\"layer" + std::to_string(idx) + ".coeffs\",\"dtype\":\"f32\",\"shape\":[" +
                 std::to_string(rows) + "," + std::to_string(cols) + "],\"offset\":" + std::to_string(payload.size()) +
                 ",\"bytes\":" + std::to_string(rows * cols * 4) + "}";
      const double* w = coeffs[kan];
      for (int64_t i = 0; i < rows * cols; ++i) {
        const float f = static_cast<float>(w[i]);
        uint32_t u;
        std::memcpy(&u, &f, 4);
        put_u32(payload, u);
      }
      ++kan;
    } else if (type == "maxpool") {
      lj = "{\"type\":\"maxpool\",\"window\":" + std::to_string(jl.value_int("window", 2)) + "}";
    } else if (type == "flatten") {
      lj = "{\"type\":\"flatten\"}";
    } else {
      throw Unsupported("save_container: layer type '" + type + "' has no container form");
    }
    add_sep(layers);
    layers += lj;
    ++idx;
  }
  auto add_u8 = [&](const std::string& name, const uint8_t* data, int64_t n, const std::string& quant,
                    const std::string& attrs) {
    add_sep(tensors);
    tensors += "{\"name\":\"" + name + "\",\"dtype\":\"u8\",\"shape\":[" + std::to_string(n) + "],\"offset\":" +
               std::to_string(payload.size()) + ",\"bytes\":" + std::to_string(n) + ",\"quant\":" + quant +
               ",\"attrs\":" + attrs + "}";
    payload.insert(payload.end(), data, data + n);
  };
  if (lut) {  // BsplineLut::value_qp = compute_quant_params(0, 1, h) (lut.hpp:112)
    const double s = 1.0 / static_cast<double>((int64_t{1} << lut_h) - 1);
    add_u8("bspline_lut.entries", lut, lut_n, quant_json(s, 0, lut_h),
           "{\"kind\":\"bspline_lut\",\"degree\":" + std::to_string(g.P) + ",\"bits_per_interval\":" +
               std::to_string(lut_k) + ",\"value_bits\":" + std::to_string(lut_h) + "}");
  }
  if (st_values) {
    for (int t = 0; t < kan; ++t) {
      const int64_t n = (kan_shapes[static_cast<size_t>(t)].first * kan_shapes[static_cast<size_t>(t)].second)
                        << st_bits_a;
      add_u8("spline_tables." + std::to_string(t), st_values[t], n,
             quant_json(st_qd[2 * t + 1], st_qi[4 * t + 2], st_h),
             "{\"kind\":\"spline_tables\",\"layer\":" + std::to_string(t) + ",\"n_in\":" +
                 std::to_string(kan_shapes[static_cast<size_t>(t)].first) + ",\"n_out\":" +
                 std::to_string(kan_shapes[static_cast<size_t>(t)].second) + ",\"bits_a\":" +
                 std::to_string(st_bits_a) + ",\"value_bits\":" + std::to_string(st_h) + ",\"in_quant\":" +
                 quant_json(st_qd[2 * t], st_qi[4 * t], st_bits_a) + "}");
    }
  }
  std::string input;
  for (const auto& d : j.at("input").arr) input += (input.empty() ? "" : ",") + std::to_string(d.integer());
  const std::string meta =
      "{\"input_shape\":[" + input + "],\"layers\":[" + layers + "],\"tensors\":[" + tensors + "]}";
  std::vector<uint8_t> file = {'K', 'A', 'N', 'T'};
  put_u32(file, 1);
  put_u32(file, static_cast<uint32_t>(meta.size()));
  file.insert(file.end(), meta.begin(), meta.end());
  file.insert(file.end(), payload.begin(), payload.end());
  put_u32(file, crc32(payload.data(), payload.size()));
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw IoError("save_container: cannot open " + path + " for writing");
  out.write(reinterpret_cast<const char*>(file.data()), static_cast<std::streamsize>(file.size()));
  if (!out) throw IoError("save_container: write failed for " + path);
}

template <class F>
kan_status run(std::string* err, F&& f) {
  try {
    f();
    if (err) err->clear();
    return KAN_OK;
  } catch (const IoError& x) {
    if (err) *err = x.what();
    return KAN_ERR_IO;
  } catch (const ChecksumError& x) {
    if (err) *err = x.what();
    return KAN_ERR_CHECKSUM;
  } catch (const FormatError& x) {
    if (err) *err = x.what();
    return KAN_ERR_FORMAT;
  } catch (const Unsupported& x) {
    if (err) *err = x.what();
    return KAN_ERR_UNSUPPORTED;
  } catch (const std::exception& x) {
    if (err) *err = x.what();
    return KAN_ERR_INVALID_ARGUMENT;
  }
}

thread_local std::string g_save_err;

}  // namespace
}  // namespace kan

extern "C" {

uint32_t kan_crc32(const uint8_t* data, size_t len) { return kan::crc32(data, len); }

kan_status kan_container_load(const char* path, kan_container** out) {
  if (!out || !path) return KAN_ERR_INVALID_ARGUMENT;
  auto c = std::make_unique<kan_container>();
  const kan_status st = kan::run(&c->err, [&] { kan::load(c.get(), path); });
  *out = c.release();  // on error the handle carries the message; the caller destroys it
  return st;
}

void kan_container_destroy(kan_container* c) { delete c; }

const char* kan_container_last_error(const kan_container* c) { return c ? c->err.c_str() : "null container"; }

const char* kan_container_descriptor(const kan_container* c) { return c ? c->descriptor.c_str() : ""; }

int kan_container_num_kan_layers(const kan_container* c) { return c ? static_cast<int>(c->coeffs.size()) : 0; }

int64_t kan_container_coeffs(const kan_container* c, int layer, double* out, int64_t cap) {
  if (!c || layer < 0 || layer >= static_cast<int>(c->coeffs.size())) return -KAN_ERR_INVALID_ARGUMENT;
  const auto& w = c->coeffs[static_cast<size_t>(layer)];
  const int64_t n = static_cast<int64_t>(w.size());
  if (out && cap >= n) std::memcpy(out, w.data(), w.size() * sizeof(double));
  return n;
}

int64_t kan_container_lut(const kan_container* c, uint8_t* out, int64_t cap, int* degree, int* k, int* h) {
  if (!c) return -KAN_ERR_INVALID_ARGUMENT;
  if (degree) *degree = c->lut_degree;
  if (k) *k = c->lut_k;
  if (h) *h = c->lut_h;
  const int64_t n = static_cast<int64_t>(c->lut.size());
  if (out && cap >= n && n) std::memcpy(out, c->lut.data(), c->lut.size());
  return n;
}

int kan_container_num_spline_tables(const kan_container* c) { return c ? static_cast<int>(c->tables.size()) : 0; }

int64_t kan_container_spline_table(const kan_container* c, int t, uint8_t* out, int64_t cap, int* bits_a, int* h,
                                   double* qp_d, int64_t* qp_i) {
  if (!c || t < 0 || t >= static_cast<int>(c->tables.size())) return -KAN_ERR_INVALID_ARGUMENT;
  const auto& tb = c->tables[static_cast<size_t>(t)];
  if (bits_a) *bits_a = tb.bits_a;
  if (h) *h = tb.h;
  if (qp_d) std::memcpy(qp_d, tb.qd, sizeof(tb.qd));
  if (qp_i) std::memcpy(qp_i, tb.qi, sizeof(tb.qi));
  const int64_t n = static_cast<int64_t>(tb.values.size());
  if (out && cap >= n && n) std::memcpy(out, tb.values.data(), tb.values.size());
  return n;
}

kan_status kan_container_save(const char* path, const char* descriptor_json, const double* const* coeffs,
                              const uint8_t* lut, int64_t lut_n, int lut_k, int lut_h,
                              const uint8_t* const* st_values, int st_bits_a, int st_h, const double* st_qp_d,
                              const int64_t* st_qp_i) {
  if (!path || !descriptor_json || !coeffs) return KAN_ERR_INVALID_ARGUMENT;
  return kan::run(&kan::g_save_err, [&] {
    kan::save(path, descriptor_json, coeffs, lut, lut_n, lut_k, lut_h, st_values, st_bits_a, st_h, st_qp_d,
              st_qp_i);
  });
}

const char* kan_container_save_error(void) { return kan::g_save_err.c_str(); }

}  // extern "C"
