// GBNN v1 weight container (binary, little-endian) and its JSON mirror.
// Restates the reference format and error classes (reference
// src/nn_io.cpp:19-247): magic "GBNN", u32 version = 1, u32 layer count; per
// layer u32 rows, u32 cols, u8 activation, rows*cols f64 weights row-major,
// rows f64 biases; no trailing bytes.  Activation code 4 (softplus) is this
// build's extension (the reference accepts 0..3, nn_io.cpp:77,184).
#include <atomic>
#include <bit>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fcntl.h>
#include <fstream>
#include <unistd.h>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "net.hpp"
#include "parallel_host.hpp"

#include "device_net.hpp"

static_assert(std::endian::native == std::endian::little, "GBNN I/O assumes a little-endian host");

namespace gbb {
namespace {

constexpr char kMagic[4] = {'G', 'B', 'N', 'N'};
constexpr std::uint32_t kVersion = 1;
constexpr std::uint32_t kMaxLayers = 4096;
constexpr std::uint32_t kMaxWidth = 16u * 1024u * 1024u;

template <typename T>
bool read_pod(std::istream& in, T* out) {
  char buf[sizeof(T)];
  if (!in.read(buf, sizeof(T))) return false;
  std::memcpy(out, buf, sizeof(T));
  return true;
}

template <typename T>
void write_pod(std::ostream& out, const T& v) {
  char buf[sizeof(T)];
  std::memcpy(buf, &v, sizeof(T));
  out.write(buf, sizeof(T));
}

bool ends_with_json(const std::string& path) {
  return path.size() >= 5 && path.compare(path.size() - 5, 5, ".json") == 0;
}

// ---- minimal JSON value + recursive-descent parser ------------------------
struct JVal {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0.0;
  bool is_int = false;
  long long inum = 0;
  std::string str;
  std::vector<JVal> arr;
  std::map<std::string, JVal> obj;
  const JVal* get(const std::string& k) const {
    auto it = obj.find(k);
    return it == obj.end() ? nullptr : &it->second;
  }
};

struct JsonParseError {};

class JParser {
 public:
  explicit JParser(const std::string& s) : s_(s) {}
  JVal parse_document() {
    JVal v = value();
    ws();
    if (p_ != s_.size()) throw JsonParseError{};
    return v;
  }

 private:
  void ws() {
    while (p_ < s_.size() && (s_[p_] == ' ' || s_[p_] == '\n' || s_[p_] == '\t' || s_[p_] == '\r')) ++p_;
  }
  char peek() {
    ws();
    if (p_ >= s_.size()) throw JsonParseError{};
    return s_[p_];
  }
  void expect(char c) {
    if (peek() != c) throw JsonParseError{};
    ++p_;
  }
  bool lit(const char* w) {
    size_t n = std::strlen(w);
    if (s_.compare(p_, n, w) == 0) {
      p_ += n;
      return true;
    }
    return false;
  }
  JVal value() {
    if (++depth_ > 256) throw JsonParseError{};
    JVal v;
    char c = peek();
    if (c == '{') {
      v.kind = JVal::Obj;
      ++p_;
      if (peek() == '}') {
        ++p_;
      } else {
        for (;;) {
          if (peek() != '"') throw JsonParseError{};
          std::string key = string_lit();
          expect(':');
          v.obj[key] = value();
          char d = peek();
          ++p_;
          if (d == '}') break;
          if (d != ',') throw JsonParseError{};
        }
      }
    } else if (c == '[') {
      v.kind = JVal::Arr;
      ++p_;
      if (peek() == ']') {
        ++p_;
      } else {
        for (;;) {
          v.arr.push_back(value());
          char d = peek();
          ++p_;
          if (d == ']') break;
          if (d != ',') throw JsonParseError{};
        }
      }
    } else if (c == '"') {
      v.kind = JVal::Str;
      v.str = string_lit();
    } else if (lit("true")) {
      v.kind = JVal::Bool;
      v.b = true;
    } else if (lit("false")) {
      v.kind = JVal::Bool;
    } else if (lit("null")) {
      v.kind = JVal::Null;
    } else {
      v.kind = JVal::Num;
      const char* start = s_.c_str() + p_;
      // JSON grammar check for the number token.
      size_t q = p_;
      if (q < s_.size() && s_[q] == '-') ++q;
      if (q >= s_.size() || !std::isdigit(static_cast<unsigned char>(s_[q]))) throw JsonParseError{};
      bool integral = true;
      while (q < s_.size() && std::isdigit(static_cast<unsigned char>(s_[q]))) ++q;
      if (q < s_.size() && s_[q] == '.') {
        integral = false;
        ++q;
        if (q >= s_.size() || !std::isdigit(static_cast<unsigned char>(s_[q]))) throw JsonParseError{};
        while (q < s_.size() && std::isdigit(static_cast<unsigned char>(s_[q]))) ++q;
      }
      if (q < s_.size() && (s_[q] == 'e' || s_[q] == 'E')) {
        integral = false;
        ++q;
        if (q < s_.size() && (s_[q] == '+' || s_[q] == '-')) ++q;
        if (q >= s_.size() || !std::isdigit(static_cast<unsigned char>(s_[q]))) throw JsonParseError{};
        while (q < s_.size() && std::isdigit(static_cast<unsigned char>(s_[q]))) ++q;
      }
      char* end = nullptr;
      errno = 0;
      v.num = std::strtod(start, &end);
      if (end != s_.c_str() + q) throw JsonParseError{};
      if (integral) {
        v.is_int = true;
        v.inum = std::strtoll(start, nullptr, 10);
      }
      p_ = q;
    }
    --depth_;
    return v;
  }
  std::string string_lit() {
    expect('"');
    std::string out;
    while (p_ < s_.size() && s_[p_] != '"') {
      char c = s_[p_++];
      if (c == '\\') {
        if (p_ >= s_.size()) throw JsonParseError{};
        char e = s_[p_++];
        switch (e) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'n': out += '\n'; break;
          case 'r': out += '\r'; break;
          case 't': out += '\t'; break;
          case 'u': {
            if (p_ + 4 > s_.size()) throw JsonParseError{};
            unsigned cp = static_cast<unsigned>(std::strtoul(s_.substr(p_, 4).c_str(), nullptr, 16));
            p_ += 4;
            if (cp < 0x80) out += static_cast<char>(cp);
            else out += '?';
            break;
          }
          default: throw JsonParseError{};
        }
      } else {
        out += c;
      }
    }
    if (p_ >= s_.size()) throw JsonParseError{};
    ++p_;
    return out;
  }
  const std::string& s_;
  size_t p_ = 0;
  int depth_ = 0;
};

std::int64_t as_int(const JVal& v, const std::string& path) {
  if (v.kind != JVal::Num) throw FormatError("load_weights: non-numeric field in " + path);
  if (v.is_int) return v.inum;
  return static_cast<std::int64_t>(v.num);
}

std::unique_ptr<Net> load_weights_json(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw IoError("load_weights: cannot open " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  const std::string text = ss.str();
  JVal doc;
  try {
    doc = JParser(text).parse_document();
  } catch (const JsonParseError&) {
    throw FormatError("load_weights: " + path + " is not valid JSON");
  }
  const JVal* magic = doc.kind == JVal::Obj ? doc.get("magic") : nullptr;
  if (!magic || magic->kind != JVal::Str || magic->str != "GBNN")
    throw FormatError("load_weights: " + path + " lacks the GBNN magic");
  const JVal* ver = doc.get("version");
  if (!ver || ver->kind != JVal::Num || as_int(*ver, path) != static_cast<std::int64_t>(kVersion))
    throw FormatError("load_weights: unsupported version in " + path);
  const JVal* jlayers = doc.get("layers");
  if (!jlayers || jlayers->kind != JVal::Arr || jlayers->arr.empty())
    throw DimensionError("load_weights: " + path + " declares no layers");
  std::vector<HostLayer> layers;
  for (const JVal& jl : jlayers->arr) {
    const JVal* jr = jl.kind == JVal::Obj ? jl.get("rows") : nullptr;
    const JVal* jc = jl.kind == JVal::Obj ? jl.get("cols") : nullptr;
    const JVal* ja = jl.kind == JVal::Obj ? jl.get("activation") : nullptr;
    const JVal* jw = jl.kind == JVal::Obj ? jl.get("weights") : nullptr;
    const JVal* jb = jl.kind == JVal::Obj ? jl.get("biases") : nullptr;
    if (!jr || !jc || !ja || !jw || !jb)
      throw FormatError("load_weights: layer object missing fields in " + path);
    const std::int64_t rows = as_int(*jr, path), cols = as_int(*jc, path), act = as_int(*ja, path);
    if (rows <= 0 || cols <= 0 || rows > kMaxWidth || cols > kMaxWidth)
      throw DimensionError("load_weights: implausible layer shape in " + path);
    if (act < 0 || act > kMaxActCode) throw FormatError("load_weights: unknown activation code in " + path);
    if (jw->kind != JVal::Arr || static_cast<std::int64_t>(jw->arr.size()) != rows || jb->kind != JVal::Arr ||
        static_cast<std::int64_t>(jb->arr.size()) != rows)
      throw DimensionError("load_weights: weight/bias row count mismatch in " + path);
    HostLayer lay;
    lay.rows = rows;
    lay.cols = cols;
    lay.act = static_cast<int>(act);
    lay.w.resize(static_cast<size_t>(rows * cols));
    lay.b.resize(static_cast<size_t>(rows));
    for (std::int64_t r = 0; r < rows; ++r) {
      const JVal& row = jw->arr[static_cast<size_t>(r)];
      if (row.kind != JVal::Arr || static_cast<std::int64_t>(row.arr.size()) != cols)
        throw DimensionError("load_weights: weight column count mismatch in " + path);
      for (std::int64_t c = 0; c < cols; ++c) {
        const JVal& e = row.arr[static_cast<size_t>(c)];
        if (e.kind != JVal::Num) throw FormatError("load_weights: non-numeric weight in " + path);
        lay.w[static_cast<size_t>(r * cols + c)] = e.num;
      }
    }
    for (std::int64_t r = 0; r < rows; ++r) {
      const JVal& e = jb->arr[static_cast<size_t>(r)];
      if (e.kind != JVal::Num) throw FormatError("load_weights: non-numeric bias in " + path);
      lay.b[static_cast<size_t>(r)] = e.num;
    }
    layers.push_back(std::move(lay));
  }
  return std::make_unique<Net>(std::move(layers));
}

void put_double(std::ostream& out, double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  // Keep it a JSON number token (e.g. never "inf"; values are validated finite).
  out << buf;
}

void save_weights_json(const Net& net, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw IoError("save_weights: cannot open " + path);
  out << "{\n \"layers\": [\n";
  for (size_t l = 0; l < net.layers().size(); ++l) {
    const HostLayer& lay = net.layers()[l];
    out << "  {\n   \"activation\": " << lay.act << ",\n   \"biases\": [";
    for (std::int64_t r = 0; r < lay.rows; ++r) {
      if (r) out << ", ";
      put_double(out, lay.b[static_cast<size_t>(r)]);
    }
    out << "],\n   \"cols\": " << lay.cols << ",\n   \"rows\": " << lay.rows << ",\n   \"weights\": [";
    for (std::int64_t r = 0; r < lay.rows; ++r) {
      out << (r ? ",\n    [" : "\n    [");
      for (std::int64_t c = 0; c < lay.cols; ++c) {
        if (c) out << ", ";
        put_double(out, lay.w[static_cast<size_t>(r * lay.cols + c)]);
      }
      out << "]";
    }
    out << "\n   ]\n  }" << (l + 1 < net.layers().size() ? "," : "") << "\n";
  }
  out << " ],\n \"magic\": \"GBNN\",\n \"version\": 1\n}\n";
  if (!out) throw IoError("save_weights: write failed for " + path);
}

}  // namespace

std::unique_ptr<Net> load_weights(const std::string& path) {
  if (ends_with_json(path)) return load_weights_json(path);
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("load_weights: cannot open " + path);
  struct Fd {
    int fd;
    ~Fd() {
      if (fd >= 0) ::close(fd);
    }
  } fd_guard{::open(path.c_str(), O_RDONLY)};
  const int fd = fd_guard.fd;
  char magic[4];
  if (!in.read(magic, 4) || std::memcmp(magic, kMagic, 4) != 0)
    throw FormatError("load_weights: " + path + " lacks the GBNN magic");
  std::uint32_t version = 0, layer_count = 0;
  if (!read_pod(in, &version)) throw FormatError("load_weights: header truncated in " + path);
  if (version != kVersion)
    throw FormatError("load_weights: unsupported version " + std::to_string(version) + " in " + path);
  if (!read_pod(in, &layer_count)) throw FormatError("load_weights: header truncated in " + path);
  if (layer_count == 0 || layer_count > kMaxLayers)
    throw DimensionError("load_weights: implausible layer count " + std::to_string(layer_count) + " in " + path);
  std::vector<HostLayer> layers;
  layers.reserve(layer_count);
  for (std::uint32_t l = 0; l < layer_count; ++l) {
    std::uint32_t rows = 0, cols = 0;
    std::uint8_t act = 0;
    if (!read_pod(in, &rows) || !read_pod(in, &cols) || !read_pod(in, &act))
      throw TruncatedError("load_weights: layer header truncated in " + path);
    if (rows == 0 || cols == 0 || rows > kMaxWidth || cols > kMaxWidth)
      throw DimensionError("load_weights: implausible shape " + std::to_string(rows) + "x" +
                           std::to_string(cols) + " in " + path);
    if (act > kMaxActCode)
      throw FormatError("load_weights: unknown activation code " + std::to_string(act) + " in " + path);
    if (!layers.empty() && static_cast<std::int64_t>(cols) != layers.back().rows)
      throw DimensionError("load_weights: layer " + std::to_string(l) + " input width does not chain in " + path);
    HostLayer lay;
    lay.rows = rows;
    lay.cols = cols;
    lay.act = act;
    // Row-major on disk and in host memory: large payloads are read with
    // parallel pread()s straight into the layer (no stream-buffer copy),
    // small ones through the stream.
    lay.w.resize(static_cast<size_t>(rows) * cols);
    const int64_t wbytes = static_cast<int64_t>(sizeof(double) * lay.w.size());
    if (fd >= 0 && wbytes >= (int64_t(16) << 20)) {
      const int64_t off0 = static_cast<int64_t>(in.tellg());
      std::atomic<bool> ok{off0 >= 0};
      char* dst = reinterpret_cast<char*>(lay.w.data());
      parallel_slices(wbytes, int64_t(4) << 20, [&](int64_t a, int64_t b) {
        while (a < b && ok) {
          const ssize_t got = ::pread(fd, dst + a, static_cast<size_t>(b - a), static_cast<off_t>(off0 + a));
          if (got <= 0) {
            ok = false;
            return;
          }
          a += got;
        }
      });
      if (!ok) throw TruncatedError("load_weights: weight payload truncated in " + path);
      in.seekg(off0 + wbytes);
    } else if (!in.read(reinterpret_cast<char*>(lay.w.data()), static_cast<std::streamsize>(wbytes))) {
      throw TruncatedError("load_weights: weight payload truncated in " + path);
    }
    lay.b.resize(rows);
    if (!in.read(reinterpret_cast<char*>(lay.b.data()), static_cast<std::streamsize>(sizeof(double) * rows)))
      throw TruncatedError("load_weights: bias payload truncated in " + path);
    layers.push_back(std::move(lay));
  }
  char extra;
  if (in.read(&extra, 1)) throw FormatError("load_weights: trailing bytes after payload in " + path);
  return std::make_unique<Net>(std::move(layers));
}

void save_weights(const Net& net, const std::string& path) {
  if (ends_with_json(path)) {
    save_weights_json(net, path);
    return;
  }
  std::ofstream out(path, std::ios::binary);
  if (!out) throw IoError("save_weights: cannot open " + path);
  out.write(kMagic, 4);
  write_pod(out, kVersion);
  write_pod(out, static_cast<std::uint32_t>(net.layer_count()));
  for (const HostLayer& lay : net.layers()) {
    write_pod(out, static_cast<std::uint32_t>(lay.rows));
    write_pod(out, static_cast<std::uint32_t>(lay.cols));
    write_pod(out, static_cast<std::uint8_t>(lay.act));
    out.write(reinterpret_cast<const char*>(lay.w.data()), static_cast<std::streamsize>(sizeof(double) * lay.w.size()));
    out.write(reinterpret_cast<const char*>(lay.b.data()), static_cast<std::streamsize>(sizeof(double) * lay.b.size()));
  }
  if (!out) throw IoError("save_weights: write failed for " + path);
}

}  // namespace gbb
