// Oracle restatement of the reference's container I/O (test infrastructure
// only): /root/reference/proj/src/io.cpp:133-281, binary rgf-grid /
// rgf-scale / rgf-field containers, read and written with nlohmann::json
// (the library io.cpp uses; the copy vendored in this image, v3.11.3), so it
// is an independent check of the product's own header parser/writer
// (paper_1404_5756_b200/csrc/container_io.cuh). The CSV dialect is out of
// scope on both sides.
#include <cstdint>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "rgf_oracle.h"

namespace {
using nlohmann::json;

thread_local std::string g_io_error;

std::ifstream open_input(const std::string& path) {  // io.cpp:24-28
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open " + path);
  return in;
}

json read_header(std::istream& in, const std::string& expected_format) {  // io.cpp:37-55
  std::string line;
  if (!std::getline(in, line)) throw std::runtime_error("missing container header");
  json h;
  try {
    h = json::parse(line);
  } catch (const json::exception& e) {
    throw std::runtime_error(std::string("malformed container header: ") + e.what());
  }
  if (h.value("format", "") != expected_format)
    throw std::runtime_error("expected a \"" + expected_format + "\" container");
  if (h.value("endianness", "little") != "little")
    throw std::runtime_error("only little-endian payloads are supported");
  if (!h.contains("nx") || !h.contains("ny"))
    throw std::runtime_error("container header is missing nx/ny");
  return h;
}

void read_f64(std::istream& in, double* out, int64_t n, const std::string& name) {  // :57-67
  in.read(reinterpret_cast<char*>(out), static_cast<std::streamsize>(sizeof(double) * n));
  if (!in) throw std::runtime_error("payload section \"" + name +
                                    "\" is truncated (dimension mismatch?)");
}

template <typename F>
int io_guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_io_error = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_io_error = e.what();
    return 2;
  }
}
}  // namespace

extern "C" {

const char* rgfo_io_last_error(void) { return g_io_error.c_str(); }

int rgfo_load_grid(const char* path, int64_t nx, int64_t ny, double* dx, double* dy,
                   uint8_t* mask, int64_t* ghost_width) {  // io.cpp:133-159
  return io_guarded([&] {
    std::ifstream in = open_input(path);
    const json h = read_header(in, "rgf-grid");
    if (h["nx"].get<int64_t>() != nx || h["ny"].get<int64_t>() != ny)
      throw std::invalid_argument("buffers do not match the container");
    *ghost_width = h.value("ghost_width", int64_t(0));
    bool has_dx = false, has_dy = false, has_mask = false;
    for (const auto& sec : h.value("sections", std::vector<std::string>{})) {
      if (sec == "dx") {
        read_f64(in, dx, nx * ny, "dx");
        has_dx = true;
      } else if (sec == "dy") {
        read_f64(in, dy, nx * ny, "dy");
        has_dy = true;
      } else if (sec == "mask") {  // io.cpp:69-79
        std::vector<unsigned char> raw(static_cast<size_t>(nx * ny));
        in.read(reinterpret_cast<char*>(raw.data()), static_cast<std::streamsize>(raw.size()));
        if (!in) throw std::runtime_error("mask section is truncated");
        for (size_t p = 0; p < raw.size(); ++p) mask[p] = raw[p] != 0;
        has_mask = true;
      } else {
        throw std::runtime_error("unknown grid section \"" + sec + "\"");
      }
    }
    if (!has_dx || !has_dy) throw std::runtime_error("grid container is missing dx/dy sections");
    if (!has_mask) std::memset(mask, 1, static_cast<size_t>(nx * ny));
    in.peek();
    if (!in.eof()) throw std::runtime_error("trailing bytes after grid payload");
  });
}

int rgfo_save_grid(const char* path, int64_t nx, int64_t ny, int64_t ghost_width,
                   const double* dx, const double* dy, const uint8_t* mask) {  // io.cpp:183-202
  return io_guarded([&] {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error(std::string("cannot write ") + path);
    json h{{"format", "rgf-grid"}, {"nx", nx}, {"ny", ny}, {"ghost_width", ghost_width},
           {"endianness", "little"}, {"sections", {"dx", "dy", "mask"}}};
    out << h.dump() << '\n';
    out.write(reinterpret_cast<const char*>(dx), static_cast<std::streamsize>(8 * nx * ny));
    out.write(reinterpret_cast<const char*>(dy), static_cast<std::streamsize>(8 * nx * ny));
    std::vector<unsigned char> raw(static_cast<size_t>(nx * ny));
    for (size_t p = 0; p < raw.size(); ++p) raw[p] = mask[p] ? 1 : 0;
    out.write(reinterpret_cast<const char*>(raw.data()), static_cast<std::streamsize>(raw.size()));
    if (!out) throw std::runtime_error(std::string("failed while writing ") + path);
  });
}

int rgfo_load_scale(const char* path, int64_t nx, int64_t ny, double* rx, double* ry) {
  return io_guarded([&] {  // io.cpp:204-235 (binary branch; validation is grid.cpp's)
    std::ifstream in = open_input(path);
    const json h = read_header(in, "rgf-scale");
    if (h["nx"].get<int64_t>() != nx || h["ny"].get<int64_t>() != ny)
      throw std::runtime_error("scale file dimensions do not match the grid");
    bool has_rx = false, has_ry = false;
    for (const auto& sec : h.value("sections", std::vector<std::string>{})) {
      if (sec == "rx") {
        read_f64(in, rx, nx * ny, "rx");
        has_rx = true;
      } else if (sec == "ry") {
        read_f64(in, ry, nx * ny, "ry");
        has_ry = true;
      } else {
        throw std::runtime_error("unknown scale section \"" + sec + "\"");
      }
    }
    if (!has_rx) throw std::runtime_error("scale file is missing the zonal (rx) component");
    if (!has_ry) throw std::runtime_error("scale file is missing the meridional (ry) component");
  });
}

int rgfo_save_scale(const char* path, int64_t nx, int64_t ny, const double* rx,
                    const double* ry) {  // io.cpp:237-249
  return io_guarded([&] {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error(std::string("cannot write ") + path);
    json h{{"format", "rgf-scale"}, {"nx", nx}, {"ny", ny}, {"endianness", "little"},
           {"sections", {"rx", "ry"}}};
    out << h.dump() << '\n';
    out.write(reinterpret_cast<const char*>(rx), static_cast<std::streamsize>(8 * nx * ny));
    out.write(reinterpret_cast<const char*>(ry), static_cast<std::streamsize>(8 * nx * ny));
    if (!out) throw std::runtime_error(std::string("failed while writing ") + path);
  });
}

int rgfo_load_field(const char* path, int64_t nx, int64_t ny, double* values) {
  return io_guarded([&] {  // io.cpp:251-269 (binary branch)
    std::ifstream in = open_input(path);
    const json h = read_header(in, "rgf-field");
    if (h["nx"].get<int64_t>() != nx || h["ny"].get<int64_t>() != ny)
      throw std::runtime_error("field file dimensions do not match the grid");
    read_f64(in, values, nx * ny, "values");
  });
}

int rgfo_save_field(const char* path, int64_t nx, int64_t ny, const double* values) {
  return io_guarded([&] {  // io.cpp:271-281
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error(std::string("cannot write ") + path);
    json h{{"format", "rgf-field"}, {"nx", nx}, {"ny", ny}, {"endianness", "little"},
           {"sections", {"values"}}};
    out << h.dump() << '\n';
    out.write(reinterpret_cast<const char*>(values), static_cast<std::streamsize>(8 * nx * ny));
    if (!out) throw std::runtime_error(std::string("failed while writing ") + path);
  });
}

}  // extern "C"
