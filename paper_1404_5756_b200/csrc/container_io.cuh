// Container I/O (io.cpp:133-281, README "File formats"):
// rgf-grid / rgf-scale / rgf-field binary containers -- one JSON header line,
// then raw little-endian payload sections in header order, x fastest.
//
// Fields are streamed straight into device memory: the payload is read in
// chunks into two pinned host buffers while the previous chunk's H2D copy
// runs on the caller's stream (and the reverse for saves), so a field never
// needs a full host copy. Grids and scale fields (construction inputs) are
// read into caller host buffers. Headers are written exactly as nlohmann's
// json::dump() writes them (keys sorted, no spaces), so saving and
// re-loading reproduces a container byte for byte (README).
//
// Extension: an rgf-field may hold a stack of `nlev` levels ("nlev" key,
// written only when nlev > 1); the reference's reader sees its first level.
#pragma once
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace rgfio {

struct Header {
  std::map<std::string, std::string> scalars;  // raw JSON scalar text (strings unquoted)
  std::vector<std::string> sections;
  bool has_sections = false;
};

// Minimal parser for the flat header object (strings, integers, one array of
// strings). Anything else is a malformed header.
inline Header parse_header(const std::string& line) {
  Header h;
  size_t i = 0;
  auto fail = [&](const char* why) {
    throw std::runtime_error(std::string("malformed container header: ") + why);
  };
  auto ws = [&] {
    while (i < line.size() && (line[i] == ' ' || line[i] == '\t' || line[i] == '\r')) ++i;
  };
  auto str = [&]() -> std::string {
    ws();
    if (i >= line.size() || line[i] != '"') fail("expected a string");
    std::string s;
    for (++i; i < line.size() && line[i] != '"'; ++i) {
      if (line[i] == '\\') {
        if (++i >= line.size()) fail("bad escape");
      }
      s.push_back(line[i]);
    }
    if (i >= line.size()) fail("unterminated string");
    ++i;
    return s;
  };
  ws();
  if (i >= line.size() || line[i] != '{') fail("expected an object");
  ++i;
  ws();
  if (i < line.size() && line[i] == '}') return h;
  for (;;) {
    const std::string key = str();
    ws();
    if (i >= line.size() || line[i] != ':') fail("expected ':'");
    ++i;
    ws();
    if (i >= line.size()) fail("truncated");
    if (line[i] == '"') {
      h.scalars[key] = str();
    } else if (line[i] == '[') {
      ++i;
      std::vector<std::string> v;
      ws();
      if (i < line.size() && line[i] == ']') {
        ++i;
      } else {
        for (;;) {
          v.push_back(str());
          ws();
          if (i < line.size() && line[i] == ',') {
            ++i;
            continue;
          }
          if (i < line.size() && line[i] == ']') {
            ++i;
            break;
          }
          fail("expected ',' or ']'");
        }
      }
      if (key == "sections") {
        h.sections = v;
        h.has_sections = true;
      }
    } else {
      const size_t j = i;
      while (i < line.size() && (std::isdigit(static_cast<unsigned char>(line[i])) ||
                                 line[i] == '-' || line[i] == '+'))
        ++i;
      if (i == j) fail("unsupported value");
      h.scalars[key] = line.substr(j, i - j);
    }
    ws();
    if (i < line.size() && line[i] == ',') {
      ++i;
      continue;
    }
    if (i < line.size() && line[i] == '}') break;
    fail("expected ',' or '}'");
  }
  return h;
}

struct File {
  FILE* f = nullptr;
  std::string path;
  File(const std::string& p, const char* mode) : path(p) {
    f = std::fopen(p.c_str(), mode);
    if (!f)
      throw std::runtime_error(std::string(mode[0] == 'r' ? "cannot open " : "cannot write ") + p);
  }
  ~File() {
    if (f) std::fclose(f);
  }
  File(const File&) = delete;
  File& operator=(const File&) = delete;
};

// io.cpp read_header: one line, the expected "format", little-endian, nx/ny
inline Header read_header(File& in, const std::string& expected) {
  std::string line;
  int c;
  while ((c = std::fgetc(in.f)) != EOF && c != '\n') line.push_back(static_cast<char>(c));
  if (line.empty() && c == EOF) throw std::runtime_error("missing container header");
  Header h = parse_header(line);
  const auto fmt = h.scalars.find("format");
  if (fmt == h.scalars.end() || fmt->second != expected)
    throw std::runtime_error("expected a \"" + expected + "\" container");
  const auto en = h.scalars.find("endianness");
  if (en != h.scalars.end() && en->second != "little")
    throw std::runtime_error("only little-endian payloads are supported");
  if (!h.scalars.count("nx") || !h.scalars.count("ny"))
    throw std::runtime_error("container header is missing nx/ny");
  return h;
}

inline int64_t get_int(const Header& h, const char* key, int64_t dflt) {
  const auto it = h.scalars.find(key);
  return it == h.scalars.end() ? dflt : std::stoll(it->second);
}

// nlohmann::json::dump() of the writer's object: keys in std::map order
inline std::string dump_header(const std::string& format, int64_t nx, int64_t ny,
                               const int64_t* ghost, int64_t nlev,
                               const std::vector<std::string>& sections) {
  std::string s = "{\"endianness\":\"little\",\"format\":\"" + format + "\"";
  if (ghost) s += ",\"ghost_width\":" + std::to_string(*ghost);
  if (nlev > 1) s += ",\"nlev\":" + std::to_string(nlev);
  s += ",\"nx\":" + std::to_string(nx) + ",\"ny\":" + std::to_string(ny) + ",\"sections\":[";
  for (size_t k = 0; k < sections.size(); ++k) s += (k ? ",\"" : "\"") + sections[k] + "\"";
  return s + "]}\n";
}

inline void read_exact(File& in, void* dst, size_t bytes, const std::string& what) {
  if (bytes && std::fread(dst, 1, bytes, in.f) != bytes) throw std::runtime_error(what);
}
inline void write_exact(File& out, const void* src, size_t bytes) {
  if (bytes && std::fwrite(src, 1, bytes, out.f) != bytes)
    throw std::runtime_error("failed while writing " + out.path);
}
inline void expect_eof(File& in, const char* what) {
  if (std::fgetc(in.f) != EOF) throw std::runtime_error(what);
}

}  // namespace rgfio
