// quake_b200/io.hpp — buffer files of the reference's `quake apply` path.
//
// Formats (reference proj/README.md "buffer formats", core/include/quake/
// io.hpp:44-65, behaviour of core/src/io.cpp:45-111):
//   raw: 4-byte magic "QAKE", little-endian u32 element count, then count
//        little-endian binary32 values; the file length must match exactly.
//   csv: decimal tokens separated by ',', ' ', '\t', '\n' or '\r'; written
//        one value per line with "%.9g" (round-trips every binary32).
// Errors: ParseError (malformed content; the CLI maps it to exit 2) and
// IoError (cannot open / read / write; exit 3).
#ifndef QUAKE_B200_IO_HPP_
#define QUAKE_B200_IO_HPP_

#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace quake::io {

enum class BufferFormat { Csv, Raw };

struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {

inline std::string slurp(const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw IoError("cannot open for reading: " + path);
  std::string data;
  char chunk[1 << 16];
  size_t got;
  while ((got = std::fread(chunk, 1, sizeof(chunk), f)) > 0) data.append(chunk, got);
  const bool bad = std::ferror(f) != 0;
  std::fclose(f);
  if (bad) throw IoError("read failure: " + path);
  return data;
}

inline bool is_sep(char c) { return c == ',' || c == ' ' || c == '\t' || c == '\n' || c == '\r'; }

inline uint32_t load_le32(const unsigned char* p) {
  return uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
}

inline void store_le32(unsigned char* p, uint32_t v) {
  p[0] = static_cast<unsigned char>(v);
  p[1] = static_cast<unsigned char>(v >> 8);
  p[2] = static_cast<unsigned char>(v >> 16);
  p[3] = static_cast<unsigned char>(v >> 24);
}

}  // namespace detail

inline std::vector<float> parse_raw(const std::string& bytes, const std::string& path) {
  if (bytes.size() < 8 || std::memcmp(bytes.data(), "QAKE", 4) != 0) {
    throw ParseError("not a QAKE raw buffer: " + path);
  }
  const auto* p = reinterpret_cast<const unsigned char*>(bytes.data());
  const uint64_t count = detail::load_le32(p + 4);
  if (bytes.size() - 8 != count * 4) throw ParseError("raw buffer length mismatch: " + path);
  std::vector<float> values(count);
  for (uint64_t i = 0; i < count; ++i) {
    const uint32_t w = detail::load_le32(p + 8 + 4 * i);
    std::memcpy(&values[i], &w, 4);
  }
  return values;
}

inline std::vector<float> parse_csv(const std::string& text, const std::string& path) {
  std::vector<float> values;
  size_t i = 0;
  const size_t n = text.size();
  while (i < n) {
    while (i < n && detail::is_sep(text[i])) ++i;
    if (i >= n) break;
    const char* begin = text.c_str() + i;
    char* end = nullptr;
    errno = 0;
    const float v = std::strtof(begin, &end);
    if (end == begin) throw ParseError("bad numeric token in " + path);
    values.push_back(v);
    i = static_cast<size_t>(end - text.c_str());
    if (i < n && !detail::is_sep(text[i])) throw ParseError("bad numeric token in " + path);
  }
  return values;
}

inline std::vector<float> read_buffer(const std::string& path, BufferFormat format) {
  const std::string bytes = detail::slurp(path);
  return format == BufferFormat::Raw ? parse_raw(bytes, path) : parse_csv(bytes, path);
}

inline std::string format_number(double v) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.9g", v);
  return buf;
}

inline void write_buffer(const std::string& path, std::span<const float> values,
                         BufferFormat format) {
  if (format == BufferFormat::Raw && values.size() > 0xFFFFFFFFull) {
    throw IoError("raw buffer too large for a u32 count: " + path);
  }
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw IoError("cannot open for writing: " + path);
  bool ok = true;
  if (format == BufferFormat::Raw) {
    unsigned char head[8] = {'Q', 'A', 'K', 'E', 0, 0, 0, 0};
    detail::store_le32(head + 4, static_cast<uint32_t>(values.size()));
    ok = std::fwrite(head, 1, 8, f) == 8;
    std::vector<unsigned char> body(values.size() * 4);
    for (size_t i = 0; i < values.size(); ++i) {
      uint32_t w;
      std::memcpy(&w, &values[i], 4);
      detail::store_le32(body.data() + 4 * i, w);
    }
    ok = ok && std::fwrite(body.data(), 1, body.size(), f) == body.size();
  } else {
    for (const float v : values) {
      const std::string s = format_number(v) + "\n";
      if (std::fwrite(s.data(), 1, s.size(), f) != s.size()) {
        ok = false;
        break;
      }
    }
  }
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) throw IoError("write failure: " + path);
}

}  // namespace quake::io

#endif  // QUAKE_B200_IO_HPP_
