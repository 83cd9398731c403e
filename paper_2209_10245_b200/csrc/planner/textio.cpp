// Line/block text format and stderr logging.
// Behaviour follows the reference's kv parser (proj/src/kv_format.cpp:28-116)
// and logger (proj/src/log.cpp:16-45); error classes are parse_failure with a
// "line N: ..." message.
#include <cerrno>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <string_view>

#include "poas/error.hpp"
#include "poas/kv_format.hpp"
#include "poas/log.hpp"

namespace poas {

std::optional<LogLevel> parse_log_level(const std::string& text) {
  if (text == "quiet") return LogLevel::quiet;
  if (text == "info") return LogLevel::info;
  if (text == "debug") return LogLevel::debug;
  return std::nullopt;
}

LogLevel log_level() {
  static const LogLevel cached = [] {
    const char* env = std::getenv("POAS_LOG");
    return env ? parse_log_level(env).value_or(LogLevel::info) : LogLevel::info;
  }();
  return cached;
}

namespace {
void emit(const char* fmt, va_list ap) {
  std::fputs("poas: ", stderr);
  std::vfprintf(stderr, fmt, ap);
  std::fputc('\n', stderr);
}
}  // namespace

void log_info(const char* fmt, ...) {
  if (log_level() < LogLevel::info) return;
  va_list ap;
  va_start(ap, fmt);
  emit(fmt, ap);
  va_end(ap);
}

void log_debug(const char* fmt, ...) {
  if (log_level() < LogLevel::debug) return;
  va_list ap;
  va_start(ap, fmt);
  emit(fmt, ap);
  va_end(ap);
}

namespace kv {

void fail_at(int line, const std::string& what) {
  poas::fail(errc::parse_failure, "line " + std::to_string(line) + ": " + what);
}

const Entry* Block::find(const std::string& key) const {
  for (const Entry& e : entries)
    if (e.key == key) return &e;
  return nullptr;
}

File parse(const std::string& text, const std::string& expected_header) {
  // Split into lines the way std::getline does: '\n' terminates a line and
  // a trailing '\n' does not create an extra empty line. One trailing '\r'
  // per line is dropped.
  std::vector<std::string_view> lines;
  {
    std::string_view rest(text);
    while (!rest.empty()) {
      const size_t nl = rest.find('\n');
      std::string_view ln = rest.substr(0, nl);
      if (!ln.empty() && ln.back() == '\r') ln.remove_suffix(1);
      lines.push_back(ln);
      if (nl == std::string_view::npos) break;
      rest.remove_prefix(nl + 1);
    }
  }
  if (lines.empty()) fail_at(1, "empty file, expected header '" + expected_header + "'");

  File file;
  file.header = std::string(lines[0]);
  if (file.header != expected_header)
    fail_at(1, "bad header '" + file.header + "', expected '" + expected_header + "'");

  bool open_block = false;
  for (size_t i = 1; i < lines.size(); ++i) {
    const int ln = static_cast<int>(i) + 1;
    const std::string_view s = lines[i];
    if (s.empty()) {
      open_block = false;
      continue;
    }
    if (s.front() == ' ' || s.front() == '\t') fail_at(ln, "unexpected leading whitespace");

    std::string head(s);
    std::string tail;
    const size_t sp = s.find(' ');
    if (sp != std::string_view::npos) {
      head = std::string(s.substr(0, sp));
      tail = std::string(s.substr(sp + 1));
      if (tail.empty()) fail_at(ln, "trailing space after '" + head + "'");
    }

    if (!open_block) {
      Block b;
      b.name = head;
      b.arg = tail;
      b.line = ln;
      file.blocks.push_back(std::move(b));
      open_block = true;
      continue;
    }
    if (tail.empty()) fail_at(ln, "key '" + head + "' has no value");
    Block& cur = file.blocks.back();
    if (cur.find(head)) fail_at(ln, "duplicate key '" + head + "'");
    cur.entries.push_back(Entry{head, tail, ln});
  }
  return file;
}

double parse_double(const Entry& e) {
  errno = 0;
  char* end = nullptr;
  const double v = std::strtod(e.value.c_str(), &end);
  const bool whole = !e.value.empty() && end == e.value.c_str() + e.value.size();
  if (!whole || errno == ERANGE || !std::isfinite(v))
    fail_at(e.line, "key '" + e.key + "': bad number '" + e.value + "'");
  return v;
}

std::int64_t parse_int(const Entry& e) {
  errno = 0;
  char* end = nullptr;
  const long long v = std::strtoll(e.value.c_str(), &end, 10);
  const bool whole = !e.value.empty() && end == e.value.c_str() + e.value.size();
  if (!whole || errno == ERANGE)
    fail_at(e.line, "key '" + e.key + "': bad integer '" + e.value + "'");
  return v;
}

std::uint64_t parse_uint(const Entry& e) {
  if (!e.value.empty() && e.value.front() == '-')
    fail_at(e.line, "key '" + e.key + "': negative value '" + e.value + "'");
  errno = 0;
  char* end = nullptr;
  const unsigned long long v = std::strtoull(e.value.c_str(), &end, 10);
  const bool whole = !e.value.empty() && end == e.value.c_str() + e.value.size();
  if (!whole || errno == ERANGE)
    fail_at(e.line, "key '" + e.key + "': bad integer '" + e.value + "'");
  return v;
}

bool parse_bool(const Entry& e) {
  if (e.value == "true") return true;
  if (e.value == "false") return false;
  fail_at(e.line, "key '" + e.key + "': expected true or false, got '" + e.value + "'");
}

std::string format_double(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

}  // namespace kv
}  // namespace poas
