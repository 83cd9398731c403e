#pragma once
// stderr diagnostics gated by POAS_LOG=quiet|info|debug (default info),
// "poas: " prefixed, as in the reference (proj/src/log.cpp:16-45).

#include <optional>
#include <string>

namespace poas {

enum class LogLevel { quiet = 0, info = 1, debug = 2 };

std::optional<LogLevel> parse_log_level(const std::string& text);
LogLevel log_level();

void log_info(const char* fmt, ...) __attribute__((format(printf, 1, 2)));
void log_debug(const char* fmt, ...) __attribute__((format(printf, 1, 2)));

}  // namespace poas
