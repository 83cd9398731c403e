// Exception -> error-code translation for the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>

#include "poas/error.hpp"
#include "poas_b200.h"

namespace poas_b200::capi {

// Error carrying an ABI code that is not a poas::errc (CUDA, internal).
struct AbiError : std::runtime_error {
  AbiError(int c, const std::string& what) : std::runtime_error(what), code(c) {}
  int code;
};

[[noreturn]] inline void raise(int code, const std::string& what) { throw AbiError(code, what); }

void set_last_error(const std::string& msg);

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    raise(POAS_E_CUDA, std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                           cudaGetErrorString(e) + ")");
}

inline int errc_code(poas::errc c) { return static_cast<int>(c) + 1; }

template <class F>
int guard(F&& f) {
  try {
    f();
    set_last_error("");
    return POAS_OK;
  } catch (const poas::Error& e) {
    set_last_error(e.what());
    return errc_code(e.code());
  } catch (const AbiError& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(std::string("internal error: ") + e.what());
    return POAS_E_INTERNAL;
  } catch (...) {
    set_last_error("internal error");
    return POAS_E_INTERNAL;
  }
}

inline std::string json_escape(const std::string& s) {
  std::string o;
  for (const char c : s) {
    if (c == '"' || c == '\\') {
      o += '\\';
      o += c;
    } else if (c == '\n') {
      o += "\\n";
    } else if (static_cast<unsigned char>(c) < 0x20) {
      char buf[8];
      std::snprintf(buf, sizeof buf, "\\u%04x", c);
      o += buf;
    } else {
      o += c;
    }
  }
  return o;
}

inline char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (!p) throw std::bad_alloc();
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

}  // namespace poas_b200::capi
