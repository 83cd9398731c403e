// Small C-ABI helpers: thread-local error text, free, version.
#include <cstdlib>
#include <string>

#include "capi_util.hpp"

namespace poas_b200::capi {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

}  // namespace poas_b200::capi

extern "C" {

const char* poas_b200_last_error(void) { return poas_b200::capi::g_last_error.c_str(); }

void poas_b200_free(void* p) { std::free(p); }

const char* poas_b200_version(void) { return "poas-b200 0.1 (sm_100a)"; }

}  // extern "C"
