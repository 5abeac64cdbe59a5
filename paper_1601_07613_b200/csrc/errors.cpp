// Thread-local last-error slot behind mc_last_error().
#include <string>

#include "mc_internal.h"

namespace {
thread_local std::string g_last_error;
}

void mc_set_error(const std::string& msg) { g_last_error = msg; }

int mc_fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

extern "C" MC_API const char* mc_last_error(void) { return g_last_error.c_str(); }

extern "C" MC_API int mc_abi_version(void) { return 1011; }  // 1011: mc_dg_desc.elem_kind (hybrid meshes)
