// Internal helpers shared by the host (.cpp) and device (.cu) sources.
#pragma once
#include <string>

#include "../../include/meshchroma_b200.h"

#define MC_API __attribute__((visibility("default")))

void mc_set_error(const std::string& msg);
int mc_fail(int code, const std::string& msg);
