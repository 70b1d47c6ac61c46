// Internal host helpers shared by host.cpp and capi.cu.
#pragma once
#include <string>

#include "../../include/kvgpu.h"

namespace kvg_host {
int set_error(int code, const std::string& what);
bool validate_sim(const kvg_sim_desc& d, std::string* why);
bool validate_policy(const kvg_policy& p, std::string* why);
}  // namespace kvg_host
