// Internal helpers shared by the libh2b translation units: last-error storage
// and status plumbing (C ABI functions return codes, never throw).
#pragma once

#include <string>

#include "../../include/h2b.h"

namespace h2b {

void set_error(const std::string& msg);
const std::string& get_error();

inline int fail(int code, const std::string& msg) {
    set_error(msg);
    return code;
}

inline int ok() { return H2B_OK; }

}  // namespace h2b
