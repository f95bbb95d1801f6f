#include <cstring>

#include "h2b_internal.h"

namespace h2b {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
const std::string& get_error() { return g_last_error; }

}  // namespace h2b

extern "C" int h2b_last_error(char* buf, size_t n) {
    const std::string& e = h2b::get_error();
    if (buf && n) {
        const size_t m = e.size() < n - 1 ? e.size() : n - 1;
        std::memcpy(buf, e.data(), m);
        buf[m] = '\0';
    }
    return (int)e.size();
}

extern "C" int h2b_abi_version(void) { return 1; }
