// error.hpp -- exception carried across the library and turned into a C return code at the ABI.
#pragma once
#include <stdint.h>

#include <string>

namespace hpdr {
struct Error {
    int code;
    std::string msg;
    int64_t bit_offset;
};
}  // namespace hpdr
