// device.hpp — glue between the drop-in API and the C ABI: status codes
// become the reference exception types (errors.hpp), in the order the C ABI
// reports them (which is the reference's check order).
#pragma once

#include <string>

#include "../../../include/lowbit_cuda.h"
#include "lowbit/errors.hpp"

namespace lowbit::detail {

[[noreturn]] void raise(lowbit_status st, const char* where);

inline void check(lowbit_status st, const char* where) {
    if (st != LOWBIT_OK) raise(st, where);
}

}  // namespace lowbit::detail
