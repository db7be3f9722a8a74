#include "device.hpp"

namespace lowbit::detail {

namespace {
// Strip the "<prefix>: " that the reference exception constructors add back.
std::string tail(const char* msg, const char* prefix) {
    std::string s = msg ? msg : "";
    std::string p = prefix;
    if (s.rfind(p, 0) == 0) return s.substr(p.size());
    return s;
}
}  // namespace

void raise(lowbit_status st, const char* where) {
    const char* msg = lowbit_last_error();
    long long v0 = 0, v1 = 0;
    lowbit_last_error_values(&v0, &v1);
    switch (st) {
        case LOWBIT_ZERO_IN_BINARY: throw ZeroInBinaryInput();
        case LOWBIT_INVALID_CODE: throw InvalidCode();
        case LOWBIT_OUT_OF_BOUNDS: throw OutOfBounds(tail(msg, "out of bounds: "));
        case LOWBIT_DEPTH_OVERFLOW: throw DepthOverflow(static_cast<long>(v0), static_cast<long>(v1));
        case LOWBIT_MODE_MISMATCH: throw ModeMismatch(tail(msg, "mode mismatch: "));
        case LOWBIT_CHANNEL_OVERFLOW: throw ChannelOverflow(static_cast<long>(v0), static_cast<long>(v1));
        case LOWBIT_EMPTY_OUTPUT: throw EmptyOutput();
        case LOWBIT_ERROR: throw Error(msg && *msg ? msg : where);
        default: throw DeviceError(std::string(where) + ": " + (msg ? msg : "") + " [" + lowbit_status_string(st) + "]");
    }
}

}  // namespace lowbit::detail
