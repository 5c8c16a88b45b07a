// odcsim/types.hpp — drop-in façade (B200 build).
// Same names and meaning as the reference's error taxonomy and log levels
// (/root/reference/proj/include/odcsim/types.hpp:11-59) so code written
// against the reference compiles unchanged. Each exception corresponds to one
// odc_status code of the C ABI (include/odc/odc.h); odcsim::detail::raise()
// turns a status back into the exception.
#ifndef ODCSIM_TYPES_HPP
#define ODCSIM_TYPES_HPP

#include <cstdint>
#include <stdexcept>
#include <string>

#include "odc/odc.h"

namespace odcsim {

using Tokens = std::int64_t;  // sequence lengths / token sums

struct ParamError : std::runtime_error { using std::runtime_error::runtime_error; };       // ODC_ERR_PARAM
struct FormatError : std::runtime_error { using std::runtime_error::runtime_error; };      // ODC_ERR_PARAM
struct InfeasibleError : std::runtime_error { using std::runtime_error::runtime_error; };  // ODC_ERR_INFEASIBLE
struct ModeError : std::runtime_error { using std::runtime_error::runtime_error; };        // ODC_ERR_MODE
struct ProtocolError : std::runtime_error { using std::runtime_error::runtime_error; };    // ODC_ERR_PROTOCOL
struct StateError : std::runtime_error { using std::runtime_error::runtime_error; };       // ODC_ERR_STATE
struct InvariantError : std::logic_error { using std::logic_error::logic_error; };         // ODC_ERR_INVARIANT
// No reference counterpart: CUDA failures and the device barrier watchdog.
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };      // ODC_ERR_CUDA/TIMEOUT

enum class LogLevel { Quiet = 0, Warn = 1, Info = 2, Debug = 3 };
LogLevel log_level();
void set_log_level(LogLevel level);
void set_log_level_from_env();  // ODC_SIM_LOG=quiet|warn|info|debug|0..3
void log_warn(const std::string& msg);
void log_info(const std::string& msg);
void log_debug(const std::string& msg);

namespace detail {
[[noreturn]] inline void raise(odc_status st, const std::string& what) {
    switch (st) {
        case ODC_ERR_PARAM: throw ParamError(what);
        case ODC_ERR_INFEASIBLE: throw InfeasibleError(what);
        case ODC_ERR_INVARIANT: throw InvariantError(what);
        case ODC_ERR_PROTOCOL: throw ProtocolError(what);
        case ODC_ERR_STATE: throw StateError(what);
        case ODC_ERR_MODE: throw ModeError(what);
        default: throw DeviceError(what);
    }
}
inline void check(odc_status st) {
    if (st != ODC_OK) raise(st, odc_last_error());
}
}  // namespace detail

}  // namespace odcsim

#endif
