// common.hpp — shared host helpers for libodc.so: thread-local last error and
// the exception <-> odc_status mapping used at every extern "C" entry point.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "odc/odc.h"
#include "odcsim/types.hpp"

namespace odc {

void set_last_error(const std::string& msg);

// Runs `f` and converts any exception into an odc_status + last error.
template <typename F>
odc_status guard(F&& f) {
    try {
        f();
        return ODC_OK;
    } catch (const odcsim::ParamError& e) {
        set_last_error(e.what());
        return ODC_ERR_PARAM;
    } catch (const odcsim::FormatError& e) {
        set_last_error(e.what());
        return ODC_ERR_PARAM;
    } catch (const odcsim::InfeasibleError& e) {
        set_last_error(e.what());
        return ODC_ERR_INFEASIBLE;
    } catch (const odcsim::ProtocolError& e) {
        set_last_error(e.what());
        return ODC_ERR_PROTOCOL;
    } catch (const odcsim::StateError& e) {
        set_last_error(e.what());
        return ODC_ERR_STATE;
    } catch (const odcsim::ModeError& e) {
        set_last_error(e.what());
        return ODC_ERR_MODE;
    } catch (const odcsim::InvariantError& e) {
        set_last_error(e.what());
        return ODC_ERR_INVARIANT;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return ODC_ERR_CUDA;
    }
}

}  // namespace odc
