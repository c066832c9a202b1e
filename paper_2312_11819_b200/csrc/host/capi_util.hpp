// Shared helpers of the C-ABI translation units.
#pragma once

#include <exception>
#include <string>

#include "flexrlhf/errors.hpp"

namespace flexrlhf {
extern thread_local std::string g_last_error;
// Record e.what() for rlhf_last_error() and map the exception type to the
// reference's exit codes (errors.hpp:8-22) + 5 for device errors.
int capi_status(const std::exception& e);
}  // namespace flexrlhf
