// Error model of the engine's C++ API.
//
// Mirrors the reference's exception types and exit codes
// (/root/reference/proj/include/rlhfsim/errors.hpp:8-22): 2 = config error,
// 3 = infeasible, 4 = search cap.  The engine adds DeviceError (exit code 5) for
// CUDA / NCCL failures; it never crosses the C-ABI as an exception (capi.cpp
// maps every exception to an int status).
#pragma once

#include <stdexcept>
#include <string>

namespace flexrlhf {

struct ConfigError : std::runtime_error {
  explicit ConfigError(const std::string& what) : std::runtime_error(what) {}
  static constexpr int exit_code = 2;
};

struct InfeasibleError : std::runtime_error {
  explicit InfeasibleError(const std::string& what) : std::runtime_error(what) {}
  static constexpr int exit_code = 3;
};

struct SearchCapError : std::runtime_error {
  explicit SearchCapError(const std::string& what) : std::runtime_error(what) {}
  static constexpr int exit_code = 4;
};

// CUDA / NCCL runtime failure inside the executor (no reference counterpart:
// the reference never touches a device).
struct DeviceError : std::runtime_error {
  explicit DeviceError(const std::string& what) : std::runtime_error(what) {}
  static constexpr int exit_code = 5;
};

}  // namespace flexrlhf
