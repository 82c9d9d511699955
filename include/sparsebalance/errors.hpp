// sparsebalance-b200 host layer: error convention.
//
// Mirrors the reference convention (proj/core/include/sparsebalance/errors.hpp:11-17,
// commands.cpp:325-336): ConfigError = invalid caller input (exit/return code 1);
// any other std::runtime_error = runtime / CUDA failure (code 2). The kernel C-ABI
// (include/sb_kernels.h) returns the same codes and the C++ wrappers convert back.
#pragma once

#include <stdexcept>
#include <string>

// Exported from libsparsebalance_b200.so (the library builds with -fvisibility=hidden): the
// C++ API is part of the drop-in boundary.
#pragma GCC visibility push(default)
namespace sparsebalance {

class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& what) : std::runtime_error(what) {}
};

}  // namespace sparsebalance
#pragma GCC visibility pop
