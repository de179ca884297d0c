// Error categories of the reference (proj/include/fj/error.hpp:9-33), which
// "map 1:1 onto CLI exit codes" (error.hpp:8). The integer codes live in the
// reference's absent tools/fj_main.cpp, so they are pinned here and exported
// through the C-ABI as FJG_E_* (include/fjg.h).
#pragma once

#include <stdexcept>
#include <string>

namespace fj {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
  virtual int code() const { return 5; }
};
struct IoError : Error {
  using Error::Error;
  int code() const override { return 1; }
};
struct ParseError : Error {
  using Error::Error;
  int code() const override { return 2; }
};
struct ValidationError : Error {
  using Error::Error;
  int code() const override { return 3; }
};
struct ResourceError : Error {
  using Error::Error;
  int code() const override { return 4; }
};
// Internal invariant violations (plan/schema mismatches a validated plan makes
// impossible, CUDA launch failures).
struct EngineError : Error {
  using Error::Error;
  int code() const override { return 5; }
};

}  // namespace fj
