// meshforge::Error for the B200 bake library. Source-compatible with the
// reference's proj/include/meshforge/core/error.h:8-43: same enum order (the
// C ABI returns 1 + code), same "<CodeName>: <message>" what() text and the
// same validation split (CLI exit code 2 vs 3).
#pragma once

#include <stdexcept>
#include <string>

namespace meshforge {

enum class ErrorCode {
  EmptyMesh,
  InvalidGeometry,
  OutOfBounds,
  EmptySurface,
  AllHidden,
  ChartFailure,
  PackOverflow,
  AtlasOverlap,
  ShapeMismatch,
  NothingToInpaint,
  ExportMismatch,
  InvalidConfig,
  IoError,
};

inline const char* errorCodeName(ErrorCode code) {
  static const char* const kNames[] = {"EmptyMesh",      "InvalidGeometry", "OutOfBounds",  "EmptySurface",
                                       "AllHidden",      "ChartFailure",    "PackOverflow", "AtlasOverlap",
                                       "ShapeMismatch",  "NothingToInpaint", "ExportMismatch", "InvalidConfig",
                                       "IoError"};
  const int i = static_cast<int>(code);
  return i >= 0 && i < 13 ? kNames[i] : "Unknown";
}

class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, const std::string& message)
      : std::runtime_error(std::string(errorCodeName(code)) + ": " + message), code_(code) {}
  ErrorCode code() const { return code_; }
  // Bad inputs / configuration (exit code 2) vs pipeline failures (exit code 3).
  bool isValidation() const {
    switch (code_) {
      case ErrorCode::EmptyMesh:
      case ErrorCode::InvalidGeometry:
      case ErrorCode::OutOfBounds:
      case ErrorCode::InvalidConfig:
      case ErrorCode::ShapeMismatch:
      case ErrorCode::ExportMismatch:
        return true;
      default:
        return false;
    }
  }

 private:
  ErrorCode code_;
};

}  // namespace meshforge
