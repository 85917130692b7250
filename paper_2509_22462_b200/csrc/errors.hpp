// Error taxonomy of the boundary.  Mirrors the reference's exception classes
// (reference include/gbopt/errors.hpp:10-71) so the C ABI can map each to the
// same gbopt_status code (reference src/capi.cpp:37-59); DeviceError is new
// and maps to GBOPT_ERR_DEVICE.
#pragma once

#include <stdexcept>
#include <string>

namespace gbb {

class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class StructuralError : public Error {
 public:
  using Error::Error;
};
class NumericError : public Error {
 public:
  using Error::Error;
};
class IoError : public Error {
 public:
  using Error::Error;
};
class FormatError : public IoError {
 public:
  using IoError::IoError;
};
class DimensionError : public IoError {
 public:
  using IoError::IoError;
};
class TruncatedError : public IoError {
 public:
  using IoError::IoError;
};
class SingularError : public Error {
 public:
  using Error::Error;
};
class RangeError : public Error {
 public:
  using Error::Error;
};
class ContractError : public StructuralError {
 public:
  using StructuralError::StructuralError;
};
// CUDA unavailable or a CUDA call failed.
class DeviceError : public Error {
 public:
  using Error::Error;
};

}  // namespace gbb
