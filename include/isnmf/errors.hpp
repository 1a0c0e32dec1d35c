// isnmf-b200 C++ API — exception taxonomy (same names and hierarchy as the
// reference, proj/include/isnmf/errors.hpp:9-90) and the mapping from the C ABI
// status codes (include/isnmf_b200.h) back onto it.
#pragma once

#include <stdexcept>
#include <string>

#include "../isnmf_b200.h"

namespace isnmf {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DataError : Error {
  using Error::Error;
};
struct NumericError : Error {
  using Error::Error;
};

struct IoError : DataError {
  using DataError::DataError;
};
struct BadMagic : DataError {
  using DataError::DataError;
};
struct TruncatedPayload : DataError {
  using DataError::DataError;
};
struct NonFiniteEntry : DataError {
  using DataError::DataError;
};
struct NegativeEntry : DataError {
  using DataError::DataError;
};
struct UnsupportedFormat : DataError {
  using DataError::DataError;
};
struct TooShort : DataError {
  using DataError::DataError;
};
struct AllSilent : DataError {
  using DataError::DataError;
};
struct EmptyDataset : DataError {
  using DataError::DataError;
};
struct ShapeMismatch : DataError {
  using DataError::DataError;
};

struct NegativeInput : NumericError {
  using NumericError::NumericError;
};
struct ZeroColumn : NumericError {
  using NumericError::NumericError;
};
struct NonPositiveInit : NumericError {
  using NumericError::NumericError;
};
struct InconsistentStats : NumericError {
  using NumericError::NumericError;
};
struct DivergedObjective : NumericError {
  using NumericError::NumericError;
};
struct NumericalFailure : NumericError {
  using NumericError::NumericError;
};

/// Device or driver failure of the B200 engine (no reference equivalent).
struct DeviceError : Error {
  using Error::Error;
};

namespace detail {

/// Rethrows a non-zero C ABI status as the matching reference exception.
inline void check(int rc) {
  if (rc == ISNMF_OK) return;
  const std::string msg = isnmf_last_error();
  switch (rc) {
    case ISNMF_E_SHAPE_MISMATCH: throw ShapeMismatch(msg);
    case ISNMF_E_EMPTY_DATASET: throw EmptyDataset(msg);
    case ISNMF_E_NEGATIVE_INPUT: throw NegativeInput(msg);
    case ISNMF_E_NON_POSITIVE_INIT: throw NonPositiveInit(msg);
    case ISNMF_E_ZERO_COLUMN: throw ZeroColumn(msg);
    case ISNMF_E_INCONSISTENT_STATS: throw InconsistentStats(msg);
    case ISNMF_E_NUMERICAL_FAILURE: throw NumericalFailure(msg);
    case ISNMF_E_DIVERGED_OBJECTIVE: throw DivergedObjective(msg);
    case ISNMF_E_NON_FINITE_ENTRY: throw NonFiniteEntry(msg);
    case ISNMF_E_NEGATIVE_ENTRY: throw NegativeEntry(msg);
    case ISNMF_E_IO: throw IoError(msg);
    case ISNMF_E_UNSUPPORTED_FORMAT: throw UnsupportedFormat(msg);
    case ISNMF_E_TOO_SHORT: throw TooShort(msg);
    case ISNMF_E_ALL_SILENT: throw AllSilent(msg);
    default: throw DeviceError(msg);
  }
}

}  // namespace detail
}  // namespace isnmf
