// Converts exceptions thrown inside the core into C-ABI status codes.
#pragma once
#include "common.cuh"

#define FPI_API_BEGIN(h)                                  \
  if (!(h)) return FPI_EDOMAIN;                           \
  try {                                                   \
    cudaSetDevice((h)->device);

#define FPI_API_END(h)                                    \
  }                                                       \
  catch (const ::fpi::Error& e) {                         \
    (h)->last_error = e.what();                           \
    return e.code;                                        \
  }                                                       \
  catch (const std::exception& e) {                       \
    (h)->last_error = e.what();                           \
    return FPI_ECUDA;                                     \
  }                                                       \
  return FPI_OK;
