// CUDA-event timing of kernel classes (enabled per handle by fpi_timing_enable).
#pragma once
#include "common.cuh"

namespace fpi {
struct KTimer {
  fpi_context* h;
  const char* name;
  double flops, bytes;
  bool active = false;
  void* ev_a = nullptr;
  KTimer(fpi_context* h, const char* name, double flops, double bytes);
  ~KTimer();
};
// Wall-clock trace points (env FPI_TRACE=1): synchronises the stream and prints the time since
// the previous point.  Diagnostic only; a no-op otherwise.
void trace_point(fpi_context* h, const char* label);
}  // namespace fpi
