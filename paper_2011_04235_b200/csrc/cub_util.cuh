// Thin wrappers over CUB device-wide primitives with a grow-only temp buffer.
#pragma once
#include <cub/cub.cuh>
#include "common.cuh"

namespace fpi {

struct CubTemp {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  explicit CubTemp(cudaStream_t st) : s(st) {}
  void* need(size_t b) {
    if (b > bytes) {
      if (p) cudaFreeAsync(p, s);
      bytes = b + (b >> 2) + 4096;
      FPI_CUDA(cudaMallocAsync(&p, bytes, s));
    }
    return p;
  }
  ~CubTemp() {
    if (p) cudaFreeAsync(p, s);
  }
};

// Order-preserving selection of [in, in + n) by predicate; count left on device.
template <typename InIt, typename T, typename Pred>
void select_if(CubTemp& tmp, InIt in, T* out, int* d_count, int64_t n, Pred pred, cudaStream_t s) {
  size_t b = 0;
  FPI_CUDA(cub::DeviceSelect::If(nullptr, b, in, out, d_count, (int)n, pred, s));
  FPI_CUDA(cub::DeviceSelect::If(tmp.need(b), b, in, out, d_count, (int)n, pred, s));
}

// Stable key-value radix sort.
template <typename K, typename V>
void sort_pairs(CubTemp& tmp, const K* kin, K* kout, const V* vin, V* vout, int64_t n, bool descending,
                int begin_bit, int end_bit, cudaStream_t s) {
  size_t b = 0;
  if (descending) {
    FPI_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, b, kin, kout, vin, vout, (int)n, begin_bit, end_bit, s));
    FPI_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp.need(b), b, kin, kout, vin, vout, (int)n, begin_bit, end_bit, s));
  } else {
    FPI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, kin, kout, vin, vout, (int)n, begin_bit, end_bit, s));
    FPI_CUDA(cub::DeviceRadixSort::SortPairs(tmp.need(b), b, kin, kout, vin, vout, (int)n, begin_bit, end_bit, s));
  }
}

template <typename InIt, typename OutIt>
void exclusive_sum(CubTemp& tmp, InIt in, OutIt out, int64_t n, cudaStream_t s) {
  size_t b = 0;
  FPI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b, in, out, (int)n, s));
  FPI_CUDA(cub::DeviceScan::ExclusiveSum(tmp.need(b), b, in, out, (int)n, s));
}

// Three-way partition: first / second parts in input order, the rest through `rest`; the two counts
// land on the device.
template <typename InIt, typename T, typename RestIt, typename P1, typename P2>
void three_way_partition(CubTemp& tmp, InIt in, T* first, T* second, RestIt rest, int* d_counts, int64_t n, P1 p1,
                         P2 p2, cudaStream_t s) {
  size_t b = 0;
  FPI_CUDA(cub::DevicePartition::If(nullptr, b, in, first, second, rest, d_counts, (int)n, p1, p2, s));
  FPI_CUDA(cub::DevicePartition::If(tmp.need(b), b, in, first, second, rest, d_counts, (int)n, p1, p2, s));
}

// Exclusive scan with a custom associative operator.
template <typename InIt, typename OutIt, typename Op, typename T>
void exclusive_scan(CubTemp& tmp, InIt in, OutIt out, Op op, T init, int64_t n, cudaStream_t s) {
  size_t b = 0;
  FPI_CUDA(cub::DeviceScan::ExclusiveScan(nullptr, b, in, out, op, init, (int)n, s));
  FPI_CUDA(cub::DeviceScan::ExclusiveScan(tmp.need(b), b, in, out, op, init, (int)n, s));
}

template <typename InIt, typename OutIt>
void inclusive_sum(CubTemp& tmp, InIt in, OutIt out, int64_t n, cudaStream_t s) {
  size_t b = 0;
  FPI_CUDA(cub::DeviceScan::InclusiveSum(nullptr, b, in, out, (int)n, s));
  FPI_CUDA(cub::DeviceScan::InclusiveSum(tmp.need(b), b, in, out, (int)n, s));
}

inline int bits_for(uint64_t maxval) {
  int b = 1;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b;
}

}  // namespace fpi
