// Cross-rank reductions of a sharded solve: one communicator per
// handle, stream-ordered.  Native NCCL (NVLink / NVSwitch) when the handle was given an NCCL
// unique id; a host callback otherwise (torch.distributed over gloo, the functional test of the
// exchange pattern with several ranks on one GPU).
#pragma once
#include <vector>

#include "common.cuh"

namespace fpi {

struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() = default;
  // in place: buf <- sum over ranks (op 0) or max (op 1)
  virtual void allreduce(double* buf, int64_t n, int op, cudaStream_t s) = 0;
  // recv (world * n doubles) <- concatenation of every rank's send (n doubles)
  virtual void allgather(const double* send, double* recv, int64_t n, cudaStream_t s) = 0;
  // recv (n doubles, on root) <- sum over ranks of send; recv is ignored on other ranks
  virtual void reduce(const double* send, double* recv, int64_t n, int root, cudaStream_t s) = 0;
  virtual void group_begin() {}
  virtual void group_end() {}
};

// world size of the handle's communicator (1 without one)
inline int world_of(const fpi_context* h) { return h->comm ? h->comm->world : 1; }

}  // namespace fpi
