// Handle lifecycle, error reporting and the exception -> status-code edge.
#include "common.cuh"
#include "capi_guard.cuh"

namespace fpi {
void note_launch(fpi_context* h, int count) { h->kernel_launches += count; }
}  // namespace fpi

extern "C" {

int fpi_abi_version(void) { return FPI_ABI_VERSION; }

int fpi_create(fpi_handle* out, int device) {
  if (!out) return FPI_EDOMAIN;
  fpi_context* h = new fpi_context();
  h->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete h;
    *out = nullptr;
    return FPI_ECUDA;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) {
    h->num_sms = prop.multiProcessorCount;
    h->smem_optin = prop.sharedMemPerBlockOptin;
  }
  // Keep freed scratch in the pool: the solve reallocates the same sizes every step.
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = h;
  return FPI_OK;
}

int fpi_destroy(fpi_handle h) {
  if (!h) return FPI_OK;
  if (h->d_spans) cudaFree(h->d_spans);
  if (h->host_scalars) cudaFreeHost(h->host_scalars);
  fpi::fastpi_free(h);
  fpi::comm_free(h);
  for (auto& e : h->copy_ev)
    if (e) cudaEventDestroy(e);
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  delete h;
  return FPI_OK;
}

int fpi_set_stream(fpi_handle h, void* stream) {
  if (!h) return FPI_EDOMAIN;
  h->stream = (cudaStream_t)stream;
  return FPI_OK;
}

const char* fpi_last_error(fpi_handle h) { return h ? h->last_error.c_str() : "null handle"; }

int64_t fpi_kernel_launches(fpi_handle h) { return h ? h->kernel_launches : 0; }

int fpi_get_svd_diag(fpi_handle h, fpi_svd_diag* out) {
  if (!h || !out) return FPI_EDOMAIN;
  *out = h->diag;
  return FPI_OK;
}

int fpi_sparse_core_info(fpi_handle h, int64_t* h_out) {
  if (!h || !h_out) return FPI_EDOMAIN;
  for (int i = 0; i < 4; ++i) h_out[i] = h->sparse_core[i];
  return FPI_OK;
}

}  // extern "C"
