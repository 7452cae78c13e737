// Shared C-ABI plumbing: thread-local error message and the exception ->
// return-code guard used by every extern "C" entry point.
#pragma once

#include <exception>
#include <string>

#include "common.cuh"
#include "emoe.h"

namespace emoe {

std::string& last_error_slot();

template <typename F>
int guard(F&& f) {
  try {
    f();
    return EMOE_OK;
  } catch (const ValidationError& e) {
    last_error_slot() = e.what();
    return EMOE_ERR_VALIDATION;
  } catch (const InvariantError& e) {
    last_error_slot() = e.what();
    return EMOE_ERR_INVARIANT;
  } catch (const std::exception& e) {
    last_error_slot() = e.what();
    return EMOE_ERR_RUNTIME;
  }
}

// RAII device buffer for the host-pointer entry points
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  explicit DevBuf(size_t count) : n(count) {
    if (count) EMOE_CUDA(cudaMalloc(&p, count * sizeof(T)));
  }
  DevBuf(const T* host, size_t count) : DevBuf(count) {
    if (count) EMOE_CUDA(cudaMemcpy(p, host, count * sizeof(T), cudaMemcpyHostToDevice));
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void to_host(T* host) const {
    if (n) EMOE_CUDA(cudaMemcpy(host, p, n * sizeof(T), cudaMemcpyDeviceToHost));
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

}  // namespace emoe
