// rr_internal.h -- host-side helpers shared by the library's translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <new>

namespace rr {

// owning device buffer (throws std::bad_alloc on allocation failure; mapped to RR_E_OOM at the ABI)
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), cap(o.cap) { o.p = nullptr; o.n = 0; o.cap = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; cap = o.cap; o.p = nullptr; o.n = 0; o.cap = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count == 0) return;
    if (cudaMalloc(&p, count * sizeof(T)) != cudaSuccess) {
      p = nullptr;
      n = 0;
      throw std::bad_alloc();
    }
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cap = 0;
  }
  void upload(const T* h, size_t count) {
    alloc(count);
    if (count) cudaMemcpy(p, h, count * sizeof(T), cudaMemcpyHostToDevice);
  }
  // per-frame data (set_edit): keep the allocation when it is large enough (no cudaFree / cudaMalloc and their
  // device-wide synchronisation); the caller has waited for the renders that read the old contents
  void upload_reuse(const T* h, size_t count) {
    if (count > cap || !p) {
      alloc(count);
      cap = count;
    }
    n = count;
    if (count) cudaMemcpy(p, h, count * sizeof(T), cudaMemcpyHostToDevice);
  }
  size_t cap = 0;
};

int build_lbvh(const float4* d_tris, int n, float4* d_nodes, float4* d_ltris, float4* d_lxf, int node_base,
               int leaf_base, cudaStream_t st, const unsigned long long* h_keys = nullptr);

}  // namespace rr
