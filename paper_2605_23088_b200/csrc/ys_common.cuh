// ys_common.cuh — shared host/device definitions of the B200 YASPS hot path.
//
// Everything here is plumbing: error mapping onto the reference's exception
// classes (core.hpp:33-71), RAII device buffers, and the POD structs that the
// kernels receive by value.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/yasps_b200.h"

namespace ys {

struct Error : std::runtime_error {
  int cls;
  Error(int c, const std::string& m) : std::runtime_error(m), cls(c) {}
};

[[noreturn]] inline void fail(int cls, const std::string& m) { throw Error(cls, m); }

#define YS_CUDA(x)                                                                       \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess)                                                               \
      ::ys::fail(YS_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));          \
  } while (0)

#define YS_LAUNCH_CHECK() YS_CUDA(cudaGetLastError())

// Bytes currently allocated through DevBuf (ys_device_bytes).
int64_t& device_bytes_counter();

// Growable device buffer: capacity only grows, so the per-Newton-iteration
// dynamic rebuilds reuse their storage (no allocator on the hot path).
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  size_t cap = 0;

  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), cap(o.cap) { o.p = nullptr; o.n = o.cap = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; cap = o.cap;
      o.p = nullptr; o.n = o.cap = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }

  void release() {
    if (p) {
      cudaFree(p);
      device_bytes_counter() -= int64_t(cap * sizeof(T));
    }
    p = nullptr;
    n = cap = 0;
  }
  // Resize without preserving contents.
  void resize(size_t m) {
    if (m > cap) {
      release();
      size_t c = m + m / 4 + 16;
      void* q = nullptr;
      YS_CUDA(cudaMalloc(&q, c * sizeof(T)));
      p = static_cast<T*>(q);
      cap = c;
      device_bytes_counter() += int64_t(cap * sizeof(T));
    }
    n = m;
  }
  void upload(const T* h, size_t m, cudaStream_t s) {
    resize(m);
    if (m) YS_CUDA(cudaMemcpyAsync(p, h, m * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void upload(const std::vector<T>& h, cudaStream_t s) { upload(h.data(), h.size(), s); }
  void download(T* h, size_t m, cudaStream_t s) const {
    if (m) YS_CUDA(cudaMemcpyAsync(h, p, m * sizeof(T), cudaMemcpyDeviceToHost, s));
  }
  std::vector<T> to_host(cudaStream_t s) const {
    std::vector<T> h(n);
    download(h.data(), n, s);
    YS_CUDA(cudaStreamSynchronize(s));
    return h;
  }
  void zero(cudaStream_t s) {
    if (n) YS_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  size_t size() const { return n; }
  T* data() { return p; }
  const T* data() const { return p; }
};

// ---------------------------------------------------------------------------
// Device-side POD views

// SlotEntry (index_gen.hpp:61-65): idx is the 1-based placement index
// (gstart + 1, 0 = padded slot), len the block length, col the column offset
// in the uncompressed local gradient/Hessian.
struct DSlot {
  int32_t idx;
  int16_t len;
  int16_t col;
};

// One point domain (a UNION child or an inertia host).
struct DomainDev {
  int32_t kind;    // YS_POINTS_*
  int32_t startA;  // DoF start of target_a (free position / affine matrix)
  int32_t startB;  // DoF start of target_b (affine translation)
  int32_t pad;
  int64_t n;
  const int32_t* v2b;   // affine: vertex -> body
  const double* rest;   // affine: rest positions n x 3
  const double* fixed;  // fixed: positions n x 3
};

constexpr int kMaxUnionChildren = 4096;

struct UnionDev {
  int32_t nchild;
  int32_t kappa_u;  // max slots over the active branches
  int32_t width;    // max width over the active branches
  int32_t pad;
  const DomainDev* child;  // device array [nchild]
  const int64_t* offsets;  // device array [nchild] prefix offsets
};

// Block-row view of the DoF layout: one entry per target instance (the
// DiagAccumulator granularity, assembly.hpp:63-71).
struct BlocksDev {
  int64_t nb;
  const int32_t* start;  // first DoF
  const int32_t* rc;     // block length
  const int64_t* voff;   // offset of the rc x rc diag / inverse block
  const int32_t* dof2block;
};

}  // namespace ys
