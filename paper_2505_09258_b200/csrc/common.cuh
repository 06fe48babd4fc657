// common.cuh -- error plumbing shared by the CUDA sources.
#pragma once

#include <cstdio>

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

namespace lgd {

// Exceptions mirror the reference's classes; the C ABI maps them to codes
// (include/legend_b200.h).
struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    throw cuda_error(std::string("CUDA error in ") + what + " (" + file + ":" +
                     std::to_string(line) + "): " + cudaGetErrorString(e));
  }
}

#define LGD_CUDA(expr) ::lgd::cuda_check((expr), #expr, __FILE__, __LINE__)
#define LGD_LAUNCH_CHECK() ::lgd::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// Checked build (make checked -> liblegend_b200_checked.so): device-side
// bounds and invariant checks on every gather / scatter index of the hot
// kernels; a violation prints its site and traps the context.  (The pool's
// compute-sanitizer is unavailable; tests/test_gpu_checked.py runs the
// small workloads of profiles/sanitize_workload.py through this build.)
#ifdef LGD_CHECKED
#define LGD_DCHECK(cond, what, v)                                                          \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("LGD_CHECKED %s:%d: %s (value %llu)\n", __FILE__, __LINE__, what,            \
             (unsigned long long)(v));                                                     \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define LGD_DCHECK(cond, what, v) \
  do {                            \
  } while (0)
#endif

constexpr uint32_t kNone32 = 0xffffffffu;
constexpr int kWarp = 32;

inline unsigned ceil_div(uint64_t a, uint64_t b) { return static_cast<unsigned>((a + b - 1) / b); }

// Kernel attributes (dynamic shared memory limits) are per device: the
// launch helpers cache what they set per device ordinal.
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  LGD_CUDA(cudaGetDevice(&d));
  return d < kMaxDevices ? d : kMaxDevices - 1;
}

inline int bits_for(uint64_t max_value) {  // bits needed to represent values <= max_value
  int b = 0;
  while (b < 64 && (max_value >> b)) ++b;
  return b < 1 ? 1 : b;
}

// Device buffer with RAII; grows but never shrinks.
template <class T>
struct DevBuf {
  T* ptr = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    n = 0;
  }
  void reserve(size_t count) {
    if (count <= n) return;
    release();
    if (count) LGD_CUDA(cudaMalloc(&ptr, count * sizeof(T)));
    n = count;
  }
  T* get() const { return ptr; }
  size_t bytes() const { return n * sizeof(T); }
  void swap(DevBuf& o) {
    std::swap(ptr, o.ptr);
    std::swap(n, o.n);
  }
};

}  // namespace lgd
