// Shared device/host helpers for the B200 QR-TEBD engine.
//
// Storage convention (matches the reference ComplexTensor,
// proj/include/qrtebd/tensor.hpp:14-61): row-major, last axis fastest,
// interleaved complex128 (re, im) == double2.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace qt {

using cplx_t = double2;

// Error taxonomy of proj/include/qrtebd/errors.hpp:9-30, carried through the
// engine as C++ exceptions and mapped onto qt_status at the C-ABI boundary.
enum class Err : int { shape = 1, input = 2, numeric = 3, capacity = 4, cuda = 5, nccl = 6, internal = 7 };

struct Error : std::runtime_error {
  Err code;
  Error(Err c, const std::string& w) : std::runtime_error(w), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(Err::cuda, std::string(what) + ": " + cudaGetErrorString(e));
}
#define QT_CUDA(x) ::qt::cuda_check((x), #x)

// every kernel launch of the library is counted (bench "gpu_launches")
inline std::atomic<unsigned long long> g_kernel_launches{0};
#define QT_LAUNCHED()                                        \
  do {                                                       \
    ::qt::cuda_check(cudaGetLastError(), "kernel launch");   \
    ::qt::g_kernel_launches.fetch_add(1, std::memory_order_relaxed); \
  } while (0)

constexpr int kNumSMs = 148;

__host__ __device__ inline long long ceil_div(long long a, long long b) { return (a + b - 1) / b; }

// ---- device complex helpers -------------------------------------------------
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double cabs2(double2 a) { return fma(a.x, a.x, a.y * a.y); }

// gauge phase of reflector column i of a factored QR (R on the upper
// triangle of a, ld lda): R_ii / |R_ii| (1 when R_ii == 0), the phase
// gauge_q applies to column i of Q (proj/src/linalg.cpp:25-36)
__device__ __forceinline__ double2 qr_phase(const double2* __restrict__ a, long long lda, long long i) {
  const double2 d = a[i * lda + i];
  const double ad = hypot(d.x, d.y);
  return ad == 0.0 ? make_double2(1.0, 0.0) : make_double2(d.x / ad, d.y / ad);
}

// sign flip without touching the FP64 pipe (integer xor on the high word)
__device__ __forceinline__ double dneg(double x) {
  return __hiloint2double(__double2hiint(x) ^ 0x80000000, __double2loint(x));
}

}  // namespace qt
