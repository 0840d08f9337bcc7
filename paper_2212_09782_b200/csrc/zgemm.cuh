// Complex128 GEMM on the sm_100a FP64 tensor pipe (DMMA), TMA-staged.
//
// Replaces every Eigen complex product on the hot path
// (proj/src/tensor.cpp:227-231, proj/src/gates.cpp:157-179, :298, :300,
// :408-409, :422-423, :441-442, :480-484) with one kernel family:
//
//   C[b] = alpha * op(A[b]) * op(B[b]) + beta * C[b]        (mode STORE)
//   sum |C[b] - alpha * op(A[b]) * op(B[b])|^2               (mode RESID)
//
// op in {N, H}; H = conjugate transpose of the stored row-major matrix.
// The output row r is stored at (r % rsplit) * ldc + (r / rsplit) * ldc_hi so
// tensor permutations of the reference (e.g. gates.cpp:171, :189) are folded
// into the store instead of running as separate copies.
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "common.cuh"

namespace qt {

enum class Op : int { N = 0, H = 1 };
enum class GemmMode : int { store = 0, resid = 1 };

struct GemmDesc {
  long long M = 0, N = 0, K = 0;
  int batch = 1;
  Op opA = Op::N, opB = Op::N;
  const double2* A = nullptr;
  long long lda = 0, strideA = 0;  // strides in complex elements
  const double2* B = nullptr;
  long long ldb = 0, strideB = 0;
  double2* C = nullptr;
  long long ldc = 0, strideC = 0;
  long long rsplit = 0, ldc_hi = 0;  // rsplit == 0: plain row-major store
  double alpha = 1.0, beta = 0.0;
  GemmMode mode = GemmMode::store;
  int splits = 0;  // split-K factor; 0 = choose automatically
};

// Scratch owned by the caller (the engine arena): split-K partials and the
// per-tile partial sums of RESID mode.
struct GemmScratch {
  double2* partial = nullptr;
  size_t partial_elems = 0;
  double* tile_sums = nullptr;
  size_t tile_sums_elems = 0;
};

// Launches the GEMM on `stream`. In RESID mode the squared residual is
// reduced deterministically into *resid_out (device pointer, one double).
void zgemm(const GemmDesc& d, const GemmScratch& s, cudaStream_t stream,
           double* resid_out = nullptr);

// number of library kernels launched since process start (bench bookkeeping)
unsigned long long zgemm_launch_count();

// GEMM launch profiler: CUDA events around every DMMA GEMM launch between
// begin and end; end synchronizes and returns the summed algorithmic flops
// (8 per complex MAC) and device time.
struct GemmProfile {
  double flops = 0.0, ms = 0.0;
  unsigned long long launches = 0;
};
void gemm_profile_begin(double min_flops = 0.0);
GemmProfile gemm_profile_end();
bool gemm_profile_active();
// GEMM launches captured into a CUDA graph while profiling is active record
// their event pairs here; the graph owner takes them after capture and
// accumulates their elapsed times after every replay.
struct GemmProfRec {
  cudaEvent_t e0, e1;
  double flops;
};
std::vector<GemmProfRec> gemm_profile_take_captured();
void gemm_profile_add_replay(const std::vector<GemmProfRec>& recs);

}  // namespace qt
