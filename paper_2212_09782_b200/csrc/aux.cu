// Engine arena and the HBM-bound helper kernels (K7 permutes, norms,
// copies).  The permutes replace the reference's ComplexTensor::transpose
// copies (proj/src/tensor.cpp:100-147) where the layout cannot be folded
// into a GEMM store.
#include <cstdlib>

#include "engine.cuh"

namespace qt {

// ---------------------------------------------------------------- Engine
void Engine::init(int dev, cudaStream_t st) {
  device = dev;
  QT_CUDA(cudaSetDevice(dev));
  int sms = 0;
  QT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  num_sms = sms;
  // the context's own stream carries the latency-bound critical path (QR
  // panels); it gets the highest priority so that CTAs of the side-stream
  // GEMMs never hold SMs a pending panel cluster is waiting for
  int prio_least = 0, prio_greatest = 0;
  QT_CUDA(cudaDeviceGetStreamPriorityRange(&prio_least, &prio_greatest));
  static const bool no_prio = std::getenv("QT_NO_STREAM_PRIORITY") != nullptr;
  if (st) {
    stream = st;
    own_stream = false;
  } else {
    QT_CUDA(cudaStreamCreateWithPriority(&stream, cudaStreamNonBlocking, no_prio ? prio_least : prio_greatest));
    own_stream = true;
  }
  QT_CUDA(cudaMalloc(&dscal, SC_COUNT * sizeof(double)));
  QT_CUDA(cudaMemset(dscal, 0, SC_COUNT * sizeof(double)));
  QT_CUDA(cudaMallocHost(&hscal, SC_COUNT * sizeof(double)));
  QT_CUDA(cudaMalloc(&barrier, 64 * sizeof(unsigned)));
  QT_CUDA(cudaMemset(barrier, 0, 64 * sizeof(unsigned)));
  QT_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
  QT_CUDA(cudaStreamCreateWithFlags(&side2, cudaStreamNonBlocking));
  QT_CUDA(cudaStreamCreateWithPriority(&side3, cudaStreamNonBlocking, no_prio ? prio_least : prio_greatest));
  QT_CUDA(cudaStreamCreateWithFlags(&side4, cudaStreamNonBlocking));
  QT_CUDA(cudaStreamCreateWithFlags(&side5, cudaStreamNonBlocking));
}

cudaEvent_t Engine::event(size_t i) {
  while (events.size() <= i) {
    cudaEvent_t ev;
    QT_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    events.push_back(ev);
  }
  return events[i];
}

void Engine::destroy() {
  if (stream) cudaStreamSynchronize(stream);
  for (void*& p : slot_ptr)
    if (p) {
      cudaFree(p);
      p = nullptr;
    }
  if (dscal) cudaFree(dscal);
  if (hscal) cudaFreeHost(hscal);
  if (barrier) cudaFree(barrier);
  if (side) {
    cudaStreamSynchronize(side);
    cudaStreamDestroy(side);
  }
  side = nullptr;
  if (side2) {
    cudaStreamSynchronize(side2);
    cudaStreamDestroy(side2);
  }
  side2 = nullptr;
  if (side3) {
    cudaStreamSynchronize(side3);
    cudaStreamDestroy(side3);
  }
  side3 = nullptr;
  if (side4) {
    cudaStreamSynchronize(side4);
    cudaStreamDestroy(side4);
  }
  side4 = nullptr;
  if (side5) {
    cudaStreamSynchronize(side5);
    cudaStreamDestroy(side5);
  }
  side5 = nullptr;
  for (cudaEvent_t ev : events) cudaEventDestroy(ev);
  events.clear();
  dscal = nullptr;
  hscal = nullptr;
  barrier = nullptr;
  if (own_stream && stream) cudaStreamDestroy(stream);
  stream = nullptr;
}

void* Engine::raw(int slot, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (slot_bytes[slot] < bytes) {
    if (slot_ptr[slot]) {
      QT_CUDA(cudaStreamSynchronize(stream));
      QT_CUDA(cudaFree(slot_ptr[slot]));
      slot_ptr[slot] = nullptr;
      slot_bytes[slot] = 0;
      ++arena_gen;
    }
    // round up to limit regrowth churn
    size_t want = bytes + bytes / 8;
    want = (want + 4095) & ~size_t(4095);
    cudaError_t err = cudaMalloc(&slot_ptr[slot], want);
    if (err != cudaSuccess) {
      cudaGetLastError();
      throw Error(Err::capacity, "device workspace allocation failed (" + std::to_string(want) + " bytes)");
    }
    slot_bytes[slot] = want;
  }
  return slot_ptr[slot];
}

GemmScratch Engine::gemm_scratch() {
  GemmScratch s;
  // split-K partials: enough for every split configuration the dispatcher
  // picks on the hot-path shapes; it falls back to fewer splits otherwise
  const size_t part = size_t(1) << 24;  // 16M complex = 256 MB (a 2-way split of 5120 x 1024 outputs)
  s.partial = cbuf(S_GEMM_PART, part);
  s.partial_elems = part;
  const size_t ts = size_t(1) << 20;
  s.tile_sums = dbuf(S_TILE_SUMS, ts);
  s.tile_sums_elems = ts;
  return s;
}

GemmScratch Engine::gemm_scratch2() {
  GemmScratch s;
  const size_t part = size_t(1) << 22;
  s.partial = cbuf(S_GEMM_PART2, part);
  s.partial_elems = part;
  const size_t ts = size_t(1) << 16;
  s.tile_sums = dbuf(S_TILE_SUMS2, ts);
  s.tile_sums_elems = ts;
  return s;
}

GemmScratch Engine::gemm_scratch3() {
  GemmScratch s;
  const size_t part = size_t(1) << 21;
  s.partial = cbuf(S_GEMM_PART3, part);
  s.partial_elems = part;
  const size_t ts = size_t(1) << 16;
  s.tile_sums = dbuf(S_TILE_SUMS3, ts);
  s.tile_sums_elems = ts;
  return s;
}

GemmScratch Engine::gemm_scratch4() {
  GemmScratch s;
  const size_t part = size_t(1) << 21;
  s.partial = cbuf(S_GEMM_PART4, part);
  s.partial_elems = part;
  const size_t ts = size_t(1) << 16;
  s.tile_sums = dbuf(S_TILE_SUMS4, ts);
  s.tile_sums_elems = ts;
  return s;
}

// ---------------------------------------------------------------- kernels
namespace {

struct Perm4 {
  long long out_shape[4];
  long long in_stride_for_out[4];  // input stride of output axis k
  int rank;
};

__global__ void permute_kernel(const double2* __restrict__ in, Perm4 p, long long total, bool conj,
                               double scale, const double* dscale, double2* __restrict__ out) {
  double s = scale;
  if (dscale) s *= *dscale;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long rem = e, src = 0;
    for (int k = p.rank - 1; k >= 0; --k) {
      const long long idx = rem % p.out_shape[k];
      rem /= p.out_shape[k];
      src += idx * p.in_stride_for_out[k];
    }
    double2 v = in[src];
    if (conj) v.y = -v.y;
    v.x *= s;
    v.y *= s;
    out[e] = v;
  }
}

// (batch, R, C) -> (batch, C, R) tiled transpose through shared memory, for
// the large axis swaps (Q' -> B~n) where the gather above would be uncoalesced
__global__ void transpose_tiled_kernel(const double2* __restrict__ in, long long R, long long Cc, bool conj,
                                       double2* __restrict__ out) {
  __shared__ double2 tile[32][33];
  const long long b = blockIdx.z;
  const long long r0 = static_cast<long long>(blockIdx.y) * 32, c0 = static_cast<long long>(blockIdx.x) * 32;
  const double2* src = in + b * R * Cc;
  double2* dst = out + b * R * Cc;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const long long r = r0 + i, c = c0 + threadIdx.x;
    if (r < R && c < Cc) tile[i][threadIdx.x] = src[r * Cc + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const long long c = c0 + i, r = r0 + threadIdx.x;
    if (r < R && c < Cc) {
      double2 v = tile[threadIdx.x][i];
      if (conj) v.y = -v.y;
      dst[c * R + r] = v;
    }
  }
}

constexpr int kNormBlocks = 296;

__global__ void norm2_partial_kernel(const double2* __restrict__ x, long long rows, long long cols, long long ld,
                                     double* part) {
  // block b sums rows b, b + gridDim.x, ... (no per-element index division;
  // two accumulation chains); fixed assignment and order -> deterministic
  __shared__ double sh[256];
  double s = 0.0, s1 = 0.0;
  for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
    const double2* row = x + r * ld;
    long long c = threadIdx.x;
    for (; c + blockDim.x < cols; c += 2 * blockDim.x) {
      const double2 v = row[c], w = row[c + blockDim.x];
      s = fma(v.x, v.x, fma(v.y, v.y, s));
      s1 = fma(w.x, w.x, fma(w.y, w.y, s1));
    }
    if (c < cols) {
      const double2 v = row[c];
      s = fma(v.x, v.x, fma(v.y, v.y, s));
    }
  }
  s += s1;
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void norm2_final_kernel(const double* __restrict__ part, int n, double* out) {
  __shared__ double sh[512];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

__global__ void copy2d_kernel(const double2* __restrict__ src, long long lds, double2* __restrict__ dst,
                              long long ldd, long long rows, long long cols) {
  const long long total = rows * cols;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = e / cols, c = e % cols;
    dst[r * ldd + c] = src[r * lds + c];
  }
}

__global__ void identity_kernel(double2* q, long long rows, long long cols, long long ld) {
  const long long total = rows * cols;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = e / cols, c = e % cols;
    q[r * ld + c] = make_double2(r == c ? 1.0 : 0.0, 0.0);
  }
}

__global__ void finite_kernel(const double2* __restrict__ x, long long n, int* flag) {
  bool bad = false;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double2 v = x[e];
    bad |= !isfinite(v.x) || !isfinite(v.y);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

__global__ void finite2d_kernel(const double2* __restrict__ x, long long rows, long long cols, long long ld,
                                int* flag) {
  bool bad = false;
  const long long n = rows * cols;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double2 v = x[(e / cols) * ld + e % cols];
    bad |= !isfinite(v.x) || !isfinite(v.y);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

int grid_for(long long total, int per = 256) {
  const long long b = ceil_div(total, per);
  return static_cast<int>(b < 16LL * kNumSMs ? (b > 0 ? b : 1) : 16LL * kNumSMs);
}

}  // namespace

void permute(Engine& e, const double2* in, int rank, const long long* shape, const int* perm, bool conj,
             double2* out, double scale, const double* dscale, cudaStream_t st) {
  if (!st) st = e.stream;
  if (rank < 1 || rank > 4) throw Error(Err::shape, "permute: rank must be 1..4");
  long long in_strides[4];
  long long s = 1;
  for (int k = rank - 1; k >= 0; --k) {
    in_strides[k] = s;
    s *= shape[k];
  }
  const long long total = s;
  if (total == 0) return;
  // fast path: swap of the last two axes with everything else leading
  bool last_two_swap = rank >= 2 && perm[rank - 1] == rank - 2 && perm[rank - 2] == rank - 1 && dscale == nullptr &&
                       scale == 1.0;
  for (int k = 0; k < rank - 2 && last_two_swap; ++k) last_two_swap = perm[k] == k;
  if (last_two_swap) {
    const long long R = shape[rank - 2], C = shape[rank - 1];
    const long long batch = total / (R * C);
    dim3 grid(static_cast<unsigned>(ceil_div(C, 32)), static_cast<unsigned>(ceil_div(R, 32)),
              static_cast<unsigned>(batch));
    transpose_tiled_kernel<<<grid, dim3(32, 8), 0, st>>>(in, R, C, conj, out);
    QT_LAUNCHED();
    return;
  }
  Perm4 p{};
  p.rank = rank;
  for (int k = 0; k < rank; ++k) {
    p.out_shape[k] = shape[perm[k]];
    p.in_stride_for_out[k] = in_strides[perm[k]];
  }
  permute_kernel<<<grid_for(total), 256, 0, st>>>(in, p, total, conj, scale, dscale, out);
  QT_LAUNCHED();
}

void norm2(Engine& e, const double2* x, long long rows, long long cols, long long ld, double* out) {
  double* part = e.dbuf(S_NORM_PART, kNormBlocks);
  norm2_partial_kernel<<<kNormBlocks, 256, 0, e.stream>>>(x, rows, cols, ld, part);
  QT_LAUNCHED();
  norm2_final_kernel<<<1, 512, 0, e.stream>>>(part, kNormBlocks, out);
  QT_LAUNCHED();
}

void copy2d(Engine& e, const double2* src, long long lds, double2* dst, long long ldd, long long rows,
            long long cols, cudaStream_t st) {
  if (rows * cols == 0) return;
  copy2d_kernel<<<grid_for(rows * cols), 256, 0, st ? st : e.stream>>>(src, lds, dst, ldd, rows, cols);
  QT_LAUNCHED();
}

void set_identity(Engine& e, double2* q, long long rows, long long cols, long long ld, cudaStream_t st) {
  if (rows * cols == 0) return;
  identity_kernel<<<grid_for(rows * cols), 256, 0, st ? st : e.stream>>>(q, rows, cols, ld);
  QT_LAUNCHED();
}

void check_finite(Engine& e, const double2* x, long long n, int* dflag) {
  if (n == 0) return;
  finite_kernel<<<grid_for(n), 256, 0, e.stream>>>(x, n, dflag);
  QT_LAUNCHED();
}

void check_finite_2d(Engine& e, const double2* x, long long rows, long long cols, long long ld, int* dflag,
                     cudaStream_t st) {
  if (rows * cols == 0) return;
  finite2d_kernel<<<grid_for(rows * cols), 256, 0, st ? st : e.stream>>>(x, rows, cols, ld, dflag);
  QT_LAUNCHED();
}

}  // namespace qt
