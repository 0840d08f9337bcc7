// Complex128 GEMM for sm_100a: TMA producer warp + mbarrier ring feeding
// register-fragment DMMA consumers (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4).
//
// Why not tcgen05: the 5th-gen tensor core has no kind::f64 (ptxas rejects
// it); the FP64 tensor path on sm_100a is the
// warp-synchronous DMMA, fed here from 128B-swizzled TMA tiles.
//
// Shared-memory tile layout.  Every operand tile is a set of "chunk blocks":
// 8 consecutive complex values along the operand's contiguous (stored) axis
// form one 128-byte row; a block stacks those rows along the strided axis.
// TMA writes each block with SWIZZLE_128B, i.e. the 16-byte slot of element
// e in row r lands at slot (e ^ r) & 7.  Fragment lanes use the row
// permutation rho(g) = (g >> 1) | ((g & 1) << 2), which makes every
// quarter-warp LDS.128 hit 8 distinct slots for all four op(A)/op(B)
// combinations ("K-GEMM").
//
// Complex arithmetic: 3M (Gauss) -- per 8x8x4 complex step three real DMMAs,
// P1 = Re a Re b, P2 = Im a Im b, P3 = (Re a + Im a)(Re b + Im b), and
// Re c = P1 - P2, Im c = P3 - P1 - P2 at the epilogue, instead of four.  The
// FP64 tensor pipe is the bound: 1.17-1.24x on the north-star GEMMs.  Error
// stays normwise ~u |A||B| (measured max |dC| / (max|A| max|B| K) 5.7e-18
// vs 6.4e-18 for the 4-product form, tools/gemm_check.py).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdio>
#include <mutex>
#include <vector>

#include "zgemm.cuh"

namespace qt {

namespace {

// launch profiler: CUDA events around every DMMA GEMM launch (bench roofline)
struct Prof {
  bool active = false;
  double min_flops = 0.0;  // only launches at least this large are bracketed
  using Rec = GemmProfRec;
  std::vector<Rec> recs;
  std::vector<Rec> captured;  // recorded while a stream was being captured into a graph
  GemmProfile replayed;       // accumulated from graph replays
  std::vector<cudaEvent_t> pool;
  size_t next = 0;
  cudaEvent_t event() {
    if (next == pool.size()) {
      cudaEvent_t e;
      QT_CUDA(cudaEventCreate(&e));
      pool.push_back(e);
    }
    return pool[next++];
  }
} g_prof;

// ---------------------------------------------------------------- PTX glue
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n"
      "DONE:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x,
                                            int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
// 4-D box over chunked operands: {16 doubles, rows, chunks, batch}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y, int z,
                                            int w) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(w), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ void consumer_bar(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

struct KParams {
  long long M, N, K;
  int splits, kt_per_split;
  int a_bz, b_bz;  // 1: operand is batched, 0: shared by every batch entry
  int a4, b4;      // 1: the operand has a 4-D chunked map: one TMA per stage
  double2* C;
  long long ldc, strideC, rsplit, ldc_hi;
  double alpha, beta;
  double2* partial;  // split-K partials, dense [z][M][N]
  double* tile_sums;
};

__host__ __device__ constexpr int rho(int g) { return (g >> 1) | ((g & 1) << 2); }

template <int OPA, int OPB, int WGM, int WGN, int WTM, int WTN, int BK, int STAGES>
struct Cfg {
  static constexpr int BM = WGM * WTM, BN = WGN * WTN, NCW = WGM * WGN;
  static constexpr int THREADS = NCW * 32;
  static constexpr uint32_t A_BYTES = BM * BK * 16, B_BYTES = BN * BK * 16;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_BYTES + 1024 + 2 * STAGES * 8;
  static_assert(WTM % 8 == 0 && WTN % 8 == 0 && BK % 8 == 0, "tile shape");
  static_assert(A_BYTES % 1024 == 0 && B_BYTES % 1024 == 0, "swizzle-128B blocks need 1 KB alignment");
};

template <int OPA, int OPB, int WGM, int WGN, int WTM, int WTN, int BK, int STAGES, int MODE>
__global__ void __launch_bounds__(WGM * WGN * 32, 1)
    zgemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const KParams p) {
  using C_ = Cfg<OPA, OPB, WGM, WGN, WTM, WTN, BK, STAGES>;
  constexpr int BM = C_::BM, BN = C_::BN, NCW = C_::NCW;
  constexpr int MI = WTM / 8, NJ = WTN / 8;
  constexpr uint32_t A_BYTES = C_::A_BYTES, STAGE_BYTES = C_::STAGE_BYTES;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(STAGES) * STAGE_BYTES);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grouped rasterization: runs of up to 16 M-tiles share each N-tile, so the
  // CTAs resident at once stream every B tile (and A panel) from HBM once
  const long long tiles_m_all = ceil_div(p.M, BM), tiles_n_all = ceil_div(p.N, BN);
  long long m_tile, n_tile;
  {
    constexpr long long GROUP_M = 16;
    const long long t = blockIdx.x;
    const long long per_group = GROUP_M * tiles_n_all;
    const long long first_m = (t / per_group) * GROUP_M;
    const long long group_m = min(tiles_m_all - first_m, GROUP_M);
    m_tile = first_m + (t % per_group) % group_m;
    n_tile = (t % per_group) / group_m;
  }
  const long long n0 = n_tile * BN;
  const long long m0 = m_tile * BM;
  const int z = blockIdx.z;
  const int b = z / p.splits, split = z % p.splits;
  const int nkt = static_cast<int>(ceil_div(p.K, BK));
  const int kt_begin = split * p.kt_per_split;
  const int kt_end = min(nkt, kt_begin + p.kt_per_split);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // Thread 0 doubles as the TMA producer (a dedicated producer warp would put
  // 3 warps on one SM sub-partition and cap the DMMA warps at 168 registers).
  const int ntiles = kt_end - kt_begin;
  auto issue = [&](int it) {
    const int s = it % STAGES;
    mbar_expect_tx(&full[s], STAGE_BYTES);
    uint8_t* As = smem + size_t(s) * STAGE_BYTES;
    uint8_t* Bs = As + A_BYTES;
    const int k0 = (kt_begin + it) * BK;
    const int za = b * p.a_bz, zb = b * p.b_bz;
    if (OPA == 0 && p.a4) {
      tma_load_4d(As, &tmA, &full[s], 0, (int)m0, k0 / 8, za);
    } else if (OPA == 0) {
#pragma unroll
      for (int c = 0; c < BK / 8; ++c)
        tma_load_3d(As + c * BM * 128, &tmA, &full[s], 2 * (k0 + 8 * c), (int)m0, za);
    } else if (p.a4) {
      tma_load_4d(As, &tmA, &full[s], 0, k0, (int)m0 / 8, za);
    } else {
#pragma unroll
      for (int c = 0; c < BM / 8; ++c)
        tma_load_3d(As + c * BK * 128, &tmA, &full[s], 2 * ((int)m0 + 8 * c), k0, za);
    }
    if (OPB == 0 && p.b4) {
      tma_load_4d(Bs, &tmB, &full[s], 0, k0, (int)n0 / 8, zb);
    } else if (OPB == 0) {
#pragma unroll
      for (int c = 0; c < BN / 8; ++c)
        tma_load_3d(Bs + c * BK * 128, &tmB, &full[s], 2 * ((int)n0 + 8 * c), k0, zb);
    } else if (p.b4) {
      tma_load_4d(Bs, &tmB, &full[s], 0, (int)n0, k0 / 8, zb);
    } else {
#pragma unroll
      for (int c = 0; c < BK / 8; ++c)
        tma_load_3d(Bs + c * BN * 128, &tmB, &full[s], 2 * (k0 + 8 * c), (int)n0, zb);
    }
  };
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int it = 0; it < STAGES && it < ntiles; ++it) issue(it);
  }

  // -------------------------------------------------------------- consumers
  const int g = lane >> 2, t = lane & 3, r8 = rho(g);
  (void)p.K;
  const int wm0 = (warp % WGM) * WTM, wn0 = (warp / WGM) * WTN;

  // 3M (Gauss) products: P1 = Re a Re b, P2 = Im A Im B (raw operands),
  // P3 = (Re a + Im a)(Re b + Im b), a = op(A), b = op(B) entries
  double pacc[MI][NJ][3][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int c = 0; c < 3; ++c) pacc[i][j][c][0] = pacc[i][j][c][1] = 0.0;

  for (int it = 0; it < ntiles; ++it) {
    const int s = it % STAGES;
    const unsigned ph = (it / STAGES) & 1;
    mbar_wait(&full[s], ph);
    const uint8_t* As = smem + size_t(s) * STAGE_BYTES;
    const uint8_t* Bs = As + A_BYTES;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      const int k = ks * 4 + t;
      const int sw = ((k ^ r8) & 7) << 4;  // swizzled 16B slot (row&7 == r8 or k&7)
      double ar[MI], ai[MI], br[NJ], bi[NJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int m = wm0 + 8 * i + r8;
        const int off = (OPA == 0) ? (((k >> 3) * BM + m) * 128 + sw) : (((m >> 3) * BK + k) * 128 + sw);
        const double2 v = *reinterpret_cast<const double2*>(As + off);
        ar[i] = v.x;
        ai[i] = v.y;
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int n = wn0 + 8 * j + r8;
        const int off = (OPB == 0) ? (((n >> 3) * BK + k) * 128 + sw) : (((k >> 3) * BN + n) * 128 + sw);
        const double2 v = *reinterpret_cast<const double2*>(Bs + off);
        br[j] = v.x;
        bi[j] = v.y;
      }
      // 3M: with Im a = sA ai, Im b = sB bi (s = -1 for a conjugated operand),
      // Cre = P1 - sA sB P2 and Cim = P3 - P1 - sA sB P2 -- three real DMMAs per
      // complex 8x8x4 step instead of four, two FP64 adds per fragment pair
      double sa[MI], sb[NJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) sa[i] = OPA == 0 ? ar[i] + ai[i] : ar[i] - ai[i];
#pragma unroll
      for (int j = 0; j < NJ; ++j) sb[j] = OPB == 0 ? br[j] + bi[j] : br[j] - bi[j];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          dmma(pacc[i][j][0][0], pacc[i][j][0][1], ar[i], br[j]);
          dmma(pacc[i][j][1][0], pacc[i][j][1][1], ai[i], bi[j]);
          dmma(pacc[i][j][2][0], pacc[i][j][2][1], sa[i], sb[j]);
        }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    // refill the stage released one iteration ago (slack for slower warps)
    if (threadIdx.x == 0 && it >= 1 && it - 1 + STAGES < ntiles) {
      const int sp = (it - 1) % STAGES;
      mbar_wait(&empty[sp], ((it - 1) / STAGES) & 1);
      issue(it - 1 + STAGES);
    }
  }

  // --------------------------------------------------------------- epilogue
  double acc[MI][NJ][2][2];
  {
    constexpr double sab = (OPA == 0) == (OPB == 0) ? 1.0 : -1.0;  // sA sB
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double p1 = pacc[i][j][0][h], p2 = pacc[i][j][1][h], p3 = pacc[i][j][2][h];
          acc[i][j][0][h] = fma(-sab, p2, p1);
          acc[i][j][1][h] = p3 - fma(sab, p2, p1);
        }
  }
  if (MODE == 0) {
    const bool partial_out = p.splits > 1;
    const bool has_beta = !partial_out && p.beta != 0.0;
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const long long row = m0 + wm0 + 8 * i + r8;
      if (row >= p.M) continue;
      long long rbase;
      if (partial_out)
        rbase = (static_cast<long long>(z) * p.M + row) * p.N;
      else if (p.rsplit > p.M)
        rbase = static_cast<long long>(b) * p.strideC + row * p.ldc;
      else
        rbase = static_cast<long long>(b) * p.strideC + (row % p.rsplit) * p.ldc + (row / p.rsplit) * p.ldc_hi;
      // beta != 0: issue every C load of this row before the first store so
      // the DRAM/L2 round trips overlap (C aliases the stores)
      double2 old[NJ][2];
      if (has_beta) {
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const long long col = n0 + wn0 + 8 * j + t + 4 * h;
            old[j][h] = col < p.N ? p.C[rbase + col] : make_double2(0.0, 0.0);
          }
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const long long col = n0 + wn0 + 8 * j + t + 4 * h;
          if (col >= p.N) continue;
          double2 v = make_double2(acc[i][j][0][h], acc[i][j][1][h]);
          if (partial_out) {
            p.partial[rbase + col] = v;
          } else {
            v.x *= p.alpha;
            v.y *= p.alpha;
            if (has_beta) {
              v.x = fma(p.beta, old[j][h].x, v.x);
              v.y = fma(p.beta, old[j][h].y, v.y);
            }
            p.C[rbase + col] = v;
          }
        }
      }
    }
  } else {
    // RESID: sum |C - alpha * acc|^2 over the tile, deterministic order
    double s2 = 0.0;
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const long long row = m0 + wm0 + 8 * i + r8;
      if (row >= p.M) continue;
      const long long rbase =
          static_cast<long long>(b) * p.strideC + (row % p.rsplit) * p.ldc + (row / p.rsplit) * p.ldc_hi;
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const long long col = n0 + wn0 + 8 * j + t + 4 * h;
          if (col >= p.N) continue;
          const double2 o = p.C[rbase + col];
          const double dr = fma(-p.alpha, acc[i][j][0][h], o.x);
          const double di = fma(-p.alpha, acc[i][j][1][h], o.y);
          s2 = fma(dr, dr, fma(di, di, s2));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    double* red = reinterpret_cast<double*>(full);  // barriers are dead now: reuse after sync
    __syncthreads();
    if (lane == 0) red[warp] = s2;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
      for (int w = 0; w < NCW; ++w) tot += red[w];
      const long long tiles_m = ceil_div(p.M, BM), tiles_n = ceil_div(p.N, BN);
      p.tile_sums[(static_cast<long long>(z) * tiles_m + m_tile) * tiles_n + n_tile] = tot;
    }
  }
}

// split-K reduction: C = alpha * sum_s partial[s] + beta * C, fixed order
__global__ void splitk_reduce_kernel(const double2* __restrict__ partial, int splits, int batch, long long M,
                                     long long N, double2* C, long long ldc, long long strideC,
                                     long long rsplit, long long ldc_hi, double alpha, double beta) {
  const long long total = static_cast<long long>(batch) * M * N;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long col = e % N;
    const long long row = (e / N) % M;
    const long long b = e / (M * N);
    double2 s = make_double2(0.0, 0.0);
    for (int k = 0; k < splits; ++k) {
      const double2 v = partial[((static_cast<long long>(b) * splits + k) * M + row) * N + col];
      s.x += v.x;
      s.y += v.y;
    }
    const long long addr = b * strideC + (row % rsplit) * ldc + (row / rsplit) * ldc_hi + col;
    s.x *= alpha;
    s.y *= alpha;
    if (beta != 0.0) {
      const double2 o = C[addr];
      s.x = fma(beta, o.x, s.x);
      s.y = fma(beta, o.y, s.y);
    }
    C[addr] = s;
  }
}

// one block, fixed reduction tree
__global__ void sum_reduce_kernel(const double* __restrict__ v, long long n, double* out) {
  __shared__ double sh[256];
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) s += v[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// ------------------------------------------------------------ host helpers
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw Error(Err::cuda, "cuTensorMapEncodeTiled entry point unavailable");
  return fn;
}

// 3-D map over a batch of row-major complex matrices: dim0 = 2*contig doubles,
// dim1 = rows (stride ld), dim2 = batch; box = one 128-byte chunk x box_rows.
CUtensorMap make_map(const double2* base, long long contig, long long rows, long long ld, int batch,
                     long long bstride, int box_rows) {
  CUtensorMap m;
  if (batch <= 1) bstride = ld * (rows > 0 ? rows : 1);
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(2 * contig), static_cast<cuuint64_t>(rows),
                        static_cast<cuuint64_t>(batch)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 16, static_cast<cuuint64_t>(bstride) * 16};
  cuuint32_t box[3] = {16, static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double2*>(base), dims, strides,
                           box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[256];
    std::snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (%d): contig=%lld rows=%lld ld=%lld batch=%d",
                  static_cast<int>(r), contig, rows, ld, batch);
    throw Error(Err::cuda, buf);
  }
  return m;
}

// 4-D map over a batch of row-major complex matrices whose contiguous axis is
// cut into 8-element (128-byte) chunks: dim0 = 16 doubles, dim1 = rows
// (stride ld), dim2 = chunks (stride 128 B), dim3 = batch; one box = box_rows
// x box_chunks chunk blocks, laid out in shared memory exactly like box_chunks
// 3-D boxes side by side (chunk-major, 1 KB-aligned blocks: same swizzle).
// Needs contig % 8 == 0 (a ragged last chunk would read past the row).
CUtensorMap make_map4(const double2* base, long long contig, long long rows, long long ld, int batch,
                      long long bstride, int box_rows, int box_chunks) {
  CUtensorMap m;
  if (batch <= 1) bstride = ld * (rows > 0 ? rows : 1);
  cuuint64_t dims[4] = {16, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(contig / 8),
                        static_cast<cuuint64_t>(batch)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(ld) * 16, 128, static_cast<cuuint64_t>(bstride) * 16};
  cuuint32_t box[4] = {16, static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(box_chunks), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double2*>(base), dims, strides,
                           box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[256];
    std::snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled (4-D) failed (%d): contig=%lld rows=%lld ld=%lld batch=%d",
                  static_cast<int>(r), contig, rows, ld, batch);
    throw Error(Err::cuda, buf);
  }
  return m;
}

template <int OPA, int OPB, int WGM, int WGN, int WTM, int WTN, int BK, int STAGES, int MODE>
void launch_cfg(const GemmDesc& d, const GemmScratch& s, cudaStream_t st, double* resid_out) {
  using C_ = Cfg<OPA, OPB, WGM, WGN, WTM, WTN, BK, STAGES>;
  constexpr int BM = C_::BM, BN = C_::BN;
  auto kern = zgemm_kernel<OPA, OPB, WGM, WGN, WTM, WTN, BK, STAGES, MODE>;
  static std::once_flag attr_once;
  std::call_once(attr_once, [&] {
    QT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C_::SMEM)));
  });
  const int a_bz = (d.batch > 1 && d.strideA != 0) ? 1 : 0;
  const int b_bz = (d.batch > 1 && d.strideB != 0) ? 1 : 0;
  const int ba = a_bz ? d.batch : 1, bb = b_bz ? d.batch : 1;
  // the strided-chunk operands (op(A) = A^H: chunks along m; op(B) = B:
  // chunks along n) take one 4-D TMA per stage instead of BM/8 or BN/8 3-D
  // ones when their contiguous extent is a multiple of 8
  // (likewise the K-contiguous operands: BK/8 = 2 -> 1 copies)
  static const bool no4 = std::getenv("QT_GEMM_NO_TMA4D") != nullptr;
  const bool a4 = !no4 && (OPA == 1 ? d.M : d.K) % 8 == 0;
  const bool b4 = !no4 && (OPB == 0 ? d.N : d.K) % 8 == 0;
  const CUtensorMap tA = OPA == 0 ? (a4 ? make_map4(d.A, d.K, d.M, d.lda, ba, d.strideA, BM, BK / 8)
                                        : make_map(d.A, d.K, d.M, d.lda, ba, d.strideA, BM))
                                  : (a4 ? make_map4(d.A, d.M, d.K, d.lda, ba, d.strideA, BK, BM / 8)
                                        : make_map(d.A, d.M, d.K, d.lda, ba, d.strideA, BK));
  const CUtensorMap tB = OPB == 1 ? (b4 ? make_map4(d.B, d.K, d.N, d.ldb, bb, d.strideB, BN, BK / 8)
                                        : make_map(d.B, d.K, d.N, d.ldb, bb, d.strideB, BN))
                                  : (b4 ? make_map4(d.B, d.N, d.K, d.ldb, bb, d.strideB, BK, BN / 8)
                                        : make_map(d.B, d.N, d.K, d.ldb, bb, d.strideB, BK));
  const long long tiles_m = ceil_div(d.M, BM), tiles_n = ceil_div(d.N, BN);
  const int nkt = static_cast<int>(ceil_div(d.K, BK));
  int splits = d.splits;
  if (MODE == 1) splits = 1;
  if (splits <= 0) {
    const long long ctas = tiles_m * tiles_n * d.batch;
    splits = 1;
    // fill roughly two waves when the output tiling alone is too small
    while (ctas * splits * 2 <= 2 * kNumSMs && nkt / (splits * 2) >= 4) splits *= 2;
  }
  if (splits > 1 && static_cast<size_t>(splits) * d.batch * d.M * d.N > s.partial_elems) splits = 1;
  const int kt_per = static_cast<int>(ceil_div(nkt, splits));
  splits = static_cast<int>(ceil_div(nkt, kt_per));
  if (splits < 1) splits = 1;

  KParams p;
  p.M = d.M;
  p.N = d.N;
  p.K = d.K;
  p.splits = splits;
  p.kt_per_split = kt_per > 0 ? kt_per : 1;
  p.a_bz = a_bz;
  p.b_bz = b_bz;
  p.a4 = a4 ? 1 : 0;
  p.b4 = b4 ? 1 : 0;
  p.C = d.C;
  p.ldc = d.ldc;
  p.strideC = d.strideC;
  p.rsplit = d.rsplit > 0 ? d.rsplit : (1LL << 62);
  p.ldc_hi = d.ldc_hi;
  p.alpha = d.alpha;
  p.beta = d.beta;
  p.partial = s.partial;
  p.tile_sums = s.tile_sums;
  if (MODE == 1 && static_cast<size_t>(tiles_m * tiles_n * d.batch) > s.tile_sums_elems)
    throw Error(Err::capacity, "zgemm: tile_sums scratch too small");

  dim3 grid(static_cast<unsigned>(tiles_n * tiles_m), 1, static_cast<unsigned>(d.batch * splits));
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool capturing = false;
  const double gflops = 8.0 * d.M * d.N * d.K * d.batch;
  const bool prof = g_prof.active && gflops >= g_prof.min_flops;
  if (prof) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    QT_CUDA(cudaStreamIsCapturing(st, &cs));
    capturing = cs == cudaStreamCaptureStatusActive;
    if (capturing) {
      // events baked into a CUDA graph: fresh ones, owned by that graph
      QT_CUDA(cudaEventCreate(&ev0));
      QT_CUDA(cudaEventCreate(&ev1));
      QT_CUDA(cudaEventRecordWithFlags(ev0, st, cudaEventRecordExternal));
    } else {
      ev0 = g_prof.event();
      ev1 = g_prof.event();
      QT_CUDA(cudaEventRecord(ev0, st));
    }
  }
  kern<<<grid, C_::THREADS, C_::SMEM, st>>>(tA, tB, p);
  QT_LAUNCHED();
  if (prof) {
    if (capturing)
      QT_CUDA(cudaEventRecordWithFlags(ev1, st, cudaEventRecordExternal));
    else
      QT_CUDA(cudaEventRecord(ev1, st));
    (capturing ? g_prof.captured : g_prof.recs).push_back({ev0, ev1, gflops});
  }
  if (MODE == 0 && splits > 1) {
    const long long total = static_cast<long long>(d.batch) * d.M * d.N;
    const int blocks = static_cast<int>(std::min<long long>(ceil_div(total, 256), 8 * kNumSMs));
    splitk_reduce_kernel<<<blocks, 256, 0, st>>>(s.partial, splits, d.batch, d.M, d.N, d.C, d.ldc, d.strideC,
                                                 p.rsplit, d.ldc_hi, d.alpha, d.beta);
    QT_LAUNCHED();
  }
  if (MODE == 1) {
    sum_reduce_kernel<<<1, 256, 0, st>>>(s.tile_sums, tiles_m * tiles_n * d.batch, resid_out);
    QT_LAUNCHED();
  }
}

template <int OPA, int OPB, int MODE>
void dispatch_shape(const GemmDesc& d, const GemmScratch& s, cudaStream_t st, double* r) {
  // Tile shape and split-K count from a makespan model: every SM runs
  // ceil(units / 148) units of bm x bn x (K / splits) complex MACs at the
  // per-SM FP64 rate (16 CMAC/clk) times a per-tile efficiency, plus the
  // split-K partial traffic and reduction launch.  Wave quantization is what
  // matters for the chi <= 512 products (e.g. 1280 x 256 x 1280: 160 tiles of
  // 32 x 64 = two rounds on 12 SMs; 40 tiles of 64 x 128 split 7 ways = 280
  // units, 94% balanced on 148 SMs).
  struct Cand {
    long long bm, bn;
    double eff;
    bool ok;
  };
  const Cand cands[4] = {{64, 128, 1.0, d.M > 32}, {64, 64, 0.9, d.M > 32}, {32, 128, 0.95, d.M <= 32},
                         {32, 64, 0.85, true}};
  static const bool fixed_split = std::getenv("QT_GEMM_NO_MODEL") != nullptr;
  const long long nkt = ceil_div(d.K, 16);
  int best = -1, best_s = 1;
  double best_t = 1e300;
  for (int c = 0; c < 4; ++c) {
    if (!cands[c].ok) continue;
    const long long tiles = ceil_div(d.M, cands[c].bm) * ceil_div(d.N, cands[c].bn) * d.batch;
    // split-K for products of up to eight waves: below two the imbalance of
    // the last wave dominates; up to eight a 2-4 way split still beats a
    // mostly empty last wave (north-star X and Hastings, 640 tiles = 4.3
    // waves: 5 rounds unsplit, 9 rounds of half the K split two ways)
    const bool may_split = tiles < 8 * kNumSMs;
    for (int sp = 1; sp <= 16; ++sp) {
      if (sp > 1 && (!may_split || MODE == 1 || d.splits > 0 || fixed_split || nkt / sp < 4 ||
                     static_cast<size_t>(sp) * d.batch * d.M * d.N > s.partial_elems))
        break;
      const double rounds = static_cast<double>(ceil_div(tiles * sp, static_cast<long long>(kNumSMs)));
      const double unit = static_cast<double>(cands[c].bm * cands[c].bn) * 16.0 * ceil_div(nkt, sp);
      double t = rounds * unit / (31.4e3 * cands[c].eff);  // us
      if (sp > 1) t += (2.0 * sp + 1.0) * static_cast<double>(d.M * d.N * d.batch) * 16.0 / 6.0e6 + 4.0;
      if (t < best_t * 0.98) {
        best_t = t;
        best = c;
        best_s = sp;
      }
    }
  }
  // short-K products (K <= 1024) with many tiles: 64 x 64 tiles run two
  // CTAs per SM (97 KB of shared memory, 128 threads each), so one CTA's
  // pipeline fill and C epilogue overlap the other's DMMA work -- 1.12x over
  // 64 x 128 at K = 128 (block-reflector updates), 1.04x at K = 512, 1.02x at
  // K = 1024 (theta); longer K keeps the larger tile (5120 x 1024 x 5120:
  // 0.97x with 64 x 64)
  if (best == 0 && nkt <= 64 && ceil_div(d.M, 64) * ceil_div(d.N, 128) * d.batch >= 2 * kNumSMs) {
    best = 1;
    best_s = 1;
  }
  GemmDesc dd = d;
  if (d.splits <= 0 && !fixed_split) dd.splits = best_s;
  switch (best) {
    case 0: launch_cfg<OPA, OPB, 2, 4, 32, 32, 16, 4, MODE>(dd, s, st, r); break;
    case 1: launch_cfg<OPA, OPB, 2, 2, 32, 32, 16, 3, MODE>(dd, s, st, r); break;
    case 2: launch_cfg<OPA, OPB, 1, 4, 32, 32, 16, 4, MODE>(dd, s, st, r); break;
    default: launch_cfg<OPA, OPB, 2, 2, 16, 32, 16, 4, MODE>(dd, s, st, r); break;
  }
}

template <int MODE>
void dispatch_ops(const GemmDesc& d, const GemmScratch& s, cudaStream_t st, double* r) {
  const int code = static_cast<int>(d.opA) * 2 + static_cast<int>(d.opB);
  switch (code) {
    case 0: dispatch_shape<0, 0, MODE>(d, s, st, r); break;
    case 1: dispatch_shape<0, 1, MODE>(d, s, st, r); break;
    case 2: dispatch_shape<1, 0, MODE>(d, s, st, r); break;
    default: dispatch_shape<1, 1, MODE>(d, s, st, r); break;
  }
}

}  // namespace

void zgemm(const GemmDesc& d, const GemmScratch& s, cudaStream_t stream, double* resid_out) {
  if (d.M < 0 || d.N < 0 || d.K < 0 || d.batch < 1) throw Error(Err::shape, "zgemm: bad dimensions");
  if (d.M == 0 || d.N == 0) return;
  if (d.K == 0) throw Error(Err::shape, "zgemm: K == 0 is not supported");
  if (d.mode == GemmMode::resid && resid_out == nullptr) throw Error(Err::internal, "zgemm: resid_out missing");
  if (d.mode == GemmMode::store)
    dispatch_ops<0>(d, s, stream, nullptr);
  else
    dispatch_ops<1>(d, s, stream, resid_out);
}

unsigned long long zgemm_launch_count() { return g_kernel_launches.load(); }

void gemm_profile_begin(double min_flops) {
  g_prof.min_flops = min_flops;
  g_prof.active = true;
  g_prof.recs.clear();
  g_prof.next = 0;
  g_prof.replayed = GemmProfile();
}

bool gemm_profile_active() { return g_prof.active; }

std::vector<GemmProfRec> gemm_profile_take_captured() {
  std::vector<GemmProfRec> out;
  out.swap(g_prof.captured);
  return out;
}

void gemm_profile_add_replay(const std::vector<GemmProfRec>& recs) {
  if (!g_prof.active) return;
  for (const auto& rec : recs) {
    QT_CUDA(cudaEventSynchronize(rec.e1));
    float ms = 0.f;
    QT_CUDA(cudaEventElapsedTime(&ms, rec.e0, rec.e1));
    g_prof.replayed.ms += ms;
    g_prof.replayed.flops += rec.flops;
    g_prof.replayed.launches += 1;
  }
}

GemmProfile gemm_profile_end() {
  GemmProfile r = g_prof.replayed;
  g_prof.replayed = GemmProfile();
  g_prof.active = false;
  for (const auto& rec : g_prof.recs) {
    QT_CUDA(cudaEventSynchronize(rec.e1));
    float ms = 0.f;
    QT_CUDA(cudaEventElapsedTime(&ms, rec.e0, rec.e1));
    r.ms += ms;
    r.flops += rec.flops;
    r.launches += 1;
  }
  g_prof.recs.clear();
  g_prof.next = 0;
  return r;
}

}  // namespace qt
