// Latency model of the per-column critical path (cycles): FP64 chains, MUFU
// based reciprocals, shared-memory round trips, CTA barriers with 16 warps,
// and DSMEM ping-pong between two CTAs of a cluster (st.async and bulk copy).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o latency_probe latency_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

__global__ void chains(double* out, long long* cyc, double a, double b, int n) {
  double x = a, y = b;
  long long t[16];
  int q = 0;
  t[q++] = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, a);
  t[q++] = clock64();
  for (int i = 0; i < n; ++i) x = x + y;
  t[q++] = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 2.0);
  t[q++] = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x + 2.0);
  t[q++] = clock64();
  for (int i = 0; i < n; ++i) x = rcp_nr(x + 2.0);
  t[q++] = clock64();
  for (int i = 0; i < n; ++i) x = a / (x + 2.0);
  t[q++] = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (i + threadIdx.x) & 31) + y;
  t[q++] = clock64();
  __shared__ double2 s[64];
  s[threadIdx.x] = make_double2(x, y);
  __syncwarp();
  double2 v = s[threadIdx.x];
  for (int i = 0; i < n; ++i) v = s[static_cast<int>(v.y * 0.0) + (i & 31)];
  t[q++] = clock64();
  out[threadIdx.x] = x + v.x;
  if (threadIdx.x == 0)
    for (int i = 0; i + 1 < q; ++i) cyc[i] = t[i + 1] - t[i];
}

// 16 warps: cost of one __syncthreads round when all warps arrive together
__global__ void barriers(long long* cyc, int n) {
  __shared__ double2 s[512];
  double2 v = make_double2(threadIdx.x, 0.0);
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    s[threadIdx.x] = v;
    __syncthreads();
    v = s[(threadIdx.x + 32) & 511];
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 2;
  if (v.x < -1) cyc[1] = 0;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cl_map(const void* p, unsigned rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_arm(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned par) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "W:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\nD:\n\t}" ::"r"(
          smem_u32(b)),
      "r"(par)
      : "memory");
}

// ping-pong between CTA 0 and CTA 1 of a 2-CTA cluster: lane 0..31 each push
// one double2 (st.async) or lane 0 one 512-byte bulk copy; n round trips
__global__ void __cluster_dims__(2, 1, 1) pingpong(long long* cyc, int n, int bulk) {
  __shared__ __align__(16) double2 buf[2][32];
  __shared__ __align__(16) double2 src[32];
  __shared__ uint64_t bar[2];
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int k = threadIdx.x;
  if (k == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  src[k] = make_double2(k, rank);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  const unsigned peer = rank ^ 1u;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const int par = i & 1;
    if (k == 0) mbar_arm(&bar[par], 512);
    __syncwarp();
    const bool my_turn = (rank == 0);
    if (my_turn || i > 0 || true) {
      // rank 0 sends first, rank 1 replies after receiving
      if (rank == 1) mbar_wait(&bar[par], (i >> 1) & 1);
      if (bulk) {
        if (k == 0)
          asm volatile(
              "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" ::"r"(
                  cl_map(&buf[par][0], peer)),
              "r"(smem_u32(src)), "r"(cl_map(&bar[par], peer))
              : "memory");
      } else {
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                         cl_map(&buf[par][k], peer)),
                     "d"(static_cast<double>(k)), "d"(1.0), "r"(cl_map(&bar[par], peer))
                     : "memory");
      }
      if (rank == 0) mbar_wait(&bar[par], (i >> 1) & 1);
    }
  }
  long long t1 = clock64();
  if (rank == 0 && k == 0) cyc[bulk] = (t1 - t0) / n;
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// all-to-all of 512 B per CTA pair inside a 16-CTA cluster (the panel's
// per-column exchange): warp w pushes to CTA w (st.async), warp 0 waits and
// combines; n rounds; mode 1 = only CTA 0 receives (gather), mode 2 = gather
// to CTA 0 + broadcast of 512 B back
__global__ void alltoall(long long* cyc, int n, int mode) {
  __shared__ __align__(16) double2 recv[2][16][32];
  __shared__ __align__(16) double2 out[2][32];
  __shared__ uint64_t bar[2];
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int CS = 16;
  const int w = threadIdx.x >> 5, k = threadIdx.x & 31;
  const unsigned bytes = mode == 0 ? CS * 512 : (rank == 0 ? CS * 512 : 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_arm(&bar[0], bytes);
    mbar_arm(&bar[1], bytes);
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  double2 acc = make_double2(rank, k);
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const int par = i & 1;
    __syncthreads();
    if (mode == 0) {
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                       cl_map(&recv[par][rank][k], w)),
                   "d"(acc.x), "d"(acc.y), "r"(cl_map(&bar[par], w))
                   : "memory");
    } else if (w == 0) {
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                       cl_map(&recv[par][rank][k], 0)),
                   "d"(acc.x), "d"(acc.y), "r"(cl_map(&bar[par], 0))
                   : "memory");
    }
    if (w == 0) {
      if (mode == 0 || rank == 0) {
        mbar_wait(&bar[par], (i >> 1) & 1);
        if (k == 0) mbar_arm(&bar[par], bytes);
        double2 s = make_double2(0.0, 0.0);
#pragma unroll
        for (int r = 0; r < 16; ++r) s.x += recv[par][r][k].x, s.y += recv[par][r][k].y;
        acc.x = s.x * 1e-3;
        acc.y = s.y * 1e-3;
        if (mode == 2) out[par][k] = acc;
      }
    }
    if (mode == 2) {
      __syncthreads();
      if (rank == 0 && w < CS)
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                         cl_map(&out[par][k], w)),
                     "d"(out[par][k].x), "d"(out[par][k].y), "r"(cl_map(&bar[par], w))
                     : "memory");
      if (rank != 0 && w == 0) {
        mbar_wait(&bar[par], (i >> 1) & 1);
        if (k == 0) mbar_arm(&bar[par], bytes);
        acc = out[par][k];
      }
    }
  }
  long long t1 = clock64();
  if (rank == 0 && threadIdx.x == 0) cyc[mode] = (t1 - t0) / n;
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 4096);
  cudaMallocManaged(&c, 256);
  const int n = 1000;
  for (int r = 0; r < 2; ++r) chains<<<1, 32>>>(o, c, 1.0000001, 0.9999999, n);
  cudaDeviceSynchronize();
  printf("cycles/op: dfma %.1f dadd %.1f dsqrt %.1f rsqrt %.1f rcp_nr %.1f ddiv %.1f shfl+dadd %.1f lds128(dep) %.1f\n",
         c[0] / (double)n, c[1] / (double)n, c[2] / (double)n, c[3] / (double)n, c[4] / (double)n, c[5] / (double)n,
         c[6] / (double)n, c[7] / (double)n);
  for (int r = 0; r < 2; ++r) barriers<<<1, 512>>>(c, n);
  cudaDeviceSynchronize();
  printf("syncthreads (512 threads, STS+LDS between): %.1f cycles\n", c[0] / (double)n);
  for (int bulk = 0; bulk < 2; ++bulk)
    for (int r = 0; r < 2; ++r) pingpong<<<2, 32>>>(c, n, bulk);
  cudaError_t err = cudaDeviceSynchronize();
  printf("DSMEM round trip (2-CTA cluster): st.async x32 lanes %lld cycles, bulk 512B %lld cycles (%s)\n", c[0], c[1],
         cudaGetErrorString(err));
  cudaFuncSetAttribute(alltoall, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int mode = 0; mode < 3; ++mode) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(512);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    for (int r = 0; r < 2; ++r) cudaLaunchKernelEx(&cfg, alltoall, c, n, mode);
    err = cudaDeviceSynchronize();
    printf("16-CTA cluster, mode %d (%s): %lld cycles/round (%s)\n", mode,
           mode == 0 ? "all-to-all 512B" : mode == 1 ? "gather to CTA0" : "gather + broadcast", c[mode],
           cudaGetErrorString(err));
  }
  return 0;
}
