// Probe: QR of an m x n panel-chain matrix with and without the Q^H C
// application on the side stream (QrOpts::capply), CUDA events on the main
// stream.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17
//   -I paper_2212_09782_b200/csrc tools/probes/qtheta_probe.cu
//   -L paper_2212_09782_b200 -lqrtebd_b200 -o tools/probes/qtheta_probe
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "engine.cuh"

using namespace qt;

__global__ void ext_kernel(const double2* c, long long nc, long long k, double2* yh, long long r0, long long nr) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nr * nc; e += (long long)gridDim.x * blockDim.x) {
    const long long i = r0 + e / nc, col = e % nc;
    const double2 v = c[i * nc + col];
    yh[col * k + i] = make_double2(v.x, -v.y);
  }
}

int main(int argc, char** argv) {
  const long long m = argc > 1 ? atoll(argv[1]) : 1280, n = argc > 2 ? atoll(argv[2]) : 256;
  const long long nc = argc > 3 ? atoll(argv[3]) : m;
  Engine e;
  e.init(0, nullptr);
  std::vector<double2> h(m * (n > nc ? n : nc));
  srand(1);
  for (auto& v : h) v = make_double2(rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5);
  double2 *A0, *A, *C0, *C, *Q, *R;
  cudaMalloc(&A0, m * n * 16); cudaMalloc(&A, m * n * 16);
  cudaMalloc(&C0, m * nc * 16); cudaMalloc(&C, m * nc * 16);
  cudaMalloc(&Q, m * n * 16); cudaMalloc(&R, n * n * 16);
  cudaMemcpy(A0, h.data(), m * n * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(C0, h.data(), m * nc * 16, cudaMemcpyHostToDevice);
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0); cudaEventCreate(&t1);
  auto run = [&](int mode) {  // 0: Q + R, 1: capply, no Q, 2: capply + Q
    float best = 1e9;
    for (int it = 0; it < 6; ++it) {
      cudaMemcpyAsync(A, A0, m * n * 16, cudaMemcpyDeviceToDevice, e.stream);
      cudaMemcpyAsync(C, C0, m * nc * 16, cudaMemcpyDeviceToDevice, e.stream);
      QrOpts o;
      if (mode >= 1) { o.capply = C; o.ldc = nc; o.nc = nc; o.want_q = mode == 2; o.want_r = false; }
      cudaEventRecord(t0, e.stream);
      qr_inplace(e, A, m, n, n, Q, n, R, n, o);
      cudaEventRecord(t1, e.stream);
      cudaStreamSynchronize(e.stream);
      float ms;
      cudaEventElapsedTime(&ms, t0, t1);
      if (it > 0 && ms < best) best = ms;
    }
    return best * 1000.f;
  };
  double2 *YH, *QY, *RY;
  cudaMalloc(&YH, nc * n * 16); cudaMalloc(&QY, nc * n * 16); cudaMalloc(&RY, n * n * 16);
  auto run_pair = [&]() {
    float best = 1e9;
    for (int it = 0; it < 6; ++it) {
      cudaMemcpyAsync(A, A0, m * n * 16, cudaMemcpyDeviceToDevice, e.stream);
      cudaMemcpyAsync(C, C0, m * nc * 16, cudaMemcpyDeviceToDevice, e.stream);
      cudaEventRecord(t0, e.stream);
      qr_pair_pipelined(e, A, m, n, C, nc, YH, QY, RY, [&](long long r0, long long nr, cudaStream_t st) {
        ext_kernel<<<296, 256, 0, st>>>(C, nc, n, YH, r0, nr);
      });
      cudaEventRecord(t1, e.stream);
      cudaStreamSynchronize(e.stream);
      float ms;
      cudaEventElapsedTime(&ms, t0, t1);
      if (it > 0 && ms < best) best = ms;
    }
    return best * 1000.f;
  };
  if (qr_pair_fits(m, nc) && n <= m && n <= nc)
    printf("pipelined pair (QR(X) + apply + QR(Y^H) + Q_y): %.1f us\n", run_pair());
  printf("m=%lld n=%lld nc=%lld: QR with Q+R %.1f us | QR + apply to C (no Q) %.1f us | QR + apply + Q %.1f us\n", m,
         n, nc, run(0), run(1), run(2));
  return 0;
}
