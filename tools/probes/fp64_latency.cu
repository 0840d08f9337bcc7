// Dependent-chain latency of FP64 ops on this GPU (cycles per op).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  double x = a, y = b;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, a);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x * y;
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = x + y;
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = a / x;
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 2.0);
  long long t5 = clock64();
  __shared__ double2 s[64];
  s[threadIdx.x] = make_double2(x, y);
  __syncwarp();
  double2 v = s[threadIdx.x];
  for (int i = 0; i < n; ++i) { v = s[(int)(v.x) & 31]; }
  long long t6 = clock64();
  out[threadIdx.x] = x + v.x;
  if (threadIdx.x == 0) { cyc[0]=t1-t0; cyc[1]=t2-t1; cyc[2]=t3-t2; cyc[3]=t4-t3; cyc[4]=t5-t4; cyc[5]=t6-t5; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024); cudaMallocManaged(&c, 64);
  const int n = 1000;
  k<<<1, 32>>>(o, c, 1.0000001, 0.9999999, n); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 1.0000001, 0.9999999, n); cudaDeviceSynchronize();
  printf("cycles/op: dfma %.1f dmul %.1f dadd %.1f ddiv %.1f dsqrt %.1f lds(dep) %.1f\n", c[0]/(double)n, c[1]/(double)n,
         c[2]/(double)n, c[3]/(double)n, c[4]/(double)n, c[5]/(double)n);
  return 0;
}
