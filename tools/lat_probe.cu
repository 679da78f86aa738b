// Dependent-latency probe (one warp): DFMA chain, shared-memory load->use, cinv-like division.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double a, double b) {
  double x = a;
  __shared__ double sm[64];
  sm[threadIdx.x] = b;
  __syncwarp();
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  int idx = threadIdx.x;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { idx = (int)sm[idx & 31] & 31; }
  long long t2 = clock64();
  double y = b;
#pragma unroll 1
  for (int i = 0; i < 256; ++i) y = 1.0 / (y + a);
  long long t3 = clock64();
  double z = b;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) z = z * a;
  long long t4 = clock64();
  out[threadIdx.x] = x + idx + y + z;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
  lat<<<1, 32>>>(o, c, 0.999, 0.5);
  lat<<<1, 32>>>(o, c, 0.999, 0.5);
  long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  printf("DFMA dependent: %.1f cycles\n", h[0] / 1024.0);
  printf("LDS.64 load->use (+cvt): %.1f cycles\n", h[1] / 1024.0);
  printf("DP reciprocal+add chain: %.1f cycles\n", h[2] / 256.0);
  printf("DMUL dependent: %.1f cycles\n", h[3] / 1024.0);
  return 0;
}
