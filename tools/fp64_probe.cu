// Microbenchmark: FP64 throughput on B200 via DFMA (CUDA cores) vs DMMA (mma.sync f64 tensor path).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += acc[i];
  if (s == 12345.678) out[blockIdx.x] = s;
}

template <int TILES>
__global__ void dmma884_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[TILES][2];
#pragma unroll
  for (int t = 0; t < TILES; ++t) { c[t][0] = t; c[t][1] = -t; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < TILES; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < TILES; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.678) out[blockIdx.x] = s;
}

template <int TILES>
__global__ void dmma1684_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = 0.5 + a0, b = 1.0 - threadIdx.x * 1e-4;
  double c[TILES][4];
#pragma unroll
  for (int t = 0; t < TILES; ++t) { c[t][0] = t; c[t][1] = -t; c[t][2] = 1; c[t][3] = 2; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < TILES; ++t) {
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3]) : "d"(a0), "d"(a1), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < TILES; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  if (s == 12345.678) out[blockIdx.x] = s;
}

template <int TILES>
__global__ void dmma16816_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 + i;
  double c[TILES][4];
#pragma unroll
  for (int t = 0; t < TILES; ++t) { c[t][0] = t; c[t][1] = -t; c[t][2] = 1; c[t][3] = 2; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < TILES; ++t) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < TILES; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  if (s == 12345.678) out[blockIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  printf("device %s SMs %d\n", p.name, sms);
  double* out; cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch, double flop_per_launch) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s %8.2f TFLOP/s  (%.3f ms/launch) err=%s\n", name, 5 * flop_per_launch / (ms * 1e-3) / 1e12, ms / 5,
           cudaGetErrorString(cudaGetLastError()));
  };
  const int iters = 4096;
  for (int bpsm : {1, 2, 4, 8}) {
    for (int threads : {128, 256, 512}) {
      int blocks = sms * bpsm;
      char nm[64];
      snprintf(nm, 64, "DFMA8 b%d t%d", bpsm, threads);
      run(nm, [&] { dfma_kernel<8><<<blocks, threads>>>(out, iters, 0.999, 1e-3); }, 2.0 * 8 * iters * blocks * threads);
      snprintf(nm, 64, "DMMA884x8 b%d t%d", bpsm, threads);
      run(nm, [&] { dmma884_kernel<8><<<blocks, threads>>>(out, iters); }, 2.0 * 256 * 8 * iters * blocks * (threads / 32));
      snprintf(nm, 64, "DMMA1684x4 b%d t%d", bpsm, threads);
      run(nm, [&] { dmma1684_kernel<4><<<blocks, threads>>>(out, iters); }, 2.0 * 512 * 4 * iters * blocks * (threads / 32));
      snprintf(nm, 64, "DMMA16816x4 b%d t%d", bpsm, threads);
      run(nm, [&] { dmma16816_kernel<4><<<blocks, threads>>>(out, iters / 4); }, 2.0 * 2048 * 4 * (iters / 4) * blocks * (threads / 32));
    }
  }
  return 0;
}
