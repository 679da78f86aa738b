// Accuracy of DMMA.8x8x4 (mma.sync m8n8k4 f64) against scalar DFMA on long dot products:
// a warp computes an 8x8 block of A[8 x K] B[K x 8] with DMMA (K/4 steps) and one thread per
// output computes the same dot product with sequential fma(); both are compared with a host
// reference in long double.  Positive data exposes a rounding bias (error ~ K eps instead of
// sqrt(K) eps).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_accuracy tools/dmma_accuracy.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void dmma_dot(const double* A, const double* B, double* C, int K) {
  // A [8][K] row-major, B [K][8] row-major; one warp
  const int lane = threadIdx.x, fr = lane >> 2, fc = lane & 3;
  double c0 = 0, c1 = 0;
  for (int k = 0; k < K; k += 4) {
    const double a = A[fr * K + k + fc];
    const double b = B[(k + fc) * 8 + fr];  // B fragment: B[k = fc][n = fr]
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
  }
  C[fr * 8 + 2 * fc] = c0;
  C[fr * 8 + 2 * fc + 1] = c1;
}

__global__ void fma_dot(const double* A, const double* B, double* C, int K) {
  const int r = threadIdx.x >> 3, c = threadIdx.x & 7;
  double acc = 0;
  for (int k = 0; k < K; ++k) acc = fma(A[r * K + k], B[k * 8 + c], acc);
  C[r * 8 + c] = acc;
}

int main() {
  for (int mode = 0; mode < 2; ++mode)
    for (int K : {64, 1024, 16384, 262144}) {
      std::vector<double> a(8 * (size_t)K), b((size_t)K * 8);
      srand(7 + K);
      for (auto& x : a) x = mode ? (rand() / (double)RAND_MAX - 0.5) : rand() / (double)RAND_MAX;
      for (auto& x : b) x = mode ? (rand() / (double)RAND_MAX - 0.5) : rand() / (double)RAND_MAX;
      double *dA, *dB, *dC, *dF;
      cudaMalloc(&dA, a.size() * 8);
      cudaMalloc(&dB, b.size() * 8);
      cudaMalloc(&dC, 64 * 8);
      cudaMalloc(&dF, 64 * 8);
      cudaMemcpy(dA, a.data(), a.size() * 8, cudaMemcpyHostToDevice);
      cudaMemcpy(dB, b.data(), b.size() * 8, cudaMemcpyHostToDevice);
      dmma_dot<<<1, 32>>>(dA, dB, dC, K);
      fma_dot<<<1, 64>>>(dA, dB, dF, K);
      double hc[64], hf[64];
      cudaMemcpy(hc, dC, 64 * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(hf, dF, 64 * 8, cudaMemcpyDeviceToHost);
      double em = 0, ef = 0, bm = 0, bf = 0, mx = 0;
      for (int r = 0; r < 8; ++r)
        for (int c = 0; c < 8; ++c) {
          long double s = 0;
          for (int k = 0; k < K; ++k) s += (long double)a[r * K + k] * (long double)b[k * 8 + c];
          const double ex = (double)s;
          mx = std::fmax(mx, std::fabs(ex));
          em = std::fmax(em, std::fabs(hc[r * 8 + c] - ex));
          ef = std::fmax(ef, std::fabs(hf[r * 8 + c] - ex));
          bm += (hc[r * 8 + c] - ex) / 64;
          bf += (hf[r * 8 + c] - ex) / 64;
        }
      std::printf("%s K=%7d  max rel err DMMA %.2e  FMA %.2e   mean signed err / max: DMMA %+.2e FMA %+.2e\n",
                  mode ? "signed  " : "positive", K, em / mx, ef / mx, bm / mx, bf / mx);
      cudaFree(dA);
      cudaFree(dB);
      cudaFree(dC);
      cudaFree(dF);
    }
  return 0;
}
