// Panel-step microbenchmark: times the NB = 32 panel variants of find_solve.cu on
// identical random panels and checks them bit for bit against panel_kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        tools/panel_bench.cu -o tools/panel_bench && tools/panel_bench [s] [b] [count] [nE]
#include "../paper_1104_0623_b200/csrc/find_solve.cu"

#include <random>

using namespace findb200;

static int64_t scratch_elems(int64_t n, int64_t s, int nb) {  // find_scratch_elems (plan.cpp)
  int64_t e = 2 * n * n + (3 * s + 264 + 3) / 4 + 1 + (n + 31) / 32;
  if (nb > 0) e += 2 * ((s + nb - 1) / nb) * (int64_t)nb * nb + (n - s) * s;
  return (e + 1) & ~int64_t(1);
}

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      std::printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                 \
    }                                                                               \
  } while (0)

int main(int argc, char** argv) {
  const int s = argc > 1 ? std::atoi(argv[1]) : 132;
  const int b = argc > 2 ? std::atoi(argv[2]) : 8;
  const int count = argc > 3 ? std::atoi(argv[3]) : 64;
  const int nE = argc > 4 ? std::atoi(argv[4]) : 16;
  const int n = s + b;
  const int64_t per = scratch_elems(n, s, 32);
  std::vector<ElimDesc> el(count);
  for (int i = 0; i < count; ++i) {
    std::memset(&el[i], 0, sizeof(ElimDesc));
    el[i].s = s; el[i].b = b; el[i].n = n;
    el[i].ws_off = (int64_t)i * per;
  }
  const int64_t total = per * count;  // per energy
  std::vector<double2> h((size_t)total * nE);
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd;
  for (auto& x : h) x = make_double2(nd(rng), nd(rng));
  // pmax chunks = 1.0 (scale), PIV etc. are outputs
  for (int e = 0; e < nE; ++e)
    for (int i = 0; i < count; ++i) {
      double2* M = h.data() + (size_t)e * total + (size_t)i * per;
      const int64_t nn = (int64_t)n * n;
      const int64_t ints = (3 * s + 264 + 3) / 4;
      double* scale = reinterpret_cast<double*>(M + 2 * nn + ints);
      for (int q = 0; q < (n + 31) / 32 * 2; ++q) scale[2 + q] = 1.0;
    }
  double2 *d0, *d1;
  ElimDesc* de;
  Task* dt;
  unsigned long long* dst;
  CK(cudaMalloc(&d0, h.size() * sizeof(double2)));
  CK(cudaMalloc(&d1, h.size() * sizeof(double2)));
  CK(cudaMalloc(&de, count * sizeof(ElimDesc)));
  CK(cudaMalloc(&dt, count * sizeof(Task)));
  CK(cudaMalloc(&dst, 8));
  CK(cudaMemcpy(d0, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(de, el.data(), count * sizeof(ElimDesc), cudaMemcpyHostToDevice));
  std::vector<Task> tk(count);
  for (int i = 0; i < count; ++i) tk[i] = {i, 0, 0, 0};
  CK(cudaMemcpy(dt, tk.data(), count * sizeof(Task), cudaMemcpyHostToDevice));
  SolveParams P;
  std::memset(&P, 0, sizeof(P));
  P.elims = de;
  P.scratch = d1;
  P.scratch_elems = total;
  P.rtol = 1e-12;
  P.status = dst;
  const dim3 grid(count, nE);
  std::vector<double2> ref, out;
  auto run = [&](int variant, int reps, bool keep) -> float {
    cudaEvent_t a, z;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&z));
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
      CK(cudaMemcpy(d1, d0, h.size() * sizeof(double2), cudaMemcpyDeviceToDevice));
      CK(cudaEventRecord(a));
      switch (variant) {
        case 0: panel_kernel<32, 256><<<grid, 256>>>(P, dt); break;
        case 1:
          if (s <= 64) panel1_kernel<32, 64><<<grid, 64>>>(P, dt);
          else if (s <= 96) panel1_kernel<32, 96><<<grid, 96>>>(P, dt);
          else if (s <= 128) panel1_kernel<32, 128><<<grid, 128>>>(P, dt);
          else if (s <= 160) panel1_kernel<32, 160><<<grid, 160>>>(P, dt);
          else if (s <= 192) panel1_kernel<32, 192><<<grid, 192>>>(P, dt);
          else if (s <= 224) panel1_kernel<32, 224><<<grid, 224>>>(P, dt);
          else panel1_kernel<32, 256><<<grid, 256>>>(P, dt);
          break;
        case 3:
          CK(cudaFuncSetAttribute(panel_smem_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem));
          panel_smem_kernel<16><<<grid, 256, (size_t)s * 17 * sizeof(double2)>>>(P, dt);
          break;
        case 4:
          if (s <= 64) panel1_kernel<16, 64><<<grid, 64>>>(P, dt);
          else if (s <= 96) panel1_kernel<16, 96><<<grid, 96>>>(P, dt);
          else if (s <= 128) panel1_kernel<16, 128><<<grid, 128>>>(P, dt);
          else if (s <= 160) panel1_kernel<16, 160><<<grid, 160>>>(P, dt);
          else if (s <= 192) panel1_kernel<16, 192><<<grid, 192>>>(P, dt);
          else if (s <= 224) panel1_kernel<16, 224><<<grid, 224>>>(P, dt);
          else panel1_kernel<16, 256><<<grid, 256>>>(P, dt);
          break;
        case 2: {
          const size_t pb = warp_panel_bytes(s, 32);
          const int w = (int)std::max<size_t>(1, std::min<size_t>(8, kMaxSmem / pb));
          CK(cudaFuncSetAttribute(warp_panel_kernel<32, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem));
          warp_panel_kernel<32, 8><<<dim3((count + w - 1) / w, nE), 32 * w, pb * w>>>(P, dt, count, s);
          break;
        }
      }
      CK(cudaEventRecord(z));
      CK(cudaEventSynchronize(z));
      CK(cudaGetLastError());
      float ms;
      CK(cudaEventElapsedTime(&ms, a, z));
      best = std::min(best, ms);
    }
    if (keep) {
      std::vector<double2>& o = (variant == 0 || variant == 3) ? ref : out;
      o.resize(h.size());
      CK(cudaMemcpy(o.data(), d1, h.size() * sizeof(double2), cudaMemcpyDeviceToHost));
    }
    return best;
  };
  const char* names[] = {"panel_kernel<32,256>", "panel1_kernel<32>", "warp_panel_kernel", "panel_smem<16>",
                         "panel1_kernel<16>"};
  std::printf("s=%d b=%d count=%d nE=%d\n", s, b, count, nE);
  float t0 = run(0, 5, true);
  std::printf("%-22s %9.1f us\n", names[0], t0 * 1e3);
  for (int v = 1; v < 5; ++v) {
    if (v == 2 && s > 256) continue;
    if (v == 3) {
      std::printf("%-22s %9.1f us   (16-column panel reference)\n", names[3], run(3, 5, true) * 1e3);
      continue;
    }
    float tv = run(v, 5, true);
    const int ncol = v == 4 ? 16 : 32;
    // compare M panel columns, PIV
    size_t diff = 0;
    double maxrel = 0.0;
    for (int e = 0; e < nE; ++e)
      for (int i = 0; i < count; ++i) {
        const size_t o = (size_t)e * total + (size_t)i * per;
        for (int r = 0; r < s; ++r)
          for (int c = 0; c < ncol; ++c) {
            const double2 x = ref[o + (size_t)r * n + c], y = out[o + (size_t)r * n + c];
            if (std::memcmp(&x, &y, sizeof(x))) ++diff;
            const double dx = std::hypot(x.x - y.x, x.y - y.y), nx = std::hypot(x.x, x.y);
            maxrel = std::max(maxrel, dx / std::max(nx, 1e-300));
          }
        const int* p0 = reinterpret_cast<const int*>(ref.data() + o + 2 * (size_t)n * n);
        const int* p1 = reinterpret_cast<const int*>(out.data() + o + 2 * (size_t)n * n);
        for (int k = 0; k < ncol; ++k) diff += p0[k] != p1[k];
      }
    std::printf("%-22s %9.1f us  bit mismatches %zu  max rel diff %.2e\n", names[v], tv * 1e3, diff, maxrel);
  }
#ifdef FIND_PANEL_CLOCKS
  {
    CK(cudaMemcpy(d1, d0, h.size() * sizeof(double2), cudaMemcpyDeviceToDevice));
    panel1_kernel<32, 160><<<dim3(1, 1), 160>>>(P, dt);
    CK(cudaDeviceSynchronize());
    long long c[64][8];
    CK(cudaMemcpyFromSymbol(c, g_pclk, sizeof(c)));
    std::printf("one CTA (T=160), warp %d: cycles per stage [argmax, publish, barrier, xwarp, update] per column\n", PCLK_WARP);
    for (int jj = 0; jj < 32; jj += 4)
      std::printf("col %2d: %5lld %5lld %5lld %5lld %5lld  | col total %lld\n", jj, c[jj][1] - c[jj][0], c[jj][2] - c[jj][1],
                  c[jj][3] - c[jj][2], c[jj][4] - c[jj][3], c[jj][5] - c[jj][4], c[jj + 1][0] - c[jj][0]);
  }
#endif
  return 0;
}
