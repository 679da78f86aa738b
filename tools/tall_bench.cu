// Tall-panel microbenchmark: the one-CTA tall panel kernel against the register-row cluster
// kernel on identical random panels (bit-for-bit check), time per launch for `count` x `nE`
// concurrent panels of `s` rows, and (with -DFIND_PANEL_CLOCKS) the per-column cycle breakdown
// of one CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include [-DFIND_PANEL_CLOCKS] \
//        tools/tall_bench.cu -o tools/tall_bench && tools/tall_bench [s] [b] [count] [nE]
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
  const int s = argc > 1 ? std::atoi(argv[1]) : 1026;
  const int b = argc > 2 ? std::atoi(argv[2]) : 4;
  const int count = argc > 3 ? std::atoi(argv[3]) : 32;
  const int nE = argc > 4 ? std::atoi(argv[4]) : 4;
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
  const int rpt = s <= kTallMaxT ? 1 : (s <= 2 * kTallMaxT ? 2 : 3);
  const int T = 32 * (((s + rpt - 1) / rpt + 31) / 32);
  auto run = [&](int variant, int reps, std::vector<double2>* keep) -> float {
    cudaEvent_t a, z;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&z));
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
      CK(cudaMemcpy(d1, d0, h.size() * sizeof(double2), cudaMemcpyDeviceToDevice));
      CK(cudaEventRecord(a));
      if (variant == 0) {
        const unsigned cs = (unsigned)((s + kRegClusterRows - 1) / kRegClusterRows);
        const int rows = (s + (int)cs - 1) / (int)cs;
        const dim3 cg(count * cs, (unsigned)nE);
        switch ((rows + 31) / 32) {
          case 1: launch_cluster(panel_cluster_reg_kernel<32>, cg, 32, cs, 0, 0, P, dt); break;
          case 2: launch_cluster(panel_cluster_reg_kernel<64>, cg, 64, cs, 0, 0, P, dt); break;
          case 3: launch_cluster(panel_cluster_reg_kernel<96>, cg, 96, cs, 0, 0, P, dt); break;
          case 4: launch_cluster(panel_cluster_reg_kernel<128>, cg, 128, cs, 0, 0, P, dt); break;
          case 5: launch_cluster(panel_cluster_reg_kernel<160>, cg, 160, cs, 0, 0, P, dt); break;
          case 6: launch_cluster(panel_cluster_reg_kernel<192>, cg, 192, cs, 0, 0, P, dt); break;
          case 7: launch_cluster(panel_cluster_reg_kernel<224>, cg, 224, cs, 0, 0, P, dt); break;
          default: launch_cluster(panel_cluster_reg_kernel<256>, cg, 256, cs, 0, 0, P, dt); break;
        }
      } else {
        if (rpt == 1) panel_tall_kernel<1><<<grid, T>>>(P, dt);
        else if (rpt == 2) panel_tall_kernel<2><<<grid, T>>>(P, dt);
        else panel_tall_kernel<3><<<grid, T>>>(P, dt);
      }
      CK(cudaEventRecord(z));
      CK(cudaEventSynchronize(z));
      CK(cudaGetLastError());
      float ms;
      CK(cudaEventElapsedTime(&ms, a, z));
      best = std::min(best, ms);
    }
    if (keep) {
      keep->resize(h.size());
      CK(cudaMemcpy(keep->data(), d1, h.size() * sizeof(double2), cudaMemcpyDeviceToHost));
    }
    return best;
  };
  std::printf("s=%d b=%d count=%d nE=%d  (tall: %d rows/thread, %d threads)\n", s, b, count, nE, rpt, T);
  const float t0 = run(0, 5, &ref), t1 = run(1, 5, &out);
  size_t diff = 0;
  for (int e = 0; e < nE; ++e)
    for (int i = 0; i < count; ++i) {
      const size_t o = (size_t)e * total + (size_t)i * per;
      for (int r = 0; r < s; ++r)
        for (int c = 0; c < 32; ++c) diff += std::memcmp(&ref[o + (size_t)r * n + c], &out[o + (size_t)r * n + c], 16) != 0;
      const int* p0 = reinterpret_cast<const int*>(ref.data() + o + 2 * (size_t)n * n);
      const int* p1 = reinterpret_cast<const int*>(out.data() + o + 2 * (size_t)n * n);
      for (int k = 0; k < 32; ++k) diff += p0[k] != p1[k];
    }
  std::printf("cluster register rows %9.1f us\none-CTA tall          %9.1f us   bit mismatches %zu\n", t0 * 1e3, t1 * 1e3, diff);
#ifdef FIND_PANEL_CLOCKS
  {
    CK(cudaMemcpy(d1, d0, h.size() * sizeof(double2), cudaMemcpyDeviceToDevice));
    if (rpt == 1) panel_tall_kernel<1><<<dim3(1, 1), T>>>(P, dt);
    else if (rpt == 2) panel_tall_kernel<2><<<dim3(1, 1), T>>>(P, dt);
    else panel_tall_kernel<3><<<dim3(1, 1), T>>>(P, dt);
    CK(cudaDeviceSynchronize());
    long long c[64][8];
    CK(cudaMemcpyFromSymbol(c, g_pclk, sizeof(c)));
    std::printf("one CTA, warp %d: cycles [argmax, barrier1, pick+publish, barrier2, update->next col] per column;"
                " rest phase [stage+load, solve, apply]\n", PCLK_WARP);
    for (int jj = 0; jj < 32; ++jj) {
      std::printf("col %2d: %5lld %5lld %5lld %5lld %5lld", jj, c[jj][1] - c[jj][0], c[jj][2] - c[jj][1], c[jj][3] - c[jj][2],
                  c[jj][4] - c[jj][3], (jj + 1 < 32 && (jj & 7) != 7 ? c[jj + 1][0] : c[jj][5]) - c[jj][4]);
      if ((jj & 7) == 7 && jj < 31)
        std::printf("   rest: %6lld (to solve done %6lld) apply %6lld", c[jj][6] - c[jj][5], c[jj][6] - c[jj][5],
                    c[jj][7] - c[jj][6]);
      std::printf("\n");
    }
    std::printf("panel total %lld cycles\n", c[31][5] - c[0][0]);
  }
#endif
  return 0;
}
