// B200 (sm_100a) device path of the FIND selected inversion.
//
// One launch per (tree level, size class), batched over every elimination of
// the level and every energy point (grid.y).  Each elimination is one merge +
// Schur/Sigma update (solver.py:188-232 -> kernels.py:363-392):
//
//   gather  M  = merged A in [S_l, S_r, B_l, B_r] order      (solver.py:97-132)
//   partial LU of M, pivoting only among the S rows:
//       M[:s,:s] = L11\U11, M[s:,:s] = Y = A(B,S) U11^-1, M[s:,s:] = U (Schur)
//       -> exactly the reference's s^3/3 + s^2 b + s b^2 (kernels.py:90)
//   X = Y L11^-1            (L = A(B,S) A(S,S)^-1 = X P)
//   gather  MS = merged Sigma with the S rows/cols permuted by P
//   T = MS[s:,:] - X MS[:s,:];  R = T[:,s:] - T[:,:s] X^H     (kernels.py:383-392)
//   store U, R re-sorted to ascending B labels (solver.py:234-243)
//   final leaf step: G = U_f^-1, G^< = G R_f G^H, diag harvest (solver.py:383-389, 644-669)
//
// Two paths:
//   * small  (s+b <= 32): one warp per elimination, everything in shared memory.
//   * blocked (s+b > 32): one CTA per elimination, matrices in a global (L2-
//     resident) workspace; panel LU in shared memory with CTA-wide argmax
//     pivot search; all O(n^3) work as FP64 tensor-core tiles (mma.sync
//     m8n8k4 f64 -> SASS DMMA.8x8x4; B200 has no tcgen05 f64 kind).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <type_traits>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <vector>

#include "../../include/find_b200.h"
#include "dmma_engine.cuh"
#include "plan.h"
#include "tmap_host.h"

using namespace findb200;

int64_t find_scratch_elems(int64_t n, int64_t s, int nb);
void find_build_tasks(find_plan* P);

namespace {

// ------------------------------------------------------------------ complex
__device__ __forceinline__ double2 cz() { return make_double2(0.0, 0.0); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// acc - a*b
__device__ __forceinline__ double2 cfms(double2 acc, double2 a, double2 b) {
  acc.x = fma(-a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(-a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
  return acc;
}
// acc + a*b
__device__ __forceinline__ double2 cfma(double2 acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double cabs1(double2 a) { return fabs(a.x) + fabs(a.y); }  // LAPACK izamax metric
// Programmatic dependent launch: let the next kernel of the stream be scheduled
// now (its CTAs only take resources this grid has left), then wait until the
// previous kernel of the stream has completed and its writes are visible.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
// 1 / a as conj(a) / |a|^2: one reciprocal (pivots are far from the overflow / underflow range
// of |a|^2; tiny pivots are rejected by the pivot test anyway)
__device__ __forceinline__ double2 crcp(double2 a) {
  const double r = 1.0 / fma(a.x, a.x, a.y * a.y);
  return make_double2(a.x * r, -a.y * r);
}
__device__ __forceinline__ double cabs(double2 a) { return hypot(a.x, a.y); }
__device__ __forceinline__ double2 cinv(double2 a) {  // Smith's algorithm
  if (a.x == 0.0 && a.y == 0.0) return cz();
  if (fabs(a.x) >= fabs(a.y)) {
    double r = a.y / a.x, d = a.x + a.y * r;
    return make_double2(1.0 / d, -r / d);
  }
  double r = a.x / a.y, d = a.y + a.x * r;
  return make_double2(r / d, -1.0 / d);
}


// ------------------------------------------------------------------ params
struct SolveParams {
  const ElimDesc* elims;
  const int32_t* i32;
  const SparseEntry* sparse;
  const double2* a_vals;  // [nE][nnz]
  const double2* s_vals;  // [nnz] or [nE][nnz]
  int64_t nnz;
  int32_t s_broadcast;
  int32_t compute_gless;
  int32_t rsym;  // 0 general; +1 Sigma (hence every R) Hermitian; -1 skew-Hermitian
  double rtol;
  double2* arena[kNumArenas];
  int64_t arena_elems[kNumArenas];
  double2* scratch;
  int64_t scratch_elems;
  double2* gr_out;  // [nE][n]
  double2* gl_out;
  int64_t n_nodes;
  unsigned long long* status;  // first failing (elim << 32 | energy << 16 | pos)
  int64_t elim_base;           // global index of elims[0] in the plan
  double2* dbg_l;              // unit-test shim only: L = A(B,S) A(S,S)^-1 (b x s), elimination 0 / energy 0
  // off-diagonal extraction (find_solve_offdiag): [nE][n_pairs] outputs, items per final elimination
  double2* off_gr;
  double2* off_gl;
  const OffItem* off_items;
  const int64_t* off_item_off;
  int64_t n_pairs;
  int32_t off_sym;  // +1 / -1: Sigma^< exactly Hermitian / skew-Hermitian (then G^< is too), 0 general
  int32_t zskip;    // skip the products of structurally zero (B_r, S_l) blocks (ElimDesc::zsplit)
  int32_t use_tma;  // DMMA tiles of trail / Schur / T / R through the TMA engine (tmaps valid)
  unsigned long long* tile_ctr;  // one tile counter per launch spec (TMA engine's dynamic tile order)
  const CUtensorMap* tmaps;  // [n_tmap][3]: M, MS, X of each CTA-path elimination (ElimDesc::tmap)
};

__device__ __forceinline__ void report_bad(const SolveParams& P, int64_t elim_global, int e, int pos) {
  unsigned long long key = ((unsigned long long)elim_global << 32) | ((unsigned long long)(e & 0xffff) << 16) |
                           (unsigned long long)min(pos, 0xffff);
  atomicMin(P.status, key);
}

__device__ __forceinline__ double2 ldg2(const double2* p) { return __ldg(p); }

// value of merged entry (i, j) that comes from a stored child block (or zero);
// CSR-sourced entries are scattered afterwards from the sparse list.
__device__ __forceinline__ double2 block_entry(const ElimDesc& d, const double2* lblk, const double2* rblk, int si,
                                               int sj) {
  const bool li = si < d.p, lj = sj < d.p;
  if (li && lj) return lblk ? lblk[(int64_t)si * d.p + sj] : cz();
  if (!li && !lj) {
    const int q = d.n - d.p;
    return rblk ? rblk[(int64_t)(si - d.p) * q + (sj - d.p)] : cz();
  }
  return cz();
}

// ================================================================== small path
// One warp per (elimination, energy); merged size n <= 32.
constexpr int kSmallWarps = 1;

__device__ void warp_gj_inverse(double2* a, int lda, int c, int lane, bool* singular) {
  // In-place Gauss-Jordan inversion with partial pivoting (row interchanges),
  // lane = column.  Mirrors np.linalg.inv (solver.py:385) up to roundoff.
  int ip[32];
  for (int k = 0; k < c; ++k) {
    double best = -1.0;
    int bi = k;
    for (int i = k; i < c; ++i) {
      double v = cabs1(a[i * lda + k]);
      if (v > best) { best = v; bi = i; }
    }
    ip[k] = bi;
    if (best == 0.0) *singular = true;
    __syncwarp();
    if (bi != k && lane < c) {
      double2 t = a[k * lda + lane];
      a[k * lda + lane] = a[bi * lda + lane];
      a[bi * lda + lane] = t;
    }
    __syncwarp();
    double2 pivinv = cinv(a[k * lda + k]);
    __syncwarp();
    if (lane < c) {
      double2 v = (lane == k) ? make_double2(1.0, 0.0) : a[k * lda + lane];
      a[k * lda + lane] = cmul(v, pivinv);
    }
    __syncwarp();
    for (int i = 0; i < c; ++i) {
      if (i == k) continue;
      double2 f = a[i * lda + k];
      __syncwarp();
      if (lane < c) {
        double2 v = (lane == k) ? cz() : a[i * lda + lane];
        a[i * lda + lane] = cfms(v, f, a[k * lda + lane]);
      }
      __syncwarp();
    }
  }
  for (int k = c - 1; k >= 0; --k) {
    if (ip[k] != k && lane < c) {
      double2 t = a[lane * lda + k];
      a[lane * lda + k] = a[lane * lda + ip[k]];
      a[lane * lda + ip[k]] = t;
    }
    __syncwarp();
  }
}

// Final leaf epilogue on one warp: U_f, R_f (c x c, in shared memory, ld),
// writes diag(G^r), diag(G^<) at the leaf's mesh nodes.
__device__ void final_epilogue_warp(const SolveParams& P, const ElimDesc& d, int64_t elim_global, int e, double2* uf,
                                    int ldu, const double2* rf, int ldr, int lane) {
  const int c = d.b;
  bool singular = false;
  warp_gj_inverse(uf, ldu, c, lane, &singular);
  if (singular) {
    if (lane == 0) report_bad(P, elim_global, e, 0xfffe);
    return;
  }
  const int32_t* nodes = P.i32 + d.rank_off;
  if (lane < c) {
    const int64_t node = nodes[lane];
    P.gr_out[(int64_t)e * P.n_nodes + node] = uf[lane * ldu + lane];
    if (P.compute_gless) {
      // (G R G^H)_ii = sum_a G_ia sum_b R_ab conj(G_ib)
      double2 acc = cz();
      for (int a = 0; a < c; ++a) {
        double2 t = cz();
        for (int b = 0; b < c; ++b) t = cfma(t, rf[a * ldr + b], cconj(uf[lane * ldu + b]));
        acc = cfma(acc, uf[lane * ldu + a], t);
      }
      P.gl_out[(int64_t)e * P.n_nodes + node] = acc;
    }
  }
}

// Per-warp shared memory (complex elements): M [nmax][ld] (A, later Sigma),
// XC [xcap] (X = Y L11^-1, and U_f for final steps), 3 x 32 ints.
__host__ __device__ constexpr int small_warp_elems(int nmax, int ld, int xcap) { return nmax * ld + xcap + 24; }

__global__ void __launch_bounds__(kSmallWarps * 32) small_elim_kernel(SolveParams P, int64_t count, int nmax, int ld,
                                                                      int xcap) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t idx = (int64_t)blockIdx.x * kSmallWarps + warp;
  if (idx >= count) return;
  const int e = blockIdx.y;
  const ElimDesc d = P.elims[idx];
  const int64_t elim_global = P.elim_base + idx;
  const int n = d.n, s = d.s, b = d.b;
  double2* MA = reinterpret_cast<double2*>(smem_raw) + (size_t)warp * small_warp_elems(nmax, ld, xcap);
  double2* XC = MA + nmax * ld;
  int* piv = reinterpret_cast<int*>(XC + xcap);  // piv, sig, isg: 3 x 32 ints
  int* sig = piv + 32;
  int* isg = sig + 32;
  const int32_t* map = P.i32 + d.map_off;
  const int32_t* rank = P.i32 + d.rank_off;
  const double2* lblk = d.left_arena >= 0 ? P.arena[d.left_arena] + (int64_t)e * P.arena_elems[d.left_arena] + d.left_off : nullptr;
  const double2* rblk = d.right_arena >= 0 ? P.arena[d.right_arena] + (int64_t)e * P.arena_elems[d.right_arena] + d.right_off : nullptr;
  const double2* av = P.a_vals + (int64_t)e * P.nnz;
  const SparseEntry* sp = P.sparse + d.sparse_off;

  // ---- gather A (solver.py:203-205) ----
  const int mj = lane < n ? map[lane] : 0;
  for (int i = 0; i < n; ++i) {
    const int mi = map[i];
    if (lane < n) MA[i * ld + lane] = block_entry(d, lblk, rblk, mi, mj);
  }
  __syncwarp();
  for (int t = lane; t < d.nsparse; t += 32) {
    const SparseEntry en = sp[t];
    MA[en.i * ld + en.j] = ldg2(av + en.csr);
  }
  __syncwarp();

  // ---- partial LU, pivoting among S rows (kernels.py:237-252, 376); lane = row ----
  double scale = 0.0;
  if (lane < s)
    for (int j = 0; j < s; ++j) scale = fmax(scale, cabs(MA[lane * ld + j]));
  for (int o = 16; o; o >>= 1) scale = fmax(scale, __shfl_xor_sync(0xffffffffu, scale, o));
  int bad = (s > 0 && scale == 0.0) ? 0 : INT32_MAX;
  for (int k = 0; k < s; ++k) {
    double v = (lane >= k && lane < s) ? cabs1(MA[lane * ld + k]) : -1.0;
    int vi = lane;
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int oi = __shfl_xor_sync(0xffffffffu, vi, o);
      if (ov > v || (ov == v && oi < vi)) { v = ov; vi = oi; }
    }
    const int pr = [&] { const int q = __shfl_sync(0xffffffffu, vi, 0); return q >= k && q < s ? q : k; }();
    if (lane == 0) piv[k] = pr;
    if (pr != k && lane < n) {  // lane = column for the interchange
      const double2 tmp = MA[k * ld + lane];
      MA[k * ld + lane] = MA[pr * ld + lane];
      MA[pr * ld + lane] = tmp;
    }
    __syncwarp();
    const double2 ukk = MA[k * ld + k];
    if (cabs(ukk) < P.rtol * scale && bad == INT32_MAX) bad = k;
    const double2 uinv = cinv(ukk);
    if (lane > k && lane < n) {  // lane = row: multiplier and rank-1 update of its own row
      double2* rw = MA + lane * ld;
      const double2 l = cmul(rw[k], uinv);
      rw[k] = l;
      for (int j = k + 1; j < n; ++j) rw[j] = cfms(rw[j], l, MA[k * ld + j]);
    }
    __syncwarp();
  }
  if (bad != INT32_MAX && lane == 0) report_bad(P, elim_global, e, bad);

  // ---- X = Y L11^-1 (row per lane), stashed in XC [b][s] ----
  if (lane < b) {
    double2* rw = MA + (s + lane) * ld;
    for (int k = s - 1; k >= 0; --k) {
      double2 acc = rw[k];
      for (int m = k + 1; m < s; ++m) acc = cfms(acc, rw[m], MA[m * ld + k]);
      rw[k] = acc;
    }
    for (int k = 0; k < s; ++k) XC[lane * s + k] = rw[k];
  }
  // permutation sigma from the pivot sequence: pivoted row k = merged row sig[k]
  if (lane == 0) {
    for (int k = 0; k < s; ++k) sig[k] = k;
    for (int k = 0; k < s; ++k) { const int tmp = sig[k]; sig[k] = sig[piv[k]]; sig[piv[k]] = tmp; }
  }
  __syncwarp();
  if (P.dbg_l && idx == 0 && e == 0 && lane < b)
    for (int k = 0; k < s; ++k) P.dbg_l[(int64_t)lane * s + sig[k]] = XC[lane * s + k];
  double2* UF = XC + b * s;  // final step: U_f kept for the epilogue
  if (d.kind == kFinal) {
    if (lane < b)
      for (int j = 0; j < b; ++j) UF[lane * b + j] = MA[(s + lane) * ld + s + j];
  } else if (d.out_arena >= 0) {  // store U sorted (solver.py:234-243)
    double2* out = P.arena[d.out_arena] + (int64_t)e * P.arena_elems[d.out_arena] + d.out_off;
    const int rj = lane < b ? rank[lane] : 0;
    for (int i = 0; i < b; ++i)
      if (lane < b) out[(int64_t)rank[i] * b + rj] = MA[(s + i) * ld + s + lane];
  }
  __syncwarp();
  double2* MS = MA;  // Sigma reuses the A buffer
  if (P.compute_gless) {
    const double2* lr = lblk ? lblk + (int64_t)d.p * d.p : nullptr;
    const int q = n - d.p;
    const double2* rr = rblk ? rblk + (int64_t)q * q : nullptr;
    const double2* sv = P.s_vals + (P.s_broadcast ? 0 : (int64_t)e * P.nnz);
    if (lane < n && lane >= s) isg[lane] = lane;
    if (lane < s) isg[sig[lane]] = lane;
    __syncwarp();
    const int pj = lane < n ? map[lane < s ? sig[lane] : lane] : 0;
    for (int i = 0; i < n; ++i) {
      const int pi = map[i < s ? sig[i] : i];
      if (lane < n) MS[i * ld + lane] = block_entry(d, lr, rr, pi, pj);
    }
    __syncwarp();
    for (int t = lane; t < d.nsparse; t += 32) {
      const SparseEntry en = sp[t];
      MS[isg[en.i] * ld + isg[en.j]] = ldg2(sv + en.csr);
    }
    __syncwarp();
    // T = MS[s:,:] - X MS[:s,:]  (lane = column)
    if (lane < n)
      for (int i = 0; i < b; ++i) {
        double2 acc = MS[(s + i) * ld + lane];
        for (int k = 0; k < s; ++k) acc = cfms(acc, XC[i * s + k], MS[k * ld + lane]);
        MS[(s + i) * ld + lane] = acc;
      }
    __syncwarp();
    // R = T[:, s:] - T[:, :s] X^H  (lane = column j < b)
    if (lane < b)
      for (int i = 0; i < b; ++i) {
        double2 acc = MS[(s + i) * ld + s + lane];
        for (int k = 0; k < s; ++k) acc = cfms(acc, MS[(s + i) * ld + k], cconj(XC[lane * s + k]));
        MS[(s + i) * ld + s + lane] = acc;
      }
    __syncwarp();
    if (d.kind != kFinal && d.out_arena >= 0) {
      double2* out = P.arena[d.out_arena] + (int64_t)e * P.arena_elems[d.out_arena] + d.out_off + (int64_t)b * b;
      const int rj = lane < b ? rank[lane] : 0;
      for (int i = 0; i < b; ++i)
        if (lane < b) out[(int64_t)rank[i] * b + rj] = MS[(s + i) * ld + s + lane];
    }
  }
  if (d.kind == kFinal) {
    __syncwarp();
    final_epilogue_warp(P, d, elim_global, e, UF, b, MS + s * ld + s, ld, lane);
  }
}

// ================================================================== CTA path: phase launches
// Every phase of the blocked elimination is one launch over a flattened task
// list covering all eliminations of the level and (grid.y) all energy points,
// so the trailing updates and the T / R products of a level spread over all
// 148 SMs and many CTAs per SM hide the latency of the sequential panel steps.
constexpr int kThreads = 256;
constexpr int kKC = 16, kSK = kKC + 4;  // K chunk; smem row stride 20 complex = 320 B (conflict-free frags)

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int NT = 256>
__device__ void block_argmax(double& v, int& vi, double* cv, int* ci) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, v, o);
    int oi = __shfl_xor_sync(0xffffffffu, vi, o);
    if (ov > v || (ov == v && oi < vi)) { v = ov; vi = oi; }
  }
  if (lane == 0) { cv[warp] = v; ci[warp] = vi; }
  __syncthreads();
  v = cv[0]; vi = ci[0];
#pragma unroll
  for (int w = 1; w < NT / 32; ++w) {
    double ov = cv[w];
    int oi = ci[w];
    if (ov > v || (ov == v && oi < vi)) { v = ov; vi = oi; }
  }
}

// ================================================================== mid path
// One 128-thread CTA per (elimination, energy) for 32 < s+b <= 64: the merged
// matrix, LU, X and the U / R products all in shared memory (the warp path's
// algorithm, CTA-wide).
constexpr int kMidThreads = 128;
constexpr int kMidMaxN = 64;
// M [nmax][nmax+1], XC [xcap], then piv / sig / isg (3 x 64 ints); sized tightly (occupancy
// of the mid path is set by this shared-memory footprint)
__host__ __device__ constexpr int mid_smem_elems(int nmax, int xcap) { return nmax * (nmax + 1) + xcap + 3 * kMidMaxN / 4; }

template <int NT>
__device__ __forceinline__ void block_max(double& v, double* cv) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) cv[warp] = v;
  __syncthreads();
  v = cv[0];
  for (int w = 1; w < NT / 32; ++w) v = fmax(v, cv[w]);
  __syncthreads();
}

__global__ void __launch_bounds__(kMidThreads) mid_elim_kernel(SolveParams P, int64_t count, int nmax, int xcap) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int NT = kMidThreads;
  __shared__ double cv[2][NT / 32];
  __shared__ int ci[2][NT / 32];
  __shared__ double2 s_uinv;
  __shared__ int s_bad;
  const int tid = threadIdx.x;
  const int64_t idx = blockIdx.x;
  const int e = blockIdx.y;
  const ElimDesc d = P.elims[idx];
  const int64_t elim_global = P.elim_base + idx;
  const int n = d.n, s = d.s, b = d.b;
  const int ld = nmax + 1;
  double2* MA = reinterpret_cast<double2*>(smem_raw);
  double2* XC = MA + nmax * ld;
  int* piv = reinterpret_cast<int*>(XC + xcap);
  int* sig = piv + kMidMaxN;
  int* isg = sig + kMidMaxN;
  const int32_t* map = P.i32 + d.map_off;
  const int32_t* rank = P.i32 + d.rank_off;
  const double2* lblk = d.left_arena >= 0 ? P.arena[d.left_arena] + (int64_t)e * P.arena_elems[d.left_arena] + d.left_off : nullptr;
  const double2* rblk = d.right_arena >= 0 ? P.arena[d.right_arena] + (int64_t)e * P.arena_elems[d.right_arena] + d.right_off : nullptr;
  const double2* av = P.a_vals + (int64_t)e * P.nnz;
  const SparseEntry* sp = P.sparse + d.sparse_off;
  if (tid == 0) s_bad = INT32_MAX;

  // ---- gather A ----
  for (int q = tid; q < n * n; q += NT) {
    const int i = q / n, j = q % n;
    MA[i * ld + j] = block_entry(d, lblk, rblk, map[i], map[j]);
  }
  __syncthreads();
  for (int q = tid; q < d.nsparse; q += NT) {
    const SparseEntry en = sp[q];
    MA[en.i * ld + en.j] = ldg2(av + en.csr);
  }
  __syncthreads();
  double scale = 0.0;
  for (int q = tid; q < s * s; q += NT) scale = fmax(scale, cabs(MA[(q / s) * ld + q % s]));
  block_max<NT>(scale, cv[0]);
  if (tid == 0 && s > 0 && scale == 0.0) s_bad = 0;

  // ---- partial LU, pivot search among the S rows ----
  for (int k = 0; k < s; ++k) {
    double v = -1.0;
    int vi = INT32_MAX;
    for (int r = k + tid; r < s; r += NT) {
      const double a = cabs1(MA[r * ld + k]);
      if (a > v) { v = a; vi = r; }
    }
    block_argmax<NT>(v, vi, cv[k & 1], ci[k & 1]);
    const int pr = vi >= k && vi < s ? vi : k;  // NaN / Inf entries: no interchange
    if (tid == 0) {
      piv[k] = pr;
      const double2 u = MA[pr * ld + k];
      s_uinv = cinv(u);
      if (cabs(u) < P.rtol * scale) atomicMin(&s_bad, k);
    }
    if (pr != k)
      for (int c = tid; c < n; c += NT) {
        const double2 tmp = MA[k * ld + c];
        MA[k * ld + c] = MA[pr * ld + c];
        MA[pr * ld + c] = tmp;
      }
    __syncthreads();
    const double2 uinv = s_uinv;
    const int rows = n - k - 1;
    {  // multiplier and rank-1 update: warp = row (stride 4), lane = column (rows <= 63: two columns
       // per lane); every lane forms its row's multiplier from the broadcast column-k entry
      const int warp = tid >> 5, lane = tid & 31;
      const double2* pr_row = MA + k * ld + k + 1;
      const double2 u0 = lane < rows ? pr_row[lane] : cz();
      const double2 u1 = lane + 32 < rows ? pr_row[lane + 32] : cz();
      for (int r = warp; r < rows; r += NT / 32) {
        double2* row = MA + (k + 1 + r) * ld + k + 1;
        const double2 l = cmul(row[-1], uinv);
        __syncwarp();
        if (lane == 0) row[-1] = l;
        if (lane < rows) row[lane] = cfms(row[lane], l, u0);
        if (lane + 32 < rows) row[lane + 32] = cfms(row[lane + 32], l, u1);
      }
    }
    __syncthreads();
  }
  if (tid == 0 && s_bad != INT32_MAX) report_bad(P, elim_global, e, s_bad);

  // ---- X = Y L11^-1 -> XC [b][s]: warp per B row, lane = column (s <= 63: two per lane);
  // column-oriented back substitution, x_k broadcast by shuffle from its owner lane
  {
    const int warp = tid >> 5, lane = tid & 31;
    for (int i = warp; i < b; i += NT / 32) {
      const double2* rw = MA + (s + i) * ld;
      double2 x0 = lane < s ? rw[lane] : cz();
      double2 x1 = lane + 32 < s ? rw[lane + 32] : cz();
      for (int k = s - 1; k >= 0; --k) {
        const double2 own = k < 32 ? x0 : x1;
        const double2 xk = make_double2(__shfl_sync(0xffffffffu, own.x, k & 31), __shfl_sync(0xffffffffu, own.y, k & 31));
        const double2* lk = MA + k * ld;  // L11[k][m], m < k
        if (lane < k) x0 = cfms(x0, xk, lk[lane]);
        if (lane + 32 < k) x1 = cfms(x1, xk, lk[lane + 32]);
      }
      if (lane < s) XC[i * s + lane] = x0;
      if (lane + 32 < s) XC[i * s + lane + 32] = x1;
    }
  }
  if (tid == 0) {
    for (int k = 0; k < s; ++k) sig[k] = k;
    for (int k = 0; k < s; ++k) { const int tmp = sig[k]; sig[k] = sig[piv[k]]; sig[piv[k]] = tmp; }
  }
  __syncthreads();
  if (P.dbg_l && idx == 0 && e == 0)
    for (int q = tid; q < b * s; q += NT) P.dbg_l[(int64_t)(q / s) * s + sig[q % s]] = XC[q];
  double2* UF = XC + b * s;
  if (d.kind == kFinal) {
    for (int q = tid; q < b * b; q += NT) UF[q] = MA[(s + q / b) * ld + s + q % b];
  } else if (d.out_arena >= 0) {
    double2* out = P.arena[d.out_arena] + (int64_t)e * P.arena_elems[d.out_arena] + d.out_off;
    for (int q = tid; q < b * b; q += NT) {
      const int i = q / b, j = q % b;
      out[(int64_t)rank[i] * b + rank[j]] = MA[(s + i) * ld + s + j];
    }
  }
  __syncthreads();
  double2* MS = MA;
  if (P.compute_gless) {
    const double2* lr = lblk ? lblk + (int64_t)d.p * d.p : nullptr;
    const int q0 = n - d.p;
    const double2* rr = rblk ? rblk + (int64_t)q0 * q0 : nullptr;
    const double2* sv = P.s_vals + (P.s_broadcast ? 0 : (int64_t)e * P.nnz);
    for (int k = tid; k < n; k += NT) {
      if (k >= s) isg[k] = k;
      else isg[sig[k]] = k;
    }
    __syncthreads();
    for (int q = tid; q < n * n; q += NT) {
      const int i = q / n, j = q % n;
      MS[i * ld + j] = block_entry(d, lr, rr, map[i < s ? sig[i] : i], map[j < s ? sig[j] : j]);
    }
    __syncthreads();
    for (int q = tid; q < d.nsparse; q += NT) {
      const SparseEntry en = sp[q];
      MS[isg[en.i] * ld + isg[en.j]] = ldg2(sv + en.csr);
    }
    __syncthreads();
    // T_S = S'_BS - X S'_SS (two accumulators: half-length dependent chains)
    for (int q = tid; q < b * s; q += NT) {
      const int i = q / s, c = q % s;
      double2 acc = MS[(s + i) * ld + c], acc2 = cz();
      int m = 0;
      for (; m + 1 < s; m += 2) {
        acc = cfms(acc, XC[i * s + m], MS[m * ld + c]);
        acc2 = cfma(acc2, XC[i * s + m + 1], MS[(m + 1) * ld + c]);
      }
      if (m < s) acc = cfms(acc, XC[i * s + m], MS[m * ld + c]);
      MS[(s + i) * ld + c] = csub(acc, acc2);
    }
    __syncthreads();
    // R = S'_BB - X S'_SB - T_S X^H
    const bool store = d.kind != kFinal && d.out_arena >= 0;
    const bool mirror = store && P.rsym != 0;
    const double sgn = P.rsym < 0 ? -1.0 : 1.0;
    double2* out = store ? P.arena[d.out_arena] + (int64_t)e * P.arena_elems[d.out_arena] + d.out_off + (int64_t)b * b
                         : nullptr;
    for (int q = tid; q < b * b; q += NT) {
      const int i = q / b, j = q % b;
      if (mirror && j > i) continue;
      double2 acc = MS[(s + i) * ld + s + j], acc2 = cz();
      for (int m = 0; m < s; ++m) {
        acc = cfms(acc, XC[i * s + m], MS[m * ld + s + j]);
        acc2 = cfma(acc2, MS[(s + i) * ld + m], cconj(XC[j * s + m]));
      }
      acc = csub(acc, acc2);
      if (!store) {
        MS[(s + i) * ld + s + j] = acc;
      } else {
        out[(int64_t)rank[i] * b + rank[j]] = acc;
        if (mirror && i != j) out[(int64_t)rank[j] * b + rank[i]] = make_double2(sgn * acc.x, -sgn * acc.y);
      }
    }
    __syncthreads();
  }
  if (d.kind == kFinal && tid < 32) final_epilogue_warp(P, d, elim_global, e, UF, b, MS + s * ld + s, ld, tid);
}

struct Scr {
  double2* M;   // merged A, then L\U, Y/X, U               [n][n]
  double2* MS;  // merged, pivot-permuted Sigma, then T, R  [n][n]
  int* PIV;     // pivot rows (global S index)              [s]
  int* SIG;     // pivoted position -> merged position      [s]
  int* ISG;     // merged position -> pivoted position      [s]
  int* PERM;    // current panel's net row interchange: {nd, src[64], dst[64]}
  int* PERM2;   // the first panel's PERM of a wide (two-panel) block, saved for the wide TRSM
  double* scale;
  double* pmax;   // per gather row chunk: max |A(S,S)| over its rows   [ceil(n/kRowChunk)]
  double2* LINV;  // per panel j: L_jj^-1  [NB][NB]   (valid when nb > 0)
  double2* UINV;  // per panel j: U_jj^-1  [NB][NB]
  double2* X;     // X = Y L11^-1   [b][s]            (valid when nb > 0)
};
// Layout must match find_scratch_elems() in plan.cpp.
__device__ __forceinline__ Scr scratch_of(const SolveParams& P, const ElimDesc& d, int e, int nb = 0) {
  Scr r;
  r.M = P.scratch + (int64_t)e * P.scratch_elems + d.ws_off;
  const int64_t nn = (int64_t)d.n * d.n;
  r.MS = r.M + nn;
  r.PIV = reinterpret_cast<int*>(r.M + 2 * nn);
  r.SIG = r.PIV + d.s;
  r.ISG = r.SIG + d.s;
  r.PERM = r.ISG + d.s;
  r.PERM2 = r.PERM + 132;
  const int64_t ints = (3 * d.s + 264 + 3) / 4;
  r.scale = reinterpret_cast<double*>(r.M + 2 * nn + ints);
  r.pmax = r.scale + 2;
  r.LINV = r.M + 2 * nn + ints + 1 + (d.n + 2 * kRowChunk - 1) / (2 * kRowChunk);
  r.UINV = nb ? r.LINV + (int64_t)((d.s + nb - 1) / nb) * nb * nb : r.LINV;
  r.X = nb ? r.UINV + (int64_t)((d.s + nb - 1) / nb) * nb * nb : r.LINV;
  return r;
}

// One DMMA output tile: acc[BM x BN] = A[BM x K] * op(B)[K x BN], operands
// streamed global -> shared memory with a 2-stage cp.async pipeline.
// op(B)[k][c] = B[k*ldb + c] (BT = false) or conj(B[c*ldb + k]) (BT = true).
template <int WM, int WN, int MT, int NT, bool BT>
struct Tile {
  static constexpr int BM = WM * MT * 8, BN = WN * NT * 8;
  static constexpr int STAGE = (BM + BN) * kSK;
  static constexpr size_t SMEM = 2 * STAGE * sizeof(double2);
  double acc[MT][NT][2][2];

  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int a = 0; a < MT; ++a)
#pragma unroll
      for (int c = 0; c < NT; ++c) acc[a][c][0][0] = acc[a][c][0][1] = acc[a][c][1][0] = acc[a][c][1][1] = 0.0;
  }

  template <bool BT2 = BT>
  __device__ __forceinline__ void load(const double2* A, int64_t lda, const double2* B, int64_t ldb, int Mv, int Nv,
                                       int K, int kc, double2* st) {
    const int tid = threadIdx.x;
    double2* As = st;
    double2* Bs = st + BM * kSK;
    const int k0 = kc * kKC;
#pragma unroll
    for (int q = tid; q < BM * kKC; q += kThreads) {
      const int row = q / kKC, kk = q % kKC;
      const bool ok = row < Mv && k0 + kk < K;
      cp_async16(As + row * kSK + kk, ok ? A + (int64_t)row * lda + k0 + kk : A, ok);
    }
    if (BT2) {
#pragma unroll
      for (int q = tid; q < BN * kKC; q += kThreads) {
        const int col = q / kKC, kk = q % kKC;
        const bool ok = col < Nv && k0 + kk < K;
        cp_async16(Bs + col * kSK + kk, ok ? B + (int64_t)col * ldb + k0 + kk : B, ok);
      }
    } else {
#pragma unroll
      for (int q = tid; q < BN * kKC; q += kThreads) {
        const int kk = q / BN, col = q % BN;
        const bool ok = col < Nv && k0 + kk < K;
        cp_async16(Bs + col * kSK + kk, ok ? B + (int64_t)(k0 + kk) * ldb + col : B, ok);
      }
    }
    cp_async_commit();
  }

  // acc += A op(B), or acc -= A op(B) with NEG (acc seeded by load_c: C - A op(B) tiles).
  // NS shared-memory stages (NS - 1 K chunks in flight; smem must hold NS * STAGE elements).
  template <bool BT2 = BT, bool NEG = false, int NS = 2>
  __device__ __forceinline__ void mma(const double2* A, int64_t lda, const double2* B, int64_t ldb, int Mv, int Nv,
                                      int K, double2* smem) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp % WM, wn = warp / WM;
    const int fr = lane >> 2, fc = lane & 3;
    const int nk = (K + kKC - 1) / kKC;
    if (nk <= 0) return;
    // fragments of this warp that hold valid rows / cols (warp-uniform); the
    // zero padding of partial tiles is not multiplied
    const int mtv = min(MT, max(0, (Mv - wm * MT * 8 + 7) / 8));
    const int ntv = min(NT, max(0, (Nv - wn * NT * 8 + 7) / 8));
#pragma unroll
    for (int p = 0; p < NS - 1; ++p) {
      if (p < nk) load<BT2>(A, lda, B, ldb, Mv, Nv, K, p, smem + p * STAGE);
      else cp_async_commit();
    }
    for (int kc = 0; kc < nk; ++kc) {
      // one commit group per iteration (empty past the end), so wait<NS - 1> always means "chunk kc landed"
      if (kc + NS - 1 < nk) load<BT2>(A, lda, B, ldb, Mv, Nv, K, kc + NS - 1, smem + ((kc + NS - 1) % NS) * STAGE);
      else cp_async_commit();
      cp_async_wait<NS - 1>();
      __syncthreads();
      const double2* As = smem + (kc % NS) * STAGE;
      const double2* Bs = As + BM * kSK;
      const int kv = K - kc * kKC;
      if (kv >= kKC && mtv == MT && ntv == NT) {
        // whole chunk, every fragment valid: no predicates; the two DMMAs into one accumulator
        // are MT*NT*2 instructions apart (each accumulator still sums ax*bx, -ay*by / ax*by, ay*bx
        // in this order: bit-identical to the general path below)
#pragma unroll
        for (int kk = 0; kk < kKC; kk += 4) {
          double2 a[MT], b[NT];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) a[mt] = As[(wm * MT * 8 + mt * 8 + fr) * kSK + kk + fc];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            b[nt] = Bs[(wn * NT * 8 + nt * 8 + fr) * kSK + kk + fc];
            if (BT2) b[nt].y = -b[nt].y;
          }
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const double ax = NEG ? -a[mt].x : a[mt].x;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              dmma(acc[mt][nt][0][0], acc[mt][nt][0][1], ax, b[nt].x);
              dmma(acc[mt][nt][1][0], acc[mt][nt][1][1], ax, b[nt].y);
            }
          }
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const double ay = NEG ? -a[mt].y : a[mt].y, nai = -ay;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              dmma(acc[mt][nt][0][0], acc[mt][nt][0][1], nai, b[nt].y);
              dmma(acc[mt][nt][1][0], acc[mt][nt][1][1], ay, b[nt].x);
            }
          }
        }
        __syncthreads();
        continue;
      }
#pragma unroll
      for (int kk = 0; kk < kKC; kk += 4) {
        if (kk >= kv || mtv == 0 || ntv == 0) break;
        double2 a[MT], b[NT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) a[mt] = As[(wm * MT * 8 + mt * 8 + fr) * kSK + kk + fc];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          b[nt] = Bs[(wn * NT * 8 + nt * 8 + fr) * kSK + kk + fc];
          if (BT2) b[nt].y = -b[nt].y;
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          if (mt >= mtv) break;
          const double ax = NEG ? -a[mt].x : a[mt].x, ay = NEG ? -a[mt].y : a[mt].y, nai = -ay;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            if (nt >= ntv) break;
            dmma(acc[mt][nt][0][0], acc[mt][nt][0][1], ax, b[nt].x);
            dmma(acc[mt][nt][0][0], acc[mt][nt][0][1], nai, b[nt].y);
            dmma(acc[mt][nt][1][0], acc[mt][nt][1][1], ax, b[nt].y);
            dmma(acc[mt][nt][1][0], acc[mt][nt][1][1], ay, b[nt].x);
          }
        }
      }
      __syncthreads();
    }
  }

  // acc = this thread's elements of C[Mv x Nv] (row stride ld; zero outside), loaded before the
  // K loop so the C - A op(B) epilogue only stores (the loads overlap the operand staging)
  __device__ __forceinline__ void load_c(const double2* C, int64_t ld, int Mv, int Nv) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp % WM, wn = warp / WM;
    const int fr = lane >> 2, fc = lane & 3;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int r = wm * MT * 8 + mt * 8 + fr, c = wn * NT * 8 + nt * 8 + 2 * fc + i;
          const double2 v = (r < Mv && c < Nv) ? C[(int64_t)r * ld + c] : cz();
          acc[mt][nt][0][i] = v.x;
          acc[mt][nt][1][i] = v.y;
        }
  }

  template <class F>
  __device__ __forceinline__ void for_each(F f) const {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp % WM, wn = warp / WM;
    const int fr = lane >> 2, fc = lane & 3;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int i = 0; i < 2; ++i)
          f(wm * MT * 8 + mt * 8 + fr, wn * NT * 8 + nt * 8 + 2 * fc + i,
            make_double2(acc[mt][nt][0][i], acc[mt][nt][1][i]));
  }
};
using Tile64 = Tile<2, 4, 4, 2, false>;

template <int NB>
struct XTileSel;
template <>
struct XTileSel<32> { using T = Tile<4, 2, 2, 2, false>; };
template <>
struct XTileSel<16> { using T = Tile<4, 2, 2, 1, false>; };
template <>
struct XTileSel<8> { using T = Tile<8, 1, 1, 1, false>; };
template <>
struct XTileSel<4> { using T = Tile<8, 1, 1, 1, false>; };

__device__ __forceinline__ const double2* child_block(const SolveParams& P, const ElimDesc& d, int e, bool left,
                                                      bool sigma) {
  const int a = left ? d.left_arena : d.right_arena;
  if (a < 0) return nullptr;
  const int sz = left ? d.p : d.n - d.p;
  const double2* base = P.arena[a] + (int64_t)e * P.arena_elems[a] + (left ? d.left_off : d.right_off);
  return sigma ? base + (int64_t)sz * sz : base;
}

// ---- merged A / pivot-permuted Sigma into scratch (solver.py:97-132, 203-205, 227-228)
template <bool SIGMA>
__device__ void gather_body(const SolveParams& P, const Task& t, int e) {
  const ElimDesc d = P.elims[t.e];
  const int n = d.n, s = d.s;
  const Scr S = scratch_of(P, d, e);
  double2* dst = SIGMA ? S.MS : S.M;
  const int32_t* map = P.i32 + d.map_off;
  const int32_t* rowoff = P.i32 + d.sprow_off;
  const double2* lb = child_block(P, d, e, true, SIGMA);
  const double2* rb = child_block(P, d, e, false, SIGMA);
  const double2* vals = SIGMA ? P.s_vals + (P.s_broadcast ? 0 : (int64_t)e * P.nnz) : P.a_vals + (int64_t)e * P.nnz;
  const int r0 = t.a, nr = t.b;
  // flat (row, column) walk over the chunk with the position stepped incrementally (one
  // division per thread instead of one per element)
  const int istep = kThreads / n, jstep = kThreads % n;
  int i = r0 + threadIdx.x / n, j = threadIdx.x % n;
  for (int q = threadIdx.x; q < nr * n; q += kThreads) {
    const int mi = map[(SIGMA && i < s) ? S.SIG[i] : i];
    const int mj = map[(SIGMA && j < s) ? S.SIG[j] : j];
    dst[(int64_t)i * n + j] = block_entry(d, lb, rb, mi, mj);
    i += istep;
    j += jstep;
    if (j >= n) {
      j -= n;
      ++i;
    }
  }
  __syncthreads();
  const SparseEntry* sp = P.sparse + d.sparse_off;
  // rows in merged order (A, and the B rows of Sigma) own one contiguous range of the
  // sparse list: one flat loop; pivot-permuted Sigma S rows one range per row
  const int flat0 = SIGMA ? max(r0, min(s, r0 + nr)) : r0;
  // (one warp per row: a row holds a handful of entries)
  for (int ri = threadIdx.x / 32; ri < flat0 - r0; ri += kThreads / 32) {
    const int i = r0 + ri;
    const int mr = S.SIG[i];
    for (int q = rowoff[mr] + (threadIdx.x & 31); q < rowoff[mr + 1]; q += 32) {
      const SparseEntry en = sp[q];
      const int j = en.j < s ? S.ISG[en.j] : en.j;
      dst[(int64_t)i * n + j] = ldg2(vals + en.csr);
    }
  }
  for (int q = rowoff[flat0] + threadIdx.x; q < rowoff[r0 + nr]; q += kThreads) {
    const SparseEntry en = sp[q];
    const int j = (SIGMA && en.j < s) ? S.ISG[en.j] : en.j;
    dst[(int64_t)en.i * n + j] = ldg2(vals + en.csr);
  }
  if (!SIGMA && r0 < s) {  // partial pivot scale max |A(S,S)| of these rows (kernels.py:241)
    __shared__ double cv[kThreads / 32];
    __shared__ int ci[kThreads / 32];
    __syncthreads();
    double mx = 0.0;
    const int rs = min(nr, max(0, s - r0));
    for (int q = threadIdx.x; q < rs * s; q += kThreads) mx = fmax(mx, cabs(dst[(int64_t)(r0 + q / s) * n + q % s]));
    int dummy = 0;
    block_argmax<kThreads>(mx, dummy, cv, ci);
    if (threadIdx.x == 0) S.pmax[r0 / kRowChunk] = mx;
  }
}

template <bool SIGMA>
__global__ void __launch_bounds__(kThreads) gather_kernel(SolveParams P, const Task* tasks) {
  pdl_entry();
  gather_body<SIGMA>(P, tasks[blockIdx.x], blockIdx.y);
}

// Inverse of one triangle of the jb x jb diagonal block D (smem, ld NB+1) of a
// factored panel, with all kThreads threads, by recursive doubling:
//   LOWER (unit L):  [A 0; C B]^-1 = [A^-1 0; -B^-1 C A^-1  B^-1]
//   upper (U):       [A C; 0 B]^-1 = [A^-1 -A^-1 C B^-1; 0  B^-1]
// X, W: smem [NB][NB+1]; rows/cols >= jb act as identity.
// Barrier over the NT threads [bar_base, bar_base + NT) of the CTA (named barrier bar_id when
// NT is not the whole CTA, so two halves can run independent inverses).
template <int NT>
__device__ __forceinline__ void part_sync(int bar_id) {
  if (NT == kThreads) __syncthreads();
  else asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(NT) : "memory");
}

template <int NB, bool LOWER, int NT>
__device__ void block_tri_inverse_t(const double2 (*D)[NB + 1], int jb, double2 (*X)[NB + 1], double2 (*W)[NB + 1],
                                    int tid = -1, int bar_id = 0) {
  if (tid < 0) tid = threadIdx.x;
  for (int q = tid; q < NB * NB; q += NT) {
    const int r = q / NB, c = q % NB;
    X[r][c] = r != c ? cz() : ((LOWER || r >= jb) ? make_double2(1.0, 0.0) : cinv(D[r][r]));
  }
  part_sync<NT>(bar_id);
  // Fixed-length inner products: the triangle's structural zeros (X triangular, D zero
  // outside jb) add exact zeros, so the sums equal the triangular ranges term for term and
  // every loop has a compile-time trip count (operand loads hoisted out of the FMA chain).
#pragma unroll
  for (int bs = 1; bs < NB; bs *= 2) {
#pragma unroll
    for (int q = tid; q < (NB / 2) * bs; q += NT) {
      const int pair = q / (bs * bs), loc = q % (bs * bs);
      const int k = pair * 2 * bs, a = loc / bs, b = loc % bs;
      double2 acc = cz();
      if (LOWER) {  // W[i][j] = sum_q L[i][q] X[q][j], i in B, q and j in A
        const int i = k + bs + a, jc = k + b;
#pragma unroll
        for (int qq = k; qq < k + bs; ++qq) acc = cfma(acc, D[i][qq], X[qq][jc]);
        W[i][jc] = acc;
      } else {  // W[i][j] = sum_q X[i][q] U[q][j], i and q in A, j in B
        const int i = k + a, jc = k + bs + b;
#pragma unroll
        for (int qq = k; qq < k + bs; ++qq) acc = cfma(acc, X[i][qq], D[qq][jc]);
        W[i][jc] = acc;
      }
    }
    part_sync<NT>(bar_id);
#pragma unroll
    for (int q = tid; q < (NB / 2) * bs; q += NT) {
      const int pair = q / (bs * bs), loc = q % (bs * bs);
      const int k = pair * 2 * bs, a = loc / bs, b = loc % bs;
      double2 acc = cz();
      if (LOWER) {  // X[i][j] = -sum_p X[i][p] W[p][j], p in B
        const int i = k + bs + a, jc = k + b;
#pragma unroll
        for (int p = k + bs; p < k + 2 * bs; ++p) acc = cfma(acc, X[i][p], W[p][jc]);
        X[i][jc] = make_double2(-acc.x, -acc.y);
      } else {  // X[i][j] = -sum_p W[i][p] X[p][j], p in B
        const int i = k + a, jc = k + bs + b;
#pragma unroll
        for (int p = k + bs; p < k + 2 * bs; ++p) acc = cfma(acc, W[i][p], X[p][jc]);
        X[i][jc] = make_double2(-acc.x, -acc.y);
      }
    }
    part_sync<NT>(bar_id);
  }
}

template <int NB, bool LOWER>
__device__ void block_tri_inverse(const double2 (*D)[NB + 1], int jb, double2 (*X)[NB + 1], double2 (*W)[NB + 1]) {
  block_tri_inverse_t<NB, LOWER, kThreads>(D, jb, X, W);
}

#ifdef FIND_PANEL_CLOCKS  // tools/tall_bench.cu latency breakdown of one panel CTA
__device__ long long g_pclk[64][8];
#define PCLK(k) do { if (blockIdx.x == 0 && blockIdx.y == 0 && (threadIdx.x & 31) == 0 && threadIdx.x / 32 == PCLK_WARP && jj < 64) g_pclk[jj][k] = clock64(); } while (0)
#ifndef PCLK_WARP
#define PCLK_WARP 0
#endif
#else
#define PCLK(k) do {} while (0)
#endif

// ---- panel step with ONE CTA barrier per column: T = 32 * ceil(R / 32) threads,
// one S row per thread in registers.  Per column, every warp reduces its best
// candidate (max |re|+|im|, lowest position on ties) and the candidate's lane
// publishes its whole row and the pivot inverse in a per-warp slot (double
// buffered); after the barrier every thread picks the winning slot and updates
// its row from it.  Row interchanges are logical positions; rows are written to
// their final positions at the end (LAPACK zgetf2 pivots: max |re|+|im|, lowest row on ties).
// two or three CTAs per SM up to 192 rows (the panel is latency-bound: throughput comes from
// concurrent panels); above that the row registers leave room for one without spilling
template <int NB, int T>
__global__ void __launch_bounds__(T, (T <= 96 ? 3 : (T <= 192 ? 2 : 1))) panel1_kernel(SolveParams P, const Task* tasks) {
  pdl_entry();
  constexpr int NW = T / 32;
  __shared__ double2 cand[2][NW][NB + 1];
  __shared__ double candv[2][NW];
  __shared__ int candi[2][NW];
  __shared__ int s_bad, s_nd;
  __shared__ double s_scale[NW];
  __shared__ double2 s_pval[NB];         // pivot values (test after the column loop)
  __shared__ int s_piv[NB];
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Task t = tasks[blockIdx.x];
  const int e = blockIdx.y;
  const ElimDesc d = P.elims[t.e];
  const int n = d.n, s = d.s, j = t.a;
  const int j0 = j * NB, jb = min(NB, s - j0), R = s - j0;
  const Scr S = scratch_of(P, d, e, NB);
  double2* M = S.M;
  double2* Lst = S.MS + (int64_t)tid * NB;
  const bool has = tid < R;
  int pos = tid;
  double2 row[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) row[c] = (has && c < jb) ? M[(int64_t)(j0 + tid) * n + j0 + c] : cz();
  if (tid == 0) { s_bad = INT32_MAX; s_nd = 0; }
  double scale;
  if (j == 0) {
    scale = 0.0;
    for (int q = tid; q < (s + kRowChunk - 1) / kRowChunk; q += T) scale = fmax(scale, S.pmax[q]);
    for (int o = 16; o; o >>= 1) scale = fmax(scale, __shfl_xor_sync(0xffffffffu, scale, o));
    if (lane == 0) s_scale[warp] = scale;
    __syncthreads();
    scale = s_scale[0];
    for (int w = 1; w < NW; ++w) scale = fmax(scale, s_scale[w]);
    if (tid == 0) {
      *S.scale = scale;
      if (scale == 0.0) s_bad = 0;
    }
  } else {
    scale = *reinterpret_cast<volatile double*>(S.scale);
  }
#pragma unroll 1
  for (int jj = 0; jj < jb; ++jj) {
    const int buf = jj & 1;
    const int rem = jb - jj - 1;  // panel columns right of the pivot column (row[1..rem])
    const bool act = has && pos >= jj;
    PCLK(0);
    // every candidate row's pivot inverse, off the reduction's critical path
    const double2 rinv = crcp(row[0]);
    // warp argmax: max |re|+|im| (>= 0, so its IEEE bits order like integers: high word,
    // then low word), then the lowest position holding it
    const double v0 = cabs1(row[0]);
    const double v = v0 >= 0.0 ? v0 : 0.0;  // NaN (after a zero pivot) ranks lowest; the status already failed
    const int vhi = act ? __double2hiint(v) : -1;
    const int mhi = __reduce_max_sync(0xffffffffu, vhi);
    const unsigned vlo = (unsigned)__double2loint(v);
    const unsigned mlo = __reduce_max_sync(0xffffffffu, vhi == mhi ? vlo : 0u);
    const bool best = act && vhi == mhi && vlo == mlo;
    const int wpos = (int)__reduce_min_sync(0xffffffffu, (unsigned)(best ? pos : INT32_MAX));
    PCLK(1);
    if (lane == 0) {
      candv[buf][warp] = mhi < 0 ? -1.0 : __hiloint2double(mhi, (int)mlo);
      candi[buf][warp] = wpos;
    }
    PCLK(2);
    __syncthreads();
    PCLK(3);
    // block argmax over the warp candidates (same rule), lane w looks at warp w
    const double cvw = lane < NW ? candv[buf][lane] : -1.0;
    const int ciw = lane < NW ? candi[buf][lane] : INT32_MAX;
    const int whi = cvw < 0.0 ? -1 : __double2hiint(cvw);
    const int bhi = __reduce_max_sync(0xffffffffu, whi);
    const unsigned wlo = (unsigned)__double2loint(cvw);
    const unsigned blo = __reduce_max_sync(0xffffffffu, whi == bhi ? wlo : 0u);
    const int pr0 = (int)__reduce_min_sync(0xffffffffu, (unsigned)((whi == bhi && wlo == blo) ? ciw : INT32_MAX));
    const int pr = pr0 >= jj && pr0 < R ? pr0 : jj;  // NaN / Inf entries: no interchange
    // only the pivot row is published (live part + its inverse), then a second barrier
    if (has && pos == pr) {
      double2* slot = cand[buf][0];
      slot[NB] = rinv;
#pragma unroll
      for (int c0 = 0; c0 < NB; c0 += 4)
        if (c0 <= rem) {
#pragma unroll
          for (int c = c0; c < c0 + 4; ++c) slot[c] = row[c];
        }
    }
    __syncthreads();
    const int wsel = 0;
    const double2* prow = cand[buf][wsel];
    PCLK(4);
    if (tid == 0) {
      s_piv[jj] = pr;
      s_pval[jj] = prow[0];
    }
    if (has && pos == pr) pos = -1 - jj;  // pivot row of column jj (final position jj)
    else if (has && pos == jj) pos = pr;
    if (has && pos > jj) {
      const double2 l = cmul(row[0], prow[NB]);
      Lst[jj] = l;
      // 8-column chunks of the live part: each chunk's shared loads issue together
#pragma unroll
      for (int c0 = 1; c0 < NB; c0 += 8)
        if (c0 <= rem) {
          double2 pv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (c0 + q < NB) pv[q] = prow[c0 + q];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (c0 + q < NB) row[c0 + q - 1] = cfms(row[c0 + q], l, pv[q]);
        }
    }
    PCLK(5);
  }
  __syncthreads();
  for (int k = tid; k < jb; k += T) {  // pivot rows and the pivot test of kernels.py:241 (abs < rtol * scale)
    S.PIV[j0 + k] = j0 + s_piv[k];
    if (cabs(s_pval[k]) < P.rtol * scale) atomicMin(&s_bad, j0 + k);
  }
  // final positions: pivot rows (pos = -1 - jj) hold U row jj shifted by jj
  int fp = pos < 0 ? -1 - pos : pos;
  if (has) {
    double2* dst = M + (int64_t)(j0 + fp) * n + j0;
    const int nl = min(fp, jb);
#pragma unroll 8
    for (int c = 0; c < nl; ++c) dst[c] = Lst[c];
    if (pos < 0) {
#pragma unroll
      for (int c = 0; c < NB; ++c)
        if (fp + c < jb) dst[fp + c] = row[c];
    }
    if (fp != tid) {
      const int k = atomicAdd(&s_nd, 1);
      S.PERM[1 + k] = tid;
      S.PERM[1 + 2 * NB + k] = fp;
    }
  }
  __syncthreads();
  if (tid == 0) {
    S.PERM[0] = s_nd;
    if (s_bad != INT32_MAX) report_bad(P, t.e, e, s_bad);
  }
}

// ---- same panel step with the S-row panel in shared memory (R > 256 rows):
// 256 threads, row per thread in a strided loop, 2 barriers per column.
template <int NB>
__global__ void __launch_bounds__(kThreads) panel_smem_kernel(SolveParams P, const Task* tasks) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* panel = reinterpret_cast<double2*>(smem_raw);  // [R][NB+1]
  constexpr int PS = NB + 1;
  __shared__ double cand_v[2][kThreads / 32];
  __shared__ int cand_i[2][kThreads / 32];
  __shared__ double2 s_uinv;
  __shared__ int s_bad, s_nd;
  __shared__ int lpiv[NB], dsrc[2 * NB], ddst[2 * NB];
  const int tid = threadIdx.x;
  const Task t = tasks[blockIdx.x];
  const int e = blockIdx.y;
  const ElimDesc d = P.elims[t.e];
  const int n = d.n, s = d.s;
  const int j = t.a, j0 = j * NB, jb = min(NB, s - j0), R = s - j0;
  const Scr S = scratch_of(P, d, e, NB);
  double2* M = S.M;
  if (tid == 0) s_bad = INT32_MAX;
  for (int q = tid; q < R * jb; q += kThreads) {
    const int r = q / jb, c = q % jb;
    panel[r * PS + c] = M[(int64_t)(j0 + r) * n + j0 + c];
  }
  double scale;
  if (j == 0) {
    scale = 0.0;
    for (int q = tid; q < (s + kRowChunk - 1) / kRowChunk; q += kThreads) scale = fmax(scale, S.pmax[q]);
    int dummy = 0;
    block_argmax<kThreads>(scale, dummy, cand_v[1], cand_i[1]);
    if (tid == 0) {
      *S.scale = scale;
      if (scale == 0.0) s_bad = 0;
    }
  } else {
    scale = *reinterpret_cast<volatile double*>(S.scale);
  }
  __syncthreads();
  for (int jj = 0; jj < jb; ++jj) {
    double v = -1.0;
    int vi = INT32_MAX;
    for (int r = tid; r < R; r += kThreads) {  // fixed row ownership: r = tid (mod 256)
      if (r < jj) continue;
      const double a = cabs1(panel[r * PS + jj]);
      if (a > v) { v = a; vi = r; }
    }
    block_argmax<kThreads>(v, vi, cand_v[jj & 1], cand_i[jj & 1]);
    const int pr = vi >= jj && vi < R ? vi : jj;  // NaN / Inf entries: no interchange
    if (tid == 0) {
      lpiv[jj] = pr;
      S.PIV[j0 + jj] = j0 + pr;
      s_uinv = cinv(panel[pr * PS + jj]);
      if (cabs(panel[pr * PS + jj]) < P.rtol * scale) atomicMin(&s_bad, j0 + jj);
    }
    if (pr != jj && tid < jb) {
      const double2 tmp = panel[jj * PS + tid];
      panel[jj * PS + tid] = panel[pr * PS + tid];
      panel[pr * PS + tid] = tmp;
    }
    __syncthreads();
    const double2 uinv = s_uinv;
    for (int r = tid; r < R; r += kThreads) {
      if (r <= jj) continue;
      double2* rw = panel + r * PS;
      const double2 l = cmul(rw[jj], uinv);
      rw[jj] = l;
#pragma unroll
      for (int c = 1; c < NB; ++c)
        if (c > jj && c < jb) rw[c] = cfms(rw[c], l, panel[jj * PS + c]);
    }
  }
  __syncthreads();
  for (int q = tid; q < R * jb; q += kThreads) {
    const int r = q / jb, c = q % jb;
    M[(int64_t)(j0 + r) * n + j0 + c] = panel[r * PS + c];
  }
  if (tid == 0) {
    int key[2 * NB], val[2 * NB], cnt = 0;
    for (int jj = 0; jj < jb; ++jj) {
      if (lpiv[jj] == jj) continue;
      int ia = -1, ib = -1;
      for (int k = 0; k < cnt; ++k) {
        if (key[k] == jj) ia = k;
        if (key[k] == lpiv[jj]) ib = k;
      }
      if (ia < 0) { key[cnt] = jj; val[cnt] = jj; ia = cnt++; }
      if (ib < 0) { key[cnt] = lpiv[jj]; val[cnt] = lpiv[jj]; ib = cnt++; }
      const int tmp = val[ia];
      val[ia] = val[ib];
      val[ib] = tmp;
    }
    int nd = 0;
    for (int k = 0; k < cnt; ++k)
      if (key[k] != val[k]) { ddst[nd] = key[k]; dsrc[nd] = val[k]; ++nd; }
    s_nd = nd;
  }
  __syncthreads();
  {
    const int nd = s_nd;
    if (tid == 0) S.PERM[0] = nd;
    for (int k = tid; k < nd; k += kThreads) {
      S.PERM[1 + k] = dsrc[k];
      S.PERM[1 + 2 * NB + k] = ddst[k];
    }
  }
  if (tid == 0 && s_bad != INT32_MAX) report_bad(P, t.e, e, s_bad);
}

// ---- U12 = L_jj^-1 A12 (type 0, 64-column tiles) and L21 = A21 U_jj^-1 (type 1, 64-row tiles), DMMA

// ---- NB = 32 panel step over a thread-block CLUSTER (S rows beyond one CTA's shared
// memory, s > 426): the R panel rows are split into CS contiguous chunks, one per CTA of
// the cluster, in shared memory.  Per column (two cluster barriers): every CTA posts its
// best candidate to every CTA (DSMEM stores); after the barrier all pick the same winner
// (max |re|+|im|, lowest row on ties, as panel_smem_kernel); the winner's owner broadcasts
// the pivot row and 1/u, the owner of row jj sends that row to the winner's owner; after
// the second barrier rows jj / pr are exchanged (LAPACK order) and every CTA updates its
// rows.  Same pivots, multipliers and outputs (M rows, PIV, PERM) as panel_smem_kernel<32>.
constexpr int kClusterMax = 8;
constexpr int kClusterRows = 384;  // rows per CTA: 384 * 33 * 16 B = 198 KB
__host__ __device__ constexpr size_t cluster_panel_smem() {
  return ((size_t)kClusterRows * 33 + 2 * kClusterMax * 33 + 2 * 33) * sizeof(double2);
}

__global__ void __launch_bounds__(kThreads) panel_cluster_kernel(SolveParams P, const Task* tasks) {
  namespace cg = cooperative_groups;
  constexpr int NB = 32, PS = NB + 1;
  cg::cluster_group cluster = cg::this_cluster();
  const int CS = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* panel = reinterpret_cast<double2*>(smem_raw);  // [chunk][PS]
  // per column parity: every CTA's candidate row [kClusterMax][PS] (+ its |.| and row index) and
  // the current row jj, posted by their owners to every CTA of the cluster
  double2* crow = panel + (size_t)kClusterRows * PS;       // [2][kClusterMax][PS]
  double2* jrow = crow + 2 * kClusterMax * PS;             // [2][PS]
  __shared__ double cand_v[2][kClusterMax];
  __shared__ int cand_i[2][kClusterMax];
  __shared__ double wv[kThreads / 32];
  __shared__ int wi[kThreads / 32];
  __shared__ int lpiv[NB], dsrc[2 * NB], ddst[2 * NB];
  __shared__ int s_bad, s_nd;
  const int tid = threadIdx.x;
  const Task t = tasks[blockIdx.x / CS];
  const int e = blockIdx.y;
  const ElimDesc d = P.elims[t.e];
  const int n = d.n, s = d.s;
  const int j = t.a, j0 = j * NB, jb = min(NB, s - j0), R = s - j0;
  const int chunk = (R + CS - 1) / CS;
  const int r_lo = min(R, rank * chunk), r_hi = min(R, r_lo + chunk), nloc = r_hi - r_lo;
  const Scr S = scratch_of(P, d, e, NB);
  double2* M = S.M;
  if (tid == 0) s_bad = INT32_MAX;
  for (int q = tid; q < nloc * jb; q += kThreads) {
    const int r = q / jb, c = q % jb;
    panel[r * PS + c] = M[(int64_t)(j0 + r_lo + r) * n + j0 + c];
  }
  double scale = 0.0;
  if (rank == 0) {
    if (j == 0) {
      for (int q = tid; q < (s + kRowChunk - 1) / kRowChunk; q += kThreads) scale = fmax(scale, S.pmax[q]);
      int dummy = 0;
      block_argmax<kThreads>(scale, dummy, wv, wi);
      if (tid == 0) {
        *S.scale = scale;
        if (scale == 0.0) s_bad = 0;
      }
    }
  }
  cluster.sync();
  scale = *reinterpret_cast<volatile double*>(S.scale);
  // One cluster barrier per column: before it every CTA posts its best candidate's whole row and
  // the owner of row jj posts row jj; after it all pick the same winner from their own copies.
  for (int jj = 0; jj < jb; ++jj) {
    const int buf = jj & 1;
    double v = -1.0;
    int vi = INT32_MAX;
    for (int r = max(jj - r_lo, 0) + tid; r < nloc; r += kThreads) {
      const double a = cabs1(panel[r * PS + jj]);
      if (a > v) { v = a; vi = r_lo + r; }
    }
    block_argmax<kThreads>(v, vi, wv, wi);
    const bool have = vi >= r_lo && vi < r_hi;
    for (int q = tid; q < CS * (NB + 2); q += kThreads) {  // candidate (value, index, row) to every CTA
      const int dst = q / (NB + 2), c = q % (NB + 2);
      if (c == NB) {
        *cluster.map_shared_rank(&cand_v[buf][rank], dst) = have ? v : -1.0;
        *cluster.map_shared_rank(&cand_i[buf][rank], dst) = have ? vi : INT32_MAX;
      } else if (c < NB && have) {
        cluster.map_shared_rank(crow, dst)[(buf * kClusterMax + rank) * PS + c] = panel[(vi - r_lo) * PS + c];
      }
    }
    if (jj >= r_lo && jj < r_hi)  // row jj (current diagonal position) to every CTA
      for (int q = tid; q < CS * NB; q += kThreads) {
        const int dst = q / NB, c = q % NB;
        cluster.map_shared_rank(jrow, dst)[buf * PS + c] = panel[(jj - r_lo) * PS + c];
      }
    cluster.sync();
    double bv = -1.0;
    int pr = INT32_MAX, pk = 0;
    for (int k = 0; k < CS; ++k) {
      const double ov = cand_v[buf][k];
      const int oi = cand_i[buf][k];
      if (ov > bv || (ov == bv && oi < pr)) { bv = ov; pr = oi; pk = k; }
    }
    const double2* prow = crow + (size_t)(buf * kClusterMax + pk) * PS;
    if (pr < jj || pr >= R) { pr = jj; prow = jrow + buf * PS; }  // NaN / Inf entries: no interchange
    if (tid == 0) {
      lpiv[jj] = pr;
      if (rank == 0 && cabs(prow[jj]) < P.rtol * scale) atomicMin(&s_bad, j0 + jj);
    }
    if (pr != jj) {  // exchange rows jj and pr (each owner rewrites its own copy)
      if (jj >= r_lo && jj < r_hi)
        for (int c = tid; c < NB; c += kThreads) panel[(jj - r_lo) * PS + c] = prow[c];
      if (pr >= r_lo && pr < r_hi)
        for (int c = tid; c < NB; c += kThreads) panel[(pr - r_lo) * PS + c] = jrow[buf * PS + c];
    }
    __syncthreads();
    const double2 uinv = cinv(prow[jj]);
    for (int r = max(jj + 1 - r_lo, 0) + tid; r < nloc; r += kThreads) {
      double2* rw = panel + r * PS;
      const double2 l = cmul(rw[jj], uinv);
      rw[jj] = l;
#pragma unroll
      for (int c = 1; c < NB; ++c)
        if (c > jj && c < jb) rw[c] = cfms(rw[c], l, prow[c]);
    }
  }
  cluster.sync();
  for (int q = tid; q < nloc * jb; q += kThreads) {
    const int r = q / jb, c = q % jb;
    M[(int64_t)(j0 + r_lo + r) * n + j0 + c] = panel[r * PS + c];
  }
  if (tid == 0 && s_bad != INT32_MAX) report_bad(P, t.e, e, s_bad);  // pivot test of the rows this CTA owned
  if (rank != 0) return;
  for (int k = tid; k < jb; k += kThreads) S.PIV[j0 + k] = j0 + lpiv[k];
  if (tid == 0) {
    int key[2 * NB], val[2 * NB], cnt = 0;
    for (int jj = 0; jj < jb; ++jj) {
      if (lpiv[jj] == jj) continue;
      int ia = -1, ib = -1;
      for (int k = 0; k < cnt; ++k) {
        if (key[k] == jj) ia = k;
        if (key[k] == lpiv[jj]) ib = k;
      }
      if (ia < 0) { key[cnt] = jj; val[cnt] = jj; ia = cnt++; }
      if (ib < 0) { key[cnt] = lpiv[jj]; val[cnt] = lpiv[jj]; ib = cnt++; }
      const int tmp = val[ia];
      val[ia] = val[ib];
      val[ib] = tmp;
    }
    int nd = 0;
    for (int k = 0; k < cnt; ++k)
      if (key[k] != val[k]) { ddst[nd] = key[k]; dsrc[nd] = val[k]; ++nd; }
    s_nd = nd;
  }
  __syncthreads();
  const int nd = s_nd;
  if (tid == 0) S.PERM[0] = nd;
  for (int k = tid; k < nd; k += kThreads) {
    S.PERM[1 + k] = dsrc[k];
    S.PERM[1 + 2 * NB + k] = ddst[k];
  }
}

// ---- NB = 32 panel step over a thread-block cluster with the rows in REGISTERS (panel1_kernel's
// scheme spread over CS <= 8 CTAs of T threads, one S row per thread): per column every warp
// reduces its best candidate (max |re|+|im|, lowest logical position on ties) and that lane posts
// its live row and 1/u to a per-warp slot; after one CTA barrier every CTA posts its best (value,
// position, row) to every CTA of the cluster through DSMEM (double-buffered by column parity);
// after one cluster barrier all threads pick the same winner from their local copies and update
// their own row in registers.  Interchanges only swap logical positions; every row is written once,
// to its final position, at the end.  Same pivots and arithmetic as panel1_kernel (the rank-1
// update of the panel rows runs out of registers instead of shared memory).
constexpr int kRegClusterRows = 256;  // rows per CTA (T <= 256 threads)
template <int T>
__global__ void __launch_bounds__(T, 1) panel_cluster_reg_kernel(SolveParams P, const Task* tasks) {
  pdl_entry();
  namespace cg = cooperative_groups;
  constexpr int NB = 32, NW = T / 32;
  cg::cluster_group cluster = cg::this_cluster();
  const int CS = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  __shared__ double2 wrow[2][NW][NB + 1];           // per-warp candidate rows (+ 1/u)
  __shared__ double wv[2][NW];
  __shared__ int wp[2][NW];
  __shared__ double2 crow[2][kClusterMax][NB + 1];  // every CTA's candidate row, posted by its owner CTA
  __shared__ double cv[2][kClusterMax];
  __shared__ int cp[2][kClusterMax];
  __shared__ int s_bad, s_nd;
  __shared__ double2 s_pval[NB];
  __shared__ int s_piv[NB];
  __shared__ double s_scale[NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Task t = tasks[blockIdx.x / CS];
  const int e = blockIdx.y;
  const ElimDesc d = P.elims[t.e];
  const int n = d.n, s = d.s, j = t.a;
  const int j0 = j * NB, jb = min(NB, s - j0), R = s - j0;
  const int chunk = (R + CS - 1) / CS;
  const int r_lo = min(R, rank * chunk), r_hi = min(R, r_lo + chunk);
  const int gr = r_lo + tid;  // this thread's panel row (physical, = its initial logical position)
  const Scr S = scratch_of(P, d, e, NB);
  double2* M = S.M;
  double2* Lst = S.MS + (int64_t)gr * NB;
  const bool has = gr < r_hi;
  int pos = gr;
  double2 row[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) row[c] = (has && c < jb) ? M[(int64_t)(j0 + gr) * n + j0 + c] : cz();
  if (tid == 0) { s_bad = INT32_MAX; s_nd = 0; }
  if (rank == 0 && j == 0) {
    double sc = 0.0;
    for (int q = tid; q < (s + kRowChunk - 1) / kRowChunk; q += T) sc = fmax(sc, S.pmax[q]);
    for (int o = 16; o; o >>= 1) sc = fmax(sc, __shfl_xor_sync(0xffffffffu, sc, o));
    if (lane == 0) s_scale[warp] = sc;
    __syncthreads();
    sc = s_scale[0];
    for (int w = 1; w < NW; ++w) sc = fmax(sc, s_scale[w]);
    if (tid == 0) {
      *S.scale = sc;
      if (sc == 0.0) s_bad = 0;
    }
  }
  cluster.sync();
  const double scale = *reinterpret_cast<volatile double*>(S.scale);
#pragma unroll 1
  for (int jj = 0; jj < jb; ++jj) {
    const int buf = jj & 1;
    const int rem = jb - jj - 1;
    const bool act = has && pos >= jj;
    const double2 rinv = crcp(row[0]);
    const double v0 = cabs1(row[0]);
    const double v = v0 >= 0.0 ? v0 : 0.0;  // NaN ranks lowest
    const int vhi = act ? __double2hiint(v) : -1;
    const int mhi = __reduce_max_sync(0xffffffffu, vhi);
    const unsigned vlo = (unsigned)__double2loint(v);
    const unsigned mlo = __reduce_max_sync(0xffffffffu, vhi == mhi ? vlo : 0u);
    const bool best = act && vhi == mhi && vlo == mlo;
    const int wpos = (int)__reduce_min_sync(0xffffffffu, (unsigned)(best ? pos : INT32_MAX));
    if (best && pos == wpos) {  // the warp's candidate posts its live row and pivot inverse
      double2* slot = wrow[buf][warp];
      slot[NB] = rinv;
#pragma unroll
      for (int c0 = 0; c0 < NB; c0 += 4)
        if (c0 <= rem) {
#pragma unroll
          for (int c = c0; c < c0 + 4; ++c) slot[c] = row[c];
        }
    }
    if (lane == 0) {
      wv[buf][warp] = mhi < 0 ? -1.0 : __hiloint2double(mhi, (int)mlo);
      wp[buf][warp] = wpos;
    }
    __syncthreads();
    // CTA candidate (every thread computes it) -> posted to every CTA of the cluster
    double bv = -1.0;
    int bp = INT32_MAX, bw = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const double ov = wv[buf][w];
      const int op = wp[buf][w];
      if (ov > bv || (ov == bv && op < bp)) { bv = ov; bp = op; bw = w; }
    }
    for (int q = tid; q < CS * (NB + 2); q += T) {
      const int dst = q / (NB + 2), c = q % (NB + 2);
      if (c == NB + 1) {
        *cluster.map_shared_rank(&cv[buf][rank], dst) = bv;
        *cluster.map_shared_rank(&cp[buf][rank], dst) = bp;
      } else if (bp != INT32_MAX && (c == NB || c <= rem)) {
        cluster.map_shared_rank(&crow[buf][rank][0], dst)[c] = wrow[buf][bw][c];
      }
    }
    cluster.sync();
    double gv = -1.0;
    int pr0 = INT32_MAX, pk = 0;
    for (int k = 0; k < CS; ++k) {
      const double ov = cv[buf][k];
      const int op = cp[buf][k];
      if (ov > gv || (ov == gv && op < pr0)) { gv = ov; pr0 = op; pk = k; }
    }
    const bool valid = pr0 >= jj && pr0 < R;  // NaN / Inf entries: no interchange (row jj pivots)
    const int pr = valid ? pr0 : jj;
    const double2* prow = crow[buf][pk];
    if (!valid) {
      // the row at logical position jj is this column's pivot: its owner has not posted it; every
      // thread reads it through its owner's candidate slot after a second exchange (rare path)
      __syncthreads();
      if (has && pos == jj) {
        for (int dst = 0; dst < CS; ++dst) {
          double2* o = cluster.map_shared_rank(&crow[buf][0][0], dst);
#pragma unroll
          for (int c = 0; c < NB; ++c) o[c] = row[c];
          o[NB] = rinv;
        }
      }
      cluster.sync();
      prow = crow[buf][0];
    }
    if (rank == 0 && tid == 0) {
      s_piv[jj] = pr;
      s_pval[jj] = prow[0];
    }
    if (has && pos == pr) pos = -1 - jj;  // pivot row of column jj (final position jj)
    else if (has && pos == jj) pos = pr;
    if (has && pos > jj) {
      const double2 l = cmul(row[0], prow[NB]);
      Lst[jj] = l;
#pragma unroll
      for (int c0 = 1; c0 < NB; c0 += 8)
        if (c0 <= rem) {
          double2 pv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (c0 + q < NB) pv[q] = prow[c0 + q];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (c0 + q < NB) row[c0 + q - 1] = cfms(row[c0 + q], l, pv[q]);
        }
    }
  }
  // final positions: pivot rows (pos = -1 - jj) hold U row jj shifted by jj
  const int fp = pos < 0 ? -1 - pos : pos;
  if (has) {
    double2* dst = M + (int64_t)(j0 + fp) * n + j0;
    const int nl = min(fp, jb);
#pragma unroll 8
    for (int c = 0; c < nl; ++c) dst[c] = Lst[c];
    if (pos < 0) {
#pragma unroll
      for (int c = 0; c < NB; ++c)
        if (fp + c < jb) dst[fp + c] = row[c];
    }
    if (fp != gr) {  // net interchange entry, counted on rank 0's counter
      const int k = atomicAdd(cluster.map_shared_rank(&s_nd, 0), 1);
      S.PERM[1 + k] = gr;
      S.PERM[1 + 2 * NB + k] = fp;
    }
  }
  cluster.sync();
  if (rank == 0) {
    for (int k = tid; k < jb; k += T) {  // pivot rows and the pivot test of kernels.py:241
      S.PIV[j0 + k] = j0 + s_piv[k];
      if (cabs(s_pval[k]) < P.rtol * scale) atomicMin(&s_bad, j0 + k);
    }
    __syncthreads();
    if (tid == 0) {
      S.PERM[0] = s_nd;
      if (s_bad != INT32_MAX) report_bad(P, t.e, e, s_bad);
    }
  }
}

// ---- L_jj^-1 and U_jj^-1 of panel j, once per (elimination, energy), published to LINV / UINV.
// Runs on the first kThreads threads of the CTA (every thread of the CTA must call it: the
// CTA-wide barriers are __syncthreads); smem: 5 [NB][NB+1] blocks + 64 ints.
template <int NB>
__device__ void panel_inv_body(const SolveParams& P, const Task& t, int e, unsigned char* smem_raw) {
  const int j = t.a;
  const ElimDesc d = P.elims[t.e];
  const int n = d.n, s = d.s;
  const int j0 = j * NB, jb = min(NB, s - j0);
  const Scr S = scratch_of(P, d, e, NB);
  const bool on = threadIdx.x < kThreads;
  typedef double2 Row[NB + 1];
  Row* Dm = reinterpret_cast<Row*>(smem_raw);
  Row* Xm = Dm + NB;
  Row* Wm = Xm + NB;
  // sigma (pivoted position -> merged position) kept up to date panel by panel: this panel's
  // net row interchange PERM applied to SIG[j0:s) exactly as to the rows of M (identity
  // before panel 0), so the last panel only inverts it -- no serial pass over PIV
  int* stg = reinterpret_cast<int*>(Wm + 3 * NB);
  const int nd = S.PERM[0];
  if (on) {
    if (j == 0)
      for (int k = threadIdx.x; k < s; k += kThreads) S.SIG[k] = k;
    for (int k = threadIdx.x; k < nd; k += kThreads) stg[k] = j == 0 ? S.PERM[1 + k] : S.SIG[j0 + S.PERM[1 + k]];
    for (int q = threadIdx.x; q < NB * NB; q += kThreads) {
      const int r = q / NB, c = q % NB;
      Dm[r][c] = (r < jb && c < jb) ? S.M[(int64_t)(j0 + r) * n + j0 + c] : cz();
    }
  }
  __syncthreads();
  if (on) {
    for (int k = threadIdx.x; k < nd; k += kThreads) S.SIG[j0 + S.PERM[1 + 2 * NB + k]] = stg[k];
    // L_jj^-1 on threads [0, 128), U_jj^-1 on [128, 256), concurrently (named barriers 1 and 2)
    constexpr int H = kThreads / 2;
    const bool lower = threadIdx.x < H;
    const int ht = lower ? threadIdx.x : threadIdx.x - H;
    Row* Xh = lower ? Xm : Wm + NB;
    Row* Wh = lower ? Wm : Wm + 2 * NB;
    if (lower) block_tri_inverse_t<NB, true, H>(Dm, jb, Xh, Wh, ht, 1);
    else block_tri_inverse_t<NB, false, H>(Dm, jb, Xh, Wh, ht, 2);
    double2* out = (lower ? S.LINV : S.UINV) + (int64_t)j * NB * NB;
    for (int q = ht; q < NB * NB; q += H) {
      const int r = q / NB, c = q % NB;
      out[q] = (r < jb && c < jb) ? Xh[r][c] : cz();
    }
  }
  if (j0 + jb == s) {  // last panel: sigma is final -> its inverse (the finish step)
    __syncthreads();
    if (on)
      for (int k = threadIdx.x; k < s; k += kThreads) S.ISG[S.SIG[k]] = k;
  }
}

template <int NB>
__global__ void __launch_bounds__(kThreads) panel_inv_kernel(SolveParams P, const Task* tasks) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  panel_inv_body<NB>(P, tasks[blockIdx.x], blockIdx.y, smem_raw);
}

// ---- NB = 32 panel step of a TALL panel in ONE CTA (many concurrent panels: the contact-row
// eliminations of the deep downward levels, s ~ 1000 with tiny b, hundreds per level).  The
// cluster kernels above spread one panel over up to 8 SMs and leave each of them idle at the
// per-column barriers; with more panels than SMs in flight the SM-time is what counts, so here a
// panel stays on one SM: up to 512 threads x RPT rows each.  The 32 panel columns are processed as
// four 8-column sub-panels held in registers (column steps: warp argmax, one barrier, pivot row
// published, one barrier, rank-1 update); after a sub-panel its eight pivot rows' remaining
// panel columns are solved in shared memory (8 x 24 block) and every other row applies the eight
// multipliers to its remaining columns, which round-trip through its own row of M except the
// next sub-panel's eight, which stay in registers (thread-per-row: every thread keeps its own
// 128-byte row segments in flight; a cooperative lanes-along-columns variant with the
// multipliers in shared memory measured slower, tools/tall_bench.cu).  Every element sees the
// same updates in the same order as in panel1_kernel (bit-identical results); rows are staged
// in MS and written once, to their final positions, at the end.
constexpr int kTallSP = 8;
constexpr int kTallMaxT = 512;
constexpr int tall_threads(int rpt) { return rpt >= 3 ? 352 : kTallMaxT; }  // three rows a thread need > 128 registers
constexpr int kTallMaxRows = 3 * tall_threads(3);
template <int RPT>
__global__ void __launch_bounds__(tall_threads(RPT), 1) panel_tall_kernel(SolveParams P, const Task* tasks) {
  pdl_entry();
  constexpr int NB = 32, SP = kTallSP, MAXW = kTallMaxT / 32;
  __shared__ double candv[2][MAXW];
  __shared__ int candi[2][MAXW];
  __shared__ double2 prow[2][SP + 1];  // pivot row's live sub-panel part + 1/u
  __shared__ double2 Us[SP][NB - SP];  // the sub-panel's pivot rows, remaining panel columns
  __shared__ double2 Lp[SP][SP];       // their multipliers inside the sub-panel
  __shared__ int s_bad, s_nd;
  __shared__ double s_scale[MAXW];
  __shared__ double2 s_pval[NB];
  __shared__ int s_piv[NB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = blockDim.x, NW = T >> 5;
  const Task t = tasks[blockIdx.x];
  const int e = blockIdx.y;
  const ElimDesc d = P.elims[t.e];
  const int n = d.n, s = d.s, j = t.a;
  const int j0 = j * NB, jb = min(NB, s - j0), R = s - j0;
  const Scr S = scratch_of(P, d, e, NB);
  double2* M = S.M;
  bool has[RPT];
  int pos[RPT];
  double2 a[RPT][SP];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int r = tid + i * T;
    has[i] = r < R;
    pos[i] = r;
#pragma unroll
    for (int c = 0; c < SP; ++c) a[i][c] = (has[i] && c < jb) ? M[(int64_t)(j0 + r) * n + j0 + c] : cz();
  }
  if (tid == 0) { s_bad = INT32_MAX; s_nd = 0; }
  double scale;
  if (j == 0) {
    scale = 0.0;
    for (int q = tid; q < (s + kRowChunk - 1) / kRowChunk; q += T) scale = fmax(scale, S.pmax[q]);
    for (int o = 16; o; o >>= 1) scale = fmax(scale, __shfl_xor_sync(0xffffffffu, scale, o));
    if (lane == 0) s_scale[warp] = scale;
    __syncthreads();
    scale = s_scale[0];
    for (int w = 1; w < NW; ++w) scale = fmax(scale, s_scale[w]);
    if (tid == 0) {
      *S.scale = scale;
      if (scale == 0.0) s_bad = 0;
    }
  } else {
    scale = *reinterpret_cast<volatile double*>(S.scale);
  }
#pragma unroll 1
  for (int c0 = 0; c0 < jb; c0 += SP) {
    const int cw = min(SP, jb - c0);
#pragma unroll
    for (int k = 0; k < SP; ++k) {
      if (k >= cw) break;
      const int jj = c0 + k, buf = jj & 1;
      PCLK(0);
      // this thread's best active row (max |re|+|im|, lowest position), then the warp's
      int vhi = -1, bpos = INT32_MAX;
      unsigned vlo = 0;
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const double v0 = cabs1(a[i][k]);
        const double v = v0 >= 0.0 ? v0 : 0.0;  // NaN ranks lowest
        const int hi = (has[i] && pos[i] >= jj) ? __double2hiint(v) : -1;
        const unsigned lo = (unsigned)__double2loint(v);
        if (hi > vhi || (hi == vhi && hi >= 0 && (lo > vlo || (lo == vlo && pos[i] < bpos)))) {
          vhi = hi;
          vlo = lo;
          bpos = pos[i];
        }
      }
      const int mhi = __reduce_max_sync(0xffffffffu, vhi);
      const unsigned mlo = __reduce_max_sync(0xffffffffu, vhi == mhi ? vlo : 0u);
      const bool best = vhi >= 0 && vhi == mhi && vlo == mlo;
      const int wpos = (int)__reduce_min_sync(0xffffffffu, (unsigned)(best ? bpos : INT32_MAX));
      if (lane == 0) {
        candv[buf][warp] = mhi < 0 ? -1.0 : __hiloint2double(mhi, (int)mlo);
        candi[buf][warp] = wpos;
      }
      PCLK(1);
      __syncthreads();
      PCLK(2);
      const double cvw = lane < NW ? candv[buf][lane] : -1.0;
      const int ciw = lane < NW ? candi[buf][lane] : INT32_MAX;
      const int whi = cvw < 0.0 ? -1 : __double2hiint(cvw);
      const int bhi = __reduce_max_sync(0xffffffffu, whi);
      const unsigned wlo = (unsigned)__double2loint(cvw);
      const unsigned blo = __reduce_max_sync(0xffffffffu, whi == bhi ? wlo : 0u);
      const int pr0 = (int)__reduce_min_sync(0xffffffffu, (unsigned)((whi == bhi && wlo == blo) ? ciw : INT32_MAX));
      const int pr = pr0 >= jj && pr0 < R ? pr0 : jj;  // NaN / Inf entries: no interchange
#pragma unroll
      for (int i = 0; i < RPT; ++i)
        if (has[i] && pos[i] == pr) {
          prow[buf][SP] = crcp(a[i][k]);
#pragma unroll
          for (int c = k; c < SP; ++c) prow[buf][c - k] = a[i][c];
        }
      PCLK(3);
      __syncthreads();
      PCLK(4);
      const double2 rinv = prow[buf][SP];
      if (tid == 0) {
        s_piv[jj] = pr;
        s_pval[jj] = prow[buf][0];
      }
      double2 pv[SP];
#pragma unroll
      for (int c = k + 1; c < SP; ++c) pv[c] = prow[buf][c - k];
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        if (has[i] && pos[i] == pr) pos[i] = -1 - jj;  // pivot row of column jj (final position jj)
        else if (has[i] && pos[i] == jj) pos[i] = pr;
        if (has[i] && pos[i] > jj) {
          const double2 l = cmul(a[i][k], rinv);
          a[i][k] = l;
#pragma unroll
          for (int c = k + 1; c < SP; ++c) a[i][c] = cfms(a[i][c], l, pv[c]);
        }
      }
    }
    const int jj = c0 + SP - 1;  // (clock stamps of the rest phase: slots 5-7 of the sub-panel's last column)
    (void)jj;
    PCLK(5);
    // the sub-panel's columns are final: stage them (L multipliers / U values) in MS
#pragma unroll
    for (int i = 0; i < RPT; ++i)
      if (has[i] && (pos[i] >= 0 || pos[i] <= -1 - c0)) {  // not earlier sub-panels' pivot rows (staged with their U values)
        double2* Lst = S.MS + (int64_t)(tid + i * T) * NB + c0;
#pragma unroll
        for (int c = 0; c < SP; ++c)
          if (c < cw) Lst[c] = a[i][c];
      }
    const int nrest = jb - (c0 + SP);  // panel columns right of the sub-panel
    if (nrest <= 0) break;
    // the sub-panel's pivot rows: raw remaining columns and their multipliers to shared memory
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int kk = -1 - pos[i] - c0;  // pivot index inside the sub-panel
      if (has[i] && pos[i] < 0 && kk >= 0 && kk < SP) {
        const double2* src = M + (int64_t)(j0 + tid + i * T) * n + j0 + c0 + SP;
        for (int c = 0; c < nrest; ++c) Us[kk][c] = src[c];
#pragma unroll
        for (int c = 0; c < SP; ++c) Lp[kk][c] = a[i][c];
      }
    }
    __syncthreads();
    if (tid < nrest) {  // U rows of the sub-panel: row kk minus its multipliers times the rows above
#pragma unroll
      for (int kk = 1; kk < SP; ++kk) {
        double2 u = Us[kk][tid];
#pragma unroll
        for (int q = 0; q < kk; ++q) u = cfms(u, Lp[kk][q], Us[q][tid]);
        Us[kk][tid] = u;
      }
    }
    __syncthreads();
    PCLK(6);
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      if (!has[i]) continue;
      const int r = tid + i * T;
      const int kk = -1 - pos[i] - c0;
      if (pos[i] < 0 && kk >= 0 && kk < SP) {  // a pivot row of this sub-panel: its U values are final
        double2* Lst = S.MS + (int64_t)r * NB + c0 + SP;
        for (int c = 0; c < nrest; ++c) Lst[c] = Us[kk][c];
      } else if (pos[i] >= 0) {  // still active: apply the eight multipliers to the remaining columns
        double2* mrow = M + (int64_t)(j0 + r) * n + j0 + c0 + SP;
        double2 l[SP];
#pragma unroll
        for (int q = 0; q < SP; ++q) l[q] = a[i][q];
#pragma unroll 1
        for (int cc = 0; cc < nrest; cc += SP) {
          double2 x[SP];
#pragma unroll
          for (int c = 0; c < SP; ++c) x[c] = cc + c < nrest ? mrow[cc + c] : cz();
#pragma unroll 2
          for (int q = 0; q < SP; ++q)
#pragma unroll
            for (int c = 0; c < SP; ++c) x[c] = cfms(x[c], l[q], Us[q][cc + c]);
          if (cc == 0) {
#pragma unroll
            for (int c = 0; c < SP; ++c) a[i][c] = x[c];  // the next sub-panel stays in registers
          } else {
#pragma unroll
            for (int c = 0; c < SP; ++c)
              if (cc + c < nrest) mrow[cc + c] = x[c];
          }
        }
      }
    }
    PCLK(7);
    // (Us / Lp are next written after the next sub-panel's column barriers)
  }
  __syncthreads();
  for (int k = tid; k < jb; k += T) {  // pivot rows and the pivot test of kernels.py:241 (abs < rtol * scale)
    S.PIV[j0 + k] = j0 + s_piv[k];
    if (cabs(s_pval[k]) < P.rtol * scale) atomicMin(&s_bad, j0 + k);
  }
#pragma unroll
  for (int i = 0; i < RPT; ++i)
    if (has[i]) {
      const int r = tid + i * T;
      const int fp = pos[i] < 0 ? -1 - pos[i] : pos[i];
      const double2* Lst = S.MS + (int64_t)r * NB;
      double2* dst = M + (int64_t)(j0 + fp) * n + j0;
#pragma unroll 8
      for (int c = 0; c < jb; ++c) dst[c] = Lst[c];
      if (fp != r) {
        const int k = atomicAdd(&s_nd, 1);
        S.PERM[1 + k] = r;
        S.PERM[1 + 2 * NB + k] = fp;
      }
    }
  __syncthreads();
  if (tid == 0) {
    S.PERM[0] = s_nd;
    if (s_bad != INT32_MAX) report_bad(P, t.e, e, s_bad);
  }
}

template <int NB>
struct TrsmTiles;
template <>
struct TrsmTiles<32> { using U = Tile<4, 2, 1, 4, false>; using L = Tile<4, 2, 2, 2, false>; };
template <>
struct TrsmTiles<16> { using U = Tile<2, 4, 1, 2, false>; using L = Tile<4, 2, 2, 1, false>; };
template <>
struct TrsmTiles<8> { using U = Tile<1, 8, 1, 1, false>; using L = Tile<8, 1, 1, 1, false>; };
template <>
struct TrsmTiles<4> { using U = Tile<1, 8, 1, 1, false>; using L = Tile<8, 1, 1, 1, false>; };

// ---- wide (two-panel) block TRSM for columns [c0, c0+64) right of the block [J0, J0+2NB):
// both panels' row interchanges in order (PERM2 of panel j-1 at J0, PERM of panel j at
// J0+NB), then U12 = L_JJ^-1 A12 as top = L1^-1 A_top, A_bot -= L21 top, bot = L2^-1 A_bot.
template <int NB>
__device__ void wide_trsm_tile(const Scr& S, int n, int s, int j, int c0, double2* smem) {
  using TT = typename TrsmTiles<NB>::U;
  double2* M = S.M;
  const int J0 = (j - 1) * NB, jb2 = min(NB, s - j * NB);
  const int cn = min(kTile, n - c0);
  double2* st = smem;  // [2 NB][64] staging of the moved rows
  for (int pass = 0; pass < 2; ++pass) {
    const int* perm = pass == 0 ? S.PERM2 : S.PERM;
    const int base = pass == 0 ? J0 : J0 + NB;
    const int nd = perm[0];
    for (int q = threadIdx.x; q < nd * kTile; q += kThreads) {
      const int k = q / kTile, c = q % kTile;
      if (c < cn) st[q] = M[(int64_t)(base + perm[1 + k]) * n + c0 + c];
    }
    __syncthreads();
    for (int q = threadIdx.x; q < nd * kTile; q += kThreads) {
      const int k = q / kTile, c = q % kTile;
      if (c < cn) M[(int64_t)(base + perm[1 + 2 * NB + k]) * n + c0 + c] = st[q];
    }
    __syncthreads();
  }
  double2* top = M + (int64_t)J0 * n + c0;
  double2* bot = M + (int64_t)(J0 + NB) * n + c0;
  {
    TT T;
    T.zero();
    T.mma(S.LINV + (int64_t)(j - 1) * NB * NB, NB, top, n, NB, cn, NB, smem);
    T.for_each([&](int r, int c, double2 v) {
      if (r < NB && c < cn) top[(int64_t)r * n + c] = v;
    });
  }
  __syncthreads();
  {
    TT T;
    T.zero();
    T.mma(M + (int64_t)(J0 + NB) * n + J0, n, top, n, jb2, cn, NB, smem);
    T.for_each([&](int r, int c, double2 v) {
      if (r < jb2 && c < cn) bot[(int64_t)r * n + c] = csub(bot[(int64_t)r * n + c], v);
    });
  }
  __syncthreads();
  TT T;
  T.zero();
  T.mma(S.LINV + (int64_t)j * NB * NB, NB, bot, n, jb2, cn, jb2, smem);
  T.for_each([&](int r, int c, double2 v) {
    if (r < jb2 && c < cn) bot[(int64_t)r * n + c] = v;
  });
}

template <int NB>
__device__ void trsm_body(const SolveParams& P, const Task& t, int e, int j, double2* smem, bool inv_ready = false) {
  const ElimDesc d = P.elims[t.e];
  const int n = d.n, s = d.s;
  const int j0 = j * NB, jb = min(NB, s - j0);
  const Scr S = scratch_of(P, d, e, NB);
  double2* M = S.M;
  if (t.a == 5) {  // wide block: keep the first panel's interchanges for the wide TRSM
    for (int k = threadIdx.x; k < 1 + 4 * NB; k += kThreads) S.PERM2[k] = S.PERM[k];
    return;
  }
  if (t.a == 3) {  // wide TRSM: this is the block's second panel j; columns [c0, c0+64) right of it
    wide_trsm_tile<NB>(S, n, s, j, t.b, smem);
    return;
  }
  if (t.a == 1 && inv_ready && P.zskip && d.zsplit && j0 + jb <= (d.zsplit & 0xffff) && t.b >= (d.zsplit >> 16))
    return;  // L21 rows in B_r of a panel inside S_l: A(B_r, S_l) structurally zero, L21 stays zero
  if (t.a != 1) {
    // this panel's row interchanges on columns [c0, c0+64) (solver-side zgetrf laswp), or the
    // t.c-wide strip of the next panel of a wide block: all moved rows are read before any is written
    const int c0 = t.b, cn = min(t.c > 0 ? t.c : kTile, (t.a == 2 ? j0 : n) - c0);
    const int nd = S.PERM[0];
    if (nd > 0) {  // (uniform over the CTA)
      double2* st = smem;  // [2 NB][64]
      for (int q = threadIdx.x; q < nd * kTile; q += kThreads) {
        const int k = q / kTile, c = q % kTile;
        if (c < cn) st[q] = M[(int64_t)(j0 + S.PERM[1 + k]) * n + c0 + c];
      }
      __syncthreads();
      for (int q = threadIdx.x; q < nd * kTile; q += kThreads) {
        const int k = q / kTile, c = q % kTile;
        if (c < cn) M[(int64_t)(j0 + S.PERM[1 + 2 * NB + k]) * n + c0 + c] = st[q];
      }
      __syncthreads();
    }
    if (t.a == 2) return;
  }
  if (!inv_ready) {  // the diagonal block's inverse this tile needs (L for U12 tiles, U for L21 tiles),
     // published to the elimination's LINV/UINV slot; every tile of the elimination writes the same values
    typedef double2 Row[NB + 1];
    Row* Dm = reinterpret_cast<Row*>(smem);
    Row* Xm = Dm + NB;
    Row* Wm = Xm + NB;
    for (int q = threadIdx.x; q < NB * NB; q += kThreads) {
      const int r = q / NB, c = q % NB;
      Dm[r][c] = (r < jb && c < jb) ? M[(int64_t)(j0 + r) * n + j0 + c] : cz();
    }
    __syncthreads();
    if (t.a == 0) block_tri_inverse<NB, true>(Dm, jb, Xm, Wm);
    else block_tri_inverse<NB, false>(Dm, jb, Xm, Wm);
    double2* out = (t.a == 0 ? S.LINV : S.UINV) + (int64_t)j * NB * NB;
    for (int q = threadIdx.x; q < NB * NB; q += kThreads) {
      const int r = q / NB, c = q % NB;
      out[q] = (r < jb && c < jb) ? Xm[r][c] : cz();
    }
    __syncthreads();
  }
  if (t.a == 0) {
    using TT = typename TrsmTiles<NB>::U;
    const int c0 = t.b;
    double2* B = M + (int64_t)j0 * n + c0;
    TT T;
    T.zero();
    const int cn = min(t.c > 0 ? t.c : kTile, n - c0);
    T.mma(S.LINV + (int64_t)j * NB * NB, NB, B, n, jb, cn, jb, smem);
    T.for_each([&](int r, int c, double2 v) {
      if (r < jb && c < cn) B[(int64_t)r * n + c] = v;
    });
  } else {
    using TT = typename TrsmTiles<NB>::L;
    const int r0 = s + t.b;
    double2* A = M + (int64_t)r0 * n + j0;
    TT T;
    T.zero();
    T.mma(A, n, S.UINV + (int64_t)j * NB * NB, NB, min(kTile, n - r0), jb, jb, smem);
    T.for_each([&](int r, int c, double2 v) {
      if (r0 + r < n && c < jb) A[(int64_t)r * n + c] = v;
    });
  }
}

template <int NB>
__global__ void __launch_bounds__(kThreads) trsm_kernel(SolveParams P, const Task* tasks, int j, int inv_ready) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  trsm_body<NB>(P, tasks[blockIdx.x], blockIdx.y, j, reinterpret_cast<double2*>(smem_raw), inv_ready != 0);
}

// ---- trailing update M[j1:, j1:] -= M[j1:, j0:j1] M[j0:j1, j1:]
// t.c: 0 the full trailing update of panel j; 2 only the next panel's columns (the strip of
// a wide block); 1 the wide block's update, K = both panels (j-1, j)
__device__ void trail_body(const SolveParams& P, const Task& t, int e, int j, int nb, double2* smem) {
  const ElimDesc d = P.elims[t.e];
  const int n = d.n, s = d.s;
  const int j0 = (t.c == 1 ? j - 1 : j) * nb, j1 = min(s, (j + 1) * nb), jb = j1 - j0;
  double2* M = scratch_of(P, d, e).M;
  const int r0 = j1 + t.a * kTile, c0 = j1 + t.b * kTile;
  const int cw = t.c == 2 ? min(nb, s - j1) : kTile;
  // all rows in B_r and the panel inside S_l with A(B_r, S_l) structurally zero: L21 = 0 there
  if (P.zskip && d.zsplit && j1 <= (d.zsplit & 0xffff) && r0 >= s + (d.zsplit >> 16)) return;
  Tile64 T;
  T.load_c(M + (int64_t)r0 * n + c0, n, min(kTile, n - r0), min(cw, n - c0));
  T.mma<false, true>(M + (int64_t)r0 * n + j0, n, M + (int64_t)j0 * n + c0, n, min(kTile, n - r0), min(cw, n - c0), jb,
                     smem);
  T.for_each([&](int r, int c, double2 v) {
    if (r0 + r < n && c < cw && c0 + c < n && (r0 + r < s || c0 + c < s)) M[(int64_t)(r0 + r) * n + c0 + c] = v;
  });
}

__global__ void __launch_bounds__(kThreads, 2) trail_kernel(SolveParams P, const Task* tasks, int j, int nb) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  trail_body(P, tasks[blockIdx.x], blockIdx.y, j, nb, reinterpret_cast<double2*>(smem_raw));
}

// ---- U = A_BB - Y U12 in one K = s pass (Y = M[s:, :s] = A_BS U11^-1, U12 = M[:s, s:]),
// stored sorted (solver.py:234-243); final steps keep U_f in M for the epilogue
__device__ void schur_body(const SolveParams& P, const Task& t, int e, double2* smem) {
  const ElimDesc d = P.elims[t.e];
  const int n = d.n, s = d.s, b = d.b;
  double2* M = scratch_of(P, d, e).M;
  const int i0 = t.a * kTile, c0 = t.b * kTile;
  // rows in B_r with A(B_r, S_l) structurally zero: Y is zero on the first s_l columns, so
  // K starts at s_l (rounded down to the K chunk: the same products in the same order)
  const int k0 = (P.zskip && d.zsplit && i0 >= (d.zsplit >> 16)) ? ((d.zsplit & 0xffff) / kKC) * kKC : 0;
  Tile64 T;
  T.load_c(M + (int64_t)(s + i0) * n + s + c0, n, min(kTile, b - i0), min(kTile, b - c0));
  T.mma<false, true>(M + (int64_t)(s + i0) * n + k0, n, M + (int64_t)k0 * n + s + c0, n, min(kTile, b - i0),
                     min(kTile, b - c0), s - k0, smem);
  const bool store = d.kind != kFinal && d.out_arena >= 0;
  double2* out = store ? P.arena[d.out_arena] + (int64_t)e * P.arena_elems[d.out_arena] + d.out_off : nullptr;
  const int32_t* rank = P.i32 + d.rank_off;
  T.for_each([&](int r, int c, double2 v) {
    const int i = i0 + r, jj = c0 + c;
    if (i < b && jj < b) {
      if (store) out[(int64_t)rank[i] * b + rank[jj]] = v;
      else M[(int64_t)(s + i) * n + s + jj] = v;
    }
  });
}

__global__ void __launch_bounds__(kThreads, 2) schur_kernel(SolveParams P, const Task* tasks) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  schur_body(P, tasks[blockIdx.x], blockIdx.y, reinterpret_cast<double2*>(smem_raw));
}

// ---- X_j = (Y_j - X_{>j} L11[>j, j]) L_jj^-1 for 64 B rows: Z = Y_j - X_{>j} L11[>j, j]
// (one DMMA tile, K = s - j1) is written to X_j, then X_j = Z L_jj^-1 (second DMMA
// tile, K = jb) with the inverse published by the panel / TRSM launch of step j.
template <int NB, class TT = typename XTileSel<NB>::T, int NS = 2>
__device__ void xsolve_tile(const Scr& S, int n, int s, int j, int r0, double2* smem, int rows = kTile) {
  double2* M = S.M;
  const int b = n - s;
  const int j0 = j * NB, jb = min(NB, s - j0), j1 = j0 + jb;
  const int nr = min(rows, b - r0);
  {
    TT T;
    T.load_c(M + (int64_t)(s + r0) * n + j0, n, nr, jb);
    if (s > j1)
      T.template mma<false, true, NS>(S.X + (int64_t)r0 * s + j1, s, M + (int64_t)j1 * n + j0, n, nr, jb, s - j1, smem);
    T.for_each([&](int r, int c, double2 v) {
      if (r < nr && c < jb) S.X[(int64_t)(r0 + r) * s + j0 + c] = v;
    });
  }
  __syncthreads();
  TT T;
  T.zero();
  T.template mma<false, false, NS>(S.X + (int64_t)r0 * s + j0, s, S.LINV + (int64_t)j * NB * NB, NB, nr, jb, jb, smem);
  T.for_each([&](int r, int c, double2 v) {
    if (r < nr && c < jb) S.X[(int64_t)(r0 + r) * s + j0 + c] = v;
  });
  __syncthreads();
}

// ---- X_j = (Y_j - X_{>j} L11[>j, j]) L_jj^-1 for 64 B rows (X in its own buffer; Y stays for the Schur launch)
template <int NB>
__global__ void __launch_bounds__(kThreads) xsolve_kernel(SolveParams P, const Task* tasks) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Task t = tasks[blockIdx.x];
  const int e = blockIdx.y;
  const ElimDesc d = P.elims[t.e];
  const Scr S = scratch_of(P, d, e, NB);
  if (NB == 32 && t.b == 16) {  // 16-row tiles: 4x the CTAs for groups with few row tiles
    for (int j = (d.s + NB - 1) / NB - 1; j >= 0; --j)
      xsolve_tile<NB, Tile<2, 4, 1, 1, false>, 4>(S, d.n, d.s, j, t.a * 16, reinterpret_cast<double2*>(smem_raw), 16);
    return;
  }
  for (int j = (d.s + NB - 1) / NB - 1; j >= 0; --j)
    xsolve_tile<NB>(S, d.n, d.s, j, t.a * kTile, reinterpret_cast<double2*>(smem_raw));
}

// ---- pivot permutation sigma and its inverse (+ L for the unit-test shim)
__device__ void finish_body(const SolveParams& P, int64_t eidx, const ElimDesc& d, int e, int nb, int* sig) {
  const int tid = threadIdx.x;
  const int s = d.s, b = d.b;
  const Scr S = scratch_of(P, d, e, nb);
  for (int k = tid; k < s; k += kThreads) sig[k] = k;
  __syncthreads();
  if (tid == 0)
    for (int k = 0; k < s; ++k) {
      const int pk = S.PIV[k];
      const int tmp = sig[k];
      sig[k] = sig[pk];
      sig[pk] = tmp;
    }
  __syncthreads();
  for (int k = tid; k < s; k += kThreads) {
    S.SIG[k] = sig[k];
    S.ISG[sig[k]] = k;
  }
  if (P.dbg_l && eidx == 0 && e == 0)
    for (int64_t q = tid; q < (int64_t)b * s; q += kThreads) P.dbg_l[(q / s) * s + sig[q % s]] = S.X[q];
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads) finish_kernel(SolveParams P, const Task* tasks, int nb) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Task t = tasks[blockIdx.x];
  const ElimDesc d = P.elims[t.e];
  finish_body(P, t.e, d, blockIdx.y, nb, reinterpret_cast<int*>(smem_raw));
}

// ---- T_S = MS[s:, :s] - X MS[:s, :s]   (the S columns of T = Sigma'_B: - X Sigma'_S:)
__device__ void tgemm_body(const SolveParams& P, const Task& t, int e, int nb, double2* smem) {
  const ElimDesc d = P.elims[t.e];
  const int n = d.n, s = d.s, b = d.b;
  const Scr S = scratch_of(P, d, e);
  const int i0 = t.a * kTile, c0 = t.b * kTile;
  Tile64 T;
  T.load_c(S.MS + (int64_t)(s + i0) * n + c0, n, min(kTile, b - i0), min(kTile, s - c0));
  const Scr SX = scratch_of(P, d, e, nb);
  T.mma<false, true>(SX.X + (int64_t)i0 * s, s, S.MS + c0, n, min(kTile, b - i0), min(kTile, s - c0), s, smem);
  T.for_each([&](int r, int c, double2 v) {
    if (i0 + r < b && c0 + c < s) S.MS[(int64_t)(s + i0 + r) * n + c0 + c] = v;
  });
}

__global__ void __launch_bounds__(kThreads, 2) tgemm_kernel(SolveParams P, const Task* tasks, int nb) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  tgemm_body(P, tasks[blockIdx.x], blockIdx.y, nb, reinterpret_cast<double2*>(smem_raw));
}

// ---- R = Sigma'_BB - X Sigma'_SB - T_S X^H in one pass (two K = s products into one
// accumulator), stored sorted (or kept in MS for the final step).  Symmetric mode:
// lower-triangle tiles only; the upper triangle is written as the (skew-)conjugate
// mirror of elements (i >= j), so results stay deterministic.
__device__ void rgemm_body(const SolveParams& P, const Task& t, int e, int nb, double2* smem) {
  if (t.c == 2 && P.rsym != 0) return;
  const ElimDesc d = P.elims[t.e];
  const int n = d.n, s = d.s, b = d.b;
  const Scr S = scratch_of(P, d, e);
  const int i0 = t.a * kTile, c0 = t.b * kTile;
  const int mv = min(kTile, b - i0), nv = min(kTile, b - c0);
  Tile64 T;
  T.load_c(S.MS + (int64_t)(s + i0) * n + s + c0, n, mv, nv);
  const Scr SX = scratch_of(P, d, e, nb);
  T.mma<false, true>(SX.X + (int64_t)i0 * s, s, S.MS + s + c0, n, mv, nv, s, smem);          // - X Sigma'_SB
  T.mma<true, true>(S.MS + (int64_t)(s + i0) * n, n, SX.X + (int64_t)c0 * s, s, mv, nv, s, smem);  // - T_S X^H
  const bool store = d.kind != kFinal && d.out_arena >= 0;
  const bool mirror = store && P.rsym != 0;
  const double sg = P.rsym < 0 ? -1.0 : 1.0;
  double2* out = store ? P.arena[d.out_arena] + (int64_t)e * P.arena_elems[d.out_arena] + d.out_off + (int64_t)b * b
                       : nullptr;
  const int32_t* rank = P.i32 + d.rank_off;
  T.for_each([&](int r, int c, double2 v) {
    const int i = i0 + r, jj = c0 + c;
    if (i < b && jj < b) {
      const double2 val = v;
      if (!store) {
        S.MS[(int64_t)(s + i) * n + s + jj] = val;
      } else if (!mirror) {
        out[(int64_t)rank[i] * b + rank[jj]] = val;
      } else if (i >= jj) {
        out[(int64_t)rank[i] * b + rank[jj]] = val;
        if (i != jj) out[(int64_t)rank[jj] * b + rank[i]] = make_double2(sg * val.x, -sg * val.y);
      }
    }
  });
}

__global__ void __launch_bounds__(kThreads, 2) rgemm_kernel(SolveParams P, const Task* tasks, int nb) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  rgemm_body(P, tasks[blockIdx.x], blockIdx.y, nb, reinterpret_cast<double2*>(smem_raw));
}

// ---- the same four DMMA tile kinds (trailing update, Schur, T_S, R) through the TMA engine
// (dmma_engine.cuh): one persistent CTA per SM walks the launch's (task, energy) tiles in order;
// a producer warp streams the operands (UTMALDG boxes of the A / X^H operands through the
// elimination's tensor maps, UBLKCP rows of the [k][n] operands) into a 4-stage mbarrier ring
// and prefetches the next tile's C block into L2; eight consumer warps run the DMMA fragments.
// Same products, operand order and epilogues as trail_body / schur_body / tgemm_body /
// rgemm_body (bit-identical results).
using TmaEng = dmma::Eng64;

struct TileJob {
  dmma::Seg seg[2];
  int nseg;
  double2* C;     // C block (row stride n)
  int mv, nv;     // valid rows / columns of the tile
  const CUtensorMap* cmap;
  int cr, cc;     // C block origin in cmap's matrix
};

template <int KIND>
__device__ __forceinline__ bool tile_job(const SolveParams& P, const Task& t, int e, int j, int nb, TileJob& J) {
  const ElimDesc d = P.elims[t.e];
  const int n = d.n, s = d.s, b = d.b;
  const CUtensorMap* tm = P.tmaps + 3 * (int64_t)d.tmap;
  double2* M = scratch_of(P, d, e).M;
  double2* MS = M + (int64_t)n * n;
  if (KIND == kLTrail) {
    const int j0 = (t.c == 1 ? j - 1 : j) * nb, j1 = min(s, (j + 1) * nb), jb = j1 - j0;
    const int r0 = j1 + t.a * kTile, c0 = j1 + t.b * kTile;
    const int cw = t.c == 2 ? min(nb, s - j1) : kTile;
    if (P.zskip && d.zsplit && j1 <= (d.zsplit & 0xffff) && r0 >= s + (d.zsplit >> 16)) return false;
    J.seg[0] = {tm + 0, nullptr, M + (int64_t)j0 * n + c0, n, r0, j0, 0, 0, jb, 0};
    J.nseg = 1;
    J.C = M + (int64_t)r0 * n + c0;
    J.mv = min(kTile, n - r0);
    J.nv = min(cw, n - c0);
    J.cmap = tm + 0;
    J.cr = r0;
    J.cc = c0;
  } else if (KIND == kLSchur) {
    const int i0 = t.a * kTile, c0 = t.b * kTile;
    const int k0 = (P.zskip && d.zsplit && i0 >= (d.zsplit >> 16)) ? ((d.zsplit & 0xffff) / kKC) * kKC : 0;
    J.seg[0] = {tm + 0, nullptr, M + (int64_t)k0 * n + s + c0, n, s + i0, k0, 0, 0, s - k0, 0};
    J.nseg = 1;
    J.C = M + (int64_t)(s + i0) * n + s + c0;
    J.mv = min(kTile, b - i0);
    J.nv = min(kTile, b - c0);
    J.cmap = tm + 0;
    J.cr = s + i0;
    J.cc = s + c0;
  } else if (KIND == kLTGemm) {
    const int i0 = t.a * kTile, c0 = t.b * kTile;
    J.seg[0] = {tm + 2, nullptr, MS + c0, n, i0, 0, 0, 0, s, 0};
    J.nseg = 1;
    J.C = MS + (int64_t)(s + i0) * n + c0;
    J.mv = min(kTile, b - i0);
    J.nv = min(kTile, s - c0);
    J.cmap = tm + 1;
    J.cr = s + i0;
    J.cc = c0;
  } else {  // kLRGemm: R = Sigma'_BB - X Sigma'_SB - T_S X^H
    if (t.c == 2 && P.rsym != 0) return false;
    const int i0 = t.a * kTile, c0 = t.b * kTile;
    J.seg[0] = {tm + 2, nullptr, MS + s + c0, n, i0, 0, 0, 0, s, 0};
    J.seg[1] = {tm + 1, tm + 2, nullptr, 0, s + i0, 0, c0, 0, s, 1};
    J.nseg = 2;
    J.C = MS + (int64_t)(s + i0) * n + s + c0;
    J.mv = min(kTile, b - i0);
    J.nv = min(kTile, b - c0);
    J.cmap = tm + 1;
    J.cr = s + i0;
    J.cc = s + c0;
  }
  return true;
}

template <int KIND, class Eng>
__device__ __forceinline__ void tile_store(const SolveParams& P, const Task& t, int e, int j, int nb, const TileJob& J,
                                           const Eng& eng) {
  const ElimDesc d = P.elims[t.e];
  const int n = d.n, s = d.s, b = d.b;
  if (KIND == kLTrail) {
    const int j1 = min(s, (j + 1) * nb);
    const int r0 = j1 + t.a * kTile, c0 = j1 + t.b * kTile;
    const int cw = t.c == 2 ? min(nb, s - j1) : kTile;
    eng.for_each([&](int r, int c, double2 v) {
      if (r0 + r < n && c < cw && c0 + c < n && (r0 + r < s || c0 + c < s)) J.C[(int64_t)r * n + c] = v;
    });
  } else if (KIND == kLTGemm) {
    eng.for_each([&](int r, int c, double2 v) {
      if (r < J.mv && c < J.nv) J.C[(int64_t)r * n + c] = v;
    });
  } else {
    const int i0 = t.a * kTile, c0 = t.b * kTile;
    const bool store = d.kind != kFinal && d.out_arena >= 0;
    const int32_t* rank = P.i32 + d.rank_off;
    if (KIND == kLSchur) {
      double2* out = store ? P.arena[d.out_arena] + (int64_t)e * P.arena_elems[d.out_arena] + d.out_off : nullptr;
      eng.for_each([&](int r, int c, double2 v) {
        const int i = i0 + r, jj = c0 + c;
        if (i < b && jj < b) {
          if (store) out[(int64_t)rank[i] * b + rank[jj]] = v;
          else J.C[(int64_t)r * n + c] = v;
        }
      });
    } else {
      const bool mirror = store && P.rsym != 0;
      const double sg = P.rsym < 0 ? -1.0 : 1.0;
      double2* out = store ? P.arena[d.out_arena] + (int64_t)e * P.arena_elems[d.out_arena] + d.out_off + (int64_t)b * b
                           : nullptr;
      eng.for_each([&](int r, int c, double2 v) {
        const int i = i0 + r, jj = c0 + c;
        if (i < b && jj < b) {
          if (!store) {
            J.C[(int64_t)r * n + c] = v;
          } else if (!mirror) {
            out[(int64_t)rank[i] * b + rank[jj]] = v;
          } else if (i >= jj) {
            out[(int64_t)rank[i] * b + rank[jj]] = v;
            if (i != jj) out[(int64_t)rank[jj] * b + rank[i]] = make_double2(sg * v.x, -sg * v.y);
          }
        }
      });
    }
  }
}

template <int KIND, bool CS = false>
__global__ void __launch_bounds__(TmaEng::THREADS, 1) tile_tma_kernel(SolveParams P, const Task* tasks, int64_t cnt,
                                                                     int nE, int j, int nb,
                                                                     unsigned long long* counter) {
  using Eng = typename std::conditional<CS, dmma::Eng64cs, TmaEng>::type;
  pdl_entry();
  extern __shared__ __align__(16) unsigned char smem_raw[];  // Engine::init aligns to 1024
  Eng eng;
  eng.init(smem_raw);
  const int64_t total = cnt * nE;
  // tiles are drawn in order from the launch's counter (zeroed by the solve call): the tiles of
  // one launch differ in K, in skipped work and in their epilogues
  if (Eng::producer()) {
    for (;;) {
      const int64_t q = eng.next_tile_p(counter, total);
      if (q < 0) break;
      const int e = (int)(q / cnt);
      const Task t = tasks[q % cnt];
      TileJob J;
      if (!tile_job<KIND>(P, t, e, j, nb, J)) continue;
      if (CS) eng.stage_c(J.cmap, J.cr, J.cc, e);
      else Eng::prefetch_c(J.cmap, J.cr, J.cc, e);
      eng.produce(J.seg, J.nseg, e, J.nv);
    }
  } else {
    for (;;) {
      const int64_t q = eng.next_tile_c();
      if (q < 0) break;
      const int e = (int)(q / cnt);
      const Task t = tasks[q % cnt];
      TileJob J;
      if (!tile_job<KIND>(P, t, e, j, nb, J)) continue;
      if (CS) eng.load_c_staged();
      else eng.load_c(J.C, P.elims[t.e].n, J.mv, J.nv);
      eng.template consume<true>(J.seg, J.nseg, J.mv, J.nv);
      tile_store<KIND>(P, t, e, j, nb, J, eng);
    }
  }
}

// ================================================================== dense batched primitives
// The block-tridiagonal RGF comparison path (find_selinv/rgf.py:108-208) runs on the same DMMA
// tiles and elimination kernels as FIND: a strided-batched complex GEMM and a batched dense
// inverse (the Schur complement of [[A, I], [I, 0]] is -A^-1: one blocked elimination per matrix).
struct GemmArgs {
  const double2* A;  // [m][k], row stride lda, batch stride sa
  const double2* B;  // [k][n] (bt = 0) or [n][k], used as its conjugate transpose (bt = 1)
  double2* C;        // [m][n]
  int64_t lda, sa, ldb, sb, ldc, sc;
  int m, n, k, bt, mode;  // mode 0: C = AB;  +1: C += AB;  -1: C -= AB
};

__global__ void __launch_bounds__(kThreads, 2) zgemm_kernel(GemmArgs g) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* smem = reinterpret_cast<double2*>(smem_raw);
  const int tn = (g.n + kTile - 1) / kTile;
  const int i0 = (blockIdx.x / tn) * kTile, c0 = (blockIdx.x % tn) * kTile;
  const int mv = min(kTile, g.m - i0), nv = min(kTile, g.n - c0);
  const double2* A = g.A + (int64_t)blockIdx.y * g.sa + (int64_t)i0 * g.lda;
  const double2* B = g.B + (int64_t)blockIdx.y * g.sb + (g.bt ? (int64_t)c0 * g.ldb : (int64_t)c0);
  double2* C = g.C + (int64_t)blockIdx.y * g.sc + (int64_t)i0 * g.ldc + c0;
  Tile64 T;
  if (g.mode != 0) T.load_c(C, g.ldc, mv, nv);
  else T.zero();
  if (g.bt) {
    if (g.mode < 0) T.mma<true, true>(A, g.lda, B, g.ldb, mv, nv, g.k, smem);
    else T.mma<true, false>(A, g.lda, B, g.ldb, mv, nv, g.k, smem);
  } else {
    if (g.mode < 0) T.mma<false, true>(A, g.lda, B, g.ldb, mv, nv, g.k, smem);
    else T.mma<false, false>(A, g.lda, B, g.ldb, mv, nv, g.k, smem);
  }
  T.for_each([&](int r, int c, double2 v) {
    if (r < mv && c < nv) C[(int64_t)r * g.ldc + c] = v;
  });
}

// merged block [[A, I], [I, 0]] (2n x 2n, row-major) of every matrix of the batch
__global__ void __launch_bounds__(kThreads) dense_pack_kernel(const double2* a, double2* up, int64_t up_stride, int n) {
  const int n2 = 2 * n;
  double2* M = up + (int64_t)blockIdx.y * up_stride;
  const double2* A = a + (int64_t)blockIdx.y * n * n;
  for (int64_t q = blockIdx.x * (int64_t)kThreads + threadIdx.x; q < (int64_t)n2 * n2; q += (int64_t)gridDim.x * kThreads) {
    const int i = (int)(q / n2), j = (int)(q % n2);
    double2 v = cz();
    if (i < n && j < n) v = A[(int64_t)i * n + j];
    else if ((i < n && j == i + n) || (j < n && i == j + n)) v = make_double2(1.0, 0.0);
    M[q] = v;
  }
}

// A^-1 = -(Schur complement)
__global__ void __launch_bounds__(kThreads) dense_unpack_kernel(const double2* u, int64_t u_stride, double2* out, int n) {
  const double2* U = u + (int64_t)blockIdx.y * u_stride;
  double2* O = out + (int64_t)blockIdx.y * n * n;
  for (int64_t q = blockIdx.x * (int64_t)kThreads + threadIdx.x; q < (int64_t)n * n; q += (int64_t)gridDim.x * kThreads) {
    const double2 v = U[q];
    O[q] = make_double2(-v.x, -v.y);
  }
}

// ---- final leaf step epilogue, warp per (leaf, energy)
__device__ void final_body_warp(const SolveParams& P, const Task& t, int e, double2* uf, int cmax, int lane) {
  const ElimDesc d = P.elims[t.e];
  const int n = d.n, s = d.s, c = d.b;
  const int ld = cmax + 1;
  double2* rf = uf + cmax * ld;
  const Scr S = scratch_of(P, d, e);
  for (int q = lane; q < c * c; q += 32) {
    uf[(q / c) * ld + q % c] = S.M[(int64_t)(s + q / c) * n + s + q % c];
    rf[(q / c) * ld + q % c] = P.compute_gless ? S.MS[(int64_t)(s + q / c) * n + s + q % c] : cz();
  }
  __syncwarp();
  final_epilogue_warp(P, d, t.e, e, uf, ld, rf, ld, lane);
}

__global__ void __launch_bounds__(kSmallWarps * 32) final_kernel(SolveParams P, const Task* tasks, int64_t count,
                                                                 int cmax) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t idx = (int64_t)blockIdx.x * kSmallWarps + warp;
  if (idx >= count) return;
  final_body_warp(P, tasks[idx], blockIdx.y, reinterpret_cast<double2*>(smem_raw) + (size_t)warp * 2 * cmax * (cmax + 1),
                  cmax, lane);
}


// ================================================================== off-diagonal extraction
// G^r and G^< between each leaf C and its ring r = B_{-C} (solver.py:454-484; the
// G^< cross blocks as in _extended_extraction, solver.py:487-507, which the
// reference computes by inverting [[U_r, A_rC], [A_Cr, A_CC]] and sandwiching
// [[R_r, S_rC], [S_Cr, S_CC]]).  With K = A_rr^-1 A_rC, L = A_Cr A_rr^-1,
// G = U_f^-1, G^<_CC = G R_f G^H:
//   G(r, C)   = -K G                       G(C, r) = -G L
//   G^<(r, C) = A_rr^-1 (S_rC - R_r L^H) G^H - K G^<_CC
//   G^<(C, r) = [same with Sigma^H]^H   (= +-G^<(r, C)^H when Sigma^< is (skew-)Hermitian)
// Outputs are written only for the pairs this leaf owns (first in DFS order).
constexpr int kOffMaxC = 16;
constexpr int kOffT = 256;

// CTA-path final steps reuse the factorization left in scratch: M[:s,:s] = L11\U11 of
// P A_rr, M[:s, s:] = U12 = L11^-1 P A_rC, M[s:, s:] = U_f, X = A_Cr U11^-1 L11^-1
// (L = X P), the inverted diagonal blocks L_jj^-1 / U_jj^-1, and in MS the pivot-
// permuted Sigma rows of S (P S_rr P^T | P S_rC), T_S and R_f.  Then
//   P (S_rC - R_r L^H) = MS_SB - MS_SS X^H,  P (S^H_rC - R_r^H L^H) = T_S^H,
// and A_rr^-1 = U11^-1 L11^-1 P: blocked substitutions with the published inverses.
__global__ void __launch_bounds__(kOffT) offdiag_cta_kernel(SolveParams P, const Task* tasks, int nb) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sm = reinterpret_cast<double2*>(smem_raw);
  const Task t = tasks[blockIdx.x];
  const int e = blockIdx.y, tid = threadIdx.x;
  const int64_t it0 = P.off_item_off[t.e], it1 = P.off_item_off[t.e + 1];
  if (it0 == it1) return;
  const ElimDesc d = P.elims[t.e];
  const int n = d.n, s = d.s, c = d.b;
  const Scr S = scratch_of(P, d, e, nb);
  const double2* M = S.M;
  const double2* MS = S.MS;
  const bool gl = P.off_gl != nullptr;
  const bool gen = gl && P.off_sym == 0;
  const int nc = gl ? (gen ? 3 * c : 2 * c) : c;
  const int ldc = c + 1;
  double2* G = sm;
  double2* GL = G + c * ldc;
  double2* RF = GL + c * ldc;
  double2* Z = RF + c * ldc;           // [s][nc]: K | x2 | x3
  double2* TM = Z + (int64_t)s * nc;   // [nb][nc]
  for (int q = tid; q < c * c; q += kOffT) {
    const int i = q / c, j = q % c;
    G[i * ldc + j] = M[(int64_t)(s + i) * n + s + j];
    RF[i * ldc + j] = gl ? MS[(int64_t)(s + i) * n + s + j] : cz();
  }
  __syncthreads();
  if (tid < 32) {
    bool sing = false;  // a singular U_f is reported by the final launch
    warp_gj_inverse(G, ldc, c, tid, &sing);
  }
  __syncthreads();
  if (gl)
    for (int q = tid; q < c * c; q += kOffT) {
      const int i = q / c, j = q % c;
      double2 acc = cz();
      for (int a = 0; a < c; ++a) {
        double2 tt = cz();
        for (int b2 = 0; b2 < c; ++b2) tt = cfma(tt, RF[a * ldc + b2], cconj(G[j * ldc + b2]));
        acc = cfma(acc, G[i * ldc + a], tt);
      }
      GL[i * ldc + j] = acc;
    }
  // right-hand sides, rows in pivoted order
  for (int k = tid; k < s; k += kOffT) {
    double2* z = Z + (int64_t)k * nc;
    for (int j = 0; j < c; ++j) z[j] = M[(int64_t)k * n + s + j];
    if (!gl) continue;
    double2 v[kOffMaxC];
    const double2* mr = MS + (int64_t)k * n;
    for (int j = 0; j < c; ++j) {
      double2 acc = mr[s + j];
      const double2* xr = S.X + (int64_t)j * s;
      for (int m = 0; m < s; ++m) acc = cfms(acc, mr[m], cconj(xr[m]));
      v[j] = acc;
    }
    for (int j = 0; j < c; ++j) {
      double2 acc = cz();
      for (int i = 0; i < c; ++i) acc = cfma(acc, v[i], cconj(G[j * ldc + i]));
      z[c + j] = acc;
    }
    if (gen)
      for (int j = 0; j < c; ++j) {
        double2 acc = cz();
        for (int i = 0; i < c; ++i) acc = cfma(acc, cconj(MS[(int64_t)(s + i) * n + k]), cconj(G[j * ldc + i]));
        z[2 * c + j] = acc;
      }
  }
  __syncthreads();
  const int nblk = (s + nb - 1) / nb;
  if (gl) {  // unit-lower L11 on the Sigma columns
    const int w = nc - c;
    for (int j = 0; j < nblk; ++j) {
      const int j0 = j * nb, jb = min(nb, s - j0), j1 = j0 + jb;
      const double2* Li = S.LINV + (int64_t)j * nb * nb;
      for (int q = tid; q < jb * w; q += kOffT) {
        const int r = q / w, col = c + q % w;
        double2 acc = cz();
        for (int kk = 0; kk < jb; ++kk) acc = cfma(acc, Li[r * nb + kk], Z[(int64_t)(j0 + kk) * nc + col]);
        TM[r * nc + col] = acc;
      }
      __syncthreads();
      for (int q = tid; q < jb * w; q += kOffT) {
        const int r = q / w, col = c + q % w;
        Z[(int64_t)(j0 + r) * nc + col] = TM[r * nc + col];
      }
      __syncthreads();
      for (int q = tid; q < (s - j1) * w; q += kOffT) {
        const int i = j1 + q / w, col = c + q % w;
        double2 acc = Z[(int64_t)i * nc + col];
        const double2* lr = M + (int64_t)i * n + j0;
        for (int kk = 0; kk < jb; ++kk) acc = cfms(acc, lr[kk], Z[(int64_t)(j0 + kk) * nc + col]);
        Z[(int64_t)i * nc + col] = acc;
      }
      __syncthreads();
    }
  }
  for (int j = nblk - 1; j >= 0; --j) {  // U11 on every column; rows become merged ring positions
    const int j0 = j * nb, jb = min(nb, s - j0);
    const double2* Ui = S.UINV + (int64_t)j * nb * nb;
    for (int q = tid; q < jb * nc; q += kOffT) {
      const int r = q / nc, col = q % nc;
      double2 acc = cz();
      for (int kk = 0; kk < jb; ++kk) acc = cfma(acc, Ui[r * nb + kk], Z[(int64_t)(j0 + kk) * nc + col]);
      TM[r * nc + col] = acc;
    }
    __syncthreads();
    for (int q = tid; q < jb * nc; q += kOffT) Z[(int64_t)(j0 + q / nc) * nc + q % nc] = TM[q];
    __syncthreads();
    for (int q = tid; q < j0 * nc; q += kOffT) {
      const int i = q / nc, col = q % nc;
      double2 acc = Z[(int64_t)i * nc + col];
      const double2* ur = M + (int64_t)i * n + j0;
      for (int kk = 0; kk < jb; ++kk) acc = cfms(acc, ur[kk], Z[(int64_t)(j0 + kk) * nc + col]);
      Z[(int64_t)i * nc + col] = acc;
    }
    __syncthreads();
  }
  const double sg = P.off_sym < 0 ? -1.0 : 1.0;
  for (int64_t q = it0 + tid; q < it1; q += kOffT) {
    const OffItem I = P.off_items[q];
    double2 gr = cz(), gv = cz();
    if (I.type == 2) {
      gr = G[I.r * ldc + I.c];
      if (gl) gv = GL[I.r * ldc + I.c];
    } else {
      const double2* z = Z + (int64_t)I.r * nc;
      const int cj = I.c;
      if (I.type == 0) {
        for (int k = 0; k < c; ++k) gr = cfms(gr, z[k], G[k * ldc + cj]);
        if (gl) {
          gv = z[c + cj];
          for (int k = 0; k < c; ++k) gv = cfms(gv, z[k], GL[k * ldc + cj]);
        }
      } else {
        const int pc = S.ISG[I.r];
        for (int k = 0; k < c; ++k) gr = cfms(gr, G[cj * ldc + k], S.X[(int64_t)k * s + pc]);
        if (gl) {
          double2 v;
          if (gen) {
            v = z[2 * c + cj];
            for (int k = 0; k < c; ++k) v = cfms(v, z[k], cconj(GL[cj * ldc + k]));
            gv = cconj(v);
          } else {
            v = z[c + cj];
            for (int k = 0; k < c; ++k) v = cfms(v, z[k], GL[k * ldc + cj]);
            gv = make_double2(sg * v.x, -sg * v.y);
          }
        }
      }
    }
    P.off_gr[(int64_t)e * P.n_pairs + I.pair] = gr;
    if (gl) P.off_gl[(int64_t)e * P.n_pairs + I.pair] = gv;
  }
}

// Warp- and mid-path final steps (s + c <= 64): the trailing system
// M = [[U_r, A_rC], [A_Cr, A_CC]] and its Sigma counterpart are rebuilt in shared
// memory and M is inverted in place (Gauss-Jordan, partial pivoting), as the
// reference's _extended_extraction does (solver.py:487-507).
template <int NMAX>
__host__ __device__ constexpr size_t offdiag_small_smem() {
  return (size_t)(2 * NMAX * (NMAX + 1) + 2 * NMAX * kOffMaxC + NMAX) * sizeof(double2);
}

template <int NMAX, int NT>
__global__ void __launch_bounds__(NT) offdiag_small_kernel(SolveParams P, int64_t elim_begin) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int LD = NMAX + 1;
  __shared__ int ip[NMAX];
  __shared__ int piv;
  const int64_t k = elim_begin + blockIdx.x;
  const int e = blockIdx.y, tid = threadIdx.x;
  const int64_t it0 = P.off_item_off[k], it1 = P.off_item_off[k + 1];
  if (it0 == it1) return;
  const ElimDesc d = P.elims[k];
  const int n = d.n, s = d.s, c = d.b;
  double2* A = reinterpret_cast<double2*>(smem_raw);  // [NMAX][LD]: M, then M^-1
  double2* SG = A + NMAX * LD;                          // [NMAX][LD]: merged Sigma
  double2* Q = SG + NMAX * LD;                          // [NMAX][kOffMaxC]: Sigma G(C,:)^H
  double2* Q2 = Q + NMAX * kOffMaxC;                    // [NMAX][kOffMaxC]: Sigma^H G(C,:)^H
  double2* F = Q2 + NMAX * kOffMaxC;                    // [NMAX]
  const bool gl = P.off_gl != nullptr;
  const bool gen = gl && P.off_sym == 0;
  const int32_t* map = P.i32 + d.map_off;
  const SparseEntry* sp = P.sparse + d.sparse_off;
  for (int sig = 0; sig < (gl ? 2 : 1); ++sig) {
    double2* dst = sig ? SG : A;
    const double2* lb = child_block(P, d, e, true, sig != 0);
    const double2* rb = child_block(P, d, e, false, sig != 0);
    for (int q = tid; q < n * n; q += NT) dst[(q / n) * LD + q % n] = block_entry(d, lb, rb, map[q / n], map[q % n]);
    __syncthreads();
    const double2* vals = sig ? P.s_vals + (P.s_broadcast ? 0 : (int64_t)e * P.nnz) : P.a_vals + (int64_t)e * P.nnz;
    for (int q = tid; q < d.nsparse; q += NT) {
      const SparseEntry en = sp[q];
      dst[en.i * LD + en.j] = ldg2(vals + en.csr);
    }
    __syncthreads();
  }
  for (int kk = 0; kk < n; ++kk) {
    if (tid < 32) {
      double best = -1.0;
      int bi = kk;
      for (int i = kk + tid; i < n; i += 32) {
        const double v = cabs1(A[i * LD + kk]);
        if (v > best) { best = v; bi = i; }
      }
      for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (tid == 0) { piv = bi; ip[kk] = bi; }
    }
    __syncthreads();
    const int p = piv;
    if (p != kk)
      for (int j = tid; j < n; j += NT) {
        const double2 tmp = A[kk * LD + j];
        A[kk * LD + j] = A[p * LD + j];
        A[p * LD + j] = tmp;
      }
    __syncthreads();
    const double2 pinv = cinv(A[kk * LD + kk]);
    for (int i = tid; i < n; i += NT) F[i] = A[i * LD + kk];
    __syncthreads();
    for (int j = tid; j < n; j += NT) A[kk * LD + j] = cmul(j == kk ? make_double2(1.0, 0.0) : A[kk * LD + j], pinv);
    __syncthreads();
    for (int q = tid; q < n * n; q += NT) {
      const int i = q / n, j = q % n;
      if (i == kk) continue;
      A[i * LD + j] = cfms(j == kk ? cz() : A[i * LD + j], F[i], A[kk * LD + j]);
    }
    __syncthreads();
  }
  for (int kk = n - 1; kk >= 0; --kk) {
    const int p = ip[kk];
    if (p != kk)
      for (int i = tid; i < n; i += NT) {
        const double2 tmp = A[i * LD + kk];
        A[i * LD + kk] = A[i * LD + p];
        A[i * LD + p] = tmp;
      }
    __syncthreads();
  }
  if (gl) {
    for (int q = tid; q < n * c; q += NT) {
      const int i = q / c, cj = q % c;
      const double2* grow = A + (s + cj) * LD;
      double2 a1 = cz(), a2 = cz();
      for (int m = 0; m < n; ++m) {
        a1 = cfma(a1, SG[i * LD + m], cconj(grow[m]));
        if (gen) a2 = cfma(a2, cconj(SG[m * LD + i]), cconj(grow[m]));
      }
      Q[i * kOffMaxC + cj] = a1;
      Q2[i * kOffMaxC + cj] = a2;
    }
    __syncthreads();
  }
  const double sg = P.off_sym < 0 ? -1.0 : 1.0;
  for (int64_t q = it0 + tid; q < it1; q += NT) {
    const OffItem I = P.off_items[q];
    const int row = I.type == 2 ? s + I.r : I.r;  // G^< row: ring r (types 0, 1) or leaf node a
    const int cj = I.c;
    double2 gr, gv = cz();
    if (I.type == 0) gr = A[I.r * LD + s + cj];
    else if (I.type == 1) gr = A[(s + cj) * LD + I.r];
    else gr = A[(s + I.r) * LD + s + cj];
    if (gl) {
      const double2* QQ = (I.type == 1 && gen) ? Q2 : Q;
      double2 acc = cz();
      for (int m = 0; m < n; ++m) acc = cfma(acc, A[row * LD + m], QQ[m * kOffMaxC + cj]);
      if (I.type == 1) gv = gen ? cconj(acc) : make_double2(sg * acc.x, -sg * acc.y);
      else gv = acc;
    }
    P.off_gr[(int64_t)e * P.n_pairs + I.pair] = gr;
    if (gl) P.off_gl[(int64_t)e * P.n_pairs + I.pair] = gv;
  }
}

// ================================================================== host side
#define CUDA_TRY(x)                                                                                   \
  do {                                                                                                \
    cudaError_t err__ = (x);                                                                          \
    if (err__ != cudaSuccess) {                                                                       \
      if (st) {                                                                                       \
        st->code = FIND_ECUDA;                                                                        \
        std::snprintf(st->message, sizeof(st->message), "%s: %s", #x, cudaGetErrorString(err__));    \
      }                                                                                               \
      return FIND_ECUDA;                                                                              \
    }                                                                                                 \
  } while (0)

void status_ok(find_status* st) {
  if (!st) return;
  st->code = FIND_OK;
  st->energy_idx = -1;
  st->cluster_label = 0;
  st->node_id = -1;
  st->pivot_ratio = NAN;
  std::snprintf(st->message, sizeof(st->message), "ok");
}

int fail_status(find_status* st, int code, const char* msg) {
  if (st) {
    st->code = code;
    std::snprintf(st->message, sizeof(st->message), "%s", msg);
  }
  return code;
}

// Kernel launches, optionally with programmatic stream serialization
// (FIND_B200_PDL=1; measured neutral on cfg1, so off by default): every kernel
// starts with pdl_entry(), so a launch may begin while its predecessor in the
// stream drains; errors surface through cudaGetLastError().
const bool g_pdl = [] {
  const char* f = std::getenv("FIND_B200_PDL");
  return f && f[0] == '1';
}();
template <typename... KArgs, typename... Args>
void launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
void launch_cluster(void (*k)(KArgs...), dim3 grid, dim3 block, unsigned cs, size_t smem, cudaStream_t st,
                    Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

constexpr size_t kMaxSmem = 227 * 1024 - 1024;  // dynamic budget (static smem of the kernels < 1 KB)
size_t ws_header_bytes() { return 256; }
// tile counters of the TMA engine launches (one per launch spec), at the end of the workspace
size_t tile_ctr_bytes(const find_plan* P) { return (P->specs.size() * 8 + 255) / 256 * 256 + 256; }

template <int NB>
size_t xsolve_smem() {
  using TT = typename XTileSel<NB>::T;
  return TT::SMEM;
}

template <int NB>
size_t trsm_smem() {
  return std::max(std::max(std::max(TrsmTiles<NB>::U::SMEM, TrsmTiles<NB>::L::SMEM), (size_t)2 * NB * kTile * sizeof(double2)),
                  (size_t)3 * NB * (NB + 1) * sizeof(double2));
}

// The dynamic shared-memory opt-ins are per device: tracked per device index (a process may drive
// several GPUs, one host thread each).
constexpr int kMaxDevices = 64;
bool g_attrs_done[kMaxDevices] = {};
std::mutex g_attrs_mu;

int set_attrs(find_status* st) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return fail_status(st, FIND_EINVAL, "device index out of range");
  std::lock_guard<std::mutex> lk(g_attrs_mu);
  if (g_attrs_done[dev]) return FIND_OK;
  const int mx = (int)kMaxSmem;
  CUDA_TRY(cudaFuncSetAttribute(small_elim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CUDA_TRY(cudaFuncSetAttribute(zgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Tile64::SMEM));
  CUDA_TRY(cudaFuncSetAttribute(mid_elim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CUDA_TRY(cudaFuncSetAttribute(panel_smem_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));

  CUDA_TRY(cudaFuncSetAttribute(panel_smem_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CUDA_TRY(cudaFuncSetAttribute(panel_smem_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CUDA_TRY(cudaFuncSetAttribute(panel_smem_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CUDA_TRY(cudaFuncSetAttribute(trsm_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)trsm_smem<4>()));
  CUDA_TRY(cudaFuncSetAttribute(panel_inv_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CUDA_TRY(cudaFuncSetAttribute(panel_inv_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CUDA_TRY(cudaFuncSetAttribute(panel_inv_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CUDA_TRY(cudaFuncSetAttribute(panel_inv_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CUDA_TRY(cudaFuncSetAttribute(xsolve_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xsolve_smem<4>()));
  CUDA_TRY(cudaFuncSetAttribute(trsm_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)trsm_smem<32>()));
  CUDA_TRY(cudaFuncSetAttribute(trsm_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)trsm_smem<16>()));
  CUDA_TRY(cudaFuncSetAttribute(trsm_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)trsm_smem<8>()));
  CUDA_TRY(cudaFuncSetAttribute(trail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Tile64::SMEM));
  CUDA_TRY(cudaFuncSetAttribute(tgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Tile64::SMEM));
  CUDA_TRY(cudaFuncSetAttribute(rgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Tile64::SMEM));
  CUDA_TRY(cudaFuncSetAttribute(schur_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Tile64::SMEM));
  CUDA_TRY(cudaFuncSetAttribute(xsolve_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xsolve_smem<32>()));
  CUDA_TRY(cudaFuncSetAttribute(xsolve_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xsolve_smem<16>()));
  CUDA_TRY(cudaFuncSetAttribute(xsolve_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xsolve_smem<8>()));
  CUDA_TRY(cudaFuncSetAttribute(finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CUDA_TRY(cudaFuncSetAttribute(final_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CUDA_TRY(cudaFuncSetAttribute(offdiag_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  CUDA_TRY(cudaFuncSetAttribute(panel_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)cluster_panel_smem()));
  CUDA_TRY(cudaFuncSetAttribute(offdiag_small_kernel<32, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)offdiag_small_smem<32>()));
  CUDA_TRY(cudaFuncSetAttribute(offdiag_small_kernel<64, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)offdiag_small_smem<64>()));
  CUDA_TRY(cudaFuncSetAttribute(tile_tma_kernel<kLTrail>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TmaEng::SMEM));
  CUDA_TRY(cudaFuncSetAttribute(tile_tma_kernel<kLTrail, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)dmma::Eng64cs::SMEM));
  CUDA_TRY(cudaFuncSetAttribute(tile_tma_kernel<kLSchur>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TmaEng::SMEM));
  CUDA_TRY(cudaFuncSetAttribute(tile_tma_kernel<kLTGemm>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TmaEng::SMEM));
  CUDA_TRY(cudaFuncSetAttribute(tile_tma_kernel<kLRGemm>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TmaEng::SMEM));
  g_attrs_done[dev] = true;
  return FIND_OK;
}

// Side streams for the concurrent groups of a phase (per device, created once):
// kSideStreams at normal priority and kHiStreams at the device's greatest
// priority for the groups on the phase's critical path (the longest launch
// chains), whose CTAs the scheduler then places first.
constexpr int kSideStreams = 16;
constexpr int kHiStreams = 8;
struct SideStreams {
  int device = -1;
  cudaStream_t s[kSideStreams + kHiStreams] = {};
  cudaEvent_t fork[64] = {}, join[64] = {};
  int next = 0;
  cudaStream_t joiner = nullptr;     // dependency scheduling: per-phase join events are recorded here
  std::vector<cudaEvent_t> gev, jev;  // per launch group / per phase completion
};
// one set per device; g_side_mu[dev] is held while a solve enqueues on that device's side streams
SideStreams g_sides[kMaxDevices];
std::mutex g_side_mu[kMaxDevices];

int side_init(SideStreams& g_side, int dev, find_status* st) {
  if (g_side.device == dev) return FIND_OK;
  int least = 0, greatest = 0;
  CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  for (int i = 0; i < kSideStreams + kHiStreams; ++i)
    CUDA_TRY(cudaStreamCreateWithPriority(&g_side.s[i], cudaStreamNonBlocking, i < kSideStreams ? least : greatest));
  for (int i = 0; i < 64; ++i) {
    CUDA_TRY(cudaEventCreateWithFlags(&g_side.fork[i], cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&g_side.join[i], cudaEventDisableTiming));
  }
  CUDA_TRY(cudaStreamCreateWithFlags(&g_side.joiner, cudaStreamNonBlocking));
  g_side.device = dev;
  return FIND_OK;
}

int run_one_group(const find_plan* P, const SolveParams& prm, int64_t gi, int nE, cudaStream_t stream,
                  find_status* st);
// NB = 32 panel steps up to kRegPanelMaxS rows: register rows with one barrier per column, or the
// CTA with shared-memory rows (FIND_B200_SMEM_PANEL=1)
const bool g_reg_panel = [] {
  const char* f = std::getenv("FIND_B200_SMEM_PANEL");
  return !(f && f[0] == '1');
}();

// Diagonal-block inverses once per (elimination, panel) in their own launch (default), or
// recomputed by every TRSM tile that needs one (FIND_B200_INV_LAUNCH=0).
const bool g_inv_launch = [] {
  const char* f = std::getenv("FIND_B200_INV_LAUNCH");
  return !(f && f[0] == '0');
}();

// Structural-zero skips (ElimDesc::zsplit), on unless FIND_B200_STRUCT=0.
const bool g_zskip = [] {
  const char* f = std::getenv("FIND_B200_STRUCT");
  return !(f && f[0] == '0');
}();

// Opt-in per-launch timing (find_solve_timing_enable): one event pair per launch.
struct LaunchTimer {
  bool on = false;
  std::vector<cudaEvent_t> ev;  // 2 per launch
  std::vector<int32_t> kind;
  std::vector<int32_t> group;
  size_t used = 0;
};
LaunchTimer g_timer;

int timer_mark(cudaStream_t stream, int32_t kind, int32_t group, bool begin, find_status* st) {
  if (!g_timer.on) return FIND_OK;
  if (begin) {
    if (2 * g_timer.used + 2 > g_timer.ev.size()) {
      for (int k = 0; k < 64; ++k) {
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreate(&e));
        g_timer.ev.push_back(e);
      }
    }
    g_timer.kind.resize(g_timer.used + 1);
    g_timer.group.resize(g_timer.used + 1);
    g_timer.kind[g_timer.used] = kind;
    g_timer.group[g_timer.used] = group;
    CUDA_TRY(cudaEventRecord(g_timer.ev[2 * g_timer.used], stream));
  } else {
    CUDA_TRY(cudaEventRecord(g_timer.ev[2 * g_timer.used + 1], stream));
    ++g_timer.used;
  }
  return FIND_OK;
}

// critical-path groups on high-priority streams (FIND_B200_PRIO=0 disables)
const bool g_prio = [] {
  const char* f = std::getenv("FIND_B200_PRIO");
  return !(f && f[0] == '0');
}();

// Dependency scheduling (plans built with dag): every group waits only for the groups that
// produce its input blocks and for every group two or more phases back (the scratch half and
// the down arena it reuses), so a phase's tail overlaps the next phase's first launches.
// FIND_B200_DAG=0 falls back to phase barriers.
const bool g_dag = [] {
  const char* f = std::getenv("FIND_B200_DAG");
  return !(f && f[0] == '0');
}();

int grow_events(std::vector<cudaEvent_t>& v, size_t n, find_status* st) {
  while (v.size() < n) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    v.push_back(e);
  }
  return FIND_OK;
}

int run_groups_dag(const find_plan* P, const SolveParams& prm, int64_t g_begin, int64_t g_end, int nE,
                   cudaStream_t stream, SideStreams& g_side, find_status* st) {
  const int np = P->groups.back().phase + 1;
  int rc = grow_events(g_side.gev, P->groups.size(), st);
  if (!rc) rc = grow_events(g_side.jev, (size_t)np, st);
  if (rc) return rc;
  const int slot = g_side.next;
  g_side.next = (g_side.next + 1) % 64;
  CUDA_TRY(cudaEventRecord(g_side.fork[slot], stream));
  for (int k = 0; k < kSideStreams + kHiStreams; ++k) CUDA_TRY(cudaStreamWaitEvent(g_side.s[k], g_side.fork[slot], 0));
  CUDA_TRY(cudaStreamWaitEvent(g_side.joiner, g_side.fork[slot], 0));
  const int p_first = P->groups[g_begin].phase;
  int lo = 0, hi = 0, last_phase = p_first;
  int64_t gi = g_begin;
  while (gi < g_end) {
    int64_t ge = gi;
    const int p = P->groups[gi].phase;
    while (ge < g_end && P->groups[ge].phase == p) ++ge;
    int64_t longest = 0;
    for (int64_t g = gi; g < ge; ++g) longest = std::max(longest, P->groups[g].spec_end - P->groups[g].spec_begin);
    for (int pass = 0; pass < 2; ++pass)  // critical chains first, on the high-priority streams
      for (int64_t g = gi; g < ge; ++g) {
        const bool crit = g_prio && 4 * (P->groups[g].spec_end - P->groups[g].spec_begin) >= 3 * longest;
        if (crit != (pass == 0)) continue;
        cudaStream_t sg = crit ? g_side.s[kSideStreams + (hi++ % kHiStreams)] : g_side.s[lo++ % kSideStreams];
        for (int32_t dgp : P->group_deps[g])
          if (dgp >= g_begin && dgp < g) CUDA_TRY(cudaStreamWaitEvent(sg, g_side.gev[dgp], 0));
        if (p - 2 >= p_first) CUDA_TRY(cudaStreamWaitEvent(sg, g_side.jev[p - 2], 0));
        if ((rc = run_one_group(P, prm, g, nE, sg, st))) return rc;
        CUDA_TRY(cudaEventRecord(g_side.gev[g], sg));
      }
    for (int64_t g = gi; g < ge; ++g) CUDA_TRY(cudaStreamWaitEvent(g_side.joiner, g_side.gev[g], 0));
    CUDA_TRY(cudaEventRecord(g_side.jev[p], g_side.joiner));  // every group of phases <= p done
    last_phase = p;
    gi = ge;
  }
  CUDA_TRY(cudaStreamWaitEvent(stream, g_side.jev[last_phase], 0));
  return FIND_OK;
}

// Enqueue the launches of groups [g_begin, g_end): phase by phase; the groups
// of a phase fork onto side streams and join back into `stream`.
int run_groups(const find_plan* P, const SolveParams& prm, int64_t g_begin, int64_t g_end, int nE,
               cudaStream_t stream, find_status* st) {
  int rc = set_attrs(st);
  if (rc) return rc;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_side_mu[dev]);
  SideStreams& g_side = g_sides[dev];
  if ((rc = side_init(g_side, dev, st))) return rc;
  if (P->dag && g_dag && g_end > g_begin) return run_groups_dag(P, prm, g_begin, g_end, nE, stream, g_side, st);
  int64_t gi = g_begin;
  while (gi < g_end) {
    int64_t ge = gi;
    while (ge < g_end && P->groups[ge].phase == P->groups[gi].phase) ++ge;
    if (ge - gi == 1) {
      if ((rc = run_one_group(P, prm, gi, nE, stream, st))) return rc;
    } else {
      // critical groups: launch chains at least 3/4 as long as the phase's longest
      int64_t longest = 0;
      for (int64_t g = gi; g < ge; ++g) longest = std::max(longest, P->groups[g].spec_end - P->groups[g].spec_begin);
      const int slot = g_side.next;
      g_side.next = (g_side.next + 1) % 64;
      CUDA_TRY(cudaEventRecord(g_side.fork[slot], stream));
      bool used[kSideStreams + kHiStreams] = {};
      int nlo = 0, nhi = 0;
      std::vector<int> sid((size_t)(ge - gi));
      for (int64_t g = gi; g < ge; ++g) {
        const int64_t len = P->groups[g].spec_end - P->groups[g].spec_begin;
        const bool hi = g_prio && 4 * len >= 3 * longest;
        sid[(size_t)(g - gi)] = hi ? kSideStreams + (nhi++ % kHiStreams) : (nlo++ % kSideStreams);
      }
      for (int64_t g = gi; g < ge; ++g) {
        const int k = sid[(size_t)(g - gi)];
        if (!used[k]) {
          used[k] = true;
          CUDA_TRY(cudaStreamWaitEvent(g_side.s[k], g_side.fork[slot], 0));
        }
      }
      // critical chains first so their first launches are queued ahead of the rest
      for (int pass = 0; pass < 2; ++pass)
        for (int64_t g = gi; g < ge; ++g) {
          const int k = sid[(size_t)(g - gi)];
          if ((k >= kSideStreams) != (pass == 0)) continue;
          if ((rc = run_one_group(P, prm, g, nE, g_side.s[k], st))) return rc;
        }
      for (int k = 0, js = 0; k < kSideStreams + kHiStreams; ++k) {
        if (!used[k]) continue;
        const int ev = (slot + 1 + js++) % 64;
        CUDA_TRY(cudaEventRecord(g_side.join[ev], g_side.s[k]));
        CUDA_TRY(cudaStreamWaitEvent(stream, g_side.join[ev], 0));
      }
    }
    gi = ge;
  }
  return FIND_OK;
}

// profiling hook (results invalid): FIND_B200_SKIP=tall skips blocked groups with s >= 128 and b <= 64,
// FIND_B200_SKIP=other skips every other group
const int g_skip = [] {
  const char* f = std::getenv("FIND_B200_SKIP");
  if (!f) return 0;
  return std::string(f) == "tall" ? 1 : (std::string(f) == "other" ? 2 : 0);
}();

// persistent grid of the TMA tile kernels: one CTA per SM at most (a CTA holds ~132 KB of smem)
int g_num_sms[kMaxDevices] = {};
// FIND_B200_TMA_SMS: CTAs of a TMA tile launch (default: every SM); fewer leave SMs to the
// latency-bound launches of the concurrent groups
const int g_tma_sms = [] {
  const char* f = std::getenv("FIND_B200_TMA_SMS");
  return f ? std::atoi(f) : 0;
}();
dim3 tma_grid(unsigned cnt, int nE) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (g_num_sms[dev] == 0) cudaDeviceGetAttribute(&g_num_sms[dev], cudaDevAttrMultiProcessorCount, dev);
  const int64_t total = (int64_t)cnt * nE;
  const int sms = g_tma_sms > 0 ? std::min(g_tma_sms, g_num_sms[dev]) : g_num_sms[dev];
  return dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(total, sms)), 1);
}

// NB = 32 panels of more than kRegPanelMaxS rows on register-row clusters (FIND_B200_CREG=0: the
// shared-memory-row panel / cluster kernels)
const bool g_creg = [] {
  const char* f = std::getenv("FIND_B200_CREG");
  return !(f && f[0] == '0');
}();

// TMA engine switch (FIND_B200_TMA=0: the cp.async tile kernels everywhere)
const bool g_tma = [] {
  const char* f = std::getenv("FIND_B200_TMA");
  return !(f && f[0] == '0');
}();
// Launch groups that use the engine.  Measured per group on cfg4 / cfg1 (tools/group_kinds.py,
// gpurun_out/t_gk*: every max_s bucket): with the predicate-free full-chunk path and the dynamic
// tile order the engine is faster than the 2-CTA/SM cp.async tiles on every Schur / T / R group
// (cfg4 serialized: rgemm 885 -> 821 ms, schur 522 -> 469, tgemm 391 -> 360) and on the trailing
// updates (1970 -> 1637 ms), so it runs all of them; FIND_B200_TMA_MIN_S / _TRAIL_MIN_N raise the
// group-size bounds for A/B runs.
const int g_tma_min_s = [] {
  const char* f = std::getenv("FIND_B200_TMA_MIN_S");
  return f ? std::atoi(f) : 192;  // below: cfg4 loses < 1 % serialized, cfg1 (latency-bound, many small concurrent groups) gains 2 %
}();
// ... or launches of at least this many tiles whatever their s (cfg4's boundary-carrying eliminations: tens of
// thousands of tiles per launch, where the engine wins; cfg1's stay below)
const int64_t g_tma_min_tiles = [] {
  const char* f = std::getenv("FIND_B200_TMA_MIN_TILES");
  return f ? std::atoll(f) : 16384;
}();
const int g_tma_trail_min_n = [] {
  const char* f = std::getenv("FIND_B200_TMA_TRAIL_MIN_N");
  return f ? std::atoi(f) : 0;
}();

// One-CTA tall panels (panel_tall_kernel): for panel steps with more than g_tall_min_rows rows
// when the launch holds at least g_tall_min_panels (elimination, energy) panels.
const int g_tall_min_rows = [] {
  const char* f = std::getenv("FIND_B200_TALL_MIN_ROWS");
  return f ? std::atoi(f) : (int)kRegPanelMaxS;
}();
const int64_t g_tall_min_panels = [] {
  const char* f = std::getenv("FIND_B200_TALL_MIN_PANELS");
  return f ? std::atoll(f) : 48;
}();

bool use_tall_panel(const LaunchGroup& G, const LaunchSpec& L, int nE) {
  const int rmax = G.max_s - L.step * L.nb;  // rows of this step's largest panel
  return L.nb == 32 && rmax > g_tall_min_rows && rmax <= kTallMaxRows && L.task_count * nE >= g_tall_min_panels;
}
// rows per thread and CTA size of a tall panel launch
void tall_shape(const LaunchGroup& G, const LaunchSpec& L, int& rpt, int& T) {
  const int rmax = G.max_s - L.step * L.nb;
  rpt = rmax <= kTallMaxT ? 1 : (rmax <= 2 * kTallMaxT ? 2 : 3);
  T = 32 * (((rmax + rpt - 1) / rpt + 31) / 32);
}

// Trailing updates with the C block staged through the TMA unit (FIND_B200_CSTAGE=1; dmma_engine.cuh:
// faster standalone, slower inside the solver)
const bool g_cstage = [] {
  const char* f = std::getenv("FIND_B200_CSTAGE");
  return f && f[0] == '1';
}();

const bool g_rsym_down = [] {
  const char* f = std::getenv("FIND_B200_RSYM_DOWN");
  return f && f[0] == '1';
}();

int run_one_group(const find_plan* P, const SolveParams& prm_in, int64_t gi, int nE, cudaStream_t stream,
                  find_status* st) {
  const Task* dtasks = (const Task*)P->d_tasks;
  {
    const LaunchGroup& G = P->groups[gi];
    if (g_skip) {
      const bool tall = G.path == 1 && G.max_s >= 128 && G.max_b <= 64;
      if ((g_skip == 1) == tall) return FIND_OK;
    }
    // The lower-triangle (mirrored) R mode is used in the upward pass only: in the
    // downward recurrence the re-symmetrised blocks drift from the general result
    // level after level (2.3e-3 relative at 256x1024, tools/bisect_gl.py), while
    // the upward pass agrees to roundoff.
    SolveParams prm = prm_in;
    if (G.pass != 0 && !g_rsym_down) prm.rsym = 0;
    if (G.path == 1 && G.nb == 0) return fail_status(st, FIND_EINVAL, "elimination block too large for this build");
    for (int64_t si = G.spec_begin; si < G.spec_end; ++si) {
      const LaunchSpec& L = P->specs[si];
      if (!prm.compute_gless && (L.kind == kLGatherS || L.kind == kLTGemm || L.kind == kLRGemm)) continue;
      if (L.kind == kLPanelInv && !g_inv_launch) continue;
      // sigma comes from the last panel's inverse launch; the finish launch remains for the
      // unit-test shim's L output (and when the inverse launches are off)
      if (L.kind == kLFinish && g_inv_launch && !prm.dbg_l) continue;
      const Task* tk = dtasks + L.task_off;
      const unsigned cnt = (unsigned)L.task_count;
      const dim3 grid(cnt, (unsigned)nE);
      if (int rt = timer_mark(stream, L.kind, (int32_t)gi, true, st)) return rt;
      switch (L.kind) {
        case kLSmall: {
          SolveParams p = prm;
          p.elims = prm.elims + L.task_off;
          p.elim_base = L.task_off;
          const int nmax = std::max(1, G.max_n), ld = nmax + 1;
          // X [b][s], plus U_f [b][b] for final steps (pass 2 groups hold exactly those)
          const int xcap = G.max_b * G.max_s + (G.pass == 2 ? G.max_b * G.max_b : 0);
          const size_t smem = (size_t)kSmallWarps * small_warp_elems(nmax, ld, xcap) * sizeof(double2);
          launch_k(small_elim_kernel, dim3((unsigned)((L.task_count + kSmallWarps - 1) / kSmallWarps), (unsigned)nE), kSmallWarps * 32, smem, stream, p, L.task_count, nmax, ld, xcap);
          break;
        }
        case kLMid: {
          SolveParams p = prm;
          p.elims = prm.elims + L.task_off;
          p.elim_base = L.task_off;
          const int nmax = std::max(1, G.max_n);
          const int xcap = G.max_b * G.max_s + (G.pass == 2 ? G.max_b * G.max_b : 0);  // X, U_f of final steps
          const size_t smem = (size_t)mid_smem_elems(nmax, xcap) * sizeof(double2);
          launch_k(mid_elim_kernel, dim3((unsigned)L.task_count, (unsigned)nE), kMidThreads, smem, stream, p, L.task_count, nmax,
                                                                                                   xcap);
          break;
        }
        case kLGatherA: launch_k(gather_kernel<false>, grid, kThreads, 0, stream, prm, tk); break;
        case kLGatherS: launch_k(gather_kernel<true>, grid, kThreads, 0, stream, prm, tk); break;
        case kLPanel: {
          const int rmax = G.max_s - L.step * L.nb;  // rows of this step's largest panel
          if (use_tall_panel(G, L, nE)) {
            // many tall panels in flight: one CTA per panel (SM-time, not latency, is what counts).
            // (Running the diagonal-block inverses in the same launch measured neutral: the panel CTA
            // holds its SM that much longer.)
            int rpt, T;
            tall_shape(G, L, rpt, T);
            if (rpt == 1) launch_k(panel_tall_kernel<1>, grid, T, 0, stream, prm, tk);
            else if (rpt == 2) launch_k(panel_tall_kernel<2>, grid, T, 0, stream, prm, tk);
            else launch_k(panel_tall_kernel<3>, grid, T, 0, stream, prm, tk);
          } else if (L.nb == 32 && g_creg && rmax > (int)kRegPanelMaxS && rmax <= kClusterMax * kRegClusterRows) {
            // register rows over a thread-block cluster of cs CTAs
            const unsigned cs = (unsigned)((rmax + kRegClusterRows - 1) / kRegClusterRows);
            const int rows = (rmax + (int)cs - 1) / (int)cs;
            const dim3 cg(cnt * cs, (unsigned)nE);
            switch ((rows + 31) / 32) {
              case 1: launch_cluster(panel_cluster_reg_kernel<32>, cg, 32, cs, 0, stream, prm, tk); break;
              case 2: launch_cluster(panel_cluster_reg_kernel<64>, cg, 64, cs, 0, stream, prm, tk); break;
              case 3: launch_cluster(panel_cluster_reg_kernel<96>, cg, 96, cs, 0, stream, prm, tk); break;
              case 4: launch_cluster(panel_cluster_reg_kernel<128>, cg, 128, cs, 0, stream, prm, tk); break;
              case 5: launch_cluster(panel_cluster_reg_kernel<160>, cg, 160, cs, 0, stream, prm, tk); break;
              case 6: launch_cluster(panel_cluster_reg_kernel<192>, cg, 192, cs, 0, stream, prm, tk); break;
              case 7: launch_cluster(panel_cluster_reg_kernel<224>, cg, 224, cs, 0, stream, prm, tk); break;
              default: launch_cluster(panel_cluster_reg_kernel<256>, cg, 256, cs, 0, stream, prm, tk); break;
            }
          } else if (L.nb == 32 && rmax > (int)kSmemPanelMaxS32) {  // rows over a thread-block cluster
            const unsigned cs = (unsigned)((rmax + kClusterRows - 1) / kClusterRows);
            if (cs > (unsigned)kClusterMax) return fail_status(st, FIND_EINVAL, "panel too tall for one cluster");
            launch_cluster(panel_cluster_kernel, dim3(cnt * cs, (unsigned)nE), kThreads, cs, cluster_panel_smem(), stream,
                           prm, tk);
          } else if (L.nb == 32 && rmax > (int)kRegPanelMaxS) {  // more rows than the register panel holds
            launch_k(panel_smem_kernel<32>, grid, kThreads, (size_t)rmax * 33 * sizeof(double2), stream, prm, tk);
          } else if (L.nb == 32 && g_reg_panel) {
            switch ((std::max(rmax, 1) + 31) / 32) {
              case 1: launch_k(panel1_kernel<32, 32>, grid, 32, 0, stream, prm, tk); break;
              case 2: launch_k(panel1_kernel<32, 64>, grid, 64, 0, stream, prm, tk); break;
              case 3: launch_k(panel1_kernel<32, 96>, grid, 96, 0, stream, prm, tk); break;
              case 4: launch_k(panel1_kernel<32, 128>, grid, 128, 0, stream, prm, tk); break;
              case 5: launch_k(panel1_kernel<32, 160>, grid, 160, 0, stream, prm, tk); break;
              case 6: launch_k(panel1_kernel<32, 192>, grid, 192, 0, stream, prm, tk); break;
              case 7: launch_k(panel1_kernel<32, 224>, grid, 224, 0, stream, prm, tk); break;
              case 8: launch_k(panel1_kernel<32, 256>, grid, 256, 0, stream, prm, tk); break;
              default: launch_k(panel1_kernel<32, 288>, grid, 288, 0, stream, prm, tk); break;
            }
          } else if (L.nb == 32)
            launch_k(panel_smem_kernel<32>, grid, kThreads, (size_t)std::max(rmax, 1) * 33 * sizeof(double2), stream, prm, tk);
          else if (L.nb == 16)
            launch_k(panel_smem_kernel<16>, grid, kThreads, (size_t)G.max_s * 17 * sizeof(double2), stream, prm, tk);
          else if (L.nb == 8)
            launch_k(panel_smem_kernel<8>, grid, kThreads, (size_t)G.max_s * 9 * sizeof(double2), stream, prm, tk);
          else launch_k(panel_smem_kernel<4>, grid, kThreads, (size_t)G.max_s * 5 * sizeof(double2), stream, prm, tk);
          break;
        }
        case kLPanelInv:
        {
          const size_t si = (size_t)G.max_s * sizeof(int);  // + sigma scratch (last panel)
          if (L.nb == 32) launch_k(panel_inv_kernel<32>, grid, kThreads, 5 * 32 * 33 * sizeof(double2) + si, stream, prm, tk);
          else if (L.nb == 16) launch_k(panel_inv_kernel<16>, grid, kThreads, 5 * 16 * 17 * sizeof(double2) + si, stream, prm, tk);
          else if (L.nb == 8) launch_k(panel_inv_kernel<8>, grid, kThreads, 5 * 8 * 9 * sizeof(double2) + si, stream, prm, tk);
          else launch_k(panel_inv_kernel<4>, grid, kThreads, 5 * 4 * 5 * sizeof(double2) + si, stream, prm, tk);
        }
          break;
        case kLTrsm: {
          const int ir = g_inv_launch ? 1 : 0;  // inverses published by the kLPanelInv launch
          if (L.nb == 32)
            launch_k(trsm_kernel<32>, grid, kThreads, trsm_smem<32>(), stream, prm, tk, L.step, ir);
          else if (L.nb == 16) launch_k(trsm_kernel<16>, grid, kThreads, trsm_smem<16>(), stream, prm, tk, L.step, ir);
          else if (L.nb == 8) launch_k(trsm_kernel<8>, grid, kThreads, trsm_smem<8>(), stream, prm, tk, L.step, ir);
          else launch_k(trsm_kernel<4>, grid, kThreads, trsm_smem<4>(), stream, prm, tk, L.step, ir);
          break;
        }
        case kLTrail:
          if (prm.use_tma && G.max_n >= g_tma_trail_min_n)
            if (g_cstage)
              launch_k(tile_tma_kernel<kLTrail, true>, tma_grid(cnt, nE), TmaEng::THREADS, dmma::Eng64cs::SMEM, stream, prm,
                       tk, (int64_t)cnt, nE, L.step, L.nb, prm.tile_ctr + si);
            else
              launch_k(tile_tma_kernel<kLTrail>, tma_grid(cnt, nE), TmaEng::THREADS, TmaEng::SMEM, stream, prm, tk,
                       (int64_t)cnt, nE, L.step, L.nb, prm.tile_ctr + si);
          else
            launch_k(trail_kernel, grid, kThreads, Tile64::SMEM, stream, prm, tk, L.step, L.nb);
          break;
        case kLXSolve:
          if (L.nb == 32) launch_k(xsolve_kernel<32>, grid, kThreads, xsolve_smem<32>(), stream, prm, tk);
          else if (L.nb == 16) launch_k(xsolve_kernel<16>, grid, kThreads, xsolve_smem<16>(), stream, prm, tk);
          else if (L.nb == 8) launch_k(xsolve_kernel<8>, grid, kThreads, xsolve_smem<8>(), stream, prm, tk);
          else launch_k(xsolve_kernel<4>, grid, kThreads, xsolve_smem<4>(), stream, prm, tk);
          break;
        case kLFinish:
          launch_k(finish_kernel, grid, kThreads, std::max<size_t>((size_t)G.max_s * sizeof(int), 16), stream, prm, tk, L.nb);
          break;
        case kLTGemm:
          if (prm.use_tma && (G.max_s >= g_tma_min_s || (int64_t)cnt * nE >= g_tma_min_tiles))
            launch_k(tile_tma_kernel<kLTGemm>, tma_grid(cnt, nE), TmaEng::THREADS, TmaEng::SMEM, stream, prm, tk,
                     (int64_t)cnt, nE, 0, L.nb, prm.tile_ctr + si);
          else
            launch_k(tgemm_kernel, grid, kThreads, Tile64::SMEM, stream, prm, tk, L.nb);
          break;
        case kLRGemm:
          if (prm.use_tma && (G.max_s >= g_tma_min_s || (int64_t)cnt * nE >= g_tma_min_tiles))
            launch_k(tile_tma_kernel<kLRGemm>, tma_grid(cnt, nE), TmaEng::THREADS, TmaEng::SMEM, stream, prm, tk,
                     (int64_t)cnt, nE, 0, L.nb, prm.tile_ctr + si);
          else
            launch_k(rgemm_kernel, grid, kThreads, Tile64::SMEM, stream, prm, tk, L.nb);
          break;
        case kLSchur:
          if (prm.use_tma && (G.max_s >= g_tma_min_s || (int64_t)cnt * nE >= g_tma_min_tiles))
            launch_k(tile_tma_kernel<kLSchur>, tma_grid(cnt, nE), TmaEng::THREADS, TmaEng::SMEM, stream, prm, tk,
                     (int64_t)cnt, nE, 0, L.nb, prm.tile_ctr + si);
          else
            launch_k(schur_kernel, grid, kThreads, Tile64::SMEM, stream, prm, tk);
          break;
        case kLFinal: {
          const int cmax = std::max(1, G.max_b);
          const size_t smem = (size_t)kSmallWarps * 2 * cmax * (cmax + 1) * sizeof(double2);
          launch_k(final_kernel, dim3((cnt + kSmallWarps - 1) / kSmallWarps, (unsigned)nE), kSmallWarps * 32, smem, stream, 
              prm, tk, L.task_count, cmax);
          break;
        }
        default: return fail_status(st, FIND_EINVAL, "unknown launch kind");
      }
      CUDA_TRY(cudaGetLastError());
      if (int rt = timer_mark(stream, L.kind, (int32_t)gi, false, st)) return rt;
    }
    if (prm.off_gr && G.pass == 2) {  // off-diagonal extraction right after the group's final step
      if (G.max_b > kOffMaxC) return fail_status(st, FIND_EINVAL, "off-diagonal extraction supports leaves of <= 16 nodes");
      if (int rt = timer_mark(stream, kLOffdiag, (int32_t)gi, true, st)) return rt;
      const unsigned ne = (unsigned)nE;
      if (G.path == 1) {
        const LaunchSpec* fl = nullptr;
        for (int64_t si = G.spec_begin; si < G.spec_end; ++si)
          if (P->specs[si].kind == kLFinal) fl = &P->specs[si];
        if (!fl) return fail_status(st, FIND_EINVAL, "final group without a final launch");
        const bool gl = prm.off_gl != nullptr, gen = gl && prm.off_sym == 0;
        const int c = G.max_b, nc = gl ? (gen ? 3 * c : 2 * c) : c;
        const size_t smem = ((size_t)3 * c * (c + 1) + (size_t)G.max_s * nc + (size_t)G.nb * nc) * sizeof(double2);
        if (smem > kMaxSmem) return fail_status(st, FIND_EINVAL, "leaf ring too large for off-diagonal extraction");
        launch_k(offdiag_cta_kernel, dim3((unsigned)fl->task_count, ne), kOffT, smem, stream, prm, dtasks + fl->task_off,
                 G.nb);
      } else if (G.max_n <= 32) {
        launch_k(offdiag_small_kernel<32, 64>, dim3((unsigned)(G.end - G.begin), ne), 64, offdiag_small_smem<32>(), stream,
                 prm, G.begin);
      } else {
        if (G.max_n > 64) return fail_status(st, FIND_EINVAL, "unexpected final group size");
        launch_k(offdiag_small_kernel<64, 128>, dim3((unsigned)(G.end - G.begin), ne), 128, offdiag_small_smem<64>(),
                 stream, prm, G.begin);
      }
      CUDA_TRY(cudaGetLastError());
      if (int rt = timer_mark(stream, kLOffdiag, (int32_t)gi, false, st)) return rt;
    }
  }
  return FIND_OK;
}

// Every kernel launch of a full solve, in enqueue order: f(kind, step, group, tasks).
template <class F>
void for_each_launch(const find_plan* P, int nE, F f) {
  for (const LaunchGroup& G : P->groups) {
    for (int64_t si = G.spec_begin; si < G.spec_end; ++si) {
      if (P->specs[si].kind == kLPanelInv && !g_inv_launch) continue;
      if (P->specs[si].kind == kLFinish && g_inv_launch) continue;  // folded into the last inverse launch
      f(P->specs[si].kind, P->specs[si].step, P->specs[si].group, P->specs[si].task_count);
    }
  }
}

SolveParams make_params(const find_plan* P, void* ws, int nE) {
  SolveParams prm;
  std::memset(&prm, 0, sizeof(prm));
  unsigned char* base = (unsigned char*)ws;
  prm.elims = (const ElimDesc*)P->d_elims;
  prm.i32 = (const int32_t*)P->d_i32;
  prm.sparse = (const SparseEntry*)P->d_sparse;
  prm.nnz = P->nnz;
  prm.status = (unsigned long long*)base;
  size_t off = ws_header_bytes();
  for (int a = 0; a < kNumArenas; ++a) {
    prm.arena[a] = (double2*)(base + off);
    prm.arena_elems[a] = P->arena_elems[a];
    off += (size_t)nE * P->arena_elems[a] * sizeof(double2);
  }
  prm.scratch = (double2*)(base + off);
  prm.scratch_elems = P->ws_elems;
  off += (size_t)nE * P->ws_elems * sizeof(double2);
  prm.tile_ctr = (unsigned long long*)(base + off);
  prm.n_nodes = P->n;
  return prm;
}


// Complex-element offset of X inside an elimination's scratch (scratch_of with the group's nb).
int64_t x_offset(int64_t n, int64_t s, int nb) {
  const int64_t nn = n * n, ints = (3 * s + 264 + 3) / 4;
  const int64_t linv = 2 * nn + ints + 1 + (n + 2 * kRowChunk - 1) / (2 * kRowChunk);
  const int64_t blocks = nb ? (s + nb - 1) / nb * (int64_t)nb * nb : 0;
  return linv + 2 * blocks;
}

// Tensor maps {M, MS, X} of every CTA-path elimination for this scratch base and energy count,
// cached per plan (a few entries; an entry is never rewritten, so solves in flight on other
// streams keep valid maps).  The device copy is enqueued on `stream` (a memcpy node when the
// stream is being captured).  Leaves prm.use_tma = 0 when the maps are unavailable.
int ensure_tmaps(find_plan* P, SolveParams& prm, int nE, cudaStream_t stream, find_status* st) {
  prm.use_tma = 0;
  prm.tmaps = nullptr;
  if (!g_tma || P->n_tmap == 0) return FIND_OK;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  for (auto& E : P->tmap_cache)
    if (E.device == dev && E.scratch == prm.scratch && E.n_energies == nE) {
      E.stamp = ++P->tmap_clock;
      prm.tmaps = (const CUtensorMap*)E.dev;
      prm.use_tma = 1;
      return FIND_OK;
    }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CUDA_TRY(cudaStreamIsCapturing(stream, &cs));
  constexpr size_t kMaxEntries = 4;
  if (P->tmap_cache.size() >= kMaxEntries) {
    if (cs != cudaStreamCaptureStatusNone) return FIND_OK;  // no eviction inside a capture: cp.async tiles
    size_t lru = 0;
    for (size_t i = 1; i < P->tmap_cache.size(); ++i)
      if (P->tmap_cache[i].stamp < P->tmap_cache[lru].stamp) lru = i;
    CUDA_TRY(cudaDeviceSynchronize());  // the evicted maps may still be read by queued work
    auto& E = P->tmap_cache[lru];
    int cur = dev;
    if (E.device != dev) cudaSetDevice(E.device);
    cudaFree(E.dev);
    cudaFreeHost(E.host);
    if (E.device != dev) cudaSetDevice(cur);
    P->tmap_cache.erase(P->tmap_cache.begin() + (std::ptrdiff_t)lru);
  }
  const size_t bytes = (size_t)P->n_tmap * 3 * sizeof(CUtensorMap);
  find_plan::TmapEntry E;
  E.device = dev;
  E.scratch = prm.scratch;
  E.n_energies = nE;
  CUDA_TRY(cudaMallocHost(&E.host, bytes));
  if (cudaMalloc(&E.dev, bytes) != cudaSuccess) {
    cudaGetLastError();
    cudaFreeHost(E.host);
    return FIND_OK;  // no room: cp.async tiles
  }
  CUtensorMap* h = (CUtensorMap*)E.host;
  bool ok = true;
  for (const LaunchGroup& G : P->groups) {
    if (G.path != 1) continue;
    for (int64_t k = G.begin; k < G.end && ok; ++k) {
      const ElimDesc& d = P->elims[k];
      if (d.tmap < 0) continue;
      const double2* M = prm.scratch + d.ws_off;
      const int64_t n = d.n, s = d.s, b = d.b;
      CUtensorMap* t = h + 3 * (int64_t)d.tmap;
      ok = encode_complex_tmap(t + 0, M, n, n, n, P->ws_elems, nE) &&
           encode_complex_tmap(t + 1, M + n * n, n, n, n, P->ws_elems, nE) &&
           encode_complex_tmap(t + 2, M + x_offset(n, s, G.nb), std::max<int64_t>(s, 1), std::max<int64_t>(b, 1),
                               std::max<int64_t>(s, 1), P->ws_elems, nE);
    }
  }
  if (!ok) {
    cudaFree(E.dev);
    cudaFreeHost(E.host);
    return FIND_OK;
  }
  CUDA_TRY(cudaMemcpyAsync(E.dev, E.host, bytes, cudaMemcpyHostToDevice, stream));
  E.stamp = ++P->tmap_clock;
  P->tmap_cache.push_back(E);
  prm.tmaps = (const CUtensorMap*)E.dev;
  prm.use_tma = 1;
  return FIND_OK;
}

}  // namespace

extern "C" {

void find_plan_free_device(find_plan* P) {
  if (!P) return;
  if (P->d_elims) cudaFree(P->d_elims);
  if (P->d_i32) cudaFree(P->d_i32);
  if (P->d_sparse) cudaFree(P->d_sparse);
  if (P->d_tasks) cudaFree(P->d_tasks);
  if (P->d_off_items) cudaFree(P->d_off_items);
  if (P->d_off_item_off) cudaFree(P->d_off_item_off);
  P->d_elims = P->d_i32 = P->d_sparse = P->d_tasks = nullptr;
  P->d_off_items = P->d_off_item_off = nullptr;
  P->off_device = -1;
  P->device = -1;
  if (!P->tmap_cache.empty()) {
    cudaDeviceSynchronize();
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& E : P->tmap_cache) {
      cudaSetDevice(E.device);
      cudaFree(E.dev);
      cudaFreeHost(E.host);
    }
    cudaSetDevice(cur);
    P->tmap_cache.clear();
  }
}

int find_plan_upload(find_plan* P, find_status* st) {
  status_ok(st);
  if (!P) return FIND_EINVAL;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (P->d_elims && P->device == dev) return FIND_OK;
  find_plan_free_device(P);
  // tensor-map slots of the CTA-path eliminations (ensure_tmaps fills them per scratch base)
  for (auto& d : P->elims) d.tmap = -1;
  int32_t nt = 0;
  for (const LaunchGroup& G : P->groups)
    if (G.path == 1)
      for (int64_t k = G.begin; k < G.end; ++k) P->elims[k].tmap = nt++;
  P->n_tmap = nt;
  auto up = [&](void** dst, const void* src, size_t bytes) -> cudaError_t {
    cudaError_t e = cudaMalloc(dst, bytes ? bytes : 16);
    if (e != cudaSuccess) return e;
    if (bytes) e = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
    return e;
  };
  CUDA_TRY(up(&P->d_elims, P->elims.data(), P->elims.size() * sizeof(ElimDesc)));
  CUDA_TRY(up(&P->d_i32, P->i32.data(), P->i32.size() * sizeof(int32_t)));
  CUDA_TRY(up(&P->d_sparse, P->sparse.data(), P->sparse.size() * sizeof(SparseEntry)));
  CUDA_TRY(up(&P->d_tasks, P->tasks.data(), P->tasks.size() * sizeof(Task)));
  P->device = dev;
  return FIND_OK;
}

size_t find_solve_workspace_bytes(const find_plan* P, int32_t nE, int32_t compute_gless) {
  (void)compute_gless;
  if (!P || nE < 1) return 0;
  size_t b = ws_header_bytes();
  for (int a = 0; a < kNumArenas; ++a) b += (size_t)nE * P->arena_elems[a] * sizeof(double2);
  b += (size_t)nE * P->ws_elems * sizeof(double2);
  b += tile_ctr_bytes(P);
  return b;
}

int64_t find_solve_launch_count(const find_plan* P, int32_t nE) {
  if (!P) return 0;
  int64_t k = 0;
  for_each_launch(P, nE, [&](int32_t, int32_t, int32_t, int64_t) { ++k; });
  return k;
}

int find_plan_group_phases(const find_plan* P, int32_t* phase) {
  if (!P) return FIND_EINVAL;
  for (size_t g = 0; g < P->groups.size(); ++g)
    if (phase) phase[g] = P->groups[g].phase;
  return FIND_OK;
}

int find_plan_offdiag_build(find_plan* P);  // plan.cpp

int find_solve_offdiag_groups(find_plan* P, const void* a_vals, const void* s_vals, int32_t s_broadcast, int32_t nE,
                              int32_t compute_gless, double rtol, void* gr_out, void* gl_out, void* off_gr,
                              void* off_gl, void* ws, size_t ws_bytes, int64_t g_begin, int64_t g_end, void* stream_,
                              find_status* st) {
  status_ok(st);
  if (!P || !a_vals || !gr_out || !ws || nE < 1) return fail_status(st, FIND_EINVAL, "invalid argument");
  if (compute_gless && (!s_vals || !gl_out)) return fail_status(st, FIND_EINVAL, "compute_gless needs s_vals and gl_out");
  if (nE > 0xffff) return fail_status(st, FIND_EINVAL, "too many energy points in one call");
  if (ws_bytes < find_solve_workspace_bytes(P, nE, compute_gless)) return fail_status(st, FIND_ENOMEM, "workspace too small");
  if (off_gl && !compute_gless) return fail_status(st, FIND_EINVAL, "off_gl needs compute_gless");
  int rc = find_plan_upload(P, st);
  if (rc) return rc;
  if (off_gr) {
    try {
      if (find_plan_offdiag_build(P) != FIND_OK) return fail_status(st, FIND_EINVAL, "off-diagonal plan failed");
    } catch (const std::exception& ex) {
      return fail_status(st, FIND_ENOMEM, ex.what());
    }
    if (P->off_device != P->device) {
      if (P->d_off_items) cudaFree(P->d_off_items);
      if (P->d_off_item_off) cudaFree(P->d_off_item_off);
      P->d_off_items = P->d_off_item_off = nullptr;
      const size_t bi = std::max<size_t>(16, P->off_items.size() * sizeof(OffItem));
      const size_t bo = P->off_item_off.size() * sizeof(int64_t);
      CUDA_TRY(cudaMalloc(&P->d_off_items, bi));
      CUDA_TRY(cudaMalloc(&P->d_off_item_off, bo));
      if (!P->off_items.empty())
        CUDA_TRY(cudaMemcpy(P->d_off_items, P->off_items.data(), P->off_items.size() * sizeof(OffItem),
                            cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(P->d_off_item_off, P->off_item_off.data(), bo, cudaMemcpyHostToDevice));
      P->off_device = P->device;
    }
  }
  cudaStream_t stream = (cudaStream_t)stream_;
  SolveParams prm = make_params(P, ws, nE);
  prm.a_vals = (const double2*)a_vals;
  prm.s_vals = (const double2*)s_vals;
  prm.s_broadcast = s_broadcast;
  prm.compute_gless = compute_gless ? 1 : 0;
  prm.rsym = compute_gless == 2 ? 1 : (compute_gless == 3 ? -1 : 0);
  prm.rtol = rtol;
  prm.gr_out = (double2*)gr_out;
  prm.gl_out = (double2*)gl_out;
  prm.zskip = g_zskip ? 1 : 0;
  if (off_gr) {
    prm.off_gr = (double2*)off_gr;
    prm.off_gl = (double2*)off_gl;
    prm.off_items = (const OffItem*)P->d_off_items;
    prm.off_item_off = (const int64_t*)P->d_off_item_off;
    prm.n_pairs = (int64_t)P->off_u.size();
    prm.off_sym = prm.rsym;
  }
  if (g_begin < 0) g_begin = 0;
  if (g_end < 0 || g_end > (int64_t)P->groups.size()) g_end = (int64_t)P->groups.size();
  if (g_begin == 0) CUDA_TRY(cudaMemsetAsync(ws, 0xff, 8, stream));
  if ((rc = ensure_tmaps(P, prm, nE, stream, st))) return rc;
  if (prm.use_tma) CUDA_TRY(cudaMemsetAsync(prm.tile_ctr, 0, tile_ctr_bytes(P), stream));
  return run_groups(P, prm, g_begin, g_end, nE, stream, st);
}

int find_solve_offdiag(find_plan* P, const void* a_vals, const void* s_vals, int32_t s_broadcast, int32_t nE,
                       int32_t compute_gless, double rtol, void* gr_out, void* gl_out, void* off_gr, void* off_gl,
                       void* ws, size_t ws_bytes, void* stream_, find_status* st) {
  return find_solve_offdiag_groups(P, a_vals, s_vals, s_broadcast, nE, compute_gless, rtol, gr_out, gl_out, off_gr,
                                   off_gl, ws, ws_bytes, 0, -1, stream_, st);
}

int find_solve_groups(find_plan* P, const void* a_vals, const void* s_vals, int32_t s_broadcast, int32_t nE,
                      int32_t compute_gless, double rtol, void* gr_out, void* gl_out, void* ws, size_t ws_bytes,
                      int64_t g_begin, int64_t g_end, void* stream_, find_status* st) {
  return find_solve_offdiag_groups(P, a_vals, s_vals, s_broadcast, nE, compute_gless, rtol, gr_out, gl_out, nullptr,
                                   nullptr, ws, ws_bytes, g_begin, g_end, stream_, st);
}

int find_solve(find_plan* P, const void* a_vals, const void* s_vals, int32_t s_broadcast, int32_t nE,
               int32_t compute_gless, double rtol, void* gr_out, void* gl_out, void* ws, size_t ws_bytes,
               void* stream_, find_status* st) {
  return find_solve_groups(P, a_vals, s_vals, s_broadcast, nE, compute_gless, rtol, gr_out, gl_out, ws, ws_bytes, 0,
                           -1, stream_, st);
}

int find_plan_groups(const find_plan* P, int32_t* pass, int32_t* level, int32_t* path, int64_t* count,
                     int32_t* max_n, int32_t* max_s, int32_t* max_b) {
  if (!P) return FIND_EINVAL;
  for (size_t g = 0; g < P->groups.size(); ++g) {
    const LaunchGroup& G = P->groups[g];
    if (pass) pass[g] = G.pass;
    if (level) level[g] = G.level;
    if (path) path[g] = G.path;
    if (count) count[g] = G.end - G.begin;
    if (max_n) max_n[g] = G.max_n;
    if (max_s) max_s[g] = G.max_s;
    if (max_b) max_b[g] = G.max_b;
  }
  return FIND_OK;
}

int find_plan_specs(const find_plan* P, int32_t nE, int32_t* kind, int32_t* step, int32_t* group, int64_t* tasks) {
  if (!P) return FIND_EINVAL;
  int64_t i = 0;
  for_each_launch(P, nE, [&](int32_t k, int32_t s, int32_t g, int64_t t) {
    if (kind) kind[i] = k;
    if (step) step[i] = s;
    if (group) group[i] = g;
    if (tasks) tasks[i] = t;
    ++i;
  });
  return FIND_OK;
}

void find_solve_timing_enable(int32_t enable) {
  g_timer.on = enable != 0;
  if (g_timer.on) g_timer.used = 0;  // enabling clears the record; disabling keeps it for reading
}

int64_t find_solve_timing_read(int32_t* kind, int32_t* group, float* ms, int64_t cap) {
  const int64_t n = (int64_t)g_timer.used;
  for (int64_t i = 0; i < std::min(n, cap); ++i) {
    if (kind) kind[i] = g_timer.kind[i];
    if (group) group[i] = g_timer.group[i];
    if (ms) {
      float v = 0.f;
      if (cudaEventSynchronize(g_timer.ev[2 * i + 1]) == cudaSuccess)
        cudaEventElapsedTime(&v, g_timer.ev[2 * i], g_timer.ev[2 * i + 1]);
      ms[i] = v;
    }
  }
  return n;
}

int64_t find_solve_timing_read2(int32_t* kind, int32_t* group, float* t_begin, float* t_end, int64_t cap) {
  const int64_t n = (int64_t)g_timer.used;
  for (int64_t i = 0; i < std::min(n, cap); ++i) {
    if (kind) kind[i] = g_timer.kind[i];
    if (group) group[i] = g_timer.group[i];
    float a = 0.f, b = 0.f;
    if (cudaEventSynchronize(g_timer.ev[2 * i + 1]) == cudaSuccess) {
      cudaEventElapsedTime(&a, g_timer.ev[0], g_timer.ev[2 * i]);
      cudaEventElapsedTime(&b, g_timer.ev[0], g_timer.ev[2 * i + 1]);
    }
    if (t_begin) t_begin[i] = a;
    if (t_end) t_end[i] = b;
  }
  return n;
}

int find_solve_status(find_plan* P, void* ws, int32_t nE, void* stream_, find_status* st) {
  status_ok(st);
  if (!P || !ws) return FIND_EINVAL;
  unsigned long long key = ~0ull;
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream_));
  CUDA_TRY(cudaMemcpy(&key, ws, 8, cudaMemcpyDeviceToHost));
  if (key == ~0ull) return FIND_OK;
  const int64_t elim = (int64_t)(key >> 32);
  const int e = (int)((key >> 16) & 0xffff);
  const int pos = (int)(key & 0xffff);
  (void)nE;
  if (st) {
    st->code = FIND_ESINGULAR;
    st->energy_idx = e;
    if (elim >= 0 && elim < (int64_t)P->elims.size()) {
      const ElimDesc& d = P->elims[elim];
      st->cluster_label = d.label;
      if (pos == 0xfffe) {
        st->node_id = -1;
        std::snprintf(st->message, sizeof(st->message), "singular final block (cluster %lld, energy %d)",
                      (long long)d.label, e);
      } else {
        const int k = std::min(pos, std::max(d.s - 1, 0));
        st->node_id = d.s > 0 ? P->slabels[d.slabel_off + k] : -1;
        std::snprintf(st->message, sizeof(st->message),
                      "singular pivot at elimination position %d (cluster %lld, energy %d)", pos, (long long)d.label, e);
      }
    }
  }
  return FIND_ESINGULAR;
}

int find_schur_sigma_update(int32_t s, int32_t b, const void* ass, const void* asb, const void* abs_, const void* abb,
                            const void* sss, const void* ssb, const void* sbs, const void* sbb, double rtol,
                            void* u_out, void* r_out, void* l_out, int32_t force_path, void* stream_,
                            find_status* st) {
  status_ok(st);
  if (s < 0 || b < 0 || s + b < 1 || (b > 0 && !u_out)) return fail_status(st, FIND_EINVAL, "invalid sizes");
  cudaStream_t stream = (cudaStream_t)stream_;
  const int n = s + b;
  const bool gless = (r_out != nullptr || b == 0) && (s == 0 || sss) && (s == 0 || b == 0 || (ssb && sbs)) &&
                     (b == 0 || sbb);
  int path = force_path >= 0 ? force_path : (n <= 32 ? 0 : (n <= kMidMaxN ? 2 : 1));
  if (path == 0 && n > 32) path = 1;
  if (path == 2 && n > kMidMaxN) path = 1;
  // a one-elimination plan: left block = [[ass, asb], [abs, abb]] (+ Sigma), identity maps
  find_plan Q;
  Q.n = n;
  Q.nnz = 0;
  ElimDesc d;
  std::memset(&d, 0, sizeof(d));
  d.s = s; d.b = b; d.n = n; d.p = n; d.kind = kUpMerge; d.label = 1;
  d.left_arena = kArenaUp; d.left_off = 0; d.right_arena = kArenaNone; d.right_off = -1;
  d.out_arena = kArenaDown0; d.out_off = 0;
  d.map_off = 0; d.rank_off = n; d.sprow_off = n + b; d.sparse_off = 0; d.nsparse = 0; d.ws_off = 0;
  Q.i32.resize(n + b + n + 1, 0);
  for (int k = 0; k < n; ++k) Q.i32[k] = k;
  for (int k = 0; k < b; ++k) Q.i32[n + k] = k;
  Q.elims.push_back(d);
  Q.slabels.assign(std::max(s, 1), 0);
  for (int k = 0; k < s; ++k) Q.slabels[k] = k;
  LaunchGroup G;
  std::memset(&G, 0, sizeof(G));
  G.begin = 0; G.end = 1; G.path = path; G.max_n = n; G.max_s = s; G.max_b = b;
  G.nb = path == 1 ? pick_nb_host(s) : 0;
  if (path == 1 && G.nb == 0) return fail_status(st, FIND_EINVAL, "block too large");
  G.ws_elems = path == 1 ? find_scratch_elems(n, s, G.nb) : 0;
  Q.groups.push_back(G);
  Q.arena_elems[kArenaUp] = 2 * (int64_t)n * n;
  Q.arena_elems[kArenaDown0] = 2 * (int64_t)b * b + 2;
  Q.arena_elems[kArenaDown1] = 0;
  Q.arena_elems[kArenaDown2] = 0;
  Q.ws_elems = G.ws_elems;
  find_build_tasks(&Q);
  int rc = find_plan_upload(&Q, st);
  if (rc) { find_plan_free_device(&Q); return rc; }
  const size_t wsb = find_solve_workspace_bytes(&Q, 1, 1);
  void* ws = nullptr;
  cudaError_t ce = cudaMalloc(&ws, wsb);
  if (ce != cudaSuccess) { find_plan_free_device(&Q); return fail_status(st, FIND_ECUDA, cudaGetErrorString(ce)); }
  SolveParams prm = make_params(&Q, ws, 1);
  prm.compute_gless = gless;
  prm.rtol = rtol;
  prm.a_vals = prm.arena[kArenaUp];  // unused: no sparse entries
  prm.s_vals = prm.arena[kArenaUp];
  prm.s_broadcast = 1;
  prm.dbg_l = (double2*)l_out;
  double2* up = prm.arena[kArenaUp];
  auto put = [&](double2* dst, const void* src, int rows, int cols) -> cudaError_t {
    if (!rows || !cols) return cudaSuccess;
    return cudaMemcpy2DAsync(dst, (size_t)n * 16, src, (size_t)cols * 16, (size_t)cols * 16, rows,
                             cudaMemcpyDeviceToDevice, stream);
  };
  int out = FIND_OK;
  do {
    if ((ce = cudaMemsetAsync(ws, 0, wsb, stream)) != cudaSuccess) break;
    if ((ce = cudaMemsetAsync(ws, 0xff, 8, stream)) != cudaSuccess) break;
    if ((ce = put(up, ass, s, s)) != cudaSuccess) break;
    if ((ce = put(up + s, asb, s, b)) != cudaSuccess) break;
    if ((ce = put(up + (int64_t)s * n, abs_, b, s)) != cudaSuccess) break;
    if ((ce = put(up + (int64_t)s * n + s, abb, b, b)) != cudaSuccess) break;
    if (gless) {
      double2* rs = up + (int64_t)n * n;
      if ((ce = put(rs, sss, s, s)) != cudaSuccess) break;
      if ((ce = put(rs + s, ssb, s, b)) != cudaSuccess) break;
      if ((ce = put(rs + (int64_t)s * n, sbs, b, s)) != cudaSuccess) break;
      if ((ce = put(rs + (int64_t)s * n + s, sbb, b, b)) != cudaSuccess) break;
    }
    out = run_groups(&Q, prm, 0, 1, 1, stream, st);
    if (out) break;
    if (b && (ce = cudaMemcpyAsync(u_out, prm.arena[kArenaDown0], (size_t)b * b * 16, cudaMemcpyDeviceToDevice,
                                   stream)) != cudaSuccess) break;
    if (gless && b &&
        (ce = cudaMemcpyAsync(r_out, prm.arena[kArenaDown0] + (int64_t)b * b, (size_t)b * b * 16,
                              cudaMemcpyDeviceToDevice, stream)) != cudaSuccess) break;
    unsigned long long key = ~0ull;
    if ((ce = cudaMemcpyAsync(&key, ws, 8, cudaMemcpyDeviceToHost, stream)) != cudaSuccess) break;
    if ((ce = cudaStreamSynchronize(stream)) != cudaSuccess) break;
    if (key != ~0ull) {
      if (st) {
        st->code = FIND_ESINGULAR;
        st->node_id = (int64_t)(key & 0xffff);
        st->cluster_label = 0;
        st->energy_idx = 0;
        std::snprintf(st->message, sizeof(st->message), "singular pivot at elimination position %d", (int)(key & 0xffff));
      }
      out = FIND_ESINGULAR;
    }
  } while (0);
  cudaFree(ws);
  find_plan_free_device(&Q);
  if (ce != cudaSuccess) return fail_status(st, FIND_ECUDA, cudaGetErrorString(ce));
  return out;
}

// ---- dense batched primitives (include/find_b200.h)
struct find_dense {
  find_plan Q;
  int32_t n = 0, batch = 0;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  int device = -1;
};

void find_dense_destroy(find_dense* H) {
  if (!H) return;
  int cur = 0;
  cudaGetDevice(&cur);
  if (H->device >= 0 && H->device != cur) cudaSetDevice(H->device);
  if (H->ws) cudaFree(H->ws);
  find_plan_free_device(&H->Q);
  if (H->device >= 0 && H->device != cur) cudaSetDevice(cur);
  delete H;
}

int find_dense_create(int32_t n, int32_t batch, find_dense** out, find_status* st) {
  status_ok(st);
  if (!out || n < 1 || batch < 1 || batch > 0xffff) return fail_status(st, FIND_EINVAL, "invalid sizes");
  find_dense* H = new find_dense;
  H->n = n;
  H->batch = batch;
  const int n2 = 2 * n;
  find_plan& Q = H->Q;
  Q.n = n2;
  Q.nnz = 0;
  ElimDesc d;
  std::memset(&d, 0, sizeof(d));
  d.s = n; d.b = n; d.n = n2; d.p = n2; d.kind = kUpMerge; d.label = 1;
  d.left_arena = kArenaUp; d.left_off = 0; d.right_arena = kArenaNone; d.right_off = -1;
  d.out_arena = kArenaDown0; d.out_off = 0;
  d.map_off = 0; d.rank_off = n2; d.sprow_off = n2 + n; d.sparse_off = 0; d.nsparse = 0; d.ws_off = 0;
  Q.i32.resize((size_t)n2 + n + n2 + 1, 0);
  for (int k = 0; k < n2; ++k) Q.i32[k] = k;
  for (int k = 0; k < n; ++k) Q.i32[n2 + k] = k;
  Q.elims.push_back(d);
  Q.slabels.assign((size_t)n, 0);
  for (int k = 0; k < n; ++k) Q.slabels[k] = k;
  LaunchGroup G;
  std::memset(&G, 0, sizeof(G));
  const int path = n2 <= 32 ? 0 : (n2 <= kMidMaxN ? 2 : 1);
  G.begin = 0; G.end = 1; G.path = path; G.max_n = n2; G.max_s = n; G.max_b = n;
  G.nb = path == 1 ? pick_nb_host(n) : 0;
  if (path == 1 && G.nb == 0) {
    delete H;
    return fail_status(st, FIND_EINVAL, "block too large");
  }
  G.ws_elems = path == 1 ? find_scratch_elems(n2, n, G.nb) : 0;
  Q.groups.push_back(G);
  Q.arena_elems[kArenaUp] = 2 * (int64_t)n2 * n2;
  Q.arena_elems[kArenaDown0] = 2 * (int64_t)n * n + 2;
  Q.arena_elems[kArenaDown1] = 0;
  Q.arena_elems[kArenaDown2] = 0;
  Q.ws_elems = G.ws_elems;
  find_build_tasks(&Q);
  int rc = find_plan_upload(&Q, st);
  if (rc) { find_dense_destroy(H); return rc; }
  cudaGetDevice(&H->device);
  H->ws_bytes = find_solve_workspace_bytes(&Q, batch, 0);
  cudaError_t ce = cudaMalloc(&H->ws, H->ws_bytes);
  if (ce != cudaSuccess) {
    find_dense_destroy(H);
    return fail_status(st, FIND_ENOMEM, cudaGetErrorString(ce));
  }
  if ((ce = cudaMemset(H->ws, 0, H->ws_bytes)) != cudaSuccess) {
    find_dense_destroy(H);
    return fail_status(st, FIND_ECUDA, cudaGetErrorString(ce));
  }
  *out = H;
  return FIND_OK;
}

int find_dense_inverse(find_dense* H, const void* a, void* inv_out, void* status_out, void* stream_, find_status* st) {
  status_ok(st);
  if (!H || !a || !inv_out) return fail_status(st, FIND_EINVAL, "invalid argument");
  cudaStream_t stream = (cudaStream_t)stream_;
  SolveParams prm = make_params(&H->Q, H->ws, H->batch);
  prm.compute_gless = 0;
  prm.rtol = 1e-300;  // LAPACK getrf semantics: only an exactly zero pivot is singular
  prm.a_vals = prm.arena[kArenaUp];  // unused: no sparse entries
  prm.s_vals = prm.arena[kArenaUp];
  prm.s_broadcast = 1;
  const int n = H->n, n2 = 2 * n;
  CUDA_TRY(cudaMemsetAsync(H->ws, 0xff, 8, stream));
  const unsigned gx = (unsigned)std::min<int64_t>(((int64_t)n2 * n2 + kThreads - 1) / kThreads, 1184);
  dense_pack_kernel<<<dim3(gx, (unsigned)H->batch), kThreads, 0, stream>>>((const double2*)a, prm.arena[kArenaUp],
                                                                         H->Q.arena_elems[kArenaUp], n);
  CUDA_TRY(cudaGetLastError());
  int rc = run_groups(&H->Q, prm, 0, 1, H->batch, stream, st);
  if (rc) return rc;
  dense_unpack_kernel<<<dim3(gx, (unsigned)H->batch), kThreads, 0, stream>>>(prm.arena[kArenaDown0],
                                                                           H->Q.arena_elems[kArenaDown0],
                                                                           (double2*)inv_out, n);
  CUDA_TRY(cudaGetLastError());
  if (status_out) CUDA_TRY(cudaMemcpyAsync(status_out, H->ws, 8, cudaMemcpyDeviceToDevice, stream));
  return FIND_OK;
}

int find_zgemm_batched(int32_t batch, int32_t m, int32_t n, int32_t k, const void* A, int64_t lda, int64_t sa,
                       const void* B, int64_t ldb, int64_t sb, int32_t b_conj_trans, void* C, int64_t ldc, int64_t sc,
                       int32_t mode, void* stream_, find_status* st) {
  status_ok(st);
  if (batch < 1 || m < 1 || n < 1 || k < 0 || !A || !B || !C || batch > 0xffff)
    return fail_status(st, FIND_EINVAL, "invalid argument");
  int rc = set_attrs(st);
  if (rc) return rc;
  GemmArgs g;
  g.A = (const double2*)A; g.B = (const double2*)B; g.C = (double2*)C;
  g.lda = lda; g.sa = sa; g.ldb = ldb; g.sb = sb; g.ldc = ldc; g.sc = sc;
  g.m = m; g.n = n; g.k = k; g.bt = b_conj_trans ? 1 : 0; g.mode = mode;
  const unsigned tiles = (unsigned)(((m + kTile - 1) / kTile) * ((n + kTile - 1) / kTile));
  zgemm_kernel<<<dim3(tiles, (unsigned)batch), kThreads, Tile64::SMEM, (cudaStream_t)stream_>>>(g);
  CUDA_TRY(cudaGetLastError());
  return FIND_OK;
}

}  // extern "C"
