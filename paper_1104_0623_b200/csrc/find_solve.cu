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
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/find_b200.h"
#include "plan.h"

using namespace findb200;

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
  double rtol;
  double2* arena[3];
  int64_t arena_elems[3];
  double2* scratch;
  int64_t scratch_elems;
  double2* gr_out;  // [nE][n]
  double2* gl_out;
  int64_t n_nodes;
  unsigned long long* status;  // first failing (elim << 32 | energy << 16 | pos)
  int64_t elim_base;           // global index of elims[0] in the plan
  double2* dbg_l;              // unit-test shim only: L = A(B,S) A(S,S)^-1 (b x s), elimination 0 / energy 0
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
constexpr int kSmallWarps = 4;

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

__global__ void __launch_bounds__(kSmallWarps * 32) small_elim_kernel(SolveParams P, int64_t count, int nmax, int ld) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t idx = (int64_t)blockIdx.x * kSmallWarps + warp;
  if (idx >= count) return;
  const int e = blockIdx.y;
  const ElimDesc d = P.elims[idx];
  const int64_t elim_global = P.elim_base + idx;
  const int n = d.n, s = d.s, b = d.b;
  double2* MA = reinterpret_cast<double2*>(smem_raw) + (size_t)warp * (2 * nmax * ld + 64);
  double2* MS = MA + nmax * ld;
  int* piv = reinterpret_cast<int*>(MS + nmax * ld);  // piv, sig, isg: 3 x 32 ints
  int* sig = piv + 32;
  const int32_t* map = P.i32 + d.map_off;
  const int32_t* rank = P.i32 + d.rank_off;
  const double2* lblk = d.left_arena >= 0 ? P.arena[d.left_arena] + (int64_t)e * P.arena_elems[d.left_arena] + d.left_off : nullptr;
  const double2* rblk = d.right_arena >= 0 ? P.arena[d.right_arena] + (int64_t)e * P.arena_elems[d.right_arena] + d.right_off : nullptr;
  const double2* av = P.a_vals + (int64_t)e * P.nnz;

  // ---- gather A (solver.py:203-205) ----
  const int mj = lane < n ? map[lane] : 0;
  for (int i = 0; i < n; ++i) {
    const int mi = map[i];
    if (lane < n) MA[i * ld + lane] = block_entry(d, lblk, rblk, mi, mj);
  }
  __syncwarp();
  const SparseEntry* sp = P.sparse + d.sparse_off;
  for (int t = lane; t < d.nsparse; t += 32) {
    SparseEntry en = sp[t];
    MA[en.i * ld + en.j] = ldg2(av + en.csr);
  }
  __syncwarp();

  // ---- partial LU, pivoting among S rows (kernels.py:237-252, 376) ----
  double scale = 0.0;
  for (int i = 0; i < s; ++i)
    if (lane < s) scale = fmax(scale, cabs(MA[i * ld + lane]));
  for (int o = 16; o; o >>= 1) scale = fmax(scale, __shfl_xor_sync(0xffffffffu, scale, o));
  int bad = (s > 0 && scale == 0.0) ? 0 : INT32_MAX;
  for (int k = 0; k < s; ++k) {
    double v = (lane >= k && lane < s) ? cabs1(MA[lane * ld + k]) : -1.0;
    int vi = lane;
    for (int o = 16; o; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, v, o);
      int oi = __shfl_xor_sync(0xffffffffu, vi, o);
      if (ov > v || (ov == v && oi < vi)) { v = ov; vi = oi; }
    }
    const int pr = vi;
    if (lane == 0) piv[k] = pr;
    if (pr != k && lane < n) {
      double2 t = MA[k * ld + lane];
      MA[k * ld + lane] = MA[pr * ld + lane];
      MA[pr * ld + lane] = t;
    }
    __syncwarp();
    const double2 ukk = MA[k * ld + k];
    if (cabs(ukk) < P.rtol * scale && bad == INT32_MAX) bad = k;
    const double2 uinv = cinv(ukk);
    // column below the pivot (S and B rows), then rank-1 update (lane = column)
    double2 urow = lane < n ? MA[k * ld + lane] : cz();
    __syncwarp();
    for (int i = k + 1; i < n; ++i) {
      double2 l = cmul(MA[i * ld + k], uinv);
      __syncwarp();
      if (lane == k) MA[i * ld + k] = l;
      else if (lane > k && lane < n) MA[i * ld + lane] = cfms(MA[i * ld + lane], l, urow);
    }
    __syncwarp();
  }
  if (bad != INT32_MAX && lane == 0) report_bad(P, elim_global, e, bad);

  // ---- X = Y L11^-1 (row per lane) ----
  if (lane < b) {
    double2* row = MA + (s + lane) * ld;
    for (int k = s - 1; k >= 0; --k) {
      double2 acc = row[k];
      for (int m = k + 1; m < s; ++m) acc = cfms(acc, row[m], MA[m * ld + k]);
      row[k] = acc;
    }
  }
  __syncwarp();

  if (d.kind != kFinal && d.out_arena >= 0) {  // store U sorted (solver.py:234-243)
    double2* out = P.arena[d.out_arena] + (int64_t)e * P.arena_elems[d.out_arena] + d.out_off;
    const int rj = lane < b ? rank[lane] : 0;
    for (int i = 0; i < b; ++i)
      if (lane < b) out[(int64_t)rank[i] * b + rj] = MA[(s + i) * ld + s + lane];
  }
  // permutation sigma from the pivot sequence: pivoted row k = merged row sig[k]
  if (lane == 0) {
    for (int k = 0; k < s; ++k) sig[k] = k;
    for (int k = 0; k < s; ++k) { int t = sig[k]; sig[k] = sig[piv[k]]; sig[piv[k]] = t; }
  }
  __syncwarp();
  if (P.dbg_l && idx == 0 && e == 0 && lane < b)
    for (int k = 0; k < s; ++k) P.dbg_l[(int64_t)lane * s + sig[k]] = MA[(s + lane) * ld + k];
  if (P.compute_gless) {
    const double2* lr = lblk ? lblk + (int64_t)d.p * d.p : nullptr;
    const int q = n - d.p;
    const double2* rr = rblk ? rblk + (int64_t)q * q : nullptr;
    const double2* sv = P.s_vals + (P.s_broadcast ? 0 : (int64_t)e * P.nnz);
    // inverse permutation for the sparse scatter: merged pos -> pivoted pos
    int* isg = sig + 32;
    if (lane < n && lane >= s) isg[lane] = lane;  // B part: identity
    __syncwarp();
    if (lane < s) isg[sig[lane]] = lane;
    __syncwarp();
    const int pj = lane < n ? map[lane < s ? sig[lane] : lane] : 0;
    for (int i = 0; i < n; ++i) {
      const int pi = map[i < s ? sig[i] : i];
      if (lane < n) MS[i * ld + lane] = block_entry(d, lr, rr, pi, pj);
    }
    __syncwarp();
    for (int t = lane; t < d.nsparse; t += 32) {
      SparseEntry en = sp[t];
      MS[isg[en.i] * ld + isg[en.j]] = ldg2(sv + en.csr);
    }
    __syncwarp();
    // T = MS[s:,:] - X MS[:s,:]  (lane = column)
    if (lane < n)
      for (int i = 0; i < b; ++i) {
        double2 acc = MS[(s + i) * ld + lane];
        for (int k = 0; k < s; ++k) acc = cfms(acc, MA[(s + i) * ld + k], MS[k * ld + lane]);
        MS[(s + i) * ld + lane] = acc;
      }
    __syncwarp();
    // R = T[:, s:] - T[:, :s] X^H  (lane = column j < b)
    if (lane < b)
      for (int i = 0; i < b; ++i) {
        double2 acc = MS[(s + i) * ld + s + lane];
        for (int k = 0; k < s; ++k) acc = cfms(acc, MS[(s + i) * ld + k], cconj(MA[(s + lane) * ld + k]));
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
    final_epilogue_warp(P, d, elim_global, e, MA + s * ld + s, ld, MS + s * ld + s, ld, lane);
  }
}

// ================================================================== blocked path
constexpr int kThreads = 256;
constexpr int kTM = 64, kTN = 64, kKC = 16, kSK = kKC + 4;  // smem row stride 20 complex = 320 B

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// C[M x N] (-)= A[M x K] * op(B).  op(B)[k][n] = B[k*ldb + n] (CONJT = false) or
// conj(B[n*ldb + k]) (CONJT = true).  SUB: C -= AB, else C = AB.  Whole CTA.
// In-place use is safe when each output tile's K-range of its own rows/cols
// is the only aliased region (the LU/TRSM uses below).
template <bool CONJT, bool SUB>
__device__ void cta_gemm(double2* C, int64_t ldc, const double2* A, int64_t lda, const double2* B, int64_t ldb, int M,
                         int N, int K, double2* smem) {
  if (M <= 0 || N <= 0) return;
  double2* As = smem;
  double2* Bs = smem + kTM * kSK;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int tiles_m = (M + kTM - 1) / kTM, tiles_n = (N + kTN - 1) / kTN;
  const int fr = lane >> 2, fc = lane & 3;
  for (int tile = 0; tile < tiles_m * tiles_n; ++tile) {
    const int m0 = (tile / tiles_n) * kTM, n0 = (tile % tiles_n) * kTN;
    double acc[4][2][2][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 2; ++c) { acc[a][c][0][0] = acc[a][c][0][1] = acc[a][c][1][0] = acc[a][c][1][1] = 0.0; }
    for (int k0 = 0; k0 < K; k0 += kKC) {
#pragma unroll
      for (int r = 0; r < (kTM * kKC) / kThreads; ++r) {
        const int q = tid + r * kThreads;
        const int row = q >> 4, kk = q & 15;
        double2 v = cz();
        if (m0 + row < M && k0 + kk < K) v = A[(int64_t)(m0 + row) * lda + k0 + kk];
        As[row * kSK + kk] = v;
      }
      if (!CONJT) {
#pragma unroll
        for (int r = 0; r < (kTN * kKC) / kThreads; ++r) {
          const int q = tid + r * kThreads;
          const int kk = q >> 6, col = q & 63;
          double2 v = cz();
          if (k0 + kk < K && n0 + col < N) v = B[(int64_t)(k0 + kk) * ldb + n0 + col];
          Bs[col * kSK + kk] = v;
        }
      } else {
#pragma unroll
        for (int r = 0; r < (kTN * kKC) / kThreads; ++r) {
          const int q = tid + r * kThreads;
          const int col = q >> 4, kk = q & 15;
          double2 v = cz();
          if (k0 + kk < K && n0 + col < N) v = cconj(B[(int64_t)(n0 + col) * ldb + k0 + kk]);
          Bs[col * kSK + kk] = v;
        }
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < kKC; kk += 4) {
        double2 a[4], b[2];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) a[mt] = As[(wm * 32 + mt * 8 + fr) * kSK + kk + fc];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) b[nt] = Bs[(wn * 16 + nt * 8 + fr) * kSK + kk + fc];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          const double nai = -a[mt].y;
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            dmma(acc[mt][nt][0][0], acc[mt][nt][0][1], a[mt].x, b[nt].x);
            dmma(acc[mt][nt][0][0], acc[mt][nt][0][1], nai, b[nt].y);
            dmma(acc[mt][nt][1][0], acc[mt][nt][1][1], a[mt].x, b[nt].y);
            dmma(acc[mt][nt][1][0], acc[mt][nt][1][1], a[mt].y, b[nt].x);
          }
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int r = m0 + wm * 32 + mt * 8 + fr;
          const int c = n0 + wn * 16 + nt * 8 + 2 * fc + i;
          if (r < M && c < N) {
            double2* p = C + (int64_t)r * ldc + c;
            double2 v = make_double2(acc[mt][nt][0][i], acc[mt][nt][1][i]);
            *p = SUB ? csub(*p, v) : v;
          }
        }
  }
  __syncthreads();
}

__device__ void block_argmax(double& v, int& vi, double* cv, int* ci) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, v, o);
    int oi = __shfl_xor_sync(0xffffffffu, vi, o);
    if (ov > v || (ov == v && oi < vi)) { v = ov; vi = oi; }
  }
  if (lane == 0) { cv[warp] = v; ci[warp] = vi; }
  __syncthreads();
  v = cv[0]; vi = ci[0];
  for (int w = 1; w < kThreads / 32; ++w) {
    double ov = cv[w];
    int oi = ci[w];
    if (ov > v || (ov == v && oi < vi)) { v = ov; vi = oi; }
  }
}

// Triangular inverse of the jb x jb diagonal block T (shared, ld ldt) into
// `out` (shared, ld ldo).  lower: unit lower L; else upper U.  One warp,
// lane = column.
__device__ void warp_tri_inverse(const double2* T, int ldt, int jb, bool lower, double2* out, int ldo, int lane) {
  if (lane >= jb) return;
  const int c = lane;
  if (lower) {
    for (int r = 0; r < jb; ++r) {
      double2 x = cz();
      if (r == c) x = make_double2(1.0, 0.0);
      else if (r > c)
        for (int m = c; m < r; ++m) x = cfms(x, T[r * ldt + m], out[m * ldo + c]);
      out[r * ldo + c] = x;
    }
  } else {
    for (int r = jb - 1; r > c; --r) out[r * ldo + c] = cz();
    out[c * ldo + c] = cinv(T[c * ldt + c]);
    for (int r = c - 1; r >= 0; --r) {
      double2 acc = cz();
      for (int m = r + 1; m <= c; ++m) acc = cfms(acc, T[r * ldt + m], out[m * ldo + c]);
      out[r * ldo + c] = cmul(acc, cinv(T[r * ldt + r]));
    }
  }
}

template <int NB>
__host__ __device__ constexpr size_t cta_panel_smem(int max_s) {
  return (size_t)max_s * (NB + 1) * sizeof(double2) + 2 * NB * NB * sizeof(double2);
}
constexpr size_t kGemmSmem = 2 * kTM * kSK * sizeof(double2);

template <int NB>
__global__ void __launch_bounds__(kThreads, 1) cta_elim_kernel(SolveParams P, int64_t count) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* smem = reinterpret_cast<double2*>(smem_raw);
  __shared__ double cand_v[2][kThreads / 32];
  __shared__ int cand_i[2][kThreads / 32];
  __shared__ int s_bad;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t idx = blockIdx.x;
  const int e = blockIdx.y;
  const ElimDesc d = P.elims[idx];
  const int64_t elim_global = P.elim_base + idx;
  const int n = d.n, s = d.s, b = d.b;
  double2* M = P.scratch + (int64_t)e * P.scratch_elems + d.ws_off;
  double2* MS = M + (int64_t)n * n;
  double2* LINV = MS + (int64_t)n * n;  // block j at j*NB*NB (ld NB); U^-1 of the current panel after them
  const int nblk = (s + NB - 1) / NB;
  double2* UINV = LINV + (int64_t)nblk * NB * NB;
  int* PIV = reinterpret_cast<int*>(UINV + NB * NB);
  int* SIG = PIV + n;
  const int32_t* map = P.i32 + d.map_off;
  const int32_t* rank = P.i32 + d.rank_off;
  const double2* lblk = d.left_arena >= 0 ? P.arena[d.left_arena] + (int64_t)e * P.arena_elems[d.left_arena] + d.left_off : nullptr;
  const double2* rblk = d.right_arena >= 0 ? P.arena[d.right_arena] + (int64_t)e * P.arena_elems[d.right_arena] + d.right_off : nullptr;
  const SparseEntry* sp = P.sparse + d.sparse_off;
  const double2* av = P.a_vals + (int64_t)e * P.nnz;
  if (tid == 0) s_bad = INT32_MAX;

  // ---- gather A (solver.py:203-205) ----
  for (int64_t q = tid; q < (int64_t)n * n; q += kThreads) {
    const int i = (int)(q / n), j = (int)(q % n);
    M[q] = block_entry(d, lblk, rblk, map[i], map[j]);
  }
  __syncthreads();
  for (int t = tid; t < d.nsparse; t += kThreads) {
    SparseEntry en = sp[t];
    M[(int64_t)en.i * n + en.j] = ldg2(av + en.csr);
  }
  __syncthreads();
  // pivot scale = max |A(S,S)| (kernels.py:241)
  double scale = 0.0;
  for (int64_t q = tid; q < (int64_t)s * s; q += kThreads) scale = fmax(scale, cabs(M[(q / s) * n + q % s]));
  {
    int dummy = 0;
    block_argmax(scale, dummy, cand_v[0], cand_i[0]);
  }
  if (tid == 0 && s > 0 && scale == 0.0) s_bad = 0;
  __syncthreads();

  // ---- blocked right-looking partial LU; pivot search among S rows only ----
  constexpr int PS = NB + 1;
  for (int j0 = 0; j0 < s; j0 += NB) {
    const int jb = min(NB, s - j0), j1 = j0 + jb, R = s - j0;
    double2* panel = smem;                      // [R][PS]
    double2* tinv = smem + (size_t)R * PS;      // [2][NB*NB]: L^-1, U^-1 of the diagonal block
    for (int q = tid; q < R * jb; q += kThreads) {
      const int r = q / jb, c = q % jb;
      panel[r * PS + c] = M[(int64_t)(j0 + r) * n + j0 + c];
    }
    __syncthreads();
    for (int jj = 0; jj < jb; ++jj) {
      double v = -1.0;
      int vi = INT32_MAX;
      for (int r = jj + tid; r < R; r += kThreads) {
        const double a = cabs1(panel[r * PS + jj]);
        if (a > v) { v = a; vi = r; }
      }
      block_argmax(v, vi, cand_v[jj & 1], cand_i[jj & 1]);
      const int pr = vi;
      if (tid == 0) PIV[j0 + jj] = j0 + pr;
      if (pr != jj && tid < jb) {
        double2 t = panel[jj * PS + tid];
        panel[jj * PS + tid] = panel[pr * PS + tid];
        panel[pr * PS + tid] = t;
      }
      __syncthreads();
      const double2 ukk = panel[jj * PS + jj];
      if (tid == 0 && cabs(ukk) < P.rtol * scale) atomicMin(&s_bad, j0 + jj);
      const double2 uinv = cinv(ukk);
      for (int r = jj + 1 + tid; r < R; r += kThreads) {
        double2* row = panel + r * PS;
        const double2 l = cmul(row[jj], uinv);
        row[jj] = l;
        for (int c = jj + 1; c < jb; ++c) row[c] = cfms(row[c], l, panel[jj * PS + c]);
      }
      __syncthreads();
    }
    // inverses of the diagonal block (warp 0: unit-lower L, warp 1: upper U)
    if (warp == 0) warp_tri_inverse(panel, PS, jb, true, tinv, NB, lane);
    if (warp == 1) warp_tri_inverse(panel, PS, jb, false, tinv + NB * NB, NB, lane);
    for (int q = tid; q < R * jb; q += kThreads) {
      const int r = q / jb, c = q % jb;
      M[(int64_t)(j0 + r) * n + j0 + c] = panel[r * PS + c];
    }
    // row interchanges of this panel on the other columns of the S rows
    for (int c = tid; c < n; c += kThreads) {
      if (c >= j0 && c < j1) continue;
      for (int jj = 0; jj < jb; ++jj) {
        const int pr = PIV[j0 + jj];
        if (pr != j0 + jj) {
          double2* pa = M + (int64_t)(j0 + jj) * n + c;
          double2* pb = M + (int64_t)pr * n + c;
          const double2 t = *pa;
          *pa = *pb;
          *pb = t;
        }
      }
    }
    __syncthreads();
    double2* linv = LINV + (int64_t)(j0 / NB) * NB * NB;
    for (int q = tid; q < NB * NB; q += kThreads) {
      linv[q] = tinv[q];
      UINV[q] = tinv[NB * NB + q];
    }
    __syncthreads();
    // U12 = L_jj^-1 A(j0:j1, j1:n)         (in place)
    cta_gemm<false, false>(M + (int64_t)j0 * n + j1, n, linv, NB, M + (int64_t)j0 * n + j1, n, jb, n - j1, jb, smem);
    // L21 (B rows) = A(s:n, j0:j1) U_jj^-1 (in place; S rows below came out of the panel)
    cta_gemm<false, false>(M + (int64_t)s * n + j0, n, M + (int64_t)s * n + j0, n, UINV, NB, b, jb, jb, smem);
    // trailing update over all remaining rows/cols (S and B)
    cta_gemm<false, true>(M + (int64_t)j1 * n + j1, n, M + (int64_t)j1 * n + j0, n, M + (int64_t)j0 * n + j1, n,
                          n - j1, n - j1, jb, smem);
  }
  if (tid == 0 && s_bad != INT32_MAX) report_bad(P, elim_global, e, s_bad);

  // ---- X = Y L11^-1, block columns right to left ----
  for (int j = nblk - 1; j >= 0; --j) {
    const int j0 = j * NB, jb = min(NB, s - j0), j1 = j0 + jb;
    if (j1 < s)
      cta_gemm<false, true>(M + (int64_t)s * n + j0, n, M + (int64_t)s * n + j1, n, M + (int64_t)j1 * n + j0, n, b,
                            jb, s - j1, smem);
    cta_gemm<false, false>(M + (int64_t)s * n + j0, n, M + (int64_t)s * n + j0, n, LINV + (int64_t)j * NB * NB, NB,
                           b, jb, jb, smem);
  }

  // ---- store U sorted (solver.py:234-243) ----
  if (d.kind != kFinal && d.out_arena >= 0) {
    double2* out = P.arena[d.out_arena] + (int64_t)e * P.arena_elems[d.out_arena] + d.out_off;
    for (int64_t q = tid; q < (int64_t)b * b; q += kThreads) {
      const int i = (int)(q / b), j = (int)(q % b);
      out[(int64_t)rank[i] * b + rank[j]] = M[(int64_t)(s + i) * n + s + j];
    }
  }
  if (tid == 0) {
    for (int k = 0; k < s; ++k) SIG[k] = k;
    for (int k = 0; k < s; ++k) {
      const int pk = PIV[k];
      const int t = SIG[k];
      SIG[k] = SIG[pk];
      SIG[pk] = t;
    }
  }
  __syncthreads();
  if (P.dbg_l && idx == 0 && e == 0)
    for (int64_t q = tid; q < (int64_t)b * s; q += kThreads)
      P.dbg_l[(q / s) * s + SIG[q % s]] = M[(int64_t)(s + q / s) * n + q % s];
  if (P.compute_gless) {
    int* ISG = SIG + s;  // merged position -> pivoted position (S part)
    for (int k = tid; k < s; k += kThreads) ISG[SIG[k]] = k;
    __syncthreads();
    const double2* lr = lblk ? lblk + (int64_t)d.p * d.p : nullptr;
    const int q = n - d.p;
    const double2* rr = rblk ? rblk + (int64_t)q * q : nullptr;
    const double2* sv = P.s_vals + (P.s_broadcast ? 0 : (int64_t)e * P.nnz);
    for (int64_t t = tid; t < (int64_t)n * n; t += kThreads) {
      const int i = (int)(t / n), j = (int)(t % n);
      MS[t] = block_entry(d, lr, rr, map[i < s ? SIG[i] : i], map[j < s ? SIG[j] : j]);
    }
    __syncthreads();
    for (int t = tid; t < d.nsparse; t += kThreads) {
      SparseEntry en = sp[t];
      const int i = en.i < s ? ISG[en.i] : en.i, j = en.j < s ? ISG[en.j] : en.j;
      MS[(int64_t)i * n + j] = ldg2(sv + en.csr);
    }
    __syncthreads();
    // T = MS[s:, :] - X MS[:s, :]
    cta_gemm<false, true>(MS + (int64_t)s * n, n, M + (int64_t)s * n, n, MS, n, b, n, s, smem);
    // R = T[:, s:] - T[:, :s] X^H
    cta_gemm<true, true>(MS + (int64_t)s * n + s, n, MS + (int64_t)s * n, n, M + (int64_t)s * n, n, b, b, s, smem);
    if (d.kind != kFinal && d.out_arena >= 0) {
      double2* out = P.arena[d.out_arena] + (int64_t)e * P.arena_elems[d.out_arena] + d.out_off + (int64_t)b * b;
      for (int64_t t = tid; t < (int64_t)b * b; t += kThreads) {
        const int i = (int)(t / b), j = (int)(t % b);
        out[(int64_t)rank[i] * b + rank[j]] = MS[(int64_t)(s + i) * n + s + j];
      }
    }
  }
  if (d.kind == kFinal) {
    // U_f, R_f (c x c) to shared memory, then the warp epilogue
    const int c = b;
    double2* uf = smem;
    double2* rf = smem + c * c;
    for (int t = tid; t < c * c; t += kThreads) {
      uf[t] = M[(int64_t)(s + t / c) * n + s + t % c];
      rf[t] = P.compute_gless ? MS[(int64_t)(s + t / c) * n + s + t % c] : cz();
    }
    __syncthreads();
    if (warp == 0) final_epilogue_warp(P, d, elim_global, e, uf, c, rf, c, lane);
  }
}

// ================================================================== host side
#define CUDA_TRY(x)                                                                        \
  do {                                                                                     \
    cudaError_t err__ = (x);                                                               \
    if (err__ != cudaSuccess) {                                                            \
      if (st) {                                                                            \
        st->code = FIND_ECUDA;                                                             \
        std::snprintf(st->message, sizeof(st->message), "%s: %s", #x, cudaGetErrorString(err__)); \
      }                                                                                    \
      return FIND_ECUDA;                                                                   \
    }                                                                                      \
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

constexpr size_t kMaxSmem = 227 * 1024 - 1024;  // dynamic budget (static smem of the kernels < 1 KB)

int pick_nb(int max_s) {
  if (cta_panel_smem<32>(max_s) <= kMaxSmem) return 32;
  if (cta_panel_smem<16>(max_s) <= kMaxSmem) return 16;
  if (cta_panel_smem<8>(max_s) <= kMaxSmem) return 8;
  return 0;
}

size_t ws_header_bytes() { return 256; }

int64_t group_launches(const find_plan* P) { return (int64_t)P->groups.size(); }

}  // namespace

extern "C" {

void find_plan_free_device(find_plan* P) {
  if (!P) return;
  if (P->d_elims) cudaFree(P->d_elims);
  if (P->d_i32) cudaFree(P->d_i32);
  if (P->d_sparse) cudaFree(P->d_sparse);
  P->d_elims = P->d_i32 = P->d_sparse = nullptr;
  P->device = -1;
}

int find_plan_upload(find_plan* P, find_status* st) {
  status_ok(st);
  if (!P) return FIND_EINVAL;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (P->d_elims && P->device == dev) return FIND_OK;
  find_plan_free_device(P);
  auto up = [&](void** dst, const void* src, size_t bytes) -> cudaError_t {
    cudaError_t e = cudaMalloc(dst, bytes ? bytes : 16);
    if (e != cudaSuccess) return e;
    if (bytes) e = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
    return e;
  };
  CUDA_TRY(up(&P->d_elims, P->elims.data(), P->elims.size() * sizeof(ElimDesc)));
  CUDA_TRY(up(&P->d_i32, P->i32.data(), P->i32.size() * sizeof(int32_t)));
  CUDA_TRY(up(&P->d_sparse, P->sparse.data(), P->sparse.size() * sizeof(SparseEntry)));
  P->device = dev;
  return FIND_OK;
}

size_t find_solve_workspace_bytes(const find_plan* P, int32_t nE, int32_t compute_gless) {
  (void)compute_gless;
  if (!P || nE < 1) return 0;
  size_t b = ws_header_bytes();
  for (int a = 0; a < 3; ++a) b += (size_t)nE * P->arena_elems[a] * sizeof(double2);
  b += (size_t)nE * P->ws_elems * sizeof(double2);
  return b;
}

int64_t find_solve_launch_count(const find_plan* P) { return P ? group_launches(P) : 0; }

int find_solve_groups(find_plan* P, const void* a_vals, const void* s_vals, int32_t s_broadcast, int32_t nE,
                      int32_t compute_gless, double rtol, void* gr_out, void* gl_out, void* ws, size_t ws_bytes,
                      int64_t g_begin, int64_t g_end, void* stream_, find_status* st) {
  status_ok(st);
  auto fail = [&](int code, const char* msg) {
    if (st) { st->code = code; std::snprintf(st->message, sizeof(st->message), "%s", msg); }
    return code;
  };
  if (!P || !a_vals || !gr_out || !ws || nE < 1) return fail(FIND_EINVAL, "invalid argument");
  if (compute_gless && (!s_vals || !gl_out)) return fail(FIND_EINVAL, "compute_gless needs s_vals and gl_out");
  if (nE > 0xffff) return fail(FIND_EINVAL, "too many energy points in one call");
  if (ws_bytes < find_solve_workspace_bytes(P, nE, compute_gless)) return fail(FIND_ENOMEM, "workspace too small");
  int rc = find_plan_upload(P, st);
  if (rc) return rc;
  cudaStream_t stream = (cudaStream_t)stream_;
  unsigned char* base = (unsigned char*)ws;
  SolveParams prm;
  std::memset(&prm, 0, sizeof(prm));
  prm.elims = (const ElimDesc*)P->d_elims;
  prm.i32 = (const int32_t*)P->d_i32;
  prm.sparse = (const SparseEntry*)P->d_sparse;
  prm.a_vals = (const double2*)a_vals;
  prm.s_vals = (const double2*)s_vals;
  prm.nnz = P->nnz;
  prm.s_broadcast = s_broadcast;
  prm.compute_gless = compute_gless;
  prm.rtol = rtol;
  prm.status = (unsigned long long*)base;
  size_t off = ws_header_bytes();
  for (int a = 0; a < 3; ++a) {
    prm.arena[a] = (double2*)(base + off);
    prm.arena_elems[a] = P->arena_elems[a];
    off += (size_t)nE * P->arena_elems[a] * sizeof(double2);
  }
  prm.scratch = (double2*)(base + off);
  prm.scratch_elems = P->ws_elems;
  prm.gr_out = (double2*)gr_out;
  prm.gl_out = (double2*)gl_out;
  prm.n_nodes = P->n;
  if (g_begin < 0) g_begin = 0;
  if (g_end < 0 || g_end > (int64_t)P->groups.size()) g_end = (int64_t)P->groups.size();
  if (g_begin == 0) CUDA_TRY(cudaMemsetAsync(base, 0xff, 8, stream));
  static bool attr_done = false;
  if (!attr_done) {
    CUDA_TRY(cudaFuncSetAttribute(cta_elim_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem));
    CUDA_TRY(cudaFuncSetAttribute(cta_elim_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem));
    CUDA_TRY(cudaFuncSetAttribute(cta_elim_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem));
    CUDA_TRY(cudaFuncSetAttribute(small_elim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem));
    attr_done = true;
  }
  for (int64_t gi = g_begin; gi < g_end; ++gi) {
    const LaunchGroup& G = P->groups[gi];
    const int64_t count = G.end - G.begin;
    SolveParams p = prm;
    p.elims = prm.elims + G.begin;
    p.elim_base = G.begin;
    if (G.path == 0) {
      const int nmax = std::max(1, G.max_n), ld = nmax + 1;
      const size_t smem = (size_t)kSmallWarps * (2 * nmax * ld + 64) * sizeof(double2);
      dim3 grid((unsigned)((count + kSmallWarps - 1) / kSmallWarps), (unsigned)nE);
      small_elim_kernel<<<grid, kSmallWarps * 32, smem, stream>>>(p, count, nmax, ld);
    } else {
      const int nb = pick_nb(G.max_s);
      if (nb == 0) return fail(FIND_EINVAL, "elimination block too large for the single-CTA path");
      dim3 grid((unsigned)count, (unsigned)nE);
      size_t smem = kGemmSmem;
      if (nb == 32) {
        smem = std::max(smem, cta_panel_smem<32>(G.max_s));
        cta_elim_kernel<32><<<grid, kThreads, smem, stream>>>(p, count);
      } else if (nb == 16) {
        smem = std::max(smem, cta_panel_smem<16>(G.max_s));
        cta_elim_kernel<16><<<grid, kThreads, smem, stream>>>(p, count);
      } else {
        smem = std::max(smem, cta_panel_smem<8>(G.max_s));
        cta_elim_kernel<8><<<grid, kThreads, smem, stream>>>(p, count);
      }
    }
    CUDA_TRY(cudaGetLastError());
  }
  return FIND_OK;
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
        std::snprintf(st->message, sizeof(st->message), "singular pivot at elimination position %d (cluster %lld, energy %d)",
                      pos, (long long)d.label, e);
      }
    }
  }
  return FIND_ESINGULAR;
}

}  // extern "C"

extern "C" int find_schur_sigma_update(int32_t s, int32_t b, const void* ass, const void* asb, const void* abs_,
                                       const void* abb, const void* sss, const void* ssb, const void* sbs,
                                       const void* sbb, double rtol, void* u_out, void* r_out, void* l_out,
                                       int32_t force_path, void* stream_, find_status* st) {
  status_ok(st);
  if (s < 0 || b < 0 || s + b < 1 || (b > 0 && !u_out)) {
    if (st) { st->code = FIND_EINVAL; std::snprintf(st->message, sizeof(st->message), "invalid sizes"); }
    return FIND_EINVAL;
  }
  cudaStream_t stream = (cudaStream_t)stream_;
  const int n = s + b;
  const bool gless = (r_out != nullptr || b == 0) && (s == 0 || sss) && (s == 0 || b == 0 || (ssb && sbs)) &&
                     (b == 0 || sbb);
  int path = force_path >= 0 ? force_path : (n <= 32 ? 0 : 1);
  if (path == 0 && n > 32) path = 1;
  // one elimination: left block = [[ass, asb], [abs, abb]] (+ Sigma block), map = identity
  ElimDesc d;
  std::memset(&d, 0, sizeof(d));
  d.s = s; d.b = b; d.n = n; d.p = n; d.kind = kUpMerge; d.label = 1;
  d.left_arena = kArenaUp; d.left_off = 0; d.right_arena = kArenaNone; d.right_off = -1;
  d.out_arena = kArenaDown0; d.out_off = 0;
  d.map_off = 0; d.rank_off = n; d.sparse_off = 0; d.nsparse = 0; d.ws_off = 0;
  std::vector<int32_t> i32(n + b);
  for (int k = 0; k < n; ++k) i32[k] = k;
  for (int k = 0; k < b; ++k) i32[n + k] = k;
  const int64_t up_elems = 2 * (int64_t)n * n, out_elems = 2 * (int64_t)b * b;
  const int64_t scr = 2 * (int64_t)n * n + ((s + 31) / 32) * 1024 + 1024 + (3 * n + 3) / 4 + 2;
  void *d_desc = nullptr, *d_i32 = nullptr, *d_up = nullptr, *d_out = nullptr, *d_scr = nullptr, *d_stat = nullptr;
  CUDA_TRY(cudaMalloc(&d_desc, sizeof(ElimDesc)));
  CUDA_TRY(cudaMalloc(&d_i32, i32.size() * 4));
  CUDA_TRY(cudaMalloc(&d_up, up_elems * 16));
  CUDA_TRY(cudaMalloc(&d_out, (out_elems + 2) * 16));
  CUDA_TRY(cudaMalloc(&d_scr, scr * 16));
  CUDA_TRY(cudaMalloc(&d_stat, 16));
  CUDA_TRY(cudaMemcpyAsync(d_desc, &d, sizeof(d), cudaMemcpyHostToDevice, stream));
  CUDA_TRY(cudaMemcpyAsync(d_i32, i32.data(), i32.size() * 4, cudaMemcpyHostToDevice, stream));
  CUDA_TRY(cudaMemsetAsync(d_up, 0, up_elems * 16, stream));
  CUDA_TRY(cudaMemsetAsync(d_stat, 0xff, 8, stream));
  double2* up = (double2*)d_up;
  auto put = [&](double2* dst, const void* src, int rows, int cols) -> cudaError_t {
    if (!rows || !cols) return cudaSuccess;
    return cudaMemcpy2DAsync(dst, (size_t)n * 16, src, (size_t)cols * 16, (size_t)cols * 16, rows,
                             cudaMemcpyDeviceToDevice, stream);
  };
  CUDA_TRY(put(up, ass, s, s));
  CUDA_TRY(put(up + s, asb, s, b));
  CUDA_TRY(put(up + (int64_t)s * n, abs_, b, s));
  CUDA_TRY(put(up + (int64_t)s * n + s, abb, b, b));
  if (gless) {
    double2* rs = up + (int64_t)n * n;
    CUDA_TRY(put(rs, sss, s, s));
    CUDA_TRY(put(rs + s, ssb, s, b));
    CUDA_TRY(put(rs + (int64_t)s * n, sbs, b, s));
    CUDA_TRY(put(rs + (int64_t)s * n + s, sbb, b, b));
  }
  SolveParams p;
  std::memset(&p, 0, sizeof(p));
  p.elims = (const ElimDesc*)d_desc;
  p.i32 = (const int32_t*)d_i32;
  p.sparse = nullptr;
  p.a_vals = (const double2*)d_up;  // unused (no sparse entries)
  p.s_vals = (const double2*)d_up;
  p.compute_gless = gless;
  p.rtol = rtol;
  p.arena[kArenaUp] = up;
  p.arena[kArenaDown0] = (double2*)d_out;
  p.arena[kArenaDown1] = (double2*)d_out;
  p.scratch = (double2*)d_scr;
  p.scratch_elems = scr;
  p.status = (unsigned long long*)d_stat;
  p.dbg_l = (double2*)l_out;
  if (path == 0) {
    const int nmax = n, ld = n + 1;
    const size_t smem = (size_t)kSmallWarps * (2 * nmax * ld + 64) * sizeof(double2);
    CUDA_TRY(cudaFuncSetAttribute(small_elim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem));
    small_elim_kernel<<<dim3(1, 1), kSmallWarps * 32, smem, stream>>>(p, 1, nmax, ld);
  } else {
    const int nb = pick_nb(s);
    if (nb == 0) {
      if (st) { st->code = FIND_EINVAL; std::snprintf(st->message, sizeof(st->message), "block too large"); }
      return FIND_EINVAL;
    }
    size_t smem = kGemmSmem;
    if (nb == 32) {
      smem = std::max(smem, cta_panel_smem<32>(s));
      CUDA_TRY(cudaFuncSetAttribute(cta_elim_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem));
      cta_elim_kernel<32><<<dim3(1, 1), kThreads, smem, stream>>>(p, 1);
    } else if (nb == 16) {
      smem = std::max(smem, cta_panel_smem<16>(s));
      CUDA_TRY(cudaFuncSetAttribute(cta_elim_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem));
      cta_elim_kernel<16><<<dim3(1, 1), kThreads, smem, stream>>>(p, 1);
    } else {
      smem = std::max(smem, cta_panel_smem<8>(s));
      CUDA_TRY(cudaFuncSetAttribute(cta_elim_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem));
      cta_elim_kernel<8><<<dim3(1, 1), kThreads, smem, stream>>>(p, 1);
    }
  }
  CUDA_TRY(cudaGetLastError());
  if (b) CUDA_TRY(cudaMemcpyAsync(u_out, d_out, (size_t)b * b * 16, cudaMemcpyDeviceToDevice, stream));
  if (gless && b) CUDA_TRY(cudaMemcpyAsync(r_out, (double2*)d_out + (int64_t)b * b, (size_t)b * b * 16, cudaMemcpyDeviceToDevice, stream));
  unsigned long long key = ~0ull;
  CUDA_TRY(cudaMemcpyAsync(&key, d_stat, 8, cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  cudaFree(d_desc); cudaFree(d_i32); cudaFree(d_up); cudaFree(d_out); cudaFree(d_scr); cudaFree(d_stat);
  if (key != ~0ull) {
    if (st) {
      st->code = FIND_ESINGULAR;
      st->node_id = (int64_t)(key & 0xffff);
      st->cluster_label = 0;
      st->energy_idx = 0;
      std::snprintf(st->message, sizeof(st->message), "singular pivot at elimination position %d", (int)(key & 0xffff));
    }
    return FIND_ESINGULAR;
  }
  return FIND_OK;
}
