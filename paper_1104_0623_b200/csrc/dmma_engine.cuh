// TMA-fed FP64 tensor-core (DMMA) tile engine for sm_100a.
//
// One CTA computes BM x BN complex output tiles, acc (+/-)= A[M x K] op(B)[K x N], over a
// sequence of product segments.  Operands are streamed global -> shared memory by the TMA
// bulk-copy engine (cp.async.bulk ... mbarrier::complete_tx, SASS UBLKCP): one PRODUCER warp
// issues one bulk copy per operand row of every K chunk into an S-stage ring of shared-memory
// buffers guarded by full / empty mbarriers; the CONSUMER warps wait on the full barrier of a
// stage, run the DMMA fragments (mma.sync m8n8k4 f64 -> DMMA.8x8x4; B200 has no tcgen05 f64
// kind) and release the stage on its empty barrier.  The producer therefore runs up to S chunks
// ahead, across tile boundaries of a persistent CTA (the next tile's operands arrive while the
// consumers run the previous tile's epilogue).
//
// Shared-memory layouts (padded rows; TMA writes each row at any 16-byte aligned address):
//   A and conjugated B ("BT", given as B[n][k]): [rows][KC + 4] complex (row stride 320 B:
//       the eight rows of a fragment start 64 B apart -> conflict-free 16-byte fragment loads)
//   B given as B[k][n]: [KC][BN + 2] complex (row stride = 32 B mod 128 -> conflict-free)
// Stale shared memory outside the valid rows / K range is never multiplied into a stored
// output: fragments beyond the valid K are zeroed in registers (both operands), fragments of
// rows / columns beyond the valid range only feed outputs that are not stored.
#pragma once

#include <cstdint>

namespace dmma {

constexpr int KC = 16;        // complex per K chunk
constexpr int SKA = KC + 4;   // A / BT row stride (complex)

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  unsigned ok;
  do {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!ok);
}
// TMA bulk copy global -> this CTA's shared memory, completion counted on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// One product segment: acc +/-= A op(B), A [Mv x K] row stride lda; op(B)[k][c] = B[k*ldb + c]
// (bt = false) or conj(B[c*ldb + k]) (bt = true).
struct Seg {
  const double2* A;
  const double2* B;
  int64_t lda, ldb;
  int K;
  int bt;
};

// WM x WN consumer warps, each MT x NT 8x8 fragments; S stages.
template <int WM, int WN, int MT, int NT, int S>
struct Engine {
  static constexpr int NW = WM * WN;              // consumer warps
  static constexpr int THREADS = (NW + 1) * 32;   // + one producer warp
  static constexpr int BM = WM * MT * 8, BN = WN * NT * 8;
  static constexpr int SKB = BN + 2;              // B[k][n] row stride (complex)
  static constexpr int A_ELEMS = BM * SKA;
  static constexpr int B_ELEMS = (BN * SKA > KC * SKB) ? BN * SKA : KC * SKB;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr size_t SMEM = (size_t)S * STAGE * 16 + 2 * S * sizeof(uint64_t) + 16;

  double2* st;        // S stages
  uint64_t* full;     // [S]
  uint64_t* empty;    // [S]
  unsigned pchunk;    // producer's running chunk counter
  unsigned cchunk;    // consumer's running chunk counter

  __device__ __forceinline__ void init(unsigned char* smem_raw) {
    st = reinterpret_cast<double2*>(smem_raw);
    full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)S * STAGE * 16);
    empty = full + S;
    pchunk = cchunk = 0;
    if (threadIdx.x == 0) {
      for (int i = 0; i < S; ++i) {
        mbar_init(&full[i], 1);
        mbar_init(&empty[i], NW);
      }
      mbar_fence_init();
    }
    __syncthreads();
  }

  __device__ __forceinline__ static bool producer() { return threadIdx.x >= NW * 32; }

  // ---- producer warp: stream every K chunk of the segments of one tile
  __device__ __forceinline__ void produce(const Seg* seg, int nseg, int Mv, int Nv) {
    const int lane = threadIdx.x & 31;
    const int mv = Mv < BM ? Mv : BM, nv = Nv < BN ? Nv : BN;
    for (int g = 0; g < nseg; ++g) {
      const Seg sg = seg[g];
      for (int k0 = 0; k0 < sg.K; k0 += KC) {
        const int kv = (sg.K - k0) < KC ? (sg.K - k0) : KC;
        const unsigned stage = pchunk % S, round = pchunk / S;
        ++pchunk;
        mbar_wait(&empty[stage], (round & 1) ^ 1);
        double2* As = st + (size_t)stage * STAGE;
        double2* Bs = As + A_ELEMS;
        const unsigned bytes = (unsigned)(mv * kv + (sg.bt ? nv * kv : kv * nv)) * 16u;
        if (lane == 0) mbar_expect_tx(&full[stage], bytes);
        __syncwarp();
        for (int r = lane; r < mv; r += 32)
          bulk_g2s(As + r * SKA, sg.A + (int64_t)r * sg.lda + k0, (unsigned)kv * 16u, &full[stage]);
        if (sg.bt) {
          for (int c = lane; c < nv; c += 32)
            bulk_g2s(Bs + c * SKA, sg.B + (int64_t)c * sg.ldb + k0, (unsigned)kv * 16u, &full[stage]);
        } else {
          for (int k = lane; k < kv; k += 32)
            bulk_g2s(Bs + k * SKB, sg.B + (int64_t)(k0 + k) * sg.ldb, (unsigned)nv * 16u, &full[stage]);
        }
      }
    }
  }

  // ---- consumer warps
  double acc[MT][NT][2][2];

  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int a = 0; a < MT; ++a)
#pragma unroll
      for (int c = 0; c < NT; ++c) acc[a][c][0][0] = acc[a][c][0][1] = acc[a][c][1][0] = acc[a][c][1][1] = 0.0;
  }

  // acc = C (this thread's elements of C[Mv x Nv], zero outside)
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
          const double2 v = (r < Mv && c < Nv) ? C[(int64_t)r * ld + c] : make_double2(0.0, 0.0);
          acc[mt][nt][0][i] = v.x;
          acc[mt][nt][1][i] = v.y;
        }
  }

  // consume the chunks of the segments (same sequence as produce); NEG: acc -= A op(B)
  template <bool NEG>
  __device__ __forceinline__ void consume(const Seg* seg, int nseg, int Mv, int Nv) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp % WM, wn = warp / WM;
    const int fr = lane >> 2, fc = lane & 3;
    const int mtv = min(MT, max(0, (Mv - wm * MT * 8 + 7) / 8));
    const int ntv = min(NT, max(0, (Nv - wn * NT * 8 + 7) / 8));
    for (int g = 0; g < nseg; ++g) {
      const int K = seg[g].K;
      const bool bt = seg[g].bt != 0;
      for (int k0 = 0; k0 < K; k0 += KC) {
        const int kv = (K - k0) < KC ? (K - k0) : KC;
        const unsigned stage = cchunk % S, round = cchunk / S;
        ++cchunk;
        mbar_wait(&full[stage], round & 1);
        const double2* As = st + (size_t)stage * STAGE;
        const double2* Bs = As + A_ELEMS;
        if (mtv > 0 && ntv > 0) {
#pragma unroll
          for (int kk = 0; kk < KC; kk += 4) {
            if (kk >= kv) break;
            const bool kok = kk + fc < kv;
            double2 a[MT], b[NT];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              a[mt] = As[(wm * MT * 8 + mt * 8 + fr) * SKA + kk + fc];
              if (!kok) a[mt] = make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const int col = wn * NT * 8 + nt * 8 + fr;
              if (bt) {
                b[nt] = Bs[col * SKA + kk + fc];
                b[nt].y = -b[nt].y;
              } else {
                b[nt] = Bs[(kk + fc) * SKB + col];
              }
              if (!kok) b[nt] = make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              if (mt >= mtv) break;
              const double ax = NEG ? -a[mt].x : a[mt].x, ay = NEG ? -a[mt].y : a[mt].y, nai = -ay;
#pragma unroll
              for (int nt = 0; nt < NT; ++nt) {
                if (nt >= ntv) break;
                dmma884(acc[mt][nt][0][0], acc[mt][nt][0][1], ax, b[nt].x);
                dmma884(acc[mt][nt][0][0], acc[mt][nt][0][1], nai, b[nt].y);
                dmma884(acc[mt][nt][1][0], acc[mt][nt][1][1], ax, b[nt].y);
                dmma884(acc[mt][nt][1][0], acc[mt][nt][1][1], ay, b[nt].x);
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
      }
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

}  // namespace dmma
