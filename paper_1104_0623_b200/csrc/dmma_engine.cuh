// TMA-fed FP64 tensor-core (DMMA) tile engine for sm_100a.
//
// One persistent CTA computes BM x BN complex output tiles, acc (+/-)= A[M x K] op(B)[K x N]
// summed over up to two product segments.  One PRODUCER warp streams the operands global ->
// shared memory with the TMA unit into an S-stage ring guarded by full / empty mbarriers; the
// CONSUMER warps wait on a stage's full barrier, run the DMMA fragments (mma.sync m8n8k4 f64 ->
// SASS DMMA.8x8x4: B200 has no tcgen05 f64 kind) and release the stage on its empty barrier.
// The producer runs up to S chunks ahead, across tile boundaries (the next tile's operands and an
// L2 prefetch of its C block arrive while the consumers run the previous tile's epilogue).
//
//   A operand (rows x K, row-major complex) and a conjugated B given as B^T[n][k] ("bt"):
//       cp.async.bulk.tensor.3d (SASS UTMALDG) from a per-matrix 3-D tensor map
//       {2*cols doubles, rows, energy}, box {8 complex, 64 rows}, SWIZZLE_128B: two boxes per
//       K chunk, each a [64][8] complex sub-tile with 128-byte rows whose 16-byte chunks are
//       XOR-ed with (row & 7).
//   B given as B[k][n] (rows of the scratch matrices): one cp.async.bulk (SASS UBLKCP) per k row
//       (BN complex, 1 KB) into a padded [KC][BN + 1] layout (row stride = 16 B mod 128).
//
// Fragment rows / columns are permuted within each group of 8 by rho(x) = (x >> 1) | (x & 1) << 2
// so that the eight lanes of a quarter warp hit eight distinct 16-byte bank groups in every
// layout above (conflict-free 16-byte fragment loads); the accumulator's rows and columns carry
// the same permutation, which load_c / for_each undo.
// Shared memory outside the valid K range is never multiplied: fragments beyond the valid K are
// zeroed in registers (both operands); rows / columns beyond the valid range (TMA zero-fills
// outside the tensor, stale data inside it) only feed outputs that are not stored.
#pragma once

#include <cstdint>

namespace dmma {

constexpr int KC = 16;  // complex per K chunk (two 8-complex TMA boxes)
constexpr int BOXR = 64;  // rows per TMA box (the tensor maps' box)

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ int rho(int x) { return (x >> 1) | ((x & 1) << 2); }

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
// TMA bulk copy global -> this CTA's shared memory (UBLKCP), completion counted on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// TMA tensor tile load (UTMALDG): box at element coordinates {x, y, z} of a 3-D tensor map in global memory
__device__ __forceinline__ void tensor_g2s(void* dst, const void* tmap, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tensor_prefetch_l2(const void* tmap, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];\n" ::"l"(tmap), "r"(x), "r"(y), "r"(z)
               : "memory");
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// One product segment of a tile: acc +/-= A op(B) over K.
//   A: rows [ar, ar + BM) x complex columns [ac, ac + K) of the matrix behind tensor map amap
//   op(B)[k][c]: bt ? conj(B^T[bc_row + c][bk + k]) from tensor map bmap
//                   : B[(k) * ldb + c] read from the pointer B (row k of the K range)
struct Seg {
  const void* amap;
  const void* bmap;
  const double2* B;
  int64_t ldb;
  int ar, ac, br, bk;
  int K, bt;
};

// WM x WN consumer warps (8), each MT x NT 8x8 fragments; S stages; CS: with the C staging buffer
// (stage_c / load_c_staged).
template <int WM, int WN, int MT, int NT, int S, bool CS = false>
struct Engine {
  static constexpr int NW = WM * WN;
  static constexpr int THREADS = (NW + 1) * 32;  // + one producer warp
  static constexpr int BM = WM * MT * 8, BN = WN * NT * 8;
  static_assert(BM == BOXR && BN == BOXR, "tiles are one TMA box tall and wide");
  static constexpr int SKB = BN + 1;                   // B[k][n] row stride (complex): 16 B mod 128
  static constexpr int A_BYTES = BM * KC * 16;         // two swizzled [BM][8] sub-tiles
  static constexpr int B_BYTES_RAW = (BN * KC > KC * SKB ? BN * KC : KC * SKB) * 16;
  static constexpr int B_BYTES = (B_BYTES_RAW + 1023) & ~1023;
  static constexpr int STAGE = A_BYTES + B_BYTES;      // multiple of 1024 (swizzle-128B alignment)
  static constexpr int QD = 2;                         // depth of the dynamic tile queue
  static constexpr int C_BYTES = CS ? BM * BN * 16 : 0;  // the next tile's C block: BN / 8 swizzled [BM][8] boxes
  // stages, the C block, then one 1 KB block of barriers / tile-queue slots; + 1 KB alignment slack
  static constexpr size_t SMEM = (size_t)S * STAGE + C_BYTES + 2048;
  static_assert((2 * S + 2 * QD + 2) * sizeof(uint64_t) + QD * sizeof(long long) <= 1024, "barrier block");

  unsigned char* st;  // S stages, 1024-byte aligned
  uint64_t* full;
  uint64_t* empty;
  unsigned chunk;  // running chunk counter (producer and consumers each keep their own copy)
  // dynamic tile queue (next_tile): the producer warp draws tile indices from a global counter
  // and hands them to the consumer warps through QD slots guarded by their own barriers
  uint64_t* qfull;
  uint64_t* qempty;
  long long* qslot;
  unsigned qn;
  // C staging (stage_c / load_c_staged, CS = true): the producer brings the tile's C block in with the TMA
  // unit while the consumers still multiply the previous tile, so seeding the accumulators is a
  // shared-memory read instead of 32 dependent global loads per thread at the head of every tile.
  // Standalone (tools/dmma_bench.cu) +8 % on the K = 64 trailing shape (32.6 TFLOP/s, cuBLAS 31.5); inside
  // the solver the trailing updates ran 7 % slower with it (ncu: same DRAM traffic, the consumer warps
  // run in lockstep and contend for the FP64 pipe instead of overlapping one warp's epilogue with
  // another's MMAs), so find_solve.cu uses load_c + the L2 prefetch unless FIND_B200_CSTAGE=1.
  unsigned char* cbuf;
  uint64_t* cfull;
  uint64_t* cempty;
  unsigned cn;

  __device__ __forceinline__ void init(unsigned char* smem_raw) {
    st = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    full = reinterpret_cast<uint64_t*>(st + (size_t)S * STAGE + C_BYTES);
    empty = full + S;
    qfull = empty + S;
    qempty = qfull + QD;
    cfull = qempty + QD;
    cempty = cfull + 1;
    qslot = reinterpret_cast<long long*>(cempty + 1);
    cbuf = st + (size_t)S * STAGE;
    chunk = 0;
    qn = 0;
    cn = 0;
    if (threadIdx.x == 0) {
      for (int i = 0; i < S; ++i) {
        mbar_init(&full[i], 1);
        mbar_init(&empty[i], NW);
      }
      for (int i = 0; i < QD; ++i) {
        mbar_init(&qfull[i], 1);
        mbar_init(&qempty[i], NW);
      }
      mbar_init(cfull, 1);
      mbar_init(cempty, NW);
      mbar_fence_init();
    }
    __syncthreads();
  }

  // Next tile index of this group, drawn from the launch's global counter (dynamic scheduling:
  // tiles differ in K and in skipped work, so a static round-robin leaves SMs idle at the end).
  // The producer warp draws (next_tile_p) and hands the index to its consumer warps
  // (next_tile_c); -1 when the counter passed `total`.
  __device__ __forceinline__ long long next_tile_p(unsigned long long* counter, long long total) {
    const int lane = threadIdx.x & 31;
    const unsigned slot = qn % QD, round = qn / QD;
    ++qn;
    mbar_wait(&qempty[slot], (round & 1) ^ 1);
    long long t = 0;
    if (lane == 0) {
      t = (long long)atomicAdd(counter, 1ull);
      if (t >= total) t = -1;
      qslot[slot] = t;
      mbar_arrive(&qfull[slot]);
    }
    return __shfl_sync(0xffffffffu, t, 0);
  }
  __device__ __forceinline__ long long next_tile_c() {
    const int lane = threadIdx.x & 31;
    const unsigned slot = qn % QD, round = qn / QD;
    ++qn;
    mbar_wait(&qfull[slot], round & 1);
    const long long t = qslot[slot];
    __syncwarp();
    if (lane == 0) mbar_arrive(&qempty[slot]);
    return t;
  }

  __device__ __forceinline__ static bool producer() { return (int)threadIdx.x >= NW * 32; }

  // ---- producer warp: every K chunk of the segments of one tile (Nv: valid B columns)
  __device__ __forceinline__ void produce(const Seg* seg, int nseg, int e, int Nv) {
    const int lane = threadIdx.x & 31;
    const int nv = Nv < BN ? Nv : BN;
#pragma unroll 1
    for (int g = 0; g < nseg; ++g) {
      const Seg sg = seg[g];
#pragma unroll 1
      for (int k0 = 0; k0 < sg.K; k0 += KC) {
        const int kv = (sg.K - k0) < KC ? (sg.K - k0) : KC;
        const unsigned stage = chunk % S, round = chunk / S;
        ++chunk;
        mbar_wait(&empty[stage], (round & 1) ^ 1);
        unsigned char* As = st + (size_t)stage * STAGE;
        unsigned char* Bs = As + A_BYTES;
        const int nbox = kv > 8 ? 2 : 1;  // 8-complex boxes the valid K range touches
        const unsigned bytes = (unsigned)nbox * BOXR * 128u + (sg.bt ? (unsigned)nbox * BOXR * 128u : (unsigned)(kv * nv) * 16u);
        if (lane == 0) {
          mbar_expect_tx(&full[stage], bytes);
          for (int h = 0; h < nbox; ++h) {
            tensor_g2s(As + h * (BM * 128), sg.amap, 2 * (sg.ac + k0 + 8 * h), sg.ar, e, &full[stage]);
            if (sg.bt) tensor_g2s(Bs + h * (BN * 128), sg.bmap, 2 * (sg.bk + k0 + 8 * h), sg.br, e, &full[stage]);
          }
        }
        __syncwarp();
        if (!sg.bt)
          for (int k = lane; k < kv; k += 32)
            bulk_g2s(Bs + k * SKB * 16, sg.B + (int64_t)(k0 + k) * sg.ldb, (unsigned)nv * 16u, &full[stage]);
      }
    }
  }

  // producer warp: the C block [r0, r0 + 64) x [c0, c0 + 64) of the tile into the C buffer (BN / 8 boxes
  // through the matrix's tensor map; rows / columns outside the matrix arrive as zeros)
  __device__ __forceinline__ void stage_c(const void* cmap, int r0, int c0, int e) {
    const unsigned round = cn++;
    mbar_wait(cempty, (round & 1) ^ 1);
    if ((threadIdx.x & 31) == 0) {
      mbar_expect_tx(cfull, (unsigned)C_BYTES);
#pragma unroll
      for (int h = 0; h < BN / 8; ++h) tensor_g2s(cbuf + h * (BM * 128), cmap, 2 * (c0 + 8 * h), r0, e, cfull);
    }
    __syncwarp();
  }

  // consumer warps: acc = the staged C block (this thread's elements), then the buffer is released
  __device__ __forceinline__ void load_c_staged() {
    const int lane = threadIdx.x & 31;
    const int fr = lane >> 2, fc = lane & 3;
    const unsigned round = cn++;
    mbar_wait(cfull, round & 1);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int r = row_of(mt, fr), c = col_of(nt, 2 * fc + i);
          const double2 v = *reinterpret_cast<const double2*>(cbuf + (c >> 3) * (BM * 128) + r * 128 +
                                                              (((c & 7) ^ (r & 7)) << 4));
          acc[mt][nt][0][i] = v.x;
          acc[mt][nt][1][i] = v.y;
        }
    __syncwarp();
    if (lane == 0) mbar_arrive(cempty);
  }

  // L2 prefetch of a C block [r0, r0 + 64) x [c0, c0 + 64) through its matrix's tensor map
  __device__ __forceinline__ static void prefetch_c(const void* cmap, int r0, int c0, int e) {
    const int lane = threadIdx.x & 31;
    if (lane < 8) tensor_prefetch_l2(cmap, 2 * (c0 + 8 * lane), r0, e);
  }

  // ---- consumer warps
  double acc[MT][NT][2][2];

  __device__ __forceinline__ static int row_of(int mt, int fr) {
    const int warp = (int)threadIdx.x >> 5;
    return (warp % WM) * MT * 8 + mt * 8 + rho(fr);
  }
  __device__ __forceinline__ static int col_of(int nt, int x) {
    const int warp = (int)threadIdx.x >> 5;
    return (warp / WM) * NT * 8 + nt * 8 + rho(x);
  }

  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int a = 0; a < MT; ++a)
#pragma unroll
      for (int c = 0; c < NT; ++c) acc[a][c][0][0] = acc[a][c][0][1] = acc[a][c][1][0] = acc[a][c][1][1] = 0.0;
  }

  // acc = C (this thread's elements of C[Mv x Nv], zero outside)
  __device__ __forceinline__ void load_c(const double2* C, int64_t ld, int Mv, int Nv) {
    const int lane = threadIdx.x & 31;
    const int fr = lane >> 2, fc = lane & 3;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int r = row_of(mt, fr), c = col_of(nt, 2 * fc + i);
          const double2 v = (r < Mv && c < Nv) ? C[(int64_t)r * ld + c] : make_double2(0.0, 0.0);
          acc[mt][nt][0][i] = v.x;
          acc[mt][nt][1][i] = v.y;
        }
  }

  // One full K chunk (KC complex) for a warp whose MT x NT fragments are all valid: no
  // predicates, constant shared-memory offsets, and the two DMMAs into one accumulator
  // MT*NT*2 instructions apart (every accumulator chain still sums its products in the same
  // order as the generic path: ax*bx then -ay*by; ax*by then ay*bx -> bit-identical).
  template <bool NEG, bool BTc>
  __device__ __forceinline__ void chunk_full(const unsigned char* a0, const unsigned char* a1, const unsigned char* b0,
                                             const unsigned char* b1) {
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      const unsigned char* ap = ((kk & 4) ? a1 : a0) + (kk >> 3) * (BOXR * 128);
      double2 a[MT], b[NT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) a[mt] = *reinterpret_cast<const double2*>(ap + mt * (8 * 128));
      if (BTc) {
        const unsigned char* bp = ((kk & 4) ? b1 : b0) + (kk >> 3) * (BOXR * 128);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          b[nt] = *reinterpret_cast<const double2*>(bp + nt * (8 * 128));
          b[nt].y = -b[nt].y;
        }
      } else {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) b[nt] = *reinterpret_cast<const double2*>(b0 + (kk * SKB + nt * 8) * 16);
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const double ax = NEG ? -a[mt].x : a[mt].x;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          dmma884(acc[mt][nt][0][0], acc[mt][nt][0][1], ax, b[nt].x);
          dmma884(acc[mt][nt][1][0], acc[mt][nt][1][1], ax, b[nt].y);
        }
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const double ay = NEG ? -a[mt].y : a[mt].y, nai = -ay;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          dmma884(acc[mt][nt][0][0], acc[mt][nt][0][1], nai, b[nt].y);
          dmma884(acc[mt][nt][1][0], acc[mt][nt][1][1], ay, b[nt].x);
        }
      }
    }
  }

  // the chunks of the segments (same sequence as produce); NEG: acc -= A op(B)
  template <bool NEG>
  __device__ __forceinline__ void consume(const Seg* seg, int nseg, int Mv, int Nv) {
    const int lane = threadIdx.x & 31, warp = (int)threadIdx.x >> 5;
    const int wm = warp % WM, wn = warp / WM;
    const int fr = lane >> 2, fc = lane & 3, rf = rho(fr);
    const int mtv = min(MT, max(0, (Mv - wm * MT * 8 + 7) / 8));
    const int ntv = min(NT, max(0, (Nv - wn * NT * 8 + 7) / 8));
    const bool whole = mtv == MT && ntv == NT;
    // per-thread fragment offsets inside a stage (fast path): swizzled A / B^T rows, padded B rows
    const int x0 = (fc ^ rf) << 4, x1 = x0 ^ 64;
    const int aoff = (wm * MT * 8 + rf) * 128;
    const int btoff = A_BYTES + (wn * NT * 8 + rf) * 128;
    const int bnoff = A_BYTES + (fc * SKB + wn * NT * 8 + rf) * 16;
#pragma unroll 1
    for (int g = 0; g < nseg; ++g) {
      const int K = seg[g].K;
      const bool bt = seg[g].bt != 0;
#pragma unroll 1
      for (int k0 = 0; k0 < K; k0 += KC) {
        const int kv = (K - k0) < KC ? (K - k0) : KC;
        const unsigned stage = chunk % S, round = chunk / S;
        ++chunk;
        mbar_wait(&full[stage], round & 1);
        const unsigned char* As = st + (size_t)stage * STAGE;
        const unsigned char* Bs = As + A_BYTES;
        if (whole && kv == KC) {
          if (bt)
            chunk_full<NEG, true>(As + aoff + x0, As + aoff + x1, As + btoff + x0, As + btoff + x1);
          else
            chunk_full<NEG, false>(As + aoff + x0, As + aoff + x1, As + bnoff, nullptr);
        } else if (mtv > 0 && ntv > 0) {
#pragma unroll
          for (int kk = 0; kk < KC; kk += 4) {
            if (kk >= kv) break;
            const int k = kk + fc;
            const bool kok = k < kv;
            // swizzled sub-tile offsets: row r (r & 7 == rf), 16-byte chunk (k & 7) ^ rf
            const int soff = (k >> 3) * (BOXR * 128) + ((((k & 7) ^ rf)) << 4);
            double2 a[MT], b[NT];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              a[mt] = *reinterpret_cast<const double2*>(As + soff + (wm * MT * 8 + mt * 8 + rf) * 128);
              if (!kok) a[mt] = make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const int col = wn * NT * 8 + nt * 8 + rf;
              if (bt) {
                b[nt] = *reinterpret_cast<const double2*>(Bs + soff + col * 128);
                b[nt].y = -b[nt].y;
              } else {
                b[nt] = *reinterpret_cast<const double2*>(Bs + (k * SKB + col) * 16);
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
                dmma884(acc[mt][nt][1][0], acc[mt][nt][1][1], ax, b[nt].y);
                dmma884(acc[mt][nt][0][0], acc[mt][nt][0][1], nai, b[nt].y);
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

  // f(tile row, tile col, value) for this thread's accumulator elements
  template <class F>
  __device__ __forceinline__ void for_each(F f) const {
    const int lane = threadIdx.x & 31;
    const int fr = lane >> 2, fc = lane & 3;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int i = 0; i < 2; ++i)
          f(row_of(mt, fr), col_of(nt, 2 * fc + i), make_double2(acc[mt][nt][0][i], acc[mt][nt][1][i]));
  }
};

using Eng64 = Engine<2, 4, 4, 2, 4>;   // 8 consumer warps (32 x 16 each), one CTA per SM
using Eng64cs = Engine<2, 4, 4, 2, 4, true>;  // + C staging

}  // namespace dmma
