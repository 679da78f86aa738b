// Internal plan structures shared by the host plan builder (plan.cpp) and the
// device driver (find_solve.cu).  Not part of the public ABI.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

namespace findb200 {

// Elimination kinds (execution semantics of solver.py):
enum ElimKind : int32_t {
  kLeafSeed = 0,   // upward leaf: order = S u B seeded from A (solver.py:276-291)
  kUpMerge = 1,    // upward internal merge of the two children (solver.py:293-307)
  kDownMerge = 2,  // complement of c = parent complement (+) sibling (solver.py:339-364)
  kFinal = 3,      // final leaf step S = ring, B = leaf nodes (solver.py:392-418, 644-669)
};

// Arenas that hold per-cluster (U, R) blocks, one copy per energy point.
enum Arena : int32_t { kArenaNone = -1, kArenaUp = 0, kArenaDown0 = 1, kArenaDown1 = 2, kArenaDown2 = 3 };
constexpr int kNumArenas = 4;

// One elimination (one merge + Schur/Sigma update), POD, device-visible.
struct alignas(16) ElimDesc {
  int32_t s, b, n, p;        // |S|, |B|, s+b, |left|
  int32_t kind, nsparse;     // ElimKind, number of sparse (CSR-sourced) entries
  int32_t left_arena, right_arena;
  int32_t out_arena, zsplit;  // zsplit: s_l | b_l << 16 when A(B_r, S_l) is structurally zero, else 0
  int64_t label;             // cluster label (negative = complement); final: leaf label
  int64_t left_off, right_off;  // complex-element offsets of child U blocks in their arena (R follows at +sz*sz)
  int64_t out_off;           // offset of the output U block (R at +b*b); final: unused
  int64_t map_off;           // int32[n]: merged position -> index into [left ++ right]
  int64_t rank_off;          // int32[b]: merged B position -> sorted rank (final: mesh node id)
  int64_t sparse_off;        // sparse entries [sparse_off, sparse_off+nsparse)
  int64_t ws_off;            // complex-element offset of this elimination's scratch (per energy)
  int64_t slabel_off;        // int64 host-only array: S labels in merged order (error reporting)
  int64_t sprow_off;         // int32[n+1]: per merged row, offsets of its sparse entries (relative)
  int32_t tmap;              // CTA-path eliminations: index of its tensor-map triple (M, MS, X); else -1
  int32_t tmap_pad;
};
static_assert(sizeof(ElimDesc) == 128, "ElimDesc layout");

// Phase launches of the CTA path (one launch = one kind over a task list).
enum LaunchKind : int32_t {
  kLSmall = 0,     // warp-per-elimination fused kernel (s+b <= 32)
  kLGatherA = 1,   // merged A into scratch                    tasks {e, row0, nrows}
  kLPanel = 2,     // panel LU with pivot search (step j)       tasks {e, j}
  kLTrsm = 3,      // U12 = L_jj^-1 A12 / L21 = A21 U_jj^-1     tasks {e, type, start}
  kLTrail = 4,     // trailing update (DMMA tiles)              tasks {e, tm, tn}
  kLXSolve = 5,    // X = Y L11^-1, block column j              tasks {e, tm}
  kLFinish = 6,    // pivot permutation + store U               tasks {e}
  kLGatherS = 7,   // merged, pivot-permuted Sigma              tasks {e, row0, nrows}
  kLTGemm = 8,     // T_S = S_BS - X S_SS                       tasks {e, tm, tn}
  kLRGemm = 9,     // R = S_BB - X S_SB - T_S X^H (+ store)     tasks {e, tm, tn, sym-skip}
  kLFinal = 10,    // leaf inverse + G^< sandwich               tasks {e}
  kLSchur = 11,    // U = A_BB - Y U12 (K = s), stored sorted  tasks {e, tm, tn}
  kLLuFused = 12,  // (retired: whole blocked LU in one CTA; the value stays reserved)
  kLMid = 13,      // CTA-per-elimination smem kernel (32 < s+b <= 64)
  kLOffdiag = 14,  // off-diagonal G^r / G^< of a final group (after its final launch)
  kLPanelInv = 15, // diagonal-block inverses L_jj^-1, U_jj^-1 of panel j  tasks {e, j}
};

struct Task { int32_t e, a, b, c; };

struct LaunchSpec {
  int32_t kind, step, nb, group;
  int64_t task_off, task_count;
};

// Panel width of a group.  NB = 32: register panel, one S row per thread, up to
// kRegPanelMaxS rows; NB = 16/8/4: shared-memory panel for larger S.
constexpr int64_t kRegPanelMaxS = 288;
constexpr int64_t kSmemPanelMaxS32 = 426;     // NB = 32 rows in one CTA's shared memory (426 * 33 * 16 B)
constexpr int64_t kClusterPanelMaxS = 8 * 384;  // NB = 32 rows over a cluster of <= 8 CTAs (panel_cluster_kernel)
inline int pick_nb_host(int64_t max_s) {
  if (const char* f = std::getenv("FIND_B200_NB")) {  // test hook: force the panel width
    const int nb = std::atoi(f);
    if ((nb == 32 && max_s <= kClusterPanelMaxS) || (nb == 16 && max_s * 17 * 16 <= 220 * 1024) ||
        (nb == 8 && max_s * 9 * 16 <= 220 * 1024) || (nb == 4 && max_s * 5 * 16 <= 220 * 1024))
      return nb;
  }
  if (max_s <= kClusterPanelMaxS) return 32;  // register / shared-memory / cluster panels: K = 32 updates
  if (max_s * 17 * 16 <= 220 * 1024) return 16;
  if (max_s * 9 * 16 <= 220 * 1024) return 8;
  if (max_s * 5 * 16 <= 220 * 1024) return 4;
  return 0;
}
constexpr int kTile = 64;       // DMMA output tile edge
constexpr int64_t kSplitDownElems = int64_t(1) << 29;  // complex elements (8 GiB) of one level's complement blocks
constexpr int64_t kGroupScratchCap = int64_t(1) << 28;  // complex elements of CTA-path scratch per energy per phase (4 GiB)
constexpr int kRowChunk = 16;  // gather rows per CTA (8: gathers 5 % faster serialized, solve 323 -> 321)

struct LaunchGroup {
  int64_t begin, end;  // ElimDesc range
  int32_t path;        // 0 = warp-per-elimination, 1 = blocked (phase launches), 2 = CTA-per-elimination smem
  int32_t pass;        // 0 up, 1 down, 2 final
  int32_t level;
  int32_t max_n, max_s, max_b;
  int64_t ws_elems;    // scratch per energy used by this group
  int32_t nb;          // panel width of the CTA path (0: unsupported size)
  int32_t phase;       // groups of one phase are independent and run concurrently
  int64_t spec_begin, spec_end;    // launches of this group (level-batched phase launches)
};

struct SparseEntry {  // merged (row, col) <- csr value slot
  int32_t i, j;
  int64_t csr;
};

// One off-diagonal output of a final leaf step (solver.py:454-484): the directed
// adjacent pair `pair` is read from this leaf's extraction as
//   type 0: G(ring r, leaf node c)   type 1: G(leaf node c, ring r)   type 2: G(leaf a=r, leaf b=c)
// with r the merged S position of the ring node (type 0/1) or the leaf position (type 2).
struct OffItem {
  int32_t type, r, c, pad;
  int64_t pair;
};

struct Cluster {
  int64_t label;
  int32_t x0, y0, w, h, level;
  int32_t parent;   // index, -1 for root
  int32_t child0, child1;  // indices, -1 if leaf
  std::vector<int64_t> B, S, CB, CS;
  bool leaf() const { return child0 < 0; }
};

}  // namespace findb200

struct find_plan {
  int64_t nx = 0, ny = 0, n = 0, nnz = 0;
  int32_t leaf_max = 2;
  std::vector<int64_t> indptr, indices;
  std::vector<findb200::Cluster> clusters;  // preorder
  std::vector<int64_t> label_keys;          // sorted labels for lookup
  std::vector<int32_t> label_index;         // parallel to label_keys
  std::vector<findb200::ElimDesc> elims;
  std::vector<findb200::LaunchGroup> groups;
  std::vector<int32_t> i32;                 // maps and ranks
  std::vector<int64_t> slabels;             // S labels (merged order) per elimination
  std::vector<findb200::SparseEntry> sparse;
  std::vector<int64_t> exc_slots[2];         // CSR slots of structure-exception entries (up, down)
  std::vector<findb200::Task> tasks;
  std::vector<findb200::LaunchSpec> specs;
  int64_t arena_elems[findb200::kNumArenas] = {0, 0, 0, 0};
  // dependency scheduling (plans small enough for the extra memory): consecutive phases may
  // overlap; three rotating down arenas and two scratch halves (phase parity); per group the
  // groups producing its input blocks
  bool dag = false;
  int32_t split_level = 0;  // > 0: downward levels >= split_level run subtree by subtree
  std::vector<std::vector<int32_t>> group_deps;
  int64_t ws_elems = 0;
  int32_t max_n = 0, max_s = 0, max_b = 0, depth = 0, n_leaves = 0;
  int32_t n_levels_up = 0, n_levels_down = 0;
  // off-diagonal extraction (built on first request, find_plan_offdiag_pairs)
  bool off_ready = false;
  std::vector<int64_t> off_u, off_v;        // directed adjacent pairs, (u, v) ascending
  std::vector<findb200::OffItem> off_items; // grouped by final elimination
  std::vector<int64_t> off_item_off;        // [n_elims + 1]
  void* d_off_items = nullptr;
  void* d_off_item_off = nullptr;
  int off_device = -1;
  // device copies (owned), set by find_plan_upload
  int device = -1;
  void* d_elims = nullptr;
  void* d_i32 = nullptr;
  void* d_sparse = nullptr;
  void* d_tasks = nullptr;
  // TMA tensor maps of the CTA-path scratch matrices (find_solve.cu ensure_tmaps): a few entries,
  // one per (device, scratch base, energy count) seen, each a pinned host + a device array of
  // n_tmap x {M, MS, X} CUtensorMap (128 B each)
  int32_t n_tmap = 0;
  struct TmapEntry {
    int device = -1;
    const void* scratch = nullptr;
    int32_t n_energies = 0;
    void* host = nullptr;
    void* dev = nullptr;
    uint64_t stamp = 0;
  };
  std::vector<TmapEntry> tmap_cache;
  uint64_t tmap_clock = 0;
};
