// Host plan builder: nested-dissection tree, node sets, elimination schedule.
//
// Restates (from scratch, O(nnz * depth) instead of the reference's
// O(n * #clusters) sparse mat-vec per cluster):
//   build_cluster_tree        mesh.py:176-206
//   boundary_nodes            mesh.py:209-221
//   adjacent_nodes            mesh.py:224-232
//   private_inner_nodes       mesh.py:235-252
//   annotate_boundaries       mesh.py:255-264
//   complement_boundary_sets  mesh.py:267-290
//   _merge_permutation        solver.py:111-132   ([S_l, S_r, B_l, B_r])
//   _Engine.store             solver.py:234-243   (U/R re-sorted to ascending B)
//   FlopLedger charges        kernels.py:88-146, 379, 391, 436; solver.py:388, 664
#include <algorithm>
#include <map>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <stdexcept>

#include "../../include/find_b200.h"
#include "plan.h"

using namespace findb200;

int64_t find_scratch_elems(int64_t n, int64_t s, int nb);
void find_build_tasks(find_plan* P);
void find_assign_phases(find_plan* P);

namespace {

void set_status(find_status* st, int code, const char* msg) {
  if (!st) return;
  st->code = code;
  st->energy_idx = -1;
  st->cluster_label = 0;
  st->node_id = -1;
  st->pivot_ratio = NAN;
  std::snprintf(st->message, sizeof(st->message), "%s", msg);
}

}  // namespace

// Scratch (complex elements) of one CTA-path elimination: M (n x n), MS
// (n x n), pivots / permutation / inverse permutation (3 s int32), scale, and
// the inverted diagonal blocks L_jj^-1, U_jj^-1 of every panel (nb x nb).
// Must match scratch_of() in find_solve.cu.
int64_t find_scratch_elems(int64_t n, int64_t s, int nb) {
  int64_t e = 2 * n * n + (3 * s + 264 + 3) / 4 + 1 + (n + 2 * kRowChunk - 1) / (2 * kRowChunk);
  if (nb > 0) e += 2 * ((s + nb - 1) / nb) * (int64_t)nb * nb + (n - s) * s;  // + X [b][s]
  return (e + 1) & ~int64_t(1);
}

// Phases: the groups of one upward level; or the downward merges of level L
// together with the final leaf steps of level L-1 (both depend only on the
// downward level L-1).  Groups of a phase run concurrently on side streams,
// so each gets a disjoint scratch range (offsets are rebased here).
void find_assign_phases(find_plan* P) {
  int32_t phase = -1;
  int32_t cur_key = INT32_MIN;
  int64_t base = 0;
  P->ws_elems = 0;
  for (auto& G : P->groups) {
    // key of the phase this group belongs to; a phase whose scratch would exceed
    // the cap is continued as a new (sequential) phase
    int32_t key = G.pass == 0 ? -1000 - G.level : (G.pass == 1 ? G.level : G.level + 1);
    if (key != cur_key || (G.path == 1 && base > 0 && base + G.ws_elems > kGroupScratchCap)) {
      ++phase;
      cur_key = key;
      base = 0;
    }
    G.phase = phase;
    if (G.path == 1) {
      for (int64_t k = G.begin; k < G.end; ++k) P->elims[k].ws_off += base;
      base += G.ws_elems;
    }
    P->ws_elems = std::max(P->ws_elems, base);
  }
  if (P->dag) {  // phase parity halves: a phase may still run while the next one starts
    for (auto& G : P->groups)
      if (G.path == 1 && (G.phase & 1))
        for (int64_t k = G.begin; k < G.end; ++k) P->elims[k].ws_off += P->ws_elems;
    P->ws_elems *= 2;
  }
  // producer of every group's input blocks: the latest earlier group that wrote that
  // (arena, offset) — down arenas are reused every two or three levels
  P->group_deps.assign(P->groups.size(), {});
  std::map<std::pair<int32_t, int64_t>, int32_t> prod;
  for (int32_t g = 0; g < (int32_t)P->groups.size(); ++g) {
    std::vector<int32_t>& dv = P->group_deps[g];
    for (int64_t k = P->groups[g].begin; k < P->groups[g].end; ++k) {
      const ElimDesc& d = P->elims[k];
      for (int side = 0; side < 2; ++side) {
        const int32_t a = side ? d.right_arena : d.left_arena;
        if (a < 0) continue;
        auto it = prod.find({a, side ? d.right_off : d.left_off});
        if (it != prod.end() && it->second != g) dv.push_back(it->second);
      }
    }
    std::sort(dv.begin(), dv.end());
    dv.erase(std::unique(dv.begin(), dv.end()), dv.end());
    for (int64_t k = P->groups[g].begin; k < P->groups[g].end; ++k)
      if (P->elims[k].out_arena >= 0) prod[{P->elims[k].out_arena, P->elims[k].out_off}] = g;
  }
}

// Flattened task lists of every phase launch (see LaunchKind).
// X solve with 16-row tiles for large-S groups with fewer than 148 row tiles of 64 (long, narrow
// chains: cfg2-4 near the root); FIND_B200_XS16=0 disables.
bool xsolve16_enabled() {
  const char* f = std::getenv("FIND_B200_XS16");
  return !(f && f[0] == '0');
}
int xsolve16_min_s() {  // groups with a larger S qualify (FIND_B200_XS16_MIN_S)
  const char* f = std::getenv("FIND_B200_XS16_MIN_S");
  return f ? std::atoi(f) : 288;
}

// Groups whose largest S exceeds this use wide (K = 64) trailing updates (FIND_B200_WIDE_MIN_S).
int wide_min_s() {
  const char* f = std::getenv("FIND_B200_WIDE_MIN_S");
  return f ? std::atoi(f) : 200;
}

void find_build_tasks(find_plan* P) {
  P->tasks.clear();
  P->specs.clear();
  auto spec = [&](int32_t kind, int32_t step, int32_t nb, int32_t g, int64_t off) {
    LaunchSpec L;
    L.kind = kind; L.step = step; L.nb = nb; L.group = g;
    L.task_off = off;
    L.task_count = (int64_t)P->tasks.size() - off;
    if (L.task_count > 0 || kind == kLSmall) P->specs.push_back(L);
  };
  for (int32_t gi = 0; gi < (int32_t)P->groups.size(); ++gi) {
    LaunchGroup& G = P->groups[gi];
    G.spec_begin = (int64_t)P->specs.size();
    if (G.path == 0 || G.path == 2) {
      LaunchSpec L;
      L.kind = G.path == 0 ? kLSmall : kLMid; L.step = 0; L.nb = 0; L.group = gi;
      L.task_off = G.begin; L.task_count = G.end - G.begin;
      P->specs.push_back(L);
      G.spec_end = (int64_t)P->specs.size();
      continue;
    }
    const int nb = G.nb;
    auto push = [&](int32_t e, int32_t a, int32_t b, int32_t c) { P->tasks.push_back({e, a, b, c}); };
    int64_t off = (int64_t)P->tasks.size();
    for (int64_t e = G.begin; e < G.end; ++e) {
      const ElimDesc& d = P->elims[e];
      for (int r0 = 0; r0 < d.n; r0 += kRowChunk) push((int32_t)e, r0, std::min(kRowChunk, d.n - r0), 0);
    }
    spec(kLGatherA, 0, nb, gi, off);
    const int steps = nb ? (G.max_s + nb - 1) / nb : 0;
    // Wide blocks (large S, NB = 32): panels (2k, 2k+1) of an elimination share one trailing
    // update with K = 64.  After panel 2k only the next panel's columns (the strip) get its
    // interchanges, U12 and update; after panel 2k+1 a wide TRSM applies both panels'
    // interchanges and L_JJ^-1 to the columns right of the block, then one K = 64 update.
    const bool wide = nb == 32 && G.max_s > wide_min_s();
    auto first_of_wide = [&](const ElimDesc& d, int j) { return wide && j % 2 == 0 && d.s > (j + 1) * nb; };
    auto second_of_wide = [&](const ElimDesc& d, int j) { return wide && j % 2 == 1 && d.s > j * nb; };
    for (int j = 0; j < steps; ++j) {
      off = (int64_t)P->tasks.size();
      for (int64_t e = G.begin; e < G.end; ++e)
        if (P->elims[e].s > j * nb) push((int32_t)e, j, 0, 0);
      spec(kLPanel, j, nb, gi, off);
      {  // the diagonal block's inverses, once per (elimination, panel), for the TRSM and X-solve tiles
        LaunchSpec L = P->specs.back();
        L.kind = kLPanelInv;
        P->specs.push_back(L);
      }
      off = (int64_t)P->tasks.size();
      for (int64_t e = G.begin; e < G.end; ++e) {
        const ElimDesc& d = P->elims[e];
        if (d.s <= j * nb) continue;
        const int j1 = std::min(d.s, (j + 1) * nb);
        if (first_of_wide(d, j)) {
          push((int32_t)e, 0, j1, std::min(nb, d.s - j1));  // the strip: next panel's columns
          push((int32_t)e, 5, 0, 0);                        // keep this panel's interchanges
        } else if (!second_of_wide(d, j)) {
          for (int c0 = j1; c0 < d.n; c0 += kTile) push((int32_t)e, 0, c0, 0);
        }
        for (int r0 = 0; r0 < d.b; r0 += kTile) push((int32_t)e, 1, r0, 0);
        for (int c0 = 0; c0 < j * nb; c0 += kTile) push((int32_t)e, 2, c0, 0);  // interchanges on L columns
      }
      spec(kLTrsm, j, nb, gi, off);
      off = (int64_t)P->tasks.size();
      for (int64_t e = G.begin; e < G.end; ++e) {  // wide TRSM, columns right of the block
        const ElimDesc& d = P->elims[e];
        if (!second_of_wide(d, j)) continue;
        for (int c0 = std::min(d.s, (j + 1) * nb); c0 < d.n; c0 += kTile) push((int32_t)e, 3, c0, 0);
      }
      spec(kLTrsm, j, nb, gi, off);
      off = (int64_t)P->tasks.size();
      for (int64_t e = G.begin; e < G.end; ++e) {
        const ElimDesc& d = P->elims[e];
        if (d.s <= j * nb) continue;
        const int j1 = std::min(d.s, (j + 1) * nb), m = d.n - j1;
        const int t = (m + kTile - 1) / kTile;
        if (first_of_wide(d, j)) {  // strip columns only, every row below the panel
          for (int tm = 0; tm < t; ++tm) push((int32_t)e, tm, 0, 2);
          continue;
        }
        const int mode = second_of_wide(d, j) ? 1 : 0;
        for (int tm = 0; tm < t; ++tm)
          for (int tn = 0; tn < t; ++tn)  // the B x B block is updated once, by the Schur launch
            if (j1 + tm * kTile < d.s || j1 + tn * kTile < d.s) push((int32_t)e, tm, tn, mode);
      }
      spec(kLTrail, j, nb, gi, off);
    }
    off = (int64_t)P->tasks.size();
    for (int64_t e = G.begin; e < G.end; ++e) {
      const ElimDesc& d = P->elims[e];
      if (d.b == 0) continue;
      const int tb = (d.b + kTile - 1) / kTile;
      for (int tm = 0; tm < tb; ++tm)
        for (int tn = 0; tn < tb; ++tn) push((int32_t)e, tm, tn, 0);
    }
    spec(kLSchur, 0, nb, gi, off);
    // X = Y L11^-1: one task per 64-row tile of B, each walking the block columns right to
    // left (a row tile depends only on its own rows of X)
    off = (int64_t)P->tasks.size();
    {
      int64_t tiles = 0;  // few 64-row tiles (large-S groups): 16-row tiles, 4x the parallelism
      for (int64_t e = G.begin; e < G.end; ++e)
        if (P->elims[e].s > 0) tiles += (P->elims[e].b + kTile - 1) / kTile;
      const int rows = (nb == 32 && tiles < 148 && G.max_s > xsolve16_min_s() && xsolve16_enabled()) ? 16 : kTile;
      for (int64_t e = G.begin; e < G.end; ++e) {
        const ElimDesc& d = P->elims[e];
        if (d.s == 0 || d.b == 0) continue;
        for (int tm = 0; tm < (d.b + rows - 1) / rows; ++tm) push((int32_t)e, tm, rows == 16 ? 16 : 0, 0);
      }
    }
    spec(kLXSolve, -1, nb, gi, off);
    off = (int64_t)P->tasks.size();
    for (int64_t e = G.begin; e < G.end; ++e) push((int32_t)e, 0, 0, 0);
    spec(kLFinish, 0, nb, gi, off);
    off = (int64_t)P->tasks.size();
    for (int64_t e = G.begin; e < G.end; ++e) {
      const ElimDesc& d = P->elims[e];
      for (int r0 = 0; r0 < d.n; r0 += kRowChunk) push((int32_t)e, r0, std::min(kRowChunk, d.n - r0), 0);
    }
    spec(kLGatherS, 0, nb, gi, off);
    // T = S_B: - X S_S: : tiles over the S columns (c = 0) and the B columns
    // (c = 1); with (skew-)Hermitian Sigma only the lower-triangle B tiles
    // (c = 2 marks tiles the symmetric mode may skip: tn > tm, non-final)
    off = (int64_t)P->tasks.size();
    for (int64_t e = G.begin; e < G.end; ++e) {
      const ElimDesc& d = P->elims[e];
      if (d.s == 0 || d.b == 0) continue;
      const int tb = (d.b + kTile - 1) / kTile;
      for (int tm = 0; tm < tb; ++tm)
        for (int tn = 0; tn < (d.s + kTile - 1) / kTile; ++tn) push((int32_t)e, tm, tn, 0);
    }
    spec(kLTGemm, 0, nb, gi, off);
    off = (int64_t)P->tasks.size();
    for (int64_t e = G.begin; e < G.end; ++e) {
      const ElimDesc& d = P->elims[e];
      if (d.b == 0) continue;
      const int tb = (d.b + kTile - 1) / kTile;
      for (int tm = 0; tm < tb; ++tm)
        for (int tn = 0; tn < tb; ++tn) push((int32_t)e, tm, tn, (tn > tm && d.kind != kFinal) ? 2 : 1);
    }
    spec(kLRGemm, 0, nb, gi, off);
    off = (int64_t)P->tasks.size();
    for (int64_t e = G.begin; e < G.end; ++e)
      if (P->elims[e].kind == kFinal) push((int32_t)e, 0, 0, 0);
    spec(kLFinal, 0, nb, gi, off);
    G.spec_end = (int64_t)P->specs.size();
  }
}

namespace {

constexpr int32_t kSmallMaxN = 32;  // warp-per-elimination path up to this merged size
constexpr int32_t kMidMaxN = 64;    // CTA-per-elimination shared-memory path up to this merged size
constexpr int32_t kLanesDefault = 4;  // concurrent sub-groups per blocked-path size class
int32_t lanes_setting() {  // FIND_B200_LANES overrides (tuning experiments)
  const char* f = std::getenv("FIND_B200_LANES");
  const int v = f ? std::atoi(f) : 0;
  return v >= 1 && v <= 16 ? v : kLanesDefault;
}

struct Builder {
  find_plan* P;
  std::vector<int32_t> mark;  // generation marks over nodes
  std::vector<int32_t> posv;  // position lookup over nodes
  int32_t gen = 0;

  explicit Builder(find_plan* p) : P(p), mark(p->n, 0), posv(p->n, -1) {}

  void build_tree() {
    // mesh.py:176-206: bisect the longer side (ties -> x), ceil half first.
    struct Item { int64_t label; int32_t x0, y0, w, h, level, parent; int32_t slot_child; };
    std::vector<Item> stack;
    stack.push_back({1, 0, 0, (int32_t)P->nx, (int32_t)P->ny, 0, -1, -1});
    while (!stack.empty()) {
      Item it = stack.back();
      stack.pop_back();
      Cluster c;
      c.label = it.label;
      c.x0 = it.x0; c.y0 = it.y0; c.w = it.w; c.h = it.h; c.level = it.level;
      c.parent = it.parent;
      c.child0 = c.child1 = -1;
      int32_t idx = (int32_t)P->clusters.size();
      P->clusters.push_back(c);
      if (it.parent >= 0) {
        if (it.slot_child == 0) P->clusters[it.parent].child0 = idx;
        else P->clusters[it.parent].child1 = idx;
      }
      P->depth = std::max(P->depth, it.level);
      if (it.w <= P->leaf_max && it.h <= P->leaf_max) {
        P->n_leaves++;
        continue;
      }
      Item l = it, r = it;
      l.label = 2 * it.label; r.label = 2 * it.label + 1;
      l.level = r.level = it.level + 1;
      l.parent = r.parent = idx;
      l.slot_child = 0; r.slot_child = 1;
      if (it.w >= it.h) {
        int32_t wl = (it.w + 1) / 2;
        l.w = wl; r.x0 = it.x0 + wl; r.w = it.w - wl;
      } else {
        int32_t hl = (it.h + 1) / 2;
        l.h = hl; r.y0 = it.y0 + hl; r.h = it.h - hl;
      }
      stack.push_back(r);  // preorder: left popped first
      stack.push_back(l);
    }
    std::vector<std::pair<int64_t, int32_t>> kv;
    kv.reserve(P->clusters.size());
    for (int32_t i = 0; i < (int32_t)P->clusters.size(); ++i) kv.push_back({P->clusters[i].label, i});
    std::sort(kv.begin(), kv.end());
    for (auto& e : kv) { P->label_keys.push_back(e.first); P->label_index.push_back(e.second); }
  }

  inline bool in_rect(const Cluster& c, int64_t v) const {
    int64_t x = v % P->nx, y = v / P->nx;
    return x >= c.x0 && x < c.x0 + c.w && y >= c.y0 && y < c.y0 + c.h;
  }

  // mesh.py:209-221 (B) and mesh.py:224-232 (complement boundary).
  void boundary_sets(Cluster& c) {
    c.B.clear();
    c.CB.clear();
    for (int32_t y = c.y0; y < c.y0 + c.h; ++y) {
      for (int32_t x = c.x0; x < c.x0 + c.w; ++x) {
        int64_t v = x + P->nx * (int64_t)y;
        bool outside = false;
        for (int64_t k = P->indptr[v]; k < P->indptr[v + 1]; ++k) {
          int64_t u = P->indices[k];
          if (u == v) continue;
          if (!in_rect(c, u)) {
            outside = true;
            c.CB.push_back(u);
          }
        }
        if (outside) c.B.push_back(v);
      }
    }
    // rect iteration is ascending in id (row-major)
    std::sort(c.CB.begin(), c.CB.end());
    c.CB.erase(std::unique(c.CB.begin(), c.CB.end()), c.CB.end());
  }

  static std::vector<int64_t> set_union(const std::vector<int64_t>& a, const std::vector<int64_t>& b) {
    std::vector<int64_t> out;
    out.reserve(a.size() + b.size());
    std::set_union(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(out));
    return out;
  }
  static std::vector<int64_t> set_diff(const std::vector<int64_t>& a, const std::vector<int64_t>& b) {
    std::vector<int64_t> out;
    out.reserve(a.size());
    std::set_difference(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(out));
    return out;
  }

  void annotate() {
    auto& C = P->clusters;
    for (auto& c : C) boundary_sets(c);
    // S: leaves = C \ B (mesh.py:259-261); internal = (B_l u B_r) \ B (mesh.py:249-251)
    for (auto& c : C) {
      if (c.leaf()) {
        std::vector<int64_t> nodes;
        nodes.reserve((size_t)c.w * c.h);
        for (int32_t y = c.y0; y < c.y0 + c.h; ++y)
          for (int32_t x = c.x0; x < c.x0 + c.w; ++x) nodes.push_back(x + P->nx * (int64_t)y);
        c.S = set_diff(nodes, c.B);
      } else {
        c.S = set_diff(set_union(C[c.child0].B, C[c.child1].B), c.B);
      }
    }
    // complement private inner (mesh.py:280-289), preorder so parents come first
    for (auto& c : C) {
      if (c.parent < 0) {
        c.CB.clear();
        c.CS.clear();
        continue;
      }
      const Cluster& par = C[c.parent];
      int32_t me = (int32_t)(&c - &C[0]);
      const Cluster& sib = C[par.child0 == me ? par.child1 : par.child0];
      c.CS = set_diff(set_union(par.CB, sib.B), c.CB);
    }
  }

  // ---- elimination descriptors ----
  int32_t next_gen() {
    if (++gen == INT32_MAX) { std::fill(mark.begin(), mark.end(), 0); gen = 1; }
    return gen;
  }

  // Build one elimination: merged order [S_l, S_r, B_l, B_r] (solver.py:111-132).
  // left/right are ascending label lists (the stored blocks' order); `lblock`
  // / `rblock` tell whether a stored (U, R) block exists for that side; sparse
  // entries are generated for every (i, j) not covered by a block and present
  // in the CSR pattern.
  void add_elim(int32_t kind, int64_t label, const std::vector<int64_t>& left,
                const std::vector<int64_t>& right, const std::vector<int64_t>& S,
                const std::vector<int64_t>& Bsorted, int32_t left_arena, int64_t left_off,
                int32_t right_arena, int64_t right_off, int32_t out_arena, int64_t out_off,
                const std::vector<int64_t>* final_nodes, bool order_is_leaf_seed) {
    ElimDesc d;
    std::memset(&d, 0, sizeof(d));
    const int32_t p = (int32_t)left.size(), q = (int32_t)right.size();
    d.p = p;
    d.kind = kind;
    d.label = label;
    d.left_arena = left_arena;
    d.right_arena = right_arena;
    d.left_off = left_off;
    d.right_off = right_off;
    d.out_arena = out_arena;
    d.out_off = out_off;
    // membership of S
    int32_t g = next_gen();
    for (int64_t v : S) mark[v] = g;
    std::vector<int32_t> perm;
    perm.reserve(p + q);
    for (int32_t i = 0; i < p; ++i) if (mark[left[i]] == g) perm.push_back(i);
    for (int32_t i = 0; i < q; ++i) if (mark[right[i]] == g) perm.push_back(p + i);
    int32_t s = (int32_t)perm.size();
    for (int32_t i = 0; i < p; ++i) if (mark[left[i]] != g) perm.push_back(i);
    for (int32_t i = 0; i < q; ++i) if (mark[right[i]] != g) perm.push_back(p + i);
    int32_t n = p + q, b = n - s;
    if ((size_t)s != S.size() || (size_t)b != Bsorted.size()) {
      std::fprintf(stderr, "find_b200: merge labels do not split into S and B (label %lld)\n", (long long)label);
      throw std::runtime_error("merge labels do not split into the given S and B sets");
    }
    d.s = s; d.b = b; d.n = n;
    auto lab = [&](int32_t k) { return k < p ? left[k] : right[k - p]; };
    d.map_off = (int64_t)P->i32.size();
    for (int32_t k = 0; k < n; ++k) P->i32.push_back(perm[k]);
    d.rank_off = (int64_t)P->i32.size();
    if (final_nodes) {
      for (int32_t k = s; k < n; ++k) P->i32.push_back((int32_t)lab(perm[k]));
    } else {
      int32_t gb = next_gen();
      for (size_t r = 0; r < Bsorted.size(); ++r) { mark[Bsorted[r]] = gb; posv[Bsorted[r]] = (int32_t)r; }
      for (int32_t k = s; k < n; ++k) P->i32.push_back(posv[lab(perm[k])]);
    }
    d.slabel_off = (int64_t)P->slabels.size();
    for (int32_t k = 0; k < s; ++k) P->slabels.push_back(lab(perm[k]));
    // merged position of every label
    int32_t gm = next_gen();
    for (int32_t k = 0; k < n; ++k) { int64_t v = lab(perm[k]); mark[v] = gm; posv[v] = k; }
    // side of every merged position
    d.sparse_off = (int64_t)P->sparse.size();
    const bool lb = left_arena != kArenaNone && !order_is_leaf_seed;
    const bool rb = right_arena != kArenaNone;
    for (int32_t k = 0; k < n; ++k) {
      int32_t src = perm[k];
      bool from_left = src < p;
      int64_t v = lab(src);
      for (int64_t e = P->indptr[v]; e < P->indptr[v + 1]; ++e) {
        int64_t u = P->indices[e];
        if (mark[u] != gm) continue;
        int32_t j = posv[u];
        bool u_left = perm[j] < p;
        bool covered = (from_left == u_left) && (from_left ? lb : rb);
        if (covered) continue;
        P->sparse.push_back({k, j, e});
      }
    }
    d.nsparse = (int32_t)((int64_t)P->sparse.size() - d.sparse_off);
    {  // structural zero block A(B_r, S_l) (the paper's zero sub-blocks, kernels.py:400-463): then
       // Y = A(B,S) U11^-1 is zero on (B_r, S_l), and the kernels skip those products.
       // (Reordering B_r to put its clean rows last widens this but breaks the contiguous child-
       // block reads: measured -7 % on cfg3, so B keeps the reference's merge order.)
      int32_t ml = 0, nl = 0;
      for (int32_t k = 0; k < s; ++k) ml += perm[k] < p;
      for (int32_t k = s; k < n; ++k) nl += perm[k] < p;
      bool zero = ml > 0 && nl < b && ml < 0x8000 && nl < 0x8000;
      for (int64_t t = d.sparse_off; zero && t < (int64_t)P->sparse.size(); ++t)
        if (P->sparse[t].i >= s + nl && P->sparse[t].j < ml) zero = false;
      d.zsplit = zero ? (ml | (nl << 16)) : 0;
    }
    d.sprow_off = (int64_t)P->i32.size();
    {
      int64_t t = d.sparse_off;
      for (int32_t k = 0; k <= n; ++k) {
        while (t < (int64_t)P->sparse.size() && P->sparse[t].i < k) ++t;
        P->i32.push_back((int32_t)(t - d.sparse_off));
      }
    }
    if (kind == kUpMerge || kind == kDownMerge) {
      // structure exceptions (kernels.py:192-202): off-diagonal entries of the
      // S_l x S_r / S_r x S_l blocks and any entry of X, Y, Q, R.  All of them
      // are cross entries, i.e. CSR-sourced.
      int32_t ml = 0, nl = 0;
      for (int32_t k = 0; k < s; ++k) ml += perm[k] < p;
      for (int32_t k = s; k < n; ++k) nl += perm[k] < p;
      auto& out = P->exc_slots[kind == kUpMerge ? 0 : 1];
      for (int64_t t = d.sparse_off; t < (int64_t)P->sparse.size(); ++t) {
        const int32_t i = P->sparse[t].i, j = P->sparse[t].j;
        bool exc = false;
        if (i < ml && j >= ml && j < s) exc = (i != j - ml);                   // B12 off-diagonal
        else if (i >= ml && i < s && j < ml) exc = (i - ml != j);              // C21 off-diagonal
        else if (i < ml && j >= s + nl) exc = true;                            // X
        else if (i >= ml && i < s && j >= s && j < s + nl) exc = true;         // Y
        else if (i >= s && i < s + nl && j >= ml && j < s) exc = true;         // Q
        else if (i >= s + nl && j < ml) exc = true;                            // R
        if (exc) out.push_back(P->sparse[t].csr);
      }
    }
    P->elims.push_back(d);
  }

  void schedule() {
    auto& C = P->clusters;
    const int32_t D = P->depth;
    std::vector<std::vector<int32_t>> by_level(D + 1);
    for (int32_t i = 0; i < (int32_t)C.size(); ++i) by_level[C[i].level].push_back(i);
    for (auto& v : by_level)
      std::sort(v.begin(), v.end(), [&](int32_t a, int32_t b) { return C[a].label < C[b].label; });
    std::vector<int64_t> up_off(C.size(), -1), down_off(C.size(), -1);
    // upward arena: every non-root cluster, 2*b^2 (U then R)
    int64_t acc = 0;
    for (int32_t L = D; L >= 1; --L)
      for (int32_t i : by_level[L]) { up_off[i] = acc; acc += 2 * (int64_t)C[i].B.size() * C[i].B.size(); }
    P->arena_elems[kArenaUp] = acc;
    int64_t down_max = 0;
    for (int32_t L = 1; L <= D; ++L) {
      int64_t a = 0;
      for (int32_t i : by_level[L]) { down_off[i] = a; a += 2 * (int64_t)C[i].CB.size() * C[i].CB.size(); }
      down_max = std::max(down_max, a);
    }
    // Memory-bounded downward pass: when one level's complement blocks
    // exceed kSplitDownElems per energy, levels >= K run subtree by subtree (one level-K cluster
    // and its descendants at a time, the down arenas reused per subtree); the complements of
    // level K-1 stay in the third arena for all subtrees.  More energy points then fit at once.
    int32_t split = 0;
    if (!P->dag) {
      const char* f = std::getenv("FIND_B200_SPLIT_K");
      if (f) split = std::max(0, std::min(std::atoi(f), D));
      else if (down_max > kSplitDownElems)
        for (split = 1; split < std::min<int32_t>(D, 6); ++split) {
          int64_t mx = 0;  // largest (subtree, level) block set with this split
          for (int32_t r : by_level[split]) {
            std::vector<int32_t> cur{r};
            while (!cur.empty()) {
              int64_t a = 0;
              std::vector<int32_t> nxt;
              for (int32_t i : cur) {
                a += 2 * (int64_t)C[i].CB.size() * C[i].CB.size();
                if (!C[i].leaf()) { nxt.push_back(C[i].child0); nxt.push_back(C[i].child1); }
              }
              mx = std::max(mx, a);
              cur.swap(nxt);
            }
          }
          if (mx <= kSplitDownElems) break;
        }
    }
    P->split_level = split;
    std::vector<int32_t> sub_of(C.size(), -1);  // subtree (level-K ancestor index) of clusters at level >= K
    if (split > 0) {
      for (int32_t r : by_level[split]) {
        std::vector<int32_t> st{r};
        while (!st.empty()) {
          const int32_t i = st.back();
          st.pop_back();
          sub_of[i] = r;
          if (!C[i].leaf()) { st.push_back(C[i].child0); st.push_back(C[i].child1); }
        }
      }
      down_max = 0;
      for (int32_t L = split; L <= D; ++L) {
        std::map<int32_t, int64_t> a;  // per subtree
        for (int32_t i : by_level[L]) {
          int64_t& x = a[sub_of[i]];
          down_off[i] = x;
          x += 2 * (int64_t)C[i].CB.size() * C[i].CB.size();
          down_max = std::max(down_max, x);
        }
      }
      int64_t top = 0;
      for (int32_t L = 1; L < split; ++L) {
        int64_t a = 0;
        for (int32_t i : by_level[L]) {
          if (L == split - 1) down_off[i] = a;
          a += 2 * (int64_t)C[i].CB.size() * C[i].CB.size();
        }
        if (L == split - 1) top = a;
        else down_max = std::max(down_max, a);
      }
      for (int32_t L = 1; L < split - 1; ++L) {  // levels above K-1: ping-pong as usual
        int64_t a = 0;
        for (int32_t i : by_level[L]) { down_off[i] = a; a += 2 * (int64_t)C[i].CB.size() * C[i].CB.size(); }
      }
      P->arena_elems[kArenaDown2] = top;
    }
    P->arena_elems[kArenaDown0] = P->arena_elems[kArenaDown1] = down_max;
    if (split == 0) P->arena_elems[kArenaDown2] = P->dag ? down_max : 0;
    const std::vector<int64_t> empty;

    auto emit_groups = [&](int64_t begin, int32_t pass, int32_t level) {
      // sort the level's eliminations by size class; warp path for s+b <= 32,
      // CTA path split by s so every launch gets a right-sized panel kernel
      int64_t end = (int64_t)P->elims.size();
      if (end == begin) return;
      auto cls = [](const ElimDesc& d) -> int {
        if (d.n <= kSmallMaxN) return 0;
        if (d.n <= kMidMaxN) return 5;
        if (d.s <= 64) return 1;
        if (d.s <= 128) return 2;
        if (d.s <= kRegPanelMaxS) return 3;
        return 4;
      };
      std::stable_sort(P->elims.begin() + begin, P->elims.end(), [&](const ElimDesc& a, const ElimDesc& b) {
        const int ca = cls(a), cb = cls(b);
        return ca != cb ? ca < cb : a.n < b.n;
      });
      auto make_group = [&](int64_t gb, int64_t ge, int path) {
        LaunchGroup G;
        std::memset(&G, 0, sizeof(G));
        G.begin = gb; G.end = ge; G.path = path; G.pass = pass; G.level = level;
        for (int64_t k = gb; k < ge; ++k) {
          const ElimDesc& d = P->elims[k];
          G.max_n = std::max(G.max_n, d.n); G.max_s = std::max(G.max_s, d.s); G.max_b = std::max(G.max_b, d.b);
        }
        G.nb = path == 1 ? pick_nb_host(G.max_s) : 0;
        int64_t ws = 0;
        for (int64_t k = gb; k < ge; ++k) {
          ElimDesc& d = P->elims[k];
          d.ws_off = ws;
          if (path == 1) ws += find_scratch_elems(d.n, d.s, G.nb);
        }
        G.ws_elems = ws;
        P->ws_elems = std::max(P->ws_elems, ws);
        P->groups.push_back(G);
        P->max_n = std::max(P->max_n, G.max_n);
        P->max_s = std::max(P->max_s, G.max_s);
        P->max_b = std::max(P->max_b, G.max_b);
      };
      int64_t cb = begin;
      while (cb < end) {
        const int c = cls(P->elims[cb]);
        int64_t ce = cb;
        while (ce < end && cls(P->elims[ce]) == c) ++ce;
        const int path = c == 0 ? 0 : (c == 5 ? 2 : 1);
        if (path != 1) {
          make_group(cb, ce, path);
          cb = ce;
          continue;
        }
        // blocked path: up to kLanes interleaved lanes (concurrent sub-groups on side
        // streams, so one lane's latency-bound panel steps overlap another lane's DMMA
        // tiles); each lane further split so one group's scratch stays under the cap
        const int64_t cnt = ce - cb;
        const int lanes = (int)std::min<int64_t>(lanes_setting(), std::max<int64_t>(1, cnt / 2));
        if (lanes > 1) {
          std::vector<ElimDesc> tmp(P->elims.begin() + cb, P->elims.begin() + ce);
          int64_t w = cb;
          for (int l = 0; l < lanes; ++l)
            for (int64_t k = l; k < cnt; k += lanes) P->elims[w++] = tmp[k];
        }
        int64_t lb = cb;
        for (int l = 0; l < lanes; ++l) {
          const int64_t le = cb + (cnt * (l + 1)) / lanes;  // lane l = [lb, le) after the reorder
          (void)le;
          const int64_t lcount = (cnt - l + lanes - 1) / lanes;
          const int64_t lend = lb + lcount;
          int32_t ms = 0;
          for (int64_t k = lb; k < lend; ++k) ms = std::max(ms, P->elims[k].s);
          const int nbc = pick_nb_host(ms);
          int64_t gb = lb;
          while (gb < lend) {
            int64_t acc = 0, k = gb;
            for (; k < lend; ++k) {
              const int64_t wsz = find_scratch_elems(P->elims[k].n, P->elims[k].s, nbc);
              if (k > gb && acc + wsz > kGroupScratchCap) break;
              acc += wsz;
            }
            make_group(gb, k, 1);
            gb = k;
          }
          lb = lend;
        }
        cb = ce;
      }
    };

    // ---- upward pass (solver.py:256-308), deepest level first ----
    for (int32_t L = D; L >= 1; --L) {
      int64_t begin = (int64_t)P->elims.size();
      for (int32_t i : by_level[L]) {
        const Cluster& c = C[i];
        if (c.leaf()) {
          std::vector<int64_t> order(c.S);
          order.insert(order.end(), c.B.begin(), c.B.end());
          add_elim(kLeafSeed, c.label, order, empty, c.S, c.B, kArenaNone, -1, kArenaNone, -1, kArenaUp, up_off[i],
                   nullptr, true);
        } else {
          const Cluster& l = C[c.child0];
          const Cluster& r = C[c.child1];
          add_elim(kUpMerge, c.label, l.B, r.B, c.S, c.B, kArenaUp, up_off[c.child0], kArenaUp, up_off[c.child1],
                   kArenaUp, up_off[i], nullptr, false);
        }
      }
      if ((int64_t)P->elims.size() > begin) P->n_levels_up++;
      emit_groups(begin, 0, L);
    }
    // ---- downward pass (solver.py:311-375) level by level, finals right after; with a split,
    // levels >= K subtree by subtree ----
    auto arena_of = [&](int32_t L) -> int32_t {
      if (split > 0 && L == split - 1) return kArenaDown2;  // kept for every subtree
      const int32_t rot = P->dag ? 3 : 2;  // ping-pong by level parity; three when phases may overlap
      return kArenaDown0 + L % rot;
    };
    auto down_level = [&](int32_t L, const std::vector<int32_t>& clusters) {
      int64_t begin = (int64_t)P->elims.size();
      int32_t arena = arena_of(L);
      int32_t parena = arena_of(L - 1);
      for (int32_t i : clusters) {
        const Cluster& c = C[i];
        const Cluster& par = C[c.parent];
        int32_t sib = par.child0 == i ? par.child1 : par.child0;
        bool par_root = par.parent < 0;
        add_elim(kDownMerge, -c.label, par.CB, C[sib].B, c.CS, c.CB, par_root ? kArenaNone : parena,
                 par_root ? -1 : down_off[c.parent], kArenaUp, up_off[sib], arena, down_off[i], nullptr, false);
      }
      if ((int64_t)P->elims.size() > begin) P->n_levels_down++;
      emit_groups(begin, 1, L);
      begin = (int64_t)P->elims.size();
      for (int32_t i : clusters) {
        const Cluster& c = C[i];
        if (!c.leaf()) continue;
        std::vector<int64_t> nodes;
        for (int32_t y = c.y0; y < c.y0 + c.h; ++y)
          for (int32_t x = c.x0; x < c.x0 + c.w; ++x) nodes.push_back(x + P->nx * (int64_t)y);
        add_elim(kFinal, c.label, c.CB, nodes, c.CB, nodes, arena, down_off[i], kArenaNone, -1, kArenaNone, -1,
                 &nodes, false);
      }
      emit_groups(begin, 2, L);
    };
    for (int32_t L = 1; L <= D && (split == 0 || L < split); ++L) down_level(L, by_level[L]);
    if (split > 0)
      for (int32_t r : by_level[split])
        for (int32_t L = split; L <= D; ++L) {
          std::vector<int32_t> cl;
          for (int32_t i : by_level[L])
            if (sub_of[i] == r) cl.push_back(i);
          if (!cl.empty()) down_level(L, cl);
        }
    if (C[0].leaf()) {  // single-cluster mesh: only the final step of the root
      int64_t begin = (int64_t)P->elims.size();
      const Cluster& c = C[0];
      std::vector<int64_t> nodes;
      for (int32_t y = c.y0; y < c.y0 + c.h; ++y)
        for (int32_t x = c.x0; x < c.x0 + c.w; ++x) nodes.push_back(x + P->nx * (int64_t)y);
      add_elim(kFinal, c.label, empty, nodes, empty, nodes, kArenaNone, -1, kArenaNone, -1, kArenaNone, -1, &nodes,
               false);
      emit_groups(begin, 2, 0);
    }
  }
};

// ---- ledger (kernels.py:88-146) over a common denominator of 48 ----
enum LedgerKey {
  kNaiveDense = 0, kSigmaNaive, kDenseInverse, kGlessSandwich, kParallel, kSequential, kBlockLU, kNaiveLU,
  kSigmaSparse, kKeyPad1, kKeyPad2, kKeyPad3
};
const char* kKeyNames[FIND_LEDGER_KEYS] = {"naive_dense", "sigma_naive", "dense_inverse", "gless_sandwich",
                                            "parallel_inverse", "sequential_inverse", "block_lu", "naive_lu",
                                            "sigma_sparse", "", "", ""};

typedef __int128 i128;
// 48 * polynomial, exact
i128 p48_naive_dense(i128 s, i128 b) { return 16 * s * s * s + 48 * s * s * b + 48 * s * b * b; }
i128 p48_sigma_naive(i128 s, i128 b) { return 48 * s * s * b + 144 * s * b * b; }
i128 p48_sigma_sparse(i128 s, i128 b) { return 24 * s * s * b + 96 * s * b * b; }
// m = s/2, n = b/2: c3*m^3 + c21*m^2 n + c12*m n^2 -> over 48: 48*c3/8 s^3 + 48*c21/8 s^2 b + 48*c12/8 s b^2
i128 p48_mn(i128 s, i128 b, i128 c3_num, i128 c3_den, i128 c21_num, i128 c21_den, i128 c12_num, i128 c12_den) {
  return (6 * c3_num / c3_den) * s * s * s + (6 * c21_num / c21_den) * s * s * b + (6 * c12_num / c12_den) * s * b * b;
}

}  // namespace

extern "C" {

int find_plan_create(int64_t nx, int64_t ny, const int64_t* indptr, const int64_t* indices, int64_t nnz,
                     int32_t leaf_max, find_plan** out, find_status* st) {
  set_status(st, FIND_OK, "ok");
  if (!out) { set_status(st, FIND_EINVAL, "out is NULL"); return FIND_EINVAL; }
  *out = nullptr;
  if (nx < 1 || ny < 1) { set_status(st, FIND_EINVAL, "mesh dimensions must be positive"); return FIND_EINVAL; }
  if (leaf_max < 1) { set_status(st, FIND_EINVAL, "leaf_max must be >= 1"); return FIND_EINVAL; }
  if (nx * ny > (int64_t)INT32_MAX) { set_status(st, FIND_EINVAL, "mesh too large"); return FIND_EINVAL; }
  const int64_t n = nx * ny;
  if (!indptr || (nnz > 0 && !indices) || indptr[0] != 0 || indptr[n] != nnz) {
    set_status(st, FIND_EINVAL, "invalid CSR pattern");
    return FIND_EINVAL;
  }
  for (int64_t v = 0; v < n; ++v)
    if (indptr[v + 1] < indptr[v]) { set_status(st, FIND_EINVAL, "indptr not monotone"); return FIND_EINVAL; }
  for (int64_t k = 0; k < nnz; ++k)
    if (indices[k] < 0 || indices[k] >= n) { set_status(st, FIND_EINVAL, "entry index out of range"); return FIND_EINVAL; }
  find_plan* P = new (std::nothrow) find_plan();
  if (!P) { set_status(st, FIND_ENOMEM, "out of host memory"); return FIND_ENOMEM; }
  try {
    P->nx = nx; P->ny = ny; P->n = n; P->nnz = nnz; P->leaf_max = leaf_max;
    P->indptr.assign(indptr, indptr + n + 1);
    P->indices.assign(indices, indices + nnz);
    {  // dependency scheduling for meshes up to FIND_B200_DAG_MAX_N nodes: off by default (measured
       // neutral on cfg1 while it costs a third down arena and a second scratch half)
      const char* f = std::getenv("FIND_B200_DAG_MAX_N");
      const int64_t lim = f ? std::atoll(f) : 0;
      P->dag = n <= lim;
    }
    Builder B(P);
    B.build_tree();
    B.annotate();
    B.schedule();
    find_assign_phases(P);
    find_build_tasks(P);
  } catch (const std::exception& e) {
    set_status(st, FIND_EINVAL, e.what());
    delete P;
    return FIND_EINVAL;
  }
  *out = P;
  return FIND_OK;
}

int find_plan_info(const find_plan* P, int64_t* o) {
  if (!P || !o) return FIND_EINVAL;
  int64_t sp = (int64_t)P->sparse.size();
  int64_t v[16] = {P->n, P->nnz, (int64_t)P->clusters.size(), (int64_t)P->elims.size(), P->n_levels_up,
                   P->n_levels_down, P->arena_elems[0], P->arena_elems[1], P->ws_elems, P->max_n, P->max_s,
                   P->max_b, (int64_t)P->groups.size(), sp, P->depth, P->n_leaves};
  std::memcpy(o, v, sizeof(v));
  return FIND_OK;
}

int64_t find_plan_cluster_set(const find_plan* P, int64_t label, int32_t which, int64_t* out, int64_t cap) {
  if (!P) return -1;
  auto it = std::lower_bound(P->label_keys.begin(), P->label_keys.end(), label);
  if (it == P->label_keys.end() || *it != label) return -1;
  const Cluster& c = P->clusters[P->label_index[it - P->label_keys.begin()]];
  std::vector<int64_t> nodes;
  const std::vector<int64_t>* src = nullptr;
  switch (which) {
    case 0:
      for (int32_t y = c.y0; y < c.y0 + c.h; ++y)
        for (int32_t x = c.x0; x < c.x0 + c.w; ++x) nodes.push_back(x + P->nx * (int64_t)y);
      src = &nodes;
      break;
    case 1: src = &c.B; break;
    case 2: src = &c.S; break;
    case 3: src = &c.CB; break;
    case 4: src = &c.CS; break;
    default: return -1;
  }
  int64_t sz = (int64_t)src->size();
  if (out) for (int64_t k = 0; k < std::min(sz, cap); ++k) out[k] = (*src)[k];
  return sz;
}

int find_plan_elims(const find_plan* P, int32_t* kind, int32_t* s, int32_t* b, int64_t* label) {
  if (!P) return FIND_EINVAL;
  for (size_t k = 0; k < P->elims.size(); ++k) {
    if (kind) kind[k] = P->elims[k].kind;
    if (s) s[k] = P->elims[k].s;
    if (b) b[k] = P->elims[k].b;
    if (label) label[k] = P->elims[k].label;
  }
  return FIND_OK;
}

int find_plan_elim_splits(const find_plan* P, int32_t* s_left, int32_t* b_left) {
  if (!P) return FIND_EINVAL;
  for (size_t k = 0; k < P->elims.size(); ++k) {
    const int32_t z = P->elims[k].zsplit;
    if (s_left) s_left[k] = z & 0xffff;
    if (b_left) b_left[k] = z ? (z >> 16) : 0;
  }
  return FIND_OK;
}

int find_plan_arena_elems(const find_plan* P, int64_t* out4) {
  if (!P || !out4) return FIND_EINVAL;
  for (int a = 0; a < kNumArenas; ++a) out4[a] = P->arena_elems[a];
  return FIND_OK;
}

int find_plan_elim_out(const find_plan* P, int32_t* out_arena, int64_t* out_off) {
  if (!P) return FIND_EINVAL;
  for (size_t k = 0; k < P->elims.size(); ++k) {
    if (out_arena) out_arena[k] = P->elims[k].out_arena;
    if (out_off) out_off[k] = P->elims[k].out_off;
  }
  return FIND_OK;
}

int64_t find_plan_exception_slots(const find_plan* P, int32_t pass, int64_t* out, int64_t cap) {
  if (!P || pass < 0 || pass > 1) return -1;
  const auto& v = P->exc_slots[pass];
  if (out) for (int64_t k = 0; k < std::min<int64_t>((int64_t)v.size(), cap); ++k) out[k] = v[k];
  return (int64_t)v.size();
}

const char* find_ledger_key_name(int32_t key) {
  if (key < 0 || key >= FIND_LEDGER_KEYS) return "";
  return kKeyNames[key];
}

int find_plan_ledger(const find_plan* P, int32_t kernel, int32_t compute_gless, int64_t* num, int64_t* den) {
  if (!P || !num || !den || kernel < 0 || kernel > 4) return FIND_EINVAL;
  i128 acc[FIND_LEDGER_KEYS] = {0};
  for (const ElimDesc& d : P->elims) {
    i128 s = d.s, b = d.b;
    const bool split = d.kind == kUpMerge || d.kind == kDownMerge;
    if (d.kind == kFinal) {
      // solver.py:404 naive schur, 410 sigma, 388 inverse c^3, 664 sandwich 2c^3
      if (s > 0) {
        acc[kNaiveDense] += p48_naive_dense(s, b);
        if (compute_gless) acc[kSigmaNaive] += p48_sigma_naive(s, b);
      }
      acc[kDenseInverse] += 48 * b * b * b;
      if (compute_gless) acc[kGlessSandwich] += 96 * b * b * b;
      continue;
    }
    if (s == 0) continue;  // kernels.py:372-375 / 387-388 / 423-427: no charge
    if (!split || kernel == 0) {
      acc[kNaiveDense] += p48_naive_dense(s, b);
      if (compute_gless) acc[kSigmaNaive] += p48_sigma_naive(s, b);
      continue;
    }
    // block kernels (kernels.py:100-111), *_with_factor when G^< is requested
    i128 v = 0;
    const bool wf = compute_gless != 0;
    switch (kernel) {
      case 1: v = wf ? p48_mn(s, b, 8, 3, 6, 1, 4, 1) : p48_mn(s, b, 8, 3, 4, 1, 4, 1); break;
      case 2: v = p48_mn(s, b, 4, 3, 5, 1, 4, 1); break;
      case 3: v = wf ? p48_mn(s, b, 4, 3, 5, 1, 4, 1) : p48_mn(s, b, 4, 3, 4, 1, 5, 1); break;
      case 4: v = wf ? p48_mn(s, b, 8, 3, 15, 2, 4, 1) : p48_mn(s, b, 8, 3, 13, 2, 4, 1); break;
    }
    acc[3 + kernel] += v;
    if (compute_gless) acc[kSigmaSparse] += p48_sigma_sparse(s, b);
  }
  for (int k = 0; k < FIND_LEDGER_KEYS; ++k) num[k] = (int64_t)acc[k];
  *den = 48;
  return FIND_OK;
}

// ---- off-diagonal extraction plan (solver.py:454-484, 644-669) ----
// Every directed adjacent pair (u, v), u != v in A's pattern (operators.py:84-93),
// ascending.  The reference harvests pairs leaf by leaf in the downward DFS
// order, first writer wins (solver.py:666-669): a pair inside one leaf comes
// from that leaf's block G(C, C); a pair across two leaves from the leaf that
// is visited first, as G(ring, C) or G(C, ring) of its extraction.
int find_plan_offdiag_build(find_plan* P) {
  if (P->off_ready) return FIND_OK;
  const int64_t n = P->n, ne = (int64_t)P->elims.size();
  std::vector<int32_t> leaf_elim((size_t)n, -1), pos((size_t)n, -1);
  std::vector<int64_t> dfs((size_t)ne, -1);
  for (int64_t k = 0; k < ne; ++k) {
    const ElimDesc& d = P->elims[k];
    if (d.kind != kFinal) continue;
    auto it = std::lower_bound(P->label_keys.begin(), P->label_keys.end(), d.label);
    if (it == P->label_keys.end() || *it != d.label) return FIND_EINVAL;
    dfs[k] = P->label_index[it - P->label_keys.begin()];  // preorder index = DFS leaf order
    for (int32_t j = 0; j < d.b; ++j) {
      const int32_t node = P->i32[d.rank_off + j];
      leaf_elim[node] = (int32_t)k;
      pos[node] = j;
    }
  }
  for (int64_t v = 0; v < n; ++v)
    if (leaf_elim[v] < 0) return FIND_EINVAL;
  P->off_u.clear();
  P->off_v.clear();
  std::vector<int32_t> owner;
  for (int64_t u = 0; u < n; ++u)
    for (int64_t q = P->indptr[u]; q < P->indptr[u + 1]; ++q) {
      const int64_t v = P->indices[q];
      if (v == u) continue;
      P->off_u.push_back(u);
      P->off_v.push_back(v);
      const int32_t lu = leaf_elim[u], lv = leaf_elim[v];
      owner.push_back(dfs[lu] <= dfs[lv] ? lu : lv);
    }
  const int64_t np = (int64_t)P->off_u.size();
  P->off_item_off.assign((size_t)ne + 1, 0);
  for (int64_t p = 0; p < np; ++p) P->off_item_off[owner[p] + 1]++;
  for (int64_t k = 0; k < ne; ++k) P->off_item_off[k + 1] += P->off_item_off[k];
  P->off_items.assign((size_t)np, OffItem{0, 0, 0, 0, 0});
  std::vector<int64_t> fill(P->off_item_off.begin(), P->off_item_off.end() - 1);
  for (int64_t p = 0; p < np; ++p) {
    const int64_t u = P->off_u[p], v = P->off_v[p];
    const int32_t k = owner[p];
    OffItem it{0, 0, 0, 0, p};
    if (leaf_elim[u] == leaf_elim[v]) {
      it.type = 2; it.r = pos[u]; it.c = pos[v];
    } else if (leaf_elim[v] == k) {
      it.type = 0; it.r = (int32_t)u; it.c = pos[v];  // r resolved below (ring node id -> S position)
    } else {
      it.type = 1; it.r = (int32_t)v; it.c = pos[u];
    }
    P->off_items[fill[k]++] = it;
  }
  std::vector<int32_t> rp((size_t)n, -1);
  for (int64_t k = 0; k < ne; ++k) {
    const int64_t b0 = P->off_item_off[k], b1 = P->off_item_off[k + 1];
    if (b0 == b1) continue;
    const ElimDesc& d = P->elims[k];
    for (int32_t q = 0; q < d.s; ++q) rp[P->slabels[d.slabel_off + q]] = q;
    for (int64_t t = b0; t < b1; ++t) {
      OffItem& it = P->off_items[t];
      if (it.type == 2) continue;
      const int32_t r = rp[it.r];
      if (r < 0) return FIND_EINVAL;  // not in the leaf's ring: cannot happen for a symmetric pattern
      it.r = r;
    }
    for (int32_t q = 0; q < d.s; ++q) rp[P->slabels[d.slabel_off + q]] = -1;
  }
  P->off_ready = true;
  return FIND_OK;
}

int64_t find_plan_offdiag_pairs(find_plan* P, int64_t* u, int64_t* v, int64_t cap) {
  if (!P) return -1;
  try {
    if (find_plan_offdiag_build(P) != FIND_OK) return -1;
  } catch (const std::exception&) {
    return -1;
  }
  const int64_t np = (int64_t)P->off_u.size();
  for (int64_t p = 0; p < std::min(np, cap); ++p) {
    if (u) u[p] = P->off_u[p];
    if (v) v[p] = P->off_v[p];
  }
  return np;
}

void find_plan_free_device(find_plan* P);  // find_solve.cu

void find_plan_destroy(find_plan* P) {
  if (!P) return;
  find_plan_free_device(P);
  delete P;
}

}  // extern "C"
