/*
 * find_b200.h — C ABI of the B200-native FIND selected-inversion path.
 *
 * Drop-in boundary for the reference package find_selinv 0.1.0
 * (/root/reference/pkg/src/find_selinv).  The reference is pure Python; its
 * "FFI" for this path is the Python call
 *     solve(mesh, a, sigma, config) -> SelectedInverse      (solver.py:586-701)
 * which the Python host package paper_1104_0623_b200 keeps verbatim and
 * implements on top of the entry points below (ctypes binding, see
 * INTEGRATION.md).  No torch types cross this boundary: plain pointers,
 * sizes and a cudaStream_t passed as void*.
 *
 * Complex numbers are interleaved (re, im) doubles — the memory layout of
 * numpy/torch complex128.
 *
 * Return codes: FIND_OK 0, FIND_EINVAL 1 (invalid argument, maps to
 * ValueError, solver.py:591-608), FIND_ESINGULAR 2 (singular pivot, maps to
 * SingularPivotError, kernels.py:237-252 / solver.py:383-389),
 * FIND_ECUDA 3 (CUDA error), FIND_ENOMEM 4 (workspace too small).
 */
#ifndef FIND_B200_H
#define FIND_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FIND_OK 0
#define FIND_EINVAL 1
#define FIND_ESINGULAR 2
#define FIND_ECUDA 3
#define FIND_ENOMEM 4

typedef struct find_plan find_plan;

/* Status of one find_solve call (device-side pivot test mapped back to the
 * reference's SingularPivotError(node, cluster), errors.py:8-18). */
typedef struct find_status {
  int32_t code;          /* FIND_* */
  int32_t energy_idx;    /* energy point of the failing elimination, -1 if none */
  int64_t cluster_label; /* cluster label (negative: complement cluster), 0 if none */
  int64_t node_id;       /* mesh node of the failing pivot, -1 if none */
  double pivot_ratio;    /* |u_kk| / max|A(S,S)| at the failing pivot (NaN if unknown) */
  char message[160];
} find_status;

/* ---- energy-independent plan (host only; replaces build_cluster_tree +
 *      annotate_boundaries + complement_boundary_sets, mesh.py:176-290, and
 *      the merge bookkeeping of solver.py:97-132, 234-243) ---- */

/* Build the nested-dissection plan for an nx*ny mesh whose operator has CSR
 * pattern (indptr[n+1], indices[nnz]); node id = x + nx*y.  The pattern
 * must be structurally symmetric (solver.py:593-594).  leaf_max as
 * SolverConfig.leaf_max (mesh.py:176-206). */
int find_plan_create(int64_t nx, int64_t ny, const int64_t* indptr, const int64_t* indices,
                     int64_t nnz, int32_t leaf_max, find_plan** out, find_status* st);
void find_plan_destroy(find_plan* plan);

/* Plan statistics: out[0..15] = {n, nnz, n_clusters, n_elims, n_levels_up,
 * n_levels_down, up_arena_elems, down_arena_elems, ws_elems, max_n, max_s,
 * max_b, n_launch_groups, sparse_entries, tree_depth, n_leaves}. */
int find_plan_info(const find_plan* plan, int64_t* out16);

/* Node sets of one cluster, ascending ids (for set-for-set validation
 * against mesh.py:209-290).  which: 0 = nodes, 1 = boundary B,
 * 2 = private inner S, 3 = complement boundary B_{-c}, 4 = complement
 * private inner S_{-c}.  Returns the set size (writes min(size, cap)
 * entries), or -1 if the label does not exist. */
int64_t find_plan_cluster_set(const find_plan* plan, int64_t label, int32_t which, int64_t* out,
                              int64_t cap);

/* Per-elimination shapes in execution order: kind (0 leaf seed, 1 upward
 * merge, 2 downward merge, 3 final leaf step), s, b, label.  Arrays of
 * n_elims entries (find_plan_info out[3]). */
int find_plan_elims(const find_plan* plan, int32_t* kind, int32_t* s, int32_t* b, int64_t* label);

/* Per elimination (find_plan_elims order): when the block A(B_r, S_l) of the merged
 * matrix [S_l, S_r, B_l, B_r] is structurally zero (no exception entry; the paper's zero
 * sub-blocks, kernels.py:400-463), s_left = |S_l| and b_left = |B_l| (the kernels then skip
 * the products with Y(B_r, S_l) = 0); otherwise both 0.  Any pointer may be NULL. */
int find_plan_elim_splits(const find_plan* plan, int32_t* s_left, int32_t* b_left);

/* Per elimination (find_plan_elims order): the arena (-1: none) and complex-element offset of
 * its output block pair U [b][b], R [b][b] (sorted-B order; R at +b*b) within one energy
 * point's slice of that arena; the arenas follow the 256-byte status header of the workspace in
 * order, arena a holding n_energies * arena_elems[a] complex elements (find_plan_arena_elems). */
int find_plan_elim_out(const find_plan* plan, int32_t* out_arena, int64_t* out_off);

/* Complex elements per energy point of each of the four block arenas (0: upward U/R blocks,
 * 1-3: downward complement blocks). */
int find_plan_arena_elems(const find_plan* plan, int64_t* out4);

/* CSR slots of the merge-structure exception entries (kernels.py:192-202,
 * counted into SelectedInverse.stats at solver.py:217-219) for pass 0
 * (upward merges) or 1 (downward merges); an entry counts when its value is
 * nonzero.  Returns the number of slots (writes min(count, cap)). */
int64_t find_plan_exception_slots(const find_plan* plan, int32_t pass, int64_t* out, int64_t cap);

/* Exact multiplication count of the reference FlopLedger (kernels.py:48-146,
 * charged at kernels.py:379,391,436, solver.py:388,664) for one energy
 * point.  kernel: 0 naive, 1 parallel_inverse, 2 sequential_inverse,
 * 3 block_lu, 4 naive_lu (KERNEL_NAMES order, solver.py:49).  Writes
 * per-ledger-key numerators over the common denominator *den (=48) into
 * num[FIND_LEDGER_KEYS] in the key order of find_ledger_key_name(). */
#define FIND_LEDGER_KEYS 12
int find_plan_ledger(const find_plan* plan, int32_t kernel, int32_t compute_gless, int64_t* num,
                     int64_t* den);
const char* find_ledger_key_name(int32_t key);

/* ---- device side ---- */

/* Bytes of device workspace find_solve needs for n_energies points. */
size_t find_solve_workspace_bytes(const find_plan* plan, int32_t n_energies, int32_t compute_gless);

/* Upload the plan's index maps to the current device (idempotent). */
int find_plan_upload(find_plan* plan, find_status* st);

/* Selected inversion for n_energies operators sharing the plan's pattern.
 *   a_vals   device, [n_energies][nnz] complex128 (values of A(E_k) on the pattern)
 *   s_vals   device, [nnz] complex128 if s_broadcast else [n_energies][nnz]
 *            (Sigma^< on A's pattern; zeros where Sigma^< has no entry);
 *            may be NULL when compute_gless == 0
 *   gr_out   device, [n_energies][n] complex128  diag(G^r)
 *   gl_out   device, [n_energies][n] complex128  diag(G^<) (NULL if !compute_gless)
 *   compute_gless  0: diag(G^r) only; 1: also diag(G^<); 2 / 3: also diag(G^<)
 *            and Sigma^< is Hermitian / skew-Hermitian (e.g. i*Gamma), so every
 *            R block is too; the upward pass then computes only the lower
 *            triangle of each R and mirrors it (the paper's symmetry saving
 *            for R; the downward pass keeps the general product)
 *   ws       device workspace of >= find_solve_workspace_bytes()
 *   stream   cudaStream_t
 * Stream-ordered; on return the work is enqueued.  Call find_solve_status()
 * (synchronises the stream) to obtain the pivot status. */
int find_solve(find_plan* plan, const void* a_vals, const void* s_vals, int32_t s_broadcast,
               int32_t n_energies, int32_t compute_gless, double pivot_rtol, void* gr_out,
               void* gl_out, void* ws, size_t ws_bytes, void* stream, find_status* st);

/* Same as find_solve restricted to launch groups [g_begin, g_end) of the
 * plan's schedule (upward levels deepest-first, then per level the downward
 * merges and the final leaf steps).  The device status word is reset only
 * when g_begin == 0.  Used for per-level timing. */
int find_solve_groups(find_plan* plan, const void* a_vals, const void* s_vals, int32_t s_broadcast,
                      int32_t n_energies, int32_t compute_gless, double pivot_rtol, void* gr_out,
                      void* gl_out, void* ws, size_t ws_bytes, int64_t g_begin, int64_t g_end,
                      void* stream, find_status* st);

/* ---- off-diagonal extraction (SolverConfig.compute_offdiag, solver.py:454-484,
 *      637-642, 666-669; the G^< cross blocks of _extended_extraction,
 *      solver.py:487-507) ---- */

/* Directed adjacent pairs (u, v), u != v in the plan's pattern (a.adjacency(),
 * operators.py:84-93), in ascending (u, v) order: the index space of the
 * off_gr / off_gl outputs of find_solve_offdiag.  Builds the per-leaf
 * extraction lists on first use.  Returns the pair count (writes
 * min(count, cap) entries; u / v may be NULL), or -1 on failure. */
int64_t find_plan_offdiag_pairs(find_plan* plan, int64_t* u, int64_t* v, int64_t cap);

/* find_solve that also writes G^r(u, v) (off_gr) and, when compute_gless and
 * off_gl != NULL, G^<(u, v) (off_gl) for every pair of find_plan_offdiag_pairs:
 * device arrays [n_energies][n_pairs] complex128.  Each pair is taken from the
 * extraction of the leaf the reference's downward DFS visits first
 * (solver.py:666-669).  Leaves of more than 16 nodes are rejected (FIND_EINVAL). */
int find_solve_offdiag(find_plan* plan, const void* a_vals, const void* s_vals, int32_t s_broadcast,
                       int32_t n_energies, int32_t compute_gless, double pivot_rtol, void* gr_out,
                       void* gl_out, void* off_gr, void* off_gl, void* ws, size_t ws_bytes, void* stream,
                       find_status* st);
int find_solve_offdiag_groups(find_plan* plan, const void* a_vals, const void* s_vals, int32_t s_broadcast,
                              int32_t n_energies, int32_t compute_gless, double pivot_rtol, void* gr_out,
                              void* gl_out, void* off_gr, void* off_gl, void* ws, size_t ws_bytes,
                              int64_t g_begin, int64_t g_end, void* stream, find_status* st);

/* Launch-group table (find_plan_info out[12] entries): pass (0 upward,
 * 1 downward, 2 final), tree level, path (0 warp-per-elimination, 1 CTA),
 * number of eliminations, and the largest s+b, s, b in the group.  Any
 * pointer may be NULL. */
int find_plan_groups(const find_plan* plan, int32_t* pass, int32_t* level, int32_t* path, int64_t* count,
                     int32_t* max_n, int32_t* max_s, int32_t* max_b);

/* Kernel-launch table of a find_solve over n_energies points, in issue order
 * (find_solve_launch_count() entries): launch kind (0 warp path, 1 gather A,
 * 2 panel, 3 TRSM, 4 trailing, 5 X solve, 6 finish, 7 gather Sigma, 8 T_S,
 * 9 R, 10 final, 11 Schur, 12 fused LU, 13 mid path, 14 off-diagonal, 15 panel inverses), panel step, launch
 * group, task count.  Any pointer may be NULL. */
int find_plan_specs(const find_plan* plan, int32_t n_energies, int32_t* kind, int32_t* step, int32_t* group,
                    int64_t* tasks);

/* Per launch group: its phase (the groups of a phase are independent and run
 * concurrently; phases run in order). */
int find_plan_group_phases(const find_plan* plan, int32_t* phase);

/* Opt-in per-launch device timing (process-wide, for benchmarks): while
 * enabled every kernel launch of find_solve is bracketed by CUDA events on its
 * stream.  find_solve_timing_enable(1) also clears the record;
 * find_solve_timing_read() synchronises the events and returns the number of
 * recorded launches (writes launch kind as in find_plan_specs, group, ms). */
void find_solve_timing_enable(int32_t enable);
int64_t find_solve_timing_read(int32_t* kind, int32_t* group, float* ms, int64_t cap);
/* Same record as start / end times (ms) relative to the first recorded launch
 * (a timeline across the side streams). */
int64_t find_solve_timing_read2(int32_t* kind, int32_t* group, float* t_begin, float* t_end, int64_t cap);

/* Synchronise `stream` and decode the device status of the last find_solve
 * that used `ws`. */
int find_solve_status(find_plan* plan, void* ws, int32_t n_energies, void* stream, find_status* st);

/* Number of kernel launches one find_solve over n_energies points enqueues. */
int64_t find_solve_launch_count(const find_plan* plan, int32_t n_energies);

/* Unit-test shim with the reference's kernel-level signature
 * schur_update + sigma_update (kernels.py:363-392) for ONE dense
 * elimination input: ass[s*s], asb[s*b], abs[b*s], abb[b*b], and the four
 * Sigma blocks (may be NULL), all row-major device buffers; writes
 * u_out[b*b], r_out[b*b], l_out[b*s] (L = A(B,S) A(S,S)^{-1}).  Runs the
 * same device code path as find_solve (force_path: -1 auto, 0 warp path,
 * 1 blocked CTA path, 2 CTA-per-elimination shared-memory path).  Returns FIND_ESINGULAR with st->node_id = position k of the
 * failing pivot. */
int find_schur_sigma_update(int32_t s, int32_t b, const void* ass, const void* asb, const void* abs_,
                            const void* abb, const void* sss, const void* ssb, const void* sbs,
                            const void* sbb, double pivot_rtol, void* u_out, void* r_out, void* l_out,
                            int32_t force_path, void* stream, find_status* st);

/* ---- Dense batched primitives on the FIND kernels (the RGF comparison path,
 * find_selinv/rgf.py:108-208: g_i = (D_i - F g E)^-1 and the G / Sigma sandwiches).
 *
 * find_dense: batched inverse of `batch` complex128 n x n matrices (row-major, contiguous,
 * device).  Each matrix is one blocked elimination of [[A, I], [I, 0]] by the same panel /
 * TRSM / DMMA kernels as find_solve (replaces numpy.linalg.inv at rgf.py:84-87); the handle owns
 * the one-elimination plan and its workspace.  find_dense_inverse is asynchronous on `stream`;
 * status_out (device, 8 bytes, may be NULL) receives the call's status word: all ones when
 * every pivot was nonzero, else (energy << 16 | position) of the first zero pivot. */
typedef struct find_dense find_dense;
int find_dense_create(int32_t n, int32_t batch, find_dense** out, find_status* st);
void find_dense_destroy(find_dense* h);
int find_dense_inverse(find_dense* h, const void* a, void* inv_out, void* status_out, void* stream,
                       find_status* st);

/* Strided-batched complex128 GEMM on the DMMA tiles (replaces the `@` products of
 * rgf.py:92-105, 121-136, 139-208): C[i] (mode 0: =, +1: +=, -1: -=) A[i] op(B[i]) for
 * i < batch, A [m][k] row stride lda, B [k][n] row stride ldb (b_conj_trans = 0) or B [n][k]
 * used as its conjugate transpose (b_conj_trans = 1), C [m][n] row stride ldc; sa / sb / sc are
 * the batch strides in complex elements (0 broadcasts an operand). */
int find_zgemm_batched(int32_t batch, int32_t m, int32_t n, int32_t k, const void* a, int64_t lda, int64_t sa,
                       const void* b, int64_t ldb, int64_t sb, int32_t b_conj_trans, void* c, int64_t ldc,
                       int64_t sc, int32_t mode, void* stream, find_status* st);

#ifdef __cplusplus
}
#endif

#endif /* FIND_B200_H */
