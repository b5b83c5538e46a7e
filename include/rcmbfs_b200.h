/*
 * rcmbfs_b200.h -- C ABI of the B200-native RCM + direction-optimizing BFS.
 *
 * The reference package (rcmbfs, /root/reference/pkg/src/rcmbfs) has no FFI;
 * its drop-in boundary is the public Python surface (__init__.py:12-105).
 * These entry points are what that surface binds to (see INTEGRATION.md for
 * the ctypes binding).  Every pointer named d_* is a caller-owned DEVICE
 * pointer on the current device; h_* pointers are host memory; stream is a
 * cudaStream_t passed as void*.  Return codes: RB_OK, RB_ERR_ARG (the shim
 * raises ValueError with the reference's message), RB_ERR_CUDA, RB_ERR_OOM.
 * rb_last_error() gives a thread-local message for the last failure.
 */
#ifndef RCMBFS_B200_H
#define RCMBFS_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { RB_OK = 0, RB_ERR_ARG = 1, RB_ERR_CUDA = 2, RB_ERR_NCCL = 3, RB_ERR_OOM = 4 };

const char* rb_last_error(void);
int rb_version(void);

/* ---- input: replaces generator.py:114-148 (kronecker_generate) ---------- */
/* Writes n*edgefactor (u,v) uint32 pairs, byte-identical with the reference
 * (numpy Philox4x64-10 streams keyed (seed, chunk), 65,536-edge chunks). */
int rb_kronecker_generate(int scale, int64_t edgefactor, uint64_t seed, double a, double b, double c,
                          uint32_t* d_edges, void* stream);

/* Edges [e_lo, e_hi) of the same stream (the sharded scale-29 build: each
 * rank draws its share of the 65,536-edge chunks). */
int rb_kronecker_generate_range(int scale, int64_t edgefactor, uint64_t seed, double a, double b, double c,
                                int64_t e_lo, int64_t e_hi, uint32_t* d_edges, void* stream);

/* Chung-Lu power-law graph (BASELINE configs[4]; no reference generator --
 * recipe in paper_2012_10026_b200/generator.py).  d_weights: n positive
 * int64 integer weights; writes m_pairs (u,v) uint32 pairs, each endpoint
 * drawn with probability weight / total from Philox4x64-10 streams keyed
 * (seed, 2^32 + chunk).  Workspace: rb_chunglu_workspace_bytes(n). */
size_t rb_chunglu_workspace_bytes(int64_t n);
int rb_chunglu_generate(const int64_t* d_weights, int64_t n, int64_t m_pairs, uint64_t seed, void* d_ws,
                        size_t ws_bytes, uint32_t* d_edges, void* stream);

/* ---- CSR build: replaces graph.py:85-120 (build_csr) -------------------- */
/* Stage 1 (sizes + error check).  d_edges: m_raw (u,v) uint32 pairs.
 * On an out-of-range edge returns RB_ERR_ARG with *bad_index = first index.
 * ws: workspace of rb_csr_workspace_bytes(m_raw, n) bytes.
 * On success *m_directed = deduplicated directed edge count and the sorted
 * unique keys are kept in ws for stage 2. */
size_t rb_csr_workspace_bytes(int64_t m_raw, int64_t n);
int rb_csr_build(const uint32_t* d_edges, int64_t m_raw, int64_t n, void* d_ws, size_t ws_bytes,
                 int64_t* m_directed, int64_t* bad_index, void* stream);
/* Stage 2: materialize CSR from ws (row_starts n+1 int64, col m_directed
 * int32, degrees n int32). */
int rb_csr_emit(const void* d_ws, int64_t m_directed, int64_t n, int64_t* d_row_starts,
                int32_t* d_col, int32_t* d_degrees, void* stream);

/* Sharded build / relabel (configs[3], paper_2012_10026_b200/sharded.py):
 * rb_csr_keys: the sorted unique keys (u << 32 | v) rb_csr_build left in its
 * workspace (what a rank routes to the owners of u);
 * rb_keys_sort_unique: sort keys[0, m) on the low end_bit bits and drop
 * duplicates in place (workspace rb_keys_workspace_bytes(m));
 * rb_keys_to_csr: CSR rows of the vertex block [v_lo, v_lo + n_local) from
 * its sorted unique keys (row starts from 0, global column ids, degrees);
 * rb_relabel_keys: keys inv[v] << 32 | inv[w] of a block's rows (its part of
 * apply_permutation, to be routed to the owners of the new ids). */
int rb_csr_keys(const void* d_ws, const uint64_t** d_keys, int64_t* m_directed);
size_t rb_keys_workspace_bytes(int64_t m);
int rb_keys_sort_unique(uint64_t* d_keys, int64_t m, int end_bit, void* d_ws, size_t ws_bytes, int64_t* m_out,
                        void* stream);
int rb_keys_to_csr(const uint64_t* d_keys, int64_t m, int64_t v_lo, int64_t n_local, int64_t* d_row_starts,
                   int32_t* d_col, int32_t* d_degrees, void* stream);
int rb_relabel_keys(const int64_t* d_row_starts, const int32_t* d_col, int64_t n_local, int64_t v_lo,
                    const uint32_t* d_inv, uint64_t* d_keys, void* stream);

/* ---- RCM: replaces reorder.py:198-237 (rcm / _rcm_impl / _rcm_walk) ----- */
/* Outputs perm (new->old) and inv (old->new), |V+|, component ranges (pairs of
 * new-id [start,end), ascending by start; capacity n pairs).  Bit-exact with
 * the reference's sequential walk. */
size_t rb_rcm_workspace_bytes(int64_t n, int64_t m_directed);
int rb_rcm(const int64_t* d_row_starts, const int32_t* d_col, const int32_t* d_degrees, int64_t n,
           void* d_ws, size_t ws_bytes, uint32_t* d_perm, uint32_t* d_inv, int64_t* n_plus,
           int64_t* d_comp_ranges, int64_t* n_components, void* stream);

/* ---- relabel: replaces reorder.py:254-271 (apply_permutation) ----------- */
size_t rb_permute_workspace_bytes(int64_t n, int64_t m_directed);
int rb_apply_permutation(const int64_t* d_row_starts, const int32_t* d_col, const int32_t* d_degrees,
                         int64_t n, int64_t m_directed, const uint32_t* d_perm, const uint32_t* d_inv,
                         void* d_ws, size_t ws_bytes, int64_t* d_row_starts_out, int32_t* d_col_out,
                         int32_t* d_degrees_out, void* stream);
/* degree_sort_adjacency (reorder.py:151-195): rows re-sorted by (deg, id)
 * ascending or by (deg desc, id asc). */
int rb_degree_sort_adjacency(const int64_t* d_row_starts, const int32_t* d_col, const int32_t* d_degrees,
                             int64_t n, int64_t m_directed, int descending, void* d_ws, size_t ws_bytes,
                             int32_t* d_col_out, void* stream);

/* ---- BFS engine: replaces engine.py:478-617 (BfsEngine / bfs_run) ------- */
typedef struct rb_bfs rb_bfs;

typedef struct {
  int64_t level;
  int64_t direction; /* 0 = top_down, 1 = bottom_up (the reference policy's label) */
  int64_t n_f;
  int64_t m_f;
  int64_t m_u;
  int64_t scanned_edges; /* TD: edges examined; BU: neighbour checks */
  int64_t t_ns;          /* device %globaltimer duration of the level */
  int64_t n_next;
  int64_t t_queue_ns;    /* part of t_ns before the top-down hub phase (phase A) */
  int64_t reserved;      /* executed direction: 0 = top_down, 1 = bottom_up */
  /* LevelRecord fields of the partitioned modes (engine.py:166-180), -1 = None:
   * pass1_hits: bottom-up vertices found by their first scanned neighbour
   * (bu_reduced pass 1, _kernels.py:254-266; counted when the engine was given
   * RB_PART_COUNT_PASS1); live_vertices: PartitionSet.live_total() after the
   * bottom-up level (partition.py:70-72, live bounds shrunk past all-visited
   * 512-vertex blocks; RB_PART_SHRINK); claimed: partitions claimed (set by
   * the host shim: every partition is claimed once per bottom-up step). */
  int64_t pass1_hits;
  int64_t live_vertices;
  int64_t claimed;
  int64_t reserved2;
} rb_level_record;

typedef struct {
  int32_t alpha;      /* engine.py:85 */
  int32_t beta;       /* engine.py:86 */
  int32_t hybrid;     /* 0 = level_sync (top-down only) */
  int32_t bu_reverse; /* scan bottom-up rows from their end */
  int64_t n_policy;   /* g.n incl. isolated (engine.py:593) */
  int64_t m_directed; /* g.m_directed */
  int32_t record_levels; /* also keep a per-vertex level array (not part of
                            the reference's BfsResult; costs 4 B per reached
                            vertex in the traversal); 0 = parents only */
  int32_t reserved0;
} rb_bfs_params;

/* d_col_bu may equal d_col.  n_dev: vertices [0,n_dev) live on the device
 * (isolated tail dropped); d_isolated_words marks isolated vertices inside
 * [0,n_dev) (uint32 words, bit v -> word v>>5), may be NULL. */
int rb_bfs_create(const int64_t* d_row_starts, const int32_t* d_col, const int32_t* d_col_bu,
                  const int32_t* d_degrees, int64_t n_dev, const uint32_t* d_isolated_words,
                  const rb_bfs_params* params, rb_bfs** out);
int rb_bfs_destroy(rb_bfs* h);

/* 1D vertex-block partition (multi-GPU): this engine owns global
 * vertices [v_lo, v_lo + n_dev); its CSR rows (d_row_starts local, columns
 * GLOBAL ids) serve bottom-up; top-down expands every global frontier vertex
 * through the transpose slice d_td_row_starts / d_td_col (the owned
 * neighbours of each of the n_glob global vertices). */
typedef struct {
  int64_t v_lo;
  int64_t n_glob;
  const int64_t* d_td_row_starts;
  const int32_t* d_td_col;
} rb_bfs_partition;
int rb_bfs_create_part(const int64_t* d_row_starts, const int32_t* d_col, const int32_t* d_col_bu,
                       const int32_t* d_degrees, int64_t n_dev, const uint32_t* d_isolated_words,
                       const rb_bfs_params* params, const rb_bfs_partition* part, rb_bfs** out);
/* Partitioned traversal, driven level by level by the host (which exchanges
 * frontier bitmaps and counters, e.g. with NCCL): reset (seeds the source if
 * owned), then one level from the all-gathered global frontier bitmap (+ its
 * nonzero summary, rb_make_nz).  Returns the local next-frontier words and the
 * local counters n_next, deg_next, maxdeg, scanned. */
int rb_bfs_reset_part(rb_bfs* h, int64_t source_global, void* stream);
int rb_bfs_dist_level(rb_bfs* h, int64_t level, int direction, int hubs, const uint32_t* d_fcur_glob,
                      const uint8_t* d_nz_glob, uint32_t** d_next_local, int64_t* h_counters, void* stream);
int rb_bfs_words(rb_bfs* h, int64_t* n_words_local, int64_t* n_words_glob);

/* Device-side exchange for the 1D partition (the level loop stays on the
 * device; replaces the per-level all-gather / all-reduce of the host-driven
 * path above).  Per rank: rb_bfs_xchg_alloc (three global frontier bitmaps +
 * summaries, counter slots, barrier counter in one allocation), then either
 *   multi-process: rb_bfs_xchg_handle -> exchange the world handles (e.g.
 *   torch.distributed.all_gather_object) -> rb_bfs_xchg_open (cudaIpc, NVLink
 *   peer mappings), and per root rb_bfs_dist_reset + rb_bfs_dist_traverse on
 *   every rank (ONE persistent launch each: at every level a rank stores its
 *   next-frontier words and counters into every peer's buffers and meets the
 *   others at a system-scope barrier), rb_bfs_dist_results;
 *   one GPU (emulation of `world` ranks): rb_bfs_xchg_connect_local over the
 *   ranks' engines of this process, rb_bfs_dist_reset each, then
 *   rb_bfs_dist_traverse_emu (ONE cooperative launch over all ranks' data).
 * Records are written by rank 0's engine.  world <= 8; v_lo % 128 == 0. */
int rb_bfs_xchg_alloc(rb_bfs* h, int32_t world, int32_t rank);
size_t rb_bfs_xchg_handle_bytes(void);
int rb_bfs_xchg_handle(rb_bfs* h, void* h_handle_out);
int rb_bfs_xchg_open(rb_bfs* h, const void* h_handles /* world handles, rank order */);
int rb_bfs_xchg_connect_local(rb_bfs* const* hs, int32_t world);
int rb_bfs_dist_reset(rb_bfs* h, int64_t source_global, int64_t deg_source, void* stream);
int rb_bfs_dist_traverse(rb_bfs* h, void* stream);
int rb_bfs_dist_traverse_emu(rb_bfs* const* hs, int32_t world, void* stream);
int rb_bfs_dist_results(rb_bfs* h, rb_level_record* h_records, int64_t cap, int64_t* n_records, double* elapsed_s,
                        void* stream);
/* Nonzero summary of a bitmap: d_nz[i] = (d_words[i] != 0), one byte per word. */
int rb_make_nz(const uint32_t* d_words, int64_t n_words, uint8_t* d_nz, void* stream);
/* Transpose slice for a partition: for every global vertex u < n_glob, the
 * owned vertices adjacent to u (ascending). */
size_t rb_transpose_workspace_bytes(int64_t m_local, int64_t n_glob);
int rb_transpose_rows(const int64_t* d_row_starts_local, const int32_t* d_col_local, int64_t n_local, int64_t v_lo,
                      int64_t m_local, int64_t n_glob, void* d_ws, size_t ws_bytes, int64_t* d_td_row_starts,
                      int32_t* d_td_col, void* stream);
/* Partition bookkeeping of the reference's partitioned modes (hybrid_balanced,
 * hybrid_reduced; engine.py:499-500, partition.py:67-171).  h_bounds: n_parts+1
 * vertex boundaries of get_partitions(n_full, partition_factor, threads)
 * (host memory; starts 512-aligned, last = n_full = g.n).  flags:
 *   RB_PART_EXACT        every level runs the direction the policy labels (no
 *                        cost-model execution), so scanned_edges is the
 *                        reference's count for the scan order given;
 *   RB_PART_COUNT_PASS1  records carry pass1_hits;
 *   RB_PART_SHRINK       records carry live_vertices (bounds shrunk as
 *                        bu_reduced does).
 * n_parts = 0 clears it. */
enum { RB_PART_EXACT = 1, RB_PART_COUNT_PASS1 = 2, RB_PART_SHRINK = 4 };
int rb_bfs_set_partitions(rb_bfs* h, const int64_t* h_bounds, int64_t n_parts, int64_t n_full, int32_t flags);
/* Reset per-root state (not timed; engine.py:526-532). */
int rb_bfs_reset(rb_bfs* h, int64_t source, void* stream);
/* The traversal (engine.py:534-598): one cooperative persistent launch. */
int rb_bfs_traverse(rb_bfs* h, void* stream);
/* Device time of the last traversal (all of its launches), seconds. */
int rb_bfs_elapsed(rb_bfs* h, double* seconds);
/* Copy results; parents/levels cover [0,n_dev); n_records <= cap. */
/* Asynchronous result path (BfsEngine.run, engine.py:518-604): enqueue the
 * copies of the launch state (rb_bfs_state_bytes() bytes), of the first `cap`
 * level records and (if h_parent) of the parents in `chunks` pieces behind
 * the traversal on `stream`, without waiting.
 * After the caller synchronizes the stream, rb_bfs_complete() returns 0 and
 * the record count when that launch finished the traversal, or 1 when the
 * caller must drain with rb_bfs_results (continuation launches). */
int rb_bfs_results_async(rb_bfs* h, void* h_state, rb_level_record* h_records, int64_t cap, int32_t* h_parent,
                         int32_t chunks, void* stream);
/* Wait for those copies: what = -1 the state + records, what = i (< chunks,
 * <= 32) the i-th of `chunks` equal pieces of the parents [0, n_dev) that were
 * enqueued into h_parent (pinned host memory). */
int rb_bfs_wait(rb_bfs* h, int32_t what);
int rb_bfs_complete(rb_bfs* h, const void* h_state, const rb_level_record* h_records, int64_t cap,
                    int64_t* n_records);
size_t rb_bfs_state_bytes(void);
int rb_bfs_results(rb_bfs* h, int32_t* d_or_h_parent, int32_t* d_or_h_level, rb_level_record* h_records,
                   int64_t cap, int64_t* n_records, void* stream);
/* One step from an explicit state (top_down_step / bottom_up_step,
 * engine.py:252-429): state words are uint32 over [0,n_dev). */
int rb_bfs_step(rb_bfs* h, int direction, const uint32_t* d_visited_words, const uint32_t* d_frontier_words,
                const int32_t* d_parent_in, uint32_t* d_visited_out, uint32_t* d_next_out,
                int32_t* d_parent_out, int64_t* h_counters /* n_next, deg_next, scanned */, void* stream);
/* Device pointers of the engine-owned parent / level arrays. */
int32_t* rb_bfs_parent_ptr(rb_bfs* h);
int32_t* rb_bfs_level_ptr(rb_bfs* h);
int rb_bfs_grid(rb_bfs* h, int* blocks, int* threads);
/* Diagnostics: average cost of one grid barrier of the traversal grid. */
int rb_bfs_barrier_probe(rb_bfs* h, int iters, double* ns_per_barrier, void* stream);
/* Diagnostics (engine created with RB_DEBUG_TS set): per level (first 64),
 * per CTA: globaltimer at level start, after the work + block reduction,
 * after the grid barrier, 0. */
int rb_bfs_debug_timestamps(rb_bfs* h, uint64_t* out, int64_t cap, int* blocks);

/* ---- tree validation (validate.py:63-225) ----------- */
/* Component labels = min vertex id of the component (validate.py:63-84),
 * by device union-find over the raw edge list d_edges (m_raw pairs, may hold
 * duplicates / self loops) or, if d_edges is NULL, over the CSR. */
int rb_components(const int64_t* d_row_starts, const int32_t* d_col, int64_t n, const uint32_t* d_edges,
                  int64_t m_raw, int32_t* d_labels, void* stream);
size_t rb_validate_workspace_bytes(int64_t n);
/* The five rules of Validator.validate (validate.py:123-225) for one
 * predecessor array.  d_levels receives the derived levels (-1 unreached or
 * unresolved).  h_first_bad[5]: per rule -1 if it passed, else the first
 * counterexample the reference reports -- rule 1: the source; 2: vertex
 * (out-of-range parents take precedence); 3: vertex; 4: CSR edge index;
 * 5: vertex.  RB_ERR_ARG if source is out of range. */
int rb_validate(const int64_t* d_row_starts, const int32_t* d_col, int64_t n, const int32_t* d_labels,
                int64_t source, const int32_t* d_parent, void* d_ws, size_t ws_bytes, int32_t* d_levels,
                int64_t* h_first_bad, void* stream);

/* ---- sequential BFS parents (_kernels.py:26-54 seq_bfs_kernel) ---------- */
/* The parent array of the reference's queue BFS from `source` -- parent[w] =
 * the neighbour that discovers w first in queue order -- computed from the
 * level array of a level-synchronous traversal (d_level[v] = depth, < 0 for
 * unreached vertices; n_levels = depth + 1).  Bit-exact with seq_bfs_kernel
 * for any row order.  d_parent: n int32 (-1 unreached). */
int rb_bfs_first_parents(const int64_t* d_row_starts, const int32_t* d_col, int64_t n, const int32_t* d_level,
                         int64_t source, int64_t n_levels, int32_t* d_parent, void* stream);

/* ---- host-side result assembly ------------------------------------------ */
/* h_dst[0, n) = value with streaming stores from up to `threads` host threads:
 * the -1 tail of BfsResult.predecessor for the isolated vertices behind n_dev
 * (engine.py:598), written while the parents are DMA'd into the head. */
int rb_host_fill_i32(int32_t* h_dst, int64_t n, int32_t value, int threads);

#ifdef __cplusplus
}
#endif
#endif
