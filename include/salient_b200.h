/*
 * salient_b200.h — C-ABI of the B200-native SALIENT batch-preparation library
 * (libsalient_b200.so, built from paper_2110_08450_b200/csrc for sm_100a).
 *
 * The reference (`mfgprep`, /root/reference/pkg/src/mfgprep) has no native
 * boundary of its own: its operator layer is a set of numba @njit functions
 * over numpy arrays (`_kernels.py`).  Each entry point below replaces one of
 * those operators, or one step of the Python driver that chains them; the
 * reference symbol is cited on every declaration.  INTEGRATION.md shows the
 * ctypes stub a maintainer adds to `mfgprep` to bind this library.
 *
 * Conventions
 *   - every pointer argument named *_dev or typed as device data is a CUDA
 *     device pointer; `stream` is a cudaStream_t (NULL = legacy default);
 *   - calls only enqueue work (asynchronous); device faults surface at the
 *     caller's next synchronisation;
 *   - return value: 0 = SAL_OK, <0 = error; sal_last_error() returns a
 *     thread-local message describing the last failure on this thread;
 *   - node ids on device are int32 (graphs up to 2^31-1 nodes), the graph
 *     row pointer is int64, MFG row pointers / source locals are int32;
 *   - nothing here allocates device memory: callers pass workspaces sized by
 *     the *_bytes / layout helpers.  No global mutable state apart from the
 *     per-thread error message; reentrant across streams and threads.
 */
#ifndef SALIENT_B200_H
#define SALIENT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SAL_OK 0
#define SAL_EINVAL (-1)
#define SAL_ECUDA (-2)

#define SAL_MAX_HOPS 8

/* RNG policies of the sampler.  SPLITMIX reproduces the reference draw
 * stream bit-exactly (rng.py:16-35, _kernels.py:30-39); PHILOX is the
 * north-star counter-based policy keyed on (seed, batch, hop, dst). */
#define SAL_RNG_SPLITMIX 0
#define SAL_RNG_PHILOX 1

/* element types (values 1/2 match graph.py:18-19 DTYPE_F16 / DTYPE_F32) */
#define SAL_F16 1
#define SAL_F32 2
#define SAL_BF16 3

/* CSR graph resident in HBM (graph.py:39-85 CsrGraph). */
typedef struct {
  int64_t num_nodes;
  int64_t num_edges;
  const int64_t* indptr;  /* device, int64[num_nodes + 1] */
  const int32_t* indices; /* device, int32[num_edges]     */
} sal_graph;

/* Device-resident descriptor of one seed batch (prep.py:40-52 SeedBatch):
 * seeds = seeds_base[seed_offset : seed_offset + n_seeds]. */
typedef struct {
  int64_t batch_id;
  int64_t seed_offset;
  int64_t n_seeds;
} sal_batch_desc;

/* Global->local map (sampler.py:106-171 IdMap, flat_probing variant).
 * table: 64-bit slots, table_cap a power of two, reset to all-ones bytes. */
typedef struct {
  unsigned long long* table;
  int64_t table_cap;
  int32_t* globals; /* local -> global, capacity globals_cap */
  int64_t globals_cap;
} sal_idmap;

/* Capacities of one multi-hop sample (sampler.py:321-346). */
typedef struct {
  int32_t num_hops;
  int32_t fanout[SAL_MAX_HOPS];         /* expansion order: per_hop[L-1-h] */
  int64_t max_seeds;
  int64_t node_cap[SAL_MAX_HOPS + 1];   /* max id-map size after h hops   */
  int64_t edge_cap[SAL_MAX_HOPS];       /* max edges emitted by hop h     */
  int64_t table_cap;
  int32_t flags;                        /* SAL_MFG_* plan flags            */
  /* SAL_MFG_LAST_HOP_FUSED plans: hop L-2's relabel second pass (its src_local) runs
   * inside sal_sample_aggregate's kernel instead of at the end of sal_sample_mfg, so
   * the fused kernel starts one launch earlier; read the MFG after the aggregate */
  int32_t resolve_in_aggregate;
  /* sampler launch shape (sal_hop_sample_tuned; 0 = default), set by the
   * caller after sal_mfg_plan_init; the caller may also raise table_cap (a
   * power of two) before sal_mfg_layout_init to lower the id-table load */
  int32_t sample_lanes;
  int32_t sample_blocks_per_sm;
  /* resident blocks per SM of sal_sample_aggregate (0 = as many as shared memory
   * allows); a trainer caps it so its weight-gradient CTAs fit beside it */
  int32_t aggregate_blocks_per_sm;
  /* SAL_MFG_LAST_HOP_FUSED plans: sal_sample_mfg skips the id-table and scan-workspace
   * resets and sal_sample_aggregate leaves them reset for the workspace's next batch
   * (the caller resets the workspace once before its first batch) — two memset nodes
   * fewer at the head of a pipelined batch preparation */
  int32_t reset_in_aggregate;
} sal_mfg_plan;

/* Plan flag: the last hop emits its edges as global ids only (layout.src_glob);
 * no id-map insertion, no relabel, sizes[L] = -1 and src_local[L-1] is not
 * written.  For training with the layer-0 aggregation read straight from the
 * feature table, where the last hop's local ids are never consumed; the id
 * map then only holds hops 0..L-2 (table_cap sized for node_cap[L-1]). */
#define SAL_MFG_LAST_HOP_EDGES 1
/* Plan flag: the last hop is not materialised at all.  sal_sample_mfg builds
 * hops 0..L-2 (the id map holds their nodes, as with SAL_MFG_LAST_HOP_EDGES);
 * sal_sample_aggregate then samples the last hop and reduces it into the
 * layer-0 mean in one pass (no src_glob, no dst_indptr for hop L-1).  Also
 * sets the SAL_MFG_LAST_HOP_EDGES sizing. */
#define SAL_MFG_LAST_HOP_FUSED 2

/* Byte offsets of the arrays inside one batch workspace. */
typedef struct {
  int64_t table;                      /* u64[table_cap]                      */
  int64_t globals;                    /* int32[node_cap[L]]                  */
  int64_t sizes;                      /* int64[L+1]: id-map size after hop h */
  int64_t etot;                       /* int64[L]:   edges of hop h          */
  int64_t dst_indptr[SAL_MAX_HOPS];   /* int32[node_cap[h]+1] (hop h)        */
  int64_t src_local[SAL_MAX_HOPS];    /* int32[edge_cap[h]]   (hop h)        */
  int64_t src_glob;                   /* int32[max edge_cap] scratch         */
  int64_t slot;                       /* int32[max edge_cap] scratch         */
  int64_t rank;                       /* int32[max edge_cap] scratch         */
  int64_t scan;                       /* look-back scan workspace            */
  int64_t scan_bytes;
  int64_t total;                      /* total workspace bytes               */
} sal_mfg_layout;

/* ---- library ------------------------------------------------------------ */
int sal_version(void);
const char* sal_last_error(void);
/* number of kernels this library has enqueued in this process (launch audit) */
long long sal_launch_count(void);

/* HopStream.key_prefix (sampler.py:238-247) */
uint64_t sal_hop_key_prefix(uint64_t global_seed, int64_t batch_id, int64_t hop);

/* ---- batch-level driver: multihop_mfg (sampler.py:328-346) -------------- */
/* per_hop is FanoutSpec.per_hop (outermost hop first, sampler.py:70-72). */
int sal_mfg_plan_init(sal_mfg_plan* plan, int32_t num_hops, const int32_t* per_hop,
                      int64_t max_seeds, int64_t num_nodes);
/* as sal_mfg_plan_init with SAL_MFG_* flags */
int sal_mfg_plan_init_ex(sal_mfg_plan* plan, int32_t num_hops, const int32_t* per_hop,
                         int64_t max_seeds, int64_t num_nodes, int32_t flags);
int sal_mfg_layout_init(const sal_mfg_plan* plan, sal_mfg_layout* layout);
/* Seeds -> L hops -> MFG, all on `stream`, no host synchronisation.
 * Outputs land in the workspace at the layout's offsets; `sizes[h]` and
 * `etot[h]` give the dynamic extents. */
int sal_sample_mfg(const sal_graph* g, const sal_mfg_plan* plan, const sal_mfg_layout* layout,
                   void* ws_dev, const int64_t* seeds_base_dev, const sal_batch_desc* desc_dev,
                   uint64_t global_seed, int32_t rng_policy, void* stream);

/* sal_plan_next + sal_sample_mfg in one: *desc_out = desc_all[*cursor] (an empty
 * batch past n_steps), ++*cursor, then the sample of that batch — the cursor step
 * rides in the seed-insertion kernel, so a captured per-step graph starts its
 * batch preparation one launch earlier. */
int sal_sample_mfg_next(const sal_graph* g, const sal_mfg_plan* plan,
                        const sal_mfg_layout* layout, void* ws_dev,
                        const int64_t* seeds_base_dev, const int64_t* desc_all_dev,
                        int64_t n_steps, int64_t* cursor_dev, sal_batch_desc* desc_out_dev,
                        uint64_t global_seed, int32_t rng_policy, void* stream);

/* Fused last hop (plan flag SAL_MFG_LAST_HOP_FUSED), after sal_sample_mfg on the
 * same stream: for each destination d < sizes[L-1] of hop L-1, draw its fanout
 * sample exactly as sal_sample_mfg would (hop_kernel + _sample_positions,
 * _kernels.py:102-185), read the sampled rows of the feature table by global id
 * and write
 *   out[d, 0:cols]                  = mean of the sampled rows (mpnn.py:57-65,
 *                                     fp32 sum in edge order, then * 1/count)
 *   out[d, self_offset:+cols]       = table[globals[d], 0:cols]   (self_offset >= 0;
 *                                     slice_features, prep.py:153-171)
 * converted to out_dtype.  Rows >= sizes[L-1] are not written.  table: fp16,
 * cols * 2 a multiple of 16 and <= 256 bytes; out_dtype SAL_BF16 or SAL_F16;
 * the last hop's fanout <= 32. */
int sal_sample_aggregate(const sal_graph* g, const sal_mfg_plan* plan,
                         const sal_mfg_layout* layout, void* ws_dev,
                         const sal_batch_desc* desc_dev, uint64_t global_seed,
                         int32_t rng_policy, const void* table_dev, int32_t table_dtype,
                         int64_t table_stride, int32_t cols, void* out_dev, int32_t out_dtype,
                         int64_t out_stride, int64_t self_offset, void* stream);

/* ---- hop-level operators (the _kernels.py operator layer) --------------- */
size_t sal_scan_ws_bytes(int64_t max_items);
/* reset every slot of the map to empty (IdMap.__init__, sampler.py:113-129) */
int sal_idmap_reset(const sal_idmap* m, void* stream);
/* rebuild the table from locals 0..n-1 after growth (sampler.py:131-145,
 * rehash_flat _kernels.py:64-73) */
int sal_idmap_rehash(const sal_idmap* m, int64_t n, void* stream);
/* insert_keys (_kernels.py:216-222): get-or-insert keys in order.
 * size_old_dev -> size_new_dev; local_out (nullable) receives each key's local. */
int sal_idmap_insert(const sal_idmap* m, const int64_t* keys_dev, int64_t n,
                     const int64_t* size_old_dev, int64_t* size_new_dev, int64_t* n_dev_scratch,
                     int32_t* scratch_glob, int32_t* scratch_slot, int32_t* scratch_rank,
                     int32_t* local_out, void* scan_ws, void* stream);
/* hop_budget (_kernels.py:42-50) + the destination CSR of hop_kernel:
 * dst_indptr[i] = sum_{j<i} min(deg(globals[j]), fanout); *e_total_dev = total. */
int sal_hop_count(const sal_graph* g, const int32_t* globals_dev, const int64_t* n_dst_dev,
                  int64_t max_dst, int32_t fanout, int32_t* dst_indptr_dev, int64_t* e_total_dev,
                  void* scan_ws, void* stream);
/* sampling half of hop_kernel (_kernels.py:161-183, _sample_positions 102-147):
 * per destination take-all or rejection sampling; writes the sampled global
 * ids and inserts them into the map.  inject_pos_dev (nullable, int64 per
 * edge, same layout as hop_kernel's pos_all, _kernels.py:186-204) replaces
 * the draws with externally supplied slot positions.  draws_out_dev
 * (nullable, int32 per destination) receives the number of draws consumed
 * (CounterRng.counter after sample_neighbors, rng.py:38-51). */
int sal_hop_sample(const sal_graph* g, const sal_idmap* m, const int64_t* n_dst_dev,
                   int64_t max_dst, int32_t fanout, uint64_t key_prefix, int32_t rng_policy,
                   uint64_t global_seed, int64_t batch_id, int32_t hop,
                   const int64_t* inject_pos_dev, const int32_t* dst_indptr_dev,
                   int32_t* src_glob_dev, int32_t* slot_dev, int32_t* draws_out_dev,
                   void* stream);
/* sal_hop_sample with the launch shape pinned, for the f3 design-space sweep
 * (bench.py:142-189 sweep over SamplerVariant): lanes = threads cooperating on
 * one destination (8 / 16 / 32; 0 = smallest group holding the fanout),
 * blocks_per_sm = grid cap per SM (0 = 8).  Output is identical for every
 * setting (the sweep checks digests). */
int sal_hop_sample_tuned(const sal_graph* g, const sal_idmap* m, const int64_t* n_dst_dev,
                         int64_t max_dst, int32_t fanout, uint64_t key_prefix,
                         int32_t rng_policy, uint64_t global_seed, int64_t batch_id, int32_t hop,
                         const int64_t* inject_pos_dev, const int32_t* dst_indptr_dev,
                         int32_t* src_glob_dev, int32_t* slot_dev, int32_t* draws_out_dev,
                         int32_t lanes, int32_t blocks_per_sm, void* stream);
/* relabel half of hop_kernel (_map_get_or_insert, _kernels.py:76-99). */
int sal_hop_relabel(const sal_idmap* m, const int64_t* e_total_dev, int64_t max_edges,
                    const int64_t* size_old_dev, int64_t* size_new_dev,
                    const int32_t* src_glob_dev, const int32_t* slot_dev, int32_t* rank_dev,
                    int32_t* src_local_dev, void* scan_ws, void* stream);

/* ---- slicing (prep.py:153-182) ------------------------------------------ */
/* gather_f16 / gather_f32 (_kernels.py:225-252): out[i,:] = X[ids[i],:]
 * converted to out_dtype.  Row count = *n_dev if n_dev != NULL else n.
 * ids are int32 (id_bytes 4) or int64 (id_bytes 8). */
int sal_gather_rows(const void* x_dev, int64_t x_rows, int32_t cols, int64_t x_stride,
                    int32_t in_dtype, const void* ids_dev, int32_t id_bytes,
                    const int64_t* n_dev, int64_t n, void* out_dev, int64_t out_stride,
                    int32_t out_dtype, void* stream);
/* gather_labels (_kernels.py:255-258): out[j] = y[seeds[j]] for j < n_seeds;
 * rows [n_seeds, max_n) are set to -1 (ignore_index of a padded loss) */
int sal_gather_labels(const int64_t* y_dev, const int64_t* seeds_base_dev,
                      const sal_batch_desc* desc_dev, int64_t max_n, int64_t* out_dev,
                      void* stream);

/* ---- mean aggregation (mpnn.py:57-65 _mean_neighbors) -------------------- */
/* out[d,:] = mean_{e in row d} h[src[e],:]  (0 when the row is empty),
 * fp32 accumulation in edge order; rows [n_dst, n_pad) are zero-filled.
 * n_dst = *n_dst_dev if non-NULL else n_pad. */
int sal_segment_mean_fwd(const int32_t* indptr_dev, const int32_t* src_dev,
                         const int64_t* n_dst_dev, int64_t n_pad, const void* h_dev,
                         int32_t h_dtype, int64_t h_stride, int32_t f, void* out_dev,
                         int32_t out_dtype, int64_t out_stride, void* stream);
/* sal_segment_mean_fwd with flags: SAL_SEG_NO_PAD_FILL leaves rows
 * [*n_dst_dev, n_pad) untouched (a consumer that never reads them, or a buffer
 * that already holds finite values there). */
#define SAL_SEG_NO_PAD_FILL 1
int sal_segment_mean_fwd_ex(const int32_t* indptr_dev, const int32_t* src_dev,
                            const int64_t* n_dst_dev, int64_t n_pad, const void* h_dev,
                            int32_t h_dtype, int64_t h_stride, int32_t f, void* out_dev,
                            int32_t out_dtype, int64_t out_stride, int32_t flags, void* stream);
/* gradient of the above w.r.t. h: g_h[src[e],:] += g_out[d,:] / deg(d).
 * g_h (fp32, n_src rows) must be zeroed by the caller. */
int sal_segment_mean_bwd(const int32_t* indptr_dev, const int32_t* src_dev,
                         const int64_t* n_dst_dev, int64_t n_pad, const void* g_out_dev,
                         int32_t g_dtype, int64_t g_stride, int32_t f, float* g_h_dev,
                         int64_t gh_stride, void* stream);
/* Fused layer-0 aggregation straight from the global feature table (no
 * materialised gather): out[d,:] = mean_e X[globals[src[e]],:]. */
int sal_segment_mean_fwd_global(const int32_t* indptr_dev, const int32_t* src_dev,
                                const int32_t* globals_dev, const int64_t* n_dst_dev,
                                int64_t n_pad, const void* x_dev, int32_t x_dtype,
                                int64_t x_stride, int32_t f, void* out_dev, int32_t out_dtype,
                                int64_t out_stride, void* stream);

/* ---- training-step helpers (PAPER.md:2577-2585 GraphSAGE step) ---------- */
/* Activations use a "cat" layout: layer i's input is [rows, 2f] with h in the
 * right half and mean (first n_pad rows) in the left half, so a SAGEConv is
 * one GEMM [mean | h_dst] @ [W_neigh | W_self]^T. */
/* device epoch cursor: *out = desc_all[*cursor] (or an empty batch past the
 * end), then ++*cursor — one captured graph prepares a new batch per replay */
int sal_plan_next(const int64_t* desc_all_dev, int64_t n_steps, int64_t* cursor_dev,
                  sal_batch_desc* out_dev, void* stream);
/* y = relu(x) * keep / (1-p), keep ~ Philox(seed, element, *salt_dev); mask
 * gets one bit per element (x > 0 && keep), dense over [rows, cols].
 * cols and both row strides (elements) multiples of 8. */
int sal_relu_dropout_fwd(const void* x_dev, int64_t x_stride, void* y_dev, int64_t y_stride,
                         int64_t rows, int32_t cols, int32_t dtype, uint8_t* mask_dev, float p,
                         uint64_t seed, const int64_t* salt_dev, void* stream);
/* dx = dy * bit / (1-p) */
int sal_relu_dropout_bwd(const void* dy_dev, int64_t dy_stride, int32_t dy_dtype,
                         const uint8_t* mask_dev, void* dx_dev, int64_t dx_stride,
                         int32_t dx_dtype, int64_t rows, int32_t cols, float p, void* stream);
/* log_softmax + NLL (labels < 0 ignored, mean over valid rows) fused with its
 * gradient: *loss += mean NLL (caller zeroes it); grad = (softmax-onehot)/count */
int sal_lsm_nll(const void* logits_dev, int64_t ld, int64_t rows, int32_t num_classes,
                int32_t dtype, const int64_t* labels_dev, float* loss_dev, void* grad_dev,
                int64_t ldg, void* stream);
/* sampled-inference scoring (PAPER.md:1428-1439 evaluation): pred[r] =
 * argmax of logits row r (first maximum, NaN as maximum — torch.argmax);
 * counts_dev[0] += #(pred == label), counts_dev[1] += #(label >= 0) over the
 * rows with label >= 0.  pred_dev is nullable.  counts are int64. */
int sal_argmax_correct(const void* logits_dev, int64_t ld, int64_t rows, int32_t num_classes,
                       int32_t dtype, const int64_t* labels_dev, int64_t* counts_dev,
                       int64_t* pred_dev, void* stream);
/* reverse adjacency of an MFG layer: tindptr[n_src_rows+1], tdst[edges] lists
 * for every source row the destinations that sampled it (order within a list
 * is unspecified); tw (nullable) receives each entry's 1/deg(dst) */
size_t sal_transpose_ws_bytes(int64_t n_src_rows);
int sal_transpose_build(const int32_t* indptr_dev, const int32_t* src_dev,
                        const int64_t* n_dst_dev, int64_t n_pad, int64_t n_src_rows,
                        int64_t max_edges, int32_t* tindptr_dev, int32_t* tdst_dev,
                        float* tw_dev, void* ws_dev, int32_t ws_zeroed, void* stream);
/* zero n <= 8 device byte ranges in one kernel (ptrs/bytes are host arrays);
 * replaces a chain of memset nodes inside a captured step */
int sal_zero_spans(void* const* ptrs, const int64_t* bytes, int32_t n, void* stream);
/* input gradient of a SAGEConv layer, gathered per source row s < rows:
 * dz[s] = mask(s) * (dA[s, f:2f] if s < n_pad) + sum_{d in T(s)} dA[d, 0:f]/deg(d),
 * scaled by 1/(1-p) — relu/dropout backward fused, no atomics, no zero fill */
int sal_mean_bwd_t(const void* dA_dev, int64_t lda, int32_t dA_dtype, int32_t f, int64_t n_pad,
                   const int32_t* indptr_dev, const int32_t* tindptr_dev, const int32_t* tdst_dev,
                   const float* tw_dev, int64_t rows, const uint8_t* mask_dev, float p,
                   void* dz_dev, int64_t ldz, int32_t dz_dtype, void* stream);
/* the same over the live rows only: source rows [0, ceil64(*m_dev)), m_dev = the
 * true row count of dz; rows past that 64-row chunk are left unwritten.  For a dz
 * whose only reader is the split-K weight gradient with the same m_dev (layer 0's
 * dz: nothing reads its padding rows, the weight gradient reads whole 64-row chunks) */
int sal_mean_bwd_t_live(const void* dA_dev, int64_t lda, int32_t dA_dtype, int32_t f,
                        int64_t n_pad, const int32_t* indptr_dev, const int32_t* tindptr_dev,
                        const int32_t* tdst_dev, const float* tw_dev, int64_t rows,
                        const int64_t* m_dev, const uint8_t* mask_dev, float p, void* dz_dev,
                        int64_t ldz, int32_t dz_dtype, void* stream);
/* the same input gradient (bit-identical to sal_mean_bwd_t) in two disjoint passes of
 * one launch: destination-major over the forward adjacency (indptr/src, n_dst_dev
 * destinations) for the rows with exactly one in-edge and no self term
 * (s >= n_pad), reading each dA[d] once for all its sources; source-major over
 * the reverse adjacency for the rest.  m_dev != NULL: live rows only, as
 * sal_mean_bwd_t_live. */
int sal_mean_bwd(const void* dA_dev, int64_t lda, int32_t dA_dtype, int32_t f, int64_t n_pad,
                 const int64_t* n_dst_dev, const int32_t* indptr_dev, const int32_t* src_dev,
                 const int32_t* tindptr_dev, const int32_t* tdst_dev, const float* tw_dev,
                 const int32_t* cplx_dev, const int32_t* n_cplx_dev, int64_t rows,
                 const int64_t* m_dev, const uint8_t* mask_dev, float p, void* dz_dev,
                 int64_t ldz, int32_t dz_dtype, void* stream);
/* byte offsets, inside a sal_transpose_build workspace, of the list (int32) of the rows
 * sal_mean_bwd handles source-major (self term, or not exactly one in-edge; any order)
 * and of its length (int32); sal_transpose_build fills both (pass them as cplx_dev /
 * n_cplx_dev, or NULL to scan every row) */
int sal_transpose_complex_list(int64_t n_src_rows, int64_t* list_offset, int64_t* count_offset);
/* Adam (torch.optim.Adam, no weight decay) on flat fp32 params; step count
 * t = *t_dev + 1; refreshes the optional bf16 shadow copy; zero_grad != 0
 * leaves grad zeroed (the next backward accumulates without a memset) */
int sal_adam_step(float* param_dev, float* grad_dev, float* m_dev, float* v_dev,
                  void* shadow_bf16_dev, int64_t n, float lr, float beta1, float beta2, float eps,
                  const int64_t* t_dev, int32_t zero_grad, void* stream);
/* per-step bookkeeping: *last = *loss; log[*step] = *loss; *loss = 0 (ready
 * for the next step's accumulation); ++*step; ++*adam_t */
/* sal_adam_step (vectorised: n % 4 == 0, 16-byte aligned) and sal_step_tail in one
 * launch: the last block to finish does the bookkeeping (ticket_dev: one zeroed
 * uint32 the kernel leaves zeroed) */
int sal_adam_step_tail(float* param_dev, float* grad_dev, float* m_dev, float* v_dev,
                       void* shadow_bf16_dev, int64_t n, float lr, float beta1, float beta2,
                       float eps, int64_t* t_dev, int32_t zero_grad, float* loss_dev,
                       float* last_dev, float* log_dev, int64_t log_len, int64_t* step_dev,
                       unsigned int* ticket_dev, void* stream);
int sal_step_tail(float* loss_dev, float* last_dev, float* log_dev, int64_t log_len,
                  int64_t* step_dev, int64_t* adam_t_dev, void* stream);

/* ---- tcgen05 GEMMs of the layer-0 SAGEConv (sm_100a tensor cores) -------- */
/* Y = act(A[M,K] @ W[N,K]^T), bf16 in, fp32 TMEM accumulate, bf16 out; with
 * relu_dropout != 0 the epilogue applies ReLU + dropout (same stream as
 * sal_relu_dropout_fwd) and writes the bit mask [M, N/8].  N = 256 and
 * K = 256 (layer 0: [mean | h] of 128-d features) or K = 512 (a hidden layer
 * of width 256: two 128-column blocks per row tile).
 * m_dev (nullable): true row count on the device; 128-row tiles past it are
 * zero-filled (Y and mask) without loading A or running the MMA, or left
 * unwritten when relu_dropout has bit 1 set (a caller that never reads the
 * padding rows, e.g. inference). */
int sal_tc_sage_fwd(const void* A_dev, int64_t lda, int64_t M, const int64_t* m_dev,
                    const void* W_dev, int32_t N, int32_t K, void* Y_dev, int64_t ldy,
                    uint8_t* mask_dev, float p, uint64_t seed, const int64_t* salt_dev,
                    int32_t relu_dropout, void* stream);
/* dW[N,K] (fp32, row stride lddw) = dz[M,N]^T @ A[M,K]; zeroes dW first
 * unless `accumulate` (then dW += ...: the caller guarantees dW was zero).
 * m_dev (nullable): true row count on the device (rows past it are skipped;
 * the caller guarantees their contributions are zero).
 * 128 x 128 output tiles x split-K over M (about one CTA per SM), partials
 * added with fp32 vector atomics.  K multiple of 128, N of 16 (the output
 * layer's c_pad rows: dz columns past N read as zero, dW rows past N untouched). */
int sal_tc_sage_wgrad(const void* dz_dev, int64_t ldz, const void* A_dev, int64_t lda, int64_t M,
                      const int64_t* m_dev, int32_t N, int32_t K, float* dW_dev, int64_t lddw,
                      int32_t accumulate, void* stream);
/* C[M,N] = A[M,K] @ B[K,N] (bf16 in, fp32 TMEM accumulate, bf16 out), both
 * operands row-major: the input gradient dA = dz @ [W_neigh | W_self] of a
 * SAGEConv layer (mpnn.py:82's contraction, backward).  K multiple of 16
 * (columns past K read as zero), N multiple of 64.  m_dev (nullable): true
 * row count on the device; 128-row tiles past it are skipped, or zero-filled
 * when pad_fill != 0.  Replaces torch.mm (cuBLAS) in the step. */
int sal_tc_gemm_nn(const void* A_dev, int64_t lda, int64_t M, const int64_t* m_dev, int32_t K,
                   const void* B_dev, int64_t ldb, int32_t N, void* C_dev, int64_t ldc,
                   int32_t pad_fill, void* stream);
/* the output layer in one tcgen05 kernel (training): logits = A[M,K] @
 * W[c_pad,K]^T (never written), *loss += mean NLL over labels >= 0 (count over
 * labels[0:min(M, n_labels)]), dlogits[M, ldd] = (softmax - onehot) / count
 * (bf16, columns >= num_classes and rows of unlabelled or padding rows zero),
 * dA[M,K] = dlogits @ W (bf16; rows of tiles past *m_dev zero) and
 * dW[c_pad,K] += dlogits^T @ A (fp32 atomics; the caller zeroes dW).  Replaces
 * cuBLAS + sal_lsm_nll + cuBLAS + cuBLAS (mpnn.py:82 and the log_softmax/NLL of
 * PAPER.md:2577-2585).  One cluster of K/64 CTAs per 128-row tile: split-K
 * logits partials summed through an L2-resident workspace of
 * sal_tc_sage_head_ws_bytes() bytes, dA and dW from the same A / W tiles.
 * K = 128, 256 or 512; c_pad multiple of 16, <= 192. */
size_t sal_tc_sage_head_ws_bytes(int64_t M, int32_t K, int32_t c_pad);
int sal_tc_sage_head(const void* A_dev, int64_t lda, int64_t M, const int64_t* m_dev, int32_t K,
                     const void* W_dev, int64_t ldw, int32_t c_pad, int32_t num_classes,
                     const int64_t* labels_dev, int64_t n_labels, float* loss_dev,
                     void* dlogits_dev, int64_t ldd, void* dA_dev, int64_t ldda, float* dW_dev,
                     int64_t lddw, void* ws_dev, size_t ws_bytes, void* stream);
/* sampled-inference scoring with the same kernel: logits as above, epilogue =
 * sal_argmax_correct's (counts_dev[0] += correct, counts_dev[1] += labelled) */
int sal_tc_sage_logits_argmax(const void* A_dev, int64_t lda, int64_t M, const int64_t* m_dev,
                              int32_t K, const void* W_dev, int64_t ldw, int32_t c_pad,
                              int32_t num_classes, const int64_t* labels_dev, int64_t n_labels,
                              int64_t* counts_dev, void* ws_dev, size_t ws_bytes, void* stream);

/* ---- on-device synthetic data (graph.py:252-298 laws) ---- */
/* Pareto degrees of the synth_graph law (graph.py:262-271): degs[v] =
 * rint(scale * (1-u_v)^(-1/a)) clipped to [0, n-1], u_v counter-based
 * (Philox on v); a = exponent - 1, scale = avg_degree (a-1)/a */
int sal_gen_degrees(int64_t n, uint64_t seed, double scale, double a, int64_t* degs_dev,
                    void* stream);
/* owner[s] = v for every slot s in [indptr[v], indptr[v+1]) */
int sal_gen_owner(const int64_t* indptr_dev, int64_t n, int32_t* owner_dev, void* stream);
/* configuration-model pairing: indices[s] = owner[partner(s)], partner a
 * seeded pseudo-random perfect matching of the n_stubs (even) slots */
int sal_gen_pairing(const int32_t* owner_dev, int64_t n_stubs, uint64_t seed,
                    int32_t* indices_dev, void* stream);
/* uniform [-1,1) features rounded to fp16, row stride `stride` elements */
int sal_gen_features_uniform(int64_t n, int32_t f, int64_t stride, uint64_t seed, void* out_dev,
                             void* stream);
/* i.i.d. uniform class labels (graph.py:295-298 law) */
int sal_gen_labels_uniform(int64_t n, int32_t num_classes, uint64_t seed, int64_t* out_dev,
                           void* stream);

/* ---- f2: binary files straight into HBM (graph.py:194-249) -------------- *
 * MFGC: "MFGC" u32 version=1, u64 num_nodes, u64 num_edges, u64 indptr[n+1],
 *       u32 indices[E]                       (save_csr / load_csr, :194-214)
 * FEAT: "FEAT" u32 version, u64 rows, u32 cols, u8 dtype (1 = f16, else f32),
 *       3 pad bytes, row-major payload        (save_features / load_features, :217-232)
 * LABL: "LABL" u32 version, u64 rows, u32 num_classes, u32 values[rows]
 *                                            (save_labels / load_labels, :235-249)
 * Header errors mirror graph.py:23-36 and _check_header/_read_exact (:176-191):
 * SAL_EBADMAGIC (BadMagicError), SAL_EVERSION (VersionMismatchError),
 * SAL_ETRUNC (TruncatedFileError, message "truncated file while reading <what>"
 * with the reference's field names), SAL_EIO (OSError). */
#define SAL_EBADMAGIC (-10)
#define SAL_EVERSION (-11)
#define SAL_ETRUNC (-12)
#define SAL_EIO (-13)

#define SAL_FILE_CSR 1
#define SAL_FILE_FEAT 2
#define SAL_FILE_LABL 3

typedef struct {
  int32_t kind;            /* SAL_FILE_*                                   */
  uint32_t version;
  uint8_t magic[4];        /* as read (for the BadMagicError message)      */
  int64_t rows;            /* CSR: num_nodes; FEAT / LABL: rows            */
  int64_t cols;            /* CSR: num_edges; FEAT: cols; LABL: classes    */
  int32_t dtype;           /* FEAT: SAL_F16 / SAL_F32 (code 1 = f16)       */
  int32_t elem_bytes;      /* FEAT: 2 / 4; LABL / CSR indices: 4           */
  int64_t payload_offset;  /* first byte after the fixed header            */
  int64_t file_bytes;
} sal_file_header;

/* Parse + size-check the header of `path` as `kind` (no device work). */
int sal_file_header_read(const char* path, int32_t kind, sal_file_header* out);
/* Stream a file's payload into HBM through a caller-provided pinned staging
 * buffer (split in two halves: read of chunk k+1 by `threads` host threads
 * overlaps the H2D copy of chunk k on `stream`).  Returns when the last copy
 * is enqueued and the staging buffer is free again (synchronises on its own
 * events only).
 *   CSR : indptr_dev int64[n+1] (u64 bytes), indices_dev int32[E] (u32 bytes)
 *   FEAT: rows into out_dev with row pitch out_stride_bytes (>= cols*elem);
 *         a padded pitch goes through scratch_dev (>= pinned_bytes/2 bytes,
 *         nullable when the pitch equals the row) and a re-pitch kernel
 *   LABL: u32 chunks into scratch_dev (>= pinned_bytes/2 bytes), widened
 *         to int64 into out_dev by a kernel                                  */
int sal_load_csr(const char* path, const sal_file_header* h, int64_t* indptr_dev,
                 int32_t* indices_dev, void* pinned, int64_t pinned_bytes, int32_t threads,
                 void* stream);
int sal_load_features(const char* path, const sal_file_header* h, void* out_dev,
                      int64_t out_stride_bytes, void* scratch_dev, void* pinned,
                      int64_t pinned_bytes, int32_t threads, void* stream);
int sal_load_labels(const char* path, const sal_file_header* h, int64_t* out_dev,
                    void* scratch_dev, void* pinned, int64_t pinned_bytes, int32_t threads,
                    void* stream);
/* CsrGraph.validate (graph.py:58-65) on device: flags_dev int32[3] |= (bad
 * endpoints, decreasing indptr, neighbour id out of range); caller zeroes. */
int sal_validate_csr(const int64_t* indptr_dev, const int32_t* indices_dev, int64_t n,
                     int64_t e, int32_t* flags_dev, void* stream);
/* LabelVector check (graph.py:96-100): flags_dev[0] |= any value outside
 * [0, num_classes). */
int sal_validate_labels(const int64_t* y_dev, int64_t n, int64_t num_classes, int32_t* flags_dev,
                        void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SALIENT_B200_H */
