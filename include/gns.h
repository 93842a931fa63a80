/*
 * gns.h — C ABI of the B200-native Global Neighbor Sampling hot path.
 *
 * libgns.so (paper_2106_06150_b200/libgns.so, sm_100a) exports exactly these
 * symbols.  All array arguments are DEVICE pointers unless stated; every call
 * is asynchronous on `stream` (a cudaStream_t passed as void*) and writes only
 * into caller-owned buffers.  Functions that need scratch take a caller-given
 * workspace whose size is queried first with the matching *_workspace_size().
 * Counts that are produced on the device (cache size, edges, unique sources)
 * are returned through device pointers so a whole mini-batch can be captured
 * in a CUDA graph; the host reads them once per batch.
 *
 * Node ids are int32 (ogbn-papers100M has 111M < 2^31 nodes), CSR offsets are
 * int64 (3.2B directed entries > 2^31), importance weights are float64 exactly
 * as the reference computes them.
 *
 * Each entry point names the reference function it replaces (paths relative
 * to /root/reference/pkg/src/gnsbench).  The reference is a Python package, so
 * "replaces" means: the Python facade paper_2106_06150_b200/ keeps the
 * reference signature and calls this function where the reference ran numpy.
 *
 * Status codes: GNS_OK, or an error whose message gns_last_error() returns.
 * The facade maps GNS_EINVAL / GNS_EZEROPROB to ValueError (sampling.py:161,
 * 202-207, 255-256; cache.py:34-37,49,57), GNS_ECAPACITY to InvariantError
 * (graph.py:48) and GNS_ECUDA to RuntimeError.
 */
#ifndef GNS_B200_H_
#define GNS_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define GNS_API __attribute__((visibility("default")))
#else
#define GNS_API
#endif

#define GNS_OK 0
#define GNS_EINVAL 1
#define GNS_ECAPACITY 2
#define GNS_ECUDA 3
#define GNS_EZEROPROB 4

/* Device-side error flags raised by kernels (bit set in a block's counts[GNS_CNT_ERR]). */
#define GNS_ERRBIT_ZEROPROB 1u  /* cached draw with inclusion 0 (sampling.py:255-256) */
#define GNS_ERRBIT_CAPACITY 2u  /* selection buffer could not converge */
#define GNS_ERRBIT_ZEROQ 4u     /* gns-exact edge with zero estimated inclusion (sampling.py:248-249) */

/* Layout of the per-block device counter array (int32[8]). */
#define GNS_CNT_DST 0      /* number of dst rows (seeds)                    */
#define GNS_CNT_EDGES 1    /* sampled edges (cached + fill)                 */
#define GNS_CNT_CACHED 2   /* cached-phase edges                            */
#define GNS_CNT_SRC 3      /* unique src nodes after relabel                */
#define GNS_CNT_HUBS 4     /* (row, phase) items for the CTA-per-item sampler */
#define GNS_CNT_ERR 5      /* GNS_ERRBIT_* flags                             */
#define GNS_CNT_WARPROWS 6 /* (row, phase) items for the warp-per-item sampler  */
#define GNS_CNT_THREADROWS 7 /* (row, phase) items for the thread-per-item sorting-network sampler */
#define GNS_CNT_STREAMROWS 8 /* (row, phase) items for the thread-per-item streaming top-k sampler */
#define GNS_CNT_TSEGS 9    /* segments of the transpose's long rows (gns_block_transpose) */
#define GNS_CNT_N 16

/* CSR graph (graph.py:52-104): indptr int64[N+1], indices int32[E]. */
typedef struct gns_graph {
  int64_t num_nodes;
  int64_t num_edges;
  const int64_t* indptr;
  const int32_t* indices;
} gns_graph_t;

/* Cache state (cache.py:130-157): cached CSR N(v)∩C, membership bitmap over
 * node ids (bit v of word v>>5), per-node inclusion probability (Eq. 9). */
typedef struct gns_cache {
  const int64_t* cached_indptr;   /* int64[N+1] */
  const int32_t* cached_indices;  /* int32[nnz_C] */
  const uint32_t* mask_bits;      /* uint32[ceil(N/32)] */
  const double* inclusion;        /* float64[N] */
  const int32_t* cached_pos;      /* int32[nnz_C]: position in the full row (gns-exact), may be NULL */
} gns_cache_t;

/* Philox4x32-10 key (oracle/philox.py): key = (seed, epoch), counter =
 * (pos>>1, node, tag<<24|layer<<16|phase<<8, batch). */
typedef struct gns_rng {
  uint32_t seed;
  uint32_t epoch;
  uint32_t batch;
  uint32_t layer;
} gns_rng_t;

/* Per-batch parameters kept in DEVICE memory so a captured CUDA graph can be
 * replayed for every batch: the Philox key and the batch's slice of the
 * epoch permutation (pool.py:60-70). */
typedef struct gns_step {
  uint32_t seed;
  uint32_t epoch;
  uint32_t batch;
  uint32_t pad;
  int64_t begin;
  int64_t count;
} gns_step_t;

/* One sampled layer (sampling.py:32-60 LayerBlock) in capacity-sized buffers. */
typedef struct gns_block {
  /* per dst row, capacity max_dst (+1 for row_scan) */
  uint64_t* row_scan;      /* exclusive scan, packed (cached_prefix<<32 | fill_prefix); [n] = totals */
  int32_t* dst_degree;     /* deg(dst) (sampling.py:149)                              */
  int32_t* self_pos;       /* searchsorted(src_nodes, dst_nodes) (model.py:137)       */
  int32_t* hub_rows;       /* (row<<1|phase) work lists, capacity 6*max_dst: sorting-network
                              thread tier in [0, 2*max_dst), streaming thread tier in [2*max_dst,
                              4*max_dst), warp tier from 4*max_dst up, CTA tier from 6*max_dst-1 down */
  /* per edge, capacity max_edges; order = cached edges then fill edges, each by (dst row, key) */
  int32_t* edge_node;      /* global id of the sampled neighbour                       */
  int32_t* edge_src;       /* relabelled: index into src_nodes (sampling.py:145)       */
  int32_t* edge_dst;       /* dst row (sampling.py:146)                                */
  double* edge_weight;     /* importance weight (sampling.py:168,252-258)              */
  uint8_t* edge_cached;    /* cached-phase flag (sampling.py:263)                      */
  /* src set, capacity max_src */
  int32_t* src_nodes;      /* sorted unique seeds ∪ neighbours (sampling.py:141)        */
  int32_t* counts;         /* int32[GNS_CNT_N] device counters                           */
} gns_block_t;

/* ---- library ------------------------------------------------------------ */
GNS_API const char* gns_last_error(void);
GNS_API int gns_version(void);

/* Record a CUDA event on a stream with cudaEventRecordExternal, so an event
 * recorded while a stream is being captured into a CUDA graph fires (and can
 * be timed / waited on) at every replay.  Used for in-graph kernel timing. */
GNS_API int gns_record_event_external(void* event, void* stream);

/* Kernel copy of `bytes` between device-addressable buffers, either of which
 * may be mapped pinned host memory (UVA): used inside captured step graphs
 * for the per-step host inputs / outputs instead of memcpy nodes.  Source
 * loads are volatile (fresh on every replay).  4-byte aligned pointers. */
GNS_API int gns_copy_mapped(void* dst, const void* src, int64_t bytes, void* stream);

/* Sticky device error word: ORs counts[l * stride + GNS_CNT_ERR] of `layers`
 * per-layer counter rows into *sticky (one thread, graph-capturable).  The
 * per-batch counters are reset by every gns_sample_layer call, so an engine
 * that reuses sampler slots accumulates each batch's error bits here and
 * reads the word once per epoch (the reference raises at the failing call,
 * sampling.py:248-249,255-256; the façade raises the same exceptions). */
GNS_API int gns_errors_accumulate(const int32_t* counts, int32_t layers, int32_t stride, int32_t* sticky,
                                  void* stream);

/* CUDA-graph plumbing for the whole-step engine (engine.py).  `graph` is a
 * captured cudaGraph_t (torch.cuda.CUDAGraph(keep_graph=True).raw_cuda_graph()).
 * gns_graph_instantiate instantiates it, optionally honouring the per-kernel
 * priorities captured from the streams (cudaGraphInstantiateFlagUseNodePriority)
 * so the sampling branch of a step is scheduled ahead of the training branch;
 * gns_graph_launch replays it on `stream`.  gns_graph_kernel_priorities fills
 * out_hist[|priority|] with the number of kernel nodes at each priority. */
GNS_API int gns_graph_instantiate(void* graph, int32_t use_node_priority, void** out_exec);
GNS_API int gns_graph_launch(void* exec, void* stream);
GNS_API int gns_graph_exec_destroy(void* exec);
GNS_API int gns_graph_kernel_priorities(void* graph, int32_t* out_hist, int32_t nbins);

/* Size-switched graph regions: called while `stream` is being captured,
 * gns_graph_switch_begin appends a kernel that reads the device row count
 * *n_dev and a SWITCH conditional node with `nbodies` empty body graphs
 * (out_bodies[k]); at every replay body k = min(ceil(n / chunk), nbodies-1)
 * runs.  The caller records body k — typically the dense op over the first
 * k*chunk rows — by capturing onto another stream between
 * gns_graph_body_capture_begin(aux, out_bodies[k]) and
 * gns_graph_body_capture_end(aux).  Lets capacity-sized GEMMs run on the
 * rows the batch actually has. */
GNS_API int gns_graph_switch_begin(void* stream, const int32_t* n_dev, int64_t chunk, int32_t nbodies,
                                   void** out_bodies);
/* Several SWITCH nodes over the same device count with one selector kernel:
 * gns_graph_switch_handles creates `count` (<= 4) conditional handles in the
 * graph being captured on `stream` and appends ONE kernel setting handle i to
 * min(ceil(n / chunk), nbodies[i] - 1); gns_graph_switch_node then appends
 * the SWITCH node of a handle (no selector kernel of its own) wherever the
 * capture has reached. */
GNS_API int gns_graph_switch_handles(void* stream, const int32_t* n_dev, int64_t chunk, int32_t count,
                                     const int32_t* nbodies, uint64_t* handles);
GNS_API int gns_graph_switch_node(void* stream, uint64_t handle, int32_t nbodies, void** out_bodies);
GNS_API int gns_graph_body_capture_begin(void* stream, void* body);
GNS_API int gns_graph_body_capture_end(void* stream);

/* Developer knobs for A/B measurements of kernel variants (defaults = the
 * measured best; every setting gives identical results):
 *   "spmm_narrow"  1: shuffle-ranked forward SpMM for float32 rows of <= 128
 *                  floats, 0: the generic shared-memory kernel;
 *   "spmm_wide"    1: shuffle-ranked hidden-layer forward (rows of <= 512
 *                  floats), 0: generic;
 *   "stream_len"   selection tier routing: items with take <= 8 scanning <=
 *                  this many positions go to the streaming thread tier (32);
 *   "thread_len"   other items scanning <= this many positions go to the
 *                  sorting-network thread tier (0 = off);
 *   "sampler_ctas" cap grid-stride sampler grids at this many CTAs per SM
 *                  (0 = no cap).
 * Not used on the product path. */
GNS_API int gns_tune(const char* name, int32_t value);

/* ---- cache engine (cache.py) ------------------------------------------- */

/* degree_probs (cache.py:53-58): out[i] = deg(i) / E in float64. */
GNS_API int gns_degree_probs(const gns_graph_t* g, double* out_probs, void* stream);

/* random_walk_probs (cache.py:61-84): p0 = 1/|train| on train_ids, then for
 * l < num_layers: p <- d*(A p) + p with d_i = min(fanouts_host[l], deg_i) /
 * max(deg_i, 1) (A p summed per row in CSR order: bit-identical to scipy),
 * then p / sum(p) with a fixed-order strided sum.  fanouts_host is a HOST
 * array of num_layers ints. */
GNS_API size_t gns_random_walk_workspace_size(int64_t num_nodes);
GNS_API int gns_random_walk_probs(const gns_graph_t* g, const int32_t* train_ids, int64_t n_train,
                                  const int32_t* fanouts_host, int32_t num_layers, double* out_probs,
                                  void* ws, size_t ws_bytes, void* stream);

/* sample_cache (cache.py:87-103) + NodeSet.from_ids (graph.py:118-125):
 * exponential race keys -log(1-U)/p over p>0, smallest min(cache_size,
 * |support|) by (key, id) via radix select, emitted as sorted ids + bitmap.
 * tag = Philox stream tag: 33 for the epoch cache (pool.py:32), 21 for the
 * gns-exact resamples (sampling.py:29).
 * out_ids int32[cache_size]; out_mask_bits uint32[ceil(N/32)];
 * out_counts int64[2] = {|C|, |support|} (device). */
GNS_API size_t gns_cache_draw_workspace_size(int64_t num_nodes);
GNS_API int gns_cache_draw(const double* probs, int64_t num_nodes, int64_t cache_size,
                   uint32_t seed, uint32_t epoch, uint32_t tag, int32_t* out_ids,
                   uint32_t* out_mask_bits, int64_t* out_counts, void* ws,
                   size_t ws_bytes, void* stream);

/* inclusion_prob (cache.py:106-117) and the forced-case pin of build_cache
 * (cache.py:174-177).  cache_size_dev / support_dev (device int64, may be
 * NULL) override cache_size and enable the pin when |C| >= |support|. */
GNS_API int gns_inclusion(const double* probs, int64_t n, int64_t cache_size,
                  const int64_t* cache_size_dev, const int64_t* support_dev,
                  double* out, void* stream);

/* Induced cached-neighbour CSR (cache.py:185-197) by filtering the full CSR
 * with the cache bitmap (rows stay ascending).  Two phases sharing one
 * workspace (it holds one keep bit per CSR entry between them): count (writes
 * out_c_indptr and *out_nnz_dev), then fill (needs c_indices capacity >= nnz;
 * out_c_pos, optional — gns-exact only — receives each entry's position in
 * the full row). */
GNS_API size_t gns_cached_csr_workspace_size(int64_t num_nodes, int64_t num_edges);
GNS_API int gns_cached_csr_count(const gns_graph_t* g, const uint32_t* mask_bits,
                         int64_t* out_c_indptr, int64_t* out_nnz_dev, void* ws,
                         size_t ws_bytes, void* stream);
GNS_API int gns_cached_csr_fill(const gns_graph_t* g, const uint32_t* mask_bits,
                        const int64_t* c_indptr, int32_t* out_c_indices,
                        int32_t* out_c_pos, void* ws, size_t ws_bytes, void* stream);

/* estimate_edge_inclusion (sampling.py:269-296): CSR-aligned float64 table
 * q[e] = mean over `resamples` Philox cache draws (key (seed, r), tag 21) of
 * the edge's selection probability min(k,nc)/nc if its neighbour is cached,
 * else fill/rest (0 when cache_only). */
GNS_API size_t gns_edge_inclusion_workspace_size(int64_t num_nodes, int64_t cache_size);
GNS_API int gns_estimate_edge_inclusion(const gns_graph_t* g, const double* probs,
                                        int64_t cache_size, int32_t k, int32_t cache_only,
                                        int32_t resamples, uint32_t seed, double* out_q, void* ws,
                                        size_t ws_bytes, void* stream);

/* ---- sampler (sampling.py) --------------------------------------------- */

/* step_dev (device, may be NULL) overrides rng->seed/epoch/batch.
 * exact_q (device float64[E], may be NULL): gns-exact weights 1/q[position]
 * (sampling.py:238-250) instead of gns-paper; needs cache->cached_pos.
 * sample_neighbors_gns (sampling.py:189-266, policy gns-paper) when cache !=
 * NULL, sample_neighbors_uniform (sampling.py:155-170) when cache == NULL.
 * seeds: sorted unique int32 (count in *n_seeds_dev, <= max_dst).  Writes
 * row_scan, dst_degree, edge_node/edge_dst/edge_weight/edge_cached, and the
 * assembled block (_assemble, sampling.py:139-152): src_nodes, edge_src,
 * self_pos, plus counts DST/EDGES/CACHED/SRC/HUBS/ERR.  Edge capacity must be
 * >= max_dst * k.  The workspace (gns_sample_workspace_size) holds the
 * two-level dedup bitmap: zero it once before first use; every call leaves it
 * zero. */
GNS_API size_t gns_sample_workspace_size(int64_t num_nodes, int64_t max_dst);
GNS_API int gns_sample_layer(const gns_graph_t* g, const gns_cache_t* cache,
                     const int32_t* seeds, const int32_t* n_seeds_dev,
                     int64_t max_dst, int32_t k, int32_t cache_only, const double* exact_q,
                     const gns_rng_t* rng, const gns_step_t* step_dev,
                     gns_block_t* block, void* ws, size_t ws_bytes, void* stream);

/* Standalone _assemble (sampling.py:139-152) for an externally produced edge
 * list: src_nodes = sorted unique(seeds ∪ edge_node), edge_src = rank of
 * edge_node, self_pos = rank of each seed.  Two-level bitmap dedup over node
 * ids; the workspace must be zero on first use and is left zero.  Writes
 * counts[GNS_CNT_SRC].  (gns_sample_layer already does this internally.) */
GNS_API size_t gns_relabel_workspace_size(int64_t num_nodes);
GNS_API int gns_relabel(int64_t num_nodes, const int32_t* seeds, const int32_t* n_seeds_dev,
                int64_t max_dst, gns_block_t* block, int64_t max_edges,
                void* ws, size_t ws_bytes, void* stream);

/* np.unique of an id list (sampling.py:208,312): sorted unique ids of
 * ids[0..n) (n = *n_dev if n_dev else n_host) into out, count into *out_n_dev. */
GNS_API int gns_unique_sorted(int64_t num_nodes, const int32_t* ids, const int32_t* n_dev,
                      int64_t n_host, int32_t* out, int32_t* out_n_dev, void* ws,
                      size_t ws_bytes, void* stream);

/* ---- data loader (pool.py) --------------------------------------------- */

/* epoch_targets (pool.py:60-66): out[j] = train_ids[perm(begin + j)] for
 * j < count, perm = 4-round Feistel bijection keyed on (seed, epoch). */
GNS_API int gns_epoch_targets(const int32_t* train_ids, int64_t n_train, uint32_t seed,
                      uint32_t epoch, int64_t begin, int64_t count, int32_t* out,
                      void* stream);

/* Same, with (seed, epoch, begin, count) read from a device gns_step_t; the
 * batch size actually written (min(count, n_train - begin)) goes to *out_n_dev. */
GNS_API int gns_epoch_targets_dev(const int32_t* train_ids, int64_t n_train,
                                  const gns_step_t* step_dev, int64_t max_count, int32_t* out,
                                  int32_t* out_n_dev, void* stream);

/* gns_epoch_targets_dev followed by np.unique (sampling.py:312) in one
 * single-CTA kernel, for batches of <= 1024 targets: out_sorted receives the
 * sorted distinct targets, *out_n_dev their number. */
GNS_API int gns_batch_targets_sorted(const int32_t* train_ids, int64_t n_train,
                                     const gns_step_t* step_dev, int64_t max_count, int32_t* out_sorted,
                                     int32_t* out_n_dev, void* stream);

/* Same from a precomputed epoch permutation (epoch_perm[j] = the j-th target
 * of the epoch, gns_epoch_targets over the whole epoch): the batch is the
 * slice [begin, begin + count), sorted and deduplicated — no per-batch
 * Feistel evaluation inside the step.  step_src may be pinned (mapped) host
 * memory written between graph replays; when step_dev_out is non-NULL the
 * kernel reads step_src once, uncached, and stores it there for the step's
 * later kernels (no separate host->device copy). */
GNS_API int gns_batch_slice_sorted(const int32_t* epoch_perm, int64_t n_train, const gns_step_t* step_src,
                                   gns_step_t* step_dev_out, int64_t max_count, int32_t* out_sorted,
                                   int32_t* out_n_dev, void* stream);

/* ---- model side (model.py) --------------------------------------------- */

/* features[input_nodes] (model.py:146): out[i,:] = table[rows[i],:], D
 * columns.  dtype_in/out: 0 = float32, 1 = float64 (float32 -> float64 for
 * the reference-parity mode).  ld_* are row strides in elements.  float32
 * rows of D <= 64 go through the TMA (tile::gather4 loads + bulk stores);
 * wider rows through the register-staged kernel (gns_tune "gather_tma"). */
GNS_API int gns_gather_rows(const void* table, int64_t ld_in, int32_t dtype_in,
                    const int32_t* rows, const int32_t* n_rows_dev, int64_t max_rows,
                    int32_t dim, void* out, int64_t ld_out, int32_t dtype_out,
                    void* stream);

/* Mixed CPU-GPU placement (paper §3.1): cached rows from an HBM cache table
 * (slot = rank of the node in the cache bitmap), the rest from a pinned host
 * table through UVA. */
GNS_API int gns_gather_rows_mixed(const float* host_table, const float* cache_table,
                          const uint32_t* mask_bits, const int32_t* mask_word_rank,
                          int64_t ld, const int32_t* rows, const int32_t* n_rows_dev,
                          int64_t max_rows, int32_t dim, float* out, int64_t ld_out,
                          void* stream);

/* Refresh of the HBM cache table from the pinned host table (paper §3.1;
 * modeled by metrics.py:83-86): cache_table[j,:] = host_table[ids[j],:]. */
GNS_API int gns_cache_refresh_rows(const float* host_table, int64_t ld, const int32_t* ids,
                           const int64_t* n_dev, int64_t max_rows, int32_t dim,
                           float* cache_table, void* stream);

/* Per-word exclusive popcount rank of a bitmap (slot lookup for the cache). */
GNS_API int gns_bitmap_rank(const uint32_t* bits, int64_t nwords, int32_t* out_rank,
                    void* ws, size_t ws_bytes, void* stream);

/* Weighted mean aggregation + self concat (model.py:131-138,153-154):
 * cat[r, 0:D]  = x(h[self_pos[r], :])
 * cat[r, D:2D] = (sum_e w_e * x(h[edge_src_e, :])) / max(deg(r), 1)
 * accumulated in ascending edge_src order (scipy CSR order); x = relu when
 * flags & GNS_SPMM_RELU_INPUT (h holds the previous layer's pre-activations,
 * model.py:156), identity otherwise.  Rows [n_dst, pad_rows) of cat are
 * zero-filled.  dtype 0 = float32 (production), 1 = float64 bit-exact vs
 * scipy (no FMA). */
#define GNS_SPMM_RELU_INPUT 1
GNS_API int gns_spmm_fwd(int32_t dtype, const void* h, int64_t ld_h, int32_t dim, int32_t flags,
                         const gns_block_t* block, int64_t max_dst, int64_t pad_rows, void* cat,
                         int64_t ld_cat, void* stream);

/* The input layer's gns_spmm_fwd fused with the feature gather (model.py:146
 * + 153): h rows are read straight from the float32 node feature table by
 * global node id — block->edge_node for the neighbours, dst_ids[r] (the
 * block's dst node ids) for the self half — instead of from a materialised
 * features[input_nodes].  Output identical to gns_gather_rows followed by
 * gns_spmm_fwd(dtype 0, flags 0).  pad_chunk > 0 zero-fills rows [n, pad_rows)
 * only up to the next multiple of pad_chunk (what a size-switched GEMM over
 * the first ceil(n / pad_chunk) * pad_chunk rows reads).  max_row_edges: an
 * upper bound on a row's edges (the layer's fanout; 0 = unknown), a hint for
 * kernel selection (a cp.async shared-memory-staged variant for D = 128,
 * fanout <= 5 measured 121 us vs 90 us for the register-staged kernel on the
 * papers100M batch and is not used). */
GNS_API int gns_spmm_fwd_gather(const float* table, int64_t ld_table, int32_t dim,
                                const gns_block_t* block, const int32_t* dst_ids, int64_t max_dst,
                                int64_t pad_rows, int64_t pad_chunk, int32_t max_row_edges, float* cat,
                                int64_t ld_cat, void* stream);

/* out[c] = sum over r < nrows of part[r * ncols + c], fixed order (the
 * reduction of split-K partial products).  dtype 0 = float32, 1 = float64. */
GNS_API int gns_sum_rows(int32_t dtype, const void* part, int64_t nrows, int64_t ncols, void* out,
                         void* stream);

/* Backward of the above (model.py:223-225):
 * dh[s,:] = sum_{e: src=s, ascending dst} w_e * (dcat[dst_e, D:2D] / max(deg,1))
 *           (+ dcat[d, 0:D] where self_pos[d] == s).
 * Builds the transposed block CSR in the workspace.  Rows [n_src, pad_rows)
 * of dh are zero-filled.  Fused epilogue of the previous layer's backward
 * (model.py:218,220): with z_mask != NULL the output is relu'(z) * dh (z has
 * the row stride ld_dh), and with db != NULL the column sums of the output
 * (the previous layer's bias gradient) are written to db. */
GNS_API size_t gns_spmm_bwd_workspace_size(int64_t max_src, int64_t max_edges, int32_t dim);
GNS_API int gns_spmm_bwd(int32_t dtype, const void* dcat, int64_t ld_dcat, int32_t dim,
                 const gns_block_t* block, int64_t max_dst, int64_t max_src,
                 int64_t max_edges, int64_t pad_rows, const void* z_mask, void* db,
                 void* dh, int64_t ld_dh, void* ws, size_t ws_bytes, void* stream);

/* The two halves of gns_spmm_bwd: gns_block_transpose builds the block's
 * transpose (per src row, its edges sorted by dst — scipy's csc order) in the
 * workspace; it depends only on the sampled block, so the engine runs it on
 * the sampling branch.  gns_spmm_bwd_transposed then runs the backward from a
 * workspace the transpose was built in (same sizes).  Long transposed rows
 * (hub sources, more than 16 entries) are also registered as 32-entry
 * segments (count in block->counts[GNS_CNT_TSEGS]); the float32 backward
 * sums them across warps, in a fixed segment order (float32 results are
 * deterministic and identical across the float32 entry points; float64
 * keeps scipy's sequential order).  The workspace carries a generation
 * counter, so any number of backward launches may follow one transpose. */
GNS_API int gns_block_transpose(const gns_block_t* block, int64_t max_dst, int64_t max_src,
                                int64_t max_edges, int32_t dim, void* ws, size_t ws_bytes, void* stream);
GNS_API int gns_spmm_bwd_transposed(int32_t dtype, const void* dcat, int64_t ld_dcat, int32_t dim,
                                    const gns_block_t* block, int64_t max_dst, int64_t max_src,
                                    int64_t max_edges, int64_t pad_rows, const void* z_mask, void* db,
                                    void* dh, int64_t ld_dh, void* ws, size_t ws_bytes, void* stream);

/* The hidden-layer pair with a compact relu' mask: gns_spmm_fwd_bits is
 * gns_spmm_fwd(dtype 0, GNS_SPMM_RELU_INPUT) that also writes, for every h
 * row it reads, the row's relu' bits (word blk*4+q, bit l <-> element
 * 4*(blk*32+l)+q; gns_relu_bits_size(rows, dim) bytes); every src row of a
 * block is read (as a dst self row or an edge source).
 * gns_spmm_bwd_transposed_bits is gns_spmm_bwd_transposed(dtype 0) with the
 * mask taken from those bits instead of the pre-activation rows z (32 bytes
 * instead of dim*4 per row); results are identical. */
GNS_API size_t gns_relu_bits_size(int64_t rows, int32_t dim);
GNS_API int gns_spmm_fwd_bits(const float* h, int64_t ld_h, int32_t dim, const gns_block_t* block,
                              int64_t max_dst, int64_t pad_rows, float* cat, int64_t ld_cat,
                              uint32_t* relu_bits, void* stream);
GNS_API int gns_spmm_bwd_transposed_bits(const float* dcat, int64_t ld_dcat, int32_t dim,
                                         const gns_block_t* block, int64_t max_dst, int64_t max_src,
                                         int64_t max_edges, int64_t pad_rows, const uint32_t* relu_bits,
                                         float* db, float* dh, int64_t ld_dh, void* ws, size_t ws_bytes,
                                         void* stream);

/* relu backward fused with the bias gradient (model.py:218,220):
 * dz = (z > 0) ? dh : 0 (skipped when z == NULL: the output layer), db[c] =
 * sum over rows of dz[:, c] in a fixed order (deterministic).  n = *n_dev if
 * n_dev else n_rows; dh, z, dz share the row stride ld. */
GNS_API size_t gns_dense_bwd_workspace_size(int64_t max_rows, int32_t ncols);
GNS_API int gns_dense_bwd_bias(int32_t dtype, const void* dh, const void* z, int64_t ld,
                               const int32_t* n_dev, int64_t n_rows, int32_t ncols, void* dz,
                               void* db, void* ws, size_t ws_bytes, void* stream);

/* Softmax cross-entropy (model.py:189-200) over rows of logits for the
 * sorted targets; labels gathered as labels[targets[r]].  Writes grad_out
 * (same layout; rows [n, pad_rows) zero) and loss_out[0] = mean loss (device,
 * float64). */
GNS_API int gns_softmax_xent(int32_t dtype, const void* logits, int64_t ld, const int32_t* n_dev,
                     int64_t max_rows, int64_t pad_rows, int32_t num_classes, const int32_t* labels,
                     const int32_t* targets, void* grad_out, double* loss_out,
                     void* ws, size_t ws_bytes, void* stream);

/* The output layer's loss and gradients in one launch (the graphed step):
 * gns_softmax_xent's rows and loss_out[0] plus grad_bias[c] = sum over rows
 * of grad_out[:, c] (model.py:218-220; the output layer's dz is dlogits),
 * both reduced in a fixed order.  num_classes <= 256.  The workspace
 * (gns_softmax_xent_bias_workspace_size) must be zeroed once before the first
 * call; every call leaves its counter at zero. */
GNS_API size_t gns_softmax_xent_bias_workspace_size(int64_t max_rows, int64_t pad_rows, int32_t num_classes);
GNS_API int gns_softmax_xent_bias(int32_t dtype, const void* logits, int64_t ld, const int32_t* n_dev,
                                  int64_t max_rows, int64_t pad_rows, int32_t num_classes,
                                  const int32_t* labels, const int32_t* targets, void* grad_out,
                                  double* loss_out, void* grad_bias, void* ws, size_t ws_bytes,
                                  void* stream);

/* Bias-corrected Adam over a flat parameter buffer (model.py:229-242);
 * grad_scale multiplies the gradient first (1/W after an allreduce). */
GNS_API int gns_adam(int32_t dtype, void* params, const void* grads, void* m, void* v,
             int64_t n, double lr, double beta1, double beta2, double eps,
             int64_t step, double grad_scale, void* stream);

/* gns_adam with the step count on the device: step_dev points to two int64,
 * the step count and a ticket that must be zero; uses t = step_dev[0] + 1,
 * then the last CTA increments step_dev[0] and leaves the ticket at zero
 * (graph-replay safe, one launch). */
GNS_API int gns_adam_dev(int32_t dtype, void* params, const void* grads, void* m, void* v,
                         int64_t n, double lr, double beta1, double beta2, double eps,
                         int64_t* step_dev, double grad_scale, void* stream);

/* ---- synthetic graphs (graph.py:172-205 analogue, device generator) ---- */

/* Power-law (Chung-Lu style) random graph with the graph.py:142-169 contract:
 * symmetric, no self loops, no duplicate edges, rows sorted ascending.
 * num_pairs undirected endpoint pairs are drawn from Philox; endpoint rank x
 * follows P(x) ~ (x + offset)^-alpha, ranks are scattered over ids by a
 * Feistel bijection.  Two phases: count (builds sorted rows in the workspace,
 * writes the final indptr and *out_nnz_dev) then fill (compacts unique
 * neighbours into out_indices, capacity >= nnz). */
GNS_API size_t gns_gen_workspace_size(int64_t num_nodes, int64_t num_pairs);
GNS_API int gns_gen_powerlaw_count(int64_t num_nodes, int64_t num_pairs, double alpha, double offset,
                           uint32_t seed, int64_t* out_indptr, int64_t* out_nnz_dev, void* ws,
                           size_t ws_bytes, void* stream);
GNS_API int gns_gen_powerlaw_fill(int64_t num_nodes, int64_t num_pairs, const int64_t* indptr,
                          int32_t* out_indices, void* ws, size_t ws_bytes, void* stream);

/* Node attributes of the synthetic graphs (graph.py:249-253 scheme), pure
 * functions of (seed, node) so oracle/gen.c rebuilds them bit for bit:
 * labels in [0, num_classes), train/val/test masks (uniform r < train_frac,
 * then halves of the rest), and class-mean + noise float32 features
 * [n, ld] (columns >= dim zero; class_means = caller scratch [classes, ld]). */
GNS_API int gns_gen_node_attrs(int64_t n, int32_t num_classes, double train_frac, uint32_t seed,
                               int32_t* labels, uint8_t* train, uint8_t* val, uint8_t* test, void* stream);
GNS_API int gns_gen_features(int64_t n, int32_t dim, int32_t ld, int32_t num_classes, float noise,
                             uint32_t seed, const int32_t* labels, float* class_means, float* out,
                             void* stream);

/* build_csr (graph.py:142-169) on the device from caller-given endpoint arrays
 * (int32 u[m], v[m], all in [0, num_nodes)): symmetrise, drop self loops and
 * duplicates, sort rows.  Same two phases / workspace as the generator. */
GNS_API int gns_build_csr_count(int64_t num_nodes, const int32_t* u, const int32_t* v, int64_t num_pairs,
                                int64_t* out_indptr, int64_t* out_nnz_dev, void* ws, size_t ws_bytes,
                                void* stream);
GNS_API int gns_build_csr_fill(int64_t num_nodes, int64_t num_pairs, const int64_t* indptr,
                               int32_t* out_indices, void* ws, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GNS_B200_H_ */
