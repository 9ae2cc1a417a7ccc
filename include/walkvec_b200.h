/*
 * walkvec_b200 — C ABI of the B200 (sm_100a) RDF2vec hot path.
 *
 * Plain C: device pointers, sizes and an opaque cudaStream_t (void*).  No
 * torch, numpy or C++ types cross this boundary.  Every function returns 0 on
 * success and a negative status on failure (-1 invalid argument, -2 CUDA
 * error); wv_last_error() returns the thread-local message.  Buffers are
 * caller-owned; functions that need scratch take (ws, ws_bytes) sized by the
 * matching *_workspace_bytes query.  Nothing here allocates device memory.
 *
 * Each entry point replaces one function of the reference's Python module
 * walkvec (/root/reference/pkg/src/walkvec/...); the citation is given per
 * function.  The reference has no FFI of its own: it is numpy all the way
 * down, so the binding a maintainer adds is a ctypes shim on the reference
 * side.
 */
#ifndef WALKVEC_B200_H
#define WALKVEC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WV_ABI_VERSION 1

/* generator kinds for walk draws (numpy-compatible streams) */
#define WV_RNG_PCG64 0  /* numpy default_rng(SeedSequence(...)) — the unmodified reference */
#define WV_RNG_PHILOX 1 /* numpy Generator(Philox(SeedSequence(...))) */

/* flat-corpus filter modes */
#define WV_KEEP_ENTITY 0   /* walks.project_corpus(..., "entity")   walks.py:323-341 */
#define WV_KEEP_PROPERTY 1 /* walks.project_corpus(..., "property") walks.py:323-341 */
#define WV_KEEP_TOKENS 2   /* w2v._filter_min_count                 w2v.py:146-158  */

/* parameter-store precision for SGNS */
#define WV_FP32 0
#define WV_FP64 1

/* SGNS pair source */
#define WV_MODEL_SKIPGRAM 0
#define WV_MODEL_CBOW 1
#define WV_PAIRS_NATIVE 0   /* device Feistel permutation + length-class decode + Philox negatives */
#define WV_PAIRS_EXPLICIT 1 /* caller-supplied pair table, epoch permutation, negatives (replay) */

const char* wv_last_error(void);
int wv_abi_version(void);
/* sizeof of the ABI structs (0 WvSgnsDevState, 1 WvSgnsModel, 2 WvSgnsBatch) for binding checks */
int64_t wv_struct_size(int which);
int wv_stream_sync(void* stream);
/* kernels this library has enqueued so far (host-side count; a CUDA-graph
 * capture counts its launches once, replays are not seen here) */
int64_t wv_launch_count(void);
/* n CUDA events for kernel timing; records made while `stream` is being
 * captured into a CUDA graph become external event-record nodes, so a
 * replayed graph still timestamps its phases (profiling / bench roofline). */
void* wv_timer_create(int n);
int wv_timer_record(void* timer, int i, void* stream);
int wv_timer_elapsed(void* timer, int i, int j, float* ms);
int wv_timer_destroy(void* timer);

/* numpy SeedSequence(prefix + [index]).generate_state(n64, uint64) on the host.
 * prefix = little-endian u32 words of the leading entropy integers. */
int wv_seedseq_generate(const uint32_t* entropy_prefix, int n_prefix, uint64_t index, int n64, uint64_t* out);
/* element k (0-based) of the numpy u64 stream of PCG64/Philox seeded by that SeedSequence */
int wv_stream_u64(const uint32_t* entropy_prefix, int n_prefix, uint64_t index, int kind, uint64_t k, uint64_t* out);

/* ---------------------------------------------------------------- graph --
 * Replaces graph.build_graph (graph.py:74-98): stable CSR by source.
 * edges: device int64 (E,3) rows (src, pred, dst), all in [0, V).
 * row_offsets: int64[V+1]; packed_edges: u64[E] = pred << 32 | dst. */
int64_t wv_csr_workspace_bytes(int64_t E, int64_t V);
int wv_csr_build(const int64_t* edges, int64_t E, int64_t V, int64_t* row_offsets, uint64_t* packed_edges, void* ws,
                 int64_t ws_bytes, void* stream);
/* Graph.col_targets / col_predicates views (graph.py:38-41); either may be NULL */
int wv_csr_unpack(const uint64_t* packed_edges, int64_t E, int64_t* col_targets, int64_t* col_predicates,
                  void* stream);

/* ---------------------------------------------------------------- walks --
 * Replaces walks.random_walks/_walk_shard (walks.py:117-204).  The global work
 * list is repeat(roots, walk_number); this call computes walkers
 * [work_begin, work_begin+work_count) of it (multi-GPU shards pass disjoint
 * ranges; the union is byte-identical to one call over everything).
 * seed_prefix = u32 words of [rng_seed, 0] (SeedSequence([seed, 0, shard])).
 * corpus: int32 [work_count, 2*depth+1] padded with -1; lengths: int32[work_count]. */
/* walk adjacency (optional, E < 2^32): per packed edge e, 16 bytes {pred, dst,
 * row start of dst, out-degree of dst}, so a walk hop is one dependent load
 * (the chosen edge names the next row) instead of offsets -> edge.  Random
 * 8-byte CSR reads cost a 64-byte DRAM fetch each (ncu: 113 B/hop at cfg5). */
int wv_walk_adjacency_build(const int64_t* row_offsets, const uint64_t* packed_edges, int64_t vertex_count,
                            int64_t edge_count, void* walk_adj, void* stream);
/* workspace: the launch's per-shard generator seeds (ws = NULL seeds per CTA) */
int64_t wv_random_walks_workspace_bytes(int64_t work_begin, int64_t work_count);
int wv_random_walks(const int64_t* row_offsets, const uint64_t* packed_edges, const void* walk_adj,
                    int64_t vertex_count, const int64_t* roots, int64_t n_roots, int64_t walk_number, int walk_depth, int64_t work_begin,
                    int64_t work_count, const uint32_t* seed_prefix, int n_prefix, int rng_kind, int32_t* corpus,
                    int32_t* lengths, void* ws, int64_t ws_bytes, void* stream);

/* fixed-width rows -> flat tokens (int32 or int64 by token_bytes) + int64 offsets[n+1]
 * (the PAD strip + concatenate + cumsum of walks.py:139-141, 181-184) */
int64_t wv_compact_workspace_bytes(int64_t n_walks);
int wv_corpus_compact(const int32_t* corpus, const int32_t* lengths, int64_t n_walks, int width, int64_t* offsets,
                      void* tokens, int token_bytes, void* ws, int64_t ws_bytes, void* stream);

/* duplicate_free (walks.py:186-202) over groups of `group` consecutive walks */
int64_t wv_dedup_workspace_bytes(int64_t n_walks);
int wv_duplicate_free(const int32_t* corpus, const int32_t* lengths, int64_t n_walks, int width, int64_t group,
                      int32_t* out_corpus, int32_t* out_lengths, int64_t* n_kept, void* ws, int64_t ws_bytes,
                      void* stream);

/* project_corpus (walks.py:323-341) and the min_count token filter (w2v.py:146-158) */
int64_t wv_filter_workspace_bytes(int64_t n_walks);
int wv_corpus_filter(const int32_t* tokens, const int64_t* offsets, int64_t n_walks, int mode,
                     const uint8_t* token_mask, int64_t* new_offsets, int32_t* new_tokens, void* ws, int64_t ws_bytes,
                     void* stream);

/* frequency = bincount(tokens, minlength=V) (w2v.py:147, pipeline.py:217) */
int wv_token_histogram(const int32_t* tokens, int64_t n_tokens, int64_t vocab_size, int64_t* counts, int zero_first,
                       void* stream);

/* ----------------------------------------------------------------- BFS ---
 * Replaces walks.bfs_walks/_bfs_tree (walks.py:207-310). */
int64_t wv_bfs_workspace_bytes(int64_t vertex_count, int64_t n_roots);
/* phase 1: walks per root, min(leaves, max_walks_per_root) (<= 0: uncapped, the reference) */
int wv_bfs_count(const int64_t* row_offsets, const uint64_t* packed_edges, int64_t vertex_count, const int64_t* roots,
                 int64_t n_roots, int walk_depth, int64_t max_walks_per_root, int64_t* walk_counts, void* ws,
                 int64_t ws_bytes, void* stream);
/* phase 2 (same ws): rows [walk_base[r], walk_base[r]+walk_counts[r]) of the
 * fixed-width int32 corpus [total, 2*depth+1] (-1 padded) + lengths */
int wv_bfs_emit(const int64_t* row_offsets, const uint64_t* packed_edges, int64_t vertex_count, const int64_t* roots,
                int64_t n_roots, int walk_depth, int64_t max_walks_per_root, const int64_t* walk_base, int32_t* corpus,
                int32_t* lengths, void* ws, int64_t ws_bytes, void* stream);
/* PathTable (walks.py:87-103, 284-293) rows of a flat BFS corpus: leaf edge first */
int wv_path_table(const int32_t* tokens, const int64_t* offsets, int64_t n_walks, int64_t* sources, int64_t* targets,
                  int64_t* walk_ids, void* stream);

/* ---------------------------------------------------------------- SGNS ---
 * Replaces w2v.train for model="skipgram" (w2v.py:507-576) together with
 * init_embeddings (:123-131), generate_pairs (:161-191), sample_negatives
 * (:225-239), sgns_batch_grads (:276-299), _coalesce (:407-416) and RowAdam
 * (:364-404). */
typedef struct WvSgnsDevState {
  int64_t lo;             /* first permuted position of the current batch */
  int64_t epoch;
  int64_t batch;          /* batch index within the epoch */
  int64_t step;           /* optimizer steps so far (dense-mode global step) */
  double epoch_loss_sum;  /* sum of batch_loss * batch_rows (w2v.py:571) */
  int64_t epoch_count;
  int64_t diverged_epoch; /* first non-finite batch (w2v.py:566-567), -1 if none */
  int64_t diverged_batch;
  double last_batch_loss;
  uint32_t block_counter;
  uint32_t pad;
  int64_t rows_updated;   /* cumulative unique (row, matrix) updates -- telemetry */
} WvSgnsDevState;

typedef struct WvSgnsModel {
  int64_t vocab_size;
  int vector_size;
  int precision; /* WV_FP32 / WV_FP64 */
  int sparse;    /* TrainConfig.use_sparse */
  int pad;
  double learning_rate;
  void* input;   /* [V,d] */
  void* output;  /* [V,d] */
  void* m_in;
  void* v_in;
  void* m_out;
  void* v_out;
  int32_t* steps_in; /* RowAdam.row_steps */
  int32_t* steps_out;
  uint8_t* touched_in; /* EmbeddingModel.touched_input */
  uint8_t* touched_out;
  uint8_t* modified_in; /* rows whose stored value differs from the init */
  uint8_t* modified_out;
  void* dense_g_in; /* [V,d] gradient staging, dense mode only */
  void* dense_g_out;
  WvSgnsDevState* state;
} WvSgnsModel;

typedef struct WvSgnsBatch {
  int mode; /* WV_PAIRS_NATIVE / WV_PAIRS_EXPLICIT */
  int negatives; /* per item: negative_samples (skip-gram) or window_size (CBOW, w2v.py:481-484) */
  int window;
  int model; /* WV_MODEL_SKIPGRAM / WV_MODEL_CBOW (TrainConfig.model) */
  int64_t batch_rows;
  int64_t n_pairs;
  uint64_t seed;
  /* native */
  const int32_t* tokens;
  const int64_t* offsets;
  const int32_t* walks_by_class;
  const int64_t* class_len;
  const int64_t* class_walk_start;
  const int64_t* class_pair_start;
  int64_t n_classes;
  const int32_t* candidates; /* NULL: identity */
  int64_t n_candidates;
  /* explicit */
  const int32_t* pairs;
  const int64_t* perm;
  const int32_t* negative_table;
  /* optional wv_timer_create handle: 7 stamps per batch from slot timer_base
   * (start, decode end, gather end, join, owner end, sort start, sort end) */
  void* timer;
  int64_t timer_base;
  /* CBOW: instance table [n_pairs, 2*window + 1] from wv_cbow_instances
   * (context columns, -1 padded, then the target); both pair modes index it */
  const int32_t* instances;
} WvSgnsBatch;

int wv_sgns_init(int64_t vocab_size, int vector_size, const uint32_t* seed_prefix, int n_prefix, int precision,
                 void* input_matrix, void* output_matrix, void* stream);
int wv_sgns_export(int64_t vocab_size, int vector_size, const uint32_t* seed_prefix, int n_prefix, int precision,
                   int matrix, const void* params, const uint8_t* modified, double* out64, void* stream);
int64_t wv_pair_index_workspace_bytes(int64_t n_walks);
int wv_pair_index_build(const int64_t* offsets, int64_t n_walks, int window, int32_t* walks_by_class,
                        int64_t* class_len, int64_t* class_walk_start, int64_t* class_pair_start, int64_t* n_classes,
                        int64_t* n_pairs, void* ws, int64_t ws_bytes, void* stream);
int64_t wv_pairs_workspace_bytes(int64_t n_walks);
int wv_generate_pairs(const int32_t* tokens, const int64_t* offsets, int64_t n_walks, int window, int32_t* pairs,
                      int64_t* n_pairs_out, void* ws, int64_t ws_bytes, void* stream);
int64_t wv_candidates_workspace_bytes(int64_t vocab_size);
int wv_candidates(const int64_t* freq, int64_t vocab_size, int64_t min_count, uint8_t* keep, int32_t* candidates,
                  int64_t* n_candidates, void* ws, int64_t ws_bytes, void* stream);
/* inspection (skip-gram): decode the epoch's permuted positions [pos_begin,
 * pos_begin + n) exactly as a batch does -> rows [n, 2 + negatives] (centre,
 * context, negatives) and, if pair_index != NULL, the pair index each position
 * maps to (native: the Feistel image in [0, n_pairs); explicit: perm[pos]).
 * The pair-order and negative-distribution tests run through this. */
int wv_sgns_decode(const WvSgnsBatch* batch, int64_t epoch, int64_t pos_begin, int64_t n, int32_t* rows,
                   int64_t* pair_index, void* stream);
/* reset the batch cursor to permuted position `start` (a worker's span start) */
int wv_sgns_epoch_begin(WvSgnsDevState* state, int64_t epoch, int64_t start, void* stream);
/* cbow_window = 0 for skip-gram, the CBOW window_size otherwise (2W context rows per item) */
int64_t wv_sgns_batch_workspace_bytes(int64_t vocab_size, int vector_size, int negatives, int64_t batch,
                                      int precision, int cbow_window);
/* copy the corpus side of `batch` (pair source, negatives) into the workspace;
 * needed before replaying a CUDA graph of wv_sgns_batch calls on a new corpus
 * (uncaptured wv_sgns_batch calls bind by themselves) */
int wv_sgns_bind(const WvSgnsBatch* batch, void* ws, int64_t ws_bytes, int64_t vocab_size, int vector_size,
                 int precision, void* stream);
/* zero the workspace's persistent per-row counters: once after allocating it */
int wv_sgns_workspace_init(void* ws, int64_t ws_bytes, int64_t vocab_size, int vector_size, int negatives,
                           int64_t batch, int precision, int cbow_window, void* stream);
int wv_sgns_batch(const WvSgnsModel* model, const WvSgnsBatch* batch, void* ws, int64_t ws_bytes, void* stream);
/* CBOW instances (w2v.generate_cbow_instances, w2v.py:194-222): one row per
 * token of every walk of length >= 2, in corpus order: 2*window context
 * columns (column 2(s-1) = token s to the left, 2(s-1)+1 = s to the right,
 * -1 when outside the walk) then the target.  Pass instances = NULL to get
 * the count only (*n_instances, device int64). */
int64_t wv_cbow_instances_workspace_bytes(int64_t n_walks);
int wv_cbow_instances(const int32_t* tokens, const int64_t* offsets, int64_t n_walks, int window, int32_t* instances,
                      int64_t* n_instances, void* ws, int64_t ws_bytes, void* stream);
/* `count` consecutive batches, software-pipelined over the workspace's two
 * halves (decode + grouping of batch i+1 on a side stream while batch i is
 * gathered and applied); equal to `count` wv_sgns_batch calls; capturable as
 * one CUDA graph.  Replaces the batch loop of w2v._train_single (w2v.py:553-565). */
int wv_sgns_batches(const WvSgnsModel* model, const WvSgnsBatch* batch, void* ws, int64_t ws_bytes, int64_t count,
                    void* stream);
/* ----------------------------------------------------------- row-sharded --
 * cfg5 mode (SGNS state too large to replicate): rank `shard` of
 * `nshard` owns rows r with r % nshard == shard of both matrices (local row
 * r / nshard) and their RowAdam state; `model` is that local store
 * (vocab_size = ceil(vocab_global / nshard)).  Per global batch:
 * decode_group -> requests -> (all-to-all) -> serve -> (all-to-all) -> place ->
 * gather -> (all-gather of U, G, coef in global pair order) -> update.  The
 * result equals single-GPU training with the same global batch. */
int wv_shard_init(int64_t vocab_global, int vector_size, const uint32_t* seed_prefix, int n_prefix, int precision,
                  int nshard, int shard, void* input_local, void* output_local, void* stream);
int wv_shard_decode_group(const WvSgnsModel* model, const WvSgnsBatch* batch, void* ws, int64_t ws_bytes,
                          int64_t vocab_global, int nshard, int shard, void* stream);
int wv_shard_requests(const WvSgnsModel* model, const WvSgnsBatch* batch, void* ws, int64_t ws_bytes,
                      int64_t vocab_global, int nshard, int shard, int64_t item_begin, int64_t n_items,
                      uint32_t* cursor, int64_t* keys, int32_t* items, int32_t* ident, int64_t* counts,
                      void* stream);
/* split sizes of a skip-gram batch's request all-to-all, computed without
 * communication: decodes positions [pos_begin, pos_begin + rows) of `epoch`
 * (into scratch_rows [rows, 2 + negatives]) and counts counts[s * nshard + o]
 * = rows requested by rank s (its pair share) from owner o.  Run one batch
 * ahead with an async copy, it removes the host round trip per batch. */
int wv_shard_count_requests(const WvSgnsBatch* batch, int64_t epoch, int64_t pos_begin, int64_t rows, int nshard,
                            int32_t* scratch_rows, int64_t* counts, void* stream);
int wv_shard_serve(const WvSgnsModel* model, const int64_t* keys, int64_t n, int64_t vocab_global, int nshard,
                   void* rows, void* stream);
int wv_shard_place(const void* rows, const int32_t* items, int64_t n, int vector_size, int precision,
                   void* itemrows, void* stream);
int wv_shard_gather(const WvSgnsModel* model, const WvSgnsBatch* batch, void* ws, int64_t ws_bytes,
                    int64_t vocab_global, int nshard, int shard, const void* itemrows, const int32_t* ident,
                    int64_t pair_count, void* U, void* G, void* coef, void* stream);
int wv_shard_update(const WvSgnsModel* model, const WvSgnsBatch* batch, void* ws, int64_t ws_bytes,
                    int64_t vocab_global, int nshard, int shard, const void* U, const void* G, const void* coef,
                    void* stream);
#define WV_PHASE_PAIRS 1  /* decode pair/negative rows; gather rows, dots, coefficients, batch loss */
#define WV_PHASE_GROUP 2  /* group contribution slots by destination row (no sort) */
#define WV_PHASE_UPDATE 4 /* per unique row: slot-ordered sum + RowAdam */
#define WV_PHASE_ALL 7
int wv_sgns_batch_phases(const WvSgnsModel* model, const WvSgnsBatch* batch, void* ws, int64_t ws_bytes, int phases,
                         void* stream);

/* Replica averaging (w2v.py:642-659 _merge_bundles + :719-724 resync), run
 * after an all-reduce(sum) of the deltas and touch counts across ranks. */
int wv_replica_delta(const void* params, const void* snapshot, int64_t n, int precision, void* delta, void* stream);
int wv_replica_apply(void* params, void* snapshot, const void* delta_sum, const float* touch_count, int64_t rows,
                     int vector_size, int precision, void* stream);

/* --------------------------------------------------------------- ingest --
 * GPU ingest: ingest.parse_ntriples / parse_edge_table +
 * build_vocabulary (ingest.py:116-257, 368-396) over raw UTF-8 file bytes.
 * Phase 1 finds universal-newline line terminators (line_end[n_terms]);
 * phase 2 parses every line (mode 0 N-Triples, 1 whitespace table, 2
 * `delim`-separated table), interns keys by first occurrence (64-bit hash of
 * the unescaped key, every occurrence verified against its first one) and
 * writes edges, roles and each token's key span.  n_lines = n_terms, + 1
 * when the text does not end with a terminator (the caller then sets
 * line_end[n_terms] = n_bytes).  Per line status: 0 skipped,
 * 1 statement, 2 ParseError, 3 ValueError; err = code (negative: -columns),
 * err_at = byte position; bad[2] = first error line, first ValueError line;
 * n_out = {statements, edges, vocabulary size, hash-collision flag}. */
int64_t wv_ingest_lines_workspace_bytes(int64_t n_bytes);
int wv_ingest_lines(const uint8_t* text, int64_t n_bytes, int64_t* line_end, int64_t* n_terms, void* ws,
                    int64_t ws_bytes, void* stream);
int64_t wv_ingest_workspace_bytes(int64_t n_lines);
/* csv.reader records of a quoted csv/tsv text (quoted fields may hold the
 * delimiter and line breaks): rec_end[r] = position of record r's terminator,
 * rec_line[r] = csv.reader's line_num after it; *n_records, *n_lines (device)
 * = terminated records, universal-newline line terminators.  Parse them with
 * wv_ingest_parse mode 3, line_end = rec_end, line_no = rec_line. */
int64_t wv_ingest_records_workspace_bytes(int64_t n_bytes);
int wv_ingest_records(const uint8_t* text, int64_t n_bytes, int delim, int64_t* rec_end, int64_t* rec_line,
                      int64_t* n_records, int64_t* n_lines, void* ws, int64_t ws_bytes, void* stream);
/* mode 3: quoted delimiter table over csv.reader records; line_no (mode 3) = each
 * record's line number (has_header skips the record at line 1); NULL otherwise */
int wv_ingest_parse(const uint8_t* text, int64_t n_bytes, const int64_t* line_end, int64_t n_lines, int mode,
                    const int64_t* line_no, uint64_t hash_seed, int delim, int has_header, int include_literals, uint8_t* status, int32_t* err, int64_t* err_at,
                    int64_t* bad, int64_t* n_out, int64_t* edges, uint32_t* roles, int64_t* tok_span, void* ws,
                    int64_t ws_bytes, void* stream);

/* -------------------------------------------------------------- formats --
 * Writers of SURVEY §8f row 3, formatted on the device.  Text export of `rows`
 * vectors (fp32 / fp64 [rows, d]) as "<lexical><sep>%.8g<sep>...\n" lines
 * (pipeline.save_embeddings_text / _tsv, pipeline.py:236-251; Python's
 * correctly rounded %.8g): plan -> *total bytes (device int64), *bad = 1 if a
 * value is outside [1e-30, 1e16) in magnitude (and not 0, inf or nan); emit ->
 * the bytes.  WVC1 corpus body (walks.save_corpus_binary, walks.py:344-364):
 * per walk a u32 length then its u32 tokens (header written by the caller). */
int64_t wv_format_workspace_bytes(int64_t rows, int d);
int wv_format_plan(const void* vec, int precision, int64_t rows, int d, const int64_t* lex_off, int64_t* total,
                   int* bad, void* ws, int64_t ws_bytes, void* stream);
int wv_format_emit(const char* lex, const int64_t* lex_off, int64_t rows, int d, char sep, char* out, void* ws,
                   int64_t ws_bytes, void* stream);
int wv_wvc1_pack(const int32_t* tokens, const int64_t* offsets, int64_t n_walks, uint32_t* body, void* stream);
/* Vocabulary TSV (Vocabulary.save_tsv, ingest.py:307-323): one line per token
 * "<token>\t<lexical, \\ \t \n \r escaped>\t<roles: e if bit 0, p if bit 1>\t<count>\n".
 * out = NULL: only *total (device int64, the file size) is computed. */
int64_t wv_vocab_tsv_workspace_bytes(int64_t rows);
int wv_vocab_tsv(const uint8_t* lex, const int64_t* lex_off, int64_t rows, const uint8_t* roles, const int64_t* counts,
                 char* out, int64_t* total, void* ws, int64_t ws_bytes, void* stream);
/* WVC1 reader (load_corpus_binary, walks.py:368-389): the body words after the
 * 12-byte header -> offsets [count + 1] and tokens [n_words - count].  Records
 * are located by speculative chunk parsing (any record length; records of 128
 * words or more take a sequential path).  *status (device int): 0 ok, 2 corrupt
 * (a record runs past the body, or words remain after `count` records), 3 the
 * body ends before `count` records. */
int64_t wv_wvc1_read_workspace_bytes(int64_t n_words);
int wv_wvc1_read(const uint32_t* body, int64_t n_words, int64_t count, int64_t* offsets, int32_t* tokens, int* status,
                 void* ws, int64_t ws_bytes, void* stream);

/* ------------------------------------------------------------ synthetic --
 * Measurement inputs (BASELINE.json configs).  gen_barabasi restates
 * benchgen.gen_barabasi (benchgen.py:78-109): vertex v >= 1 adds min(m, v)
 * distinct edges v -> t, t drawn from the degree+1 attachment bag.  Same
 * process, counter-based draws (not numpy's stream).  src/dst int64 sized
 * wv_barabasi_edge_count(n, m), ordered by source then draw slot like the
 * reference.  Synchronises `stream` (a few convergence rounds). */
int64_t wv_barabasi_edge_count(int64_t n, int m);
int64_t wv_barabasi_workspace_bytes(int64_t n, int m);
int wv_gen_barabasi(int64_t n, int m, uint64_t seed, int64_t* src, int64_t* dst, void* ws, int64_t ws_bytes,
                    void* stream);
/* benchgen.gen_erdos_renyi (benchgen.py:112-127) and gen_uniform_attachment
 * (:130-149) semantics with counter-based draws: edges in the reference's order
 * (row-major pairs; per vertex ascending distinct targets).  src = dst = NULL
 * returns the edge count in *n_edges (device int64); then call with buffers. */
int64_t wv_gen_rows_workspace_bytes(int64_t n);
int wv_gen_erdos_renyi(int64_t n, double p, uint64_t seed, int64_t* src, int64_t* dst, int64_t* n_edges, void* ws,
                       int64_t ws_bytes, void* stream);
int wv_gen_uniform_attachment(int64_t n, int m, uint64_t seed, int64_t* src, int64_t* dst, int64_t* n_edges,
                              void* ws, int64_t ws_bytes, void* stream);
/* First-occurrence token encoding of integer triples (ingest.build_vocabulary,
 * ingest.py:368-396, over benchgen.assign_predicates' "v{u}"/"P{k}" triples,
 * benchgen.py:152-161).  Keys: entity u -> u, predicate k -> n_entities + k.
 * edges_out (E,3) int64 tokens (may be NULL); token_of_key[n_keys] (-1 when
 * absent); key_of_token[n_keys] (-1 past the vocabulary; may be NULL);
 * *vocab_size is a device int64. */
int64_t wv_encode_workspace_bytes(int64_t E, int64_t n_keys);
int wv_encode_triples(const int64_t* src, const int64_t* preds, const int64_t* dst, int64_t E, int64_t n_entities,
                      int64_t n_predicates, int64_t* edges_out, int64_t* token_of_key, int64_t* key_of_token,
                      int64_t* vocab_size, void* ws, int64_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* WALKVEC_B200_H */
