/*
 * countstream_gpu.h -- C ABI of libcountgpu.so, the B200 (sm_100a) counting-query engine.
 *
 * This is the drop-in boundary for the reference's hot path (arXiv 1804.04640,
 * reference package `countstream`, /root/reference/pkg/src/countstream).  The
 * reference answers one counting query per Python call and streams the
 * non-zero cells (N_ijk, N_ij) into an aggregator; this library answers
 * thousands of queries per launch on device-resident uint8 columns and folds
 * the aggregators the reference ships (LogLikelihood, MdlScore via LL) into the
 * kernel epilogue.  Every entry point below names the reference interface it
 * replaces (file:line relative to pkg/src/countstream/).
 *
 * Conventions
 *   - Every call returns int: CS_OK (0) or a negative CS_ERR_* code; the
 *     thread-local message of the last failure is cs_last_error().
 *   - Handles are opaque.  The library owns all device memory it allocates;
 *     the caller owns every buffer it passes.  Nothing passed in is retained
 *     past the call except through a returned handle.
 *   - Query descriptor arrays (var_off, vars, states) are HOST arrays.
 *   - Output arrays may be HOST or DEVICE pointers (detected per pointer).
 *     When every output is a device pointer a single-plan call is asynchronous on
 *     the context stream; otherwise it synchronises before returning.  A chunked
 *     cs_query_batch (see there) always synchronises.
 *   - Thread safety: every call that uses a context (directly or through a
 *     database / plan handle) holds that context's mutex for its duration, so
 *     handles may be shared across threads; calls on one context serialise.
 *   - Row counts: m (and a sharded database's total) must be < 2^32, the range
 *     of the uint32 count tables (CS_ERR_UNSUPPORTED otherwise).
 *   - No torch, no C++ types cross this boundary.
 *
 * Joint-index convention (reference baselines.py:51-57, survey a11): for a
 * query with target t and parents p_0..p_{k-2} (in the given order) the dense
 * table cell of a record is
 *       idx = s_t + r_t * (s_p0 + r_p0 * (s_p1 + r_p1 * (...)))
 * i.e. the target is the least significant digit and the first parent the
 * next one, so the r_t cells of one parent configuration j are contiguous:
 * N_ijk = table[j*r_t + k],  N_ij = sum_k table[j*r_t + k].
 */
#ifndef COUNTSTREAM_GPU_H
#define COUNTSTREAM_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CS_ABI_VERSION 1

/* return codes */
#define CS_OK 0
#define CS_ERR_INVALID (-1)     /* bad argument; maps to InvalidQueryError / ValueError */
#define CS_ERR_CUDA (-2)        /* CUDA runtime failure */
#define CS_ERR_OOM (-3)         /* device allocation failed */
#define CS_ERR_UNSUPPORTED (-4) /* valid query the engine does not handle (e.g. arity > 256) */
#define CS_ERR_PARSE (-5)       /* cs_db_load_text: the text is not a valid database (info[] says why) */

/* flags for cs_plan_create / cs_query_batch */
#define CS_WANT_TABLES 0x1u  /* write dense uint32 N_ijk tables */
#define CS_WANT_LOGLIK 0x2u  /* fp64 sum N_ijk ln(N_ijk/N_ij)  (aggregators.py:147-157) */
#define CS_WANT_MI 0x4u      /* fp64 mutual information I(X_t; Pa) in nats (new, survey 8a) */
#define CS_WANT_NNZ 0x8u     /* number of non-zero cells (NullSink.count, aggregators.py:80-93) */
#define CS_PARTIAL 0x10u     /* shard-local tables only: skip scores (merge then cs_plan_score) */
#define CS_NLOGN 0x20u       /* loglik output = sum over cells of N ln N (joint-table "entropy
                              * numerator"); LL(X|Pa) = NLOGN(X u Pa) - NLOGN(Pa), which lets a
                              * batch score every family from the distinct variable subsets */

typedef struct cs_ctx cs_ctx;   /* one device + one stream + scratch */
typedef struct cs_db cs_db;     /* device-resident database (one instance shard) */
typedef struct cs_plan cs_plan; /* an uploaded batch of counting queries */

/* ---- library / context ------------------------------------------------------------- */
int cs_abi_version(void);
const char* cs_last_error(void);
int cs_device_count(int32_t* count);
int cs_ctx_create(int32_t device, cs_ctx** out);
int cs_ctx_destroy(cs_ctx* ctx);
/* use an external cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream); NULL = own stream */
int cs_ctx_set_stream(cs_ctx* ctx, void* stream);
int cs_ctx_sync(cs_ctx* ctx);
/* number of kernels this context has launched so far (bench `gpu_launches`) */
int cs_ctx_launch_count(cs_ctx* ctx, int64_t* launches);
/* device time (ms, CUDA events on the context stream) of the last histogram phase (all K1
 * launches of one cs_plan_execute) or itemset launch; waits for it.  0 if none yet. */
int cs_ctx_last_kernel_ms(cs_ctx* ctx, float* ms);
/* number of SMs / bytes of dynamic smem the histogram kernel uses (diagnostics) */
/* class that answered the last cs_itemset_supports call on this context (0 = none yet) */
#define CS_ITEMSETS_BITGEMM 1  /* K4b: Harley-Seal bit-GEMM on the CUDA cores */
#define CS_ITEMSETS_TENSOR 2   /* K4c: u8 bit-GEMM on tcgen05 tensor cores */
#define CS_ITEMSETS_SELECTOR 3 /* K4d: rarest-item selection (sparse data) */
int cs_ctx_itemset_class(cs_ctx* ctx, int32_t* cls);
int cs_ctx_info(cs_ctx* ctx, int32_t* num_sms, int32_t* hist_smem_bytes, int32_t* hist_ctas);

/* ---- database (reference database.py) ----------------------------------------------- */
/* Replaces Database(data, arities) (database.py:36-84).  cols: n x m variable-major
 * uint8 states (row i = variable i), leading dimension ld >= m; host or device pointer.
 * arities: host int32[n], 1..256, every state < its arity (checked on device). */
int cs_db_create(cs_ctx* ctx, const uint8_t* cols, int32_t n, int64_t m, int64_t ld,
                 const int32_t* arities, cs_db** out);
/* Allocate an n x m database whose columns are filled by cs_db_generate (replaces
 * generate_synthetic, database.py:221-247, for device-side data at scale). */
int cs_db_create_empty(cs_ctx* ctx, int32_t n, int64_t m, const int32_t* arities, cs_db** out);
/* Fill column `var` with the counter-based generator (twin: oracle/gen_twin.py):
 *   u(row) = hash32(seed, var, row_offset + row)
 *   pcfg   = sum_t state(parents[t]) * prod_{u<t} arity(parents[u])
 *   state  = #{ t < r-1 : u >= thresholds[pcfg*(r-1) + t] }    (thresholds ascending per pcfg)
 * nparents may be 0 (marginal).  thresholds: host uint32[q*(r-1)]. */
int cs_db_generate(cs_db* db, int32_t var, uint64_t seed, int64_t row_offset, int32_t nparents,
                   const int32_t* parents, const uint32_t* thresholds, int64_t nthresholds);
int cs_db_destroy(cs_db* db);
int cs_db_shape(cs_db* db, int32_t* n, int64_t* m, int64_t* ld);
/* device pointer to the column block (n x ld bytes), read-only for the caller */
int cs_db_columns(cs_db* db, const uint8_t** dev, int64_t* ld);
/* copy rows [row0, row0+nrows) of column var to host (oracle checks of generated data) */
int cs_db_download(cs_db* db, int32_t var, int64_t row0, int64_t nrows, uint8_t* host);
/* Total record count of the whole (possibly sharded) database: used for MI's 1/m and
 * MDL's ln m when this handle holds only an instance shard.  Default = own m. */
int cs_db_set_total_rows(cs_db* db, int64_t m_total);
/* arities of the n variables (host int32[n]) */
int cs_db_arities(cs_db* db, int32_t* arities);

/* ---- device-side text ingest (reference load_csv, database.py:160-207) ---------------- */
/* Parse delimited integer records straight into a device database: line boundaries of
 * str.splitlines, each line stripped, blank lines dropped, split on `delim` (then each token
 * stripped) or on whitespace runs, int() base-10 tokens, a file whose smallest state is 1
 * shifted down by one, arities = observed maxima + 1 unless declared (`arities`, n_arities
 * entries, checked like Database(data, arities), database.py:36-84).  ASCII grammar: bytes >=
 * 0x80 are never whitespace or digits.  text: host or device bytes.
 * delim: a byte, CS_DELIM_SNIFF (',' if the first record holds one, else whitespace; the
 * reference's default) or CS_DELIM_WHITESPACE.
 * info (int64[8], always written): [0] CS_LOAD_* status, [1] record width, [2] records,
 * [3] delimiter used (-1 = whitespace), [4..6] detail (see CS_LOAD_*), [7] 1 if shifted.
 * Returns CS_ERR_PARSE with info[0] != CS_LOAD_OK when the reference would raise
 * DatabaseLoadError; CS_ERR_UNSUPPORTED for states above 255. */
#define CS_DELIM_SNIFF (-1)
#define CS_DELIM_WHITESPACE (-2)
#define CS_LOAD_OK 0
#define CS_LOAD_NO_RECORDS 1  /* "no records found" */
#define CS_LOAD_BAD_RECORD 2  /* info[4] = first bad record (ragged or non-integer token);
                               * its stripped line is text[info[5] .. info[6]) */
#define CS_LOAD_NEGATIVE 3    /* info[4] = smallest state */
#define CS_LOAD_ARITY_COUNT 4 /* info[4] = number of declared arities */
#define CS_LOAD_ARITY_SHORT 5 /* info[4] = row, [5] = variable, [6] = state */
#define CS_LOAD_ARITY_ZERO 6  /* a declared arity < 1 */
int cs_db_load_text(cs_ctx* ctx, const char* text, int64_t nbytes, int32_t delim,
                    const int32_t* arities, int32_t n_arities, cs_db** out, int64_t* info);

/* ---- bitmap index (reference bitmap.py:29-66) ---------------------------------------- */
/* Replaces build_bitmap_index (bitmap.py:53-66): one bit plane per (variable, state),
 * bit t of word t/32 = record t (little-endian, bitmap.py:31).  vars NULL => all. */
int cs_bitmap_build(cs_db* db, int32_t nvars, const int32_t* vars);
/* words per plane (padded) and a device pointer to plane (var, state), or NULL if not built */
int cs_bitmap_plane(cs_db* db, int32_t var, int32_t state, const uint32_t** dev, int64_t* words);

/* ---- counting queries (reference radix.py:113-156, bitmap.py:69-128) ----------------- */
/* Query q uses vars[var_off[q] .. var_off[q+1]): target first, then parents in the
 * reference's given order (QuerySpec(target, parents), database.py:102-126).
 * Cells are packed: table of q starts at table_off[q] = sum_{p<q} cells[p].
 * Joint state spaces above the dense limit (2^30 cells; env CS_MAX_DENSE_LOG2) are counted in
 * device hash tables instead (any number of variables, up to 2^63 cells): such a query has
 * cells[q] = 0 in the dense layout; its LL / MI / nnz outputs and its cs_plan_compact record
 * stream (hash order) are produced as for dense queries.  Not combinable with CS_PARTIAL. */
int cs_plan_create(cs_db* db, int32_t nq, const int32_t* var_off, const int32_t* vars,
                   uint32_t flags, cs_plan** out);
/* cells: host int64[nq] (nullable); table_off: host int64[nq] (nullable); total cells */
int cs_plan_info(cs_plan* plan, int64_t* cells, int64_t* table_off, int64_t* total_cells);
/* Run the batch.  tables: uint32[total_cells] (host/device/NULL); loglik, mi: double[nq];
 * nnz: int64[nq].  Replaces one radix_query(db, q, agg) per query with agg in
 * {NullSink, LogLikelihood, MdlScore} (radix.py:113, aggregators.py:80-193). */
int cs_plan_execute(cs_plan* plan, uint32_t* tables, double* loglik, double* mi, int64_t* nnz);
/* Scores of merged tables (after a cross-shard sum of CS_PARTIAL tables): same layout. */
int cs_plan_score(cs_plan* plan, const uint32_t* tables, double* loglik, double* mi, int64_t* nnz);
/* Non-zero cell stream (K5) for aggregators that want every cell (accept_block /
 * accept_record, aggregators.py:58-77).  Needs nnz from a previous execute/score;
 * out_off: host int64[nq] exclusive prefix of nnz.  Writes cell index, N_ijk, N_ij. */
int cs_plan_compact(cs_plan* plan, const uint32_t* tables, const int64_t* out_off, int64_t total_nnz,
                    int64_t* cell_idx, int64_t* n_ijk, int64_t* n_ij);
int cs_plan_destroy(cs_plan* plan);
/* create + execute + destroy.  Batches of >= ~4K queries are split into 2-4 chunks (chunk j a
 * 2^j share, first chunk >= 1.4K queries; env CS_QB_CHUNKS / CS_QB_GROWTH / CS_QB_MIN_CHUNK
 * override) whose host planning overlaps the previous chunk's kernels; outputs land at the same
 * offsets as one plan's (tables in query order, one entry per query in loglik / mi / nnz).
 * The whole batch is validated before the first chunk launches (errors name the query's index
 * in the batch; no output is written), and a chunked call returns synchronised. */
int cs_query_batch(cs_db* db, int32_t nq, const int32_t* var_off, const int32_t* vars,
                   uint32_t flags, uint32_t* tables, double* loglik, double* mi, int64_t* nnz);

/* One query with the lowest latency (the drop-in Strategy.query path; replaces one
 * radix_query / bitmap_query call, radix.py:113-156, bitmap.py:69-128).  vars: host int32[k],
 * target first.  Outputs as cs_query_batch for nq = 1 (any may be NULL).  Small queries (k <= 8,
 * <= 49,152 cells, m <= 2^18 rows; env CS_ONE_MAX_ROWS) run as one kernel whose descriptor is a
 * launch parameter and whose results land in mapped host memory; anything else goes through
 * cs_query_batch.  Synchronous. */
int cs_query_one(cs_db* db, int32_t k, const int32_t* vars, uint32_t flags, uint32_t* table, double* loglik,
                 double* mi, int64_t* nnz);
/* The same query's non-zero cells (the reference's record stream, radix.py:143-156 /
 * bitmap.py:103-116) in cell order: cell index, N_ijk, N_ij (host int64[cells] each; *nnz =
 * how many were written).  Only for queries of the single-query class (CS_ERR_UNSUPPORTED
 * otherwise: use a plan and cs_plan_compact). */
int cs_query_one_cells(cs_db* db, int32_t k, const int32_t* vars, int64_t* cell_idx, int64_t* n_ijk,
                       int64_t* n_ij, int64_t* nnz);

/* Batched MDL parent-set scoring (learn_parents, harness.py:296-348; MdlScore,
 * aggregators.py:163-193).  nlogn[nsub]: CS_NLOGN outputs of a plan over the distinct variable
 * subsets; family f scores  ll[f] = nlogn[s_idx[f]] - (p_idx[f] >= 0 ? nlogn[p_idx[f]] : m_ln_m)
 * and mdl[f] = -ll[f] + penalty[f].  Inputs/outputs host or device. */
int cs_family_scores(cs_ctx* ctx, int64_t nfam, const double* nlogn, int64_t nsub, const int32_t* s_idx,
                     const int32_t* p_idx, const double* penalty, double m_ln_m, double* ll, double* mdl);

/* ---- multi-GPU: instance sharding (survey 8(e)) ---------------------------------------------
 * Contract.  Rank g of N holds rows [r0, r0 + m_g) of the database (cs_db_create on that row
 * range, or cs_db_generate with row_offset = r0: the generator keys every state on the GLOBAL
 * row id, so shards reproduce the unsharded columns) and declares the global row count with
 * cs_db_set_total_rows(db, m).  Every rank plans the same queries with CS_PARTIAL: tables are
 * the shard's counts and no score is computed.  Counts are additive over disjoint row ranges, so
 * summing the partial tables over ranks (cs_reduce_tables, or any all-reduce / reduce-scatter of
 * uint32 / int32 words) gives the unsharded tables bit-exactly; cs_plan_score on merged tables
 * scores with the global m (MI's 1/m, MDL's ln m).  With REDUCE_SCATTER each rank receives the
 * merged tables of the queries it owns (a contiguous, equal-size slice of the table buffer:
 * one plan per owner, each writing its own slice) and scores only those.
 * NCCL (libnccl.so.2) is opened at run time; CS_ERR_UNSUPPORTED when it cannot be. */
#define CS_REDUCE_ALLREDUCE 0
#define CS_REDUCE_SCATTER 1
/* id: 128 bytes (ncclUniqueId), created on one rank and sent to the others by the caller */
int cs_comm_unique_id(void* id);
int cs_comm_init(cs_ctx* ctx, const void* id, int32_t rank, int32_t nranks);
int cs_comm_destroy(cs_ctx* ctx);
/* Sum uint32 tables over the ranks on the context stream (asynchronous).  tables, out: device.
 * ALLREDUCE: cells words, in place when out is NULL.  REDUCE_SCATTER: cells = nranks * S;
 * rank r receives the merged words [r S, (r + 1) S) in out (S words). */
int cs_reduce_tables(cs_ctx* ctx, uint32_t* tables, int64_t cells, int32_t op, uint32_t* out);
/* Every rank's `bytes` of send, concatenated in rank order into recv (device; the owners'
 * fp64 scores after a REDUCE_SCATTER merge).  Asynchronous on the context stream. */
int cs_comm_all_gather(cs_ctx* ctx, const void* send, int64_t bytes, void* recv);

/* ---- point counts / itemset supports (reference bitmap.py:131-136, radix.py:181-193) - */
/* counts[q] = #records with vars[j] == states[j] for every j in query q.  Uses bitmap
 * planes when every (var, state) has one (AND + popcount), else a byte scan. */
int cs_count_points(cs_db* db, int32_t nq, const int32_t* var_off, const int32_t* vars,
                    const int32_t* states, int64_t* counts);
/* All-pairs/all-triples support of `nitems` binary items in state 1 (mine_rules support_of,
 * harness.py:390-392, at configs[3] scale).  pairs: int64[nitems*nitems] (row-major, only
 * a<b written; nullable); triples: int64[C(nitems,3)] in itertools.combinations order
 * (nullable). Requires planes for state 1 of every item. */
int cs_itemset_supports(cs_db* db, int32_t nitems, const int32_t* items, int64_t* pairs,
                        int64_t* triples);

#ifdef __cplusplus
}
#endif
#endif /* COUNTSTREAM_GPU_H */
