/*
 * fjg.h — C-ABI of the B200 Free Join executor (libfjg.so).
 *
 * The reference has no FFI layer; its API surface is the
 * GHT interface of Fig 5 extended in SPEC.md:286-339, the
 * executor operations of SPEC.md:387-431, the plan compiler of
 * SPEC.md:195-240 and the typed exceptions of proj/include/fj/error.hpp:9-33.
 * Each entry point below names the reference interface it replaces.
 *
 * Conventions
 *  - Every int-returning call returns FJG_OK (0) or one FJG_E_* category
 *    (error.hpp:8: "Error categories map 1:1 onto CLI exit codes").
 *    fjg_last_error() returns the thread-local message of the last failure.
 *  - No exceptions and no C++/torch types cross this boundary.
 *  - Handles are not thread-safe; distinct engines may run concurrently
 *    (reentrant with disjoint contexts).
 *  - fjg_execute is synchronous: it returns after its stream has drained.
 *  - Values are int32 columns; they are widened to int64 exactly as
 *    fj::Value (value.hpp:28-57) when hashed for the checksum.
 */
#ifndef FJG_H_
#define FJG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error.hpp:9-33 categories */
#define FJG_OK 0
#define FJG_E_IO 1
#define FJG_E_PARSE 2
#define FJG_E_VALIDATION 3
#define FJG_E_RESOURCE 4 /* cudaErrorMemoryAllocation, NCCL OOM, capacity */
#define FJG_E_ENGINE 5   /* invariant violation or CUDA launch failure */

/* plan modes (SPEC.md:463-464 RunConfig.mode) */
#define FJG_MODE_BINARY 0
#define FJG_MODE_FREE 1
#define FJG_MODE_GENERIC 2

/* output modes (SPEC.md:374 ExecOptions.output_mode) */
#define FJG_OUT_COUNT 0
#define FJG_OUT_ENUMERATE 1
#define FJG_OUT_FACTORIZED_COUNT 2

/* predicate comparators */
#define FJG_CMP_EQ 0
#define FJG_CMP_NE 1
#define FJG_CMP_LT 2
#define FJG_CMP_LE 3
#define FJG_CMP_GT 4
#define FJG_CMP_GE 5

#define FJG_MAX_NODES 32
#define FJG_MAX_ATOMS 16

typedef struct fjg_engine fjg_engine;
typedef struct fjg_relation fjg_relation;
typedef struct fjg_query fjg_query;

/* ExecOptions. batch_size is the iter_batch size of
 * Fig 13: on the device it bounds the number of cover
 * candidates expanded per node launch (0 = engine default: 2^25, up to 2^27
 * when the largest relation has more than 2^22 rows; at most 2^31, else
 * FJG_E_VALIDATION). */
typedef struct {
  uint64_t batch_size;
  int32_t dynamic_cover; /* §4.4 select_cover */
  int32_t output_mode;   /* FJG_OUT_* */
  int32_t min_var;       /* head-variable index aggregated with MIN, or -1 */
  int32_t collect_timing;/* record build/join phase times (CUDA events) */
  int32_t backend;       /* FJG_BACKEND_*: GHT backend of new() */
} fjg_exec_options;

/* GHT backends (the §5.3 ablation ladder):
 * COLT builds nothing up front and forces subtries lazily in batch; SLT
 * forces every trie's level 0 before the join and deeper levels lazily;
 * SIMPLE forces every level of every trie before the join. */
#define FJG_BACKEND_COLT 0
#define FJG_BACKEND_SLT 1
#define FJG_BACKEND_SIMPLE 2

/* Result: OutputSink counter + ExecStats/TrieStats
 * (SPEC.md:377-380, :280-283). count is 128-bit (count_hi:count_lo). */
typedef struct {
  uint64_t count_lo;
  uint64_t count_hi;
  uint64_t checksum;          /* sum mult*fmix64(TupleHash(t)) mod 2^64 */
  int64_t min_value;          /* valid iff has_min */
  int32_t has_min;
  int32_t num_nodes;
  uint64_t output_rows;       /* enumerate mode: rows available via fjg_query_output */
  uint64_t probes;            /* get() calls issued by the executor */
  uint64_t probe_misses;
  uint64_t node_body_entries[FJG_MAX_NODES]; /* cover tuples iterated per node */
  uint64_t node_probes[FJG_MAX_NODES];       /* get() calls per node */
  uint64_t node_inputs[FJG_MAX_NODES];       /* bindings entering each node */
  uint64_t maps_built;        /* subtries forced (TrieStats.maps_built) */
  uint64_t keys_inserted;     /* distinct keys inserted into COLT maps */
  uint64_t forces;            /* force batches executed on the device */
  uint64_t rows_forced;       /* offsets regrouped by forcing */
  double build_ms;            /* device time in COLT forcing (if collect_timing) */
  double join_ms;             /* device time in node kernels (if collect_timing) */
  double last_node_ms;        /* device time of the fused last-node kernel (if collect_timing) */
  uint64_t last_node_launches;
  uint64_t last_node_candidates; /* cover candidates expanded by the last node */
  double first_node_ms;       /* device time of node 0's kernels when node 0 is not the last (if collect_timing) */
  double memo_ms;             /* device time of the memoised chain passes (factorised count, if collect_timing) */
  uint64_t memo_rows_resolved;/* rows whose fresh-atom roots were probed once (k_memo_resolve) */
  uint64_t memo_rows_gathered;/* rows folded by the memo passes (k_memo_gather) */
  uint64_t memo_rows_init;    /* level-0 positions scanned to initialise memo groups (k_memo_init) */
  /* TrieStats of each atom's physical trie (renamed
   * self-join atoms that share one report the same values): subtries forced
   * into maps, and bit l set iff some map was built at schema level l. */
  uint64_t atom_maps_built[FJG_MAX_ATOMS];
  uint32_t atom_levels_forced[FJG_MAX_ATOMS];
  uint32_t kernel_launches;   /* kernels this library launched for the call */
  uint32_t host_syncs;
} fjg_result;

typedef struct {
  int32_t column;
  int32_t cmp;      /* FJG_CMP_* */
  int32_t is_column;/* 1: compare against column `rhs_column` (attr = attr form) */
  int32_t rhs_column;
  int64_t constant;
} fjg_predicate;

/* ---- errors ---- */
const char* fjg_last_error(void);
int fjg_abi_version(void);

/* ---- plan compiler (host C++) ----
 * Strings use the plan-file dialect of SPEC.md:171. Output buffers follow the
 * snprintf convention: *needed receives strlen+1; FJG_E_RESOURCE if cap is
 * too small. */
/* run pipeline SPEC.md:475 up to schemas: decompose -> binary2fj ->
 * (factor if FREE) -> (fj_to_gj_plan if GENERIC) -> validate */
int fjg_compile_plan(const char* query_json, int mode, int factor_fixpoint, char* out, size_t cap,
                     size_t* needed);
/* op: "binary2fj" (arg: JSON list of relation names, a left-deep segment),
 * "factor" / "factor_fixpoint" / "fj_to_gj" / "schemas" / "validate" /
 * "gj_order" (arg: FJ plan JSON), "covers" / "vs" / "avs" (arg:
 * {"plan": plan, "k": k}), "decompose" (arg: binary tree JSON),
 * "head_vars" (arg ignored). */
int fjg_plan_op(const char* op, const char* query_json, const char* arg_json, char* out, size_t cap,
                size_t* needed);

/* ---- ingestion ----
 * Header-less CSV of int fields into a row-major host buffer (cap_rows x
 * ncols). *rows = rows in the file (also on FJG_E_RESOURCE when cap_rows is
 * too small). Errors: FJG_E_IO (open), FJG_E_PARSE (row, column), 
 * FJG_E_VALIDATION (field count). Text columns are not supported. */
int fjg_parse_csv(const char* path, int ncols, int32_t* out, uint64_t cap_rows, uint64_t* rows);

/* ---- engine (one per device/stream) ---- */
int fjg_engine_create(int device, fjg_engine** out);
void fjg_engine_destroy(fjg_engine* eng);
/* The engine's cudaStream_t (for event timing by the caller). */
void* fjg_engine_stream(fjg_engine* eng);
/* Wait for all work of the engine's stream. */
int fjg_engine_sync(fjg_engine* eng);

/* ---- relations: immutable columnar int32 tables ---- */
/* Copies host columns to the device (cudaMemcpyAsync per column). */
int fjg_relation_create(fjg_engine* eng, const int32_t* const* host_cols, int ncols, uint64_t nrows,
                        fjg_relation** out);
/* fj::Value is an int64 (value.hpp:31): int64 host columns are staged to the
 * device in chunks and narrowed there to the engine's int32 columns (128-bit
 * loads). FJG_E_VALIDATION, naming the column and the first row, if a value
 * does not fit int32 (wide domains must be dictionary-encoded by the caller;
 * joins only need equality, MIN and the checksum need the values). */
int fjg_relation_create_i64(fjg_engine* eng, const int64_t* const* host_cols, int ncols, uint64_t nrows,
                            fjg_relation** out);
/* Wraps (copy=0: zero-copy alias, caller keeps the memory alive) or copies
 * (copy=1) device columns. */
int fjg_relation_from_device(fjg_engine* eng, const int32_t* const* dev_cols, int ncols, uint64_t nrows,
                             int copy, fjg_relation** out);
/* apply_filter: conjunction of predicates, row order kept. */
int fjg_relation_filter(const fjg_relation* in, const fjg_predicate* preds, int npreds,
                        fjg_relation** out);
uint64_t fjg_relation_rows(const fjg_relation* rel);
int fjg_relation_cols(const fjg_relation* rel);
const int32_t* fjg_relation_device_col(const fjg_relation* rel, int col);
int fjg_relation_download(const fjg_relation* rel, int col, int32_t* host_out);
void fjg_relation_destroy(fjg_relation* rel);

/* ---- multi-GPU partitioning (north_star (c)) ----
 * Hash-partition `in` on column `col` into nparts destinations:
 * out_rel holds the rows grouped by destination (stable within a
 * destination), counts[d] the rows for destination d. */
int fjg_relation_partition(const fjg_relation* in, int col, int nparts, fjg_relation** out_rel,
                           uint64_t* counts);
/* Same, into caller-provided device columns (nrows int32 each), e.g. the send
 * buffers of an NCCL all-to-all. */
int fjg_relation_partition_into(const fjg_relation* in, int col, int nparts, int32_t* const* out_dev_cols,
                                uint64_t* counts);

/* ---- GHT / COLT handle (Fig 5 new/iter/get; SPEC.md:286-339
 * force / iter_batch / estimated_key_count) ----
 * A device COLT over one relation with a caller-given GHT schema: level l keys
 * on the columns level_cols[off_l .. off_l + level_ncols[l]); columns no level
 * names form a final vector level (rows). A subtrie of level l is named by its
 * position range (p, len) in the level's ordering; the root is (0, rows). State
 * persists across calls and queries: force is lazy and idempotent, so a host
 * can own tries and reuse them. Creation does no device work (GHT new = BaseScan). */
typedef struct fjg_colt fjg_colt;
int fjg_colt_create(fjg_engine* eng, const fjg_relation* rel, const int* level_cols, const int* level_ncols,
                    int nlevels, fjg_colt** out);
/* number of levels (the map levels plus the vector level if any column is left) */
int fjg_colt_levels(const fjg_colt* colt);
/* force the n given subtries of map level `level` (level 0:
 * the root; p/len ignored). Already forced subtries are left as they are. */
int fjg_colt_force(fjg_colt* colt, int level, const uint32_t* p, const uint32_t* len, uint64_t n);
/* get (Fig 12: force, then lookup), batched: for key i (arity = the level's
 * key columns, row-major int32) in subtrie (p[i], len[i]) of map level
 * `level`: found[i], and the child subtrie (child_p[i], child_len[i]) of level
 * + 1. Host arrays. */
int fjg_colt_get(fjg_colt* colt, int level, const uint32_t* p, const uint32_t* len, const int32_t* keys, uint64_t n,
                 uint32_t* child_p, uint32_t* child_len, uint8_t* found);
/* iter (Fig 12 on a map: force, then its keys): the distinct keys of subtrie
 * (p, len) of map level `level` in the level's clustered order, with their
 * child subtries; *nkeys receives the count (FJG_E_RESOURCE if > cap). */
int fjg_colt_iter(fjg_colt* colt, int level, uint32_t p, uint32_t len, int32_t* keys_out, uint32_t* child_p,
                  uint32_t* child_len, uint64_t cap, uint64_t* nkeys);
/* iter on a vector / rows of any subtrie: column `col` of the len rows of
 * subtrie (p, len) at `level`, in the subtrie's order (no forcing). */
int fjg_colt_rows(fjg_colt* colt, int level, uint32_t p, uint32_t len, int col, int32_t* out);
/* estimated_key_count: a forced map -> its keys; otherwise
 * (unforced map, vector, BaseScan root) -> its length. Never forces. */
int fjg_colt_estimated_key_count(fjg_colt* colt, int level, uint32_t p, uint32_t len, uint64_t* out);
void fjg_colt_destroy(fjg_colt* colt);

/* ---- multi-GPU execution (north_star (c)) ----
 * The reference is single-threaded with reentrant, disjoint contexts
 * (SPEC.md:354, :447); these calls run one such context per GPU and combine
 * them. One fjg_engine + fjg_comm per rank (process or thread). NCCL is loaded
 * on first use (dlopen of libnccl.so.2; FJG_NCCL_LIB overrides the path). */
#define FJG_COMM_ID_BYTES 128 /* sizeof(ncclUniqueId) */
#define FJG_MAX_VIEWS 16
typedef struct fjg_comm fjg_comm;
typedef struct fjg_sharded fjg_sharded;
/* ncclGetUniqueId: rank 0 creates the id; the caller ships the bytes to every
 * rank over any channel (MPI, a TCP store, a file). */
int fjg_comm_unique_id(void* id_out);
/* ncclCommInitRank on the engine's device; collectives run on the engine's stream. */
int fjg_comm_create(fjg_engine* eng, const void* id, int nranks, int rank, fjg_comm** out);
int fjg_comm_size(const fjg_comm* comm);
int fjg_comm_rank(const fjg_comm* comm);
void fjg_comm_destroy(fjg_comm* comm);
/* A query sharded on its plan's first variable. local_bases: this rank's slice
 * of every base relation (filtered already; caller-owned, kept alive, contents
 * may change between executions); atom_base[a]: base of query atom a (renamed
 * self-joins share one); first_var_col[a]: column of the plan's first variable
 * in atom a, or -1 when the atom does not hold it (then the base is replicated
 * on every rank). query_json / plan_json as fjg_query_create. */
int fjg_sharded_create(fjg_comm* comm, const char* query_json, const char* plan_json,
                       fjg_relation* const* local_bases, int nbases, const int* atom_base,
                       const int* first_var_col, int natoms, fjg_sharded** out);
typedef struct {
  uint64_t local_count_lo, local_count_hi, local_checksum; /* this rank's share */
  uint64_t bytes_sent, bytes_received;                     /* NCCL payload, peers only */
  uint64_t view_rows[FJG_MAX_VIEWS];                       /* rows held after the exchange */
  int32_t nviews;
  int32_t pad_;
  double exchange_ms, reduce_ms;                           /* if collect_timing */
} fjg_multi_info;
/* fjg_execute across the communicator: partition kernel -> one metadata
 * all-gather -> grouped ncclSend/ncclRecv (all-to-all of the partitioned
 * views, all-gather of the replicated ones) -> local execution ->
 * ncclAllReduce of (count, checksum, MIN). `out` holds the GLOBAL count /
 * checksum / MIN and this rank's stats; `info` (optional) the local share and
 * exchange figures. Collective: every rank must call it. Count and
 * factorised-count modes (enumerate is single-GPU). */
int fjg_execute_multi(fjg_sharded* sq, const fjg_exec_options* opts, fjg_result* out, fjg_multi_info* info);
void fjg_sharded_destroy(fjg_sharded* sq);
/* test hook: receive layout of an exchange from gathered metadata
 * meta[src][view][dst]: recv_off[view][src], recv_rows[view]. */
int fjg_exchange_layout(const uint64_t* meta, int nviews, int nranks, int rank, const int* partitioned,
                        uint64_t* recv_off, uint64_t* recv_rows);

/* ---- queries: build phase + join phase ----
 * query_json: {"query":[{"rel":..,"vars":[..]},..], "head": [..] (optional:
 * the output/checksum variable order, default first appearance)}; plan_json: a Free Join
 * plan in the SPEC.md:171 dialect. atom_rels[i] binds query atom i; several
 * atoms may bind the same relation (renamed self-joins) and
 * then share device COLT levels. */
int fjg_query_create(fjg_engine* eng, const char* query_json, const char* plan_json,
                     fjg_relation* const* atom_rels, int natoms, fjg_query** out);
/* One full execution: GHT new (BaseScan) for every atom, then
 * join_vectorized (Fig 13) with lazy COLT forcing; the last node fuses the
 * count/checksum/MIN aggregation (or writes tuples in enumerate mode). */
int fjg_execute(fjg_query* q, const fjg_exec_options* opts, fjg_result* out);
/* Enumerate mode: copy up to cap_rows output tuples (head-variable order,
 * row-major, num_head_vars int32 each, unsorted bag) to host_out. */
int fjg_query_output(fjg_query* q, int32_t* host_out, uint64_t cap_rows, uint64_t* rows);
int fjg_query_num_head_vars(const fjg_query* q);
/* run_segments: the enumerated output as a new device
 * relation (one int32 column per head variable), for use as an atom of the
 * parent segment of a bushy plan. */
int fjg_query_output_relation(fjg_query* q, fjg_relation** out);
void fjg_query_destroy(fjg_query* q);

/* ---- test hooks ---- */
/* TupleHash (value.hpp:61-67) of `ntuples` int64 tuples of `arity` values,
 * computed by a device kernel; used to pin the device hash against the
 * reference KATs. */
int fjg_device_tuple_hash(fjg_engine* eng, const int64_t* host_vals, int arity, uint64_t ntuples,
                          uint64_t* host_out);
uint64_t fjg_host_tuple_hash(const int64_t* vals, int arity);
/* Runs one hand-written device-wide primitive of the build path on seeded
 * data and counts the elements that differ from a host restatement:
 * which = 0 radix sort of (u32 key, u32 value) pairs on key bits [lo, hi)
 * (stable), 1 inclusive u64 sum (+ total), 2 inclusive u32 max-scan,
 * 3 flagged index selection (+ count), 4 exclusive u32 sum. */
int fjg_device_primitive_check(fjg_engine* eng, int which, uint64_t n, int lo, int hi, uint64_t seed,
                               uint64_t* mismatches);

#ifdef __cplusplus
}
#endif

#endif /* FJG_H_ */
