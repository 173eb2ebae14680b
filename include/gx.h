/*
 * gx.h -- C ABI of the B200-native GPUexplore hot path (libgx.so).
 *
 * Plain C types only: pointers, sizes, integer status codes.  One opaque
 * handle per device-resident object.  Every entry point returns
 *   GX_OK (0), GX_EINPUT (1, bad argument / config -- the reference raises
 *   ValueError), GX_ETABLE_FULL (2, mirrors TABLE_FULL / CLI exit 2) or
 *   GX_EINTERNAL (3, CUDA error or invariant violation -- CLI exit 3),
 * the CLI exit codes of the reference (pkg/src/ltsmc/cli.py:28-31), and
 * leaves a message for gx_last_error().
 *
 * The reference has no FFI (it is pure Python); the interface each entry
 * point replaces is cited next to it (paths relative to
 * /root/reference/pkg/src/ltsmc/).  The Python mirror of that interface
 * lives in paper_1801_05857_b200/ and binds these symbols with ctypes; see
 * INTEGRATION.md for the binding a maintainer would add to ltsmc itself.
 *
 * Threading: one host thread drives one handle; calls are ordered on the
 * handle's CUDA stream (0 = legacy default stream).  All device memory is
 * owned by the library.
 */
#ifndef GX_H
#define GX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GX_OK 0
#define GX_EINPUT 1
#define GX_ETABLE_FULL 2
#define GX_EINTERNAL 3

/* slot status values, hashtable.py:35-38 */
#define GX_EMPTY 0
#define GX_CLAIMED 1
#define GX_OCCUPIED_NEW 2
#define GX_OCCUPIED_OLD 3

/* find_or_insert result codes, hashtable.py:41-43 */
#define GX_FOUND 0
#define GX_INSERTED 1
#define GX_TABLE_FULL 2

/* layouts, hashtable.py:45-46 */
#define GX_LAYOUT_PLAIN 0
#define GX_LAYOUT_HALF 1

/* explore outcomes, explore.py:33-35 */
#define GX_COMPLETE 0
#define GX_OUTCOME_TABLE_FULL 1
#define GX_ITERATION_CAP 2

#define GX_DEADLOCK_KEEP 100 /* explore.py:38 */

typedef struct gx_table gx_table;
typedef struct gx_net gx_net;

/* ------------------------------------------------------------------ table */

/* TableConfig (hashtable.py:75-86) + vector length.  mark_word/mark_bit
 * name a bit that no key ever sets (a spare high bit of the packing
 * scheme, statevec.py:41-66); the table then stores keys with that bit
 * set and needs no status read on the probe path (single 32/64/128-bit
 * CAS insert).  mark_word = -1: keys may use every bit, and the table runs
 * the reference's claim/publish protocol on a status byte per slot
 * (hashtable.py:252-267). */
typedef struct gx_table_cfg {
    int32_t bucket_words;       /* 4, 8, 16, 32 */
    int32_t num_hash_functions; /* K >= 1 (<= 64 here) */
    uint64_t capacity_words;    /* num_buckets = capacity_words / bucket_words */
    int32_t layout;             /* GX_LAYOUT_PLAIN / GX_LAYOUT_HALF (resolved) */
    int32_t vector_length;      /* 1..16 */
    uint64_t seed;              /* hash seed, hashtable.py:50 */
    int32_t mark_word;          /* -1: none */
    int32_t mark_bit;           /* 0..31 */
    int32_t flags;              /* GX_TABLE_NO_STATUS: see below */
    int32_t reserved;
} gx_table_cfg;

/* flags: an in-band (mark bit) table for exploration only, without the
 * per-slot status array (saves 1 byte per slot, 12.5% of a bw 32 / vlen 2
 * table).  claim_new / scan_new / dumps / status reads then fail with
 * GX_EINPUT; explore, find_or_put and occupancy work. */
#define GX_TABLE_NO_STATUS 1

/* StateTable.__init__ (hashtable.py:137-201).  Allocates and zeroes device
 * memory.  stream: a cudaStream_t or NULL. */
int gx_table_create(const gx_table_cfg *cfg, void *stream, gx_table **out);
int gx_table_destroy(gx_table *t);
/* Reset to empty (fresh table, same geometry). */
int gx_table_clear(gx_table *t);

/* num_buckets, slots_per_bucket, total_slots (hashtable.py:155-159) */
int gx_table_geometry(const gx_table *t, uint64_t *num_buckets, int32_t *slots_per_bucket,
                      uint64_t *total_slots);
/* (a_i, b_i) pairs and the fold salt (hashtable.py:199-201), for tests */
int gx_table_hash_constants(const gx_table *t, uint64_t *a, uint64_t *b, uint64_t *salt);

/* find_or_insert over a batch (hashtable.py:224-280).  keys: n * vlen
 * words (host memory), codes[n] / handles[n] out (host memory).  Equal
 * keys in one batch agree on one handle and exactly one gets INSERTED.
 * serial != 0 processes the batch one key at a time in order on one warp:
 * the reference's single-threaded placement, handle for handle. */
int gx_find_or_put(gx_table *t, const uint32_t *keys, uint64_t n, uint8_t *codes,
                   int64_t *handles, int32_t serial);
/* Same on device-resident buffers (keys/codes/handles are device
 * pointers; codes/handles may be NULL).  *inserted (host) gets the number
 * of INSERTED results, *full the number of TABLE_FULL results. */
int gx_find_or_put_device(gx_table *t, const uint32_t *d_keys, uint64_t n, uint8_t *d_codes,
                          int64_t *d_handles, uint64_t *inserted, uint64_t *full);

/* gx_find_or_put (concurrent, not serial) with the FINDORPUT kernel timed
 * alone by CUDA events in *kernel_ms (key upload and code download
 * excluded): run_insert_bench's timed region (bench.py:120-202 times only
 * the insert loop). */
int gx_find_or_put_timed(gx_table *t, const uint32_t *keys, uint64_t n, uint8_t *codes, double *kernel_ms);

/* claim_new (hashtable.py:296-313): claimed[i] = 1 iff this call moved
 * handles[i] NEW -> OLD.  Repeated handles in one batch: exactly one wins. */
int gx_claim_new(gx_table *t, const int64_t *handles, uint64_t n, uint8_t *claimed);

/* scan_new (hashtable.py:315-324): handles of NEW slots in buckets
 * [first, last), ascending (bucket-major).  Call with out = NULL to get the
 * count in *count; then with capacity >= count. */
int gx_scan_new(gx_table *t, uint64_t first, uint64_t last, int64_t *out, uint64_t capacity,
                uint64_t *count);

/* occupancy (hashtable.py:326-331): occupied and new counts. */
int gx_occupancy(gx_table *t, uint64_t *occupied, uint64_t *new_count);

/* slot_status / read_slot over a batch of handles (hashtable.py:335-342). */
int gx_read_slots(gx_table *t, const int64_t *handles, uint64_t n, uint8_t *status,
                  uint32_t *words);

/* occupied_vectors / dump_rows (hashtable.py:344-365): all slots with
 * status >= NEW in bucket-major order.  out arrays sized by a first call
 * with NULLs (count in *count). */
int gx_dump(gx_table *t, int64_t *handles, uint8_t *status, uint32_t *words, uint64_t capacity,
            uint64_t *count);

/* Order-independent multiset digest of the occupied slots: the set-level
 * counterpart of the reference's sorted state dump (statevec.py:93-100,
 * explore.py:376-383), for state spaces too large to dump.  Per occupied
 * slot, over its first `words` words w_0..w_{n-1} (the packing scheme's
 * vector length; a padding word is left out):
 *     h = 0x6A09E667F3BCC908 ^ n;  h = mix64(h ^ w_i) for each i
 * with mix64 the splitmix64 finaliser (hashtable.py:114-120 without the
 * increment).  out[0] = count, out[1] = sum of h mod 2^64, out[2] = xor of
 * h.  Shards combine by adding counts and sums and xor-ing xors. */
int gx_table_digest(gx_table *t, int32_t words, uint64_t *out);

/* The canonical state dump's order (statevec.py:93-100, dump_states: packed
 * vectors sorted lexicographically over their words) computed on the
 * device: the first `words` words of every occupied slot, sorted (stable
 * LSD radix sort), copied to out[capacity * words].  *count = occupied
 * slots; out = NULL only counts.  Works without a status array. */
int gx_dump_sorted(gx_table *t, int32_t words, uint32_t *out, uint64_t capacity, uint64_t *count);

/* --------------------------------------------------------------- network */

/* A Network (network.py:43-62) flattened to device CSR by the host
 * (paper_1801_05857_b200/network.py: to_csr).  All arrays are u32; the
 * layout of each is documented in DESIGN.md ("network CSR"). */
typedef struct gx_network_csr {
    uint32_t nproc, nrules, vlen, reserved;
    const uint32_t *proc;  uint64_t n_proc;   /* nproc x {word, shift, mask, qbase}       */
    const uint32_t *qtab;  uint64_t n_qtab;   /* per (proc, state) {off, ndst, count, trig} */
    const uint32_t *im_dst; uint64_t n_im_dst;/* independent-move destinations            */
    const uint32_t *trig;  uint64_t n_trig;   /* [n, rule ids...] lists                    */
    const uint32_t *rules; uint64_t n_rules;  /* nrules x {npart, part_off, dedup_off, res} */
    const uint32_t *parts; uint64_t n_parts;  /* participants {rq_base, word, shift, mask} */
    const uint32_t *rq;    uint64_t n_rq;     /* per (rule, part, state) {off, n}          */
    const uint32_t *rdst;  uint64_t n_rdst;   /* rule destinations                         */
    const uint32_t *dedup; uint64_t n_dedup;  /* [n, earlier rule ids...] lists            */
    const uint32_t *initial;                  /* packed initial state, vlen words         */
} gx_network_csr;

/* build_network (network.py:65-181) result, uploaded once. */
int gx_net_create(const gx_network_csr *csr, void *stream, gx_net **out);
int gx_net_destroy(gx_net *n);

/* expand (network.py:184-238) over a batch of packed states (host memory):
 * counts[i] = transition count, nsucc[i] = successors emitted (self-loops
 * of independent moves are not emitted; rule targets deduplicated by
 * (result, target)); succ gets the packed successors back to back when
 * non-NULL (capacity in vectors).  Test / debug entry point. */
int gx_expand(gx_net *n, const uint32_t *states, uint64_t nstates, uint64_t *counts,
              uint32_t *nsucc, uint32_t *succ, uint64_t capacity, uint64_t *total);

/* ---------------------------------------------------------------- explore */

/* ExploreConfig (explore.py:47-62) minus the CPU worker knobs. */
typedef struct gx_explore_cfg {
    int32_t detect_deadlocks;
    int32_t filter_log2;        /* > 0: GPU-wide L2-resident dedup filter of 2^filter_log2
                                   entries (8 B each) in front of the table; 0 = off */
    int64_t max_iterations;     /* < 0: none; else stop once rounds >= it (explore.py:256-261) */
    uint64_t frontier_capacity; /* vectors; 0 = size from free device memory */
    int32_t probe_group;        /* 0 = auto; else lanes per bucket probe (1,2,4,8) */
    int32_t cache_slots;        /* per-block shared-memory dedup cache entries (the
                                   reference's LocalCache size, explore.py:91-144);
                                   rounded down to a power of two, capped at
                                   GX_CACHE_MAX_SLOTS; < 32 = off; vlen <= 2 only */
} gx_explore_cfg;

#define GX_CACHE_MAX_SLOTS 8192

/* ExplorationReport (explore.py:65-88) */
typedef struct gx_report {
    uint64_t states, transitions, expanded, iterations, deadlocks_total;
    int32_t outcome;            /* GX_COMPLETE / GX_OUTCOME_TABLE_FULL / GX_ITERATION_CAP */
    int32_t deadlocks_kept;     /* <= GX_DEADLOCK_KEEP */
    double device_ms;           /* CUDA-event time of the level loop */
    uint64_t levels_launched;   /* expand kernels launched */
    uint64_t max_frontier;      /* widest BFS level */
    uint64_t kernels;           /* all kernels launched by this call */
    double level_ms;            /* sum of the level kernels' CUDA-event durations */
    uint64_t probes;            /* successors probed (FINDORPUT operations) */
} gx_report;

/* explore (explore.py:300-395): level-synchronous BFS from the network's
 * initial state into table t (cleared first).  deadlocks: GX_DEADLOCK_KEEP
 * * vlen words (host), the smallest deadlock states in packed form
 * (composite-order sorting is done by the caller).  Table statuses are
 * left as the reference leaves them: expanded states OLD, states of the
 * last unexpanded level NEW. */
int gx_explore(gx_net *n, gx_table *t, const gx_explore_cfg *cfg, gx_report *report,
               uint32_t *deadlocks);

/* ------------------------------------------------- per-level primitives */
/* For the hash-owner sharded multi-GPU driver (paper_1801_05857_b200/
 * distributed.py): expand one level's frontier (device buffer of n packed
 * states) and bin every successor by owner rank = owner_of(fold) across
 * `ranks` peers into d_out (device, capacity vectors); d_counts[ranks]
 * (device u64) gets per-owner counts, successors of owner r occupy
 * [d_offsets[r], d_offsets[r] + d_counts[r]) after the call (d_offsets
 * device u64[ranks]).  *transitions / *deadlocks (host) get the level's
 * totals; deadlock states append to the handle's deadlock buffer. */
int gx_expand_route(gx_net *n, const gx_table *t, const uint32_t *d_frontier, uint64_t nfront,
                    int32_t ranks, uint32_t *d_out, uint64_t capacity, uint64_t *d_counts,
                    uint64_t *d_offsets, uint64_t *transitions, uint64_t *deadlocks,
                    int32_t detect_deadlocks);
/* FINDORPUT of n received vectors; INSERTED ones are appended to
 * d_next (device, capacity vectors); *n_next (host) = appended count. */
int gx_insert_append(gx_table *t, const uint32_t *d_keys, uint64_t n, uint32_t *d_next,
                     uint64_t capacity, uint64_t *n_next, int32_t *table_full);
/* owner_of for a batch of host vectors (tests of the routing function) */
int gx_owner_of(const gx_table *t, const uint32_t *keys, uint64_t n, int32_t ranks,
                int32_t *owner);

/* ------------------------------------------- fused sharded exploration */
/* Hash-owner sharding across GPUs (the reference's
 * nearest analogue is the bucket-range worker split, explore.py:284-286).
 * One shard per GPU: shard `rank` owns the states with
 * owner_of(fold) == rank and keeps them in table t.  Per BFS level the
 * driver calls gx_shard_expand (expand the local frontier; successors owned
 * by peers are stored straight into the peers' inboxes over NVLink,
 * locally owned ones are FINDORPUT at once), then a barrier across ranks
 * (e.g. an all_reduce), then gx_shard_absorb (FINDORPUT the inbox; stats
 * of the level), then reduces the stats to decide termination exactly as
 * explore.py:255-265 does.  Only in-band (mark bit) tables are supported. */
typedef struct gx_shard gx_shard;
#define GX_IPC_HANDLE_BYTES 64
/* stats[] of gx_shard_absorb: per-level claims / new, then cumulative */
#define GX_SH_CLAIMS 0
#define GX_SH_NEW 1
#define GX_SH_TRANSITIONS 2
#define GX_SH_DEADLOCKS 3
#define GX_SH_TABLE_FULL 4
#define GX_SH_OVERFLOW 5
#define GX_SH_ROUTED 6
#define GX_SH_PROBES 7
#define GX_SH_N 8
int gx_shard_create(gx_net *n, gx_table *t, int32_t rank, int32_t world, uint64_t inbox_capacity,
                    uint64_t frontier_capacity, int32_t cache_slots, int32_t filter_log2,
                    gx_shard **out);
int gx_shard_destroy(gx_shard *s);
/* CUDA IPC handle of this shard's inbox (GX_IPC_HANDLE_BYTES bytes) */
int gx_shard_ipc_handle(gx_shard *s, uint8_t *out);
/* map every peer's inbox (world handles, rank order; own entry ignored;
 * an all-zero handle marks a peer in this process: gx_shard_link it) */
int gx_shard_connect(gx_shard *s, const uint8_t *handles);
/* point s at the inbox of a peer shard living in the same process */
int gx_shard_link(gx_shard *s, const gx_shard *peer);
/* all shards of one process (one GPU or several): connect them directly */
int gx_shard_connect_local(gx_shard *const *shards, int32_t world);
/* clear the shard's table; insert the initial state if this rank owns it */
int gx_shard_begin(gx_shard *s, int32_t owns_initial, int32_t detect_deadlocks, int32_t *table_full);
int gx_shard_expand(gx_shard *s);
int gx_shard_absorb(gx_shard *s, uint64_t *stats);
/* The same level in frontier chunks, so inboxes stay bounded: for each
 * chunk every shard calls gx_shard_expand_range (states [begin, begin +
 * count) of its current frontier), a barrier, then gx_shard_absorb_chunk;
 * after the last chunk gx_shard_end_level returns the level's stats.
 * gx_shard_frontier gives the current frontier size. */
int gx_shard_expand_range(gx_shard *s, uint64_t begin, uint64_t count);

/* Partitioned dedup mode (gx_part.cuh).  dedup != 0: the
 * expansion routes EVERY successor (own ones too) into the owner shard's
 * inbox, split into `nsub` hash sub-partitions; the absorb step filters each
 * sub-partition through a 2^set_log2 x 32-byte L2-resident set so that only
 * the first occurrence of a key in the chunk probes the table.  Results are
 * those of the fused mode (FINDORPUT is idempotent, hashtable.py:224-280).
 * gx_shard_set_partitions sets nsub for the next chunk (same on every
 * shard; world * nsub <= 128); gx_shard_chunk_status (after the expansion,
 * synchronising) gives out[0] = this shard's inbox-overflow flag, out[1] =
 * successors routed so far this run, out[2] = states expanded so far; when
 * any shard overflowed, every shard calls gx_shard_rollback (the chunk's
 * counters and routed keys are discarded) and the driver re-expands the
 * chunk in smaller pieces. */
/* Hash-partitioned isolated FINDORPUT benchmark (configs[1] at N GPUs; the
 * reference's run_insert_bench, bench.py:120-202, over shards): each shard
 * runs positions [first, first + count) of one global duplication sequence
 * (total ops over total / duplication unique keys, generated on the
 * device), stores the keys owned by peers into their inboxes and
 * FINDORPUTs its own (gx_shard_bench_route); after a barrier every shard
 * calls gx_shard_absorb_chunk; gx_shard_bench_result then gives out[0] =
 * keys INSERTED into this shard, out[1] = TABLE_FULL seen, out[2] =
 * FINDORPUTs run here, out[3] = keys routed to peers, out[4] = an inbox
 * overflowed, and *ms = the CUDA-event time of this shard's kernels.  Start
 * each run with gx_shard_begin(s, 0, 0, &full). */
int gx_shard_bench_route(gx_shard *s, uint64_t total, uint64_t duplication, uint64_t seed, int32_t key_bits,
                         uint64_t first, uint64_t count);
int gx_shard_bench_result(gx_shard *s, uint64_t *out, double *ms);

int gx_shard_set_mode(gx_shard *s, int32_t dedup, int32_t set_log2);

/* Pipelined fused levels: the inbox is split in two halves; the launch for
 * chunk c of a level (gx_shard_expand_range) routes into the peers' half
 * c & 1 and, in the same kernel, FINDORPUTs the keys routed here during
 * chunk c - 1 (half (c - 1) & 1), so the memory-bound absorb work overlaps
 * the issue-bound expansion.  Protocol per level: for each chunk every
 * shard calls gx_shard_expand_range, then a barrier; after the last chunk
 * every shard calls gx_shard_absorb_chunk once (the last half), then
 * gx_shard_end_level. */
int gx_shard_set_pipeline(gx_shard *s, int32_t on);
int gx_shard_set_partitions(gx_shard *s, uint32_t nsub);
int gx_shard_chunk_status(gx_shard *s, uint64_t *out);
int gx_shard_rollback(gx_shard *s);
int gx_shard_absorb_chunk(gx_shard *s);
int gx_shard_end_level(gx_shard *s, uint64_t *stats);
int gx_shard_frontier(const gx_shard *s, uint64_t *n);
/* finalise statuses; local report (states, transitions, expanded,
 * deadlocks of this shard; level_ms = its device time) */
int gx_shard_finish(gx_shard *s, gx_report *report, uint32_t *deadlocks);

/* ------------------------------------------------------------ benchmark */
/* Isolated FINDORPUT benchmark (bench.py:120-202 protocol on device
 * generated keys): `total` operations, each unique vector repeated
 * `duplication` times, globally shuffled by a keyed bijection.  Keys are
 * random words masked to key_bits bits per word (32 = full words).
 * ms = CUDA-event time of the insert kernel(s) only; found/inserted
 * counted on device. */
int gx_bench_find_or_put(gx_table *t, uint64_t total, uint64_t duplication, uint64_t seed,
                         int32_t key_bits, int32_t probe_group, double *ms, uint64_t *found,
                         uint64_t *inserted, uint64_t *full);

/* Same, with the unique rows numbered from row_base (so successive calls
 * can fill a table step by step with fresh keys: the fill-factor sweep);
 * *loads (may be NULL) = bucket loads issued (probe_group 0 only), so
 * loads / total is the mean number of buckets a FINDORPUT touched. */
int gx_bench_find_or_put_rows(gx_table *t, uint64_t total, uint64_t duplication, uint64_t row_base,
                              uint64_t seed, int32_t key_bits, int32_t probe_group, double *ms,
                              uint64_t *found, uint64_t *inserted, uint64_t *full, uint64_t *loads);

/* Random-access HBM roofline R(g) (SURVEY.md §8(d) denominator; no
 * reference counterpart): `reads` aligned random reads of `granularity`
 * bytes (16/32/64/128 = one bucket of bw 4/8/16/32) over a fresh device
 * buffer of buffer_bytes (>> L2), best of `repeats` CUDA-event timed
 * launches after one warm-up.  with_cas: also a 64-bit CAS on the first
 * 8 bytes of every segment read as empty (the FINDORPUT insert path). */
int gx_random_access_bench(uint64_t buffer_bytes, int32_t granularity, uint64_t reads,
                           int32_t with_cas, int32_t repeats, double *ms_best, double *gbs_best);
/* Same on a buffer from allocator alloc_kind: 0 cudaMalloc, 1 VMM
 * (cuMemCreate/cuMemMap at the recommended granularity, returned in
 * *alloc_granularity), 2 stream-ordered pool (TLB-reach experiments). */
int gx_random_access_bench_alloc(uint64_t buffer_bytes, int32_t granularity, uint64_t reads,
                                 int32_t with_cas, int32_t repeats, int32_t alloc_kind,
                                 double *ms_best, double *gbs_best, uint64_t *alloc_granularity);

/* ----------------------------------------------------------------- misc */
/* Insertion protocol chosen at create time: 0 = mark bit (single CAS),
 * 1 = status-byte claim/publish. */
int gx_table_mode(const gx_table *t);
/* Deadlock states recorded by the last gx_expand_route call (device
 * buffer, at most 65536 kept); *count gets the number recorded. */
int gx_net_deadlocks(gx_net *n, uint32_t *out, uint64_t capacity, uint64_t *count);
const char *gx_last_error(void);
/* Number of kernels this library has launched (process-wide counter). */
uint64_t gx_kernel_launches(void);
/* Device properties used for grid sizing. */
int gx_device_info(int32_t *sm_count, uint64_t *free_bytes, uint64_t *total_bytes);
/* Synchronise the handle's stream and report asynchronous errors. */
int gx_sync(void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GX_H */
