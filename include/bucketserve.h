/*
 * bucketserve.h — C-ABI of the B200-native BucketServe scheduling hot path.
 *
 * The reference (bucketsim, /root/reference/pkg/src/bucketsim) has no FFI: its
 * "operator API" is a set of Python classes.  Every entry point below replaces
 * one of those Python operations and cites the reference code it stands in for.
 * The Python host package (paper_2507_17120_b200) binds these with ctypes; the
 * binding a bucketsim maintainer would add is shown in INTEGRATION.md.
 *
 * Conventions
 *   - Plain C types only.  All array arguments are DEVICE pointers (CUDA global
 *     memory) unless the name says `host_`.  The caller owns every I/O buffer;
 *     the context owns scratch memory and nothing else.
 *   - Every call is asynchronous on the given CUDA stream (`cudaStream_t` passed
 *     as void*; NULL = legacy default stream).  Results are valid after the
 *     stream is synchronised.
 *   - No C++ exception crosses the boundary.  Every function returns an int
 *     status (BS_OK = 0, negative on failure); bs_last_error() gives the text.
 *     Data-dependent errors that can only be seen on the device (a length
 *     outside [0, l_max), a zero mean length) are latched into
 *     bs_summary.flags and surface when the caller reads the summary.
 *   - One context per host thread / stream (the reference is single-writer,
 *     bucket_manager.py:73-77, batch_controller.py:70-71).
 *
 * Semantics (window mode): one call schedules a window of N pending requests,
 * given in arrival order (index = arrival rank; traces are arrival-sorted with
 * ids in file order on ties, workload.py:389-399):
 *   K1 histogram        per-(class, length) counts         bucket_manager.py:31-32,126-127
 *   K2 boundaries       Alg. 1 split/merge on prefix sums   bucket_manager.py:133-191
 *                       + n_max (current_n_max)             batch_controller.py:93-104
 *   K3 assign           bucket id per request               bucket_manager.py:110-131
 *   K4 order            stable (bucket, class, policy key)  batch_controller.py:33-41,154-156
 *   K5 size             greedy memory-safe admission        batch_controller.py:136-191
 *   K6 pack             padded [n, pitch] int32 tokens + u8 mask + waste_ratio
 *                       (no reference; stats restate memory_model.py:92-100)
 */
#ifndef BUCKETSERVE_H
#define BUCKETSERVE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BS_ABI_VERSION 2

/* ---- status codes (mapped by the Python shim to the reference exceptions) -- */
#define BS_OK                 0
#define BS_ERR_INVALID_ARG   -1  /* ValueError   (bucket_manager.py:81-84, memory_model.py:69-76) */
#define BS_ERR_CONFIG        -2  /* ConfigError  (errors.py:4-5)                                 */
#define BS_ERR_CUDA          -3  /* RuntimeError: CUDA runtime failure                           */
#define BS_ERR_CAPACITY      -4  /* a caller buffer is too small (size in bs_last_error)         */
#define BS_ERR_NOT_BUILT     -5  /* library built without device code for this GPU              */

/* ---- device-latched flags in bs_summary.flags ------------------------------- */
#define BS_FLAG_LEN_RANGE     0x1  /* input_len outside [0, l_max): ValueError, bucket_manager.py:112-115 */
#define BS_FLAG_CLASS_RANGE   0x2  /* class id >= n_classes: ValueError                                   */
#define BS_FLAG_ZERO_MEAN     0x4  /* all queued lengths 0: token_budget // 0.0 raises ZeroDivisionError  */
#define BS_FLAG_CHANGES_TRUNC 0x8  /* change log exceeded changes_cap (count still exact)                 */
#define BS_FLAG_PACK_CAPACITY 0x10 /* packed output exceeded out_capacity; batches beyond it not packed   */
#define BS_FLAG_NONPOS_LEN    0x20 /* a batch holds a length < 1: waste_ratio raises, memory_model.py:96  */
#define BS_FLAG_BATCH_CAP     0x40 /* more batches than batches_cap                                       */
#define BS_FLAG_BAD_EDGES     0x80 /* init_edges not strictly increasing from 0 to l_max: ValueError      */
#define BS_FLAG_DISPATCH_RANGE 0x100 /* dispatch keys out of range (token mass >= 2^43 or > 2^17 buckets) */
#define BS_FLAG_PEER_TIMEOUT  0x200 /* a peer rank's histogram did not arrive within the timeout   */

/* ---- enums ------------------------------------------------------------------ */
/* Dispatch order inside one (bucket, class) segment, batch_controller.py:33-41.
 * EARLIEST_ARRIVAL and FCFS share one rule (batch_controller.py:39-40).          */
enum bs_policy { BS_POLICY_FCFS = 0, BS_POLICY_SJF = 1, BS_POLICY_LJF = 2 };
/* batch_controller.py:28-30 / _footprint :136-139 */
enum bs_accounting { BS_ACCOUNTING_PADDED = 0, BS_ACCOUNTING_EXACT = 1 };
/* StructuralChange.kind, bucket_manager.py:56-63 */
enum bs_change_kind { BS_CHANGE_SPLIT = 1, BS_CHANGE_MERGE = 2, BS_CHANGE_SKIP = 3 };
/* per-request outcome in bs_window_out.req_batch when not admitted */
#define BS_REQ_PENDING  (-1)   /* left in its bucket (drain stopped before it) */
#define BS_REQ_REJECTED (-2)   /* OversizeRejection, batch_controller.py:44-67,165-169 */

#define BS_MAX_CLASSES 8
#define BS_PACK_ALIGN  16      /* packed row pitch = round_up(max_input_len, 16) tokens: every
                                  row starts on a 64-byte boundary (tokens) / 16 bytes (mask), so
                                  16-token mask words never straddle rows */

/* ---- parameter block (host memory) ------------------------------------------ */
typedef struct bs_window_params {
  int32_t l_max;             /* ModelConfig.max_seq_len: lengths live in [0, l_max)       */
  int32_t n_classes;         /* 1..BS_MAX_CLASSES; class 0 dispatches first                */
  int32_t policy[BS_MAX_CLASSES]; /* bs_policy per class (ref: ONLINE=EARLIEST_ARRIVAL,
                                     OFFLINE=offline_policy, pd_sim.py:315-320)            */
  double  split_threshold;   /* theta in (0, 1], bucket_manager.py:83                      */
  int32_t adjust;            /* 1: run adjust_buckets passes; 0: keep init edges
                                (continuous proxy, pd_sim.py:308-313)                      */
  int32_t max_passes;        /* <= 0: until a pass yields no split (window fixpoint)       */
  int64_t n_max;             /* <= 0: derive with current_n_max from the histogram         */
  int64_t kv_bytes_per_token;/* ModelConfig.kv_bytes_per_token, memory_model.py:36-39      */
  int64_t current_safe;      /* BatchController.current_safe (bytes), batch_controller.py:78 */
  int64_t pledged;           /* form_batch(pledged=...), batch_controller.py:150           */
  int32_t accounting;        /* bs_accounting                                              */
  int32_t truncate;          /* 1: len >= l_max -> l_max-1 (pd_sim.py:382-383); 0: flag    */
  int32_t pad_id;            /* token id written into padding                              */
  int32_t dispatch;          /* 1: also compute the simulator's global dispatch order (f3,
                                bs_dispatch) inside bs_window_schedule / _from_hist        */
} bs_window_params;

/* ---- one batch descriptor (device memory), BatchPlan, batch_controller.py:44-56 */
typedef struct bs_batch {
  int32_t segment;        /* bucket * n_classes + class                               */
  int32_t start;          /* first sorted position visited by this form_batch call    */
  int32_t end;            /* one past the last sorted position it consumed            */
  int32_t n;              /* admitted requests (len(BatchPlan))                       */
  int32_t max_input_len;  /* BatchPlan.max_input_len                                  */
  int32_t pitch;          /* round_up(max_input_len, BS_PACK_ALIGN)                   */
  int64_t token_sum;      /* BatchPlan.token_sum                                      */
  int64_t footprint;      /* BatchPlan.footprint (bytes, accounting mode)             */
  int64_t out_offset;     /* element offset of row 0 in the packed token/mask buffers */
  double  waste;          /* waste_ratio(lengths), memory_model.py:92-100             */
  int64_t row_base;       /* admitted rows of the window before this batch            */
} bs_batch;               /* 64 bytes */

/* ---- window summary (device memory) ----------------------------------------- */
typedef struct bs_summary {
  int64_t n_requests;     /* N in the window (this rank)                              */
  int64_t total_global;   /* requests counted by the (possibly all-reduced) histogram */
  int64_t sum_len_global; /* sum of lengths in that histogram                         */
  int64_t n_max;          /* split floor used by adjust_buckets                       */
  int64_t k_buckets;      /* number of buckets after adjustment                       */
  int64_t n_changes;      /* StructuralChange records produced                        */
  int64_t n_passes;       /* adjust_buckets passes executed                            */
  int64_t n_batches;
  int64_t n_rejected;
  int64_t n_pending;
  int64_t admitted_tokens;/* sum of admitted lengths                                  */
  int64_t padded_tokens;  /* sum over batches of n * max_input_len                    */
  int64_t packed_elems;   /* sum over batches of n * pitch (packed buffer extent)     */
  int64_t peak_footprint; /* max BatchPlan.footprint                                  */
  double  waste_sum;      /* sum of per-batch waste_ratio                             */
  int64_t sort_passes;    /* radix passes run by K4                                   */
  int64_t flags;          /* BS_FLAG_* bits                                           */
  int64_t n_dispatched;   /* plans in the dispatch sequence (bs_dispatch; else 0)     */
  int64_t reserved[14];
} bs_summary;             /* 256 bytes */

typedef struct bs_ctx bs_ctx;

/* ---- context ------------------------------------------------------------------ */
/* Allocates scratch for windows of up to max_n requests, lengths < l_max_cap and
 * up to max_classes classes on `device`. */
int  bs_create(bs_ctx** ctx, int device, int64_t max_n, int32_t l_max_cap, int32_t max_classes);
int  bs_destroy(bs_ctx* ctx);
const char* bs_last_error(const bs_ctx* ctx);  /* ctx may be NULL: last global error */
int  bs_abi_version(void);
/* bytes of device scratch held by ctx */
int64_t bs_scratch_bytes(const bs_ctx* ctx);

/* ---- K1: histogram ---------------------------------------------------------------
 * hist_out[c * l_max + x] = #{i : cls[i] == c, min(len[i], l_max-1 if truncate) == x}
 * Replaces the per-bucket request/short counting of bucket_manager.py:31-32,126-127
 * and the O(N) mean in current_n_max (batch_controller.py:100-104).
 * hist_out is zeroed by the call.  summary (may be NULL) receives n_requests/flags. */
int bs_histogram(bs_ctx* ctx, const int32_t* len, const uint8_t* cls, int64_t n,
                 const bs_window_params* p, uint32_t* hist_out, bs_summary* summary,
                 void* stream);

/* ---- K2: boundaries ------------------------------------------------------------
 * BucketSet.adjust_buckets (bucket_manager.py:133-191) run for up to max_passes
 * passes (<= 0: until a pass yields no split) from init_edges (NULL: the single
 * bucket [0, l_max), bucket_manager.py:87) on the counts in hist_global (for
 * multi-GPU windows: the all-reduced histogram, identical on every rank).
 * edges_out[0..k] (device, capacity l_max+1); k and n_max land in summary.
 * changes_out: int32[4] records (kind, parent_low, parent_up, midpoint|-1), in
 * the reference's emission order, capacity changes_cap records.
 * Also prepares the internal lookup tables used by bs_assign/bs_order, so it must
 * precede them on the same ctx.  init_edges is a device array of k_init+1 edges. */
int bs_boundaries(bs_ctx* ctx, const uint32_t* hist_local, const uint32_t* hist_global,
                  const bs_window_params* p, const int32_t* init_edges, int32_t k_init,
                  int32_t* edges_out, int32_t* changes_out, int32_t changes_cap,
                  bs_summary* summary, void* stream);

/* ---- K3: assign -------------------------------------------------------------------
 * bucket_out[i] = index of the bucket whose [low, up) holds len[i]; the value
 * BucketSet.assign returns (bucket_manager.py:110-131).  Uses the tables of the
 * last bs_boundaries call on ctx. */
int bs_assign(bs_ctx* ctx, const int32_t* len, int64_t n, const bs_window_params* p,
              int32_t* bucket_out, void* stream);

/* ---- K4: order --------------------------------------------------------------------
 * perm_out: the window's requests in drain order — bucket ascending, then class
 * ascending, then order_requests(policy[class]) (batch_controller.py:33-41), ties
 * by arrival rank.  seg_off_out[s] (s = bucket*n_classes+class, capacity
 * l_max*n_classes+1) = first sorted position of segment s; seg_off_out[K*C] = N.
 * bucket_out (may be NULL) receives the K3 result as a side product. */
int bs_order(bs_ctx* ctx, const int32_t* len, const uint8_t* cls, int64_t n,
             const bs_window_params* p, int32_t* perm_out, int32_t* seg_off_out,
             int32_t* bucket_out, bs_summary* summary, void* stream);

/* ---- K5: size ---------------------------------------------------------------------
 * Drains every segment with BatchController.form_batch semantics
 * (batch_controller.py:141-191): oversize requests are rejected, batches are the
 * longest policy-ordered prefixes within headroom = current_safe - pledged, the
 * drain of a segment stops at the first call that admits nothing.
 * batches_out: capacity batches_cap; count in summary->n_batches.
 * req_batch_out[i]: batch index, BS_REQ_PENDING or BS_REQ_REJECTED; req_row_out[i]:
 * row inside its batch (-1 if none).  out_offset of each batch is the exclusive
 * prefix of n * pitch in emission order.  perm / seg_off must be the last bs_order
 * result on ctx (its sorted slots give each position's segment and SJF/LJF length). */
int bs_size(bs_ctx* ctx, const int32_t* len, const int32_t* perm, const int32_t* seg_off,
            int64_t n, const bs_window_params* p, bs_batch* batches_out, int32_t batches_cap,
            int32_t* req_batch_out, int32_t* req_row_out, bs_summary* summary, void* stream);

/* ---- K6: pack ------------------------------------------------------------------------
 * For batches [batch_begin, batch_end) (batch_end < 0: all), writes row q of batch b —
 * the q-th admitted request i of that form_batch call — as
 * out_tokens[out_offset + q*pitch + t] = tokens[tok_off[i] + t] for t < len_i, pad_id
 * beyond, and out_mask (1 for real tokens, 0 for padding; may be NULL).  Offsets are
 * relative to the first packed batch of the call (chunked packing into a reusable
 * buffer); out_capacity is in elements.  Uses the row map of the last bs_size call on
 * ctx.  out_tokens must be 16-byte aligned, out_mask 4-byte aligned.  With both 16-byte
 * aligned (the usual case) the bulk-staged kernel runs: the output is cut into
 * 1024-token chunks filled in shared memory by bulk copies (rows whose tokens start
 * 16-byte aligned, i.e. tok_off[i] % 4 == 0 for an aligned store; other rows by scalar
 * loads) and stored by bulk copies; otherwise a 128-bit register stream. */
int bs_pack(bs_ctx* ctx, const int32_t* len, const int32_t* perm, const int64_t* tok_off,
            const int32_t* tokens, const bs_window_params* p, const bs_batch* batches,
            int64_t batch_begin, int64_t batch_end, int32_t* out_tokens, uint8_t* out_mask,
            int64_t out_capacity, bs_summary* summary, void* stream);

/* ---- K7: dispatch order ----------------------------------------
 * The order in which the simulator would hand the window's batches to prefill:
 * Simulator._next_plan (pd_sim.py:448-462) repeated while it makes progress — per
 * call, classes in priority order, BatchController.select_bucket
 * (batch_controller.py:106-134: class 0 the bucket holding the oldest queued request
 * of the class, other classes the largest queued token mass of the class, ties to the
 * lower bucket, zero mass never) then form_batch on it; the first plan ends the call.
 * emit_order[t] = batch of the t-th plan (t < summary->n_dispatched); batch_emit[b] =
 * t, or -1 for a batch the loop never forms (its bucket is never selected again: a
 * blocked drain under pledged memory, or zero token mass).  Requests of calls the
 * loop never reaches are rewritten to BS_REQ_PENDING in req_batch / req_row and the
 * summary's n_rejected / n_pending follow.  Uses the drain of the last bs_size call
 * on ctx (same perm / seg_off / batches), which must have been made with
 * p->dispatch = 1 (it then also records the per-call keys K7 sorts). */
int bs_dispatch(bs_ctx* ctx, const int32_t* perm, const int32_t* seg_off, int64_t n,
                const bs_window_params* p, const bs_batch* batches, int32_t batches_cap,
                int32_t* req_batch, int32_t* req_row, int32_t* emit_order, int32_t* batch_emit,
                bs_summary* summary, void* stream);

/* ---- fused window ------------------------------------------------------------------
 * K1..K6 (+ K7 when p->dispatch) in one call on one stream.  Single rank: the local
 * histogram is the global one.  Sharded window: attach NCCL once (bs_nccl_connect /
 * bs_set_nccl) or connect the contexts' peer memory once (bs_peer_*) and call
 * bs_window_schedule, which runs C1 between K1 and K2 into io->hist_global; or call
 * bs_histogram, all-reduce the histogram with any collective, then
 * bs_window_from_hist on every rank. */
typedef struct bs_window_io {
  /* inputs */
  const int32_t* len;         /* [n]  */
  const uint8_t* cls;         /* [n]  */
  const int64_t* tok_off;     /* [n+1] or NULL (no pack) */
  const int32_t* tokens;      /* token store or NULL     */
  int64_t        n;
  const int32_t* init_edges;  /* NULL = [0, l_max] */
  int32_t        k_init;
  int32_t        changes_cap;
  int32_t        batches_cap;
  int32_t        reserved0;
  int64_t        out_capacity;/* elements in out_tokens / out_mask */
  /* outputs (device; any may be NULL except where noted) */
  uint32_t*      hist;        /* [n_classes * l_max]  required */
  const uint32_t* hist_global;/* NULL = hist (single rank); with a peer-connected ctx
                                 bs_window_schedule writes the reduced histogram here */
  int32_t*       edges;       /* [l_max + 1]          required */
  int32_t*       changes;     /* [changes_cap * 4]             */
  int32_t*       bucket;      /* [n]                           */
  int32_t*       perm;        /* [n]                  required */
  int32_t*       seg_off;     /* [l_max*n_classes+1]  required */
  bs_batch*      batches;     /* [batches_cap]        required */
  int32_t*       req_batch;   /* [n]                  required */
  int32_t*       req_row;     /* [n]                  required */
  int32_t*       out_tokens;  /* [out_capacity]                */
  uint8_t*       out_mask;    /* [out_capacity]                */
  bs_summary*    summary;     /* required */
  int32_t*       emit_order;  /* [batches_cap] dispatch sequence (p->dispatch)  */
  int32_t*       batch_emit;  /* [batches_cap] rank in it or -1 (p->dispatch)   */
} bs_window_io;

int bs_window_schedule(bs_ctx* ctx, const bs_window_io* io, const bs_window_params* p, void* stream);
/* K2..K6 given io->hist (local) and io->hist_global (all-reduced). */
int bs_window_from_hist(bs_ctx* ctx, const bs_window_io* io, const bs_window_params* p, void* stream);

/* ---- C1 over peer memory (alternative to an NCCL all-reduce) --------------------------
 * One process per GPU; every rank's context owns an exchange buffer (two histogram
 * slots + an epoch flag) that the other ranks map with CUDA IPC (NVLink / NVSwitch
 * peer memory on a multi-GPU node).  bs_peer_export writes the buffer's
 * cudaIpcMemHandle_t (BS_PEER_HANDLE_BYTES) into handle_out; after the handles of all
 * ranks are gathered (any host transport), bs_peer_connect maps them (handles[r] is
 * rank r's handle; the own entry is ignored).  bs_peer_reduce then runs C1 on the
 * device, after bs_histogram on the same stream: it publishes this rank's histogram
 * for the next epoch (device-side counter: graph-capturable), waits on every peer's
 * epoch flag (acquire, system scope) and sums the peers' slots into hist_global
 * (read straight from peer memory).  Two slots per rank make a rank that runs one
 * window ahead safe.  A peer that does not arrive within ~5 s latches
 * BS_FLAG_PEER_TIMEOUT instead of hanging. */
#define BS_PEER_HANDLE_BYTES 64
int bs_peer_export(bs_ctx* ctx, void* handle_out);
int bs_peer_connect(bs_ctx* ctx, int32_t rank, int32_t world, const void* handles);
int bs_peer_reduce(bs_ctx* ctx, const uint32_t* hist_local, const bs_window_params* p,
                   uint32_t* hist_global, bs_summary* summary, void* stream);

/* ---- C1 over NCCL (the library's own communicator, SURVEY §8b "bs_set_nccl") --------
 * Attaching a communicator makes bs_window_schedule run C1 itself: after K1 it
 * all-reduces (sum) io->hist into io->hist_global (required, distinct) with
 * ncclAllReduce on the window's stream, then K2..K6 on the global histogram — every
 * rank gets the same edges.  The whole window is then one stream
 * sequence a CUDA graph can capture.  libnccl.so.2 is resolved at run time (the
 * instance already loaded in the process is reused; BS_NCCL_LIB overrides).
 *   bs_nccl_unique_id: ncclGetUniqueId into 128 opaque bytes (rank 0; the caller
 *                      broadcasts them over any host transport);
 *   bs_nccl_connect:   ncclCommInitRank on ctx's device; ctx owns the communicator;
 *   bs_set_nccl:       attach a caller-owned ncclComm_t instead (NULL detaches);
 *   bs_nccl_allreduce: C1 alone, for callers composing bs_histogram /
 *                      bs_window_from_hist themselves. */
#define BS_NCCL_ID_BYTES 128
int bs_nccl_unique_id(void* id_out);
int bs_nccl_connect(bs_ctx* ctx, int32_t rank, int32_t world, const void* unique_id);
int bs_set_nccl(bs_ctx* ctx, void* nccl_comm, int32_t rank, int32_t world);
int bs_nccl_allreduce(bs_ctx* ctx, const uint32_t* hist_local, const bs_window_params* p,
                      uint32_t* hist_global, void* stream);

/* ---- monitor statistics ------------------------------------------
 * Bin counts only (= bs_monitor without edges): out[b] for the window histogram,
 * summed over classes; out is uint64[bins]. */
int bs_monitor_bins(bs_ctx* ctx, const uint32_t* hist, const bs_window_params* p, int32_t bins,
                    uint64_t* out, void* stream);

/* Monitor histogram + expected_waste, one kernel (K8).
 * counts_out[b] (uint64[bins]) = LengthHistogram.from_samples(lengths, bins,
 * range=(0, l_max)).counts (memory_model.py:125-130, pd_sim.py:829-831) — np.histogram's
 * uniform-bin rule, exact for every bins — summed over classes.  With edges (device
 * int32[k+1], the bucket partition e_0 = 0 < ... < e_k) also
 * stats_out[0] = expected_waste(hist, [(e_j, e_j+1)]) (memory_model.py:160-191: bins
 * left to right, cnt * (1 - mid / up) in float64, / total mass; NaN when the histogram
 * is empty or a midpoint lies beyond e_k — the reference raises ValueError there),
 * stats_out[1] = total mass, stats_out[2] = the unnormalised sum (device double[3]).
 * Replaces the per-tick O(queued) np.histogram + Python loop of pd_sim.py:828-833. */
int bs_monitor(bs_ctx* ctx, const uint32_t* hist, const bs_window_params* p, int32_t bins,
               const int32_t* edges, int32_t k, uint64_t* counts_out, double* stats_out,
               void* stream);

/* ---- trace ingestion (host side) ---------------------------------
 * Parses the reference's trace files (workload.py:343-437: `_load_csv`, `_load_jsonl`,
 * `load_trace`) into structure-of-arrays host memory: records in arrival order
 * (stable sort, ids = file order), the reference's validation, and on the first
 * malformed record BS_ERR_CONFIG with err_line / err_msg set to the reference's
 * TraceFormatError text ("line N: ...", errors.py:8-13).  `threads` <= 0: all host
 * threads (inputs under 1 MiB parse on one thread).  Arrays are malloc'ed by the
 * library; release them with bs_trace_free.  No GPU needed.
 * The .bst binary format stores the same arrays (64-byte header, then id, arrival,
 * input_len, output_len, cls, each padded to 64 bytes) for direct reloads. */
#define BS_TRACE_CSV   0
#define BS_TRACE_JSONL 1
typedef struct bs_trace {
  int64_t  n;
  int64_t* id;          /* [n] file-order id (Request.id)                       */
  double*  arrival;     /* [n] arrival_s, non-decreasing                        */
  int64_t* input_len;   /* [n] input_tokens (>= 1)                              */
  int64_t* output_len;  /* [n] output_tokens, -1 where the record omits it      */
  uint8_t* cls;         /* [n] 0 = online, 1 = offline                          */
  int64_t  err_line;    /* 1-based line of the first malformed record, else -1  */
  char     err_msg[256];
} bs_trace;
int  bs_trace_parse(const char* text, int64_t len, int32_t format, int32_t threads, bs_trace* out);
void bs_trace_free(bs_trace* t);
int  bs_trace_write_bst(const char* path, const bs_trace* t);
int  bs_trace_read_bst(const char* path, bs_trace* out);

/* ---- instrumentation ---------------------------------------------------------------
 * Stage timing of the fused window call, recorded with CUDA events on the call's
 * stream at the K1|K2|K4|K5|K6 boundaries (no host synchronisation while
 * recording).  bs_profile_enable(ctx, max_steps) arms a ring of max_steps event
 * sets (0 disarms); bs_profile_read synchronises the recorded events, writes the
 * summed milliseconds per stage (BS_STAGES floats) and the number of recorded
 * steps, and resets the ring.  bs_launch_count: kernels launched by ctx so far. */
#define BS_STAGES 11  /* 0 histogram, 1 exchange (C1: NCCL / peer all-reduce), 2 boundaries,
                         3 order, 4 size.prep, 5 size.next, 6 size.chain,
                         7 size.describe(+offsets), 8 size.outcome,
                         9 dispatch (when p->dispatch), 10 pack */
int bs_profile_enable(bs_ctx* ctx, int32_t max_steps);
int bs_profile_read(bs_ctx* ctx, float* stage_ms, int32_t* steps_out);
int64_t bs_launch_count(const bs_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* BUCKETSERVE_H */
