// ctx.cuh — the scratch-owning context behind bs_ctx and the internal launchers.
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

struct bs_ctx {
  int device = 0;
  int num_sms = 148;
  int64_t max_n = 0;
  int32_t l_cap = 0;
  int32_t c_max = 0;
  int r_cap = 0;            // doubling levels stored for the K5 chain
  int64_t max_tiles = 0;    // K4 tiles per pass
  int64_t scratch_bytes = 0;
  int64_t launches = 0;     // kernels launched through this ctx
  int pack_variant = 0;     // K6 tuning variant (env BS_PACK_VARIANT)
  int hist_agg = 0;         // K1: 1 = warp-aggregated shared atomics (env BS_HIST_AGG)
  int32_t piece_tok = 2048;  // K6 piece size of the last sized window (piece_tokens_for)
  int64_t pack_pieces = 0;   // upper bound on its K6 pieces: n * ceil(l_max / piece_tok)
  // tuning hooks, read from the environment once per context by bs_create (per-device
  // state such as shared-memory opt-ins and occupancy lives here too, not in statics)
  int hist_ept = 4;         // K1 elements per thread (BS_HIST_EPT)
  int hist_maxb = 0;        // K1 CTA cap (BS_HIST_MAXB; default 2 per SM)
  int sort_items = 0;       // K4 keys per thread: 0 = by window size, 8 | 16 (BS_SORT_ITEMS)
  int chain_pairs = 1;       // K5c walk two calls per round trip (BS_CHAIN_PAIRS=0: off)
  int chain_walk = 0;       // K5c serial-walk limit, 0 = default (BS_CHAIN_WALK)
  int pack_tma_blocks = 0;  // K6 TMA grid: co-resident CTAs per SM x SMs
  int pack_reverse = 1;     // K6 takes its 32-piece groups last batch first (BS_PACK_REVERSE=0: in order)
  int pack_bulk_blocks = 0; // K6 bulk-staged grid: co-resident CTAs per SM x SMs (pack_prepare)
  int pack_bulk_warps = 16; // warps per CTA of the bulk-staged pack (BS_BULK_WARPS: 8 | 16)
  int carveout_uniform = 0; // > 0: every kernel at this shared-memory carveout, percent of the
                            // maximum (launch_k; bs_create: 100 for max_n <= 4M, BS_CARVEOUT)
  int64_t last_n = 0;       // requests of the last sized window (grid bound of the K6 row prep)
  int pdl = 1;              // programmatic dependent launch between the window's kernels (BS_PDL)
  int prio_on = 0;          // per-launch priorities (bs_create; BS_PRIO): scheduling high, K6 low
  int prio_sched = 0, prio_pack = 0;
  mutable bool in_pack = false;  // set by launch_pack around the K6 launches
  int small_path = 1;       // K0 single-CTA path for small windows (BS_SMALL=0 disables)
  int small_smem_max = 0;   // its dynamic shared-memory opt-in (bytes)
  int small_timing = 0;     // K0 phase timestamps into summary.reserved (BS_SMALL_TIMING=1 ns, 2 cycles)
  bool window_zeroed = false;  // inside a fused window call whose k_window_init zeroed the
                               // accumulators (the launchers then skip their memsets)
  std::string err;
  // stage profiler: ring of (BS_STAGES+1) events per recorded step
  std::vector<cudaEvent_t> prof_events;
  int prof_steps = 0;       // ring capacity (0 = disabled)
  int prof_recorded = 0;    // steps recorded since the last read
  bool prof_in_window = false;  // only the fused window call records stage events

  // K2 tables
  uint32_t* P = nullptr;         // [l_cap+1] exclusive prefix of the (global) total histogram
  uint32_t* PcL = nullptr;       // [c_max][l_cap+1] exclusive prefix of the local per-class hist
  int32_t* E = nullptr;          // [l_cap+1] compacted edges of the last bs_boundaries call
  int32_t* lut = nullptr;        // [l_cap] bucket index per length
  int32_t* seg_base = nullptr;   // [l_cap*c_max] first radix slot of each segment
  int32_t* seg_off = nullptr;    // [l_cap*c_max+1] segment offsets of the last bs_boundaries
  uint32_t* slot_lut = nullptr;  // [c_max*l_cap] radix slot per (class, length)
  int32_t* slot_seg = nullptr;   // [c_max*l_cap] segment of each radix slot
  int32_t* slot_len = nullptr;  // [C*L+1] radix slot -> length (SJF / LJF slots; -1 for FCFS)
  const uint32_t* sorted_keys = nullptr;  // drain-order slots of the last bs_order (K4)
  uint32_t* bins_cnt = nullptr;  // [4][256] per-pass radix digit counts (K2c -> K4)
  uint32_t* tile_tot = nullptr;  // [ntiles][C+1] K2a tile totals (per class, then total)
  uint64_t* tile_slen = nullptr; // [ntiles] K2a tile sum of x*h[x]
  uint32_t* tile_carry = nullptr;// [ntiles+1][C+1] per-class tile carries (K2b)
  uint32_t* bmw = nullptr;       // [W] final edge bitmask over [0, L]
  uint32_t* wp = nullptr;        // [W] exclusive popc prefix of bmw
  int32_t* kinfo = nullptr;      // [8]: K, D, ...
  // K4
  uint32_t *keysA = nullptr, *keysB = nullptr, *valsA = nullptr, *valsB = nullptr;
  uint32_t* status = nullptr;    // [4][max_tiles][256]
  uint32_t* tile_ctr = nullptr;  // [4]
  // K5
  int32_t* sorted_len = nullptr; // [max_n] effective length in drain order
  int32_t* bmax = nullptr;       // [max_n/32+1] per 32-position group: max non-rejected length
  int32_t* bcnt = nullptr;       //   non-rejected count
  int32_t* bsum = nullptr;       //   non-rejected length sum
  int32_t* bmin = nullptr;       //   non-rejected length min
  uint32_t* bmask = nullptr;     //   bit l: position 32g+l is admissible (len <= S)
  int32_t* Rg = nullptr;         // [max_n/32+1] exclusive prefix of bcnt
  int32_t* rg_tiles = nullptr;   // [2][groups/8192+2] K5c Rg tile sums, then their prefix
  int32_t* rowpos = nullptr;     // [max_n] admitted window row -> drain position (K6)
  ulonglong2* rowdesc = nullptr; // [max_n] K6 row descriptors {src | x << 40, dst | pitch << 40}
  int32_t* chunk_row = nullptr;  // [chunk_cap] K6 output chunk -> the row holding its first element
  int64_t chunk_cap = 0;
  bool rowdesc_ready = false;    // K5e of the window just sized wrote rowdesc / chunk_row
  int64_t* task_base = nullptr;  // [max_n + 1] K6 pieces before each batch (row pieces of
                                 //   <= kPiece tokens; exclusive prefix, K5f)
  int32_t* node_j0 = nullptr;    // [max_n + 1] first admissible position at/after each chain node
  int32_t* segw = nullptr;       // [7][l_cap*c_max+1] per-segment chain length / tail / bases
  int32_t* J = nullptr;          // [r_cap][max_n] 2^r-th successor in the greedy chain
  uint8_t* is_start = nullptr;   // [max_n] position starts a non-empty segment
  int32_t* listA = nullptr;      // [max_n + 1] chain-node lists (expansion ping-pong)
  int32_t* listB = nullptr;
  int32_t* node_batch = nullptr; // [max_n + 1] batch id of each chain node (-1: empty tail)
  // K7 dispatch order (f3)
  int disp_blocks = 0;           // co-resident CTAs of the cooperative K7 kernel
  int32_t* disp_cseg = nullptr;  // [max_n+1] segment of each call
  int32_t* disp_cmin = nullptr;  // [max_n+1] min arrival rank over the call's range
  int64_t* disp_csum = nullptr;  // [max_n+1] length sum over the call's range
  uint64_t *disp_keys0 = nullptr, *disp_keys1 = nullptr;  // [max_n+1] sort keys (ping-pong)
  uint32_t *disp_vals0 = nullptr, *disp_vals1 = nullptr;  // [max_n+1] call ids
  uint32_t* disp_hist8 = nullptr;    // [8][256] key-byte histograms (zero between windows)
  int64_t* disp_agg = nullptr;       // [2*disp_blocks] chunk aggregates of the key scan
  uint32_t* disp_status = nullptr;   // [8][max_n/7168+2][256] look-back words
  uint32_t* disp_tctr = nullptr;     // [8] tile counters
  int32_t* disp_nulls = nullptr;     // [l_cap*c_max+1] sorted positions of null calls
  uint64_t* disp_bkeys = nullptr;    // [l_cap*c_max+1] per null call: its blocked bucket's key
  int32_t* disp_runs = nullptr;      // [2*l_cap*c_max+32][4] runs of consecutive plans
  int64_t* disp_misc = nullptr;      // [32]
  // C1 over peer memory (bs_peer_*)
  uint32_t* xbuf = nullptr;          // own exchange buffer: [2][c_max*l_cap] hist slots + flags
  int64_t xbuf_bytes = 0;
  int peer_rank = -1, peer_world = 0;
  std::vector<void*> peer_mapped;    // IPC mappings of the other ranks' exchange buffers
  uint32_t** peer_ptrs = nullptr;    // device table [world] of exchange-buffer base pointers
  // C1 over NCCL (bs_nccl_connect / bs_set_nccl)
  void* nccl_comm = nullptr;         // ncclComm_t
  bool nccl_owned = false;           // created by bs_nccl_connect (destroyed with the ctx)
  int nccl_rank = -1, nccl_world = 0;
  unsigned char* small_rows = nullptr;  // [kSmallN] K0 -> k_pack_rows copy jobs (SmallRow)
  int32_t* misc = nullptr;       // [128]: [0..63] alive flags per level, [64] M, [65] R_top,
                                 //        [66] n_batches, [67] pack rows cursor, [69] long chains,
                                 //        [70] long-segment count
};

namespace bsk {

// one admitted row of a small window: the copy job K0 hands to k_pack_rows
struct SmallRow {
  int64_t src;    // token-store offset of the request (tok_off)
  int64_t dst;    // element offset of the row in the packed buffers
  int32_t x;      // real tokens
  int32_t pitch;  // row pitch (tokens + padding)
};

constexpr int kTileX = 4096;  // lengths per K2a tile
constexpr int kPiece = 2048;  // K6 work unit: at most this many tokens of one row
constexpr int kPackChunk = 1024;  // K6 bulk-staged pack: output chunk (tokens) per work unit
// K6 piece size for a window of n requests: kPiece from 64k requests up; smaller windows
// use proportionally smaller pieces (>= 32 tokens, one 128-byte line) so the pack still
// spreads over every SM (C1's 1k requests: 32 pieces of 2048 tokens would be 32 warps)
inline int32_t piece_tokens_for(int64_t n) {
  int32_t t = kPiece;
  while (t > 32 && n * (kPiece / t) < (int64_t)65536) t >>= 1;
  return t;
}

// records boundary event `stage` (0..BS_STAGES) of the current profiled step
inline void prof_mark(bs_ctx* ctx, int stage, cudaStream_t st) {
  if (!ctx->prof_in_window || ctx->prof_steps <= 0 || ctx->prof_recorded >= ctx->prof_steps) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) return;
  cudaEventRecord(ctx->prof_events[(size_t)ctx->prof_recorded * (BS_STAGES + 1) + stage], st);
  if (stage == BS_STAGES) ++ctx->prof_recorded;
}

// Kernel launch for the window path: cudaLaunchKernelEx with programmatic stream
// serialization when ctx->pdl (see pdl_prologue in common.cuh), and the cooperative
// attribute for grid-synchronising kernels.  If the driver refuses the combination of a
// cooperative launch with PDL, the kernel is launched cooperatively without it.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(const bs_ctx* ctx, void (*kernel)(KArgs...), dim3 grid, dim3 block,
                            size_t smem, cudaStream_t st, bool cooperative, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[4];
  unsigned na = 0;
  if (ctx->carveout_uniform > 0) {
    // every kernel of the window at the maximum shared-memory carveout: an SM only runs
    // CTAs of one L1 / shared-memory split at a time, so with mixed splits the scheduling
    // kernels of the windows in flight could not start on an SM beside the (shared-memory
    // staged) pack of another window.  Windows of up to 4M requests (C2: 0.735 vs 0.759 ms
    // per window in flight); at 16M (C3) the gather-heavy K5 kernels want their L1 back.
    at[na].id = cudaLaunchAttributePreferredSharedMemoryCarveout;
    at[na].val.sharedMemCarveout = (unsigned)ctx->carveout_uniform;  // percent of the maximum
    ++na;
  }
  if (ctx->prio_on) {
    at[na].id = cudaLaunchAttributePriority;
    at[na].val.priority = ctx->in_pack ? ctx->prio_pack : ctx->prio_sched;
    ++na;
  }
  if (cooperative) {
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    ++na;
  }
  if (ctx->pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  if (e != cudaSuccess && cooperative && ctx->pdl) {
    (void)cudaGetLastError();
    cfg.numAttrs = na - 1;  // without PDL (the last attribute)
    e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  }
  return e;
}

struct SortPlan {
  int passes;  // radix passes
  int bits;    // digit bits per pass (<= 8)
};
SortPlan sort_plan(int32_t l_max, int32_t n_classes);

// launchers (return cudaError_t of the launch)
cudaError_t launch_histogram(bs_ctx* ctx, const int32_t* len, const uint8_t* cls, int64_t n,
                             const bs_window_params& p, uint32_t* hist, bs_summary* summary,
                             cudaStream_t st);
cudaError_t launch_boundaries(bs_ctx* ctx, const uint32_t* hist_local, const uint32_t* hist_global,
                              const bs_window_params& p, const int32_t* init_edges, int32_t k_init,
                              int32_t* edges_out, int32_t* changes_out, int32_t changes_cap,
                              int32_t* seg_off_out, bs_summary* summary, cudaStream_t st);
cudaError_t launch_assign(bs_ctx* ctx, const int32_t* len, int64_t n, const bs_window_params& p,
                          int32_t* bucket_out, cudaStream_t st);
cudaError_t launch_order(bs_ctx* ctx, const int32_t* len, const uint8_t* cls, int64_t n,
                         const bs_window_params& p, int32_t* perm_out, int32_t* bucket_out,
                         bs_summary* summary, cudaStream_t st);
cudaError_t launch_size(bs_ctx* ctx, const int32_t* len, const int32_t* perm,
                        const int32_t* seg_off, int64_t n, const bs_window_params& p,
                        bs_batch* batches, int32_t batches_cap, int32_t* req_batch,
                        int32_t* req_row, bs_summary* summary, cudaStream_t st,
                        const int64_t* tok_off = nullptr);
// would launch_pack use the bulk-staged pack (row records written by K5e when it does)
bool pack_uses_bulk(const bs_ctx* ctx, const bs_window_params& p, const int32_t* out_tokens,
                    const uint8_t* out_mask);
cudaError_t launch_pack(bs_ctx* ctx, const int32_t* len, const int32_t* perm,
                        const int64_t* tok_off, const int32_t* tokens, const bs_window_params& p,
                        const bs_batch* batches, int64_t batch_begin, int64_t batch_end,
                        int32_t batches_cap, int32_t* out_tokens, uint8_t* out_mask,
                        int64_t out_capacity, bs_summary* summary, cudaStream_t st);
cudaError_t launch_dispatch(bs_ctx* ctx, const int32_t* perm, const int32_t* seg_off, int64_t n,
                            const bs_window_params& p, const bs_batch* batches,
                            int32_t batches_cap, int32_t* req_batch, int32_t* req_row,
                            int32_t* emit_order, int32_t* batch_emit, bs_summary* summary,
                            cudaStream_t st);
int dispatch_smem_bytes();
int peer_flag_words();
int dispatch_threads();
cudaError_t launch_peer_reduce(bs_ctx* ctx, const uint32_t* hist_local, const bs_window_params& p,
                               uint32_t* hist_global, bs_summary* summary, cudaStream_t st);
cudaError_t launch_monitor(const bs_ctx* ctx, const uint32_t* hist, const bs_window_params& p,
                           int32_t bins, const int32_t* edges, int32_t k, uint64_t* out,
                           double* stats, cudaStream_t st);
cudaError_t launch_monitor_bins(const bs_ctx* ctx, const uint32_t* hist, const bs_window_params& p,
                                int32_t bins, uint64_t* out, cudaStream_t st);
cudaError_t launch_init_summary(const bs_ctx* ctx, bs_summary* s, int64_t n, cudaStream_t st);
cudaError_t launch_window_init(bs_ctx* ctx, bs_summary* s, int64_t n, uint32_t* hist,
                               int64_t hist_words, int64_t status_words, cudaStream_t st);
int64_t sort_status_words(const bs_ctx* ctx, int64_t n, const bs_window_params& p);
// per-context, per-device setup run by bs_create (shared-memory opt-ins, occupancy)
cudaError_t hist_prepare(bs_ctx* ctx);
cudaError_t bounds_prepare(bs_ctx* ctx);
cudaError_t pack_prepare(bs_ctx* ctx);
cudaError_t small_prepare(bs_ctx* ctx);
bool small_window_ok(const bs_ctx* ctx, int64_t n, const bs_window_params& p, int32_t k_init);
cudaError_t launch_window_small(bs_ctx* ctx, const bs_window_io* io, const bs_window_params& p,
                                cudaStream_t st);
cudaError_t launch_pack_rows(bs_ctx* ctx, const int32_t* tokens, const bs_window_params& p,
                             int32_t n, int32_t* out_tokens, uint8_t* out_mask,
                             int64_t out_capacity, bs_summary* summary, cudaStream_t st);
// nccl_c1.cu (libnccl resolved with dlopen)
int nccl_status(std::string* why);
int nccl_unique_id(void* id_out, std::string* why);
int nccl_comm_init(void** comm, int world, const void* id, int rank, std::string* why);
void nccl_comm_destroy(void* comm);
int nccl_allreduce_hist(bs_ctx* ctx, const uint32_t* hist_local, uint32_t* hist_global,
                        size_t count, cudaStream_t st, std::string* why);

}  // namespace bsk
