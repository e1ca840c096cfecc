// capi.cu — the extern "C" boundary (include/bucketserve.h): context lifetime,
// scratch layout, argument validation and stage orchestration.  No C++
// exception crosses this boundary; every entry returns a BS_* status.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "ctx.cuh"

void* bs_dispatch_kernel_ptr();  // k_dispatch.cu

namespace {

std::mutex g_err_mu;
std::string g_err;

int fail(bs_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  std::lock_guard<std::mutex> lk(g_err_mu);
  g_err = msg;
  return code;
}

int cuda_fail(bs_ctx* ctx, cudaError_t e, const char* where) {
  std::string m = std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  const bool unavailable = e == cudaErrorNoKernelImageForDevice || e == cudaErrorNoDevice ||
                           e == cudaErrorInsufficientDriver || e == cudaErrorInvalidDevice;
  return fail(ctx, unavailable ? BS_ERR_NOT_BUILT : BS_ERR_CUDA, m);
}

#define BS_CUDA(call, where)                       \
  do {                                             \
    cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, where); \
  } while (0)

int check_params(bs_ctx* ctx, const bs_window_params* p) {
  if (!p) return fail(ctx, BS_ERR_INVALID_ARG, "params is NULL");
  if (p->l_max < 1) return fail(ctx, BS_ERR_INVALID_ARG, "max_seq_len must be >= 1");
  if (p->l_max > ctx->l_cap)
    return fail(ctx, BS_ERR_CAPACITY, "l_max " + std::to_string(p->l_max) + " exceeds context capacity " +
                                          std::to_string(ctx->l_cap));
  if (p->n_classes < 1 || p->n_classes > ctx->c_max)
    return fail(ctx, BS_ERR_INVALID_ARG, "n_classes must be in [1, " + std::to_string(ctx->c_max) + "]");
  for (int c = 0; c < p->n_classes; ++c)
    if (p->policy[c] < BS_POLICY_FCFS || p->policy[c] > BS_POLICY_LJF)
      return fail(ctx, BS_ERR_INVALID_ARG, "unknown dispatch policy");
  if (!(p->split_threshold > 0.0 && p->split_threshold <= 1.0))
    return fail(ctx, BS_ERR_INVALID_ARG, "split_threshold must be in (0, 1]");
  if (p->kv_bytes_per_token < 1) return fail(ctx, BS_ERR_CONFIG, "kv_bytes_per_token must be >= 1");
  if (p->current_safe < 0) return fail(ctx, BS_ERR_INVALID_ARG, "safe memory must be >= 0");
  if (p->accounting != BS_ACCOUNTING_PADDED && p->accounting != BS_ACCOUNTING_EXACT)
    return fail(ctx, BS_ERR_INVALID_ARG, "unknown memory accounting");
  return BS_OK;
}

int check_n(bs_ctx* ctx, int64_t n) {
  if (n < 0) return fail(ctx, BS_ERR_INVALID_ARG, "n must be >= 0");
  if (n > ctx->max_n)
    return fail(ctx, BS_ERR_CAPACITY, "window of " + std::to_string(n) + " requests exceeds context capacity " +
                                          std::to_string(ctx->max_n));
  return BS_OK;
}

template <typename T>
cudaError_t alloc(bs_ctx* ctx, T** p, size_t count) {
  size_t bytes = sizeof(T) * (count ? count : 1);
  ctx->scratch_bytes += (int64_t)bytes;
  return cudaMalloc(reinterpret_cast<void**>(p), bytes);
}

void free_all(bs_ctx* c) {
  void* ptrs[] = {c->P, c->PcL, c->E, c->lut, c->seg_base, c->seg_off, c->slot_lut, c->slot_seg, c->slot_len, c->bins_cnt,
                  c->tile_tot, c->tile_slen, c->tile_carry, c->bmw, c->wp, c->kinfo,
                  c->keysA, c->keysB, c->valsA, c->valsB, c->status, c->tile_ctr, c->sorted_len,
                  c->bmax, c->bcnt, c->bsum, c->bmin, c->bmask, c->Rg, c->rg_tiles, c->J,
                  c->is_start, c->listA, c->listB, c->node_batch, c->node_j0, c->rowpos, c->rowdesc, c->chunk_row, c->task_base, c->segw,
                  c->disp_cseg, c->disp_cmin, c->disp_csum, c->disp_keys0, c->disp_keys1,
                  c->disp_vals0, c->disp_vals1, c->disp_hist8, c->disp_agg, c->disp_status, c->disp_tctr, c->disp_nulls, c->disp_bkeys, c->disp_runs, c->disp_misc,
                  c->misc, c->small_rows};
  for (void* p : ptrs)
    if (p) cudaFree(p);
}

}  // namespace

extern "C" {

int bs_abi_version(void) { return BS_ABI_VERSION; }

const char* bs_last_error(const bs_ctx* ctx) {
  if (ctx) return ctx->err.c_str();
  std::lock_guard<std::mutex> lk(g_err_mu);
  return g_err.c_str();
}

int64_t bs_scratch_bytes(const bs_ctx* ctx) { return ctx ? ctx->scratch_bytes : 0; }

int bs_create(bs_ctx** out, int device, int64_t max_n, int32_t l_max_cap, int32_t max_classes) {
  if (!out) return fail(nullptr, BS_ERR_INVALID_ARG, "ctx out-pointer is NULL");
  *out = nullptr;
  if (max_n < 0 || max_n >= (int64_t)1 << 30)
    return fail(nullptr, BS_ERR_INVALID_ARG, "max_n must be in [0, 2^30)");
  if (l_max_cap < 1 || l_max_cap > (1 << 20))
    return fail(nullptr, BS_ERR_INVALID_ARG, "l_max_cap must be in [1, 2^20]");
  if (max_classes < 1 || max_classes > BS_MAX_CLASSES)
    return fail(nullptr, BS_ERR_INVALID_ARG, "max_classes must be in [1, 8]");
  bs_ctx* ctx = new (std::nothrow) bs_ctx();
  if (!ctx) return fail(nullptr, BS_ERR_CUDA, "out of host memory");
  ctx->device = device;
  ctx->max_n = max_n;
  ctx->l_cap = l_max_cap;
  ctx->c_max = max_classes;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) { int rc = cuda_fail(ctx, e, "cudaSetDevice"); delete ctx; return rc; }
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) { int rc = cuda_fail(ctx, e, "cudaGetDeviceProperties"); delete ctx; return rc; }
  if (prop.major != 10) {
    int rc = fail(ctx, BS_ERR_NOT_BUILT, std::string("device ") + prop.name +
                                             " is not sm_100 (this library is built for B200 sm_100a)");
    delete ctx;
    return rc;
  }
  if (!prop.cooperativeLaunch) {
    int rc = fail(ctx, BS_ERR_NOT_BUILT, "device lacks cooperative launch");
    delete ctx;
    return rc;
  }
  ctx->num_sms = prop.multiProcessorCount;
  if (const char* v = getenv("BS_PACK_VARIANT")) ctx->pack_variant = atoi(v);
  if (const char* v = getenv("BS_HIST_AGG")) ctx->hist_agg = atoi(v);
  ctx->hist_maxb = 2 * ctx->num_sms;
  if (const char* v = getenv("BS_HIST_EPT")) ctx->hist_ept = std::max(1, atoi(v));
  if (const char* v = getenv("BS_HIST_MAXB")) ctx->hist_maxb = std::max(1, atoi(v));
  if (const char* v = getenv("BS_SORT_ITEMS")) ctx->sort_items = atoi(v);
  if (const char* v = getenv("BS_CHAIN_WALK")) ctx->chain_walk = std::max(1, atoi(v));
  if (const char* v = getenv("BS_CHAIN_PAIRS")) ctx->chain_pairs = atoi(v) != 0;
  if (const char* v = getenv("BS_PDL")) ctx->pdl = atoi(v) != 0;
  if (const char* v = getenv("BS_PACK_REVERSE")) ctx->pack_reverse = atoi(v) != 0;
  {  // launch priorities: the scheduling kernels of a window ahead of the packs of the
     // windows in flight when both wait for an SM (C2 0.724 -> 0.714 ms, C3 11.89 ->
     // 11.74 ms per window in flight); BS_PRIO=0 off, -1 the reverse (tuning hook)
    const char* v = getenv("BS_PRIO");
    const int mode = v ? atoi(v) : 1;
    int lo = 0, hi = 0;  // least (numerically largest) and greatest priority
    if (mode != 0 && cudaDeviceGetStreamPriorityRange(&lo, &hi) == cudaSuccess && lo != hi) {
      ctx->prio_on = 1;
      ctx->prio_sched = mode > 0 ? hi : lo;
      ctx->prio_pack = mode > 0 ? lo : hi;
    }
  }
  if (const char* v = getenv("BS_BULK_WARPS")) ctx->pack_bulk_warps = atoi(v) == 8 ? 8 : 16;
  ctx->carveout_uniform = max_n <= (4 << 20) ? 100 : 0;
  if (const char* v = getenv("BS_CARVEOUT")) ctx->carveout_uniform = std::max(0, std::min(100, atoi(v)));
  if (const char* v = getenv("BS_SMALL")) ctx->small_path = atoi(v) != 0;
  if (const char* v = getenv("BS_SMALL_TIMING")) ctx->small_timing = atoi(v);
  int r = 1;
  while (((int64_t)1 << r) < max_n + 1) ++r;
  ctx->r_cap = r + 2;
  const int64_t L = l_max_cap, C = max_classes, N = max_n;
  ctx->max_tiles = (N + 2047) / 2048 + 1;  // smallest K4 tile is 2048 keys
  const int64_t groups = (N + 31) / 32 + 1;
#define A(ptr, cnt)                                                        \
  if ((e = alloc(ctx, &ctx->ptr, (size_t)(cnt))) != cudaSuccess) {         \
    int rc = cuda_fail(ctx, e, "cudaMalloc " #ptr);                        \
    free_all(ctx);                                                         \
    delete ctx;                                                            \
    return rc;                                                             \
  }
  A(P, L + 1);
  A(PcL, C * (L + 1));
  A(E, L + 1);
  A(lut, L);
  A(seg_base, L * C);
  A(seg_off, L * C + 1);
  A(slot_lut, C * L);
  A(slot_seg, C * L + 1);
  A(slot_len, C * L + 1);
  A(bins_cnt, 4 * 256);
  const int64_t ntiles = (L + bsk::kTileX - 1) / bsk::kTileX;
  A(tile_tot, ntiles * (C + 1));
  A(tile_slen, ntiles);
  A(tile_carry, (ntiles + 1) * (C + 1));
  A(bmw, (L + 1 + 31) / 32);
  A(wp, (L + 1 + 31) / 32);
  A(kinfo, 8);
  A(keysA, N); A(keysB, N); A(valsA, N); A(valsB, N);
  A(status, 4 * ctx->max_tiles * 256);
  A(tile_ctr, 4);
  A(sorted_len, N);
  A(bmax, groups); A(bcnt, groups); A(bsum, groups); A(bmin, groups); A(bmask, groups);
  A(Rg, groups);
  A(J, (int64_t)ctx->r_cap * N);
  A(is_start, N);
  A(listA, N + 1); A(listB, N + 1);
  A(node_batch, N + 1);
  A(node_j0, N + 1);
  A(segw, 7 * (L * C + 1));
  A(rowpos, N + 1);
  A(task_base, N + 2);
  A(rowdesc, N + 1);
  // K6 output chunks: one per kPackChunk tokens of the largest packed window
  ctx->chunk_cap = (N * (((int64_t)L + 31) / 32 * 32) + bsk::kPackChunk - 1) / bsk::kPackChunk + 2;
  A(chunk_row, ctx->chunk_cap);
  A(misc, 128);
  A(small_rows, 2048 * 32);  // bsk::kSmallN SmallRow records
  // K7 dispatch order
  A(disp_cseg, N + 1); A(disp_cmin, N + 1); A(disp_csum, N + 1);
  A(disp_keys0, N + 1); A(disp_keys1, N + 1); A(disp_vals0, N + 1); A(disp_vals1, N + 1);
  A(disp_hist8, 8 * 256);
  A(disp_status, 8 * ((N + 7167) / 7168 * 256 + 256)); A(disp_tctr, 8);
  A(disp_nulls, L * C + 1); A(disp_bkeys, L * C + 1); A(disp_runs, 4 * (2 * L * C + 32)); A(disp_misc, 32);
  if ((e = cudaMemset(ctx->disp_hist8, 0, sizeof(uint32_t) * 8 * 256)) != cudaSuccess) {
    int rc = cuda_fail(ctx, e, "cudaMemset disp_hist8");
    free_all(ctx);
    delete ctx;
    return rc;
  }
  // K5c: per-tile admissible counts and their prefix (Rg tiles of 8192 groups)
  A(rg_tiles, 2 * (groups / 8192 + 2));
  int per_sm = 0;
  // the cooperative K7 dispatch kernel: one 1024-thread CTA per SM, ~211 KB of shared memory
  e = cudaFuncSetAttribute(bs_dispatch_kernel_ptr(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                           bsk::dispatch_smem_bytes());
  per_sm = 0;
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bs_dispatch_kernel_ptr(),
                                                      bsk::dispatch_threads(),
                                                      bsk::dispatch_smem_bytes());
  if (e != cudaSuccess || per_sm < 1) {
    int rc = e != cudaSuccess ? cuda_fail(ctx, e, "occupancy(k_dispatch)")
                              : fail(ctx, BS_ERR_NOT_BUILT, "k_dispatch cannot be resident");
    free_all(ctx);
    delete ctx;
    return rc;
  }
  // 16 co-resident CTAs: the multi-CTA radix path (> 8192 calls) is as fast as with one
  // CTA per SM (C3: 177 vs 187 us), and the cooperative launch only has to find 16 SMs
  // free between the packs of other windows in flight (C2 with K7, four windows in
  // flight: 0.784 vs 0.891 ms per window); tuning hook BS_DISP_CTAS
  ctx->disp_blocks = std::min(per_sm * ctx->num_sms, 16);
  if (const char* v = getenv("BS_DISP_CTAS"))
    ctx->disp_blocks = std::max(1, std::min(per_sm * ctx->num_sms, atoi(v)));
  A(disp_agg, 2 * ctx->disp_blocks);
#undef A
  // per-device kernel attributes (checked): every context sets them on its own device
  if ((e = bsk::hist_prepare(ctx)) != cudaSuccess || (e = bsk::bounds_prepare(ctx)) != cudaSuccess ||
      (e = bsk::pack_prepare(ctx)) != cudaSuccess || (e = bsk::small_prepare(ctx)) != cudaSuccess) {
    int rc = cuda_fail(ctx, e, "kernel attributes");
    free_all(ctx);
    delete ctx;
    return rc;
  }
  *out = ctx;
  return BS_OK;
}

int bs_destroy(bs_ctx* ctx) {
  if (!ctx) return BS_OK;
  cudaSetDevice(ctx->device);
  if (ctx->nccl_owned) bsk::nccl_comm_destroy(ctx->nccl_comm);
  for (void* m : ctx->peer_mapped)
    if (m) cudaIpcCloseMemHandle(m);
  if (ctx->peer_ptrs) cudaFree(ctx->peer_ptrs);
  if (ctx->xbuf) cudaFree(ctx->xbuf);
  for (cudaEvent_t e : ctx->prof_events) cudaEventDestroy(e);
  free_all(ctx);
  delete ctx;
  return BS_OK;
}

int bs_histogram(bs_ctx* ctx, const int32_t* len, const uint8_t* cls, int64_t n,
                 const bs_window_params* p, uint32_t* hist_out, bs_summary* summary, void* stream) {
  if (!ctx) return fail(nullptr, BS_ERR_INVALID_ARG, "ctx is NULL");
  int rc;
  if ((rc = check_params(ctx, p)) != BS_OK || (rc = check_n(ctx, n)) != BS_OK) return rc;
  if (!hist_out || (n > 0 && (!len || !cls))) return fail(ctx, BS_ERR_INVALID_ARG, "NULL buffer");
  BS_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (summary) {
    BS_CUDA(bsk::launch_init_summary(ctx, summary, n, st), "init_summary");
    ++ctx->launches;
  }
  BS_CUDA(bsk::launch_histogram(ctx, len, cls, n, *p, hist_out, summary, st), "k_histogram");
  return BS_OK;
}

static int boundaries_impl(bs_ctx* ctx, const uint32_t* hist_local, const uint32_t* hist_global,
                           const bs_window_params* p, const int32_t* init_edges, int32_t k_init,
                           int32_t* edges_out, int32_t* changes_out, int32_t changes_cap,
                           int32_t* seg_off_out, bs_summary* summary, cudaStream_t st) {
  if (!hist_local || !edges_out || !summary || !seg_off_out)
    return fail(ctx, BS_ERR_INVALID_ARG, "NULL buffer");
  if (init_edges && (k_init < 1 || k_init > p->l_max))
    return fail(ctx, BS_ERR_INVALID_ARG, "k_init out of range");
  if (changes_cap < 0 || (changes_cap > 0 && !changes_out))
    return fail(ctx, BS_ERR_INVALID_ARG, "bad change-log buffer");
  BS_CUDA(bsk::launch_boundaries(ctx, hist_local, hist_global, *p, init_edges, k_init, edges_out,
                                 changes_out, changes_cap, seg_off_out, summary, st),
          "k_boundaries");
  return BS_OK;
}

int bs_boundaries(bs_ctx* ctx, const uint32_t* hist_local, const uint32_t* hist_global,
                  const bs_window_params* p, const int32_t* init_edges, int32_t k_init,
                  int32_t* edges_out, int32_t* changes_out, int32_t changes_cap,
                  bs_summary* summary, void* stream) {
  if (!ctx) return fail(nullptr, BS_ERR_INVALID_ARG, "ctx is NULL");
  int rc;
  if ((rc = check_params(ctx, p)) != BS_OK) return rc;
  BS_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  // the segment table stays in ctx scratch; bs_order hands a copy to the caller
  return boundaries_impl(ctx, hist_local, hist_global, p, init_edges, k_init, edges_out,
                         changes_out, changes_cap, ctx->seg_off, summary,
                         static_cast<cudaStream_t>(stream));
}

int bs_assign(bs_ctx* ctx, const int32_t* len, int64_t n, const bs_window_params* p,
              int32_t* bucket_out, void* stream) {
  if (!ctx) return fail(nullptr, BS_ERR_INVALID_ARG, "ctx is NULL");
  int rc;
  if ((rc = check_params(ctx, p)) != BS_OK || (rc = check_n(ctx, n)) != BS_OK) return rc;
  if (n > 0 && (!len || !bucket_out)) return fail(ctx, BS_ERR_INVALID_ARG, "NULL buffer");
  BS_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  BS_CUDA(bsk::launch_assign(ctx, len, n, *p, bucket_out, static_cast<cudaStream_t>(stream)),
          "k_assign");
  return BS_OK;
}

int bs_order(bs_ctx* ctx, const int32_t* len, const uint8_t* cls, int64_t n,
             const bs_window_params* p, int32_t* perm_out, int32_t* seg_off_out,
             int32_t* bucket_out, bs_summary* summary, void* stream) {
  if (!ctx) return fail(nullptr, BS_ERR_INVALID_ARG, "ctx is NULL");
  int rc;
  if ((rc = check_params(ctx, p)) != BS_OK || (rc = check_n(ctx, n)) != BS_OK) return rc;
  if (n > 0 && (!len || !cls || !perm_out)) return fail(ctx, BS_ERR_INVALID_ARG, "NULL buffer");
  BS_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (seg_off_out)
    BS_CUDA(cudaMemcpyAsync(seg_off_out, ctx->seg_off,
                            sizeof(int32_t) * ((size_t)p->l_max * p->n_classes + 1),
                            cudaMemcpyDeviceToDevice, st),
            "copy seg_off");
  BS_CUDA(bsk::launch_order(ctx, len, cls, n, *p, perm_out, bucket_out, summary, st), "k_sort_pass");
  return BS_OK;
}

int bs_size(bs_ctx* ctx, const int32_t* len, const int32_t* perm, const int32_t* seg_off,
            int64_t n, const bs_window_params* p, bs_batch* batches_out, int32_t batches_cap,
            int32_t* req_batch_out, int32_t* req_row_out, bs_summary* summary, void* stream) {
  if (!ctx) return fail(nullptr, BS_ERR_INVALID_ARG, "ctx is NULL");
  int rc;
  if ((rc = check_params(ctx, p)) != BS_OK || (rc = check_n(ctx, n)) != BS_OK) return rc;
  if (!summary || !batches_out || batches_cap < 0 ||
      (n > 0 && (!len || !perm || !seg_off || !req_batch_out || !req_row_out)))
    return fail(ctx, BS_ERR_INVALID_ARG, "NULL buffer");
  BS_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  BS_CUDA(bsk::launch_size(ctx, len, perm, seg_off, n, *p, batches_out, batches_cap, req_batch_out,
                           req_row_out, summary, static_cast<cudaStream_t>(stream)),
          "k_size");
  return BS_OK;
}

int bs_pack(bs_ctx* ctx, const int32_t* len, const int32_t* perm, const int64_t* tok_off,
            const int32_t* tokens, const bs_window_params* p, const bs_batch* batches,
            int64_t batch_begin, int64_t batch_end, int32_t* out_tokens, uint8_t* out_mask,
            int64_t out_capacity, bs_summary* summary, void* stream) {
  if (!ctx) return fail(nullptr, BS_ERR_INVALID_ARG, "ctx is NULL");
  int rc;
  if ((rc = check_params(ctx, p)) != BS_OK) return rc;
  if (!len || !perm || !tok_off || !tokens || !batches || !out_tokens)
    return fail(ctx, BS_ERR_INVALID_ARG, "NULL buffer");
  if (batch_end < 0 && !summary)
    return fail(ctx, BS_ERR_INVALID_ARG, "batch_end < 0 needs the summary of bs_size");
  if (batch_begin < 0) return fail(ctx, BS_ERR_INVALID_ARG, "batch_begin must be >= 0");
  if (reinterpret_cast<uintptr_t>(out_tokens) & 15)
    return fail(ctx, BS_ERR_INVALID_ARG, "out_tokens must be 16-byte aligned");
  if (out_mask && (reinterpret_cast<uintptr_t>(out_mask) & 3))
    return fail(ctx, BS_ERR_INVALID_ARG, "out_mask must be 4-byte aligned");
  BS_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  BS_CUDA(bsk::launch_pack(ctx, len, perm, tok_off, tokens, *p, batches, batch_begin, batch_end,
                           INT32_MAX, out_tokens, out_mask, out_capacity, summary,
                           static_cast<cudaStream_t>(stream)),
          "k_pack");
  return BS_OK;
}

int bs_dispatch(bs_ctx* ctx, const int32_t* perm, const int32_t* seg_off, int64_t n,
                const bs_window_params* p, const bs_batch* batches, int32_t batches_cap,
                int32_t* req_batch, int32_t* req_row, int32_t* emit_order, int32_t* batch_emit,
                bs_summary* summary, void* stream) {
  if (!ctx) return fail(nullptr, BS_ERR_INVALID_ARG, "ctx is NULL");
  int rc;
  if ((rc = check_params(ctx, p)) != BS_OK || (rc = check_n(ctx, n)) != BS_OK) return rc;
  if (!summary || !batches || batches_cap < 0 || !emit_order || !batch_emit ||
      (n > 0 && (!perm || !seg_off || !req_batch || !req_row)))
    return fail(ctx, BS_ERR_INVALID_ARG, "NULL buffer");
  if (!p->dispatch)
    return fail(ctx, BS_ERR_INVALID_ARG,
                "bs_dispatch needs the bs_size call before it made with params.dispatch = 1");
  BS_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  BS_CUDA(bsk::launch_dispatch(ctx, perm, seg_off, n, *p, batches, batches_cap, req_batch, req_row,
                               emit_order, batch_emit, summary, static_cast<cudaStream_t>(stream)),
          "k_dispatch");
  return BS_OK;
}

int bs_peer_export(bs_ctx* ctx, void* handle_out) {
  if (!ctx || !handle_out) return fail(ctx, BS_ERR_INVALID_ARG, "NULL argument");
  BS_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  if (!ctx->xbuf) {
    const int64_t slot_words = (int64_t)ctx->l_cap * ctx->c_max;
    ctx->xbuf_bytes = (int64_t)sizeof(uint32_t) * 2 * slot_words +
                      (int64_t)sizeof(int64_t) * bsk::peer_flag_words();
    BS_CUDA(cudaMalloc(reinterpret_cast<void**>(&ctx->xbuf), (size_t)ctx->xbuf_bytes), "cudaMalloc xbuf");
    BS_CUDA(cudaMemset(ctx->xbuf, 0, (size_t)ctx->xbuf_bytes), "cudaMemset xbuf");
    ctx->scratch_bytes += ctx->xbuf_bytes;
  }
  cudaIpcMemHandle_t h;
  BS_CUDA(cudaIpcGetMemHandle(&h, ctx->xbuf), "cudaIpcGetMemHandle");
  static_assert(sizeof(cudaIpcMemHandle_t) == BS_PEER_HANDLE_BYTES, "IPC handle size");
  memcpy(handle_out, &h, sizeof h);
  return BS_OK;
}

int bs_peer_connect(bs_ctx* ctx, int32_t rank, int32_t world, const void* handles) {
  if (!ctx || !handles) return fail(ctx, BS_ERR_INVALID_ARG, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(ctx, BS_ERR_INVALID_ARG, "bad rank/world");
  if (!ctx->xbuf) return fail(ctx, BS_ERR_INVALID_ARG, "bs_peer_export must come first");
  if (ctx->peer_world) return fail(ctx, BS_ERR_INVALID_ARG, "context already connected");
  BS_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  std::vector<uint32_t*> table((size_t)world, nullptr);
  const unsigned char* hb = static_cast<const unsigned char*>(handles);
  for (int r = 0; r < world; ++r) {
    if (r == rank) {
      table[r] = ctx->xbuf;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, hb + (size_t)r * BS_PEER_HANDLE_BYTES, sizeof h);
    void* ptr = nullptr;
    BS_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    ctx->peer_mapped.push_back(ptr);
    table[r] = static_cast<uint32_t*>(ptr);
  }
  BS_CUDA(cudaMalloc(reinterpret_cast<void**>(&ctx->peer_ptrs), sizeof(uint32_t*) * world),
          "cudaMalloc peer table");
  BS_CUDA(cudaMemcpy(ctx->peer_ptrs, table.data(), sizeof(uint32_t*) * world, cudaMemcpyHostToDevice),
          "copy peer table");
  ctx->peer_rank = rank;
  ctx->peer_world = world;
  return BS_OK;
}

int bs_peer_reduce(bs_ctx* ctx, const uint32_t* hist_local, const bs_window_params* p,
                   uint32_t* hist_global, bs_summary* summary, void* stream) {
  if (!ctx) return fail(nullptr, BS_ERR_INVALID_ARG, "ctx is NULL");
  int rc;
  if ((rc = check_params(ctx, p)) != BS_OK) return rc;
  if (!hist_local || !hist_global) return fail(ctx, BS_ERR_INVALID_ARG, "NULL buffer");
  if (ctx->peer_world < 1) return fail(ctx, BS_ERR_INVALID_ARG, "bs_peer_connect must come first");
  BS_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  BS_CUDA(bsk::launch_peer_reduce(ctx, hist_local, *p, hist_global, summary,
                                  static_cast<cudaStream_t>(stream)),
          "k_peer_reduce");
  return BS_OK;
}

static int pack_impl(bs_ctx* ctx, const bs_window_io* io, const bs_window_params* p,
                     cudaStream_t st) {
  if (io->tok_off && io->tokens && io->out_tokens && io->n > 0) {
    if (reinterpret_cast<uintptr_t>(io->out_tokens) & 15)
      return fail(ctx, BS_ERR_INVALID_ARG, "out_tokens must be 16-byte aligned");
    if (io->out_mask && (reinterpret_cast<uintptr_t>(io->out_mask) & 3))
      return fail(ctx, BS_ERR_INVALID_ARG, "out_mask must be 4-byte aligned");
    BS_CUDA(bsk::launch_pack(ctx, io->len, io->perm, io->tok_off, io->tokens, *p, io->batches,
                             0, -1, io->batches_cap, io->out_tokens, io->out_mask,
                             io->out_capacity, io->summary, st),
            "k_pack");
  }
  return BS_OK;
}

static int window_from_hist_impl(bs_ctx* ctx, const bs_window_io* io, const bs_window_params* p,
                                 cudaStream_t st) {
  int rc;
  if ((rc = boundaries_impl(ctx, io->hist, io->hist_global ? io->hist_global : io->hist, p,
                            io->init_edges, io->k_init, io->edges, io->changes, io->changes_cap,
                            io->seg_off, io->summary, st)) != BS_OK)
    return rc;
  bsk::prof_mark(ctx, 3, st);
  BS_CUDA(bsk::launch_order(ctx, io->len, io->cls, io->n, *p, io->perm, io->bucket, io->summary, st),
          "k_sort_pass");
  bsk::prof_mark(ctx, 4, st);
  // the bulk-staged pack reads one record per row: K5e writes them when it has the token
  // offsets (the pack of this call then skips k_pack_rowprep)
  const bool recs = io->tok_off && io->tokens && io->out_tokens && io->n > 0 &&
                    bsk::pack_uses_bulk(ctx, *p, io->out_tokens, io->out_mask);
  BS_CUDA(bsk::launch_size(ctx, io->len, io->perm, io->seg_off, io->n, *p, io->batches,
                           io->batches_cap, io->req_batch, io->req_row, io->summary, st,
                           recs ? io->tok_off : nullptr),
          "k_size");
  bsk::prof_mark(ctx, 9, st);
  if (p->dispatch) {
    if (!io->emit_order || !io->batch_emit)
      return fail(ctx, BS_ERR_INVALID_ARG, "dispatch needs emit_order and batch_emit");
    BS_CUDA(bsk::launch_dispatch(ctx, io->perm, io->seg_off, io->n, *p, io->batches,
                                 io->batches_cap, io->req_batch, io->req_row, io->emit_order,
                                 io->batch_emit, io->summary, st),
            "k_dispatch");
  }
  bsk::prof_mark(ctx, 10, st);
  if ((rc = pack_impl(ctx, io, p, st)) != BS_OK) return rc;
  bsk::prof_mark(ctx, 11, st);
  return BS_OK;
}

static int check_io(bs_ctx* ctx, const bs_window_io* io) {
  if (!io) return fail(ctx, BS_ERR_INVALID_ARG, "io is NULL");
  int rc;
  if ((rc = check_n(ctx, io->n)) != BS_OK) return rc;
  if (!io->hist || !io->edges || !io->perm || !io->seg_off || !io->batches || !io->req_batch ||
      !io->req_row || !io->summary)
    return fail(ctx, BS_ERR_INVALID_ARG, "a required window buffer is NULL");
  if (io->n > 0 && (!io->len || !io->cls)) return fail(ctx, BS_ERR_INVALID_ARG, "NULL input");
  if (io->batches_cap < 0 || io->changes_cap < 0 || io->out_capacity < 0)
    return fail(ctx, BS_ERR_INVALID_ARG, "negative capacity");
  return BS_OK;
}

namespace {
struct WindowScope {
  bs_ctx* c;
  ~WindowScope() {
    c->window_zeroed = false;
    c->prof_in_window = false;
  }
};
}  // namespace

int bs_window_schedule(bs_ctx* ctx, const bs_window_io* io, const bs_window_params* p,
                       void* stream) {
  if (!ctx) return fail(nullptr, BS_ERR_INVALID_ARG, "ctx is NULL");
  int rc;
  if ((rc = check_params(ctx, p)) != BS_OK || (rc = check_io(ctx, io)) != BS_OK) return rc;
  BS_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ctx->prof_in_window = true;
  WindowScope scope{ctx};  // clears window_zeroed / prof_in_window on every return
  bsk::prof_mark(ctx, 0, st);
  if (!ctx->nccl_comm && ctx->peer_world <= 1 &&
      bsk::small_window_ok(ctx, io->n, *p, io->init_edges ? io->k_init : 0)) {
    // K0: the whole schedule of a small window in one CTA (its time reads as stage 0)
    if (io->init_edges && (io->k_init < 1 || io->k_init > p->l_max))
      return fail(ctx, BS_ERR_INVALID_ARG, "k_init out of range");
    BS_CUDA(bsk::launch_window_small(ctx, io, *p, st), "k_window_small");
    for (int s = 1; s <= 10; ++s) bsk::prof_mark(ctx, s, st);
    if (io->tok_off && io->tokens && io->out_tokens && io->n > 0) {
      if (reinterpret_cast<uintptr_t>(io->out_tokens) & 15)
        return fail(ctx, BS_ERR_INVALID_ARG, "out_tokens must be 16-byte aligned");
      if (io->out_mask && (reinterpret_cast<uintptr_t>(io->out_mask) & 3))
        return fail(ctx, BS_ERR_INVALID_ARG, "out_mask must be 4-byte aligned");
      BS_CUDA(bsk::launch_pack_rows(ctx, io->tokens, *p, (int32_t)io->n, io->out_tokens,
                                    io->out_mask, io->out_capacity, io->summary, st),
              "k_pack_rows");
    }
    bsk::prof_mark(ctx, 11, st);
    return BS_OK;
  }
  BS_CUDA(bsk::launch_window_init(ctx, io->summary, io->n, io->hist,
                                  (int64_t)p->l_max * p->n_classes,
                                  bsk::sort_status_words(ctx, io->n, *p), st),
          "k_window_init");
  ctx->window_zeroed = true;  // the launchers below skip their memsets
  cudaError_t ek = bsk::launch_histogram(ctx, io->len, io->cls, io->n, *p, io->hist, io->summary, st);
  if (ek != cudaSuccess) {
    ctx->window_zeroed = ctx->prof_in_window = false;
    return cuda_fail(ctx, ek, "k_histogram");
  }
  bsk::prof_mark(ctx, 1, st);
  bs_window_io local = *io;
  local.hist_global = io->hist;
  if (ctx->nccl_comm) {  // C1 over NCCL, on this stream (capturable)
    if (!io->hist_global || io->hist_global == io->hist) {
      ctx->prof_in_window = false;
      return fail(ctx, BS_ERR_INVALID_ARG, "an NCCL-attached context needs io->hist_global");
    }
    std::string why;
    if (bsk::nccl_allreduce_hist(ctx, io->hist, const_cast<uint32_t*>(io->hist_global),
                                 (size_t)p->l_max * p->n_classes, st, &why)) {
      ctx->prof_in_window = false;
      return fail(ctx, BS_ERR_CUDA, why);
    }
    local.hist_global = io->hist_global;
  } else if (ctx->peer_world > 1) {  // C1 over peer memory (bs_peer_connect): io->hist_global required
    if (!io->hist_global || io->hist_global == io->hist) {
      ctx->prof_in_window = false;
      return fail(ctx, BS_ERR_INVALID_ARG, "a peer-connected context needs io->hist_global");
    }
    BS_CUDA(bsk::launch_peer_reduce(ctx, io->hist, *p, const_cast<uint32_t*>(io->hist_global),
                                    io->summary, st),
            "k_peer_reduce");
    local.hist_global = io->hist_global;
  }
  bsk::prof_mark(ctx, 2, st);
  rc = window_from_hist_impl(ctx, &local, p, st);
  ctx->prof_in_window = false;
  ctx->window_zeroed = false;
  return rc;
}

int bs_window_from_hist(bs_ctx* ctx, const bs_window_io* io, const bs_window_params* p,
                        void* stream) {
  if (!ctx) return fail(nullptr, BS_ERR_INVALID_ARG, "ctx is NULL");
  int rc;
  if ((rc = check_params(ctx, p)) != BS_OK || (rc = check_io(ctx, io)) != BS_OK) return rc;
  BS_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ctx->prof_in_window = true;
  bsk::prof_mark(ctx, 0, st);  // K1 and C1 ran before this call; their stages read as ~0
  bsk::prof_mark(ctx, 1, st);
  bsk::prof_mark(ctx, 2, st);
  rc = window_from_hist_impl(ctx, io, p, st);
  ctx->prof_in_window = false;
  return rc;
}

int bs_nccl_unique_id(void* id_out) {
  bs_ctx* ctx = nullptr;
  if (!id_out) return fail(ctx, BS_ERR_INVALID_ARG, "NULL argument");
  std::string why;
  if (bsk::nccl_unique_id(id_out, &why)) return fail(ctx, BS_ERR_CUDA, why);
  return BS_OK;
}

int bs_nccl_connect(bs_ctx* ctx, int32_t rank, int32_t world, const void* unique_id) {
  if (!ctx || !unique_id) return fail(ctx, BS_ERR_INVALID_ARG, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(ctx, BS_ERR_INVALID_ARG, "bad rank/world");
  if (ctx->nccl_comm) return fail(ctx, BS_ERR_INVALID_ARG, "context already has a communicator");
  BS_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  std::string why;
  void* comm = nullptr;
  if (bsk::nccl_comm_init(&comm, world, unique_id, rank, &why)) return fail(ctx, BS_ERR_CUDA, why);
  ctx->nccl_comm = comm;
  ctx->nccl_owned = true;
  ctx->nccl_rank = rank;
  ctx->nccl_world = world;
  return BS_OK;
}

int bs_set_nccl(bs_ctx* ctx, void* nccl_comm, int32_t rank, int32_t world) {
  if (!ctx) return fail(nullptr, BS_ERR_INVALID_ARG, "ctx is NULL");
  if (nccl_comm && (world < 1 || rank < 0 || rank >= world))
    return fail(ctx, BS_ERR_INVALID_ARG, "bad rank/world");
  std::string why;
  if (nccl_comm && bsk::nccl_status(&why)) return fail(ctx, BS_ERR_NOT_BUILT, why);
  if (ctx->nccl_owned) bsk::nccl_comm_destroy(ctx->nccl_comm);
  ctx->nccl_comm = nccl_comm;
  ctx->nccl_owned = false;
  ctx->nccl_rank = nccl_comm ? rank : -1;
  ctx->nccl_world = nccl_comm ? world : 0;
  return BS_OK;
}

int bs_nccl_allreduce(bs_ctx* ctx, const uint32_t* hist_local, const bs_window_params* p,
                      uint32_t* hist_global, void* stream) {
  if (!ctx) return fail(nullptr, BS_ERR_INVALID_ARG, "ctx is NULL");
  int rc;
  if ((rc = check_params(ctx, p)) != BS_OK) return rc;
  if (!hist_local || !hist_global) return fail(ctx, BS_ERR_INVALID_ARG, "NULL buffer");
  if (!ctx->nccl_comm) return fail(ctx, BS_ERR_INVALID_ARG, "no communicator attached");
  BS_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  std::string why;
  if (bsk::nccl_allreduce_hist(ctx, hist_local, hist_global, (size_t)p->l_max * p->n_classes,
                               static_cast<cudaStream_t>(stream), &why))
    return fail(ctx, BS_ERR_CUDA, why);
  return BS_OK;
}

int bs_monitor_bins(bs_ctx* ctx, const uint32_t* hist, const bs_window_params* p, int32_t bins,
                    uint64_t* out, void* stream) {
  if (!ctx) return fail(nullptr, BS_ERR_INVALID_ARG, "ctx is NULL");
  int rc;
  if ((rc = check_params(ctx, p)) != BS_OK) return rc;
  if (!hist || !out || bins < 1 || bins > 4096) return fail(ctx, BS_ERR_INVALID_ARG, "bad arguments");
  BS_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  BS_CUDA(bsk::launch_monitor_bins(ctx, hist, *p, bins, out, static_cast<cudaStream_t>(stream)),
          "k_monitor_bins");
  return BS_OK;
}

int bs_monitor(bs_ctx* ctx, const uint32_t* hist, const bs_window_params* p, int32_t bins,
               const int32_t* edges, int32_t k, uint64_t* counts_out, double* stats_out,
               void* stream) {
  if (!ctx) return fail(nullptr, BS_ERR_INVALID_ARG, "ctx is NULL");
  int rc;
  if ((rc = check_params(ctx, p)) != BS_OK) return rc;
  if (!hist || !counts_out || bins < 1 || bins > 4096)
    return fail(ctx, BS_ERR_INVALID_ARG, "bad arguments");
  if (edges && (k < 1 || k > p->l_max || !stats_out))
    return fail(ctx, BS_ERR_INVALID_ARG, "edges need 1 <= k <= l_max and stats_out");
  BS_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  BS_CUDA(bsk::launch_monitor(ctx, hist, *p, bins, edges, k, counts_out, stats_out,
                              static_cast<cudaStream_t>(stream)),
          "k_monitor");
  ++ctx->launches;
  return BS_OK;
}

int bs_profile_enable(bs_ctx* ctx, int32_t max_steps) {
  if (!ctx) return fail(nullptr, BS_ERR_INVALID_ARG, "ctx is NULL");
  if (max_steps < 0) return fail(ctx, BS_ERR_INVALID_ARG, "max_steps must be >= 0");
  BS_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  for (cudaEvent_t e : ctx->prof_events) cudaEventDestroy(e);
  ctx->prof_events.clear();
  ctx->prof_steps = 0;
  ctx->prof_recorded = 0;
  const size_t ne = (size_t)max_steps * (BS_STAGES + 1);
  for (size_t i = 0; i < ne; ++i) {
    cudaEvent_t e;
    BS_CUDA(cudaEventCreate(&e), "cudaEventCreate");
    ctx->prof_events.push_back(e);
  }
  ctx->prof_steps = max_steps;
  return BS_OK;
}

int bs_profile_read(bs_ctx* ctx, float* stage_ms, int32_t* steps_out) {
  if (!ctx || !stage_ms || !steps_out) return fail(ctx, BS_ERR_INVALID_ARG, "NULL argument");
  BS_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
  for (int s = 0; s < BS_STAGES; ++s) stage_ms[s] = 0.f;
  for (int k = 0; k < ctx->prof_recorded; ++k) {
    cudaEvent_t* ev = &ctx->prof_events[(size_t)k * (BS_STAGES + 1)];
    BS_CUDA(cudaEventSynchronize(ev[BS_STAGES]), "cudaEventSynchronize");
    for (int s = 0; s < BS_STAGES; ++s) {
      float ms = 0.f;
      BS_CUDA(cudaEventElapsedTime(&ms, ev[s], ev[s + 1]), "cudaEventElapsedTime");
      stage_ms[s] += ms;
    }
  }
  *steps_out = ctx->prof_recorded;
  ctx->prof_recorded = 0;
  return BS_OK;
}

int64_t bs_launch_count(const bs_ctx* ctx) { return ctx ? ctx->launches : 0; }

}  // extern "C"

static_assert(sizeof(bs_window_params) == 104, "bs_window_params layout (Python binding)");
static_assert(sizeof(bs_batch) == 64, "bs_batch layout");
static_assert(sizeof(bs_summary) == 256, "bs_summary layout");
static_assert(sizeof(bs_window_io) == 192, "bs_window_io layout");
