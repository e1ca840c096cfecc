// K3 assign + K4 order — stable LSD radix sort on packed drain-order slots.
//
// Reference: the window drains buckets left to right, ONLINE before OFFLINE
// (pd_sim.py:449-450), each form_batch call re-sorting the bucket's class with
// order_requests (batch_controller.py:33-41): SJF (len, arrival, id), LJF
// (-len, arrival, id), FCFS/EARLIEST_ARRIVAL (arrival, id).  The whole drain
// order is therefore one total order on (bucket, class, policy key, arrival).
//
// B200 design: K2 maps every (class, length) pair to a dense "slot" that
// encodes (bucket, class, len | ~len | 0) in drain order (slot_lut); arrival is
// the index, so a STABLE sort of indices by slot reproduces the reference order
// exactly.  The sort is a onesweep-style LSD radix sort: <= 8-bit digits, each
// pass one kernel with decoupled look-back over tiles (dynamic tile ids), warp
// match_any ranking in shared memory, and a shared-memory local sort so the
// scatter writes contiguous runs.  Digit offsets come from K2 (derived from the
// histogram), so there is no upsweep pass.  Pass 1 reads len/cls directly and
// also emits the K3 bucket id; the last pass writes only the permutation.
#include <cooperative_groups.h>
#include <cstdlib>

#include "ctx.cuh"

namespace bsk {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
// items per thread: 8 (2048-key tiles) for windows < 4M keys (more CTAs in flight),
// 16 (4096-key tiles) above (fewer look-back steps)
constexpr int kItemsSmall = 8;
constexpr int kItemsLarge = 16;
#ifndef BS_SORT_MINB16
#define BS_SORT_MINB16 4
#endif
#ifndef BS_SORT_MINB8
#define BS_SORT_MINB8 4
#endif
constexpr int kSortMinBlocks16 = BS_SORT_MINB16;
constexpr int kSortMinBlocks8 = BS_SORT_MINB8;

__global__ void k_assign(const int32_t* __restrict__ len, int64_t n, int32_t L, int32_t truncate,
                         const int32_t* __restrict__ lut, int32_t* __restrict__ bucket_out,
                         bs_summary* sum) {
  pdl_prologue();
  unsigned fl = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    bucket_out[i] = lut[eff_len(len[i], L, truncate, fl)];
  latch_flags(sum, fl);
}

// 16-item tiles (windows >= 4M requests): at most 64 registers so 4 CTAs share an SM
// (110 registers allowed only 2 — 25 % of the warp slots, latency-bound: C3 order
// 557 -> 427 us, with a few spilled registers); 8-item tiles likewise 64 registers
// (an explicit min-blocks of 1 let them grow to 96 and cost C2 ~5 us per window)
template <bool kFirst, bool kLast, int kItems>
__global__ void __launch_bounds__(kSortThreads, kItems >= 16 ? kSortMinBlocks16 : kSortMinBlocks8)
    k_sort_pass(const int32_t* __restrict__ len, const uint8_t* __restrict__ cls,
                const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, int64_t n,
                int32_t L, int32_t C, int32_t truncate, const uint32_t* __restrict__ slot_lut,
                const int32_t* __restrict__ lut, int32_t* __restrict__ bucket_out, int shift,
                int bits, const uint32_t* __restrict__ bins_cnt, uint32_t* __restrict__ status,
                uint32_t* __restrict__ tile_ctr) {
  pdl_prologue();
  constexpr int kTile = kSortThreads * kItems;
  __shared__ uint32_t s_cnt[kSortWarps][256];
  __shared__ uint32_t s_keys[kTile];
  __shared__ uint32_t s_vals[kTile];
  __shared__ uint32_t s_dstart[256];
  __shared__ int64_t s_gbase[256];
  __shared__ uint32_t s_scan[33];
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_binbase[256];

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t nb = 1u << bits, dmask = nb - 1u;
  if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
  for (int i = tid; i < kSortWarps * 256; i += kSortThreads) (&s_cnt[0][0])[i] = 0;
  {  // global digit offsets of this pass: exclusive scan of the K2c digit counts
    uint32_t t_;
    const uint32_t o = block_excl_scan<uint32_t>(tid < (int)nb ? bins_cnt[tid] : 0u, s_scan, &t_);
    s_binbase[tid] = o;
  }
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t tbase = (int64_t)tile * kTile;
  const int64_t wbase = tbase + (int64_t)w * (32 * kItems);

  // values: the first pass sorts the indices themselves (val = e, recomputed where needed,
  // so the 16-item tiles fit 64 registers without spilling)
  uint32_t key[kItems], val[kFirst ? 1 : kItems], rank[kItems];
  unsigned fl = 0;
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int64_t e = wbase + k * 32 + lane;
    if (e < n) {
      if (kFirst) {
        const int32_t x = eff_len(len[e], L, truncate, fl);
        const int32_t c = eff_cls(cls[e], C, fl);
        key[k] = slot_lut[(int64_t)c * L + x];
        if (bucket_out) bucket_out[e] = lut[x];
      } else {
        key[k] = keys_in[e];
        val[k] = vals_in[e];
      }
    } else {
      key[k] = 0xffffffffu;
      if (!kFirst) val[k] = 0;
    }
  }
  // ---- warp-level stable ranking (items in index order: k-major, lane-minor) ----
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int64_t e = wbase + k * 32 + lane;
    const bool valid = e < n;
    const uint32_t d = valid ? ((key[k] >> shift) & dmask) : 0xffffffffu;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (valid && lane == leader) {
      old = s_cnt[w][d];
      s_cnt[w][d] = old + __popc(peers);
    }
    old = __shfl_sync(0xffffffffu, old, leader);
    rank[k] = old + __popc(peers & lanemask_lt());
    __syncwarp();
  }
  __syncthreads();
  // ---- per digit: exclusive over warps, tile totals, look-back --------------------
  uint32_t tile_cnt = 0;
  if (tid < (int)nb) {
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ++ww) {
      const uint32_t v = s_cnt[ww][tid];
      s_cnt[ww][tid] = tile_cnt;
      tile_cnt += v;
    }
  }
  uint32_t tot;
  const uint32_t dstart = block_excl_scan<uint32_t>(tid < (int)nb ? tile_cnt : 0u, s_scan, &tot);
  if (tid < (int)nb) {
    s_dstart[tid] = dstart;
    uint32_t excl = 0;
    uint32_t* my = status + (int64_t)tile * nb + tid;
    if (tile == 0) {
      st_relaxed(my, kStatPrefix | tile_cnt);
    } else {
      st_relaxed(my, kStatAgg | tile_cnt);
      int64_t t = (int64_t)tile - 1;
      for (;;) {
        uint32_t v;
        do { v = ld_relaxed(status + t * nb + tid); } while ((v >> 30) == 0);
        excl += v & kStatMask;
        if (v & kStatPrefix) break;
        --t;
      }
      st_relaxed(my, kStatPrefix | (excl + tile_cnt));
    }
    s_gbase[tid] = (int64_t)s_binbase[tid] + excl - dstart;
  }
  __syncthreads();
  // ---- local sort into shared memory -----------------------------------------------
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int64_t e = wbase + k * 32 + lane;
    if (e < n) {
      const uint32_t d = (key[k] >> shift) & dmask;
      const uint32_t lp = s_dstart[d] + s_cnt[w][d] + rank[k];
      s_keys[lp] = key[k];
      s_vals[lp] = kFirst ? (uint32_t)e : val[kFirst ? 0 : k];
    }
  }
  __syncthreads();
  // ---- scatter contiguous digit runs --------------------------------------------------
  const int64_t tn = (n - tbase) < kTile ? (n - tbase) : (int64_t)kTile;
  for (int i = tid; i < tn; i += kSortThreads) {
    const uint32_t kk = s_keys[i];
    const uint32_t d = (kk >> shift) & dmask;
    const int64_t g = s_gbase[d] + i;
    keys_out[g] = kk;  // the last pass too: K5 maps sorted slots to segments
    vals_out[g] = s_vals[i];
  }
  (void)fl;  // range errors on the same inputs are latched by K1
}

cudaError_t launch_assign(bs_ctx* ctx, const int32_t* len, int64_t n, const bs_window_params& p,
                          int32_t* bucket_out, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 8LL * ctx->num_sms);
  launch_k(ctx, k_assign, dim3((unsigned)blocks), dim3(256), 0, st, false, len, n, p.l_max, p.truncate, ctx->lut, bucket_out,
                                              nullptr);
  ++ctx->launches;
  return cudaGetLastError();
}

template <int kItems>
static cudaError_t order_passes(bs_ctx* ctx, const int32_t* len, const uint8_t* cls, int64_t n,
                                const bs_window_params& p, int32_t* perm_out,
                                int32_t* bucket_out, const SortPlan& sp, cudaStream_t st) {
  constexpr int kTile = kSortThreads * kItems;
  const int64_t tiles = (n + kTile - 1) / kTile;
  const size_t stat_words = (size_t)tiles * 256;
  cudaError_t e = cudaSuccess;
  if (!ctx->window_zeroed) {  // the fused window zeroes these in k_window_init
    e = cudaMemsetAsync(ctx->status, 0, sizeof(uint32_t) * stat_words * sp.passes, st);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(ctx->tile_ctr, 0, sizeof(uint32_t) * 4, st);
    if (e != cudaSuccess) return e;
  }
  const uint32_t* kin = nullptr;
  const uint32_t* vin = nullptr;
  uint32_t* kbuf[2] = {ctx->keysA, ctx->keysB};
  uint32_t* vbuf[2] = {ctx->valsA, ctx->valsB};
  for (int q = 0; q < sp.passes; ++q) {
    const bool first = q == 0, last = q == sp.passes - 1;
    uint32_t* kout = kbuf[q & 1];
    uint32_t* vout = last ? reinterpret_cast<uint32_t*>(perm_out) : vbuf[q & 1];
    const uint32_t* bb = ctx->bins_cnt + q * 256;
    uint32_t* stt = ctx->status + stat_words * q;
    uint32_t* tc = ctx->tile_ctr + q;
    const int shift = q * sp.bits;
#define BS_SORT_LAUNCH(F, LST)                                                                \
  launch_k(ctx, k_sort_pass<F, LST, kItems>, dim3((unsigned)tiles), dim3(kSortThreads), 0, st, false,                       \
      len, cls, kin, vin, kout, vout, n, p.l_max, p.n_classes, p.truncate, ctx->slot_lut,     \
      ctx->lut, bucket_out, shift, sp.bits, bb, stt, tc)
    if (first && last) BS_SORT_LAUNCH(true, true);
    else if (first) BS_SORT_LAUNCH(true, false);
    else if (last) BS_SORT_LAUNCH(false, true);
    else BS_SORT_LAUNCH(false, false);
#undef BS_SORT_LAUNCH
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ++ctx->launches;
    kin = kout;
    vin = vout;
  }
  ctx->sorted_keys = kin;
  return cudaSuccess;
}

// words of look-back status (all passes) launch_order zeroes for a window of n requests
int64_t sort_status_words(const bs_ctx* ctx, int64_t n, const bs_window_params& p) {
  if (n == 0) return 0;
  const SortPlan sp = sort_plan(p.l_max, p.n_classes);
  const int force = ctx->sort_items;
  const int items = (force == 8 || (force != 16 && n < (int64_t)4 << 20)) ? kItemsSmall : kItemsLarge;
  const int64_t tiles = (n + (int64_t)kSortThreads * items - 1) / ((int64_t)kSortThreads * items);
  return tiles * 256 * sp.passes;
}

cudaError_t launch_order(bs_ctx* ctx, const int32_t* len, const uint8_t* cls, int64_t n,
                         const bs_window_params& p, int32_t* perm_out, int32_t* bucket_out,
                         bs_summary* summary, cudaStream_t st) {
  (void)summary;
  if (n == 0) return cudaSuccess;
  const SortPlan sp = sort_plan(p.l_max, p.n_classes);
  const int force = ctx->sort_items;  // tuning hook BS_SORT_ITEMS=8|16 (read by bs_create)
  if (force == 8 || (force != 16 && n < (int64_t)4 << 20))
    return order_passes<kItemsSmall>(ctx, len, cls, n, p, perm_out, bucket_out, sp, st);
  return order_passes<kItemsLarge>(ctx, len, cls, n, p, perm_out, bucket_out, sp, st);
}

}  // namespace bsk
