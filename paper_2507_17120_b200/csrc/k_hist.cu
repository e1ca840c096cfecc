// K1 — per-(class, length) histogram of the window.
//
// Replaces the per-request counting the reference does on every assign
// (Bucket.short_count / len(requests), bucket_manager.py:31-32,39-40,126-127) and
// the O(N) mean in current_n_max (batch_controller.py:100-104): all bucket counts,
// short counts, N and sum(len) are prefix-sum reads of this histogram (K2).
//
// B200 mapping: HBM-bound read of len (int32) + cls (u8) with 128-bit / 32-bit
// vector loads; counts privatised per CTA in shared memory for the dense head
// bins (lengths < H); tail bins (long-context lengths >= H) go straight to L2
// atomics; non-zero shared bins are flushed with one L2 atomic each.  Two forms of
// the shared-memory update: plain per-lane atomics (default) and warp-aggregated
// (__match_any_sync: lanes holding the same (class, length) key issue one atomic,
// BS_HIST_AGG=1).  On the BASELINE length distributions the keys inside a warp are
// mostly distinct, so aggregation only adds the MATCH latency: measured on B200,
// plain 18.5 us vs aggregated 26.5 us at C2 (1M), 50 vs 152 us at C3 (16M).
#include <cstdlib>

#include "ctx.cuh"

namespace bsk {

template <bool kAgg>
__device__ __forceinline__ void hist_add(int32_t x, int32_t c, int32_t L, int32_t H,
                                         uint32_t* sh, uint32_t* __restrict__ hist) {
  if (!kAgg) {
    if (x < H) atomicAdd(&sh[(unsigned)c * (unsigned)H + (unsigned)x], 1u);
    else atomicAdd(&hist[(unsigned)c * (unsigned)L + (unsigned)x], 1u);
    return;
  }
  if (x < H) {
    const unsigned key = (unsigned)c * (unsigned)H + (unsigned)x;
    const unsigned peers = __match_any_sync(__activemask(), key);
    if ((int)lane_id() == __ffs(peers) - 1) atomicAdd(&sh[key], (uint32_t)__popc(peers));
  } else {
    const unsigned key = (unsigned)c * (unsigned)L + (unsigned)x;
    const unsigned peers = __match_any_sync(__activemask(), key);
    if ((int)lane_id() == __ffs(peers) - 1) atomicAdd(&hist[key], (uint32_t)__popc(peers));
  }
}

template <bool kAgg>
__global__ void __launch_bounds__(512) k_histogram(const int32_t* __restrict__ len,
                                                   const uint8_t* __restrict__ cls, int64_t n,
                                                   int32_t L, int32_t C, int32_t truncate,
                                                   int32_t H, int vec_ok,
                                                   uint32_t* __restrict__ hist, bs_summary* sum) {
  pdl_prologue();
  extern __shared__ uint32_t sh[];  // [C][H]
  for (int i = threadIdx.x; i < C * H; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  unsigned fl = 0;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if (vec_ok) {
    const int64_t nv = n >> 2;
    const int4* len4 = reinterpret_cast<const int4*>(len);
    const uchar4* cls4 = reinterpret_cast<const uchar4*>(cls);
    for (int64_t v = tid; v < nv; v += stride) {
      const int4 l = __ldg(len4 + v);
      const uchar4 c = __ldg(cls4 + v);
      hist_add<kAgg>(eff_len(l.x, L, truncate, fl), eff_cls(c.x, C, fl), L, H, sh, hist);
      hist_add<kAgg>(eff_len(l.y, L, truncate, fl), eff_cls(c.y, C, fl), L, H, sh, hist);
      hist_add<kAgg>(eff_len(l.z, L, truncate, fl), eff_cls(c.z, C, fl), L, H, sh, hist);
      hist_add<kAgg>(eff_len(l.w, L, truncate, fl), eff_cls(c.w, C, fl), L, H, sh, hist);
    }
    done = nv << 2;
  }
  for (int64_t i = done + tid; i < n; i += stride)
    hist_add<kAgg>(eff_len(__ldg(len + i), L, truncate, fl), eff_cls(__ldg(cls + i), C, fl), L, H, sh,
             hist);
  __syncthreads();
  for (int i = threadIdx.x; i < C * H; i += blockDim.x) {
    const uint32_t v = sh[i];
    if (v) atomicAdd(&hist[(i / H) * L + (i % H)], v);
  }
  latch_flags(sum, fl);
}

__global__ void k_init_summary(bs_summary* s, int64_t n) {
  pdl_prologue();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    bs_summary z = {};
    z.n_requests = n;
    *s = z;
  }
}

cudaError_t launch_init_summary(const bs_ctx* ctx, bs_summary* s, int64_t n, cudaStream_t st) {
  launch_k(ctx, k_init_summary, dim3(1), dim3(32), 0, st, false, s, n);
  return cudaGetLastError();
}

// The fused window's first kernel: the summary plus every buffer the window's kernels
// accumulate into (K1 histogram, K4 look-back status words and tile counters, K5 misc
// counters) zeroed in one grid instead of memset nodes, which would cut the chain of
// programmatically dependent launches.
__global__ void k_window_init(bs_summary* s, int64_t n, uint32_t* hist, int64_t hist_words,
                              uint32_t* status, int64_t status_words, uint32_t* tile_ctr,
                              int32_t* misc) {
  pdl_prologue();
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (tid == 0 && s) {
    bs_summary z = {};
    z.n_requests = n;
    *s = z;
  }
  if (tid < 4) tile_ctr[tid] = 0;
  if (tid < 128) misc[tid] = 0;
  for (int64_t i = tid; i < hist_words; i += stride) hist[i] = 0;
  for (int64_t i = tid; i < status_words; i += stride) status[i] = 0;
}

cudaError_t launch_window_init(bs_ctx* ctx, bs_summary* s, int64_t n, uint32_t* hist,
                               int64_t hist_words, int64_t status_words, cudaStream_t st) {
  const int64_t words = std::max<int64_t>(hist_words, status_words);
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((words + 1023) / 1024, 4LL * ctx->num_sms));
  launch_k(ctx, k_window_init, dim3((unsigned)blocks), dim3(256), 0, st, false, s, n, hist,
           hist_words, ctx->status, status_words, ctx->tile_ctr, ctx->misc);
  ++ctx->launches;
  return cudaGetLastError();
}

// privatised head of K1: <= 48 KB of shared counters per CTA, so a K1 CTA fits on an SM
// beside a bulk-staged pack CTA (168 KB) of another window in flight (with 64 KB, C3's
// four-class K1 waited for the pack to end); lengths beyond the head go to L2 atomics
constexpr int kHistSmem = 48 * 1024;

// per-context setup on the context's device (bs_create)
cudaError_t hist_prepare(bs_ctx* ctx) {
  (void)ctx;
  cudaError_t e = cudaFuncSetAttribute(k_histogram<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kHistSmem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_histogram<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kHistSmem);
  return e;
}

cudaError_t launch_histogram(bs_ctx* ctx, const int32_t* len, const uint8_t* cls, int64_t n,
                             const bs_window_params& p, uint32_t* hist, bs_summary* summary,
                             cudaStream_t st) {
  const int32_t L = p.l_max, C = p.n_classes;
  cudaError_t e = cudaSuccess;
  if (!ctx->window_zeroed) e = cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (size_t)L * C, st);
  if (e != cudaSuccess || n == 0) return e;
  const int32_t H = (int32_t)std::min<int64_t>(L, (kHistSmem / 4) / C);
  const size_t smem = sizeof(uint32_t) * (size_t)C * H;
  const int threads = 512;
  // >= ept elements per thread and at most 2 CTAs per SM: the per-CTA zero/flush of the
  // privatised bins stays well below the elements each CTA reads
  const int agg = ctx->hist_agg;
  const int ept = ctx->hist_ept, maxb = ctx->hist_maxb;  // tuning hooks read by bs_create
  int64_t blocks = (n + (int64_t)ept * threads - 1) / ((int64_t)ept * threads);
  blocks = std::min<int64_t>(blocks, maxb);
  blocks = std::max<int64_t>(blocks, 1);
  const int vec_ok = ((reinterpret_cast<uintptr_t>(len) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(cls) & 3) == 0);
  if (agg)
    launch_k(ctx, k_histogram<true>, dim3((unsigned)blocks), dim3(threads), smem, st, false, len, cls, n, L, C, p.truncate, H,
                                                             vec_ok, hist, summary);
  else
    launch_k(ctx, k_histogram<false>, dim3((unsigned)blocks), dim3(threads), smem, st, false, len, cls, n, L, C, p.truncate, H,
                                                              vec_ok, hist, summary);
  ++ctx->launches;
  return cudaGetLastError();
}

// f2: the monitor histogram of pd_sim.py:829-831 — LengthHistogram.from_samples(
// lengths, bins, range=(0, L)) (memory_model.py:125-130), i.e. np.histogram over
// float64 samples with uniform edges e_i = i * (L / bins) (np.linspace; e_bins = L).
// The bin of an integer length x is restated from numpy's uniform-bin path
// (numpy/lib/_histograms_impl.py:851-861 in numpy 2.3.5): i = (int)((x / L) * bins),
// clamp to bins-1, then one step down if x < e_i and one step up if x >= e_{i+1}
// (except in the last bin).  For bins dividing L exactly this equals (x*bins)//L
// (SURVEY App. B P9); the correction keeps other bin counts identical too.
__device__ __forceinline__ double mon_edge(int i, int bins, double step, double Ld) {
  return i == bins ? Ld : __dmul_rn((double)i, step);
}

__device__ __forceinline__ int mon_bin(int64_t x, int bins, double step, double Ld) {
  const double xd = (double)x;
  int i = (int)__dmul_rn(__ddiv_rn(xd, Ld), (double)bins);
  if (i == bins) --i;
  if (xd < mon_edge(i, bins, step, Ld)) --i;
  if (xd >= mon_edge(i + 1, bins, step, Ld) && i != bins - 1) ++i;
  return i;
}

// One CTA: bin the per-(class, length) histogram into shared counters, then — when
// edges are given — expected_waste (memory_model.py:160-191) of the bucket partition
// edges[0..k]: bins left to right, skipping empty ones, acc += cnt * (1 - mid / up)
// with up the first bucket upper > mid, all in float64 in the reference's order
// (explicit _rn intrinsics: no FMA contraction), divided by the total mass.
__global__ void __launch_bounds__(1024) k_monitor(const uint32_t* __restrict__ hist, int32_t L,
                                                  int32_t C, int32_t bins,
                                                  const int32_t* __restrict__ edges, int32_t k,
                                                  unsigned long long* __restrict__ out,
                                                  double* __restrict__ stats) {
  pdl_prologue();
  extern __shared__ unsigned long long sb[];
  for (int i = threadIdx.x; i < bins; i += blockDim.x) sb[i] = 0;
  __syncthreads();
  const double Ld = (double)L;
  const double step = __ddiv_rn(Ld, (double)bins);
  for (int64_t x = threadIdx.x; x < L; x += blockDim.x) {
    unsigned long long h = 0;
    for (int c = 0; c < C; ++c) h += __ldg(hist + (int64_t)c * L + x);
    if (h) atomicAdd(&sb[mon_bin(x, bins, step, Ld)], h);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < bins; i += blockDim.x) out[i] = sb[i];
  if (threadIdx.x != 0 || stats == nullptr) return;
  double acc = 0.0, total = 0.0;
  for (int i = 0; i < bins; ++i) {
    const unsigned long long cnt = sb[i];
    total = __dadd_rn(total, (double)cnt);
    if (cnt == 0 || edges == nullptr) continue;
    const double mid = __ddiv_rn(__dadd_rn(mon_edge(i, bins, step, Ld),
                                           mon_edge(i + 1, bins, step, Ld)), 2.0);
    int lo = 1, hi = k + 1;  // first upper edges[j] (j in 1..k) with edges[j] > mid
    while (lo < hi) {
      const int m = (lo + hi) >> 1;
      if ((double)edges[m] > mid) hi = m; else lo = m + 1;
    }
    if (lo > k) { acc = __longlong_as_double(0x7ff8000000000000LL); continue; }  // not covered
    const double up = (double)edges[lo];
    acc = __dadd_rn(acc, __dmul_rn((double)cnt, __dsub_rn(1.0, __ddiv_rn(mid, up))));
  }
  stats[0] = total > 0.0 ? __ddiv_rn(acc, total) : __longlong_as_double(0x7ff8000000000000LL);
  stats[1] = total;
  stats[2] = acc;
}

cudaError_t launch_monitor(const bs_ctx* ctx, const uint32_t* hist, const bs_window_params& p,
                           int32_t bins, const int32_t* edges, int32_t k, uint64_t* out,
                           double* stats, cudaStream_t st) {
  launch_k(ctx, k_monitor, dim3(1), dim3(1024), sizeof(unsigned long long) * bins, st, false, 
      hist, p.l_max, p.n_classes, bins, edges, k, reinterpret_cast<unsigned long long*>(out),
      stats);
  return cudaGetLastError();
}

cudaError_t launch_monitor_bins(const bs_ctx* ctx, const uint32_t* hist, const bs_window_params& p,
                                int32_t bins, uint64_t* out, cudaStream_t st) {
  return launch_monitor(ctx, hist, p, bins, nullptr, 0, out, nullptr, st);
}

}  // namespace bsk
