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
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    bs_summary z = {};
    z.n_requests = n;
    *s = z;
  }
}

cudaError_t launch_init_summary(bs_summary* s, int64_t n, cudaStream_t st) {
  k_init_summary<<<1, 32, 0, st>>>(s, n);
  return cudaGetLastError();
}

cudaError_t launch_histogram(bs_ctx* ctx, const int32_t* len, const uint8_t* cls, int64_t n,
                             const bs_window_params& p, uint32_t* hist, bs_summary* summary,
                             cudaStream_t st) {
  const int32_t L = p.l_max, C = p.n_classes;
  cudaError_t e = cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (size_t)L * C, st);
  if (e != cudaSuccess || n == 0) return e;
  // privatised head: <= 64 KB of shared counters per CTA (3 CTAs / SM)
  const int32_t H = (int32_t)std::min<int64_t>(L, (64 * 1024 / 4) / C);
  const size_t smem = sizeof(uint32_t) * (size_t)C * H;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_histogram<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_histogram<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    attr_set = true;
  }
  const int threads = 512;
  // >= ept elements per thread and at most 2 CTAs per SM: the per-CTA zero/flush of the
  // privatised bins stays well below the elements each CTA reads
  const int agg = ctx->hist_agg;
  static int ept = 0, maxb = 0;
  if (ept == 0) {  // tuning hooks
    const char* v = getenv("BS_HIST_EPT");
    ept = v ? atoi(v) : 4;
    const char* m = getenv("BS_HIST_MAXB");
    maxb = m ? atoi(m) : 2 * ctx->num_sms;
  }
  int64_t blocks = (n + (int64_t)ept * threads - 1) / ((int64_t)ept * threads);
  blocks = std::min<int64_t>(blocks, maxb);
  blocks = std::max<int64_t>(blocks, 1);
  const int vec_ok = ((reinterpret_cast<uintptr_t>(len) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(cls) & 3) == 0);
  if (agg)
    k_histogram<true><<<(unsigned)blocks, threads, smem, st>>>(len, cls, n, L, C, p.truncate, H,
                                                             vec_ok, hist, summary);
  else
    k_histogram<false><<<(unsigned)blocks, threads, smem, st>>>(len, cls, n, L, C, p.truncate, H,
                                                              vec_ok, hist, summary);
  ++ctx->launches;
  return cudaGetLastError();
}

// f2: 64-bin monitor view, bin = (x * bins) // L (memory_model.py:125-130 with
// range (0, L), pd_sim.py:829-831; integer identity pinned in SURVEY App. B P9).
__global__ void k_monitor_bins(const uint32_t* __restrict__ hist, int32_t L, int32_t C,
                               int32_t bins, unsigned long long* out) {
  extern __shared__ unsigned long long sb[];
  for (int i = threadIdx.x; i < bins; i += blockDim.x) sb[i] = 0;
  __syncthreads();
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < L;
       x += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long h = 0;
    for (int c = 0; c < C; ++c) h += hist[(int64_t)c * L + x];
    if (h) atomicAdd(&sb[(x * bins) / L], h);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < bins; i += blockDim.x)
    if (sb[i]) atomicAdd(&out[i], sb[i]);
}

cudaError_t launch_monitor_bins(const uint32_t* hist, const bs_window_params& p, int32_t bins,
                                uint64_t* out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(uint64_t) * bins, st);
  if (e != cudaSuccess) return e;
  int blocks = (int)std::min<int64_t>((p.l_max + 255) / 256, 64);
  k_monitor_bins<<<blocks, 256, sizeof(unsigned long long) * bins, st>>>(
      hist, p.l_max, p.n_classes, bins, reinterpret_cast<unsigned long long*>(out));
  return cudaGetLastError();
}

}  // namespace bsk
