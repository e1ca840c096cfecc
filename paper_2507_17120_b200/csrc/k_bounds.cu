// K2 — adaptive bucket boundaries (Alg. 1) + n_max + K3/K4 lookup tables.
//
// Restates BucketSet.adjust_buckets (bucket_manager.py:133-191) on prefix sums
// of the window histogram instead of per-request deques:
//   count(b) = P[up] - P[low], short(b) = P[mid] - P[low], mid = (low+up)//2
//   (bucket_manager.py:31-32).  One pass = merge when total < n_max (:148-156),
//   no change when total == n_max (:158-160), otherwise split every bucket with
//   count > n_max and short > theta*count (float64 product, :162-164) at mid;
//   width-1 buckets log a skip (:175-178).  Passes repeat up to max_passes
//   (<= 0: until one yields no split — the window fixpoint).
// n_max = BatchController.current_n_max (batch_controller.py:93-104) evaluated
// with CPython's float floor division, bit-exact.
//
// B200 mapping.  l_max <= 16384: one fused CTA (k_bounds_small, below).  Larger
// l_max (long context), three launches:
//   K2a  k_prefix_tiles  one CTA per 4096 lengths: tile-local exclusive prefixes of
//                        the total and per-class histograms, tile totals, sum(len)
//   K2b  k_boundaries    one 1024-thread CTA: carries over the tiles, n_max, the
//                        split/merge passes on an edge bitmask in shared memory
//                        (block-scan compaction + one thread per bucket, change
//                        log in bucket order), segment offsets / radix slot bases
//   K2c  k_tables        grid over (class, length): bucket LUT (K3), radix slot per
//                        (class, length) and the per-pass digit counts for K4,
//                        derived from the histogram so K4 needs no upsweep.
#include "ctx.cuh"

namespace bsk {

constexpr int kBT = 1024;
// block of the fused small-L K2 (the code is block-size agnostic; 512 threads measured
// 41 vs 35 us at C2 and gained nothing with windows in flight)
constexpr int kSmallBT = 1024;
constexpr int kSmallBTMin = 2;  // <= 32 registers: fits on an SM beside a pack CTA of another window
constexpr int kEcap = 8192;   // edges kept in shared memory when l_max < kEcap

// p.policy[c] without a dynamically indexed kernel-parameter array (which the compiler
// copies to local memory): an unrolled select over the BS_MAX_CLASSES entries
__device__ __forceinline__ int policy_of(const bs_window_params& p, int c) {
  int pol = p.policy[0];
#pragma unroll
  for (int i = 1; i < BS_MAX_CLASSES; ++i)
    if (c == i) pol = p.policy[i];
  return pol;
}

// ---------------------------------------------------------------------------- K2a
__global__ void __launch_bounds__(1024)
    k_prefix_tiles(const uint32_t* __restrict__ hist_local, const uint32_t* __restrict__ hist_global,
                   int32_t L, int32_t C, uint32_t* __restrict__ P, uint32_t* __restrict__ PcL,
                   uint32_t* __restrict__ tile_tot, unsigned long long* __restrict__ tile_slen) {
  pdl_prologue();
  __shared__ uint32_t s32[33];
  __shared__ uint64_t s64[33];
  const int t = blockIdx.x;
  const int64_t x0 = (int64_t)t * kTileX + threadIdx.x * 4;
  uint32_t h[4];
  uint32_t sum = 0;
  uint64_t sl = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t x = x0 + i;
    h[i] = 0;
    if (x < L)
      for (int c = 0; c < C; ++c) h[i] += hist_global[(int64_t)c * L + x];
    sum += h[i];
    sl += (uint64_t)h[i] * (uint64_t)x;
  }
  uint32_t tot;
  uint32_t run = block_excl_scan<uint32_t>(sum, s32, &tot);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (x0 + i < L) P[x0 + i] = run;
    run += h[i];
  }
  uint64_t sltot;
  block_excl_scan<uint64_t>(sl, s64, &sltot);
  if (threadIdx.x == 0) {
    tile_tot[(int64_t)t * (C + 1) + C] = tot;
    tile_slen[t] = sltot;
  }
  for (int c = 0; c < C; ++c) {
    uint32_t v[4], s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[i] = (x0 + i < L) ? hist_local[(int64_t)c * L + x0 + i] : 0u;
      s += v[i];
    }
    uint32_t tc;
    uint32_t rc = block_excl_scan<uint32_t>(s, s32, &tc);
    uint32_t* Pc = PcL + (int64_t)c * (L + 1);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (x0 + i < L) Pc[x0 + i] = rc;
      rc += v[i];
    }
    if (threadIdx.x == 0) tile_tot[(int64_t)t * (C + 1) + c] = tc;
  }
}

// ---------------------------------------------------------------------------- K2b
struct BoundsShared {
  uint64_t s64[33];
  uint32_t s32[33];
  int32_t si[33];
  int64_t n_max;
  uint32_t total;
  int32_t bad;
};

// compact the edge bitmask into E[0..K]; returns K (number of buckets)
__device__ int32_t compact_edges(const uint32_t* bm, int W, int32_t* E, BoundsShared& sh) {
  const int wc = (W + (int)blockDim.x - 1) / (int)blockDim.x;
  const int w0 = threadIdx.x * wc, w1 = min(W, w0 + wc);
  int32_t cnt = 0;
  for (int w = w0; w < w1; ++w) cnt += __popc(bm[w]);
  int32_t tot;
  int32_t off = block_excl_scan<int32_t>(cnt, sh.si, &tot);
  for (int w = w0; w < w1; ++w) {
    uint32_t b = bm[w];
    while (b) {
      const int bit = __ffs(b) - 1;
      E[off++] = w * 32 + bit;
      b &= b - 1;
    }
  }
  __syncthreads();
  return tot - 1;
}

__global__ void __launch_bounds__(kBT, 1)
    k_boundaries(const uint32_t* __restrict__ P, const uint32_t* __restrict__ PcL,
                 const uint32_t* __restrict__ tile_tot,
                 const unsigned long long* __restrict__ tile_slen, int32_t ntiles,
                 bs_window_params p, const int32_t* __restrict__ init_edges, int32_t k_init,
                 int32_t* __restrict__ edges_out, int32_t* __restrict__ changes_out,
                 int32_t changes_cap, int32_t* __restrict__ seg_off_out,
                 int32_t* __restrict__ gE, uint32_t* __restrict__ gbm, uint32_t* __restrict__ gwp,
                 int32_t* __restrict__ seg_base, uint32_t* __restrict__ tile_carry,
                 uint32_t* __restrict__ bins_cnt, int32_t* __restrict__ kinfo, bs_summary* sum) {
  pdl_prologue();
  extern __shared__ uint32_t dyn[];
  __shared__ BoundsShared sh;
  const int32_t L = p.l_max, C = p.n_classes;
  const int W = (L + 1 + 31) / 32;
  uint32_t* bm = dyn;                                          // [W] edge bitmask over [0, L]
  uint32_t* carry = dyn + W;                                   // [ntiles] total-hist carries
  int32_t* sE = reinterpret_cast<int32_t*>(dyn + W + ntiles);  // [kEcap] edges (small L)
  int32_t* E = (L + 1 <= kEcap) ? sE : gE;
  const int tid = threadIdx.x;

  // ---- A. carries over the K2a tiles, totals, n_max -------------------------------
  {
    uint32_t tot_all = 0;
    uint64_t sl_all = 0;
    for (int base = 0; base < ntiles; base += kBT) {
      const int t = base + tid;
      const uint32_t v = t < ntiles ? tile_tot[(int64_t)t * (C + 1) + C] : 0u;
      uint32_t tt;
      const uint32_t o = block_excl_scan<uint32_t>(v, sh.s32, &tt);
      if (t < ntiles) carry[t] = tot_all + o;
      tot_all += tt;
      const uint64_t s = t < ntiles ? tile_slen[t] : 0ull;
      uint64_t ts;
      block_excl_scan<uint64_t>(s, sh.s64, &ts);
      sl_all += ts;
    }
    for (int c = 0; c < C; ++c) {  // per-class carries (segment counts in E.)
      uint32_t run = 0;
      for (int base = 0; base < ntiles; base += kBT) {
        const int t = base + tid;
        const uint32_t v = t < ntiles ? tile_tot[(int64_t)t * (C + 1) + c] : 0u;
        uint32_t tt;
        const uint32_t o = block_excl_scan<uint32_t>(v, sh.s32, &tt);
        if (t < ntiles) tile_carry[(int64_t)t * (C + 1) + c] = run + o;
        run += tt;
      }
      if (tid == 0) tile_carry[(int64_t)ntiles * (C + 1) + c] = run;  // class total = Pc(L)
    }
    if (tid == 0) {
      sh.total = tot_all;
      int64_t nm;
      if (p.n_max > 0) {
        nm = p.n_max;
      } else if (tot_all == 0) {
        nm = 1;  // idle system reports 1 (batch_controller.py:100-102)
      } else {
        const double mean = __ddiv_rn((double)sl_all, (double)tot_all);
        if (mean == 0.0) {
          latch_flags(sum, BS_FLAG_ZERO_MEAN);
          nm = 1;
        } else {
          const int64_t tb = p.current_safe / p.kv_bytes_per_token;  // token_budget()
          const double q = py_floordiv((double)tb, mean);
          nm = (int64_t)q;
          if (nm < 1) nm = 1;
        }
      }
      sh.n_max = nm;
      sum->total_global = tot_all;
      sum->sum_len_global = (int64_t)sl_all;
      sum->n_max = nm;
    }
  }
  for (int i = tid; i < 4 * 256; i += kBT) bins_cnt[i] = 0;  // K2c accumulates here
  __syncthreads();
  const uint32_t total = sh.total;
  // P(x) = #{requests with length < x} from the tile-local prefix + tile carry
  auto Pf = [&](int32_t x) -> uint32_t { return x >= L ? total : P[x] + carry[x / kTileX]; };

  // ---- B. initial edges -------------------------------------------------------------
  for (int w = tid; w < W; w += kBT) bm[w] = 0;
  if (tid == 0) sh.bad = 0;
  __syncthreads();
  if (init_edges) {
    for (int i = tid; i <= k_init; i += kBT) {
      const int32_t e = init_edges[i];
      bool ok = e >= 0 && e <= L;
      if (i == 0) ok = ok && e == 0;
      if (i == k_init) ok = ok && e == L;
      if (i > 0) ok = ok && init_edges[i - 1] < e;
      if (!ok) sh.bad = 1;
      else atomicOr(&bm[e >> 5], 1u << (e & 31));
    }
    __syncthreads();
    if (sh.bad || k_init < 1) {
      if (tid == 0) latch_flags(sum, BS_FLAG_BAD_EDGES);
      for (int w = tid; w < W; w += kBT) bm[w] = 0;
      __syncthreads();
      if (tid == 0) { atomicOr(&bm[0], 1u); atomicOr(&bm[L >> 5], 1u << (L & 31)); }
    }
  } else if (tid == 0) {
    atomicOr(&bm[0], 1u);  // BucketSet default: one bucket [0, L) (bucket_manager.py:87)
    atomicOr(&bm[L >> 5], 1u << (L & 31));
  }
  __syncthreads();

  // ---- C. adjust_buckets passes ------------------------------------------------------
  const int64_t n_max = sh.n_max;
  int64_t nch = 0;
  int32_t passes = 0;
  if (p.adjust) {
    for (;;) {
      const int32_t K = compact_edges(bm, W, E, sh);
      ++passes;
      if ((int64_t)total < n_max) {  // merge branch (bucket_manager.py:148-156)
        if (K != 1) {
          for (int w = tid; w < W; w += kBT) bm[w] = 0;
          __syncthreads();
          if (tid == 0) {
            atomicOr(&bm[0], 1u);
            atomicOr(&bm[L >> 5], 1u << (L & 31));
            if (nch < changes_cap) {
              int32_t* r = changes_out + 4 * nch;
              r[0] = BS_CHANGE_MERGE; r[1] = 0; r[2] = L; r[3] = -1;
            }
          }
          ++nch;
          __syncthreads();
        }
        break;
      }
      if ((int64_t)total == n_max) break;  // bucket_manager.py:158-160
      int any = 0;
      for (int base = 0; base < K; base += kBT) {
        const int k = base + tid;
        int kind = 0, lo = 0, up = 0, mid = 0;
        if (k < K) {
          lo = E[k]; up = E[k + 1]; mid = (lo + up) >> 1;
          const uint32_t plo = Pf(lo);
          const uint32_t c = Pf(up) - plo, s = Pf(mid) - plo;
          if ((int64_t)c > n_max && (double)s > __dmul_rn(p.split_threshold, (double)c))
            kind = (mid <= lo) ? BS_CHANGE_SKIP : BS_CHANGE_SPLIT;
        }
        int32_t tot;
        const int32_t off = block_excl_scan<int32_t>(kind != 0, sh.si, &tot);
        if (kind) {
          const int64_t idx = nch + off;
          if (idx < changes_cap) {
            int32_t* r = changes_out + 4 * idx;
            r[0] = kind; r[1] = lo; r[2] = up; r[3] = mid;
          }
          if (kind == BS_CHANGE_SPLIT) {
            atomicOr(&bm[mid >> 5], 1u << (mid & 31));
            any = 1;
          }
        }
        nch += tot;
      }
      any = __syncthreads_or(any);
      if (!any) break;
      if (p.max_passes > 0 && passes >= p.max_passes) break;
    }
  }
  const int32_t K = compact_edges(bm, W, E, sh);
  for (int i = tid; i <= K; i += kBT) {
    edges_out[i] = E[i];
    if (E != gE) gE[i] = E[i];
  }

  // ---- D. bitmask + per-word popc prefix for the LUT (K2c) ------------------------------
  {
    const int wc = (W + kBT - 1) / kBT;
    const int w0 = tid * wc, w1 = min(W, w0 + wc);
    int32_t cnt = 0;
    for (int w = w0; w < w1; ++w) cnt += __popc(bm[w]);
    int32_t tot;
    int32_t off = block_excl_scan<int32_t>(cnt, sh.si, &tot);
    for (int w = w0; w < w1; ++w) {
      gwp[w] = off;
      gbm[w] = bm[w];
      off += __popc(bm[w]);
    }
  }

  // ---- E. segment offsets (local per-class counts) and radix slot bases ---------------
  const int32_t S = K * C;
  int32_t run_cnt = 0, run_w = 0;
  for (int base = 0; base < S; base += kBT) {
    const int s = base + tid;
    int32_t cnt = 0, width = 0;
    if (s < S) {
      const int b = s / C, c = s % C;
      const int32_t lo = E[b], up = E[b + 1];
      const uint32_t* Pc = PcL + (int64_t)c * (L + 1);
      auto Pcf = [&](int32_t x) -> uint32_t {
        const int64_t t = x >= L ? ntiles : x / kTileX;
        return (x >= L ? 0u : Pc[x]) + tile_carry[t * (C + 1) + c];
      };
      cnt = (int32_t)(Pcf(up) - Pcf(lo));
      width = policy_of(p, c) == BS_POLICY_FCFS ? 1 : (up - lo);
    }
    int32_t tcn, tw;
    const int32_t oc = block_excl_scan<int32_t>(cnt, sh.si, &tcn);
    const int32_t ow = block_excl_scan<int32_t>(width, sh.si, &tw);
    if (s < S) {
      seg_off_out[s] = run_cnt + oc;
      seg_base[s] = run_w + ow;
    }
    run_cnt += tcn;
    run_w += tw;
  }
  if (tid == 0) {
    seg_off_out[S] = run_cnt;
    kinfo[0] = K;
    kinfo[1] = run_w;  // number of radix slots D
    kinfo[2] = S;
    sum->k_buckets = K;
    sum->n_changes = nch;
    sum->n_passes = passes;
    if (nch > changes_cap) latch_flags(sum, BS_FLAG_CHANGES_TRUNC);
  }
}

// ---------------------------------------------------------------------------- K2c
__global__ void __launch_bounds__(256)
    k_tables(const uint32_t* __restrict__ hist_local, bs_window_params p, int sort_bits,
             int sort_passes, const int32_t* __restrict__ gE, const uint32_t* __restrict__ gbm,
             const uint32_t* __restrict__ gwp, const int32_t* __restrict__ seg_base,
             int32_t* __restrict__ lut, uint32_t* __restrict__ slot_lut,
             uint32_t* __restrict__ bins_cnt, int32_t* __restrict__ slot_seg,
             int32_t* __restrict__ slot_len) {
  pdl_prologue();
  __shared__ uint32_t sbins[4 * 256];
  const int32_t L = p.l_max, C = p.n_classes;
  for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) sbins[i] = 0;
  __syncthreads();
  const uint32_t dmask = (1u << sort_bits) - 1u;
  const int64_t total = (int64_t)C * L;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(idx / L), x = (int)(idx % L);
    const int w = x >> 5, bt = x & 31;
    const uint32_t lowmask = bt == 31 ? 0xffffffffu : ((2u << bt) - 1u);
    const int b = (int)(gwp[w] + __popc(gbm[w] & lowmask)) - 1;  // #{j >= 1 : e_j <= x}
    if (c == 0) lut[x] = b;
    const int pol = policy_of(p, c);
    uint32_t slot = (uint32_t)seg_base[b * C + c];
    if (pol == BS_POLICY_SJF) slot += (uint32_t)(x - gE[b]);
    else if (pol == BS_POLICY_LJF) slot += (uint32_t)(gE[b + 1] - 1 - x);
    slot_lut[idx] = slot;
    slot_seg[slot] = b * C + c;
    // length of a slot (K5a reads it instead of gathering len[perm[j]]); an FCFS slot
    // holds every length of its segment: -1 (all writers agree)
    slot_len[slot] = (pol == BS_POLICY_SJF || pol == BS_POLICY_LJF) ? x : -1;
    const uint32_t h = hist_local[idx];
    if (h)  // consecutive lengths hit distinct low digits: plain shared atomics
      for (int q = 0; q < sort_passes; ++q)
        atomicAdd(&sbins[q * 256 + ((slot >> (q * sort_bits)) & dmask)], h);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < sort_passes * 256; i += blockDim.x)
    if (sbins[i]) atomicAdd(&bins_cnt[i], sbins[i]);
}

// ---------------------------------------------------------------------------- small L
// Single-CTA fused K2 for l_max <= kSmallL: prefix sums live in shared memory and the
// window fixpoint from the root (no init edges, passes until no split) is computed
// on the implicit midpoint tree level by level: a node of depth d is a bucket of
// pass d+1 iff its parent split, so every pass costs one level of work and the
// change log is one scan over the split flags in heap (= pass-major, left-to-right)
// order — exactly the reference's emission order.  Other modes run the general
// pass loop.  The per-length LUT, radix slots and digit counts are then built grid-wide
// by k_tables from the published edge bitmask.
constexpr int kSmallL = 16384;
constexpr int kMaxDepth = 15;  // ceil(log2(kSmallL)) + 1

__device__ __forceinline__ void node_bounds(int32_t L, int d, int32_t k, int32_t& lo,
                                            int32_t& up) {
  lo = 0;
  up = L;
  for (int bit = d - 1; bit >= 0; --bit) {
    const int32_t mid = (lo + up) >> 1;
    if ((k >> bit) & 1) lo = mid; else up = mid;
  }
}

__global__ void __launch_bounds__(kSmallBT, kSmallBTMin)
    k_bounds_small(const uint32_t* __restrict__ hist_local,
                   const uint32_t* __restrict__ hist_global, bs_window_params p, int sort_bits,
                   int sort_passes, const int32_t* __restrict__ init_edges, int32_t k_init,
                   int32_t* __restrict__ edges_out, int32_t* __restrict__ changes_out,
                   int32_t changes_cap, int32_t* __restrict__ seg_off_out,
                   uint32_t* __restrict__ PcL, int32_t* __restrict__ gE,
                   int32_t* __restrict__ seg_base, int32_t* __restrict__ lut,
                   uint32_t* __restrict__ slot_lut, uint32_t* __restrict__ bins_cnt,
                   int32_t* __restrict__ kinfo, bs_summary* sum, int32_t* __restrict__ slot_seg,
                   uint32_t* __restrict__ gbm, uint32_t* __restrict__ gwp) {
  pdl_prologue();
  extern __shared__ uint32_t dyn[];
  __shared__ BoundsShared sh;
  __shared__ int32_t s_flag;
  const int32_t L = p.l_max, C = p.n_classes;
  const int W = (L + 1 + 31) / 32;
  const int tid = threadIdx.x;
  const int nt = (int)blockDim.x;
  const int NW = ((1 << kMaxDepth) + 31) / 32;     // node-bitmask words
  uint32_t* Ps = dyn;                               // [L+1]
  uint32_t* bm = Ps + (L + 1);                      // [W]
  uint32_t* split_bits = bm + W;                    // [NW] node split flags (heap order)
  int32_t* E = reinterpret_cast<int32_t*>(split_bits + NW);  // [L+1]
  const int chunk = (L + nt - 1) / nt;
  const int x0 = min(L, tid * chunk), x1 = min(L, x0 + chunk);

  // ---- A. prefix sums (global total in smem, local per class in global) ------------
  {
    uint32_t s = 0;
    uint64_t sl = 0;
    for (int x = x0; x < x1; ++x) {
      uint32_t h = 0;
      for (int c = 0; c < C; ++c) h += hist_global[(int64_t)c * L + x];
      Ps[x] = h;
      s += h;
      sl += (uint64_t)h * (uint64_t)x;
    }
    uint32_t tot;
    uint32_t run = block_excl_scan<uint32_t>(s, sh.s32, &tot);
    for (int x = x0; x < x1; ++x) {
      const uint32_t h = Ps[x];
      Ps[x] = run;
      run += h;
    }
    uint64_t sltot;
    block_excl_scan<uint64_t>(sl, sh.s64, &sltot);
    for (int c = 0; c < C; ++c) {
      uint32_t sc = 0;
      for (int x = x0; x < x1; ++x) sc += hist_local[(int64_t)c * L + x];
      uint32_t tc;
      uint32_t rc = block_excl_scan<uint32_t>(sc, sh.s32, &tc);
      uint32_t* Pc = PcL + (int64_t)c * (L + 1);
      for (int x = x0; x < x1; ++x) {
        Pc[x] = rc;
        rc += hist_local[(int64_t)c * L + x];
      }
      if (tid == 0) Pc[L] = tc;
    }
    if (tid == 0) {
      Ps[L] = tot;
      sh.total = tot;
      int64_t nm;
      if (p.n_max > 0) {
        nm = p.n_max;
      } else if (tot == 0) {
        nm = 1;
      } else {
        const double mean = __ddiv_rn((double)sltot, (double)tot);
        if (mean == 0.0) {
          latch_flags(sum, BS_FLAG_ZERO_MEAN);
          nm = 1;
        } else {
          const int64_t tb = p.current_safe / p.kv_bytes_per_token;
          nm = (int64_t)py_floordiv((double)tb, mean);
          if (nm < 1) nm = 1;
        }
      }
      sh.n_max = nm;
      sum->total_global = tot;
      sum->sum_len_global = (int64_t)sltot;
      sum->n_max = nm;
    }
  }
  for (int w = tid; w < W; w += nt) bm[w] = 0;
  for (int w = tid; w < NW; w += nt) split_bits[w] = 0;
  if (tid == 0) { sh.bad = 0; s_flag = 0; }
  __syncthreads();
  const int64_t n_max = sh.n_max;
  const uint32_t total = sh.total;
  int64_t nch = 0;
  int32_t passes = 0;
  const bool fast = init_edges == nullptr && p.adjust && p.max_passes <= 0;

  if (fast) {
    // ---- C'. window fixpoint on the midpoint tree, one level per pass ---------------
    if (tid == 0) { atomicOr(&bm[0], 1u); atomicOr(&bm[L >> 5], 1u << (L & 31)); }
    int deepest = -1;
    for (int d = 0; d < kMaxDepth; ++d) {
      const int32_t nodes = 1 << d;
      int any = 0;
      for (int32_t k = tid; k < nodes; k += nt) {
        const int32_t id = nodes - 1 + k;
        bool realized = d == 0;
        if (d > 0) {
          const int32_t par = (id - 1) >> 1;
          realized = (split_bits[par >> 5] >> (par & 31)) & 1u;
        }
        if (!realized) continue;
        int32_t lo, up;
        node_bounds(L, d, k, lo, up);
        const int32_t mid = (lo + up) >> 1;
        const uint32_t c = Ps[up] - Ps[lo], s = Ps[mid] - Ps[lo];
        if ((int64_t)c > n_max && (double)s > __dmul_rn(p.split_threshold, (double)c)) {
          if (mid <= lo) {
            s_flag = 1;  // a skip: leave it to the general loop (never happens on counts)
          } else {
            atomicOr(&split_bits[id >> 5], 1u << (id & 31));
            atomicOr(&bm[mid >> 5], 1u << (mid & 31));
            any = 1;
          }
        }
      }
      any = __syncthreads_or(any);
      if (!any) break;
      deepest = d;
    }
    passes = deepest + 2;
    __syncthreads();
    if (s_flag) {  // fall back: reset and run the general loop below
      for (int w = tid; w < W; w += nt) bm[w] = 0;
      __syncthreads();
    } else {
      // change log: split nodes in heap order == pass-major, left to right
      const int32_t nnodes = deepest >= 0 ? (2 << deepest) - 1 : 0;
      const int per = (nnodes + nt - 1) / nt;
      const int32_t n0 = tid * per, n1 = min(nnodes, n0 + per);
      int32_t cnt = 0;
      for (int32_t id = n0; id < n1; ++id) cnt += (split_bits[id >> 5] >> (id & 31)) & 1u;
      int32_t tot;
      int32_t off = block_excl_scan<int32_t>(cnt, sh.si, &tot);
      for (int32_t id = n0; id < n1; ++id) {
        if ((split_bits[id >> 5] >> (id & 31)) & 1u) {
          if (off < changes_cap) {
            const int d = 31 - __clz(id + 1);
            int32_t lo, up;
            node_bounds(L, d, id + 1 - (1 << d), lo, up);
            int32_t* r = changes_out + 4 * off;
            r[0] = BS_CHANGE_SPLIT; r[1] = lo; r[2] = up; r[3] = (lo + up) >> 1;
          }
          ++off;
        }
      }
      nch = tot;
    }
  }
  if (!fast || s_flag) {
    // ---- B/C. general adjust_buckets passes (init edges / max_passes / skips) -----------
    nch = 0;
    passes = 0;
    if (init_edges) {
      for (int i = tid; i <= k_init; i += nt) {
        const int32_t e = init_edges[i];
        bool ok = e >= 0 && e <= L;
        if (i == 0) ok = ok && e == 0;
        if (i == k_init) ok = ok && e == L;
        if (i > 0) ok = ok && init_edges[i - 1] < e;
        if (!ok) sh.bad = 1;
        else atomicOr(&bm[e >> 5], 1u << (e & 31));
      }
      __syncthreads();
      if (sh.bad || k_init < 1) {
        if (tid == 0) latch_flags(sum, BS_FLAG_BAD_EDGES);
        for (int w = tid; w < W; w += nt) bm[w] = 0;
        __syncthreads();
        if (tid == 0) { atomicOr(&bm[0], 1u); atomicOr(&bm[L >> 5], 1u << (L & 31)); }
      }
    } else if (tid == 0) {
      atomicOr(&bm[0], 1u);
      atomicOr(&bm[L >> 5], 1u << (L & 31));
    }
    __syncthreads();
    if (p.adjust) {
      for (;;) {
        const int32_t K = compact_edges(bm, W, E, sh);
        ++passes;
        if ((int64_t)total < n_max) {
          if (K != 1) {
            for (int w = tid; w < W; w += nt) bm[w] = 0;
            __syncthreads();
            if (tid == 0) {
              atomicOr(&bm[0], 1u);
              atomicOr(&bm[L >> 5], 1u << (L & 31));
              if (nch < changes_cap) {
                int32_t* r = changes_out + 4 * nch;
                r[0] = BS_CHANGE_MERGE; r[1] = 0; r[2] = L; r[3] = -1;
              }
            }
            ++nch;
            __syncthreads();
          }
          break;
        }
        if ((int64_t)total == n_max) break;
        int any = 0;
        for (int base = 0; base < K; base += nt) {
          const int k = base + tid;
          int kind = 0, lo = 0, up = 0, mid = 0;
          if (k < K) {
            lo = E[k]; up = E[k + 1]; mid = (lo + up) >> 1;
            const uint32_t c = Ps[up] - Ps[lo], s = Ps[mid] - Ps[lo];
            if ((int64_t)c > n_max && (double)s > __dmul_rn(p.split_threshold, (double)c))
              kind = (mid <= lo) ? BS_CHANGE_SKIP : BS_CHANGE_SPLIT;
          }
          int32_t tot;
          const int32_t off = block_excl_scan<int32_t>(kind != 0, sh.si, &tot);
          if (kind) {
            const int64_t idx = nch + off;
            if (idx < changes_cap) {
              int32_t* r = changes_out + 4 * idx;
              r[0] = kind; r[1] = lo; r[2] = up; r[3] = mid;
            }
            if (kind == BS_CHANGE_SPLIT) {
              atomicOr(&bm[mid >> 5], 1u << (mid & 31));
              any = 1;
            }
          }
          nch += tot;
        }
        any = __syncthreads_or(any);
        if (!any) break;
        if (p.max_passes > 0 && passes >= p.max_passes) break;
      }
    }
  }
  __syncthreads();
  const int32_t K = compact_edges(bm, W, E, sh);
  for (int i = tid; i <= K; i += nt) { edges_out[i] = E[i]; gE[i] = E[i]; }

  // ---- edge bitmask + popc prefix for the parallel tables kernel (k_tables) -------------
  {
    const int wc = (W + nt - 1) / nt;
    const int w0 = min(W, tid * wc), w1 = min(W, w0 + wc);
    uint32_t cnt = 0;
    for (int w = w0; w < w1; ++w) cnt += __popc(bm[w]);
    uint32_t tw;
    uint32_t o = block_excl_scan<uint32_t>(cnt, sh.s32, &tw);
    for (int w = w0; w < w1; ++w) {
      gbm[w] = bm[w];
      gwp[w] = o;
      o += __popc(bm[w]);
    }
  }
  // ---- E. segment offsets (local per-class counts) and radix slot bases -------------
  const int32_t S = K * C;
  __syncthreads();
  int32_t run_cnt = 0, run_w = 0;
  for (int base = 0; base < S; base += nt) {
    const int s = base + tid;
    int32_t cnt = 0, width = 0;
    if (s < S) {
      const int b = s / C, c = s % C;
      const int32_t lo = E[b], up = E[b + 1];
      const uint32_t* Pc = PcL + (int64_t)c * (L + 1);
      cnt = (int32_t)(Pc[up] - Pc[lo]);
      width = policy_of(p, c) == BS_POLICY_FCFS ? 1 : (up - lo);
    }
    int32_t tcn, tw;
    const int32_t oc = block_excl_scan<int32_t>(cnt, sh.si, &tcn);
    const int32_t ow = block_excl_scan<int32_t>(width, sh.si, &tw);
    if (s < S) {
      seg_off_out[s] = run_cnt + oc;
      seg_base[s] = run_w + ow;
    }
    run_cnt += tcn;
    run_w += tw;
  }
  if (tid == 0) seg_off_out[S] = run_cnt;
  __syncthreads();
  // lookup tables and digit counts: k_tables (grid-wide) reads gbm / gwp / gE / seg_base
  for (int i = tid; i < 4 * 256; i += nt) bins_cnt[i] = 0;
  if (tid == 0) {
    kinfo[0] = K;
    kinfo[1] = run_w;
    kinfo[2] = S;
    sum->k_buckets = K;
    sum->n_changes = nch;
    sum->n_passes = passes;
    if (nch > changes_cap) latch_flags(sum, BS_FLAG_CHANGES_TRUNC);
  }
}

SortPlan sort_plan(int32_t l_max, int32_t n_classes) {
  // slots D <= n_classes * l_max; digits of <= 8 bits, split evenly over passes
  uint64_t dmax = (uint64_t)n_classes * (uint64_t)l_max;
  int bits = 1;
  while ((1ull << bits) < dmax) ++bits;
  int passes = (bits + 7) / 8;
  int per = (bits + passes - 1) / passes;
  return SortPlan{passes, per};
}

// dynamic shared memory of the K2 kernels for a window of l_max L
static size_t bounds_small_smem(int32_t L) {
  const int W = (L + 1 + 31) / 32;
  const int NW = ((1 << kMaxDepth) + 31) / 32;
  return sizeof(uint32_t) * ((size_t)(L + 1) + W + NW + (L + 1));
}
static size_t bounds_big_smem(int32_t L) {
  const int ntiles = (L + kTileX - 1) / kTileX;
  const int W = (L + 1 + 31) / 32;
  return sizeof(uint32_t) * ((size_t)W + ntiles + (L + 1 <= kEcap ? kEcap : 0));
}

// per-context setup on the context's device (bs_create): opt the K2 kernels into the
// shared memory the largest window of this context (l_max <= l_cap) needs
cudaError_t bounds_prepare(bs_ctx* ctx) {
  const int32_t Ls = std::min<int32_t>(ctx->l_cap, kSmallL);
  size_t sm = bounds_small_smem(Ls);
  cudaError_t e = cudaSuccess;
  if (sm > 48 * 1024)
    e = cudaFuncSetAttribute(k_bounds_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess || ctx->l_cap <= kSmallL) return e;
  sm = bounds_big_smem(ctx->l_cap);
  if (sm > 48 * 1024)
    e = cudaFuncSetAttribute(k_boundaries, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  return e;
}

cudaError_t launch_boundaries(bs_ctx* ctx, const uint32_t* hist_local, const uint32_t* hist_global,
                              const bs_window_params& p, const int32_t* init_edges, int32_t k_init,
                              int32_t* edges_out, int32_t* changes_out, int32_t changes_cap,
                              int32_t* seg_off_out, bs_summary* summary, cudaStream_t st) {
  const SortPlan sp = sort_plan(p.l_max, p.n_classes);
  const int32_t L = p.l_max, C = p.n_classes;
  if (L <= kSmallL) {
    const size_t smem = bounds_small_smem(L);
    launch_k(ctx, k_bounds_small, dim3(1), dim3(kSmallBT), smem, st, false, hist_local, hist_global ? hist_global : hist_local, p,
                                         sp.bits, sp.passes, init_edges, k_init, edges_out,
                                         changes_out, changes_cap, seg_off_out, ctx->PcL, ctx->E,
                                         ctx->seg_base, ctx->lut, ctx->slot_lut, ctx->bins_cnt,
                                         ctx->kinfo, summary, ctx->slot_seg, ctx->bmw, ctx->wp);
    cudaError_t e0 = cudaGetLastError();
    if (e0 != cudaSuccess) return e0;
    const int64_t cells = (int64_t)C * L;
    const unsigned tb = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>((cells + 255) / 256, 4LL * ctx->num_sms));
    launch_k(ctx, k_tables, dim3(tb), dim3(256), 0, st, false, hist_local, p, sp.bits, sp.passes, ctx->E, ctx->bmw, ctx->wp,
                                 ctx->seg_base, ctx->lut, ctx->slot_lut, ctx->bins_cnt,
                                 ctx->slot_seg, ctx->slot_len);
    ctx->launches += 2;
    return cudaGetLastError();
  }
  const int ntiles = (L + kTileX - 1) / kTileX;
  const uint32_t* hg = hist_global ? hist_global : hist_local;
  launch_k(ctx, k_prefix_tiles, dim3(ntiles), dim3(1024), 0, st, false, hist_local, hg, L, C, ctx->P, ctx->PcL, ctx->tile_tot,
                                          reinterpret_cast<unsigned long long*>(ctx->tile_slen));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const size_t smem = bounds_big_smem(L);
  launch_k(ctx, k_boundaries, dim3(1), dim3(kBT), smem, st, false, ctx->P, ctx->PcL, ctx->tile_tot,
                                     reinterpret_cast<const unsigned long long*>(ctx->tile_slen),
                                     ntiles, p, init_edges, k_init, edges_out, changes_out,
                                     changes_cap, seg_off_out, ctx->E, ctx->bmw, ctx->wp,
                                     ctx->seg_base, ctx->tile_carry, ctx->bins_cnt, ctx->kinfo,
                                     summary);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int64_t cells = (int64_t)C * L;
  const unsigned tb = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>((cells + 1023) / 1024, 4LL * ctx->num_sms));
  launch_k(ctx, k_tables, dim3(tb), dim3(256), 0, st, false, hist_local, p, sp.bits, sp.passes, ctx->E, ctx->bmw, ctx->wp,
                               ctx->seg_base, ctx->lut, ctx->slot_lut, ctx->bins_cnt,
                               ctx->slot_seg, ctx->slot_len);
  ctx->launches += 3;
  return cudaGetLastError();
}

}  // namespace bsk
