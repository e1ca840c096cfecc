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
// B200 mapping: a single 1024-thread CTA (the whole problem is O(L + K) and sits
// in L2/shared memory).  Edges live as a bitmask over [0, L] in shared memory; a
// pass is a block-scan compaction of the bitmask + one thread per bucket; the
// change log is written in bucket order via a block scan, matching the
// reference's left-to-right emission.  The same CTA then builds the per-length
// bucket LUT (K3), the per-(class,length) radix slot table and the per-pass
// digit offsets for K4 — derived from the histogram, so K4 needs no upsweep.
#include "ctx.cuh"

namespace bsk {

constexpr int kBT = 1024;

// CPython _float_div_mod floor quotient (Objects/floatobject.c)
__device__ double py_floordiv(double vx, double wx) {
  double mod = fmod(vx, wx);
  double div = __ddiv_rn(__dsub_rn(vx, mod), wx);
  if (mod != 0.0) {
    if ((wx < 0) != (mod < 0)) { mod = __dadd_rn(mod, wx); div = __dsub_rn(div, 1.0); }
  }
  double fd;
  if (div != 0.0) {
    fd = floor(div);
    if (__dsub_rn(div, fd) > 0.5) fd = __dadd_rn(fd, 1.0);
  } else {
    fd = copysign(0.0, __ddiv_rn(vx, wx));
  }
  return fd;
}

struct BoundsShared {
  uint64_t s64[33];
  uint32_t s32[33];
  int32_t si[33];
  int64_t n_max;
  uint32_t total;
  int32_t K;
  int32_t bad;
};

// compact the edge bitmask into E[0..K]; returns K (number of buckets)
__device__ int32_t compact_edges(const uint32_t* bm, int W, int32_t* E, BoundsShared& sh) {
  const int wc = (W + kBT - 1) / kBT;
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
    k_boundaries(const uint32_t* __restrict__ hist_local, const uint32_t* __restrict__ hist_global,
                 bs_window_params p, int sort_bits, int sort_passes,
                 const int32_t* __restrict__ init_edges, int32_t k_init,
                 int32_t* __restrict__ edges_out, int32_t* __restrict__ changes_out,
                 int32_t changes_cap, int32_t* __restrict__ seg_off_out, uint32_t* __restrict__ P,
                 uint32_t* __restrict__ PcL, int32_t* __restrict__ E, int32_t* __restrict__ lut,
                 int32_t* __restrict__ seg_base, uint32_t* __restrict__ slot_lut,
                 uint32_t* __restrict__ bin_base, int32_t* __restrict__ kinfo, bs_summary* sum) {
  extern __shared__ uint32_t dyn[];
  __shared__ BoundsShared sh;
  const int32_t L = p.l_max, C = p.n_classes;
  const int W = (L + 1 + 31) / 32;
  uint32_t* bm = dyn;                 // [W] edge bitmask over [0, L]
  uint32_t* wp = dyn + W;             // [W] exclusive popc prefix per word
  uint32_t* sbins = dyn + 2 * W;      // [4][256] radix digit counts
  const int tid = threadIdx.x;
  const int chunk = (L + kBT - 1) / kBT;
  const int x0 = min(L, tid * chunk), x1 = min(L, x0 + chunk);

  // ---- A. prefix sums: global total P, local per-class PcL, sum(len) ----------
  {
    uint32_t s = 0;
    uint64_t sl = 0;
    for (int x = x0; x < x1; ++x) {
      uint32_t h = 0;
      for (int c = 0; c < C; ++c) h += hist_global[(int64_t)c * L + x];
      s += h;
      sl += (uint64_t)h * (uint64_t)x;
    }
    uint32_t tot;
    uint32_t run = block_excl_scan<uint32_t>(s, sh.s32, &tot);
    for (int x = x0; x < x1; ++x) {
      P[x] = run;
      uint32_t h = 0;
      for (int c = 0; c < C; ++c) h += hist_global[(int64_t)c * L + x];
      run += h;
    }
    uint64_t sltot;
    block_excl_scan<uint64_t>(sl, sh.s64, &sltot);
    if (tid == 0) {
      P[L] = tot;
      sh.total = tot;
      int64_t nm;
      if (p.n_max > 0) {
        nm = p.n_max;
      } else if (tot == 0) {
        nm = 1;  // idle system reports 1 (batch_controller.py:100-102)
      } else {
        const double mean = __ddiv_rn((double)sltot, (double)tot);
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
      sum->total_global = tot;
      sum->sum_len_global = (int64_t)sltot;
      sum->n_max = nm;
    }
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
  }

  // ---- B. initial edges -------------------------------------------------------
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

  // ---- C. adjust_buckets passes --------------------------------------------------
  const int64_t n_max = sh.n_max;
  const uint32_t total = sh.total;
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
          const uint32_t c = P[up] - P[lo], s = P[mid] - P[lo];
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
  for (int i = tid; i <= K; i += kBT) edges_out[i] = E[i];

  // ---- D. per-length bucket LUT (K3): bucket(x) = #{j >= 1 : e_j <= x} ------------
  {
    const int wc = (W + kBT - 1) / kBT;
    const int w0 = tid * wc, w1 = min(W, w0 + wc);
    int32_t cnt = 0;
    for (int w = w0; w < w1; ++w) cnt += __popc(bm[w]);
    int32_t tot;
    int32_t off = block_excl_scan<int32_t>(cnt, sh.si, &tot);
    for (int w = w0; w < w1; ++w) {
      wp[w] = off;
      off += __popc(bm[w]);
    }
    __syncthreads();
    for (int x = tid; x < L; x += kBT) {
      const int w = x >> 5, b = x & 31;
      const uint32_t lowmask = b == 31 ? 0xffffffffu : ((2u << b) - 1u);
      lut[x] = (int32_t)(wp[w] + __popc(bm[w] & lowmask)) - 1;
    }
  }

  // ---- E. segments, radix slots, digit offsets (K4) --------------------------------
  const int32_t S = K * C;
  int32_t run_cnt = 0, run_w = 0;
  for (int base = 0; base < S; base += kBT) {
    const int s = base + tid;
    int32_t cnt = 0, width = 0;
    if (s < S) {
      const int b = s / C, c = s % C;
      const int32_t lo = E[b], up = E[b + 1];
      const uint32_t* Pc = PcL + (int64_t)c * (L + 1);
      cnt = (int32_t)(Pc[up] - Pc[lo]);
      width = p.policy[c] == BS_POLICY_FCFS ? 1 : (up - lo);
    }
    int32_t tc, tw;
    const int32_t oc = block_excl_scan<int32_t>(cnt, sh.si, &tc);
    const int32_t ow = block_excl_scan<int32_t>(width, sh.si, &tw);
    if (s < S) {
      seg_off_out[s] = run_cnt + oc;
      seg_base[s] = run_w + ow;
    }
    run_cnt += tc;
    run_w += tw;
  }
  if (tid == 0) seg_off_out[S] = run_cnt;
  for (int i = tid; i < 4 * 256; i += kBT) sbins[i] = 0;
  __syncthreads();
  const uint32_t dmask = (1u << sort_bits) - 1u;
  for (int64_t idx = tid; idx < (int64_t)C * L; idx += kBT) {
    const int c = (int)(idx / L), x = (int)(idx % L);
    const int b = lut[x];
    const int pol = p.policy[c];
    uint32_t slot = (uint32_t)seg_base[b * C + c];
    if (pol == BS_POLICY_SJF) slot += (uint32_t)(x - E[b]);
    else if (pol == BS_POLICY_LJF) slot += (uint32_t)(E[b + 1] - 1 - x);
    slot_lut[idx] = slot;
    const uint32_t h = hist_local[idx];
    if (h)
      for (int q = 0; q < sort_passes; ++q)
        atomicAdd(&sbins[q * 256 + ((slot >> (q * sort_bits)) & dmask)], h);
  }
  __syncthreads();
  for (int q = 0; q < sort_passes; ++q) {
    const uint32_t v = tid < 256 ? sbins[q * 256 + tid] : 0u;
    uint32_t t;
    const uint32_t o = block_excl_scan<uint32_t>(v, sh.s32, &t);
    if (tid < 256) bin_base[q * 256 + tid] = o;
  }
  if (tid == 0) {
    kinfo[0] = K;
    kinfo[1] = run_w;  // number of radix slots D
    kinfo[2] = S;
    sum->k_buckets = K;
    sum->n_changes = nch;
    sum->n_passes = passes;
    sum->sort_passes = sort_passes;
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

cudaError_t launch_boundaries(bs_ctx* ctx, const uint32_t* hist_local, const uint32_t* hist_global,
                              const bs_window_params& p, const int32_t* init_edges, int32_t k_init,
                              int32_t* edges_out, int32_t* changes_out, int32_t changes_cap,
                              int32_t* seg_off_out, bs_summary* summary, cudaStream_t st) {
  const SortPlan sp = sort_plan(p.l_max, p.n_classes);
  const int W = (p.l_max + 1 + 31) / 32;
  const size_t smem = sizeof(uint32_t) * (2 * (size_t)W + 4 * 256);
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaFuncSetAttribute(k_boundaries, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  k_boundaries<<<1, kBT, smem, st>>>(hist_local, hist_global ? hist_global : hist_local, p, sp.bits,
                                     sp.passes, init_edges, k_init, edges_out, changes_out,
                                     changes_cap, seg_off_out, ctx->P, ctx->PcL, ctx->E, ctx->lut,
                                     ctx->seg_base, ctx->slot_lut, ctx->bin_base, ctx->kinfo,
                                     summary);
  ++ctx->launches;
  return cudaGetLastError();
}

}  // namespace bsk
