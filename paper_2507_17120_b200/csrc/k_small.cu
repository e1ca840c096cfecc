// K0 — the whole schedule of a small window (K1..K5) in one CTA.
//
// A window of up to kSmallN requests (C1's 1,000-request windows, the drop-in's
// per-bucket form_batch drains, the parity fixtures) is latency-bound: the multi-kernel
// path spends ~13 dependent launches (each a handful of global round trips over a few
// KB) on it.  Here one 512-thread CTA keeps the window in shared memory and runs the
// reference composition with the semantics of the oracle (oracle/bso.c)
// and of the multi-kernel path:
//   K1  per-(class, length) histogram             bucket_manager.py:31-32,126-127
//   K2  adjust_buckets passes on prefix sums, the change log in emission order, and
//       current_n_max with CPython's float floor division
//                                                 bucket_manager.py:133-191; batch_controller.py:93-104
//   K3  bucket id per request                     bucket_manager.py:110-131
//   K4  drain order as a stable counting sort: every request's group — (class, length)
//       for SJF / LJF classes, (class, bucket) for FCFS — has its sorted offset in the
//       per-class length prefix sums; the drain order is the requests stably sorted by
//       that offset: two LSD radix passes (6-bit digits) on all 16 warps, match_any
//       ranks per warp chunk, one block scan of the (digit, warp) counters
//                                                 batch_controller.py:33-41,154-156
//   K5  form_batch drained per segment: where each call starts and where the drain
//       stops.  When the average call is short (budget / mean length < 32 requests)
//       every position first scans ahead for the end of a call starting there, and one
//       warp per segment run hops call to call; calls past the scan's reach (and every
//       call otherwise) are found by the warp 32 positions per step (lane prefix of
//       count / max / sum — none needed for an ascending / descending run under the
//       padded accounting — first violating lane by ballot).  Then every position
//       learns its batch from the call-start flag scan and its row from prefix sums,
//       the batch statistics come from shared atomics, the offsets from block scans;
//       oversize rejections, the pledged-headroom stop, waste_ratio in float64
//                                                 batch_controller.py:136-191; memory_model.py:92-100
// and leaves the row map / piece prefix K6 reads, so the pack launches right after.
// Dispatch order (K7) and sharded windows take the multi-kernel path.
#include "ctx.cuh"

namespace bsk {

constexpr int kSmallT = 512;
constexpr int kSmallN = 2048;
// phase timestamps into summary.reserved[0..7]: timing 1 = globaltimer ns (its update
// granularity is ~1 us outside a profiler), 2 = the SM cycle counter (one CTA, one SM)
#define BS_SMALL_MARK(k) \
  if (timing && threadIdx.x == 0) \
    sum->reserved[k] = timing == 2 ? (int64_t)clock64() : (int64_t)globaltimer_ns()

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct SmallSh {
  int64_t s64[33];
  int32_t s32[33];
  uint32_t s32m[9 * 33];  // multi-value scans
  int32_t i32m[3 * 33];
  uint32_t total;
  int64_t n_max, sum_len;
  int32_t k, nruns, nb, bad;
  int64_t nch;
  int32_t passes;
  unsigned flags;
  unsigned long long rej, pend, adm_tok, pad_tok, peak;
  double wsum;
};

__device__ __forceinline__ int small_policy(const bs_window_params& p, int c) {
  int pol = p.policy[0];
#pragma unroll
  for (int i = 1; i < BS_MAX_CLASSES; ++i)
    if (c == i) pol = p.policy[i];
  return pol;
}

// exclusive scan of a[0..m) in place (chunked over the block); returns the total
template <typename T>
__device__ T block_scan_array(T* a, int m, T* scratch) {
  const int nt = blockDim.x, tid = threadIdx.x;
  const int chunk = (m + nt - 1) / nt;
  const int lo = min(m, tid * chunk), hi = min(m, lo + chunk);
  T s = 0;
  for (int i = lo; i < hi; ++i) s += a[i];
  T tot;
  T run = block_excl_scan<T>(s, scratch, &tot);
  for (int i = lo; i < hi; ++i) {
    const T v = a[i];
    a[i] = run;
    run += v;
  }
  __syncthreads();
  return tot;
}

// shared-memory layout, shared by the kernel and the host (small_smem_bytes)
struct SmallLayout {
  int64_t xs, seg, goff, perm, runid, aex, cs, region;  // byte offsets
  int64_t hc, P, e, ne;                                 // inside region (K1..K4)
  int64_t total;
};

__host__ __device__ inline int64_t r16(int64_t b) { return (b + 15) & ~15LL; }

// histogram rows keep one pad word per 32 entries: a thread scanning its chunk of
// consecutive lengths (x = tid * chunk + k, chunk a power of two <= 16) then hits 32
// distinct banks across the warp instead of 32 / chunk
__host__ __device__ __forceinline__ int32_t hx(int32_t x) { return x + (x >> 5); }
__host__ __device__ __forceinline__ int32_t hrow(int32_t L) { return hx(L) + 1; }

// K4 ranking counters: [64 digits][17] (16 warps + 1 pad word)
constexpr int kRankDig = 64, kRankPitch = 17;
static_assert(kSmallN <= (kSmallT / 32) * 4 * 32, "K4 ranks at most 4 steps per warp");

__host__ __device__ inline SmallLayout small_layout(int32_t n, int32_t L, int32_t C) {
  SmallLayout s;
  const int64_t n4 = 4 * (int64_t)(n + 4);
  s.xs = 0;
  s.seg = r16(s.xs + n4);
  s.goff = r16(s.seg + n4);
  s.perm = r16(s.goff + n4);
  s.runid = r16(s.perm + n4);
  s.aex = r16(s.runid + n4);
  s.cs = r16(s.aex + n4);
  s.region = r16(s.cs + n + 4);
  // K1..K4: per-class histogram -> prefix [C][L+1], total prefix P[L+1] (padded rows,
  // hx), edges e / ne; K4's ranking counters reuse the start of the region
  s.hc = 0;
  s.P = r16(s.hc + 4 * (int64_t)C * hrow(L));
  s.e = r16(s.P + 4 * (int64_t)hrow(L));
  s.ne = r16(s.e + 4 * (int64_t)(L + 1));
  int64_t phase1 = r16(s.ne + 4 * (int64_t)(L + 1));
  if (phase1 < 4 * kRankDig * kRankPitch) phase1 = 4 * kRankDig * kRankPitch;
  // K5: 10 int32 tables of n + 2 entries and one byte table of n + 2
  const int64_t phase2 = 4 * 10 * (int64_t)(n + 2) + (n + 2) + 16;
  s.total = s.region + (phase1 > phase2 ? phase1 : phase2);
  return s;
}

// K1 epilogue: every class row of Hc becomes its exclusive prefix (Hc[c][L] = the class
// total), P[x] = #{len < x} over all classes; one multi-value block scan for the CM
// class sums and sum(len) (<= n * (L - 1) < 2^24: fits 32 bits)
template <int CM>
__device__ __forceinline__ void small_prefix(uint32_t* Hc, uint32_t* P, int32_t L, int32_t C,
                                             uint32_t* scratch, uint32_t& tot, uint32_t& sltot) {
  const int nt = blockDim.x, tid = threadIdx.x;
  const int32_t LP = hrow(L);
  const int chunk = (L + nt - 1) / nt;  // <= 16 (host: L <= 8192)
  const int x0 = min(L, tid * chunk), x1 = min(L, x0 + chunk);
  uint32_t v[CM + 1], ct[CM + 1];
#pragma unroll
  for (int c = 0; c <= CM; ++c) v[c] = 0;
  for (int x = x0; x < x1; ++x) {
    const int32_t px = hx(x);
    uint32_t h = 0;
#pragma unroll
    for (int c = 0; c < CM; ++c)
      if (c < C) { const uint32_t q = Hc[c * LP + px]; v[c] += q; h += q; }
    v[CM] += h * (uint32_t)x;
  }
  block_excl_scan_k<CM + 1, uint32_t>(v, ct, scratch);
  for (int x = x0; x < x1; ++x) {
    const int32_t px = hx(x);
    uint32_t sx = 0;
#pragma unroll
    for (int c = 0; c < CM; ++c)
      if (c < C) {
        const uint32_t h = Hc[c * LP + px];
        Hc[c * LP + px] = v[c];
        sx += v[c];
        v[c] += h;
      }
    P[px] = sx;
  }
  tot = 0;
#pragma unroll
  for (int c = 0; c < CM; ++c) tot += ct[c];
  sltot = ct[CM];
  if (tid == 0) {
#pragma unroll
    for (int c = 0; c < CM; ++c)
      if (c < C) Hc[c * LP + hx(L)] = ct[c];
  }
}

__global__ void __launch_bounds__(kSmallT, 1)
    k_window_small(const int32_t* __restrict__ len, const uint8_t* __restrict__ cls, int32_t n,
                   bs_window_params p, const int32_t* __restrict__ init_edges, int32_t k_init,
                   int32_t ptok, uint32_t* __restrict__ hist, int32_t* __restrict__ edges_out,
                   int32_t* __restrict__ changes_out, int32_t changes_cap,
                   int32_t* __restrict__ bucket_out, int32_t* __restrict__ perm_out,
                   int32_t* __restrict__ seg_off_out, bs_batch* __restrict__ batches,
                   int32_t batches_cap, int32_t* __restrict__ req_batch,
                   int32_t* __restrict__ req_row, int32_t* __restrict__ rowpos,
                   int64_t* __restrict__ task_base, bs_summary* __restrict__ sum,
                   const int64_t* __restrict__ tok_off, SmallRow* __restrict__ rows,
                   int32_t* __restrict__ nrows, int timing) {
  pdl_prologue();
  BS_SMALL_MARK(0);
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ SmallSh sh;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int nwarps = nt >> 5;
  const unsigned FULL = 0xffffffffu;
  const int32_t L = p.l_max, C = p.n_classes, LP = hrow(L);
  const SmallLayout lay = small_layout(n, L, C);
  int32_t* xs = reinterpret_cast<int32_t*>(smem + lay.xs);       // [n] lengths (arrival order)
  int32_t* seg = reinterpret_cast<int32_t*>(smem + lay.seg);     // [n] segment of request i
  int32_t* goff = reinterpret_cast<int32_t*>(smem + lay.goff);   // [n] sorted offset of i's group
  int32_t* perm_s = reinterpret_cast<int32_t*>(smem + lay.perm); // [n] drain order
  int32_t* runid = reinterpret_cast<int32_t*>(smem + lay.runid); // [n] group id, then run id
  int32_t* aex = reinterpret_cast<int32_t*>(smem + lay.aex);     // [n+1] admitted prefix
  uint8_t* cs = smem + lay.cs;                                   // [n] classes
  unsigned char* region = smem + lay.region;
  uint32_t* Hc = reinterpret_cast<uint32_t*>(region + lay.hc);   // [C][hrow(L)], index hx(x)
  uint32_t* P = reinterpret_cast<uint32_t*>(region + lay.P);     // [hrow(L)], index hx(x)
  int32_t* e = reinterpret_cast<int32_t*>(region + lay.e);       // [L+1]
  int32_t* ne = reinterpret_cast<int32_t*>(region + lay.ne);     // [L+1]
  if (tid == 0) {
    sh.flags = 0; sh.bad = 0; sh.rej = sh.pend = sh.adm_tok = sh.pad_tok = sh.peak = 0;
    sh.wsum = 0.0;
  }
  // ---- K1 -------------------------------------------------------------------------------
  for (int i = tid; i < C * LP; i += nt) Hc[i] = 0;
  __syncthreads();
  {
    unsigned fl = 0;
    for (int i = tid; i < n; i += nt) {
      const int32_t x = eff_len(len[i], L, p.truncate, fl);
      const int32_t c = eff_cls(cls[i], C, fl);
      xs[i] = x;
      cs[i] = (uint8_t)c;
      atomicAdd(&Hc[c * LP + hx(x)], 1u);
    }
    if (fl) atomicOr(&sh.flags, fl);
  }
  __syncthreads();
  BS_SMALL_MARK(1);
  for (int c = 0; c < C; ++c)
    for (int x = tid; x < L; x += nt) hist[c * L + x] = Hc[c * LP + hx(x)];
  {
    uint32_t tot, sl;
    if (C <= 2) small_prefix<2>(Hc, P, L, C, sh.s32m, tot, sl);
    else if (C <= 4) small_prefix<4>(Hc, P, L, C, sh.s32m, tot, sl);
    else small_prefix<8>(Hc, P, L, C, sh.s32m, tot, sl);
    if (tid == 0) {
      const int64_t sltot = sl;
      P[hx(L)] = tot;
      sh.total = tot;
      int64_t nm;
      if (p.n_max > 0) {
        nm = p.n_max;
      } else if (tot == 0) {
        nm = 1;
      } else {
        const double mean = __ddiv_rn((double)sltot, (double)tot);
        if (mean == 0.0) {
          atomicOr(&sh.flags, (unsigned)BS_FLAG_ZERO_MEAN);
          nm = 1;
        } else {
          nm = (int64_t)py_floordiv((double)(p.current_safe / p.kv_bytes_per_token), mean);
          if (nm < 1) nm = 1;
        }
      }
      sh.n_max = nm;
      sh.sum_len = sltot;
      sum->total_global = tot;
      sum->sum_len_global = sltot;
      sum->n_max = nm;
    }
  }
  // ---- K2: initial edges, then adjust_buckets passes (bucket_manager.py:133-191) ------
  if (init_edges) {
    for (int i = tid; i <= k_init; i += nt) {
      const int32_t v = init_edges[i];
      bool ok = v >= 0 && v <= L;
      if (i == 0) ok = ok && v == 0;
      if (i == k_init) ok = ok && v == L;
      if (i > 0) ok = ok && init_edges[i - 1] < v;
      if (!ok) sh.bad = 1;
      e[i] = v;
    }
  }
  __syncthreads();
  if (tid == 0) {
    if (!init_edges || sh.bad || k_init < 1) {
      if (init_edges) atomicOr(&sh.flags, (unsigned)BS_FLAG_BAD_EDGES);
      e[0] = 0;
      e[1] = L;
      sh.k = 1;
    } else {
      sh.k = k_init;
    }
    sh.nch = 0;
    sh.passes = 0;
  }
  __syncthreads();
  const int64_t n_max = sh.n_max;
  const uint32_t total = sh.total;
  if (p.adjust) {
    for (;;) {
      const int32_t K = sh.k;
      __syncthreads();
      if (tid == 0) ++sh.passes;
      if ((int64_t)total < n_max) {  // merge branch (:148-156)
        if (tid == 0 && K != 1) {
          e[0] = 0;
          e[1] = L;
          sh.k = 1;
          if (sh.nch < changes_cap) {
            int32_t* r = changes_out + 4 * sh.nch;
            r[0] = BS_CHANGE_MERGE; r[1] = 0; r[2] = L; r[3] = -1;
          }
          ++sh.nch;
        }
        __syncthreads();
        break;
      }
      if ((int64_t)total == n_max) break;  // (:158-160)
      // one pass: every bucket decides from the counts, left to right (:162-188)
      const int chunk = (K + nt - 1) / nt;  // <= 16
      const int b0 = min(K, tid * chunk), b1 = min(K, b0 + chunk);
      uint8_t kind[16];
      int32_t ecnt = 0, ccnt = 0;
      for (int b = b0; b < b1; ++b) {
        const int32_t lo = e[b], up = e[b + 1], mid = (lo + up) >> 1;
        const uint32_t c = P[hx(up)] - P[hx(lo)], s = P[hx(mid)] - P[hx(lo)];
        uint8_t kd = 0;
        if ((int64_t)c > n_max && (double)s > __dmul_rn(p.split_threshold, (double)c))
          kd = mid <= lo ? 2 : 1;  // 2: width-1 skip (:175-178)
        kind[b - b0] = kd;
        ecnt += 1 + (kd == 1);
        ccnt += kd != 0;
      }
      int32_t sv[2] = {ecnt, ccnt}, stt[2];
      block_excl_scan_k<2, int32_t>(sv, stt, sh.i32m);
      const int32_t etot = stt[0], ctot = stt[1];
      int32_t ep = sv[0] + 1, cp = sv[1];
      int any = 0;
      const int64_t nch0 = sh.nch;
      for (int b = b0; b < b1; ++b) {
        const int32_t lo = e[b], up = e[b + 1], mid = (lo + up) >> 1;
        const uint8_t kd = kind[b - b0];
        if (kd) {
          const int64_t ci = nch0 + cp++;
          if (ci < changes_cap) {
            int32_t* r = changes_out + 4 * ci;
            r[0] = kd == 1 ? BS_CHANGE_SPLIT : BS_CHANGE_SKIP; r[1] = lo; r[2] = up; r[3] = mid;
          }
        }
        if (kd == 1) { ne[ep++] = mid; any = 1; }
        ne[ep++] = up;
      }
      any = __syncthreads_or(any);
      if (tid == 0) {
        ne[0] = 0;
        sh.k = etot;
        sh.nch = nch0 + ctot;
      }
      __syncthreads();
      for (int i = tid; i <= etot; i += nt) e[i] = ne[i];
      __syncthreads();
      if (!any) break;
      if (p.max_passes > 0 && sh.passes >= p.max_passes) break;
    }
  }
  __syncthreads();
  BS_SMALL_MARK(2);
  const int32_t K = sh.k;
  for (int i = tid; i <= K; i += nt) edges_out[i] = e[i];
  if (tid == 0) {
    sum->k_buckets = K;
    sum->n_changes = sh.nch;
    sum->n_passes = sh.passes;
    if (sh.nch > changes_cap) atomicOr(&sh.flags, (unsigned)BS_FLAG_CHANGES_TRUNC);
  }
  // ---- K3 + K4: bucket ids and the stable counting sort ---------------------------------
  const int64_t S = p.current_safe / p.kv_bytes_per_token;
  for (int i = tid; i < n; i += nt) {
    const int32_t x = xs[i];
    int lo = 0, hi = K - 1;  // first b with x < e[b+1]
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (x < e[mid + 1]) hi = mid; else lo = mid + 1;
    }
    if (bucket_out) bucket_out[i] = lo;
    const int32_t blo = e[lo], bup = e[lo + 1];
    const int c = cs[i];
    const int32_t hlo = hx(blo), hup = hx(bup);
    int32_t base = (int32_t)P[hlo];  // requests of earlier buckets, then earlier classes
    for (int c2 = 0; c2 < c; ++c2) base += (int32_t)(Hc[c2 * LP + hup] - Hc[c2 * LP + hlo]);
    const uint32_t* row = Hc + c * LP;
    const int pol = small_policy(p, c);
    int32_t off;
    if (pol == BS_POLICY_SJF) off = base + (int32_t)(row[hx(x)] - row[hlo]);
    else if (pol == BS_POLICY_LJF) off = base + (int32_t)(row[hup] - row[hx(x + 1)]);
    else off = base;
    seg[i] = lo * C + c;
    goff[i] = off;  // the sorted offset of i's group: (class, length) or (class, bucket)
  }
  const int32_t nseg = K * C;
  for (int s2 = tid; s2 <= nseg; s2 += nt) {  // segment offsets of the drain order
    int32_t v = n;
    if (s2 < nseg) {
      const int b = s2 / C, c = s2 - b * C;
      const int32_t blo = e[b], bup = e[b + 1];
      v = (int32_t)P[hx(blo)];
      for (int c2 = 0; c2 < c; ++c2) v += (int32_t)(Hc[c2 * LP + hx(bup)] - Hc[c2 * LP + hx(blo)]);
    }
    seg_off_out[s2] = v;
  }
  __syncthreads();
  BS_SMALL_MARK(10);
  {  // the drain order = the requests stably sorted by their group's offset goff[i] (< n):
     // two LSD passes of 6-bit digits; warp w ranks its contiguous chunk (match_any per
     // 32 requests, per-warp digit counters), one block scan of the counters digit-major
     // gives every (digit, warp) its output base
    int32_t* tk = runid;  // pass-0 output keys / values (dead until K5)
    int32_t* tv = aex;
    uint32_t* wc = reinterpret_cast<uint32_t*>(region);  // [kRankDig][kRankPitch]
    const int CH = ((n + nwarps - 1) / nwarps + 31) & ~31;
    const int i_lo = wid * CH, i_hi = min(n, i_lo + CH);
    for (int pass = 0; pass < 2; ++pass) {
      const int32_t* ik = pass ? tk : goff;
      const int shift = pass ? 6 : 0;
      for (int q = tid; q < kRankDig * kRankPitch; q += nt) wc[q] = 0;
      __syncthreads();
      int32_t loc[4], dg[4];
#pragma unroll
      for (int st2 = 0; st2 < 4; ++st2) {
        dg[st2] = -1;
        loc[st2] = 0;
        if (i_lo + st2 * 32 < i_hi) {  // warp-uniform
          const int i = i_lo + st2 * 32 + lane;
          const bool valid = i < i_hi;
          const int32_t d = valid ? (ik[i] >> shift) & (kRankDig - 1) : -1 - lane;
          const unsigned peers = __match_any_sync(FULL, d);
          const int leader = __ffs(peers) - 1;
          uint32_t b0 = 0;
          if (valid && lane == leader) {
            b0 = wc[d * kRankPitch + wid];
            wc[d * kRankPitch + wid] = b0 + __popc(peers);
          }
          __syncwarp();  // the next step's leaders read these counters
          b0 = __shfl_sync(FULL, b0, leader);
          dg[st2] = valid ? d : -1;
          loc[st2] = (int32_t)b0 + __popc(peers & lanemask_lt());
        }
      }
      __syncthreads();
      {  // exclusive scan over (digit, warp); kRankDig * nwarps == 2 * nt
        const int e0 = 2 * tid, e1 = e0 + 1;
        const int a0i = (e0 / nwarps) * kRankPitch + e0 % nwarps;
        const int a1i = (e1 / nwarps) * kRankPitch + e1 % nwarps;
        const int32_t a0 = (int32_t)wc[a0i], a1 = (int32_t)wc[a1i];
        int32_t tt;
        const int32_t ex = block_excl_scan<int32_t>(a0 + a1, sh.s32, &tt);
        wc[a0i] = (uint32_t)ex;
        wc[a1i] = (uint32_t)(ex + a0);
      }
      __syncthreads();
#pragma unroll
      for (int st2 = 0; st2 < 4; ++st2) {
        if (dg[st2] >= 0) {
          const int i = i_lo + st2 * 32 + lane;
          const int32_t pos = (int32_t)wc[dg[st2] * kRankPitch + wid] + loc[st2];
          if (pass == 0) { tk[pos] = goff[i]; tv[pos] = i; }
          else perm_s[pos] = tv[i];
        }
      }
      __syncthreads();
      if (pass == 0) BS_SMALL_MARK(11);
    }
  }
  BS_SMALL_MARK(3);
  for (int j = tid; j < n; j += nt) perm_out[j] = perm_s[j];
  // ---- K5 -------------------------------------------------------------------------------
  // the K1..K4 region is dead: it now holds the run / batch tables
  const int nr = n + 2;
  int32_t* run_start = reinterpret_cast<int32_t*>(region);  // [nruns+1] first position
  int32_t* run_seg = run_start + nr;                          // [nruns] segment id
  int32_t* run_pend = run_seg + nr;                           // [nruns] first pending position
  int32_t* bpos = run_pend + nr;                              // [nb+1] batch (call) start
  int32_t* bn = bpos + nr;                                    // [nb] admitted rows
  int32_t* bmx = bn + nr;                                     // [nb] max_input_len
  int32_t* bsm = bmx + nr;                                    // [nb] token_sum
  int32_t* bpk = bsm + nr;                                    // [nb+1] n * pitch, then its scan
  int32_t* bpc = bpk + nr;                                    // [nb+1] K6 pieces, then its scan
  int32_t* brw = bpc + nr;                                    // [nb+1] rows, then its scan
  uint8_t* bflag = reinterpret_cast<uint8_t*>(brw + nr);     // [n] a batch's call starts here
  {  // segment runs of the drain order; run id of every position
    const int chunk = (n + nt - 1) / nt;
    const int j0 = min(n, tid * chunk), j1 = min(n, j0 + chunk);
    int32_t cnt = 0;
    for (int j = j0; j < j1; ++j) {
      cnt += j == 0 || seg[perm_s[j]] != seg[perm_s[j - 1]];
      bflag[j] = 0;
    }
    int32_t tot;
    int32_t r = block_excl_scan<int32_t>(cnt, sh.s32, &tot);
    for (int j = j0; j < j1; ++j) {
      if (j == 0 || seg[perm_s[j]] != seg[perm_s[j - 1]]) {
        run_start[r] = j;
        run_seg[r] = seg[perm_s[j]];
        ++r;
      }
      runid[j] = r - 1;
    }
    if (tid == 0) {
      sh.nruns = tot;
      run_start[tot] = n;
    }
  }
  __syncthreads();
  BS_SMALL_MARK(4);
  const int nruns = sh.nruns;
  int32_t* bid = seg;  // [n] batch of each position (seg is dead once the runs are known)
  const int64_t Hd = p.current_safe - p.pledged;
  const bool padded = p.accounting == BS_ACCOUNTING_PADDED;
  const int64_t T = Hd > 0 ? Hd / p.kv_bytes_per_token : 0;
  // A: the form_batch calls of every segment run: where each call that admits something
  //    starts, and where the drain stops.  Every position first learns, by its own scan
  //    of at most kNextCap positions, where a call starting there would end; one warp per
  //    run then hops from call to call, and only a call longer than the cap is re-scanned
  //    by the warp, 32 positions per step
  int32_t* xd = bn;    // [n] lengths in drain order (bn / bmx are free until the batch tables)
  int32_t* nxt = bmx;  // [n] end of the call starting at j: k, or -1 - k when it admits
                       // nothing (the drain stops at k), or kNxtUnknown past the cap
  constexpr int kNextCap = 32;
  // the scan's products stay below 8192 * 33 < 2^19: clamped budgets compare the same
  const int32_t S32 = S < (1 << 30) ? (int32_t)S : (1 << 30);
  const int32_t T32 = T < (1 << 30) ? (int32_t)T : (1 << 30);
  constexpr int32_t kNxtUnknown = INT32_MIN;
  for (int j = tid; j < n; j += nt) xd[j] = xs[perm_s[j]];
  __syncthreads();
  BS_SMALL_MARK(8);
  // the per-position scan pays only where the average call (budget / mean length) is
  // shorter than the cap; otherwise every call is found by the warp
  const bool prescan = Hd > 0 && (int64_t)T * sh.total < (int64_t)kNextCap * sh.sum_len;
  if (prescan) {
    for (int j = tid; j < n; j += nt) {
      const int32_t b = run_start[runid[j] + 1];
      const int32_t kend = min(b, j + kNextCap);
      int32_t cnt = 0, m = 0, sm = 0, res = kNxtUnknown;
      for (int32_t k0 = j; k0 < kend; k0 += 8) {
        int32_t xv[8];  // eight lengths loaded ahead (lengths are >= 0; -1 = past the end)
#pragma unroll
        for (int u = 0; u < 8; ++u) xv[u] = k0 + u < kend ? xd[k0 + u] : -1;
        int hit = 8, c_hit = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {  // 32-bit: x < 8192, cnt <= kNextCap, S32 / T32 clamped
          const int32_t x = xv[u];
          const bool adm = x >= 0 && x <= S32;  // rejected ones are skipped
          const int32_t cm = x > m ? x : m;
          const bool viol = adm && (padded ? cm * (cnt + 1) : sm + x) > T32;
          if (viol && hit == 8) { hit = u; c_hit = cnt; }
          if (adm && hit == 8) { ++cnt; m = cm; sm += x; }
        }
        if (hit < 8) {
          res = c_hit ? k0 + hit : -1 - (k0 + hit);
          break;
        }
      }
      if (res == kNxtUnknown && kend == b) res = cnt ? b : -1 - b;
      nxt[j] = res;
    }
  }
  __syncthreads();
  BS_SMALL_MARK(9);
  for (int r = wid; r < nruns; r += nwarps) {
    const int32_t a = run_start[r], b = run_start[r + 1];
    // run order: SJF ascending lengths, LJF descending, FCFS arrival (K4)
    const int pol = small_policy(p, run_seg[r] % C);
    int32_t pos = a, pend = b;
    if (Hd <= 0) pend = a;  // form_batch returns None before touching the queue (:150-152)
    while (Hd > 0 && pos < b) {
      int32_t nx = prescan ? nxt[pos] : kNxtUnknown;
      if (nx == kNxtUnknown) {  // a call longer than the cap
        int32_t cnt = 0, m = 0, sm = 0, q = pos;
        for (;;) {
          if (q >= b) { nx = cnt ? b : -1 - b; break; }
          const int32_t j = q + lane;
          const bool valid = j < b;
          const int32_t x = valid ? xd[j] : 0;
          const bool adm = valid && (int64_t)x <= S;
          int32_t pc = adm, pm = adm ? x : 0, ps = adm ? x : 0;  // lane prefix over admissible
          if (__all_sync(FULL, adm || !valid)) {
            // every valid lane admissible (the valid lanes are a prefix): the count is the
            // lane, the padded accounting needs only the running max — the own length in
            // an ascending run, the step's first in a descending one — the exact one only
            // the sum
            pc = lane + 1;
            if (padded) {
              if (pol == BS_POLICY_LJF) pm = __shfl_sync(FULL, x, 0);
              else if (pol != BS_POLICY_SJF) pm = warp_incl_max(pm);
            } else {
              ps = warp_incl_scan(ps);
            }
          } else {
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int32_t tc = __shfl_up_sync(FULL, pc, o);
              const int32_t tm = __shfl_up_sync(FULL, pm, o);
              const int32_t ts = __shfl_up_sync(FULL, ps, o);
              if (lane >= o) { pc += tc; pm = tm > pm ? tm : pm; ps += ts; }
            }
          }
          const int32_t cm = pm > m ? pm : m;
          const bool viol = adm && (padded ? (int64_t)cm * (cnt + pc) : (int64_t)(sm + ps)) > T;
          const unsigned vb = __ballot_sync(FULL, viol);
          const int f = vb ? __ffs(vb) - 1 : min(32, b - q);  // lanes < f are consumed
          if (f > 0) {
            cnt += __shfl_sync(FULL, pc, f - 1);
            m = max(m, __shfl_sync(FULL, pm, f - 1));
            sm += __shfl_sync(FULL, ps, f - 1);
          }
          q += f;
          if (vb) { nx = cnt ? q : -1 - q; break; }
        }
      }
      if (nx < 0) {  // this call admits nothing: the drain of the segment stops here
        pend = -1 - nx;
        break;
      }
      bflag[pos] = 1;  // the call closes its batch; the next starts at nx (every lane: no branch)
      pos = nx;
    }
    if (lane == 0) run_pend[r] = pend;

  }
  __syncthreads();
  BS_SMALL_MARK(5);
  // batch ids in emission order (the exclusive prefix of the call-start flags) and every
  // position's admitted prefix
  {
    const int chunk = (n + nt - 1) / nt;
    const int j0 = min(n, tid * chunk), j1 = min(n, j0 + chunk);
    int32_t cf = 0, ca = 0;
    for (int j = j0; j < j1; ++j) {
      cf += bflag[j];
      ca += j < run_pend[runid[j]] && (int64_t)xs[perm_s[j]] <= S;
    }
    int32_t sv[2] = {cf, ca}, stt[2];
    block_excl_scan_k<2, int32_t>(sv, stt, sh.i32m);
    const int32_t tf = stt[0], ta = stt[1];
    int32_t q = sv[0], qa = sv[1];
    for (int j = j0; j < j1; ++j) {
      if (bflag[j]) bpos[q++] = j;
      bid[j] = q - 1;  // the last call start <= j: the batch of j when j is admitted
      aex[j] = qa;
      qa += j < run_pend[runid[j]] && (int64_t)xs[perm_s[j]] <= S;
    }
    if (tid == 0) {
      sh.nb = tf;
      aex[n] = ta;
    }
  }
  __syncthreads();
  const int nb = sh.nb;
  uint8_t* bnp = bflag;  // the call-start flags are dead: per-batch "admitted a length < 1"
  for (int bi = tid; bi < nb; bi += nt) { bn[bi] = 0; bmx[bi] = 0; bsm[bi] = 0; bnp[bi] = 0; }
  __syncthreads();
  // batch of every admitted position (last call start <= j); statistics by shared atomics
  unsigned fl = 0;
  for (int j = tid; j < n; j += nt) {
    const int32_t x = xs[perm_s[j]];
    if (!(j < run_pend[runid[j]] && (int64_t)x <= S)) continue;
    const int lo = bid[j];
    atomicAdd(&bn[lo], 1);
    atomicMax(&bmx[lo], x);
    atomicAdd(&bsm[lo], x);
    if (x < 1) {  // waste_ratio raises for it (memory_model.py:96-97)
      fl |= BS_FLAG_NONPOS_LEN;
      bnp[lo] = 1;
    }
  }
  __syncthreads();
  for (int bi = tid; bi < nb; bi += nt) {
    const int32_t pitch = (bmx[bi] + BS_PACK_ALIGN - 1) / BS_PACK_ALIGN * BS_PACK_ALIGN;
    bpk[bi] = bn[bi] * pitch;
    bpc[bi] = bn[bi] * ((pitch + ptok - 1) / ptok);
    brw[bi] = bn[bi];
  }
  __syncthreads();
  int32_t packed_tot, piece_tot;
  {  // exclusive scans of the three per-batch tables with one pair of barriers
    const int chunk = (nb + nt - 1) / nt;
    const int lo = min(nb, tid * chunk), hi = min(nb, lo + chunk);
    int32_t sv[3] = {0, 0, 0}, stt[3];
    for (int i = lo; i < hi; ++i) { sv[0] += bpk[i]; sv[1] += bpc[i]; sv[2] += brw[i]; }
    block_excl_scan_k<3, int32_t>(sv, stt, sh.i32m);
    for (int i = lo; i < hi; ++i) {
      const int32_t a0 = bpk[i], a1 = bpc[i], a2 = brw[i];
      bpk[i] = sv[0]; bpc[i] = sv[1]; brw[i] = sv[2];
      sv[0] += a0; sv[1] += a1; sv[2] += a2;
    }
    packed_tot = stt[0];
    piece_tot = stt[1];
    __syncthreads();
  }
  BS_SMALL_MARK(6);
  // outcomes, rows and the K6 row map of every position
  unsigned long long rej = 0, pend = 0;
  for (int j = tid; j < n; j += nt) {
    const int32_t idx = perm_s[j];
    const int32_t x = xs[idx];
    if (j >= run_pend[runid[j]]) {
      req_batch[idx] = BS_REQ_PENDING;
      req_row[idx] = -1;
      ++pend;
    } else if ((int64_t)x > S) {
      req_batch[idx] = BS_REQ_REJECTED;
      req_row[idx] = -1;
      ++rej;
    } else {
      const int lo = bid[j];
      const int32_t row = aex[j] - aex[bpos[lo]];
      req_batch[idx] = lo;
      req_row[idx] = row;
      rowpos[brw[lo] + row] = j;
      if (tok_off) {  // the row's copy job for k_pack_rows
        const int32_t pitch = (bmx[lo] + BS_PACK_ALIGN - 1) / BS_PACK_ALIGN * BS_PACK_ALIGN;
        SmallRow rw;
        rw.src = tok_off[idx];
        rw.dst = (int64_t)bpk[lo] + (int64_t)row * pitch;
        rw.x = x;
        rw.pitch = pitch;
        rows[brw[lo] + row] = rw;
      }
    }
  }
  // batch descriptors (BatchPlan fields, waste_ratio) and totals
  unsigned long long adm_tok = 0, pad_tok = 0, peak = 0;
  double ws = 0.0;
  for (int bi = tid; bi < nb; bi += nt) {
    const int32_t a = bpos[bi], r = runid[a];
    const int32_t e2 = (bi + 1 < nb && bpos[bi + 1] < run_start[r + 1]) ? bpos[bi + 1] : run_pend[r];
    const int32_t c = bn[bi], mx = bmx[bi], sm = bsm[bi];
    const int64_t fp = p.kv_bytes_per_token * (padded ? (int64_t)mx * c : (int64_t)sm);
    // waste_ratio (memory_model.py:98-100); NaN where the reference raises (:96-97)
    const bool np = bnp[bi] != 0;
    const double avg = __ddiv_rn((double)sm, (double)c);
    const double w = np ? __longlong_as_double(0x7ff8000000000000LL)
                        : __ddiv_rn(__dsub_rn((double)mx, avg), (double)mx);
    if (bi < batches_cap) {
      bs_batch B;
      B.segment = run_seg[r];
      B.start = a;
      B.end = e2;
      B.n = c;
      B.max_input_len = mx;
      B.pitch = (mx + BS_PACK_ALIGN - 1) / BS_PACK_ALIGN * BS_PACK_ALIGN;
      B.token_sum = sm;
      B.footprint = fp;
      B.out_offset = bpk[bi];
      B.waste = w;
      B.row_base = brw[bi];
      batches[bi] = B;
      task_base[bi] = bpc[bi];
      ws = __dadd_rn(ws, w);
    }
    adm_tok += (unsigned long long)sm;
    pad_tok += (unsigned long long)mx * (unsigned long long)c;
    peak = (unsigned long long)fp > peak ? (unsigned long long)fp : peak;
  }
  rej = warp_sum(rej);
  pend = warp_sum(pend);
  adm_tok = warp_sum(adm_tok);
  pad_tok = warp_sum(pad_tok);
  peak = warp_max(peak);
  ws = warp_sum(ws);
  fl = __reduce_or_sync(FULL, fl);
  if (lane == 0) {
    atomicAdd(&sh.rej, rej);
    atomicAdd(&sh.pend, pend);
    atomicAdd(&sh.adm_tok, adm_tok);
    atomicAdd(&sh.pad_tok, pad_tok);
    atomicMax(&sh.peak, peak);
    atomicAdd(&sh.wsum, ws);
    if (fl) atomicOr(&sh.flags, fl);
  }
  __syncthreads();
  BS_SMALL_MARK(7);
  if (tid == 0) {
    const int nbc = nb < batches_cap ? nb : batches_cap;
    task_base[nbc] = piece_tot;
    *nrows = nbc < nb ? brw[nbc] : (nb ? brw[nb - 1] + bn[nb - 1] : 0);
    sum->n_requests = n;
    sum->n_batches = nb;
    sum->n_rejected = (int64_t)sh.rej;
    sum->n_pending = (int64_t)sh.pend;
    sum->admitted_tokens = (int64_t)sh.adm_tok;
    sum->padded_tokens = (int64_t)sh.pad_tok;
    sum->packed_elems = packed_tot;
    sum->peak_footprint = (int64_t)sh.peak;
    sum->waste_sum = sh.wsum;
    sum->sort_passes = 0;
    unsigned f2 = sh.flags;
    if (nb > batches_cap) f2 |= BS_FLAG_BATCH_CAP;
    sum->flags = f2;
    sum->n_dispatched = 0;
  }
}

size_t small_smem_bytes(int32_t n, int32_t L, int32_t C) {
  return (size_t)small_layout(n, L, C).total;
}

// eligible windows: no dispatch order, one rank, n <= kSmallN, L <= 8192, C*L <= 16384
bool small_window_ok(const bs_ctx* ctx, int64_t n, const bs_window_params& p, int32_t k_init) {
  if (!ctx->small_path || p.dispatch || n > kSmallN || p.l_max > 8192 ||
      (int64_t)p.l_max * p.n_classes > 16384 || k_init > p.l_max)
    return false;
  return small_smem_bytes((int32_t)n, p.l_max, p.n_classes) <= (size_t)ctx->small_smem_max;
}

cudaError_t small_prepare(bs_ctx* ctx) {
  int optin = 0;
  cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
  if (e != cudaSuccess) return e;
  cudaFuncAttributes fa;
  if ((e = cudaFuncGetAttributes(&fa, k_window_small)) != cudaSuccess) return e;
  ctx->small_smem_max = optin - (int)fa.sharedSizeBytes;
  return cudaFuncSetAttribute(k_window_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              ctx->small_smem_max);
}

cudaError_t launch_window_small(bs_ctx* ctx, const bs_window_io* io, const bs_window_params& p,
                                cudaStream_t st) {
  const int32_t n = (int32_t)io->n;
  ctx->piece_tok = piece_tokens_for(n);
  ctx->pack_pieces = (int64_t)n * (((int64_t)p.l_max + ctx->piece_tok - 1) / ctx->piece_tok);
  const size_t smem = small_smem_bytes(n, p.l_max, p.n_classes);
  launch_k(ctx, k_window_small, dim3(1), dim3(kSmallT), smem, st, false, io->len, io->cls, n, p,
           io->init_edges, io->init_edges ? io->k_init : 0, ctx->piece_tok, io->hist, io->edges,
           io->changes, io->changes_cap, io->bucket, io->perm, io->seg_off, io->batches,
           io->batches_cap, io->req_batch, io->req_row, ctx->rowpos, ctx->task_base, io->summary,
           io->tok_off, reinterpret_cast<SmallRow*>(ctx->small_rows), ctx->misc, ctx->small_timing);
  ++ctx->launches;
  return cudaGetLastError();
}

}  // namespace bsk
