// K7 — global batch emission order.
//
// Reference: the simulator dispatches with Simulator._next_plan (pd_sim.py:448-462):
// for each class in priority order (ONLINE, OFFLINE), BatchController.select_bucket
// (batch_controller.py:106-134) picks a bucket — ONLINE: the bucket holding the
// globally oldest queued online request (:114-123); OFFLINE: the largest queued
// offline token mass, strict > from 0, ties to the lower index (:124-134) — and
// form_batch runs on it; the first plan ends the call.  Repeated while it makes
// progress (a plan, or rejections: the set is marked dirty, :457-459).
// Generalisation to C classes: class 0 uses the oldest-request rule, every other
// class the token-mass rule of its own class (C = 2 is the reference exactly).
//
// With fixed current_safe / pledged the form_batch calls of one (bucket, class)
// segment do not depend on the other segments, so K5 already produced every call:
// the chain nodes (listA, node_batch: a batch, or -1 for the segment's null tail
// call).  Only the interleaving is left, and it is data-parallel:
//   * a call's selection key is a function of what is still queued in its segment:
//     class 0: min arrival rank over [call start, segment end) (strictly increasing
//     along a segment); class c >= 1: token mass over the same range (non-increasing).
//     The greedy argmin / argmax over segments is then exactly a k-way merge of the
//     per-segment call lists, i.e. a stable sort of all calls by
//     (class, rank | (mass desc, bucket asc)).  Zero-mass calls are never selected.
//   * the classes interleave only at null calls (a call that forms no plan cascades
//     to the next class inside the same _next_plan): one thread walks the (rare)
//     null calls and emits runs of consecutive plans; everything else is parallel.
//
// Work split: K5c/K5e already reduced every call's own range (min rank, length sum
// into disp_cmin / disp_csum, segment into disp_cseg).  K7 is ONE cooperative kernel
// (one 1024-thread CTA per SM):
//   keys    reverse segmented scan over the calls (suffix min / suffix sum per
//           segment) -> 64-bit keys
//   sort    <= 8192 calls: bitonic sort of (key, call) in CTA 0 (registers, lane
//           shuffles and shared memory); more: stable onesweep LSD radix sort on the
//           key bytes that vary
//   walk    class ranges, null-call list, single-thread walk -> runs of plans
//   emit    emit_order[t] / batch_emit[b] from the runs; requests of calls the loop
//           never reaches go back to PENDING
// Windows with <= kSmallCap calls (C2: 1,911; C4: 4,591) run entirely in CTA 0's shared
// memory with no grid barrier; larger ones (C3: 24,998) use every CTA, onesweep
// radix passes with decoupled look-back, and a grid barrier between phases.
#include <cooperative_groups.h>

#include "ctx.cuh"

namespace cg = cooperative_groups;

namespace bsk {

namespace {

constexpr int kKT = 1024;                  // threads per CTA
constexpr int kKW = kKT / 32;              // warps
constexpr int kKItems = 7;
constexpr int kSmall = kKT * kKItems;      // 7168: radix tile of the multi-CTA path
constexpr int kSmallCap = 8192;            // calls sorted in CTA 0's shared memory (bitonic)
constexpr int kBucketBits = 17;
constexpr uint64_t kMassMax = (1ull << (60 - kBucketBits)) - 1;
constexpr uint64_t kUnreach = ~0ull;

// dynamic shared memory layout (bytes)
constexpr int kOffK0 = 0;
constexpr int kOffK1 = kOffK0 + 8 * kSmall;
constexpr int kOffV0 = kOffK1 + 8 * kSmall;
constexpr int kOffV1 = kOffV0 + 4 * kSmall;
constexpr int kOffCnt = kOffV1 + 4 * kSmall;        // u32 [kKW][256]
constexpr int kOffBin = kOffCnt + 4 * kKW * 256;    // u32 [8][256] bin offsets per active pass
constexpr int kOffDst = kOffBin + 4 * 8 * 256;      // u32 [256]
constexpr int kOffGb = kOffDst + 4 * 256;           // i64 [256]
constexpr int kSmem = kOffGb + 8 * 256;             // 216,064

// dmisc (int64) layout
constexpr int kEmitted = 1;  // plans in the dispatch sequence
constexpr int kRuns = 2;     // run records
constexpr int kUnr = 3;      // 1: some call is never reached
constexpr int kUBeg = 8;     // [8..16)  first unreached sorted position per class
constexpr int kCEnd = 16;    // [16..24) end of class c's sorted range
constexpr int kZBeg = 24;    // first zero-mass (never selected) sorted position

struct Run {
  int32_t start;  // sorted position of the run's first call
  int32_t len;
  int32_t t;      // dispatch rank of the run's first plan
  int32_t pad;
};

}  // namespace

struct SegVal {
  int32_t f;   // a segment head lies within the combined range
  int32_t mn;  // min arrival rank
  int64_t sm;  // length sum
};

struct DispArgs {
  const int32_t* list;        // chain nodes: call start positions (K5c listA)
  const int32_t* node_batch;  // batch of each call, -1 for a null tail call
  const int32_t* node_j0;     // null call: first admissible position of its tail
  const int32_t* misc;        // K5: [64] calls, [66] batches
  const int32_t* seg_off;
  const bs_batch* batches;
  int32_t batches_cap;
  int32_t C;
  const int32_t* perm;
  const int32_t* slen;        // lengths in drain order (K5a)
  const int32_t* cseg;        // per call: segment, min rank, length sum over its own range
  const int32_t* cmin;
  const int64_t* csum;
  uint64_t* keys0;
  uint64_t* keys1;
  uint32_t* vals0;
  uint32_t* vals1;
  uint32_t* hist8;            // [8][256] key-byte histograms (all zero between windows)
  uint32_t* status;           // [8][stat_words] look-back words
  int64_t stat_words;
  uint32_t* tctr;             // [8] tile counters
  int32_t* nulls;             // sorted positions of null calls
  uint64_t* bkeys;            // per null call: key of its blocked bucket's remaining requests
  void* runs;
  int64_t* dmisc;
  SegVal* agg;                // [gridDim.x] chunk aggregates of the key scan
  int32_t* emit_order;
  int32_t* batch_emit;
  int32_t* req_batch;
  int32_t* req_row;
  bs_summary* sum;
};

namespace {

__device__ __forceinline__ SegVal seg_id() { return SegVal{0, INT32_MAX, 0}; }

// scan order: `x` precedes `y`; a head inside `y` cuts the carry
__device__ __forceinline__ SegVal seg_combine(const SegVal& x, const SegVal& y) {
  SegVal r;
  r.f = x.f | y.f;
  r.mn = y.f ? y.mn : min(x.mn, y.mn);
  r.sm = y.f ? y.sm : x.sm + y.sm;
  return r;
}

__device__ __forceinline__ SegVal shfl_up_seg(const SegVal& v, int o) {
  SegVal y;
  y.f = __shfl_up_sync(0xffffffffu, v.f, o);
  y.mn = __shfl_up_sync(0xffffffffu, v.mn, o);
  y.sm = __shfl_up_sync(0xffffffffu, v.sm, o);
  return y;
}

// key of a call from its suffix aggregate
__device__ __forceinline__ uint64_t call_key(int32_t sg, const SegVal& x, int32_t C, unsigned& fl) {
  const int32_t c = sg % C, bucket = sg / C;
  if (c == 0) return (uint64_t)(uint32_t)x.mn;   // oldest queued request of the class
  if (x.sm == 0) return kUnreach;                // select_bucket never picks zero mass
  if ((uint64_t)x.sm > kMassMax || bucket >= (1 << kBucketBits)) fl |= BS_FLAG_DISPATCH_RANGE;
  const uint64_t m = (uint64_t)x.sm > kMassMax ? kMassMax : (uint64_t)x.sm;
  return ((uint64_t)c << 60) | ((kMassMax - m) << kBucketBits) |
         (uint64_t)(bucket & ((1 << kBucketBits) - 1));
}

// Reverse segmented inclusive scan over scan positions [u0, u1) (u = M-1-i: call
// index descending), seeded with `carry`; writes keys[i] / vals[i] when keys is
// set; returns the aggregate (carry combined with the whole range).
__device__ SegVal scan_calls(const DispArgs& a, int M, int u0, int u1, SegVal carry,
                             uint64_t* keys, uint32_t* vals, unsigned& fl) {
  __shared__ SegVal s_w[kKW];
  __shared__ SegVal s_carry;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_carry = carry;
  __syncthreads();
  for (int base = u0; base < u1; base += kKT) {
    const int u = base + tid;
    const bool valid = u < u1;
    const int i = M - 1 - u;
    SegVal x = SegVal{1, INT32_MAX, 0};
    int32_t sg = -1;
    if (valid) {
      sg = a.cseg[i];
      x.f = (u == 0) ? 1 : (sg != a.cseg[i + 1]);
      x.mn = a.cmin[i];
      x.sm = a.csum[i];
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const SegVal y = shfl_up_seg(x, o);
      if (lane >= o) x = seg_combine(y, x);
    }
    if (lane == 31) s_w[wid] = x;
    __syncthreads();
    if (wid == 0) {
      SegVal v = s_w[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const SegVal y = shfl_up_seg(v, o);
        if (lane >= o) v = seg_combine(y, v);
      }
      SegVal ex = shfl_up_seg(v, 1);
      ex = lane == 0 ? s_carry : seg_combine(s_carry, ex);
      s_w[lane] = ex;
    }
    __syncthreads();
    x = seg_combine(s_w[wid], x);
    if (valid && keys) {
      keys[i] = call_key(sg, x, a.C, fl);
      vals[i] = (uint32_t)i;
    }
    __syncthreads();
    const int last = min(base + kKT, u1) - 1 - base;
    if (tid == last) s_carry = x;
    __syncthreads();
  }
  return s_carry;
}

// Stable local rank of up to kSmall items (warp w owns items [w*32*kKItems, ...),
// k-major, lane-minor) by the byte at `shift`.  Leaves per-warp exclusive digit
// offsets in s_cnt, tile digit starts in s_dst; per-item ranks in rank[]; the tile
// count of digit `tid` (tid < 256) in *tc.
__device__ __forceinline__ void tile_rank(const uint64_t (&key)[kKItems], int tbase, int n,
                                          int shift, uint32_t* s_cnt, uint32_t* s_dst,
                                          uint32_t (&rank)[kKItems], uint32_t* tc_out) {
  __shared__ uint32_t s_scan[33];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int i = tid; i < kKW * 256; i += kKT) s_cnt[i] = 0;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kKItems; ++k) {
    const int e = tbase + w * 32 * kKItems + k * 32 + lane;
    const bool valid = e < n;
    const uint32_t d = valid ? (uint32_t)((key[k] >> shift) & 255u) : 0xffffffffu;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (valid && lane == leader) {
      old = s_cnt[w * 256 + d];
      s_cnt[w * 256 + d] = old + __popc(peers);
    }
    old = __shfl_sync(0xffffffffu, old, leader);
    rank[k] = old + __popc(peers & lanemask_lt());
    __syncwarp();
  }
  __syncthreads();
  uint32_t tc = 0;
  if (tid < 256) {
    for (int ww = 0; ww < kKW; ++ww) {
      const uint32_t v = s_cnt[ww * 256 + tid];
      s_cnt[ww * 256 + tid] = tc;
      tc += v;
    }
  }
  uint32_t tot;
  const uint32_t ds = block_excl_scan<uint32_t>(tid < 256 ? tc : 0u, s_scan, &tot);
  if (tid < 256) s_dst[tid] = ds;
  *tc_out = tc;
  __syncthreads();
}

__device__ __forceinline__ bool pair_gt(uint64_t ka, uint32_t va, uint64_t kb, uint32_t vb) {
  return ka > kb || (ka == kb && va > vb);
}

// Bitonic sort of P (power of two, 64 <= P <= 1024*E) (key, val) pairs in shared memory by
// one 1024-thread CTA.  Warp w holds elements [w*32E, (w+1)*32E) in registers (element
// e*32+lane of its span); compare distances < 32 are lane shuffles, < 32E register
// swaps, and only the longer ones go through shared memory.
template <int E>
__device__ void block_bitonic(uint64_t* K, uint32_t* V, int P) {
  constexpr int kSpan = 32 * E;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int base = w * kSpan;
  const bool active = base < P;
  uint64_t k[E];
  uint32_t v[E];
  if (active) {
#pragma unroll
    for (int e = 0; e < E; ++e) { k[e] = K[base + e * 32 + lane]; v[e] = V[base + e * 32 + lane]; }
  }
  for (int kk = 2; kk <= P; kk <<= 1) {
    if ((kk >> 1) >= kSpan) {  // long distances through shared memory
      if (active) {
#pragma unroll
        for (int e = 0; e < E; ++e) { K[base + e * 32 + lane] = k[e]; V[base + e * 32 + lane] = v[e]; }
      }
      __syncthreads();
      for (int j = kk >> 1; j >= kSpan; j >>= 1) {
        for (int i = tid; i < (P >> 1); i += kKT) {
          const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1)), hi = lo + j;
          const uint64_t ka = K[lo], kb = K[hi];
          const uint32_t va = V[lo], vb = V[hi];
          if (pair_gt(ka, va, kb, vb) == ((lo & kk) == 0)) {
            K[lo] = kb; K[hi] = ka;
            V[lo] = vb; V[hi] = va;
          }
        }
        __syncthreads();
      }
      if (active) {
#pragma unroll
        for (int e = 0; e < E; ++e) { k[e] = K[base + e * 32 + lane]; v[e] = V[base + e * 32 + lane]; }
      }
      __syncthreads();
    }
    if (!active) continue;
#pragma unroll
    for (int jb = E / 2; jb >= 1; jb >>= 1) {  // distances 32*jb: register pairs
      if ((jb << 5) <= (kk >> 1)) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int pe = e ^ jb;
          if (pe > e) {
            const bool up = ((base + e * 32 + lane) & kk) == 0;
            if (pair_gt(k[e], v[e], k[pe], v[pe]) == up) {
              const uint64_t tk = k[e]; k[e] = k[pe]; k[pe] = tk;
              const uint32_t tv = v[e]; v[e] = v[pe]; v[pe] = tv;
            }
          }
        }
      }
    }
#pragma unroll
    for (int jj = 16; jj >= 1; jj >>= 1) {  // distances < 32: lane shuffles
      if (jj <= (kk >> 1)) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint64_t ok = __shfl_xor_sync(0xffffffffu, k[e], jj);
          const uint32_t ov = __shfl_xor_sync(0xffffffffu, v[e], jj);
          const bool lower = (lane & jj) == 0;
          const bool up = ((base + e * 32 + lane) & kk) == 0;
          const bool gt = pair_gt(k[e], v[e], ok, ov);
          if ((lower == up) ? gt : !gt) { k[e] = ok; v[e] = ov; }
        }
      }
    }
  }
  if (active) {
#pragma unroll
    for (int e = 0; e < E; ++e) { K[base + e * 32 + lane] = k[e]; V[base + e * 32 + lane] = v[e]; }
  }
  __syncthreads();
}

// null calls in sorted order -> a.nulls (block-wide compaction by one CTA); returns count
__device__ int compact_nulls(const DispArgs& a, const uint32_t* V, int M) {
  __shared__ int32_t s_scan[33];
  int run = 0;
  for (int base = 0; base < M; base += kKT) {
    const int i = base + threadIdx.x;
    const int is_null = (i < M) && a.node_batch[V[i]] < 0;
    int tot;
    const int o = block_excl_scan<int32_t>(is_null, s_scan, &tot);
    if (is_null) a.nulls[run + o] = i;
    run += tot;
  }
  return run;
}

// class boundaries, then the single-thread walk (thread 0 of the calling CTA)
__device__ void walk(const DispArgs& a, const uint64_t* K, const uint32_t* V, int M) {
  __shared__ int64_t s_cb[BS_MAX_CLASSES + 2];
  __shared__ int32_t s_nn;
  const int tid = threadIdx.x, C = a.C;
  if (tid <= C) {
    const uint64_t target = tid < C ? ((uint64_t)tid << 60) : kUnreach;
    int lo = 0, hi = M;  // lower_bound
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (K[mid] < target) lo = mid + 1; else hi = mid;
    }
    s_cb[tid] = lo;
  }
  const int nn_ = compact_nulls(a, V, M);
  // the key a blocked bucket re-enters select_bucket with (min rank / length sum of the
  // requests left after its null call, i.e. from the blocking request to the segment
  // end): one warp per null call reduces its range (a blocked bucket may hold millions of
  // requests), so the single-thread walk below only reads the result
  {
    const int lane = tid & 31, wid = tid >> 5, nwarps = (int)(blockDim.x >> 5);
    unsigned kfl = 0;
    for (int i = wid; i < nn_; i += nwarps) {
      const uint32_t call = V[a.nulls[i]];
      const int32_t sg = a.cseg[call];
      const int64_t j0 = a.node_j0[call], en = a.seg_off[sg + 1];
      if (j0 >= en) continue;  // not blocked: everything left was oversize
      int32_t mn = INT32_MAX;
      int64_t sm = 0;
      for (int64_t j = j0 + lane; j < en; j += 32) {
        mn = min(mn, a.perm[j]);
        sm += a.slen[j];
      }
      mn = -warp_max(-mn);
      sm = warp_sum(sm);
      if (lane == 0) a.bkeys[i] = call_key(sg, SegVal{1, mn, sm}, C, kfl);
    }
    if (kfl) latch_flags(a.sum, kfl);
  }
  if (tid == 0) s_nn = nn_;
  __syncthreads();
  if (tid != 0) return;
  Run* runs = reinterpret_cast<Run*>(a.runs);
  const int nn = s_nn;
  const int32_t* nulls = a.nulls;
  int64_t p[BS_MAX_CLASSES], e[BS_MAX_CLASSES];
  int q[BS_MAX_CLASSES];
  bool stuck[BS_MAX_CLASSES];
  // thr[c]: key of a blocked bucket of class c after its null call.  form_batch removes
  // the oversize requests it meets before the blocking one, so the bucket re-enters
  // select_bucket with the key of its remaining requests; the class is stuck once that
  // key is the best it has left (first call whose key sorts after it)
  uint64_t thr[BS_MAX_CLASSES];
  for (int c = 0; c < C; ++c) {
    p[c] = s_cb[c];
    e[c] = s_cb[c + 1];
    stuck[c] = false;
    thr[c] = kUnreach;
    int lo = 0, hi = nn;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (nulls[mid] < p[c]) lo = mid + 1; else hi = mid;
    }
    q[c] = lo;
  }
  unsigned fl = 0;
  int64_t t = 0;
  int nr = 0;
  for (;;) {
    int c0 = -1;
    for (int c = 0; c < C; ++c)
      if (!stuck[c] && p[c] < e[c]) { c0 = c; break; }
    if (c0 < 0) break;
    // consecutive plans of c0 up to its next null call (one per _next_plan call) or up
    // to the first call that sorts after its pending blocked bucket
    int64_t lim = e[c0];
    if (thr[c0] != kUnreach) {
      int64_t lo = p[c0], hi = e[c0];
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (K[mid] <= thr[c0]) lo = mid + 1; else hi = mid;
      }
      lim = lo;
    }
    int64_t z = (q[c0] < nn && nulls[q[c0]] < e[c0]) ? (int64_t)nulls[q[c0]] : e[c0];
    z = z < lim ? z : lim;
    if (z > p[c0]) {
      runs[nr++] = Run{(int32_t)p[c0], (int32_t)(z - p[c0]), (int32_t)t, 0};
      t += z - p[c0];
      p[c0] = z;
    }
    if (p[c0] == e[c0]) continue;
    // a null call or the blocked bucket at p[c0], then the cascade inside the same
    // _next_plan call
    for (int c = c0; c < C; ++c) {
      if (stuck[c] || p[c] >= e[c]) continue;
      if (thr[c] != kUnreach && K[p[c]] > thr[c]) {
        stuck[c] = true;  // select_bucket returns the blocked bucket from now on
        continue;
      }
      const bool is_null = q[c] < nn && nulls[q[c]] == p[c];
      if (!is_null) {
        runs[nr++] = Run{(int32_t)p[c], 1, (int32_t)t, 0};
        ++t;
        ++p[c];
        break;
      }
      const uint32_t call = V[p[c]];
      if (a.node_j0[call] < a.seg_off[a.cseg[call] + 1]) {  // blocked drain
        const uint64_t k2 = a.bkeys[q[c]];  // q[c]: this null call's index in `nulls`
        thr[c] = k2 < thr[c] ? k2 : thr[c];
      }
      ++p[c];  // the call itself is spent (its oversize requests are rejected)
      ++q[c];
    }
  }
  if (fl) latch_flags(a.sum, fl);
  a.dmisc[kEmitted] = t;
  a.dmisc[kRuns] = nr;
  int unr = 0;
  for (int c = 0; c < C; ++c) {
    const int64_t u = p[c];  // calls from here on are never reached
    a.dmisc[kUBeg + c] = u;
    a.dmisc[kCEnd + c] = s_cb[c + 1];
    if (u < s_cb[c + 1]) unr = 1;
  }
  a.dmisc[kZBeg] = s_cb[C];
  if (s_cb[C] < M) unr = 1;
  a.dmisc[kUnr] = unr;
  a.sum->n_dispatched = t;
}

// emit_order / batch_emit from the runs, over dispatch ranks [t0, T) step dt
__device__ void emit(const DispArgs& a, const uint32_t* V, int64_t t0, int64_t dt) {
  const Run* runs = reinterpret_cast<const Run*>(a.runs);
  const int64_t T = a.dmisc[kEmitted];
  const int nr = (int)a.dmisc[kRuns];
  for (int64_t t = t0; t < T; t += dt) {
    int lo = 0, hi = nr;  // last run with runs[r].t <= t
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (runs[mid].t <= t) lo = mid; else hi = mid;
    }
    const int64_t pos = runs[lo].start + (t - runs[lo].t);
    const int32_t b = a.node_batch[V[pos]];
    if (b >= 0 && b < a.batches_cap) {
      a.emit_order[t] = b;
      a.batch_emit[b] = (int32_t)t;
    }
  }
}

// requests of calls the loop never reaches -> PENDING (warps w0, w0+dw, ...)
__device__ void unreached(const DispArgs& a, const uint32_t* V, int M, int64_t w0, int64_t dw) {
  if (!a.dmisc[kUnr]) return;
  const int C = a.C;
  int64_t beg[BS_MAX_CLASSES + 1], len[BS_MAX_CLASSES + 1];
  int64_t tot = 0;
  for (int c = 0; c < C; ++c) {
    beg[c] = a.dmisc[kUBeg + c];
    len[c] = max((int64_t)0, a.dmisc[kCEnd + c] - beg[c]);
    tot += len[c];
  }
  beg[C] = a.dmisc[kZBeg];
  len[C] = M - beg[C];
  tot += len[C];
  const int lane = threadIdx.x & 31;
  int64_t to_pend = 0, from_rej = 0;
  for (int64_t x = w0; x < tot; x += dw) {
    int64_t r = x;
    int k = 0;
    while (r >= len[k]) { r -= len[k]; ++k; }
    const uint32_t call = V[beg[k] + r];
    const int32_t s = a.cseg[call];
    const int32_t b = a.node_batch[call];
    const int64_t s0 = a.list[call];
    const int64_t e0 = (b >= 0 && b < a.batches_cap) ? (int64_t)a.batches[b].end
                                                     : (int64_t)a.seg_off[s + 1];
    for (int64_t j = s0 + lane; j < e0; j += 32) {
      const int32_t q = a.perm[j];
      const int32_t old = a.req_batch[q];
      if (old != BS_REQ_PENDING) {
        a.req_batch[q] = BS_REQ_PENDING;
        a.req_row[q] = -1;
        ++to_pend;
        if (old == BS_REQ_REJECTED) ++from_rej;
      }
    }
  }
  to_pend = warp_sum(to_pend);
  from_rej = warp_sum(from_rej);
  if (lane == 0 && to_pend) {
    add_i64(&a.sum->n_pending, to_pend);
    add_i64(&a.sum->n_rejected, -from_rej);
  }
}

}  // namespace

__global__ void __launch_bounds__(kKT, 1) k_dispatch(DispArgs a) {
  pdl_prologue();
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* sk0 = reinterpret_cast<uint64_t*>(smem + kOffK0);
  uint64_t* sk1 = reinterpret_cast<uint64_t*>(smem + kOffK1);
  uint32_t* sv0 = reinterpret_cast<uint32_t*>(smem + kOffV0);
  uint32_t* sv1 = reinterpret_cast<uint32_t*>(smem + kOffV1);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(smem + kOffCnt);
  uint32_t* s_bin = reinterpret_cast<uint32_t*>(smem + kOffBin);
  uint32_t* s_dst = reinterpret_cast<uint32_t*>(smem + kOffDst);
  int64_t* s_gb = reinterpret_cast<int64_t*>(smem + kOffGb);
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_sc[33];

  const int M = a.misc[64];
  const int nb = min(a.misc[66], a.batches_cap);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  unsigned fl = 0;

  if (M <= kSmallCap) {
    // ================= one CTA, everything in shared memory ==========================
    if (blockIdx.x != 0) return;
    for (int b = tid; b < nb; b += kKT) a.batch_emit[b] = -1;
    uint64_t* K = reinterpret_cast<uint64_t*>(smem + kOffK0);  // [kSmallCap], in place
    uint32_t* V = reinterpret_cast<uint32_t*>(smem + kOffV0);
    scan_calls(a, M, 0, M, seg_id(), K, V, fl);
    // bitonic sort of (key, call) pairs: (key, call) is unique, so the order is the
    // stable order by key; pad to a power of two with keys that sort last
    int P = 64;
    while (P < M) P <<= 1;
    for (int i = M + tid; i < P; i += kKT) { K[i] = kUnreach; V[i] = 0xffffffffu; }
    __syncthreads();
    if (P <= 2048) block_bitonic<2>(K, V, P);
    else if (P == 4096) block_bitonic<4>(K, V, P);
    else block_bitonic<8>(K, V, P);
    uint64_t* kin = K;
    uint32_t* vin = V;
    walk(a, kin, vin, M);
    __syncthreads();
    emit(a, vin, tid, kKT);
    __syncthreads();
    unreached(a, vin, M, w, kKW);
    latch_flags(a.sum, fl);
    return;
  }

  // ================= every CTA, grid barriers between phases ===========================
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x;
  const int64_t gt = (int64_t)blockIdx.x * kKT + tid;
  const int64_t gs = (int64_t)G * kKT;
  for (int64_t b = gt; b < nb; b += gs) a.batch_emit[b] = -1;
  // ---- keys: chunked reverse segmented scan (aggregates, then carries) ----------------
  const int chunk = (M + G - 1) / G;
  const int u0 = min(M, (int)blockIdx.x * chunk), u1 = min(M, u0 + chunk);
  const SegVal agg = scan_calls(a, M, u0, u1, seg_id(), nullptr, nullptr, fl);
  if (tid == 0) a.agg[blockIdx.x] = agg;
  // look-back words and tile counters of the 8 passes (only the tiles this window uses)
  const int tiles = (M + kSmall - 1) / kSmall;
  const int64_t need = (int64_t)tiles * 256;
  for (int64_t i = gt; i < 8 * need; i += gs) a.status[(i / need) * a.stat_words + (i % need)] = 0;
  if (gt < 8) a.tctr[gt] = 0;
  grid.sync();
  {
    SegVal carry = seg_id();
    for (int b = 0; b < (int)blockIdx.x; ++b) carry = seg_combine(carry, a.agg[b]);
    scan_calls(a, M, u0, u1, carry, a.keys0, a.vals0, fl);
  }
  grid.sync();
  // ---- key-byte histograms ------------------------------------------------------------
  for (int i = tid; i < 8 * 256; i += kKT) s_cnt[i] = 0;
  __syncthreads();
  for (int64_t i = gt; i < M; i += gs) {
    const uint64_t k = a.keys0[i];
#pragma unroll
    for (int d = 0; d < 8; ++d) atomicAdd(&s_cnt[d * 256 + ((k >> (8 * d)) & 255u)], 1u);
  }
  __syncthreads();
  for (int i = tid; i < 8 * 256; i += kKT)
    if (s_cnt[i]) atomicAdd(a.hist8 + i, s_cnt[i]);
  grid.sync();
  // ---- plan: active bytes and bin offsets (every CTA, redundantly) ----------------------
  int nact = 0;
  int act[8];
  for (int d = 0; d < 8; ++d) {
    const uint32_t v = tid < 256 ? __ldcg(a.hist8 + d * 256 + tid) : 0u;
    const int varies = __syncthreads_or(v != 0 && v != (uint32_t)M);
    uint32_t tot;
    const uint32_t off = block_excl_scan<uint32_t>(v, s_sc, &tot);
    if (varies) {
      if (tid < 256) s_bin[nact * 256 + tid] = off;
      act[nact++] = d;
    }
  }
  __syncthreads();
  // ---- onesweep passes ---------------------------------------------------------------------
  for (int q = 0; q < nact; ++q) {
    const int shift = 8 * act[q];
    const uint64_t* kin = (q & 1) ? a.keys1 : a.keys0;
    const uint32_t* vin = (q & 1) ? a.vals1 : a.vals0;
    uint64_t* kout = (q & 1) ? a.keys0 : a.keys1;
    uint32_t* vout = (q & 1) ? a.vals0 : a.vals1;
    uint32_t* st = a.status + (int64_t)q * a.stat_words;
    for (;;) {
      if (tid == 0) s_tile = atomicAdd(a.tctr + q, 1u);
      __syncthreads();
      const int tile = (int)s_tile;
      __syncthreads();
      if (tile >= tiles) break;
      const int tbase = tile * kSmall;
      uint64_t key[kKItems];
      uint32_t val[kKItems], rank[kKItems], tc = 0;
#pragma unroll
      for (int k = 0; k < kKItems; ++k) {
        const int e = tbase + w * 32 * kKItems + k * 32 + lane;
        key[k] = e < M ? kin[e] : kUnreach;
        val[k] = e < M ? vin[e] : 0u;
      }
      tile_rank(key, tbase, M, shift, s_cnt, s_dst, rank, &tc);
      if (tid < 256) {  // decoupled look-back for digit tid
        uint32_t excl = 0;
        uint32_t* my = st + (int64_t)tile * 256 + tid;
        if (tile == 0) {
          st_relaxed(my, kStatPrefix | tc);
        } else {
          st_relaxed(my, kStatAgg | tc);
          int64_t t = (int64_t)tile - 1;
          for (;;) {
            uint32_t v;
            do { v = ld_relaxed(st + t * 256 + tid); } while ((v >> 30) == 0);
            excl += v & kStatMask;
            if (v & kStatPrefix) break;
            --t;
          }
          st_relaxed(my, kStatPrefix | (excl + tc));
        }
        s_gb[tid] = (int64_t)s_bin[q * 256 + tid] + excl - s_dst[tid];
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kKItems; ++k) {  // local sort (staged in sk0 / sv0)
        const int e = tbase + w * 32 * kKItems + k * 32 + lane;
        if (e < M) {
          const uint32_t dg = (uint32_t)((key[k] >> shift) & 255u);
          const uint32_t lp = s_dst[dg] + s_cnt[w * 256 + dg] + rank[k];
          sk0[lp] = key[k];
          sv0[lp] = val[k];
        }
      }
      __syncthreads();
      const int tn = min(kSmall, M - tbase);
      for (int i = tid; i < tn; i += kKT) {  // contiguous digit runs
        const uint64_t kk = sk0[i];
        const int64_t g = s_gb[(kk >> shift) & 255u] + i;
        kout[g] = kk;
        vout[g] = sv0[i];
      }
      __syncthreads();
    }
    grid.sync();
  }
  const uint64_t* K = (nact & 1) ? a.keys1 : a.keys0;
  const uint32_t* V = (nact & 1) ? a.vals1 : a.vals0;
  if (blockIdx.x == 0) {
    for (int i = tid; i < 8 * 256; i += kKT) a.hist8[i] = 0;  // every CTA has read it
    walk(a, K, V, M);
  }
  grid.sync();
  emit(a, V, gt, gs);
  unreached(a, V, M, gt >> 5, gs >> 5);
  latch_flags(a.sum, fl);
}

int dispatch_smem_bytes() { return kSmem; }
int dispatch_threads() { return kKT; }

cudaError_t launch_dispatch(bs_ctx* ctx, const int32_t* perm, const int32_t* seg_off, int64_t n,
                            const bs_window_params& p, const bs_batch* batches,
                            int32_t batches_cap, int32_t* req_batch, int32_t* req_row,
                            int32_t* emit_order, int32_t* batch_emit, bs_summary* summary,
                            cudaStream_t st) {
  const int64_t H = p.current_safe - p.pledged;
  if (n == 0 || H <= 0) return cudaSuccess;  // no call admits anything: nothing dispatched
  if (!p.dispatch) return cudaErrorInvalidValue;  // K5 must have filled the call accumulators
  DispArgs a;
  a.list = ctx->listA;
  a.node_batch = ctx->node_batch;
  a.node_j0 = ctx->node_j0;
  a.misc = ctx->misc;
  a.seg_off = seg_off;
  a.batches = batches;
  a.batches_cap = batches_cap;
  a.C = p.n_classes;
  a.perm = perm;
  a.slen = ctx->sorted_len;
  a.cseg = ctx->disp_cseg;
  a.cmin = ctx->disp_cmin;
  a.csum = ctx->disp_csum;
  a.keys0 = ctx->disp_keys0;
  a.keys1 = ctx->disp_keys1;
  a.vals0 = ctx->disp_vals0;
  a.vals1 = ctx->disp_vals1;
  a.hist8 = ctx->disp_hist8;
  a.status = ctx->disp_status;
  a.stat_words = (ctx->max_n + kSmall - 1) / kSmall * 256 + 256;
  a.tctr = ctx->disp_tctr;
  a.nulls = ctx->disp_nulls;
  a.bkeys = ctx->disp_bkeys;
  a.runs = ctx->disp_runs;
  a.dmisc = ctx->disp_misc;
  a.agg = reinterpret_cast<SegVal*>(ctx->disp_agg);
  a.emit_order = emit_order;
  a.batch_emit = batch_emit;
  a.req_batch = req_batch;
  a.req_row = req_row;
  a.sum = summary;
  cudaError_t e = launch_k(ctx, k_dispatch, dim3(ctx->disp_blocks), dim3(kKT), kSmem, st, true, a);
  ++ctx->launches;
  return e;
}

}  // namespace bsk

void* bs_dispatch_kernel_ptr() { return reinterpret_cast<void*>(&bsk::k_dispatch); }
