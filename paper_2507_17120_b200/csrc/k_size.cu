// K5 — memory-safe batch sizing: BatchController.form_batch drained per segment.
//
// Reference (batch_controller.py:141-191), per (bucket, class) segment in drain
// order, repeated until it returns None:
//   headroom = current_safe - pledged; headroom <= 0 -> None, nothing touched
//   a request with kvpt*len > current_safe is rejected (OversizeRejection) and
//   skipped; the batch is the longest prefix whose _footprint (PADDED:
//   kvpt*max*n, EXACT: kvpt*sum, :136-139) stays <= headroom; the drain of the
//   segment stops at the first call that admits nothing.
// In token space (kvpt*x > H <=> x > floor(H/kvpt)) with T = floor(headroom/kvpt)
// and S = floor(current_safe/kvpt) this is a greedy segmentation: drop len > S,
// cut where max*(n+1) > T (PADDED) or sum+len > T (EXACT).
//
// B200 design (no sequential walk over requests; positions = drain order):
//   K5a  prep      gather lengths into drain order + per-32-position ("group")
//                  summaries of the admissible lengths: bitmask, count, sum, max, min
//   K5b  next      next(j) = where a form_batch call starting at j stops, for
//                  EVERY j.  One warp owns the 32 starts of a group: in-group
//                  suffix stats by shuffles, then a warp-cooperative gallop over
//                  32 group summaries per step (shuffle scans + per-lane binary
//                  search), then <= 32 element steps per lane.  Work per start is
//                  O(1 + span/1024) warp steps instead of O(span/32) serial loads.
//   K5c  chain     the chain next(next(...)) of every segment = its form_batch calls:
//                  one thread per segment walks up to kWalk calls (C2's longest chain is
//                  75), one CTA per longer segment doubles pointers over its positions
//                  only, then node / batch bases and every chain node in emission order
//                  (four plain kernels, no grid barrier, no cooperative launch)
//   K5d  describe  one warp per batch: n / sum / max / min from group summaries
//   K5f  offsets   one CTA: packed-buffer offsets (scan of n*pitch), row bases, totals
//   K5e  outcome   one warp per 32 positions: batch id / row / rejected / pending,
//                  and the row map (window row -> drain position) used by K6
#include <cooperative_groups.h>

#include "ctx.cuh"

namespace cg = cooperative_groups;

namespace bsk {

struct SizeArgs {
  int64_t n;
  int64_t T;      // floor(headroom / kvpt)
  int64_t S;      // floor(current_safe / kvpt)
  int64_t kvpt;
  int32_t padded;
  int32_t L;
  int32_t truncate;
  int32_t C;         // classes (segment s holds class s % C)
  int32_t sjf_mask;  // bit c: class c drains SJF (lengths ascending in its segments)
  int32_t ljf_mask;  // bit c: class c drains LJF (lengths descending)
  int32_t walk;      // K5c: chain calls followed serially before doubling is considered
  int32_t walk_forced;  // (tuning / test hook) hand every longer chain to doubling
  int32_t pairs;        // K5c walk reads J1 = J0 o J0 too (k_chain_pairs)
};

struct Stat {
  int64_t m, c, s;  // max, count, sum of the admitted lengths so far
};

__device__ __forceinline__ bool violates(const SizeArgs& a, int64_t m, int64_t c, int64_t s) {
  return a.padded ? (m * c > a.T) : (s > a.T);
}

__device__ __forceinline__ int64_t seg_of(const int32_t* __restrict__ seg_off, int32_t n_segs,
                                          int64_t j) {
  // largest s with seg_off[s] <= j  (upper_bound - 1 over seg_off[0..n_segs])
  int32_t lo = 0, hi = n_segs;
  while (hi - lo > 1) {
    const int32_t mid = (lo + hi) >> 1;
    if (seg_off[mid] <= j) lo = mid; else hi = mid;
  }
  return lo;
}

// first admissible (non-rejected) position in [j, end), or end
__device__ __forceinline__ int64_t first_nonrej(int64_t j, int64_t end,
                                                const uint32_t* __restrict__ bmask) {
  int64_t k = j;
  while (k < end) {
    const uint32_t m = bmask[k >> 5] & (0xffffffffu << (k & 31));
    if (m) {
      const int64_t p = (k & ~31LL) + (__ffs(m) - 1);
      return p < end ? p : end;
    }
    k = (k & ~31LL) + 32;
  }
  return end;
}

// admit elements from k while the batch stays feasible; first violating position or end
__device__ __forceinline__ int64_t extend_elems(int64_t k, int64_t end, Stat& st,
                                                const SizeArgs& a,
                                                const int32_t* __restrict__ slen) {
  for (; k < end; ++k) {
    const int64_t x = slen[k];
    if (x <= a.S) {
      const int64_t nm = x > st.m ? x : st.m;
      if (violates(a, nm, st.c + 1, st.s + x)) return k;
      st.m = nm; ++st.c; st.s += x;
    }
  }
  return end;
}

// per-lane greedy with a serial gallop over group summaries (rare paths only)
__device__ int64_t greedy_serial(int64_t j0, int64_t end, const SizeArgs& a,
                                 const int32_t* __restrict__ slen,
                                 const int32_t* __restrict__ bmax,
                                 const int32_t* __restrict__ bcnt,
                                 const int32_t* __restrict__ bsum) {
  Stat st{slen[j0], 1, slen[j0]};
  int64_t k = j0 + 1;
  const int64_t a32 = (k + 31) & ~31LL;
  const int64_t lim = a32 < end ? a32 : end;
  k = extend_elems(k, lim, st, a, slen);
  if (k < lim) return k;  // violated before alignment
  while (k + 32 <= end) {
    const int g = (int)(k >> 5);
    const int64_t bc = bcnt[g];
    if (bc) {
      const int64_t bm = bmax[g];
      const int64_t nm = bm > st.m ? bm : st.m;
      if (violates(a, nm, st.c + bc, st.s + bsum[g])) break;
      st.m = nm; st.c += bc; st.s += bsum[g];
    }
    k += 32;
  }
  return extend_elems(k, end, st, a, slen);
}

// ---------------------------------------------------------------------------- K5a
__global__ void __launch_bounds__(256)
    k_size_prep(const int32_t* __restrict__ len, const int32_t* __restrict__ perm, SizeArgs a,
                int32_t* __restrict__ slen, uint32_t* __restrict__ bmask,
                int32_t* __restrict__ bmax, int32_t* __restrict__ bmin,
                int32_t* __restrict__ bcnt, int32_t* __restrict__ bsum,
                const uint32_t* __restrict__ skeys, const int32_t* __restrict__ slot_len) {
  pdl_prologue();
  const int lane = threadIdx.x & 31;
  const int64_t groups = (a.n + 31) >> 5;
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned fl = 0;
  for (int64_t g = wg; g < groups; g += wstride) {
    const int64_t j = (g << 5) + lane;
    const bool valid = j < a.n;
    int32_t x = 0;
    if (valid) {
      // SJF / LJF positions: the length is the sorted slot's (no random gather); FCFS
      // positions gather it through perm
      x = skeys ? slot_len[skeys[j]] : -1;
      if (x < 0) x = eff_len(len[perm[j]], a.L, a.truncate, fl);
      slen[j] = x;
    }
    const bool nr = valid && (int64_t)x <= a.S;
    const uint32_t m = __ballot_sync(0xffffffffu, nr);
    const int32_t mx = warp_max(nr ? x : 0);
    const int32_t mn = -warp_max(nr ? -x : -INT32_MAX);
    const int32_t s = warp_sum(nr ? x : 0);
    if (lane == 0) {
      bmask[g] = m; bcnt[g] = __popc(m); bmax[g] = mx; bmin[g] = mn; bsum[g] = s;
    }
  }
}

// ---------------------------------------------------------------------------- K5b
__global__ void __launch_bounds__(256)
    k_size_next(SizeArgs a, const int32_t* __restrict__ kinfo, const int32_t* __restrict__ seg_off,
                const int32_t* __restrict__ slen, const uint32_t* __restrict__ bmask,
                const int32_t* __restrict__ bmax, const int32_t* __restrict__ bcnt,
                const int32_t* __restrict__ bsum, int32_t* __restrict__ J0,
                uint8_t* __restrict__ is_start, int32_t* __restrict__ alive,
                const uint32_t* __restrict__ skeys, const int32_t* __restrict__ slot_seg) {
  pdl_prologue();
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int32_t n_segs = kinfo[2];
  const int64_t G = (a.n + 31) >> 5;
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t g = wg; g < G; g += wstride) {
    const int64_t j = (g << 5) + lane;
    const bool valid = j < a.n;
    const uint32_t nrm = bmask[g];
    const int32_t x = valid ? slen[j] : 0;
    int64_t e = 0;
    int64_t seg_c = 0;
    bool start = false;
    {  // segment of j: one lookup per warp, then a short walk per lane
      int64_t s0 = 0;
      // the sorted radix slot names the segment (K2 slot_seg LUT); binary search otherwise
      if (lane == 0) s0 = skeys ? slot_seg[skeys[g << 5]] : seg_of(seg_off, n_segs, g << 5);
      int64_t s = __shfl_sync(FULL, s0, 0);
      if (valid) {
        while (seg_off[s + 1] <= j) ++s;
        e = seg_off[s + 1];
        start = seg_off[s] == j;
      }
      seg_c = s;
    }
    // PADDED drains of length-sorted segments have closed forms (no gallop):
    //   SJF: lengths ascend, rejected (> S) form the tail: next(j) = first k > j with
    //        slen[k] > S or slen[k] * (k - j + 1) > T (both monotone: exponential +
    //        binary search);
    //   LJF: lengths descend, rejected form the head: the call starts at the first
    //        admissible j0 and admits floor(T / slen[j0]) requests.
    int fast = 0;
    int32_t fast_nx = kEnd;
    // whole warp inside one SJF segment, every start admissible (x <= min(S, T)): with
    // A(k) = k - floor(T / slen[k]) (+inf for an oversize k), strictly increasing along
    // the segment, a call from j stops at the first k with A(k) >= j (slen[k] (k - j + 1)
    // > T  <=>  j <= A(k)).  So next(j0) by one warp-cooperative 32-ary search, and the 32
    // starts' stops all lie in the 32 positions from there: one load + a shuffle search
    // per lane instead of an exponential + binary search per lane
    const int64_t seg_l0 = __shfl_sync(FULL, seg_c, 0);
    const bool sjf_lane = valid && a.padded && seg_c == seg_l0 &&
                          ((a.sjf_mask >> (int)(seg_c % a.C)) & 1) && (int64_t)x <= a.S &&
                          (int64_t)x <= a.T;
    if (__all_sync(FULL, sjf_lane)) {
      const int64_t j0 = g << 5;
      int64_t lo = j0 + 1, hi = e;  // first k in [lo, e) bad for j0 (hi: e or a bad k)
      while (lo < hi) {
        const int64_t step = (hi - lo + 31) >> 5;
        const int64_t q = lo + lane * step;
        bool bd = false;
        if (q < hi) {
          const int64_t y = slen[q];
          bd = y > a.S || y * (q - j0 + 1) > a.T;
        }
        const unsigned bm = __ballot_sync(FULL, bd);
        if (bm) {
          const int f = __ffs(bm) - 1;
          hi = lo + f * step;
          lo = f ? lo + (f - 1) * step + 1 : lo;
        } else {
          const int64_t span_q = (hi - 1 - lo) / step;
          const int64_t last = span_q < 31 ? span_q : 31;
          lo = lo + last * step + 1;
        }
      }
      const int64_t k0 = lo;
      const int64_t kk = k0 + lane;
      int64_t A = INT64_MAX;  // past the segment or oversize: every start stops there
      if (kk < e) {
        const int64_t y = slen[kk];
        if (y <= a.S) A = y > 0 ? kk - a.T / y : INT64_MIN;
      }
      int lo2 = 0, hi2 = 32;  // first lane i with A_i >= j
#pragma unroll
      for (int it = 0; it < 6; ++it) {
        const int mid = (lo2 + hi2) >> 1;
        const int64_t am = __shfl_sync(FULL, A, mid < 31 ? mid : 31);
        if (lo2 < hi2) {
          if (am >= j) hi2 = mid; else lo2 = mid + 1;
        }
      }
      const int64_t a_idx = __shfl_sync(FULL, A, lo2 < 31 ? lo2 : 31);
      fast = 1;
      fast_nx = (lo2 < 32 && a_idx != INT64_MAX) ? (int32_t)(k0 + lo2) : kEnd;
    } else if (valid && a.padded) {
      const int c = (int)(seg_c % a.C);
      if ((a.sjf_mask >> c) & 1) {
        fast = 1;
        if ((int64_t)x <= a.S && (int64_t)x <= a.T) {
          auto bad = [&](int64_t k) {
            const int64_t y = slen[k];
            return y > a.S || y * (k - j + 1) > a.T;
          };
          int64_t lo = j + 1, hi = e, step = 1;
          for (;;) {  // exponential search: [j+1, lo) are admitted
            const int64_t q = lo + step - 1;
            if (q >= e) break;
            if (bad(q)) { hi = q; break; }
            lo = q + 1;
            step <<= 1;
          }
          while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (bad(mid)) hi = mid; else lo = mid + 1;
          }
          // lo: first violation, or the rejected tail (consumed by this call), or e
          fast_nx = (lo < e && (int64_t)slen[lo] <= a.S) ? (int32_t)lo : kEnd;
        }
      } else if ((a.ljf_mask >> c) & 1) {
        fast = 1;
        const int64_t j0 = first_nonrej(j, e, bmask);
        if (j0 < e) {
          const int64_t x0 = slen[j0];
          if (x0 <= a.T) {
            const int64_t k = j0 + a.T / x0;
            fast_nx = k < e ? (int32_t)k : kEnd;
          }
        }
      }
    }
    const int64_t gend = ((g << 5) + 32) < a.n ? ((g << 5) + 32) : a.n;
    const bool nr = valid && ((nrm >> lane) & 1u);
    // suffix max / sum of the admissible lengths at lanes >= lane
    // (sums of <= 32 lengths < 2^22 and of <= 32 group sums < 2^27 fit int32)
    int32_t vm = nr ? x : 0;
    int32_t vs = nr ? x : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t tm = __shfl_down_sync(FULL, vm, o);
      const int32_t ts = __shfl_down_sync(FULL, vs, o);
      if (lane + o < 32) { vm = tm > vm ? tm : vm; vs += ts; }
    }
    const uint32_t rem = nrm & (FULL << lane);
    int mode = 0;  // 0 done, 1 gallop, 2 serial fallback, 3 element scan from p
    int32_t nx = kEnd;
    Stat st{0, 0, 0};
    int64_t p = 0;
    if (fast) {
      nx = fast_nx;  // mode 0: done
    } else if (valid) {
      if (e <= gend || rem == 0) {
        mode = 2;
      } else {
        const int64_t f = (g << 5) + (__ffs(rem) - 1);
        const int64_t xf = slen[f];
        if (xf > a.T) {
          mode = 0;  // blocked: form_batch admits nothing, the drain stops here
        } else if (violates(a, vm, __popc(rem), vs)) {
          mode = 3; p = f + 1; st = Stat{xf, 1, xf};
        } else {
          mode = 1; st = Stat{vm, __popc(rem), vs};
        }
      }
    }
    // warp-cooperative gallop over 32 group summaries per step
    int64_t base = g + 1;
    while (__any_sync(FULL, mode == 1)) {
      const int64_t gi = base + lane;
      int32_t pc = 0, pm = 0, ps = 0;
      if (gi < G) { pc = bcnt[gi]; pm = bmax[gi]; ps = bsum[gi]; }
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t tc = __shfl_up_sync(FULL, pc, o);
        const int32_t tm = __shfl_up_sync(FULL, pm, o);
        const int32_t ts = __shfl_up_sync(FULL, ps, o);
        if (lane >= o) { pc += tc; pm = tm > pm ? tm : pm; ps += ts; }
      }
      int ng = 0;
      if (mode == 1) {
        const int64_t lim = e / 32 - base;  // full groups of this segment from `base`
        ng = lim < 0 ? 0 : (lim > 32 ? 32 : (int)lim);
      }
      int lo = 0, hi = ng;
#pragma unroll
      for (int it = 0; it < 6; ++it) {
        const int mid = (lo + hi) >> 1;
        const int src = mid < 31 ? mid : 31;
        const int32_t qc = __shfl_sync(FULL, pc, src);
        const int32_t qm = __shfl_sync(FULL, pm, src);
        const int32_t qs = __shfl_sync(FULL, ps, src);
        if (lo < hi) {
          const int64_t nm = qm > st.m ? qm : st.m;
          if (violates(a, nm, st.c + qc, st.s + qs)) hi = mid; else lo = mid + 1;
        }
      }
      const int src2 = lo - 1 < 0 ? 0 : (lo - 1 > 31 ? 31 : lo - 1);
      const int32_t bc = __shfl_sync(FULL, pc, src2);
      const int32_t bm = __shfl_sync(FULL, pm, src2);
      const int32_t bs = __shfl_sync(FULL, ps, src2);
      if (mode == 1) {
        if (lo > 0) { st.m = bm > st.m ? bm : st.m; st.c += bc; st.s += bs; }
        if (lo < ng) { mode = 4; p = (base + lo) << 5; }        // violation inside that group
        else if (ng < 32) { mode = 4; p = (base + ng) << 5; }   // segment tail (< 32 elements)
      }
      base += 32;
    }
    // warp-cooperative resolution inside the target group: the warp loads the group
    // once, builds inclusive prefixes by shuffles, and every lane aiming at that group
    // binary-searches its first violating element (first violation is admissible:
    // an inadmissible element leaves the prefix unchanged)
    unsigned pend = __ballot_sync(FULL, mode == 4);
    while (pend) {
      const int leader = __ffs(pend) - 1;
      const int64_t tp = __shfl_sync(FULL, p, leader);
      const int64_t te = __shfl_sync(FULL, e, leader);
      const int lim = (te - tp) < 32 ? (int)(te - tp) : 32;
      const int32_t xx = lane < lim ? slen[tp + lane] : 0;
      const bool ad = lane < lim && (int64_t)xx <= a.S;
      int32_t qc = ad ? 1 : 0, qm = ad ? xx : 0, qs = ad ? xx : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t tc = __shfl_up_sync(FULL, qc, o);
        const int32_t tm = __shfl_up_sync(FULL, qm, o);
        const int32_t ts = __shfl_up_sync(FULL, qs, o);
        if (lane >= o) { qc += tc; qm = tm > qm ? tm : qm; qs += ts; }
      }
      const bool serve = mode == 4 && p == tp && e == te;
      int lo = 0, hi = lim;
#pragma unroll
      for (int it = 0; it < 6; ++it) {
        const int mid = (lo + hi) >> 1;
        const int src = mid < 31 ? mid : 31;
        const int32_t c_ = __shfl_sync(FULL, qc, src);
        const int32_t m_ = __shfl_sync(FULL, qm, src);
        const int32_t s_ = __shfl_sync(FULL, qs, src);
        if (serve && lo < hi) {
          const int64_t nm = m_ > st.m ? m_ : st.m;
          if (violates(a, nm, st.c + c_, st.s + s_)) hi = mid; else lo = mid + 1;
        }
      }
      const int32_t c31 = __shfl_sync(FULL, qc, 31);
      const int32_t m31 = __shfl_sync(FULL, qm, 31);
      const int32_t s31 = __shfl_sync(FULL, qs, 31);
      if (serve) {
        if (lo < lim) {
          nx = (int32_t)(tp + lo);
          mode = 0;
        } else if (tp + lim >= e) {
          nx = kEnd;  // reached the segment end
          mode = 0;
        } else {      // (not expected) no violation in a full group: continue serially
          st.m = m31 > st.m ? m31 : st.m; st.c += c31; st.s += s31;
          mode = 3;
          p = tp + 32;
        }
      }
      pend &= ~__ballot_sync(FULL, serve);
    }
    if (mode == 3) {
      const int64_t k = extend_elems(p, e, st, a, slen);
      nx = k < e ? (int32_t)k : kEnd;
    } else if (mode == 2) {
      const int64_t j0 = first_nonrej(j, e, bmask);
      if (j0 < e && (int64_t)slen[j0] <= a.T) {
        const int64_t k = greedy_serial(j0, e, a, slen, bmax, bcnt, bsum);
        nx = k < e ? (int32_t)k : kEnd;
      }
    }
    if (valid) {
      J0[j] = nx;
      is_start[j] = start;
      if (start && nx != kEnd) alive[0] = 1;
    }
  }
}

// ---------------------------------------------------------------------------- K5c
// The chain of every segment, next(next(...)) from its start, is the sequence of its
// form_batch calls.  Plain (non-cooperative) kernels, so no launch waits for a whole
// GPU to be free beside the pack of another window in flight:
//   pairs  J1 = J0 o J0 over every position (level 1 of the doubling table)
//   walk   one thread per segment follows its chain for up to `walk` calls, two per round
//          trip (J0[pos] and J1[pos] are independent loads; C2's longest chain is 75
//          calls) into listB; longer segments are listed; extra CTAs sum the admissible
//          counts of 8192-group tiles (for Rg)
//   long   one 1024-thread CTA per listed segment: pointer doubling J[r+1] = J[r][J[r]]
//          over the segment's positions only (__syncthreads per level, no grid barrier)
//          until the start's 2^r-th successor is past the segment, then binary lifting
//          for the chain length and last node
//   bases  one CTA: node / batch bases per segment, the window's totals, the tile prefix
//   nodes  every chain node (= batch start) in emission order; extra CTAs finish Rg
// K5c walk policy.  A segment's chain is followed serially (one dependent L2 hit per call,
// ~0.25 us) for kWalk calls; if it goes on, the walk estimates the remaining calls from the
// positions consumed so far and keeps walking (up to kWalkMax calls) only while that is
// cheaper than one CTA doubling pointers over the whole segment (~0.19 ns per position and
// level): C3's first bucket (576 calls of ~3k requests over 1.4M positions) is walked in
// ~0.1 ms where doubling would take ~2.4 ms, C4's long-context tail (1,591 calls of ~8
// requests over 12.7k positions) is doubled in ~30 us instead of walked in ~0.35 ms.
constexpr int kWalk = 64;
constexpr int kWalkMax = 16384;
constexpr int kRgTile = 8192;        // 32-position groups per Rg tile (256 threads x 32)

__device__ __forceinline__ int32_t ld_rel_i32(const int32_t* p) {
  return (int32_t)ld_relaxed(reinterpret_cast<const uint32_t*>(p));
}

struct SegArrays {
  int32_t *len, *empty, *tailj0, *nbase, *ebase, *lvl, *long_list;
};
__device__ __forceinline__ SegArrays seg_arrays(int32_t* segw, int32_t n_segs) {
  const int64_t w = n_segs + 1;
  return SegArrays{segw, segw + w, segw + 2 * w, segw + 3 * w, segw + 4 * w, segw + 5 * w,
                   segw + 6 * w};
}

// J1 = J0 o J0 (the second successor) over every position, so a walk can take two calls
// per dependent load pair (the loads of J0[pos] and J1[pos] are independent)
__global__ void __launch_bounds__(256) k_chain_pairs(int64_t n, const int32_t* __restrict__ J0,
                                                     int32_t* __restrict__ J1) {
  pdl_prologue();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    const int32_t y = J0[j];
    J1[j] = y == kEnd ? kEnd : J0[y];
  }
}

__global__ void __launch_bounds__(256)
    k_chain_walk(SizeArgs a, const int32_t* __restrict__ kinfo, const int32_t* __restrict__ seg_off,
                 const int32_t* __restrict__ J0, int32_t* __restrict__ listB,
                 const int32_t* __restrict__ slen, const uint32_t* __restrict__ bmask,
                 const int32_t* __restrict__ bcnt, int32_t* __restrict__ segw,
                 int32_t* __restrict__ misc, int32_t* __restrict__ tile_sum, int32_t n_tiles) {
  pdl_prologue();
  const int tid = threadIdx.x;
  if ((int)blockIdx.x < n_tiles) {  // admissible count of one Rg tile
    const int64_t G = (a.n + 31) >> 5;
    const int64_t g0 = (int64_t)blockIdx.x * kRgTile;
    const int64_t g1 = g0 + kRgTile < G ? g0 + kRgTile : G;
    int32_t loc = 0;
    for (int64_t g = g0 + tid; g < g1; g += blockDim.x) loc += bcnt[g];
    loc = warp_sum(loc);
    __shared__ int32_t s_w[8];
    if ((tid & 31) == 0) s_w[tid >> 5] = loc;
    __syncthreads();
    if (tid == 0) {
      int32_t t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_w[w];
      tile_sum[blockIdx.x] = t;
    }
    return;
  }
  const int32_t n_segs = kinfo[2];
  const SegArrays S = seg_arrays(segw, n_segs);
  const int64_t sg = (int64_t)(blockIdx.x - n_tiles) * blockDim.x + tid;
  if (sg >= n_segs) return;
  const int64_t st = seg_off[sg], en = seg_off[sg + 1];
  int32_t len = 0, empty = 0, tj0 = 0, lng = 0;
  if (st < en) {
    int64_t pos = st;
    int32_t k = 0;
    listB[st] = (int32_t)st;
    int32_t limit = a.walk;
    const int32_t* J1 = J0 + a.n;  // second successors (k_chain_pairs)
    // one call: false when the chain is handed to doubling instead
    auto step = [&](int32_t y) -> bool {
      if (++k >= limit) {
        if (a.walk_forced || k >= kWalkMax) return false;
        // remaining calls at the average call size so far vs levels x positions
        const double avg = (double)(pos - st + 1) / (double)k;
        const double rest = (double)(en - pos) / avg;
        const double walk_us = rest * 0.25;
        const double dbl_us = 10.0 + (double)(en - st) * (log2(rest + k) + 1.0) * 1.9e-4;
        if (walk_us > dbl_us) return false;
        limit = kWalkMax;
      }
      listB[st + k] = y;
      pos = y;
      return true;
    };
    for (;;) {  // two calls per round trip
      const int32_t y = J0[pos];
      const int32_t y2 = a.pairs ? J1[pos] : kEnd;
      if (y == kEnd) break;
      if (!step(y)) { lng = 1; break; }
      if (!a.pairs) continue;
      if (y2 == kEnd) break;  // J0[y] == kEnd: the chain ends at y
      if (!step(y2)) { lng = 1; break; }
    }
    if (!lng) {
      len = k + 1;
      const int64_t j0 = first_nonrej(pos, en, bmask);
      empty = !((j0 < en) && ((int64_t)slen[j0] <= a.T));
      tj0 = (int32_t)j0;
    }
  }
  S.len[sg] = len;
  S.empty[sg] = empty;
  S.tailj0[sg] = tj0;
  S.lvl[sg] = 0;
  if (lng) {
    const int32_t idx = atomicAdd(misc + 70, 1);
    if (idx <= n_segs) S.long_list[idx] = (int32_t)sg;
  }
}

__global__ void __launch_bounds__(1024, 2)
    k_chain_long(SizeArgs a, const int32_t* __restrict__ kinfo, const int32_t* __restrict__ seg_off,
                 int32_t* J, int r_cap, const int32_t* __restrict__ slen,
                 const uint32_t* __restrict__ bmask, int32_t* __restrict__ segw,
                 const int32_t* __restrict__ misc, bs_summary* sum) {
  pdl_prologue();
  const int32_t n_segs = kinfo[2];
  const SegArrays S = seg_arrays(segw, n_segs);
  const int32_t n_long = misc[70];
  const int64_t n = a.n;
  __shared__ int s_more;
  for (int32_t li = blockIdx.x; li < n_long; li += gridDim.x) {
    const int32_t sg = S.long_list[li];
    const int64_t st = seg_off[sg], en = seg_off[sg + 1];
    int r = 0;
    if (threadIdx.x == 0) s_more = 1;
    __syncthreads();
    for (;;) {  // level r + 1 over the segment's positions (successors stay inside it)
      if (r + 1 >= r_cap) break;
      const int32_t* Jr = J + (int64_t)r * n;
      int32_t* Jn = J + (int64_t)(r + 1) * n;
      constexpr int kIlp = 4;
      const int64_t span = en - st;
      for (int64_t x0 = threadIdx.x; x0 < span; x0 += kIlp * (int64_t)blockDim.x) {
        int32_t v[kIlp];
#pragma unroll
        for (int k = 0; k < kIlp; ++k) {
          const int64_t q = x0 + k * (int64_t)blockDim.x;
          v[k] = q < span ? Jr[st + q] : kEnd;
        }
#pragma unroll
        for (int k = 0; k < kIlp; ++k) v[k] = v[k] == kEnd ? kEnd : Jr[v[k]];
#pragma unroll
        for (int k = 0; k < kIlp; ++k) {
          const int64_t q = x0 + k * (int64_t)blockDim.x;
          if (q < span) Jn[st + q] = v[k];
        }
      }
      __syncthreads();
      ++r;
      if (threadIdx.x == 0) s_more = Jn[st] != kEnd;  // the chain has >= 2^r more calls
      __syncthreads();
      if (!s_more) break;
    }
    if (threadIdx.x == 0) {
      if (s_more && r + 1 >= r_cap) latch_flags(sum, BS_FLAG_BATCH_CAP);  // table exhausted
      // chain length and last node by binary lifting over the levels just built
      int64_t pos = st;
      int32_t cnt = 0;
      for (int lv = r - 1; lv >= 0; --lv) {
        const int32_t y = J[(int64_t)lv * n + pos];
        if (y != kEnd) { pos = y; cnt += 1 << lv; }
      }
      const int64_t j0 = first_nonrej(pos, en, bmask);
      S.len[sg] = cnt + 1;
      S.empty[sg] = !((j0 < en) && ((int64_t)slen[j0] <= a.T));
      S.tailj0[sg] = (int32_t)j0;
      S.lvl[sg] = r;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024)
    k_chain_bases(const int32_t* __restrict__ kinfo, int32_t* __restrict__ segw,
                  int32_t* __restrict__ misc, const int32_t* __restrict__ tile_sum,
                  int32_t* __restrict__ tile_pre, int32_t n_tiles, int32_t batches_cap,
                  bs_summary* sum) {
  pdl_prologue();
  __shared__ int32_t s_sc[3 * 33];
  const int32_t n_segs = kinfo[2];
  const SegArrays S = seg_arrays(segw, n_segs);
  const int tid = threadIdx.x;
  // contiguous runs per thread: one block scan for the node / empty-tail bases of the
  // segments and the Rg tile prefix
  const int per = (n_segs + (int)blockDim.x - 1) / (int)blockDim.x;
  const int i0 = min(n_segs, tid * per), i1 = min(n_segs, i0 + per);
  const int tper = (n_tiles + (int)blockDim.x - 1) / (int)blockDim.x;
  const int t0 = min(n_tiles, tid * tper), t1 = min(n_tiles, t0 + tper);
  int32_t v[3] = {0, 0, 0};
  for (int i = i0; i < i1; ++i) { v[0] += S.len[i]; v[1] += S.empty[i]; }
  for (int t = t0; t < t1; ++t) v[2] += tile_sum[t];
  int32_t tot[3];
  block_excl_scan_k<3, int32_t>(v, tot, s_sc);
  int32_t rn = v[0], re = v[1], rt = v[2];
  for (int i = i0; i < i1; ++i) {
    S.nbase[i] = rn;
    S.ebase[i] = re;
    rn += S.len[i];
    re += S.empty[i];
  }
  for (int t = t0; t < t1; ++t) {
    tile_pre[t] = rt;
    rt += tile_sum[t];
  }
  if (tid == 0) {
    S.nbase[n_segs] = tot[0];
    S.ebase[n_segs] = tot[1];
    const int32_t nb = tot[0] - tot[1];
    misc[64] = tot[0];
    misc[66] = nb;
    misc[68] = 0;
    sum->n_batches = nb;
    if (nb > batches_cap) latch_flags(sum, BS_FLAG_BATCH_CAP);
  }
}

__global__ void __launch_bounds__(256)
    k_chain_nodes(SizeArgs a, const int32_t* __restrict__ kinfo, const int32_t* __restrict__ seg_off,
                  const int32_t* __restrict__ J, const int32_t* __restrict__ listB,
                  int32_t* __restrict__ listA, int32_t* __restrict__ node_batch,
                  int32_t* __restrict__ node_j0, const int32_t* __restrict__ segw_c,
                  const int32_t* __restrict__ misc, const int32_t* __restrict__ bcnt,
                  const int32_t* __restrict__ tile_pre, int32_t* __restrict__ Rg, int32_t n_tiles,
                  int32_t* dseg, int32_t* dmin, int64_t* dsum) {
  pdl_prologue();
  const int tid = threadIdx.x;
  if ((int)blockIdx.x < n_tiles) {  // Rg: exclusive prefix of the admissible counts
    __shared__ int32_t s_sc[33];
    const int64_t G = (a.n + 31) >> 5;
    const int64_t g0 = (int64_t)blockIdx.x * kRgTile;
    constexpr int kPer = kRgTile / 256;
    const int64_t gb = g0 + (int64_t)tid * kPer;
    int32_t c[kPer];
    int32_t loc = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      c[k] = gb + k < G ? bcnt[gb + k] : 0;
      loc += c[k];
    }
    int32_t tot;
    int32_t run = tile_pre[blockIdx.x] + block_excl_scan<int32_t>(loc, s_sc, &tot);
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      if (gb + k < G) Rg[gb + k] = run;
      run += c[k];
    }
    return;
  }
  const int32_t n_segs = kinfo[2];
  int32_t* segw = const_cast<int32_t*>(segw_c);
  const SegArrays S = seg_arrays(segw, n_segs);
  const int32_t M = misc[64];
  const int64_t stride = (int64_t)(gridDim.x - n_tiles) * blockDim.x;
  for (int64_t i = (int64_t)(blockIdx.x - n_tiles) * blockDim.x + tid; i < M; i += stride) {
    int32_t lo = 0, hi = n_segs;  // last segment with nbase <= i (non-empty ones win ties)
    while (hi - lo > 1) {
      const int32_t mid = (lo + hi) >> 1;
      if (S.nbase[mid] <= i) lo = mid; else hi = mid;
    }
    const int32_t k = (int32_t)(i - S.nbase[lo]);
    int64_t pos = seg_off[lo];
    const int32_t lv = S.lvl[lo];
    if (lv) {  // long segment: binary lifting over its doubling levels
      for (int l = 0; l < lv; ++l)
        if ((k >> l) & 1) pos = J[(int64_t)l * a.n + pos];
    } else {
      pos = listB[pos + k];  // walked
    }
    listA[i] = (int32_t)pos;
    const bool tail_empty = (k == S.len[lo] - 1) && S.empty[lo];
    node_batch[i] = tail_empty ? -1 : (int32_t)(i - S.ebase[lo]);
    node_j0[i] = tail_empty ? S.tailj0[lo] : (int32_t)pos;
    if (dseg) {  // K7 per-call accumulators (filled by K5e)
      dseg[i] = lo;
      dmin[i] = INT32_MAX;
      dsum[i] = 0;
    }
  }
}

// ---------------------------------------------------------------------------- K5d
__global__ void __launch_bounds__(256)
    k_size_describe(SizeArgs a, const int32_t* __restrict__ kinfo,
                    const int32_t* __restrict__ seg_off, const int32_t* __restrict__ slen,
                    const int32_t* __restrict__ bmax, const int32_t* __restrict__ bmin,
                    const int32_t* __restrict__ bcnt, const int32_t* __restrict__ bsum,
                    const int32_t* __restrict__ J0, const int32_t* __restrict__ listA,
                    const int32_t* __restrict__ listB, const int32_t* __restrict__ node_batch,
                    const int32_t* __restrict__ misc, bs_batch* __restrict__ batches,
                    int32_t batches_cap, bs_summary* sum, const uint32_t* __restrict__ skeys,
                    const int32_t* __restrict__ slot_seg) {
  pdl_prologue();
  const int M = misc[64];
  const int32_t n_segs = kinfo[2];
  const int32_t* list = misc[68] ? listB : listA;
  const int lane = threadIdx.x & 31;
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned fl = 0;
  for (int64_t i = wg; i < M; i += wstride) {
    const int32_t b = node_batch[i];
    if (b < 0 || b >= batches_cap) continue;
    const int64_t c = list[i];
    const int64_t s = skeys ? slot_seg[skeys[c]] : seg_of(seg_off, n_segs, c);
    const int32_t nx = J0[c];
    const int64_t e = nx == kEnd ? (int64_t)seg_off[s + 1] : (int64_t)nx;
    int64_t cnt = 0, tsum = 0;
    int32_t mx = 0, mn = INT32_MAX;
    const int64_t ca = (c + 31) & ~31LL, eb = e & ~31LL;
    if (ca >= eb) {
      for (int64_t k = c + lane; k < e; k += 32) {
        const int32_t x = slen[k];
        if ((int64_t)x <= a.S) { ++cnt; tsum += x; mx = x > mx ? x : mx; mn = x < mn ? x : mn; }
      }
    } else {
      for (int64_t k = c + lane; k < ca; k += 32) {
        const int32_t x = slen[k];
        if ((int64_t)x <= a.S) { ++cnt; tsum += x; mx = x > mx ? x : mx; mn = x < mn ? x : mn; }
      }
      for (int64_t gg = (ca >> 5) + lane; gg < (eb >> 5); gg += 32) {
        const int32_t bc = bcnt[gg];
        if (bc) {
          cnt += bc; tsum += bsum[gg];
          mx = bmax[gg] > mx ? bmax[gg] : mx;
          mn = bmin[gg] < mn ? bmin[gg] : mn;
        }
      }
      for (int64_t k = eb + lane; k < e; k += 32) {
        const int32_t x = slen[k];
        if ((int64_t)x <= a.S) { ++cnt; tsum += x; mx = x > mx ? x : mx; mn = x < mn ? x : mn; }
      }
    }
    cnt = warp_sum(cnt);
    tsum = warp_sum(tsum);
    mx = warp_max(mx);
    mn = -warp_max(-mn);
    if (lane == 0) {
      bs_batch B;
      B.segment = (int32_t)s;
      B.start = (int32_t)c;
      B.end = (int32_t)e;
      B.n = (int32_t)cnt;
      B.max_input_len = mx;
      B.pitch = (mx + BS_PACK_ALIGN - 1) / BS_PACK_ALIGN * BS_PACK_ALIGN;
      B.token_sum = tsum;
      B.footprint = a.kvpt * (a.padded ? (int64_t)mx * cnt : tsum);
      B.out_offset = 0;
      // waste_ratio (memory_model.py:98-100): (s_max - s_avg) / s_max, float64
      const double s_avg = __ddiv_rn((double)tsum, (double)cnt);
      double wr = __ddiv_rn(__dsub_rn((double)mx, s_avg), (double)mx);
      if (mn < 1) {  // waste_ratio raises ValueError for lengths < 1 (memory_model.py:96-97)
        wr = __longlong_as_double(0x7ff8000000000000ll);
        fl |= BS_FLAG_NONPOS_LEN;
      }
      B.waste = wr;
      B.row_base = 0;  // K5f
      batches[b] = B;
    }
  }
  if (lane == 0) latch_flags(sum, fl);
}

// ---------------------------------------------------------------------------- K5e
__global__ void __launch_bounds__(256)
    k_size_outcome(SizeArgs a, const int32_t* __restrict__ perm, const uint32_t* __restrict__ bmask,
                   const int32_t* __restrict__ Rg, const int32_t* __restrict__ listA,
                   const int32_t* __restrict__ listB, const int32_t* __restrict__ node_batch,
                   const int32_t* __restrict__ node_j0, const int32_t* __restrict__ misc,
                   const bs_batch* __restrict__ batches, int32_t batches_cap,
                   int32_t* __restrict__ req_batch, int32_t* __restrict__ req_row,
                   int32_t* __restrict__ rowpos, bs_summary* sum,
                   const int32_t* __restrict__ slen, int32_t* __restrict__ dmin,
                   int64_t* __restrict__ dsum, int32_t r_lo, int32_t r_hi, int first,
                   const int64_t* __restrict__ tok_off, ulonglong2* __restrict__ rowdesc,
                   int32_t* __restrict__ chunk_row, int2* __restrict__ pos_out) {
  pdl_prologue();
  const int M = misc[64];
  const int32_t* list = misc[68] ? listB : listA;
  const int lane = threadIdx.x & 31;
  const int64_t G = (a.n + 31) >> 5;
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t rej = 0, pend = 0;
  for (int64_t g = wg; g < G; g += wstride) {
    const int64_t j = (g << 5) + lane;
    // chain node covering j: last node position <= j (nodes ascend and every segment
    // start is a node, so the node lies in j's segment); one 32-ary search per warp
    // (every lane probes one point per step: log32(M) dependent loads instead of log2)
    int lo = 0;
    {
      int hi = M;
      const int64_t target = g << 5;
      while (hi - lo > 1) {
        const int step = (hi - lo + 31) >> 5;
        const int pidx = lo + (lane + 1) * step;
        const bool le = pidx < hi && list[pidx] <= target;
        const int cnt = __popc(__ballot_sync(0xffffffffu, le));
        lo += cnt * step;
        hi = min(hi, lo + step);
      }
    }
    const bool in = j < a.n;
    if (in)
      while (lo + 1 < M && list[lo + 1] <= j) ++lo;
    if (dmin && first) {
      // K7 per-call accumulators: min arrival rank and length sum over the call's range
      // (lanes of one call are contiguous: one atomic per call and warp)
      const unsigned peers = __match_any_sync(0xffffffffu, in ? lo : -1);
      const unsigned pr = in ? (unsigned)perm[j] : 0xffffffffu;
      const unsigned ln = in ? (unsigned)slen[j] : 0u;
      const unsigned mn = __reduce_min_sync(peers, pr);
      const unsigned sm = __reduce_add_sync(peers, ln);
      if (in && lane == __ffs(peers) - 1) {
        atomicMin(dmin + lo, (int)mn);
        atomicAdd(reinterpret_cast<unsigned long long*>(dsum + lo), (unsigned long long)sm);
      }
    }
    if (!in) continue;
    const int64_t c = list[lo];
    const int32_t b = node_batch[lo];
    const uint32_t m = bmask[g];
    const bool nr = (m >> lane) & 1u;
    const int32_t r = perm[j];
    // large windows run this kernel once per request-id range, so each pass's scattered
    // outcome writes stay inside L2 and fill whole sectors (no DRAM read-modify-write);
    // the position-ordered row map and the counters are written by the first pass
    // with pos_out (large windows) the outcomes go out in drain order, sequentially, and
    // k_outcome_scatter moves them to request ids in L2-sized ranges afterwards
    const bool mine = !pos_out && r >= r_lo && r < r_hi;
    if (b >= 0) {
      if (nr) {
        const int64_t gc = c >> 5;
        const int32_t Rj = Rg[g] + __popc(m & ((1u << lane) - 1u));
        const int32_t Rc = Rg[gc] + __popc(bmask[gc] & ((1u << (c & 31)) - 1u));
        if (mine) {
          req_batch[r] = b;
          req_row[r] = Rj - Rc;
        }
        if (pos_out) pos_out[j] = make_int2(b, Rj - Rc);
        if (first && b < batches_cap) {
          const bs_batch& B = batches[b];
          const int64_t g = B.row_base + (Rj - Rc);
          rowpos[g] = (int32_t)j;  // K6 row map
          if (rowdesc) {  // the bulk-staged K6 reads one record per row (k_pack_rowprep's)
            const int64_t dst = B.out_offset + (int64_t)(Rj - Rc) * B.pitch;
            rowdesc[g] = make_ulonglong2((uint64_t)tok_off[r] | ((uint64_t)slen[j] << 40),
                                         (uint64_t)dst | ((uint64_t)B.pitch << 40));
            for (int64_t u = (dst + kPackChunk - 1) / kPackChunk; u * kPackChunk < dst + B.pitch; ++u)
              chunk_row[u] = (int32_t)g;
          }
        }
      } else {
        if (mine) {
          req_batch[r] = BS_REQ_REJECTED;
          req_row[r] = -1;
        }
        if (pos_out) pos_out[j] = make_int2(BS_REQ_REJECTED, -1);
        rej += first;
      }
    } else {  // a segment's empty tail: rejected up to the first admissible request, pending after
      const int64_t j0 = node_j0[lo];
      if (mine) {
        req_row[r] = -1;
        req_batch[r] = j < j0 ? BS_REQ_REJECTED : BS_REQ_PENDING;
      }
      if (pos_out) pos_out[j] = make_int2(j < j0 ? BS_REQ_REJECTED : BS_REQ_PENDING, -1);
      if (j < j0) rej += first; else pend += first;
    }
  }
  rej = warp_sum(rej);
  pend = warp_sum(pend);
  if (lane == 0) {
    if (rej) add_i64(&sum->n_rejected, rej);
    if (pend) add_i64(&sum->n_pending, pend);
  }
}

// K5e' (windows whose outcome arrays exceed 32 MB): drain-order outcomes -> request ids,
// one request-id range per launch, so each pass's scattered writes fill whole sectors in
// L2 instead of read-modify-writing DRAM; the reads (perm, outcomes) are sequential
__global__ void __launch_bounds__(256)
    k_outcome_scatter(int64_t n, const int32_t* __restrict__ perm, const int2* __restrict__ pos_out,
                      int32_t r_lo, int32_t r_hi, int32_t* __restrict__ req_batch,
                      int32_t* __restrict__ req_row) {
  pdl_prologue();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    const int32_t r = perm[j];
    if (r >= r_lo && r < r_hi) {
      const int2 o = pos_out[j];
      req_batch[r] = o.x;
      req_row[r] = o.y;
    }
  }
}

// ---------------------------------------------------------------------------- K5f
// one 512-thread CTA (fits on an SM beside a pack CTA); every warp owns a contiguous run of
// batches and reads it 32 batches (2 KB, coalesced) per step: warp sums, one block scan of
// the warp totals, then a second coalesced pass writing the running offsets (warp scans)
__global__ void __launch_bounds__(512)
    k_size_offsets(bs_batch* __restrict__ batches, int32_t batches_cap,
                   const int32_t* __restrict__ misc, int64_t* __restrict__ task_base,
                   bs_summary* sum, int32_t ptok) {
  pdl_prologue();
  __shared__ int64_t s_sc[3 * 33];
  __shared__ double s_d[32];
  __shared__ int64_t s_a[32], s_p[32], s_pk[32];
  const int nb = min(misc[66], batches_cap);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = (int)(blockDim.x >> 5);
  const int per = ((nb + nw - 1) / nw + 31) & ~31;
  const int i0 = min(nb, wid * per), i1 = min(nb, i0 + per);
  int64_t v[3] = {0, 0, 0};  // packed elements, rows, K6 pieces
  int64_t adm = 0, pad = 0, peak = 0;
  double ws = 0.0;
#pragma unroll 4
  for (int i = i0 + lane; i < i1; i += 32) {
    const bs_batch& B = batches[i];
    v[0] += (int64_t)B.n * B.pitch;
    v[1] += B.n;
    v[2] += (int64_t)B.n * ((B.pitch + ptok - 1) / ptok);
    adm += B.token_sum;
    pad += (int64_t)B.n * B.max_input_len;
    peak = B.footprint > peak ? B.footprint : peak;
    ws += B.waste;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) v[k] = warp_sum(v[k]);
  if (lane != 0) v[0] = v[1] = v[2] = 0;  // one contribution per warp to the block scan
  int64_t tot[3];
  block_excl_scan_k<3, int64_t>(v, tot, s_sc);
  int64_t run[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) run[k] = __shfl_sync(0xffffffffu, v[k], 0);
  for (int base = i0; base < i1; base += 32) {
    const int i = base + lane;
    int64_t x[3] = {0, 0, 0};
    if (i < i1) {
      const bs_batch& B = batches[i];
      x[0] = (int64_t)B.n * B.pitch;
      x[1] = B.n;
      x[2] = (int64_t)B.n * ((B.pitch + ptok - 1) / ptok);
    }
    int64_t inc[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) inc[k] = warp_incl_scan(x[k]);
    if (i < i1) {
      batches[i].out_offset = run[0] + inc[0] - x[0];
      batches[i].row_base = run[1] + inc[1] - x[1];
      task_base[i] = run[2] + inc[2] - x[2];
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) run[k] += __shfl_sync(0xffffffffu, inc[k], 31);
  }
  if (tid == 0) task_base[nb] = tot[2];
  adm = warp_sum(adm);
  pad = warp_sum(pad);
  peak = warp_max(peak);
  ws = warp_sum(ws);
  if (lane == 0) { s_a[wid] = adm; s_p[wid] = pad; s_pk[wid] = peak; s_d[wid] = ws; }
  __syncthreads();
  if (tid == 0) {
    int64_t A = 0, Pd = 0, Pk = 0;
    double Ws = 0.0;
    for (int w = 0; w < nw; ++w) {
      A += s_a[w]; Pd += s_p[w]; Pk = s_pk[w] > Pk ? s_pk[w] : Pk; Ws += s_d[w];
    }
    sum->admitted_tokens = A;
    sum->padded_tokens = Pd;
    sum->packed_elems = tot[0];
    sum->peak_footprint = Pk;
    sum->waste_sum = Ws;
  }
}

__global__ void k_fill_pending(int64_t n, int32_t* req_batch, int32_t* req_row, bs_summary* sum) {
  pdl_prologue();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    req_batch[i] = BS_REQ_PENDING;
    req_row[i] = -1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) sum->n_pending = n;
}

cudaError_t launch_size(bs_ctx* ctx, const int32_t* len, const int32_t* perm,
                        const int32_t* seg_off, int64_t n, const bs_window_params& p,
                        bs_batch* batches, int32_t batches_cap, int32_t* req_batch,
                        int32_t* req_row, bs_summary* summary, cudaStream_t st,
                        const int64_t* tok_off) {
  cudaError_t e;
  ctx->rowdesc_ready = false;
  const int64_t H = p.current_safe - p.pledged;
  if (n == 0 || H <= 0)
    for (int s = 5; s <= 8; ++s) prof_mark(ctx, s, st);
  if (n == 0) return cudaSuccess;
  if (H <= 0) {  // form_batch returns None before touching the queue (:150-152)
    launch_k(ctx, k_fill_pending, dim3((unsigned)std::min<int64_t>((n + 255) / 256, 4LL * ctx->num_sms)), dim3(256), 0, st, false, n, req_batch, req_row, summary);
    ++ctx->launches;
    return cudaGetLastError();
  }
  SizeArgs a;
  a.n = n;
  a.T = H / p.kv_bytes_per_token;
  a.S = p.current_safe / p.kv_bytes_per_token;
  a.kvpt = p.kv_bytes_per_token;
  a.padded = p.accounting == BS_ACCOUNTING_PADDED;
  a.L = p.l_max;
  a.truncate = p.truncate;
  a.C = p.n_classes;
  a.sjf_mask = a.ljf_mask = 0;
  a.walk = ctx->chain_walk > 0 ? ctx->chain_walk : kWalk;
  a.walk_forced = ctx->chain_walk > 0;
  a.pairs = ctx->chain_pairs && ctx->r_cap >= 2;
  for (int c = 0; c < p.n_classes; ++c) {
    if (p.policy[c] == BS_POLICY_SJF) a.sjf_mask |= 1 << c;
    if (p.policy[c] == BS_POLICY_LJF) a.ljf_mask |= 1 << c;
  }
  int32_t* misc = ctx->misc;
  if (!ctx->window_zeroed) {  // the fused window zeroes misc in k_window_init
    e = cudaMemsetAsync(misc, 0, sizeof(int32_t) * 128, st);
    if (e != cudaSuccess) return e;
  }
  const int64_t groups = (n + 31) >> 5;
  const unsigned wblocks = (unsigned)std::min<int64_t>((groups + 7) / 8, 16LL * ctx->num_sms);
  launch_k(ctx, k_size_prep, dim3(wblocks), dim3(256), 0, st, false, len, perm, a, ctx->sorted_len, ctx->bmask, ctx->bmax,
                                       ctx->bmin, ctx->bcnt, ctx->bsum, ctx->sorted_keys,
                                       ctx->slot_len);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  prof_mark(ctx, 5, st);
  launch_k(ctx, k_size_next, dim3(wblocks), dim3(256), 0, st, false, a, ctx->kinfo, seg_off, ctx->sorted_len, ctx->bmask,
                                       ctx->bmax, ctx->bcnt, ctx->bsum, ctx->J, ctx->is_start,
                                       misc, ctx->sorted_keys, ctx->slot_seg);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  prof_mark(ctx, 6, st);
  {
    const int64_t G = (n + 31) >> 5;
    const int32_t n_tiles = (int32_t)((G + kRgTile - 1) / kRgTile);
    const int64_t segs_ub = (int64_t)p.l_max * p.n_classes;  // K2 makes at most L*C segments
    int32_t* dseg = p.dispatch ? ctx->disp_cseg : nullptr;
    int32_t* dmin = p.dispatch ? ctx->disp_cmin : nullptr;
    int64_t* dsum = p.dispatch ? ctx->disp_csum : nullptr;
    if (a.pairs) {
      launch_k(ctx, k_chain_pairs, dim3(wblocks), dim3(256), 0, st, false, n, ctx->J, ctx->J + n);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
      ++ctx->launches;
    }
    launch_k(ctx, k_chain_walk, dim3((unsigned)(n_tiles + (segs_ub + 255) / 256)), dim3(256), 0, st,
             false, a, ctx->kinfo, seg_off, ctx->J, ctx->listB, ctx->sorted_len, ctx->bmask,
             ctx->bcnt, ctx->segw, misc, ctx->rg_tiles, n_tiles);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    launch_k(ctx, k_chain_long, dim3((unsigned)ctx->num_sms), dim3(1024), 0, st, false, a,
             ctx->kinfo, seg_off, ctx->J, ctx->r_cap, ctx->sorted_len, ctx->bmask, ctx->segw,
             misc, summary);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    launch_k(ctx, k_chain_bases, dim3(1), dim3(1024), 0, st, false, ctx->kinfo, ctx->segw, misc,
             ctx->rg_tiles, ctx->rg_tiles + n_tiles, n_tiles, batches_cap, summary);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const int64_t nodes_blocks = std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 4LL * ctx->num_sms));
    launch_k(ctx, k_chain_nodes, dim3((unsigned)(n_tiles + nodes_blocks)), dim3(256), 0, st, false,
             a, ctx->kinfo, seg_off, ctx->J, ctx->listB, ctx->listA, ctx->node_batch,
             ctx->node_j0, ctx->segw, misc, ctx->bcnt, ctx->rg_tiles + n_tiles, ctx->Rg, n_tiles,
             dseg, dmin, dsum);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ctx->launches += 3;  // four chain kernels where the count below has one
  }
  prof_mark(ctx, 7, st);
  launch_k(ctx, k_size_describe, dim3(wblocks), dim3(256), 0, st, false, a, ctx->kinfo, seg_off, ctx->sorted_len, ctx->bmax,
                                           ctx->bmin, ctx->bcnt, ctx->bsum, ctx->J, ctx->listA,
                                           ctx->listB, ctx->node_batch, misc, batches,
                                           batches_cap, summary, ctx->sorted_keys, ctx->slot_seg);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  ctx->piece_tok = piece_tokens_for(n);
  ctx->last_n = n;
  ctx->pack_pieces = n * (((int64_t)p.l_max + ctx->piece_tok - 1) / ctx->piece_tok);
  launch_k(ctx, k_size_offsets, dim3(1), dim3(512), 0, st, false, batches, batches_cap, misc, ctx->task_base, summary,
                                     ctx->piece_tok);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  prof_mark(ctx, 8, st);
  // outcome arrays beyond 32 MB (4M requests) are scattered in request-id ranges of
  // <= 32 MB (C3, 16M requests: 4 passes, 0.60 vs 0.72 ms; 3 passes of 43 MB gain
  // nothing, every extra pass re-reads the positions, ~0.1 ms at 16M)
  const char* pv = getenv("BS_OUTCOME_PARTS");  // tuning / test hook
  const int parts_env = pv ? std::max(1, atoi(pv)) : 0;
  const int parts = parts_env ? parts_env
                              : (int)std::max<int64_t>(1, (n * 8 + (32LL << 20) - 1) / (32LL << 20));
  const int64_t span = (n + parts - 1) / parts;
  // more than one range: K5e runs once and writes the outcomes in drain order (into the
  // doubling table's levels >= 1, free after K5c), k_outcome_scatter moves each range
  int2* pos_out =
      parts > 1 && ctx->r_cap >= 4 ? reinterpret_cast<int2*>(ctx->J + ((n + 1) & ~1LL)) : nullptr;
  const int passes = pos_out ? 1 : parts;
  for (int q = 0; q < passes; ++q) {
    launch_k(ctx, k_size_outcome, dim3(wblocks), dim3(256), 0, st, false,
        a, perm, ctx->bmask, ctx->Rg, ctx->listA, ctx->listB, ctx->node_batch, ctx->node_j0, misc,
        batches, batches_cap, req_batch, req_row, ctx->rowpos, summary, ctx->sorted_len,
        p.dispatch ? ctx->disp_cmin : nullptr, p.dispatch ? ctx->disp_csum : nullptr,
        (int32_t)std::min<int64_t>(n, q * span), (int32_t)std::min<int64_t>(n, (q + 1) * span),
        q == 0, tok_off, tok_off ? ctx->rowdesc : nullptr, ctx->chunk_row, pos_out);
  }
  if (pos_out) {
    const unsigned sblocks = (unsigned)std::min<int64_t>((n + 255) / 256, 8LL * ctx->num_sms);
    for (int q = 0; q < parts; ++q)
      launch_k(ctx, k_outcome_scatter, dim3(sblocks), dim3(256), 0, st, false, n, perm,
               (const int2*)pos_out, (int32_t)std::min<int64_t>(n, q * span),
               (int32_t)std::min<int64_t>(n, (q + 1) * span), req_batch, req_row);
    ctx->launches += 1;  // parts scatters + one K5e instead of parts K5e
  }
  // with the token offsets, K5e wrote the bulk-staged pack's row records for the whole
  // window (the fused path then skips k_pack_rowprep)
  ctx->rowdesc_ready = tok_off != nullptr;
  ctx->launches += 5 + parts;
  return cudaGetLastError();
}

}  // namespace bsk

