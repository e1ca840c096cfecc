/*
 * oracle/bso.c — CPU restatement of the BucketServe window scheduling path.
 *
 * TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library, and
 * only as the checker or the timed CPU baseline.  The product path
 * (paper_2507_17120_b200, CUDA) never calls it.
 *
 * Every function restates the reference algorithm (bucketsim, pure Python, at
 * /root/reference/pkg/src/bucketsim) on structure-of-arrays inputs and cites the
 * file:line it follows.  The composition is the reference window of SURVEY §3.4:
 *   assign every request -> adjust_buckets(current_n_max) until a pass yields no
 *   split -> for each bucket, for each class in priority order, form_batch until
 *   it returns None.
 * It is pinned against the live reference by oracle/gen_golden.py (fixtures in
 * tests/golden/) and by tests/test_oracle_golden.py.
 *
 * Build: oracle/Makefile -> oracle/_build/libbso.so (gcc -O2 -fopenmp).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Same layout as bs_window_params in include/bucketserve.h (kept independent). */
typedef struct {
  int32_t l_max, n_classes, policy[8];
  double theta;
  int32_t adjust, max_passes;
  int64_t n_max, kvpt, current_safe, pledged;
  int32_t accounting, truncate, pad_id, reserved;
} bso_params;

typedef struct {
  int32_t segment, start, end, n, max_input_len, pitch;
  int64_t token_sum, footprint, out_offset;
  double waste;
  int64_t row_base;
} bso_batch;

typedef struct {
  int64_t n_requests, total_global, sum_len_global, n_max, k_buckets, n_changes, n_passes,
      n_batches, n_rejected, n_pending, admitted_tokens, padded_tokens, packed_elems,
      peak_footprint;
  double waste_sum;
  int64_t sort_passes, flags, reserved[15];
} bso_summary;

enum { FCFS = 0, SJF = 1, LJF = 2 };
enum { PADDED = 0, EXACT = 1 };
enum { SPLIT = 1, MERGE = 2, SKIP = 3 };
#define F_LEN 0x1
#define F_CLASS 0x2
#define F_ZERO_MEAN 0x4
#define F_CHANGES 0x8
#define F_PACK_CAP 0x10
#define F_NONPOS 0x20
#define F_BATCH_CAP 0x40
#define REQ_PENDING (-1)
#define REQ_REJECTED (-2)
#define PACK_ALIGN 16 /* BS_PACK_ALIGN */

int bso_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void bso_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* Length seen by the scheduler.  pd_sim.py:382-383 truncates len >= L to L-1
 * before BucketSet.assign; without truncation assign raises ValueError
 * (bucket_manager.py:112-115).  Out-of-range values are clamped so downstream
 * stages stay in bounds and the error is latched in *flags. */
static inline int32_t eff_len(int32_t x, const bso_params* p, int64_t* flags) {
  if (x < 0) { *flags |= F_LEN; return 0; }
  if (x >= p->l_max) {
    if (!p->truncate) *flags |= F_LEN;
    return p->l_max - 1;
  }
  return x;
}
static inline int32_t eff_cls(uint8_t c, const bso_params* p, int64_t* flags) {
  if ((int32_t)c >= p->n_classes) { *flags |= F_CLASS; return p->n_classes - 1; }
  return (int32_t)c;
}

/* K1. Per-(class, length) counts: the state behind len(bucket.requests) and
 * Bucket.short_count (bucket_manager.py:31-32, 39-40, 126-127). */
int bso_histogram(const int32_t* len, const uint8_t* cls, int64_t n, const bso_params* p,
                  uint32_t* hist, int64_t* flags) {
  const int64_t L = p->l_max, C = p->n_classes;
  memset(hist, 0, sizeof(uint32_t) * (size_t)(L * C));
  int64_t fl = 0;
  for (int64_t i = 0; i < n; ++i) {
    int32_t x = eff_len(len[i], p, &fl);
    int32_t c = eff_cls(cls[i], p, &fl);
    hist[c * L + x] += 1;
  }
  *flags |= fl;
  return 0;
}

/* CPython float floor division (Objects/floatobject.c, _float_div_mod), the
 * operation behind `self.token_budget() // mean_len` (batch_controller.py:104). */
static double py_floordiv(double vx, double wx) {
  double mod = fmod(vx, wx);
  double div = (vx - mod) / wx;
  if (mod != 0.0) {
    if ((wx < 0) != (mod < 0)) { mod += wx; div -= 1.0; }
  }
  double fd;
  if (div != 0.0) {
    fd = floor(div);
    if (div - fd > 0.5) fd += 1.0;
  } else {
    fd = copysign(0.0, vx / wx);
  }
  return fd;
}

/* BatchController.current_n_max (batch_controller.py:93-104):
 *   total == 0 -> 1; else max(1, int(token_budget() // (sum_len / total))).
 * token_budget() = current_safe // kv_per_token (batch_controller.py:90-91).
 * sum/total is Python true division of ints: correctly rounded, identical to the
 * IEEE quotient of the two exactly-representable doubles (both < 2^53). */
int64_t bso_n_max(uint64_t total, uint64_t sum_len, int64_t current_safe, int64_t kvpt,
                  int64_t* flags) {
  if (total == 0) return 1;
  double mean = (double)sum_len / (double)total;
  if (mean == 0.0) { *flags |= F_ZERO_MEAN; return 1; }
  int64_t tb = current_safe / kvpt;
  double q = py_floordiv((double)tb, mean);
  int64_t v = (int64_t)q; /* int(): truncation toward zero; q >= 0 here */
  return v < 1 ? 1 : v;
}

/* K2. BucketSet.adjust_buckets (bucket_manager.py:133-191), repeated up to
 * max_passes times (<= 0: until a pass yields no split — the window fixpoint of
 * SURVEY §3.4 / Appendix A.5), on bucket counts read from prefix sums of the
 * total histogram:  count = P[up]-P[low], short_count = P[mid]-P[low] with
 * mid = (low+up)//2 (bucket_manager.py:31-32).
 * Returns 0, or -1 for malformed init edges. */
int bso_boundaries(const uint32_t* hist, const bso_params* p, const int32_t* init_edges,
                   int32_t k_init, int32_t* edges_out, int32_t* k_out, int32_t* changes,
                   int32_t cap, bso_summary* sum) {
  const int64_t L = p->l_max, C = p->n_classes;
  uint64_t* P = (uint64_t*)calloc((size_t)L + 1, sizeof(uint64_t));
  uint64_t slen = 0;
  for (int64_t x = 0; x < L; ++x) {
    uint64_t h = 0;
    for (int64_t c = 0; c < C; ++c) h += hist[c * L + x];
    P[x + 1] = P[x] + h;
    slen += h * (uint64_t)x;
  }
  const uint64_t total = P[L];
  int64_t fl = 0;
  int64_t n_max = p->n_max > 0 ? p->n_max : bso_n_max(total, slen, p->current_safe, p->kvpt, &fl);

  int32_t* e = (int32_t*)malloc(sizeof(int32_t) * ((size_t)L + 1));
  int32_t* ne = (int32_t*)malloc(sizeof(int32_t) * ((size_t)L + 1));
  int32_t k;
  if (init_edges) {
    k = k_init;
    if (k < 1 || init_edges[0] != 0 || init_edges[k] != L) { free(P); free(e); free(ne); return -1; }
    for (int32_t i = 0; i <= k; ++i) {
      if (i > 0 && init_edges[i] <= init_edges[i - 1]) { free(P); free(e); free(ne); return -1; }
      e[i] = init_edges[i];
    }
  } else {
    k = 1; e[0] = 0; e[1] = (int32_t)L; /* bucket_manager.py:87 */
  }
  int64_t nch = 0, passes = 0;
#define LOG(kind, lo, up, mid)                                                             \
  do {                                                                                     \
    if (nch < cap) {                                                                       \
      changes[4 * nch] = kind; changes[4 * nch + 1] = lo; changes[4 * nch + 2] = up;       \
      changes[4 * nch + 3] = mid;                                                          \
    }                                                                                      \
    ++nch;                                                                                 \
  } while (0)
  if (p->adjust) {
    for (;;) {
      ++passes; /* adjust_calls += 1, bucket_manager.py:142 */
      if (total < (uint64_t)n_max) { /* merge branch, :148-156 */
        if (!(k == 1 && e[0] == 0 && e[1] == L)) {
          k = 1; e[0] = 0; e[1] = (int32_t)L;
          LOG(MERGE, 0, (int32_t)L, -1);
        }
        break;
      }
      if (total == (uint64_t)n_max) break; /* :158-160 */
      int any_split = 0, nk = 0;
      ne[0] = e[0];
      for (int32_t b = 0; b < k; ++b) { /* split_list + rebuild, :162-187 */
        int32_t lo = e[b], up = e[b + 1], mid = (lo + up) / 2;
        uint64_t c = P[up] - P[lo], s = P[mid] - P[lo];
        /* `c > n_max and b.short_count > threshold * c`, float64 product */
        int split = (c > (uint64_t)n_max) && ((double)s > p->theta * (double)c);
        if (split) {
          if (mid <= lo) { /* width-1 bucket: degenerate midpoint, :175-178 */
            LOG(SKIP, lo, up, mid);
          } else {
            ne[++nk] = mid;
            LOG(SPLIT, lo, up, mid);
            any_split = 1;
          }
        }
        ne[++nk] = up;
      }
      k = nk;
      memcpy(e, ne, sizeof(int32_t) * ((size_t)k + 1));
      if (!any_split) break;
      if (p->max_passes > 0 && passes >= p->max_passes) break;
    }
  }
#undef LOG
  memcpy(edges_out, e, sizeof(int32_t) * ((size_t)k + 1));
  *k_out = k;
  if (nch > cap) fl |= F_CHANGES;
  sum->total_global = (int64_t)total;
  sum->sum_len_global = (int64_t)slen;
  sum->n_max = n_max;
  sum->k_buckets = k;
  sum->n_changes = nch;
  sum->n_passes = passes;
  sum->flags |= fl;
  free(P); free(e); free(ne);
  return 0;
}

/* K3. BucketSet.assign (bucket_manager.py:110-131): index of the first bucket
 * with len < up in the contiguous ascending partition. */
void bso_assign(const int32_t* len, int64_t n, const bso_params* p, const int32_t* edges,
                int32_t k, int32_t* bucket_out, int64_t* flags) {
  int64_t fl = 0;
  for (int64_t i = 0; i < n; ++i) {
    int32_t x = eff_len(len[i], p, &fl);
    int32_t lo = 0, hi = k - 1; /* first b with x < edges[b+1] */
    while (lo < hi) {
      int32_t mid = (lo + hi) / 2;
      if (x < edges[mid + 1]) hi = mid; else lo = mid + 1;
    }
    bucket_out[i] = lo;
  }
  *flags |= fl;
}

typedef struct { int64_t sub; int32_t idx; } okey;
static int okey_cmp(const void* a, const void* b) {
  const okey* x = (const okey*)a; const okey* y = (const okey*)b;
  if (x->sub != y->sub) return x->sub < y->sub ? -1 : 1;
  return (x->idx > y->idx) - (x->idx < y->idx);
}

/* K4. Drain order of the window: bucket ascending (the composition visits
 * buckets left to right), class ascending (ONLINE before OFFLINE, pd_sim.py:449-450;
 * the class filter of form_batch, batch_controller.py:154-156), then
 * order_requests (batch_controller.py:33-41): SJF (len, arrival, id), LJF
 * (-len, arrival, id), FCFS/EARLIEST_ARRIVAL (arrival, id); arrival rank = index. */
void bso_order(const int32_t* len, const uint8_t* cls, int64_t n, const bso_params* p,
               const int32_t* edges, int32_t k, int32_t* perm, int32_t* seg_off,
               int64_t* flags) {
  const int64_t C = p->n_classes, S = (int64_t)k * C;
  int32_t* bucket = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  bso_assign(len, n, p, edges, k, bucket, flags);
  int64_t* cnt = (int64_t*)calloc((size_t)S + 1, sizeof(int64_t));
  int64_t fl = 0;
  for (int64_t i = 0; i < n; ++i) cnt[bucket[i] * C + eff_cls(cls[i], p, &fl)]++;
  int64_t run = 0;
  for (int64_t s = 0; s < S; ++s) { int64_t c = cnt[s]; seg_off[s] = (int32_t)run; cnt[s] = run; run += c; }
  seg_off[S] = (int32_t)run;
  okey* keys = (okey*)malloc(sizeof(okey) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) { /* stable partition by segment */
    int32_t c = eff_cls(cls[i], p, &fl);
    int64_t s = bucket[i] * C + c;
    int32_t x = eff_len(len[i], p, &fl);
    int64_t sub = p->policy[c] == SJF ? x : (p->policy[c] == LJF ? -(int64_t)x : 0);
    okey kk = {sub, (int32_t)i};
    keys[cnt[s]++] = kk;
  }
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t s = 0; s < S; ++s) {
    int64_t a = seg_off[s], b = seg_off[s + 1];
    if (b - a > 1) qsort(keys + a, (size_t)(b - a), sizeof(okey), okey_cmp);
  }
  for (int64_t i = 0; i < n; ++i) perm[i] = keys[i].idx;
  *flags |= fl;
  free(keys); free(cnt); free(bucket);
}

/* K5. Drain every (bucket, class) segment with BatchController.form_batch
 * (batch_controller.py:141-191) until it returns None.
 *   headroom = current_safe - pledged; headroom <= 0 -> None, nothing touched (:150-152)
 *   solo = kvpt*len > current_safe -> OversizeRejection, removed (:164-169)
 *   _footprint(new_max, n+1, new_sum) > headroom -> stop the prefix (:170-174)
 * Comparisons run in token space: kvpt*x > H  <=>  x > floor(H/kvpt) for integer
 * x >= 0, H >= 0, kvpt >= 1, which avoids 64-bit overflow of the byte products. */
int bso_size(const int32_t* len, const int32_t* perm, const int32_t* seg_off, int64_t n_segs,
             int64_t n, const bso_params* p, bso_batch* batches, int64_t batches_cap,
             int32_t* req_batch, int32_t* req_row, bso_summary* sum) {
  int64_t fl = 0;
  for (int64_t i = 0; i < n; ++i) { req_batch[i] = REQ_PENDING; req_row[i] = -1; }
  const int64_t kvpt = p->kvpt;
  const int64_t H = p->current_safe - p->pledged;
  int64_t nb = 0, nrej = 0, admitted = 0, padded = 0, packed = 0, peak = 0, admitted_rows = 0;
  double wsum = 0.0;
  if (H > 0) {
    const int64_t T = H / kvpt;
    const int64_t S = p->current_safe / kvpt;
    for (int64_t s = 0; s < n_segs; ++s) {
      int64_t pos = seg_off[s], end = seg_off[s + 1];
      while (pos < end) { /* one form_batch call */
        int64_t call_start = pos, cnt = 0, m = 0, tsum = 0;
        int nonpos = 0;
        while (pos < end) {
          int32_t r = perm[pos];
          int64_t x = eff_len(len[r], p, &fl);
          if (x > S) { req_batch[r] = REQ_REJECTED; ++nrej; ++pos; continue; }
          int64_t nm = x > m ? x : m, ns = tsum + x;
          int64_t need = p->accounting == PADDED ? nm * (cnt + 1) : ns;
          if (need > T) break;
          req_batch[r] = (int32_t)nb; req_row[r] = (int32_t)cnt;
          if (x < 1) nonpos = 1;
          ++cnt; m = nm; tsum = ns; ++pos;
        }
        if (cnt == 0) break; /* form_batch returned None: this segment's drain stops */
        if (nb < batches_cap) {
          bso_batch* B = &batches[nb];
          B->segment = (int32_t)s; B->start = (int32_t)call_start; B->end = (int32_t)pos;
          B->n = (int32_t)cnt; B->max_input_len = (int32_t)m;
          B->pitch = (int32_t)((m + PACK_ALIGN - 1) / PACK_ALIGN * PACK_ALIGN);
          B->token_sum = tsum;
          B->footprint = kvpt * (p->accounting == PADDED ? m * cnt : tsum);
          B->out_offset = packed;
          /* waste_ratio, memory_model.py:98-100: (s_max - s_avg) / s_max */
          double s_avg = (double)tsum / (double)cnt;
          B->waste = ((double)m - s_avg) / (double)m;
          /* waste_ratio raises for any length < 1 (memory_model.py:96-97): NaN + flag */
          if (nonpos) B->waste = NAN;
          B->row_base = admitted_rows;
          wsum += B->waste;
          if (B->footprint > peak) peak = B->footprint;
          packed += (int64_t)B->pitch * cnt;
        } else {
          fl |= F_BATCH_CAP;
        }
        if (nonpos) fl |= F_NONPOS;
        admitted += tsum; padded += m * cnt; admitted_rows += cnt;
        ++nb;
      }
    }
  }
  int64_t npend = 0;
  for (int64_t i = 0; i < n; ++i) npend += req_batch[i] == REQ_PENDING;
  sum->n_requests = n;
  sum->n_batches = nb; sum->n_rejected = nrej; sum->n_pending = npend;
  sum->admitted_tokens = admitted; sum->padded_tokens = padded; sum->packed_elems = packed;
  sum->peak_footprint = peak; sum->waste_sum = wsum;
  sum->flags |= fl;
  return 0;
}

/* K6. Pack (no reference counterpart: bucketsim never holds token ids).
 * Batch b occupies rows [0, n) x [0, pitch) at out_offset; request with row q
 * copies its len tokens, pad_id beyond; mask 1 on real tokens. */
int bso_pack(const int32_t* len, const int32_t* perm, const int32_t* req_batch,
             const int32_t* req_row, const int64_t* tok_off, const int32_t* tokens,
             const bso_params* p, const bso_batch* batches, int64_t nb, int32_t* out_tokens,
             uint8_t* out_mask, int64_t out_capacity) {
  int64_t fl = 0;
  const int64_t base = nb > 0 ? batches[0].out_offset : 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(| : fl)
  for (int64_t b = 0; b < nb; ++b) {
    const bso_batch* B = &batches[b];
    int64_t o = B->out_offset - base;
    if (o + (int64_t)B->n * B->pitch > out_capacity) { fl |= F_PACK_CAP; continue; }
    for (int64_t j = B->start; j < B->end; ++j) {
      int32_t r = perm[j];
      if (req_batch[r] != (int32_t)b) continue;
      int64_t x = eff_len(len[r], p, &fl);
      int32_t* dst = out_tokens + o + (int64_t)req_row[r] * B->pitch;
      const int32_t* src = tokens + tok_off[r];
      memcpy(dst, src, sizeof(int32_t) * (size_t)x);
      for (int64_t t = x; t < B->pitch; ++t) dst[t] = p->pad_id;
      if (out_mask) {
        uint8_t* mk = out_mask + o + (int64_t)req_row[r] * B->pitch;
        memset(mk, 1, (size_t)x);
        memset(mk + x, 0, (size_t)(B->pitch - x));
      }
    }
  }
  return (int)fl;
}

/* Checksum of the packed output without materialising it (parity at full sizes: C3's
 * 16M-request pack is ~37 GB).  Element e (offset from the first batch's out_offset) of
 * the packed token / mask streams contributes tok[e] * w1(e) and mask[e] * w2(e),
 * w_k(e) = e * A_k + B_k, all mod 2^64 — position-sensitive, so a token in the wrong
 * slot changes the sum.  Tokens come from `tokens` or, when it is NULL, are regenerated
 * from the synthetic store's hash (token at store slot q = ((q * mul + seed) mod 2^32)
 * mod vocab, workloads.token_store).  Covers the real tokens and the padding of every
 * row of every batch.  out[0] = token sum, out[1] = mask sum. */
#define CK_A1 0x9E3779B97F4A7C15ull
#define CK_B1 0x632BE59BD9B4E019ull
#define CK_A2 0xD6E8FEB86659FD93ull
#define CK_B2 0xA0761D6478BD642Full
void bso_pack_checksum(const int32_t* len, const int32_t* perm, const int32_t* req_batch,
                       const int32_t* req_row, const int64_t* tok_off, const int32_t* tokens,
                       uint32_t mul, uint32_t seed, uint32_t vocab, const bso_params* p,
                       const bso_batch* batches, int64_t nb, uint64_t* out) {
  int64_t fl = 0;
  uint64_t st = 0, sm = 0;
  const int64_t base = nb > 0 ? batches[0].out_offset : 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : st, sm) reduction(| : fl)
  for (int64_t b = 0; b < nb; ++b) {
    const bso_batch* B = &batches[b];
    for (int64_t j = B->start; j < B->end; ++j) {
      const int32_t r = perm[j];
      if (req_batch[r] != (int32_t)b) continue;
      const int64_t x = eff_len(len[r], p, &fl);
      const uint64_t e0 = (uint64_t)(B->out_offset - base + (int64_t)req_row[r] * B->pitch);
      for (int64_t t = 0; t < B->pitch; ++t) {
        const uint64_t e = e0 + (uint64_t)t;
        uint32_t tok;
        if (t < x) {
          const uint64_t q = (uint64_t)tok_off[r] + (uint64_t)t;
          tok = tokens ? (uint32_t)tokens[q] : (uint32_t)(((uint32_t)q * mul + seed) % vocab);
          sm += e * CK_A2 + CK_B2;
        } else {
          tok = (uint32_t)p->pad_id;
        }
        st += (uint64_t)tok * (e * CK_A1 + CK_B1);
      }
    }
  }
  out[0] = st;
  out[1] = sm;
}

/* f2 monitor view: LengthHistogram.from_samples(lengths, bins, range=(0, L))
 * (memory_model.py:125-130, pd_sim.py:829-831) equals bincount((len*bins)//L). */
void bso_monitor_bins(const uint32_t* hist, const bso_params* p, int32_t bins, uint64_t* out) {
  const int64_t L = p->l_max, C = p->n_classes;
  memset(out, 0, sizeof(uint64_t) * (size_t)bins);
  for (int64_t x = 0; x < L; ++x) {
    uint64_t h = 0;
    for (int64_t c = 0; c < C; ++c) h += hist[c * L + x];
    out[(x * bins) / L] += h;
  }
}

/* The whole window in one call; used by bench.py's CPU leg. */
int bso_window(const int32_t* len, const uint8_t* cls, int64_t n, const int64_t* tok_off,
               const int32_t* tokens, const bso_params* p, const int32_t* init_edges,
               int32_t k_init, uint32_t* hist, int32_t* edges, int32_t* k_out, int32_t* changes,
               int32_t changes_cap, int32_t* perm, int32_t* seg_off, bso_batch* batches,
               int64_t batches_cap, int32_t* req_batch, int32_t* req_row, int32_t* out_tokens,
               uint8_t* out_mask, int64_t out_capacity, bso_summary* sum) {
  memset(sum, 0, sizeof(*sum));
  int64_t fl = 0;
  bso_histogram(len, cls, n, p, hist, &fl);
  sum->flags |= fl;
  if (bso_boundaries(hist, p, init_edges, k_init, edges, k_out, changes, changes_cap, sum) != 0)
    return -1;
  fl = 0;
  bso_order(len, cls, n, p, edges, *k_out, perm, seg_off, &fl);
  sum->flags |= fl;
  bso_size(len, perm, seg_off, (int64_t)(*k_out) * p->n_classes, n, p, batches, batches_cap,
           req_batch, req_row, sum);
  if (out_tokens && tokens && tok_off) {
    int64_t nb = sum->n_batches < batches_cap ? sum->n_batches : batches_cap;
    sum->flags |= bso_pack(len, perm, req_batch, req_row, tok_off, tokens, p, batches, nb,
                           out_tokens, out_mask, out_capacity);
  }
  return 0;
}

/* f3. Global batch emission order: Simulator._next_plan (pd_sim.py:448-462) repeated
 * while it makes progress.  Each call tries the classes in priority order; for a
 * class, BatchController.select_bucket (batch_controller.py:106-134) picks the
 * bucket — class 0 (ONLINE): the one holding the globally oldest request of the
 * class (:114-123); other classes (OFFLINE): the largest queued token mass of the
 * class, strict > from 0, so ties go to the lower index (:124-134) — and form_batch
 * runs on it; the first plan ends the call.  A call that forms no plan but rejects
 * requests still counts as progress (the simulator marks the set dirty, :457-459).
 * Generalisation: classes >= 2 use the mass rule of their own class.
 *
 * The form_batch calls of one (bucket, class) segment do not depend on the others
 * (fixed current_safe and pledged), so each call's outcome is read from the drain
 * of bso_size (the batch starting at the segment's cursor, or the segment's null
 * tail call); this function restates only the selection loop.  Outputs:
 * emit_order[t] = batch of the t-th plan; batch_emit[b] = t or -1 (never formed);
 * req_batch / req_row are rewritten to the dispatch outcome (requests of calls the
 * loop never reaches stay queued: BS_REQ_PENDING).  Returns the number of plans. */
int64_t bso_dispatch(const int32_t* len, const int32_t* perm, const int32_t* seg_off,
                     int64_t n_segs, int64_t n, const bso_params* p, const bso_batch* batches,
                     int64_t nb, int32_t* req_batch, int32_t* req_row, int32_t* emit_order,
                     int32_t* batch_emit, bso_summary* sum) {
  const int64_t C = p->n_classes;
  int64_t fl = 0;
  for (int64_t b = 0; b < nb; ++b) batch_emit[b] = -1;
  int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_segs + 1));
  int64_t* nextb = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_segs + 1));
  int32_t* sufmin = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  int64_t* pre = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  pre[0] = 0;
  for (int64_t j = 0; j < n; ++j) pre[j + 1] = pre[j] + eff_len(len[perm[j]], p, &fl);
  for (int64_t s = 0; s < n_segs; ++s) {
    cur[s] = seg_off[s];
    int32_t m = INT32_MAX;
    for (int64_t j = seg_off[s + 1] - 1; j >= seg_off[s]; --j) {
      if (perm[j] < m) m = perm[j];
      sufmin[j] = m;
    }
  }
  for (int64_t s = 0, b = 0; s < n_segs; ++s) { /* first batch of each segment */
    while (b < nb && batches[b].segment < s) ++b;
    nextb[s] = b;
  }
  const int64_t H = p->current_safe - p->pledged;
  int64_t t = 0;
  for (;;) {
    int formed = 0, progress = 0;
    for (int64_t c = 0; c < C && !formed; ++c) {
      int64_t best = -1;
      if (c == 0) { /* oldest queued request of the class */
        int32_t best_key = INT32_MAX;
        for (int64_t s = c; s < n_segs; s += C)
          if (cur[s] < seg_off[s + 1] && sufmin[cur[s]] < best_key) { best_key = sufmin[cur[s]]; best = s; }
      } else { /* largest queued token mass, strict > from 0 */
        int64_t best_mass = 0;
        for (int64_t s = c; s < n_segs; s += C) {
          const int64_t mass = pre[seg_off[s + 1]] - pre[cur[s]];
          if (mass > best_mass) { best_mass = mass; best = s; }
        }
      }
      if (best < 0) continue;
      if (H <= 0) continue; /* form_batch returns None before touching the queue (:150-152) */
      const int64_t s = best, end = seg_off[s + 1];
      const int64_t b = nextb[s];
      if (b < nb && batches[b].segment == s && batches[b].start == cur[s]) {
        batch_emit[b] = (int32_t)t;
        emit_order[t++] = (int32_t)b;
        cur[s] = batches[b].end;
        nextb[s] = b + 1;
        formed = 1;
      } else { /* the segment's null call: rejects up to the first admissible request */
        int64_t j = cur[s];
        while (j < end && req_batch[perm[j]] == REQ_REJECTED) ++j;
        if (j > cur[s]) progress = 1;
        cur[s] = j;
      }
    }
    if (!formed && !progress) break;
  }
  int64_t nrej = 0, npend = 0;
  for (int64_t s = 0; s < n_segs; ++s)
    for (int64_t j = cur[s]; j < seg_off[s + 1]; ++j) { req_batch[perm[j]] = REQ_PENDING; req_row[perm[j]] = -1; }
  for (int64_t i = 0; i < n; ++i) { nrej += req_batch[i] == REQ_REJECTED; npend += req_batch[i] == REQ_PENDING; }
  sum->n_rejected = nrej;
  sum->n_pending = npend;
  sum->reserved[0] = t; /* n_emitted */
  sum->flags |= fl;
  free(cur); free(nextb); free(sufmin); free(pre);
  return t;
}
