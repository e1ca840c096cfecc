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
// B200 design (no sequential walk over requests):
//   K5a  gather lengths into drain order + per-32-position summaries
//        (max / count / sum of the non-rejected lengths)
//   K5b  next(j) for EVERY position in parallel: where a form_batch call that
//        starts at j would stop — a gallop over the 32-position summaries, exact
//        element steps only at the two ends
//   K5c  pointer doubling J[r] = next^(2^r) in one cooperative kernel (grid.sync
//        between levels, stops when every segment's chain is covered), then a
//        top-down expansion from the segment starts emits every batch start in
//        emission order — O(N log B) work, O(log B) depth instead of a walk of B
//        dependent steps per segment
//   K5d  one CTA per batch: rows (block scan over admitted positions),
//        reductions, BatchPlan fields, per-request outcome
//   K5e  one CTA: packed-buffer offsets (exclusive scan of n*pitch) + totals
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
  int32_t pad0;
};

__device__ __forceinline__ int64_t seg_of(const int32_t* __restrict__ seg_off, int32_t n_segs,
                                          int64_t j) {
  // largest s with seg_off[s] <= j  (upper_bound - 1 over seg_off[0..n_segs])
  int32_t lo = 0, hi = n_segs;  // answer in [0, n_segs-1]
  while (hi - lo > 1) {
    const int32_t mid = (lo + hi) >> 1;
    if (seg_off[mid] <= j) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int64_t first_nonrej(int64_t j, int64_t end,
                                                const int32_t* __restrict__ slen,
                                                const int32_t* __restrict__ bcnt, int64_t S) {
  int64_t k = j;
  while (k < end && (k & 31)) {
    if (slen[k] <= S) return k;
    ++k;
  }
  while (k + 32 <= end && bcnt[k >> 5] == 0) k += 32;
  while (k < end) {
    if (slen[k] <= S) return k;
    ++k;
  }
  return end;
}

__device__ __forceinline__ bool fits(const SizeArgs& a, int64_t m, int64_t c, int64_t s) {
  return a.padded ? (m * c <= a.T) : (s <= a.T);
}

// first position where the batch that admits j0 first stops (or `end`)
__device__ int64_t greedy_stop(int64_t j0, int64_t end, const SizeArgs& a,
                               const int32_t* __restrict__ slen, const int32_t* __restrict__ bmax,
                               const int32_t* __restrict__ bcnt,
                               const int32_t* __restrict__ bsum) {
  int64_t m = slen[j0], c = 1, s = m;
  int64_t k = j0 + 1;
  while (k < end && (k & 31)) {
    const int64_t x = slen[k];
    if (x <= a.S) {
      const int64_t nm = x > m ? x : m;
      if (!fits(a, nm, c + 1, s + x)) return k;
      m = nm; ++c; s += x;
    }
    ++k;
  }
  while (k + 32 <= end) {
    const int g = (int)(k >> 5);
    const int64_t bc = bcnt[g];
    if (bc) {
      const int64_t bm = bmax[g];
      const int64_t nm = bm > m ? bm : m;
      if (!fits(a, nm, c + bc, s + bsum[g])) break;
      m = nm; c += bc; s += bsum[g];
    }
    k += 32;
  }
  while (k < end) {
    const int64_t x = slen[k];
    if (x <= a.S) {
      const int64_t nm = x > m ? x : m;
      if (!fits(a, nm, c + 1, s + x)) return k;
      m = nm; ++c; s += x;
    }
    ++k;
  }
  return end;
}

// K5a
__global__ void k_size_prep(const int32_t* __restrict__ len, const int32_t* __restrict__ perm,
                            SizeArgs a, int32_t* __restrict__ slen, int32_t* __restrict__ bmax,
                            int32_t* __restrict__ bcnt, int32_t* __restrict__ bsum) {
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
      x = eff_len(len[perm[j]], a.L, a.truncate, fl);
      slen[j] = x;
    }
    const bool nr = valid && (int64_t)x <= a.S;
    const int32_t v = nr ? x : 0;
    const int32_t m = warp_max(v);
    const int32_t s = warp_sum(v);
    const int32_t c = __popc(__ballot_sync(0xffffffffu, nr));
    if (lane == 0) { bmax[g] = m; bcnt[g] = c; bsum[g] = s; }
  }
}

// K5b
__global__ void k_size_next(SizeArgs a, const int32_t* __restrict__ kinfo,
                            const int32_t* __restrict__ seg_off,
                            const int32_t* __restrict__ slen, const int32_t* __restrict__ bmax,
                            const int32_t* __restrict__ bcnt, const int32_t* __restrict__ bsum,
                            int32_t* __restrict__ J0, uint8_t* __restrict__ is_start,
                            int32_t* __restrict__ alive) {
  const int32_t n_segs = kinfo[2];
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < a.n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = seg_of(seg_off, n_segs, j);
    const int64_t end = seg_off[s + 1];
    const bool start = seg_off[s] == j;
    int32_t nx = kEnd;
    const int64_t j0 = first_nonrej(j, end, slen, bcnt, a.S);
    if (j0 < end && (int64_t)slen[j0] <= a.T) {
      const int64_t st = greedy_stop(j0, end, a, slen, bmax, bcnt, bsum);
      if (st < end) nx = (int32_t)st;
    }
    J0[j] = nx;
    is_start[j] = start;
    if (start && nx != kEnd) alive[0] = 1;
  }
}

// K5c
struct ChainShared {
  int32_t si[33];
  int32_t flag;
};

__device__ __forceinline__ int32_t ld_rel_i32(const int32_t* p) {
  return (int32_t)ld_relaxed(reinterpret_cast<const uint32_t*>(p));
}

__global__ void __launch_bounds__(512)
    k_chain(SizeArgs a, const int32_t* __restrict__ kinfo, const int32_t* __restrict__ seg_off,
            int32_t* J, int r_cap,
            const uint8_t* __restrict__ is_start, int32_t* alive, int32_t* listA, int32_t* listB,
            int32_t* node_batch, int32_t* misc, const int32_t* __restrict__ slen,
            const int32_t* __restrict__ bcnt, int32_t batches_cap, bs_summary* sum) {
  cg::grid_group grid = cg::this_grid();
  __shared__ ChainShared sh;
  const int64_t n = a.n;
  const int32_t n_segs = kinfo[2];
  int r = 0;
  // ---- pointer doubling -------------------------------------------------------------
  while (r + 1 < r_cap && ld_rel_i32(alive + r)) {
    const int32_t* Jr = J + (int64_t)r * n;
    int32_t* Jn = J + (int64_t)(r + 1) * n;
    bool any = false;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x) {
      const int32_t v = Jr[x];
      const int32_t w = v == kEnd ? kEnd : Jr[v];
      Jn[x] = w;
      if (w != kEnd && is_start[x]) any = true;
    }
    if (any) alive[r + 1] = 1;
    grid.sync();
    ++r;
  }
  if (blockIdx.x != 0) return;
  const int tid = threadIdx.x, bt = blockDim.x;
  if (tid == 0) sh.flag = (r + 1 >= r_cap && ld_rel_i32(alive + r)) ? 1 : 0;
  // ---- expansion (block 0): segment starts -> all chain nodes, emission order ----------
  int32_t cnt = 0;
  for (int base = 0; base < n_segs; base += bt) {
    const int s = base + tid;
    int32_t st = 0, en = 0;
    if (s < n_segs) { st = seg_off[s]; en = seg_off[s + 1]; }
    const int f = (s < n_segs) && (st < en);
    int32_t tot;
    const int32_t off = block_excl_scan<int32_t>(f, sh.si, &tot);
    if (f) listA[cnt + off] = st;
    cnt += tot;
  }
  int32_t* cur = listA;
  int32_t* nxt = listB;
  for (int lvl = r - 1; lvl >= 0; --lvl) {
    const int32_t* Jl = J + (int64_t)lvl * n;
    int32_t run = 0;
    for (int base = 0; base < cnt; base += bt) {
      const int i = base + tid;
      int32_t x = 0, y = kEnd;
      if (i < cnt) { x = cur[i]; y = Jl[x]; }
      const int32_t emit = i < cnt ? 1 + (y != kEnd) : 0;
      int32_t tot;
      const int32_t off = block_excl_scan<int32_t>(emit, sh.si, &tot);
      if (i < cnt) {
        nxt[run + off] = x;
        if (y != kEnd) nxt[run + off + 1] = y;
      }
      run += tot;
    }
    int32_t* t = cur; cur = nxt; nxt = t;
    cnt = run;
    __syncthreads();
  }
  // ---- batch ids: a chain node is a batch unless it is a segment's empty tail --------
  int32_t nb = 0;
  for (int base = 0; base < cnt; base += bt) {
    const int i = base + tid;
    int f = 0;
    if (i < cnt) {
      const int64_t c = cur[i];
      const int64_t s = seg_of(seg_off, n_segs, c);
      const int64_t end = seg_off[s + 1];
      const int64_t j0 = first_nonrej(c, end, slen, bcnt, a.S);
      f = (j0 < end) && ((int64_t)slen[j0] <= a.T);
    }
    int32_t tot;
    const int32_t off = block_excl_scan<int32_t>(f, sh.si, &tot);
    if (i < cnt) node_batch[i] = f ? nb + off : -1;
    nb += tot;
  }
  if (tid == 0) {
    misc[64] = cnt;
    misc[65] = r;
    misc[66] = nb;
    misc[68] = cur == listA ? 0 : 1;
    sum->n_batches = nb;
    if (nb > batches_cap) latch_flags(sum, BS_FLAG_BATCH_CAP);
    if (sh.flag) latch_flags(sum, BS_FLAG_BATCH_CAP);  // doubling table exhausted
  }
}

// K5d
__global__ void __launch_bounds__(256)
    k_size_describe(SizeArgs a, const int32_t* __restrict__ kinfo,
                    const int32_t* __restrict__ seg_off,
                    const int32_t* __restrict__ perm, const int32_t* __restrict__ slen,
                    const int32_t* __restrict__ bcnt, const int32_t* __restrict__ J0,
                    const int32_t* __restrict__ listA, const int32_t* __restrict__ listB,
                    const int32_t* __restrict__ node_batch, const int32_t* __restrict__ misc,
                    bs_batch* __restrict__ batches, int32_t batches_cap,
                    int32_t* __restrict__ req_batch, int32_t* __restrict__ req_row,
                    bs_summary* sum) {
  __shared__ int32_t s_i[33];
  __shared__ int64_t s_l[33];
  __shared__ int32_t s_m[32], s_mn[32];
  const int M = misc[64];
  const int32_t n_segs = kinfo[2];
  const int32_t* list = misc[68] ? listB : listA;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  int64_t rej_acc = 0, pend_acc = 0;
  for (int i = blockIdx.x; i < M; i += gridDim.x) {
    const int64_t c = list[i];
    const int32_t b = node_batch[i];
    const int64_t s = seg_of(seg_off, n_segs, c);
    const int64_t send = seg_off[s + 1];
    if (b >= 0) {
      const int32_t nx = J0[c];
      const int64_t e = nx == kEnd ? send : nx;
      int32_t run = 0, mx = 0, mn = 0x7fffffff;
      int64_t tsum = 0;
      for (int64_t base = c; base < e; base += blockDim.x) {
        const int64_t j = base + tid;
        int32_t x = 0;
        bool nr = false;
        if (j < e) { x = slen[j]; nr = (int64_t)x <= a.S; }
        int32_t tot;
        const int32_t off = block_excl_scan<int32_t>(nr, s_i, &tot);
        if (j < e) {
          const int32_t r = perm[j];
          if (nr) { req_batch[r] = b; req_row[r] = run + off; }
          else { req_batch[r] = BS_REQ_REJECTED; req_row[r] = -1; }
        }
        if (nr) { mx = x > mx ? x : mx; mn = x < mn ? x : mn; tsum += x; }
        run += tot;
      }
      // block reductions
      int32_t wm = warp_max(mx);
      int32_t wmn = -warp_max(-mn);
      int64_t ws = warp_sum(tsum);
      if (lane == 0) { s_m[wid] = wm; s_mn[wid] = wmn; s_l[wid] = ws; }
      __syncthreads();
      if (tid == 0) {
        int32_t m = 0, mnv = 0x7fffffff;
        int64_t ssum = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
          m = s_m[w] > m ? s_m[w] : m;
          mnv = s_mn[w] < mnv ? s_mn[w] : mnv;
          ssum += s_l[w];
        }
        if (b < batches_cap) {
          bs_batch B;
          B.segment = (int32_t)s;
          B.start = (int32_t)c;
          B.end = (int32_t)e;
          B.n = run;
          B.max_input_len = m;
          B.pitch = (m + BS_PACK_ALIGN - 1) / BS_PACK_ALIGN * BS_PACK_ALIGN;
          B.token_sum = ssum;
          B.footprint = a.kvpt * (a.padded ? (int64_t)m * run : ssum);
          B.out_offset = 0;
          // waste_ratio (memory_model.py:98-100): (s_max - s_avg) / s_max, float64
          const double s_avg = __ddiv_rn((double)ssum, (double)run);
          double wr = __ddiv_rn(__dsub_rn((double)m, s_avg), (double)m);
          if (mnv < 1) {  // waste_ratio raises ValueError for lengths < 1
            wr = __longlong_as_double(0x7ff8000000000000ll);
            latch_flags(sum, BS_FLAG_NONPOS_LEN);
          }
          B.waste = wr;
          B.reserved = 0;
          batches[b] = B;
        }
        rej_acc += (e - c) - run;
      }
      __syncthreads();
    } else {
      // empty tail: rejected up to the first admissible request, pending after it
      const int64_t j0 = first_nonrej(c, send, slen, bcnt, a.S);
      for (int64_t j = c + tid; j < send; j += blockDim.x) {
        const int32_t r = perm[j];
        req_batch[r] = j < j0 ? BS_REQ_REJECTED : BS_REQ_PENDING;
        req_row[r] = -1;
      }
      if (tid == 0) { rej_acc += j0 - c; pend_acc += send - j0; }
    }
  }
  if (tid == 0) {
    if (rej_acc) add_i64(&sum->n_rejected, rej_acc);
    if (pend_acc) add_i64(&sum->n_pending, pend_acc);
  }
}

// K5e
__global__ void __launch_bounds__(1024)
    k_size_offsets(bs_batch* __restrict__ batches, int32_t batches_cap,
                   const int32_t* __restrict__ misc, bs_summary* sum) {
  __shared__ int64_t s_l[33];
  __shared__ double s_d[32];
  __shared__ int64_t s_a[32], s_p[32], s_pk[32];
  const int nb = min(misc[66], batches_cap);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  int64_t run = 0, adm = 0, pad = 0, peak = 0;
  double ws = 0.0;
  for (int base = 0; base < nb; base += blockDim.x) {
    const int i = base + tid;
    int64_t v = 0;
    if (i < nb) {
      const bs_batch& B = batches[i];
      v = (int64_t)B.n * B.pitch;
      adm += B.token_sum;
      pad += (int64_t)B.n * B.max_input_len;
      peak = B.footprint > peak ? B.footprint : peak;
      ws += B.waste;
    }
    int64_t tot;
    const int64_t off = block_excl_scan<int64_t>(v, s_l, &tot);
    if (i < nb) batches[i].out_offset = run + off;
    run += tot;
  }
  adm = warp_sum(adm);
  pad = warp_sum(pad);
  peak = warp_max(peak);
  ws = warp_sum(ws);
  if (lane == 0) { s_a[wid] = adm; s_p[wid] = pad; s_pk[wid] = peak; s_d[wid] = ws; }
  __syncthreads();
  if (tid == 0) {
    int64_t A = 0, Pd = 0, Pk = 0;
    double Ws = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      A += s_a[w]; Pd += s_p[w]; Pk = s_pk[w] > Pk ? s_pk[w] : Pk; Ws += s_d[w];
    }
    sum->admitted_tokens = A;
    sum->padded_tokens = Pd;
    sum->packed_elems = run;
    sum->peak_footprint = Pk;
    sum->waste_sum = Ws;
  }
}

__global__ void k_fill_pending(int64_t n, int32_t* req_batch, int32_t* req_row, bs_summary* sum) {
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
                        int32_t* req_row, bs_summary* summary, cudaStream_t st) {
  cudaError_t e;
  const int64_t H = p.current_safe - p.pledged;
  if (n == 0) return cudaSuccess;
  if (H <= 0) {  // form_batch returns None before touching the queue (:150-152)
    k_fill_pending<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4LL * ctx->num_sms), 256, 0, st>>>(
        n, req_batch, req_row, summary);
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
  a.pad0 = 0;
  int32_t* misc = ctx->misc;
  e = cudaMemsetAsync(misc, 0, sizeof(int32_t) * 128, st);
  if (e != cudaSuccess) return e;
  const int64_t groups = (n + 31) >> 5;
  const unsigned pb = (unsigned)std::min<int64_t>((groups * 32 + 255) / 256, 8LL * ctx->num_sms);
  k_size_prep<<<pb, 256, 0, st>>>(len, perm, a, ctx->sorted_len, ctx->bmax, ctx->bcnt, ctx->bsum);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const unsigned nbk = (unsigned)std::min<int64_t>((n + 255) / 256, 8LL * ctx->num_sms);
  k_size_next<<<nbk, 256, 0, st>>>(a, ctx->kinfo, seg_off, ctx->sorted_len, ctx->bmax, ctx->bcnt, ctx->bsum,
                                   ctx->J, ctx->is_start, misc);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  {
    int r_cap = ctx->r_cap;
    const int32_t* so = seg_off;
    const int32_t* ki = ctx->kinfo;
    int32_t* J = ctx->J;
    const uint8_t* is_start = ctx->is_start;
    int32_t* alive = misc;
    int32_t *la = ctx->listA, *lb = ctx->listB, *nbp = ctx->node_batch;
    const int32_t* sl = ctx->sorted_len;
    const int32_t* bc = ctx->bcnt;
    int32_t bcap = batches_cap;
    bs_summary* sm = summary;
    void* args[] = {&a, (void*)&ki, (void*)&so, &J, &r_cap, (void*)&is_start, &alive, &la, &lb, &nbp, &misc,
                    (void*)&sl, (void*)&bc, &bcap, &sm};
    e = cudaLaunchCooperativeKernel((void*)k_chain, dim3(ctx->chain_blocks), dim3(512), args, 0,
                                    st);
    if (e != cudaSuccess) return e;
  }
  const unsigned db = (unsigned)(4 * ctx->num_sms);
  k_size_describe<<<db, 256, 0, st>>>(a, ctx->kinfo, seg_off, perm, ctx->sorted_len, ctx->bcnt, ctx->J,
                                      ctx->listA, ctx->listB, ctx->node_batch, misc, batches,
                                      batches_cap, req_batch, req_row, summary);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  k_size_offsets<<<1, 1024, 0, st>>>(batches, batches_cap, misc, summary);
  return cudaGetLastError();
}

}  // namespace bsk

void* bs_chain_kernel_ptr() { return reinterpret_cast<void*>(&bsk::k_chain); }
