/* Plain-C client of the C-ABI (include/bucketserve.h): no Python, no torch.
 *
 * Schedules one synthetic window with bs_window_schedule (K1..K7) from device
 * buffers allocated with the CUDA runtime, then checks the invariants a caller relies
 * on: every request is admitted exactly once, batch rows are contiguous per batch, the
 * packed rows hold the request's tokens followed by pad_id, the dispatch order is a
 * permutation of the batches.  Built and run by tests/test_c_abi_example.py (-m gpu):
 *   gcc -O2 -I include tests/c_abi_example.c -L paper_2507_17120_b200/_lib -lbucketserve
 *       -L /usr/local/cuda/lib64 -lcudart -o c_abi_example
 * Exit code 0 = all checks passed. */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "bucketserve.h"

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));    \
      return 2;                                                                     \
    }                                                                               \
  } while (0)
#define BS(x)                                                                       \
  do {                                                                              \
    int rc_ = (x);                                                                  \
    if (rc_ != BS_OK) {                                                             \
      fprintf(stderr, "%s:%d bs status %d: %s\n", __FILE__, __LINE__, rc_,          \
              bs_last_error(ctx));                                                  \
      return 3;                                                                     \
    }                                                                               \
  } while (0)
#define REQUIRE(c)                                                                  \
  do {                                                                              \
    if (!(c)) {                                                                     \
      fprintf(stderr, "%s:%d check failed: %s\n", __FILE__, __LINE__, #c);          \
      return 4;                                                                     \
    }                                                                               \
  } while (0)

static uint32_t lcg(uint32_t* s) { return *s = *s * 1664525u + 1013904223u; }

int main(void) {
  const int64_t n = 50000;
  const int32_t L = 4096, C = 2;
  if (bs_abi_version() != BS_ABI_VERSION) return 5;
  bs_ctx* ctx = NULL;
  BS(bs_create(&ctx, 0, n, L, C));

  /* host inputs: lengths 1..L-1 skewed short, 2 classes, dense 16-byte aligned rows */
  int32_t* len = malloc(sizeof(int32_t) * n);
  uint8_t* cls = malloc(n);
  int64_t* off = malloc(sizeof(int64_t) * (n + 1));
  uint32_t seed = 12345u;
  off[0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    uint32_t r = lcg(&seed) >> 8;
    int32_t x = 1 + (int32_t)((r % 1000u) * (r % 1000u) / 250u);  /* 1 .. ~4000 */
    if (x >= L) x = L - 1;
    len[i] = x;
    cls[i] = (uint8_t)(lcg(&seed) >> 31);
    off[i + 1] = off[i] + (x + 3) / 4 * 4;
  }
  const int64_t ntok = off[n];
  int32_t* tok = malloc(sizeof(int32_t) * ntok);
  for (int64_t t = 0; t < ntok; ++t) tok[t] = (int32_t)(t * 2654435761u % 32000u);

  bs_window_params p;
  memset(&p, 0, sizeof p);
  p.l_max = L;
  p.n_classes = C;
  p.policy[0] = BS_POLICY_FCFS;
  p.policy[1] = BS_POLICY_SJF;
  p.split_threshold = 0.5;
  p.adjust = 1;
  p.kv_bytes_per_token = 524288;
  p.current_safe = (int64_t)160417028505LL;
  p.accounting = BS_ACCOUNTING_PADDED;
  p.truncate = 1;
  p.pad_id = -1;
  p.dispatch = 1;

  /* device buffers */
  int32_t *d_len, *d_tok, *d_edges, *d_changes, *d_bucket, *d_perm, *d_seg, *d_rb, *d_rr,
      *d_out, *d_emit, *d_bemit;
  uint8_t *d_cls, *d_mask;
  int64_t* d_off;
  uint32_t* d_hist;
  bs_batch* d_batches;
  bs_summary* d_sum;
  const int32_t changes_cap = 4 * L + 64;
  const int32_t bcap = (int32_t)n;
  const int64_t out_cap = 256LL * 1024 * 1024;
  CK(cudaMalloc((void**)&d_len, sizeof(int32_t) * n));
  CK(cudaMalloc((void**)&d_cls, n));
  CK(cudaMalloc((void**)&d_off, sizeof(int64_t) * (n + 1)));
  CK(cudaMalloc((void**)&d_tok, sizeof(int32_t) * ntok));
  CK(cudaMalloc((void**)&d_hist, sizeof(uint32_t) * L * C));
  CK(cudaMalloc((void**)&d_edges, sizeof(int32_t) * (L + 1)));
  CK(cudaMalloc((void**)&d_changes, sizeof(int32_t) * 4 * changes_cap));
  CK(cudaMalloc((void**)&d_bucket, sizeof(int32_t) * n));
  CK(cudaMalloc((void**)&d_perm, sizeof(int32_t) * n));
  CK(cudaMalloc((void**)&d_seg, sizeof(int32_t) * (L * C + 1)));
  CK(cudaMalloc((void**)&d_batches, sizeof(bs_batch) * bcap));
  CK(cudaMalloc((void**)&d_rb, sizeof(int32_t) * n));
  CK(cudaMalloc((void**)&d_rr, sizeof(int32_t) * n));
  CK(cudaMalloc((void**)&d_out, sizeof(int32_t) * out_cap));
  CK(cudaMalloc((void**)&d_mask, out_cap));
  CK(cudaMalloc((void**)&d_sum, sizeof(bs_summary)));
  CK(cudaMalloc((void**)&d_emit, sizeof(int32_t) * bcap));
  CK(cudaMalloc((void**)&d_bemit, sizeof(int32_t) * bcap));
  CK(cudaMemcpy(d_len, len, sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_cls, cls, n, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_off, off, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_tok, tok, sizeof(int32_t) * ntok, cudaMemcpyHostToDevice));

  bs_window_io io;
  memset(&io, 0, sizeof io);
  io.len = d_len; io.cls = d_cls; io.tok_off = d_off; io.tokens = d_tok; io.n = n;
  io.changes_cap = changes_cap; io.batches_cap = bcap; io.out_capacity = out_cap;
  io.hist = d_hist; io.edges = d_edges; io.changes = d_changes; io.bucket = d_bucket;
  io.perm = d_perm; io.seg_off = d_seg; io.batches = d_batches; io.req_batch = d_rb;
  io.req_row = d_rr; io.out_tokens = d_out; io.out_mask = d_mask; io.summary = d_sum;
  io.emit_order = d_emit; io.batch_emit = d_bemit;
  BS(bs_window_schedule(ctx, &io, &p, NULL));
  CK(cudaDeviceSynchronize());

  bs_summary s;
  CK(cudaMemcpy(&s, d_sum, sizeof s, cudaMemcpyDeviceToHost));
  if (s.flags != 0)
    fprintf(stderr, "flags %lld total %lld sum_len %lld n_max %lld k %lld\n", (long long)s.flags,
            (long long)s.total_global, (long long)s.sum_len_global, (long long)s.n_max,
            (long long)s.k_buckets);
  REQUIRE(s.flags == 0);
  REQUIRE(s.n_requests == n && s.n_rejected == 0 && s.n_pending == 0);
  REQUIRE(s.n_batches > 0 && s.n_dispatched == s.n_batches);
  REQUIRE(s.packed_elems <= out_cap);
  const int64_t nb = s.n_batches;
  bs_batch* b = malloc(sizeof(bs_batch) * nb);
  int32_t* rb = malloc(sizeof(int32_t) * n);
  int32_t* rr = malloc(sizeof(int32_t) * n);
  int32_t* emit = malloc(sizeof(int32_t) * nb);
  int32_t* out = malloc(sizeof(int32_t) * s.packed_elems);
  uint8_t* mask = malloc(s.packed_elems);
  CK(cudaMemcpy(b, d_batches, sizeof(bs_batch) * nb, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(rb, d_rb, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(rr, d_rr, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(emit, d_emit, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(out, d_out, sizeof(int32_t) * s.packed_elems, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(mask, d_mask, s.packed_elems, cudaMemcpyDeviceToHost));

  /* batches: rows per batch, KV budget, pitch, token sums */
  int64_t rows = 0, admitted = 0;
  for (int64_t k = 0; k < nb; ++k) {
    REQUIRE(b[k].n > 0 && b[k].pitch % BS_PACK_ALIGN == 0 && b[k].pitch >= b[k].max_input_len);
    REQUIRE(b[k].footprint == p.kv_bytes_per_token * (int64_t)b[k].max_input_len * b[k].n);
    REQUIRE(b[k].footprint <= p.current_safe);
    REQUIRE(b[k].row_base == rows);
    rows += b[k].n;
    admitted += b[k].token_sum;
  }
  REQUIRE(rows == n && admitted == s.admitted_tokens);
  /* every request once; its packed row = its tokens then pad_id, mask = 1 then 0 */
  int64_t* seen = calloc(nb, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) {
    REQUIRE(rb[i] >= 0 && rb[i] < nb && rr[i] >= 0 && rr[i] < b[rb[i]].n);
    seen[rb[i]]++;
    const bs_batch* B = &b[rb[i]];
    const int32_t* row = out + B->out_offset + (int64_t)rr[i] * B->pitch;
    const uint8_t* mk = mask + B->out_offset + (int64_t)rr[i] * B->pitch;
    REQUIRE(len[i] <= B->max_input_len);
    for (int32_t t = 0; t < B->pitch; ++t) {
      if (t < len[i]) { REQUIRE(row[t] == tok[off[i] + t]); REQUIRE(mk[t] == 1); }
      else { REQUIRE(row[t] == -1); REQUIRE(mk[t] == 0); }
    }
  }
  for (int64_t k = 0; k < nb; ++k) REQUIRE(seen[k] == b[k].n);
  /* dispatch order: a permutation of the batches, online plans first */
  uint8_t* hit = calloc(nb, 1);
  int offline_seen = 0;
  for (int64_t t = 0; t < nb; ++t) {
    REQUIRE(emit[t] >= 0 && emit[t] < nb && !hit[emit[t]]);
    hit[emit[t]] = 1;
    const int cl = b[emit[t]].segment % C;
    if (cl == 1) offline_seen = 1;
    REQUIRE(!(offline_seen && cl == 0));
  }
  printf("ok: %lld requests, %lld buckets, %lld batches, %lld packed elements\n",
         (long long)n, (long long)s.k_buckets, (long long)nb, (long long)s.packed_elems);
  BS(bs_destroy(ctx));
  return 0;
}
