// K6 — gather-pack token ids into padded [n, pitch] int32 tensors + u8 mask.
//
// No reference counterpart (bucketsim never holds token ids); the layout is the
// one the memory model charges: a batch is padded to its max_input_len
// (batch_controller.py:136-139, the PADDED footprint), stored with row pitch
// round_up(max_input_len, 4) so every row is 16-byte aligned; padding carries
// pad_id and mask 0, so the padding fraction of [n, max_input_len] equals the
// batch's waste_ratio (memory_model.py:92-100).
//
// B200 mapping: purely HBM-bound (read 4*len bytes, write 5*pitch bytes per row).
// Work unit = a piece of <= kPiece tokens of one row (long-context rows split into
// many pieces, so 128k-token rows are spread over many warps).  Groups of 32
// consecutive pieces go round-robin to the warps of the resident grid, so the
// warps in flight touch neighbouring rows (DRAM-page / TLB locality; an equal-
// slice split was measured 3.6x slower).  The lanes fetch the 32 pieces' metadata
// in parallel (batch by binary search, row map -> request -> token offset /
// length), then the warp copies them with 128-bit streaming loads
// (ld.global.nc.L1::no_allocate, 4 in flight per lane) and evict-first 128-bit
// stores (st.global.cs), the mask as 32-bit stores.
#include "ctx.cuh"

namespace bsk {

constexpr int kPackThreads = 256;
constexpr int kPackU = 4;  // vectors per lane per step (128 vectors = 512 tokens per warp)

__device__ __forceinline__ uint32_t mask_word(int32_t k) {
  // bytes 0..3 = 1 for the first k (0..4) entries
  return k >= 4 ? 0x01010101u : (k <= 0 ? 0u : (0x01010101u >> (8 * (4 - k))));
}

// copy columns [4*vb, 4*ve) of one row (x real tokens, pad beyond)
__device__ __forceinline__ void copy_row_range(const int32_t* src, int32_t* dst, uint8_t* mdst,
                                               int32_t x, int32_t vb, int32_t ve, int lane,
                                               int32_t pad_id) {
  const int4 pad4 = make_int4(pad_id, pad_id, pad_id, pad_id);
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
    const int32_t full = x >> 2, rem = x & 3;
    const int4* s4 = reinterpret_cast<const int4*>(src);
    int4* d4 = reinterpret_cast<int4*>(dst);
    uint32_t* m4 = reinterpret_cast<uint32_t*>(mdst);
    for (int32_t v0 = vb + lane; v0 < ve; v0 += 32 * kPackU) {
      int4 t[kPackU];
#pragma unroll
      for (int u = 0; u < kPackU; ++u) {
        const int32_t v = v0 + u * 32;
        t[u] = (v < full && v < ve) ? ld_stream_v4(s4 + v) : pad4;
      }
#pragma unroll
      for (int u = 0; u < kPackU; ++u) {
        const int32_t v = v0 + u * 32;
        if (v < ve) {
          int4 val = t[u];
          if (v == full && rem) {
            val.x = src[4 * v];
            if (rem > 1) val.y = src[4 * v + 1];
            if (rem > 2) val.z = src[4 * v + 2];
          }
          st_stream_v4(d4 + v, val);
          if (m4) st_stream_u32(m4 + v, mask_word(x - 4 * v));
        }
      }
    }
  } else {  // token row not 16-byte aligned: scalar path
    for (int32_t t = 4 * vb + lane; t < 4 * ve; t += 32) {
      dst[t] = t < x ? src[t] : pad_id;
      if (mdst) mdst[t] = t < x ? 1 : 0;
    }
  }
}

__global__ void __launch_bounds__(kPackThreads)
    k_pack(const int32_t* __restrict__ len, const int32_t* __restrict__ perm,
           const int32_t* __restrict__ rowpos, const int64_t* __restrict__ task_base,
           const int64_t* __restrict__ tok_off, const int32_t* __restrict__ tokens, int32_t L,
           int32_t truncate, int32_t pad_id, const bs_batch* __restrict__ batches,
           int64_t b_begin, int64_t b_end_arg, const bs_summary* sum_in, int32_t batches_cap,
           int32_t* __restrict__ out_tokens, uint8_t* __restrict__ out_mask, int64_t out_cap,
           bs_summary* sum) {
  const unsigned FULL = 0xffffffffu;
  int64_t b_end = b_end_arg;
  if (b_end < 0) {
    b_end = sum_in->n_batches;
    if (b_end > batches_cap) b_end = batches_cap;
  }
  if (b_begin >= b_end) return;
  const int64_t base_off = batches[b_begin].out_offset;
  const bs_batch last = batches[b_end - 1];
  if (last.out_offset + (int64_t)last.n * last.pitch - base_off > out_cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) latch_flags(sum, BS_FLAG_PACK_CAPACITY);
    return;
  }
  const int64_t t0 = task_base[b_begin], t1 = task_base[b_end];
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned fl = 0;
  // groups of 32 consecutive tasks, round-robin over warps: concurrently active warps
  // work on neighbouring rows (DRAM-page and TLB locality), every task <= kPiece tokens
  for (int64_t gt = t0 + w * 32; gt < t1; gt += nw * 32) {
    const int64_t t = gt + lane;
    const int32_t* src = nullptr;
    int32_t* dst = nullptr;
    uint8_t* mdst = nullptr;
    int32_t x = 0, vb = 0, ve = 0;
    if (t < t1) {
      int64_t lo = b_begin, hi = b_end;  // batch of task t: last b with task_base[b] <= t
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (task_base[mid] <= t) lo = mid; else hi = mid;
      }
      const bs_batch B = batches[lo];
      const int32_t pieces = (B.pitch + kPiece - 1) / kPiece;
      const int64_t local = t - task_base[lo];
      const int64_t row = local / pieces;
      const int32_t piece = (int32_t)(local - row * pieces);
      const int64_t rstart = (B.out_offset - base_off) + row * (int64_t)B.pitch;
      const int32_t r = perm[rowpos[B.row_base + row]];
      x = eff_len(len[r], L, truncate, fl);
      src = tokens + tok_off[r];
      dst = out_tokens + rstart;
      mdst = out_mask ? out_mask + rstart : nullptr;
      vb = piece * (kPiece / 4);
      const int32_t c1 = (piece + 1) * kPiece < B.pitch ? (piece + 1) * kPiece : B.pitch;
      ve = c1 >> 2;
    }
    const int nv = __popc(__ballot_sync(FULL, t < t1));
    for (int i = 0; i < nv; ++i) {
      const int32_t* s_i = reinterpret_cast<const int32_t*>(
          __shfl_sync(FULL, reinterpret_cast<unsigned long long>(src), i));
      int32_t* d_i = reinterpret_cast<int32_t*>(
          __shfl_sync(FULL, reinterpret_cast<unsigned long long>(dst), i));
      uint8_t* m_i = reinterpret_cast<uint8_t*>(
          __shfl_sync(FULL, reinterpret_cast<unsigned long long>(mdst), i));
      const int32_t x_i = __shfl_sync(FULL, x, i);
      const int32_t vb_i = __shfl_sync(FULL, vb, i);
      const int32_t ve_i = __shfl_sync(FULL, ve, i);
      copy_row_range(s_i, d_i, m_i, x_i, vb_i, ve_i, lane, pad_id);
    }
  }
  if (fl) latch_flags(sum, fl);
}

cudaError_t launch_pack(bs_ctx* ctx, const int32_t* len, const int32_t* perm,
                        const int64_t* tok_off, const int32_t* tokens, const bs_window_params& p,
                        const bs_batch* batches, int64_t batch_begin, int64_t batch_end,
                        int32_t batches_cap, int32_t* out_tokens, uint8_t* out_mask,
                        int64_t out_capacity, bs_summary* summary, cudaStream_t st) {
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pack, kPackThreads, 0);
    if (per_sm < 1) per_sm = 1;
  }
  const unsigned blocks = (unsigned)(per_sm * ctx->num_sms);
  k_pack<<<blocks, kPackThreads, 0, st>>>(len, perm, ctx->rowpos, ctx->task_base, tok_off, tokens,
                                          p.l_max,
                                          p.truncate, p.pad_id, batches, batch_begin, batch_end,
                                          summary, batches_cap, out_tokens, out_mask, out_capacity,
                                          summary);
  ++ctx->launches;
  return cudaGetLastError();
}

}  // namespace bsk
