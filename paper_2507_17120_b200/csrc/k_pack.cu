// K6 — gather-pack token ids into padded [n, pitch] int32 tensors + u8 mask.
//
// No reference counterpart (bucketsim never holds token ids); the layout is the
// one the memory model charges: a batch is padded to its max_input_len
// (batch_controller.py:136-139, the PADDED footprint), stored with row pitch
// round_up(max_input_len, 4) so every row is 16-byte aligned; padding carries
// pad_id and mask 0, so the padding fraction of [n, max_input_len] equals the
// batch's waste_ratio (memory_model.py:92-100).
//
// B200 mapping: purely HBM-bound (read ~4*len bytes, write 5*pitch bytes per
// row).  One warp per request row, rows visited in drain order so the chip's
// writes form one sequential stream; 128-bit streaming loads
// (ld.global.nc.L1::no_allocate) and evict-first 128-bit stores (st.global.cs),
// four vectors in flight per lane; a persistent grid of 8 CTAs/SM x 8 warps.
#include "ctx.cuh"

namespace bsk {

constexpr int kPackThreads = 256;
constexpr int kPackUnroll = 4;

__device__ __forceinline__ uint32_t mask_word(int32_t k) {
  // bytes 0..3 = 1 for the first k (0..4) entries
  return k >= 4 ? 0x01010101u : (k <= 0 ? 0u : (0x01010101u >> (8 * (4 - k))));
}

__global__ void __launch_bounds__(kPackThreads)
    k_pack(const int32_t* __restrict__ len, const int32_t* __restrict__ perm,
           const int32_t* __restrict__ req_batch, const int32_t* __restrict__ req_row,
           const int64_t* __restrict__ tok_off, const int32_t* __restrict__ tokens, int32_t L,
           int32_t truncate, int32_t pad_id, const bs_batch* __restrict__ batches,
           int64_t b_begin, int64_t b_end_arg, const bs_summary* sum_in,
           int32_t batches_cap, int32_t* __restrict__ out_tokens, uint8_t* __restrict__ out_mask,
           int64_t out_cap, bs_summary* sum) {
  int64_t b_end = b_end_arg;
  if (b_end < 0) {
    b_end = sum_in->n_batches;
    if (b_end > batches_cap) b_end = batches_cap;
  }
  if (b_begin >= b_end) return;
  const int64_t base_off = batches[b_begin].out_offset;
  const int64_t p0 = batches[b_begin].start, p1 = batches[b_end - 1].end;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int4 pad4 = make_int4(pad_id, pad_id, pad_id, pad_id);
  unsigned fl = 0;
  for (int64_t j = p0 + gw; j < p1; j += nw) {
    const int32_t r = perm[j];
    const int32_t b = req_batch[r];
    if (b < b_begin || b >= b_end) continue;
    const int32_t pitch = batches[b].pitch;
    const int64_t o = batches[b].out_offset - base_off + (int64_t)req_row[r] * pitch;
    if (o + pitch > out_cap) { fl |= BS_FLAG_PACK_CAPACITY; continue; }
    const int32_t x = eff_len(len[r], L, truncate, fl);
    const int32_t* src = tokens + tok_off[r];
    int32_t* dst = out_tokens + o;
    uint8_t* mdst = out_mask ? out_mask + o : nullptr;
    if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
      const int32_t nv = pitch >> 2, full = x >> 2, rem = x & 3;
      const int4* s4 = reinterpret_cast<const int4*>(src);
      int4* d4 = reinterpret_cast<int4*>(dst);
      uint32_t* m4 = reinterpret_cast<uint32_t*>(mdst);
      for (int32_t v0 = lane; v0 < nv; v0 += 32 * kPackUnroll) {
        int4 t[kPackUnroll];
#pragma unroll
        for (int u = 0; u < kPackUnroll; ++u) {
          const int32_t v = v0 + u * 32;
          t[u] = v < full ? ld_stream_v4(s4 + v) : pad4;
        }
#pragma unroll
        for (int u = 0; u < kPackUnroll; ++u) {
          const int32_t v = v0 + u * 32;
          if (v < nv) {
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
    } else {
      for (int32_t t = lane; t < pitch; t += 32) {
        dst[t] = t < x ? src[t] : pad_id;
        if (mdst) mdst[t] = t < x ? 1 : 0;
      }
    }
  }
  latch_flags(sum, fl);
}

cudaError_t launch_pack(bs_ctx* ctx, const int32_t* len, const int32_t* perm,
                        const int32_t* req_batch, const int32_t* req_row, const int64_t* tok_off,
                        const int32_t* tokens, const bs_window_params& p, const bs_batch* batches,
                        int64_t batch_begin, int64_t batch_end, int32_t batches_cap,
                        int32_t* out_tokens, uint8_t* out_mask, int64_t out_capacity,
                        bs_summary* summary, cudaStream_t st) {
  const unsigned blocks = (unsigned)(8 * ctx->num_sms);
  k_pack<<<blocks, kPackThreads, 0, st>>>(len, perm, req_batch, req_row, tok_off, tokens, p.l_max,
                                          p.truncate, p.pad_id, batches, batch_begin, batch_end,
                                          summary, batches_cap, out_tokens, out_mask, out_capacity,
                                          summary);
  ++ctx->launches;
  return cudaGetLastError();
}

}  // namespace bsk
