// K6 — gather-pack token ids into padded [n, pitch] int32 tensors + u8 mask.
//
// No reference counterpart (bucketsim never holds token ids); the layout is the
// one the memory model charges: a batch is padded to its max_input_len
// (batch_controller.py:136-139, the PADDED footprint), stored with row pitch
// round_up(max_input_len, 32) so every row starts on a 128-byte line; padding carries
// pad_id and mask 0, so the padding fraction of [n, max_input_len] equals the
// batch's waste_ratio (memory_model.py:92-100).
//
// B200 mapping: purely HBM-bound (read 4*len bytes, write 5*pitch bytes per row).
// Work unit = a piece of <= piece_tok tokens of one row (kPiece = 2048 from 64k
// requests up, smaller for small windows; long-context rows split into many pieces,
// so 128k-token rows are spread over many warps).  Groups of 32 consecutive pieces
// go to the warps of a non-persistent grid, so the warps in flight touch
// neighbouring rows (DRAM-page / TLB locality; an equal-slice split was measured
// 3.6x slower).  The lanes fetch the 32 pieces' metadata in parallel (batch by
// binary search, row map -> request -> token offset / length), then the warp copies
// them with 128-bit streaming loads (ld.global.nc.L1::no_allocate, 4 in flight per
// lane) and evict-first 128-bit stores (st.global.cs).  Kernels: k_pack_stream with
// the uniform-group fast path (L <= 16384), k_pack_tma above (launch_pack, bottom).
#include "ctx.cuh"

namespace bsk {

constexpr int kPackThreads = 256;

__device__ __forceinline__ uint32_t mask_word(int32_t k) {
  // bytes 0..3 = 1 for the first k (0..4) entries
  return k >= 4 ? 0x01010101u : (k <= 0 ? 0u : (0x01010101u >> (8 * (4 - k))));
}

// mask bytes of 4-token words [vb, ve) of a row with x real tokens: 16-byte stores on
// the 16-byte-aligned part (rows start 4-byte aligned), 4-byte stores on the ends
__device__ __forceinline__ void store_mask_range(uint8_t* mrow, int32_t x, int32_t vb, int32_t ve,
                                                 int lane) {
  uint32_t* m4 = reinterpret_cast<uint32_t*>(mrow);
  const int32_t head = (int32_t)((4 - (((reinterpret_cast<uintptr_t>(mrow) >> 2) + vb) & 3)) & 3);
  const int32_t a = vb + head < ve ? vb + head : ve;  // first 16-byte-aligned word
  const int32_t nbody = (ve - a) >> 2;
  const int32_t t0 = a + 4 * nbody;                   // tail words [t0, ve)
  if (lane < a - vb) st_stream_u32(m4 + vb + lane, mask_word(x - 4 * (vb + lane)));
  for (int32_t c = lane; c < nbody; c += 32) {
    const int32_t w = a + 4 * c;
    const int32_t k = x - 4 * w;
    st_stream_v4(reinterpret_cast<int4*>(m4 + w),
                 make_int4((int)mask_word(k), (int)mask_word(k - 4), (int)mask_word(k - 8),
                           (int)mask_word(k - 12)));
  }
  if (lane < ve - t0) st_stream_u32(m4 + t0 + lane, mask_word(x - 4 * (t0 + lane)));
}

// copy columns [4*vb, 4*ve) of one row (x real tokens, pad beyond); kU vectors of
// 16 B in flight per lane
template <int kPackU>
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
        }
      }
    }
    if (m4) store_mask_range(mdst, x, vb, ve, lane);
  } else {  // token row not 16-byte aligned: scalar path
    for (int32_t t = 4 * vb + lane; t < 4 * ve; t += 32) {
      dst[t] = t < x ? src[t] : pad_id;
      if (mdst) mdst[t] = t < x ? 1 : 0;
    }
  }
}

// ---------------------------------------------------------------------------------
// Flattened variant: the 16-byte token vectors of the warp's 32 pieces form one
// stream (exclusive scan of the per-piece vector counts), and every iteration moves
// 32 * kU consecutive vectors of that stream, whichever pieces they belong to.  Copying
// row by row, a short row (C2's median is 245 tokens = 62 vectors) leaves most of the
// 4 x 32 vector slots of its iteration empty and every row costs one load round trip;
// here each round trip carries a full 32 * kU * 16 bytes.  A lane finds the piece of
// stream position q by a 5-step binary search over the lanes' scan values (shuffles);
// rows whose source is not 16-byte aligned take copy_row_range's scalar path after
// the stream.  The mask is written per piece.  kUni adds the fast path
// for uniform groups — 32 consecutive one-piece rows of equal pitch, i.e. nearly every
// group inside a batch: their output rows are contiguous, so a vector's row is q / V
// (one multiply, no search), tokens and mask go out as two contiguous streams and only
// the row's source pointer and length are shuffled per vector.
template <int kU, int kMinBlocks, bool kUni>
__global__ void __launch_bounds__(kPackThreads, kMinBlocks)
    k_pack_stream(const int32_t* __restrict__ len, const int32_t* __restrict__ perm,
                  const int32_t* __restrict__ rowpos, const int64_t* __restrict__ task_base,
                  const int64_t* __restrict__ tok_off, const int32_t* __restrict__ tokens,
                  int32_t L, int32_t truncate, int32_t pad_id, const bs_batch* __restrict__ batches,
                  int64_t b_begin, int64_t b_end_arg, const bs_summary* sum_in,
                  int32_t batches_cap, int32_t* __restrict__ out_tokens,
                  uint8_t* __restrict__ out_mask, int64_t out_cap, bs_summary* sum, int32_t ptok) {
  pdl_prologue();
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
  const int4 pad4 = make_int4(pad_id, pad_id, pad_id, pad_id);
  unsigned fl = 0;
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
      const int32_t pieces = (B.pitch + ptok - 1) / ptok;
      const int64_t local = t - task_base[lo];
      const int64_t row = local / pieces;
      const int32_t piece = (int32_t)(local - row * pieces);
      const int64_t rstart = (B.out_offset - base_off) + row * (int64_t)B.pitch;
      const int32_t r = perm[rowpos[B.row_base + row]];
      x = eff_len(len[r], L, truncate, fl);
      src = tokens + tok_off[r];
      dst = out_tokens + rstart;
      mdst = out_mask ? out_mask + rstart : nullptr;
      vb = piece * (ptok / 4);
      const int32_t c1 = (piece + 1) * ptok < B.pitch ? (piece + 1) * ptok : B.pitch;
      ve = c1 >> 2;
    }
    const bool aligned =
        ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
    const int32_t cnt = (t < t1 && aligned) ? ve - vb : 0;
    const int32_t incl = warp_incl_scan(cnt);
    const int32_t pre = incl - cnt;  // stream position of this lane's first vector
    const int32_t total = __shfl_sync(FULL, incl, 31);
    if constexpr (kUni) {
      // uniform group (the common case: 32 consecutive one-piece rows of one batch):
      // the output rows are contiguous, so the token and mask streams are plain
      // contiguous stores and a vector's row is q / V (no search, no dst shuffles)
      const int32_t V0 = __shfl_sync(FULL, ve - vb, 0);
      int32_t* d0 = reinterpret_cast<int32_t*>(
          __shfl_sync(FULL, reinterpret_cast<unsigned long long>(dst), 0));
      uint8_t* m0 = reinterpret_cast<uint8_t*>(
          __shfl_sync(FULL, reinterpret_cast<unsigned long long>(mdst), 0));
      const bool mine =
          t >= t1 || (aligned && vb == 0 && ve == V0 && dst == d0 + (int64_t)lane * 4 * V0 &&
                      mdst == (m0 ? m0 + (int64_t)lane * 4 * V0 : nullptr));
      if (__all_sync(FULL, mine) && V0 > 0 &&
          (reinterpret_cast<uintptr_t>(m0) & 15) == 0) {
        const int nvl = __popc(__ballot_sync(FULL, t < t1));
        const int32_t tot = nvl * V0;
        const float rcp = 1.0f / (float)V0;
        int4* d4 = reinterpret_cast<int4*>(d0);
        for (int32_t q0 = 0; q0 < tot; q0 += 32 * kU) {
          int4 val[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int32_t q = q0 + u * 32 + lane;
            int j = __float2int_rz((float)q * rcp);
            if (j * V0 > q) --j; else if ((j + 1) * V0 <= q) ++j;
            j = j > 31 ? 31 : j;
            const int32_t* s_j = reinterpret_cast<const int32_t*>(
                __shfl_sync(FULL, reinterpret_cast<unsigned long long>(src), j));
            const int32_t x_j = __shfl_sync(FULL, x, j);
            const int32_t v = q - j * V0;
            const int32_t full = x_j >> 2, rem = x_j & 3;
            int4 r = pad4;
            if (q < tot) {
              if (v < full) {
                r = ld_stream_v4(reinterpret_cast<const int4*>(s_j) + v);
              } else if (v == full && rem) {
                r.x = s_j[4 * v];
                if (rem > 1) r.y = s_j[4 * v + 1];
                if (rem > 2) r.z = s_j[4 * v + 2];
              }
            }
            val[u] = r;
          }
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int32_t q = q0 + u * 32 + lane;
            if (q < tot) st_stream_v4(d4 + q, val[u]);
          }
        }
        if (m0) {  // 16-byte mask words (16 columns; rows are 32-byte multiples)
          const int32_t words = tot >> 2;
          int4* mw = reinterpret_cast<int4*>(m0);
          const float rcpw = 4.0f / (float)V0;
          for (int32_t mb = 0; mb < words; mb += 32) {
            const int32_t m = mb + lane;
            int j = __float2int_rz((float)m * rcpw);
            if (j * V0 > 4 * m) --j; else if ((j + 1) * V0 <= 4 * m) ++j;
            j = j > 31 ? 31 : j;
            const int32_t x_j = __shfl_sync(FULL, x, j);
            const int32_t k = x_j - (16 * m - j * 4 * V0);
            if (m < words)
              st_stream_v4(mw + m, make_int4((int)mask_word(k), (int)mask_word(k - 4),
                                             (int)mask_word(k - 8), (int)mask_word(k - 12)));
          }
        }
        continue;
      }
    }
    for (int32_t q0 = 0; q0 < total; q0 += 32 * kU) {
      int4 val[kU];
      int32_t jv[kU];  // (piece lane << 26) | vector in row, -1 past the stream
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int32_t q = q0 + u * 32 + lane;
        // piece of q: the last lane with pre <= q (pre is non-decreasing and a zero-count
        // piece shares its pre with the next lane, so the last such lane has vectors)
        int j = 0;
#pragma unroll
        for (int s = 16; s >= 1; s >>= 1) {
          const int32_t pj = __shfl_sync(FULL, pre, j + s);
          if (pj <= q) j += s;
        }
        const int32_t* s_j = reinterpret_cast<const int32_t*>(
            __shfl_sync(FULL, reinterpret_cast<unsigned long long>(src), j));
        const int32_t x_j = __shfl_sync(FULL, x, j);
        const int32_t v = __shfl_sync(FULL, vb, j) + (q - __shfl_sync(FULL, pre, j));
        jv[u] = q < total ? (j << 26) | v : -1;
        const int32_t full = x_j >> 2, rem = x_j & 3;
        int4 r = pad4;
        if (q < total) {
          if (v < full) {
            r = ld_stream_v4(reinterpret_cast<const int4*>(s_j) + v);
          } else if (v == full && rem) {
            r.x = s_j[4 * v];
            if (rem > 1) r.y = s_j[4 * v + 1];
            if (rem > 2) r.z = s_j[4 * v + 2];
          }
        }
        val[u] = r;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        int4* d_j = reinterpret_cast<int4*>(__shfl_sync(
            FULL, reinterpret_cast<unsigned long long>(dst), jv[u] < 0 ? 0 : jv[u] >> 26));
        if (jv[u] >= 0) st_stream_v4(d_j + (jv[u] & 0x3ffffff), val[u]);
      }
    }
    const int nv = __popc(__ballot_sync(FULL, t < t1));
    for (int i = 0; i < nv; ++i) {
      uint8_t* m_i = reinterpret_cast<uint8_t*>(
          __shfl_sync(FULL, reinterpret_cast<unsigned long long>(mdst), i));
      const int32_t x_i = __shfl_sync(FULL, x, i);
      const int32_t vb_i = __shfl_sync(FULL, vb, i);
      const int32_t ve_i = __shfl_sync(FULL, ve, i);
      if (__shfl_sync(FULL, (int)aligned, i)) {
        if (m_i) store_mask_range(m_i, x_i, vb_i, ve_i, lane);
      } else {
        const int32_t* s_i = reinterpret_cast<const int32_t*>(
            __shfl_sync(FULL, reinterpret_cast<unsigned long long>(src), i));
        int32_t* d_i = reinterpret_cast<int32_t*>(
            __shfl_sync(FULL, reinterpret_cast<unsigned long long>(dst), i));
        copy_row_range<1>(s_i, d_i, m_i, x_i, vb_i, ve_i, lane, pad_id);
      }
    }
  }
  if (fl) latch_flags(sum, fl);
}

// ---------------------------------------------------------------------------------
// TMA variant: the token bytes of each piece are fetched by one elected lane with a
// bulk asynchronous copy (cp.async.bulk global -> shared, completion counted on an
// mbarrier), two 8 KB staging slots per warp, so every warp keeps up to 16 KB of
// reads in flight without spending registers; the lanes then stream the slot out
// with 128-bit stores (+ padding and the u32 mask words).
constexpr int kTmaWarps = 4;
constexpr int kTmaSlots = 2;
constexpr int kTmaSlotBytes = kPiece * 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gsrc, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct PieceMeta {
  const int32_t* src;
  int32_t* dst;
  uint8_t* mdst;
  int32_t x, vb, ve;
};

__global__ void __launch_bounds__(kTmaWarps * 32)
    k_pack_tma(const int32_t* __restrict__ len, const int32_t* __restrict__ perm,
               const int32_t* __restrict__ rowpos, const int64_t* __restrict__ task_base,
               const int64_t* __restrict__ tok_off, const int32_t* __restrict__ tokens, int32_t L,
               int32_t truncate, int32_t pad_id, const bs_batch* __restrict__ batches,
               int64_t b_begin, int64_t b_end_arg, const bs_summary* sum_in, int32_t batches_cap,
               int32_t* __restrict__ out_tokens, uint8_t* __restrict__ out_mask, int64_t out_cap,
               bs_summary* sum, int32_t ptok) {
  pdl_prologue();
  extern __shared__ __align__(128) uint8_t tma_smem[];
  __shared__ __align__(8) uint64_t bars[kTmaWarps][kTmaSlots];
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int4* slots = reinterpret_cast<int4*>(tma_smem + (size_t)wib * kTmaSlots * kTmaSlotBytes);
  if (lane == 0) {
    for (int k = 0; k < kTmaSlots; ++k) mbar_init(&bars[wib][k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
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
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int4 pad4 = make_int4(pad_id, pad_id, pad_id, pad_id);
  uint32_t use[kTmaSlots] = {0, 0};
  unsigned fl = 0;
  for (int64_t gt = t0 + w * 32; gt < t1; gt += nw * 32) {
    const int64_t t = gt + lane;
    PieceMeta my{nullptr, nullptr, nullptr, 0, 0, 0};
    if (t < t1) {
      int64_t lo = b_begin, hi = b_end;
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (task_base[mid] <= t) lo = mid; else hi = mid;
      }
      const bs_batch B = batches[lo];
      const int32_t pieces = (B.pitch + ptok - 1) / ptok;
      const int64_t local = t - task_base[lo];
      const int64_t row = local / pieces;
      const int32_t piece = (int32_t)(local - row * pieces);
      const int64_t rstart = (B.out_offset - base_off) + row * (int64_t)B.pitch;
      const int32_t r = perm[rowpos[B.row_base + row]];
      my.x = eff_len(len[r], L, truncate, fl);
      my.src = tokens + tok_off[r];
      my.dst = out_tokens + rstart;
      my.mdst = out_mask ? out_mask + rstart : nullptr;
      my.vb = piece * (ptok / 4);
      const int32_t c1 = (piece + 1) * ptok < B.pitch ? (piece + 1) * ptok : B.pitch;
      my.ve = c1 >> 2;
    }
    const int nv = __popc(__ballot_sync(FULL, t < t1));
    auto get = [&](int i) {
      PieceMeta m;
      m.src = reinterpret_cast<const int32_t*>(
          __shfl_sync(FULL, reinterpret_cast<unsigned long long>(my.src), i));
      m.dst = reinterpret_cast<int32_t*>(
          __shfl_sync(FULL, reinterpret_cast<unsigned long long>(my.dst), i));
      m.mdst = reinterpret_cast<uint8_t*>(
          __shfl_sync(FULL, reinterpret_cast<unsigned long long>(my.mdst), i));
      m.x = __shfl_sync(FULL, my.x, i);
      m.vb = __shfl_sync(FULL, my.vb, i);
      m.ve = __shfl_sync(FULL, my.ve, i);
      return m;
    };
    // bytes of whole 16-byte vectors of real tokens inside the piece
    auto bulk_vecs = [](const PieceMeta& m) -> int32_t {
      const int32_t full = m.x >> 2;
      const int32_t hi = full < m.ve ? full : m.ve;
      return hi > m.vb ? hi - m.vb : 0;
    };
    auto aligned = [](const PieceMeta& m) {
      return ((reinterpret_cast<uintptr_t>(m.src) | reinterpret_cast<uintptr_t>(m.dst)) & 15) == 0;
    };
    auto issue = [&](const PieceMeta& m, int slot) {
      const int32_t nvec = aligned(m) ? bulk_vecs(m) : 0;
      if (nvec > 0 && lane == 0) {
        mbar_expect_tx(&bars[wib][slot], (uint32_t)nvec * 16u);
        tma_load_1d(slots + slot * (kTmaSlotBytes / 16), m.src + 4 * m.vb, (uint32_t)nvec * 16u,
                    &bars[wib][slot]);
      }
    };
    if (nv == 0) continue;
    PieceMeta cur = get(0);
    issue(cur, 0);
    for (int i = 0; i < nv; ++i) {
      const int slot = i & 1;
      PieceMeta nxt{nullptr, nullptr, nullptr, 0, 0, 0};
      if (i + 1 < nv) {
        nxt = get(i + 1);
        issue(nxt, slot ^ 1);
      }
      if (aligned(cur)) {
        const int32_t nvec = bulk_vecs(cur);
        if (nvec > 0) {
          mbar_wait(&bars[wib][slot], use[slot] & 1u);
          ++use[slot];
        }
        const int32_t full = cur.x >> 2, rem = cur.x & 3;
        const int4* sl = slots + slot * (kTmaSlotBytes / 16);
        int4* d4 = reinterpret_cast<int4*>(cur.dst);
        uint32_t* m4 = reinterpret_cast<uint32_t*>(cur.mdst);
        for (int32_t v = cur.vb + lane; v < cur.ve; v += 32) {
          int4 val = v < full ? sl[v - cur.vb] : pad4;
          if (v == full && rem) {
            val.x = cur.src[4 * v];
            if (rem > 1) val.y = cur.src[4 * v + 1];
            if (rem > 2) val.z = cur.src[4 * v + 2];
          }
          st_stream_v4(d4 + v, val);
          if (m4) st_stream_u32(m4 + v, mask_word(cur.x - 4 * v));
        }
      } else {
        for (int32_t tt = 4 * cur.vb + lane; tt < 4 * cur.ve; tt += 32) {
          cur.dst[tt] = tt < cur.x ? cur.src[tt] : pad_id;
          if (cur.mdst) cur.mdst[tt] = tt < cur.x ? 1 : 0;
        }
      }
      __syncwarp();  // slot fully read before it is refilled
      cur = nxt;
    }
  }
  if (fl) latch_flags(sum, fl);
}

// ---------------------------------------------------------------------------------
// Small windows (K0 path): K0 leaves one copy job per admitted row (source offset,
// destination offset, length, pitch), so the pack is a single dependent load per row
// before its vectors stream — one warp per row, no batch search / row-map walk.
__global__ void __launch_bounds__(256)
    k_pack_rows(const SmallRow* __restrict__ rows, const int32_t* __restrict__ nrows,
                const int32_t* __restrict__ tokens, int32_t pad_id,
                int32_t* __restrict__ out_tokens, uint8_t* __restrict__ out_mask,
                int64_t out_cap, bs_summary* sum) {
  pdl_prologue();
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (sum->packed_elems > out_cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) latch_flags(sum, BS_FLAG_PACK_CAPACITY);
    return;
  }
  const int32_t nr = *nrows;
  for (int64_t r = w; r < nr; r += nw) {
    const SmallRow rw = rows[r];
    copy_row_range<4>(tokens + rw.src, out_tokens + rw.dst, out_mask ? out_mask + rw.dst : nullptr,
                      rw.x, 0, rw.pitch >> 2, lane, pad_id);
  }
}

cudaError_t launch_pack_rows(bs_ctx* ctx, const int32_t* tokens, const bs_window_params& p,
                             int32_t n, int32_t* out_tokens, uint8_t* out_mask,
                             int64_t out_capacity, bs_summary* summary, cudaStream_t st) {
  const unsigned blocks = (unsigned)std::max(1, (n + 7) / 8);  // a warp per row
  launch_k(ctx, k_pack_rows, dim3(blocks), dim3(256), 0, st, false,
           reinterpret_cast<const SmallRow*>(ctx->small_rows), ctx->misc, tokens, p.pad_id,
           out_tokens, out_mask, out_capacity, summary);
  ++ctx->launches;
  return cudaGetLastError();
}

// per-context setup on the context's device (bs_create): the dynamic shared-memory
// opt-in of the TMA kernel and its co-resident CTAs per SM
cudaError_t pack_prepare(bs_ctx* ctx) {
  const int smem = kTmaWarps * kTmaSlots * kTmaSlotBytes;
  cudaError_t e = cudaFuncSetAttribute(k_pack_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pack_tma, kTmaWarps * 32, smem);
  if (e != cudaSuccess) return e;
  ctx->pack_tma_blocks = std::max(1, per_sm) * ctx->num_sms;
  return cudaSuccess;
}

static cudaError_t launch_pack_tma(bs_ctx* ctx, const int32_t* len, const int32_t* perm,
                                   const int64_t* tok_off, const int32_t* tokens,
                                   const bs_window_params& p, const bs_batch* batches,
                                   int64_t batch_begin, int64_t batch_end, int32_t batches_cap,
                                   int32_t* out_tokens, uint8_t* out_mask, int64_t out_capacity,
                                   bs_summary* summary, cudaStream_t st) {
  const size_t smem = (size_t)kTmaWarps * kTmaSlots * kTmaSlotBytes;
  launch_k(ctx, k_pack_tma, dim3((unsigned)ctx->pack_tma_blocks), dim3(kTmaWarps * 32), smem, st, false, 
      len, perm, ctx->rowpos, ctx->task_base, tok_off, tokens, p.l_max, p.truncate, p.pad_id,
      batches, batch_begin, batch_end, summary, batches_cap, out_tokens, out_mask, out_capacity,
      summary, ctx->piece_tok);
  ++ctx->launches;
  return cudaGetLastError();
}

// non-persistent: one 32-piece group per warp (grid from an upper bound on the pieces of
// the last sized window), so CTAs retire as they finish and the scheduling kernels of
// other windows in flight interleave with this pack
template <int kU, int kMinB, bool kUni>
static cudaError_t launch_pack_stream(bs_ctx* ctx, const int32_t* len, const int32_t* perm,
                                      const int64_t* tok_off, const int32_t* tokens,
                                      const bs_window_params& p, const bs_batch* batches,
                                      int64_t batch_begin, int64_t batch_end, int32_t batches_cap,
                                      int32_t* out_tokens, uint8_t* out_mask, int64_t out_capacity,
                                      bs_summary* summary, cudaStream_t st) {
  const int64_t groups = (ctx->pack_pieces + 31) / 32;
  const int64_t blocks = std::max<int64_t>(1, (groups + kPackThreads / 32 - 1) / (kPackThreads / 32));
  launch_k(ctx, k_pack_stream<kU, kMinB, kUni>, dim3((unsigned)blocks), dim3(kPackThreads), 0, st, false, 
      len, perm, ctx->rowpos, ctx->task_base, tok_off, tokens, p.l_max, p.truncate, p.pad_id,
      batches, batch_begin, batch_end, summary, batches_cap, out_tokens, out_mask, out_capacity,
      summary, ctx->piece_tok);
  ++ctx->launches;
  return cudaGetLastError();
}

cudaError_t launch_pack(bs_ctx* ctx, const int32_t* len, const int32_t* perm,
                        const int64_t* tok_off, const int32_t* tokens, const bs_window_params& p,
                        const bs_batch* batches, int64_t batch_begin, int64_t batch_end,
                        int32_t batches_cap, int32_t* out_tokens, uint8_t* out_mask,
                        int64_t out_capacity, bs_summary* summary, cudaStream_t st) {
  // The TMA staging kernel for long-context windows (rows of many KB: C4 at 89-91 % of
  // the copy peak with windows in flight; the register stream packs a C4 window faster
  // alone, 96 %, but fills every SM and slows the windows in flight), the flattened
  // 128-bit register stream with the uniform-group fast path otherwise (C2 758 vs 786
  // us, C3 11.11 vs 11.45 ms against the stream without it).  ctx->pack_variant
  // (BS_PACK_VARIANT at bs_create) forces one: 5 = TMA, 21 = register stream; both are
  // bit-identical.  The slower forms measured in round 1 (per-row k_pack, persistent
  // grids, a cp.async shared-memory ring, 8 vectors per lane) are recorded in DESIGN.md.
  int v = ctx->pack_variant;
  if (v != 5 && v != 21) v = p.l_max > 16384 ? 5 : 21;
  if (v == 5)
    return launch_pack_tma(ctx, len, perm, tok_off, tokens, p, batches, batch_begin, batch_end,
                           batches_cap, out_tokens, out_mask, out_capacity, summary, st);
  return launch_pack_stream<4, 4, true>(ctx, len, perm, tok_off, tokens, p, batches, batch_begin,
                                        batch_end, batches_cap, out_tokens, out_mask, out_capacity,
                                        summary, st);
}

}  // namespace bsk
