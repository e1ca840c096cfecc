// K6 — gather-pack token ids into padded [n, pitch] int32 tensors + u8 mask.
//
// No reference counterpart (bucketsim never holds token ids); the layout is the
// one the memory model charges: a batch is padded to its max_input_len
// (batch_controller.py:136-139, the PADDED footprint), stored with row pitch
// round_up(max_input_len, 16) (BS_PACK_ALIGN) so every row starts 64-byte aligned; padding carries
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
                  uint8_t* __restrict__ out_mask, int64_t out_cap, bs_summary* sum, int32_t ptok,
                  int32_t reverse) {
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
  const int64_t n_groups = (t1 - t0 + 31) >> 5;
  unsigned fl = 0;
  // groups in reverse (last batch first): batches are emitted shortest rows first, so
  // the groups of the longest rows — the slowest per warp, up to 32 x 2048 tokens — start
  // first and the kernel's tail is made of short-row groups instead of long ones
  for (int64_t vg = w; vg < n_groups; vg += nw) {
    const int64_t gt = t0 + (reverse ? n_groups - 1 - vg : vg) * 32;
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
               bs_summary* sum, int32_t ptok, int32_t reverse) {
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
  const int64_t n_groups = (t1 - t0 + 31) >> 5;
  for (int64_t vg = w; vg < n_groups; vg += nw) {  // reverse order: see k_pack_stream
    const int64_t gt = t0 + (reverse ? n_groups - 1 - vg : vg) * 32;
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
// Bulk-staged pack (default): the packed output of a batch range is one contiguous
// stream (batches back to back, rows back to back), cut here into chunks of kPackChunk
// tokens.  A CTA of kW warps stays resident on its SM (persistent grid, one CTA per SM
// with 16 warps); each warp owns two shared-memory slots and walks its chunks u = warp,
// warp + all_warps, ...  Per chunk:
//   issue   the lanes read the records of the chunk's rows (one coalesced 16-byte record
//           per row, written by K5e for a fused window or by k_pack_rowprep below) into
//           the slot and start one cp.async.bulk global -> shared per row for the row's
//           real 16-byte token vectors inside the chunk, placed at the row's offset in the
//           slot's image of the chunk (completion counted in bytes on the slot's
//           mbarrier), and the row tail (<= 3 tokens) by 4-byte cp.async;
//   finish  once the bytes landed: every lane takes 16-token groups of the chunk (a row
//           starts on a group boundary: pitch % 16 == 0), finds the group's row from the
//           per-group row-start marks (a warp max-scan), completes the tail vector and
//           writes the padding into the image and the group's 16 mask bytes straight to
//           global (st.global.cs.v4); then one cp.async.bulk shared -> global stores the
//           whole token image.
// Bytes in flight per SM are bounded by shared memory (168 KB of slots) instead of by
// registers, with few threads (512 per SM, 64 registers), so the scheduling kernels of
// the windows in flight keep SM room beside it.  C2: 0.676 ms per 1M-request window
// (0.90 of the copy peak on the survey's bytes) against 0.69 ms for the register stream
// (tools/pack_probe.cu explored chunk size, warps and slots).  Rows whose tokens are not
// 16-byte aligned get their vectors from scalar loads in the finish step.
constexpr uint64_t kLo40 = (1ull << 40) - 1;

struct BulkSlot {
  int32_t tok[kPackChunk];                 // token image of the chunk
  ulonglong2 rows[kPackChunk / 16 + 1];    // descriptors of the rows overlapping the chunk
  uint16_t mark[kPackChunk / 16];          // 1 + local index of the row starting in each group
};

struct PackRange {
  int64_t b_begin, b_end, base_off, row_lo, rows, total;
};

// the range [b_begin, b_end) of a pack call: rows, output elements; false if empty
__device__ __forceinline__ bool pack_range(const bs_batch* __restrict__ batches, int64_t b_begin,
                                           int64_t b_end_arg, const bs_summary* sum_in,
                                           int32_t batches_cap, PackRange& r) {
  int64_t b_end = b_end_arg;
  if (b_end < 0) {
    b_end = sum_in->n_batches;
    if (b_end > batches_cap) b_end = batches_cap;
  }
  if (b_begin >= b_end) return false;
  const bs_batch first = batches[b_begin];
  const bs_batch last = batches[b_end - 1];
  r.b_begin = b_begin;
  r.b_end = b_end;
  r.base_off = first.out_offset;
  r.row_lo = first.row_base;
  r.rows = last.row_base + last.n - first.row_base;
  r.total = last.out_offset + (int64_t)last.n * last.pitch - first.out_offset;
  return true;
}

// K6a: one descriptor per packed row of the range, {src | x << 40, dst | pitch << 40}
// (src = token-store offset, x = real tokens, dst = element offset in the range's output),
// and (strided chunk order) chunk_row[u] = the row holding output element u * kPackChunk
__global__ void __launch_bounds__(256)
    k_pack_rowprep(const int32_t* __restrict__ len, const int32_t* __restrict__ perm,
                   const int32_t* __restrict__ rowpos, const int64_t* __restrict__ tok_off,
                   int32_t L, int32_t truncate, const bs_batch* __restrict__ batches,
                   int64_t b_begin, int64_t b_end_arg, const bs_summary* sum_in,
                   int32_t batches_cap, ulonglong2* __restrict__ desc,
                   int32_t* __restrict__ chunk_row, int64_t chunk_cap, bs_summary* sum) {
  pdl_prologue();
  PackRange R;
  if (!pack_range(batches, b_begin, b_end_arg, sum_in, batches_cap, R)) return;
  if (chunk_row && (R.total + kPackChunk - 1) / kPackChunk > chunk_cap) chunk_row = nullptr;
  unsigned fl = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < R.rows; i += stride) {
    const int64_t g = R.row_lo + i;
    int64_t lo = R.b_begin, hi = R.b_end;  // batch of row g: last b with row_base <= g
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (batches[mid].row_base <= g) lo = mid; else hi = mid;
    }
    const bs_batch B = batches[lo];
    const int32_t r = perm[rowpos[g]];
    const int32_t x = eff_len(len[r], L, truncate, fl);
    const int64_t dst = B.out_offset - R.base_off + (g - B.row_base) * (int64_t)B.pitch;
    desc[i] = make_ulonglong2((uint64_t)tok_off[r] | ((uint64_t)x << 40),
                              (uint64_t)dst | ((uint64_t)B.pitch << 40));
    if (chunk_row)  // chunk_row[u] = the row holding element u * kPackChunk
      for (int64_t u = (dst + kPackChunk - 1) / kPackChunk; u * kPackChunk < dst + B.pitch; ++u)
        chunk_row[u] = (int32_t)i;
  }
  if (fl) latch_flags(sum, fl);
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int kW>
__global__ void __launch_bounds__(kW * 32)
    k_pack_bulk(const ulonglong2* __restrict__ desc, const int32_t* __restrict__ chunk_row,
                int64_t chunk_cap, const int32_t* __restrict__ tokens,
                int32_t pad_id, const bs_batch* __restrict__ batches, int64_t b_begin,
                int64_t b_end_arg, const bs_summary* sum_in, int32_t batches_cap,
                int32_t* __restrict__ out_tokens, uint8_t* __restrict__ out_mask, int64_t out_cap,
                bs_summary* sum) {
  pdl_prologue();
  constexpr int kS = 2;  // slots per warp: one chunk in flight while the other finishes
  extern __shared__ __align__(128) uint8_t bulk_smem[];
  __shared__ __align__(8) uint64_t bars[kW][kS];
  constexpr int T = kPackChunk;
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  PackRange R;
  if (!pack_range(batches, b_begin, b_end_arg, sum_in, batches_cap, R)) return;
  const int64_t n_chunks = (R.total + T - 1) / T;
  if (R.total > out_cap || n_chunks > chunk_cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) latch_flags(sum, BS_FLAG_PACK_CAPACITY);
    return;
  }
  // chunk k of this warp is u = warp + k * all_warps, so the warps in flight write
  // neighbouring chunks (DRAM page locality of the output stream); the first row of each
  // chunk comes from chunk_row.  (Contiguous chunk ranges per warp measured 0.83 vs 0.69 ms
  // at C2: 2,368 far-apart write streams.)
  const int64_t nw = (int64_t)gridDim.x * kW;
  const int64_t gw = (int64_t)blockIdx.x * kW + wib;
  const int64_t K = gw < n_chunks ? (n_chunks - gw + nw - 1) / nw : 0;
  if (K == 0) return;
  auto chunk = [&](int64_t k) { return gw + k * nw; };
  BulkSlot* slots = reinterpret_cast<BulkSlot*>(bulk_smem) + wib * kS;
  uint64_t* bar = bars[wib];
  if (lane == 0) {
    for (int s = 0; s < kS; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int64_t n_rows = R.rows;
  auto load_desc = [&](int64_t g) {
    return g >= 0 && g < n_rows ? desc[g] : make_ulonglong2(0, 0);
  };
  // the packed image is written once: its bulk stores evict first, so L2 keeps the row
  // records and the scheduling data of the windows in flight (C4 pack 0.895 vs 0.877 of
  // the copy peak, C2 unchanged; an evict-first hint on the bulk loads too costs C2 3 %)
  uint64_t l2_first;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(l2_first));

  // issue chunk u into slot s from row g0 (d_first = the records of rows g0 + lane): the
  // records into the slot, one bulk copy per row for its 16-byte token vectors inside the
  // chunk, and the row tail (x % 4 tokens, where the row ends inside the chunk) by 4-byte
  // cp.async into the image
  auto issue = [&](int s, int64_t u, int64_t g0, ulonglong2 d_first) {
    BulkSlot& S = slots[s];
    const int64_t c0 = u * T, c1 = min(c0 + T, R.total);
    for (int i = lane; i < T / 32; i += 32) reinterpret_cast<uint32_t*>(S.mark)[i] = 0u;
    __syncwarp();
    int nin = 0;  // rows of the chunk so far (rows of pitch 0 hold no output and are skipped)
    for (int64_t base = g0;; base += 32) {
      const int64_t g = base + lane;
      const ulonglong2 d = base == g0 ? d_first : load_desc(g);
      const int64_t dst = (int64_t)(d.y & kLo40);
      const int32_t pitch = (int32_t)(d.y >> 40);
      const bool reach = g < n_rows && dst < c1;
      const bool in = reach && pitch > 0;
      const unsigned bal = __ballot_sync(FULL, in);
      uint32_t bytes = 0;
      const int64_t lo = max(dst, c0);
      const int32_t* row = tokens + (int64_t)(d.x & kLo40);
      const int32_t* src = row + (lo - dst);
      const bool al = (reinterpret_cast<uintptr_t>(row) & 15) == 0;
      if (in) {
        const int li = nin + __popc(bal & lanemask_lt());
        S.rows[li] = d;
        S.mark[(lo - c0) >> 4] = (uint16_t)(li + 1);
        const int32_t x = (int32_t)(d.x >> 40);
        const int64_t hi = min(dst + x, c1);
        if (hi > lo && al) {
          bytes = (uint32_t)((hi - lo) & ~3ll) * 4u;
          if (hi == dst + x)  // the row ends here: its tail, asynchronously
            for (int32_t e = x & ~3; e < x; ++e)
              asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                               smem_addr(S.tok + (dst + e - c0))),
                           "l"(row + e)
                           : "memory");
        }
      }
      const uint32_t tx = warp_sum(bytes);
      if (lane == 0 && tx)
        asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(
                         smem_addr(&bar[s])),
                     "r"(tx)
                     : "memory");
      __syncwarp();
      if (bytes)
        asm volatile(
            "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                "r"(smem_addr(S.tok + (lo - c0))),
            "l"(src), "r"(bytes), "r"(smem_addr(&bar[s]))
            : "memory");
      nin += __popc(bal);
      if (!__shfl_sync(FULL, reach && dst + pitch < c1, 31)) break;
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&bar[s])) : "memory");
  };

  // finish: wait for the chunk's bytes, add tails / padding / mask, store the image
  auto finish = [&](int s, int64_t u, uint32_t parity) {
    BulkSlot& S = slots[s];
    const int64_t c0 = u * T, c1 = min(c0 + T, R.total);
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_addr(&bar[s])),
        "r"(parity)
        : "memory");
    // this lane's tail copies of the chunk: one cp.async group is committed per chunk in
    // order, so the younger group (chunk u + 1) may stay pending
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    constexpr int kG = T / 16 / 32;  // 16-token groups per lane (contiguous)
    uint16_t mk[kG];
    int run = 0;
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      mk[j] = S.mark[lane * kG + j];
      run = max(run, (int)mk[j]);
    }
    int incl = run;  // warp inclusive max-scan: the row holding each lane's first group
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl = max(incl, y);
    }
    int cur = __shfl_up_sync(FULL, incl, 1);
    cur = lane == 0 ? 1 : max(cur, 1);
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      cur = max(cur, (int)mk[j]);
      const int m = lane * kG + j;
      const int64_t p = c0 + 16 * (int64_t)m;
      if (p >= c1) continue;
      const ulonglong2 d = S.rows[cur - 1];
      const int32_t x = (int32_t)(d.x >> 40);
      const int32_t o = (int32_t)(p - (int64_t)(d.y & kLo40));  // column of the group
      if (out_mask)
        st_stream_v4(reinterpret_cast<int4*>(out_mask + p),
                     make_int4((int)mask_word(x - o), (int)mask_word(x - o - 4),
                               (int)mask_word(x - o - 8), (int)mask_word(x - o - 12)));
      const int32_t* sp = tokens + (int64_t)(d.x & kLo40);
      const bool al = (reinterpret_cast<uintptr_t>(sp) & 15) == 0;
      const int32_t f4 = al ? (x & ~3) : 0;  // columns below f4 arrived by the bulk copy
      if (o + 16 > f4) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int32_t q = o + 4 * v;
          if (q + 4 <= f4) continue;
          int4* slot4 = reinterpret_cast<int4*>(S.tok + 16 * m + 4 * v);
          int4 r4 = make_int4(pad_id, pad_id, pad_id, pad_id);
          if (q < x) {
            if (al) {  // the tail vector: tokens below x arrived by cp.async
              const int4 t = *slot4;
              r4.x = t.x;
              if (q + 1 < x) r4.y = t.y;
              if (q + 2 < x) r4.z = t.z;
            } else {   // a row whose tokens are not 16-byte aligned: scalar loads
              r4.x = sp[q];
              if (q + 1 < x) r4.y = sp[q + 1];
              if (q + 2 < x) r4.z = sp[q + 2];
              if (q + 3 < x) r4.w = sp[q + 3];
            }
          }
          *slot4 = r4;
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(out_tokens + c0),
                   "r"(smem_addr(S.tok)), "r"((uint32_t)(c1 - c0) * 4u), "l"(l2_first)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  };

  auto row_of = [&](int64_t k) -> int64_t {  // first row of chunk k
    return k < K ? (int64_t)chunk_row[chunk(k)] : -1;
  };
  // prologue: both slots in flight.  The first rows of chunks k + 2, k + 3 and the records
  // of chunk k + 2 are loaded an iteration ahead of their use, so the dependent metadata
  // loads (chunk_row -> rowdesc) overlap the finish of chunk k.
  const int64_t g0 = row_of(0);
  issue(0, chunk(0), g0, load_desc(g0 + lane));
  if (K > 1) {
    const int64_t g1 = row_of(1);
    issue(1, chunk(1), g1, load_desc(g1 + lane));
  } else {
    asm volatile("cp.async.commit_group;" ::: "memory");  // keeps one group per chunk
  }
  int64_t nx_g = row_of(2);
  ulonglong2 nx_d = K > 2 ? load_desc(nx_g + lane) : make_ulonglong2(0, 0);
  int64_t nx2_g = row_of(3);
#pragma unroll 1
  for (int64_t k = 0; k < K; ++k) {
    const int s = (int)(k & 1);
    finish(s, chunk(k), (uint32_t)((k >> 1) & 1));
    if (k + 2 < K) {  // refill the slot once its store has read the image
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
      issue(s, chunk(k + 2), nx_g, nx_d);
      nx_g = nx2_g;
      nx2_g = row_of(k + 4);
      nx_d = k + 3 < K ? load_desc(nx_g + lane) : make_ulonglong2(0, 0);
    } else {
      asm volatile("cp.async.commit_group;" ::: "memory");  // (empty) group of chunk k + 2
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int kW>
static size_t bulk_smem() { return sizeof(BulkSlot) * kW * 2; }

template <int kW>
static cudaError_t launch_pack_bulk(bs_ctx* ctx, const int32_t* len, const int32_t* perm,
                                    const int64_t* tok_off, const int32_t* tokens,
                                    const bs_window_params& p, const bs_batch* batches,
                                    int64_t batch_begin, int64_t batch_end, int32_t batches_cap,
                                    int32_t* out_tokens, uint8_t* out_mask, int64_t out_capacity,
                                    bs_summary* summary, cudaStream_t st) {
  const bool ready = ctx->rowdesc_ready && batch_begin == 0 && batch_end < 0;
  ctx->rowdesc_ready = false;
  cudaError_t e;
  if (!ready) {  // records of the range (K5e writes them for a whole window it sized)
    const int64_t rows_ub = ctx->last_n > 0 ? ctx->last_n : ctx->max_n;
    const unsigned pblocks =
        (unsigned)std::max<int64_t>(1, std::min<int64_t>((rows_ub + 255) / 256, 8LL * ctx->num_sms));
    launch_k(ctx, k_pack_rowprep, dim3(pblocks), dim3(256), 0, st, false, len, perm, ctx->rowpos,
             tok_off, p.l_max, p.truncate, batches, batch_begin, batch_end, summary, batches_cap,
             ctx->rowdesc, ctx->chunk_row, ctx->chunk_cap, summary);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++ctx->launches;
  }
  launch_k(ctx, k_pack_bulk<kW>, dim3((unsigned)ctx->pack_bulk_blocks), dim3(kW * 32),
           bulk_smem<kW>(), st, false, ctx->rowdesc, ctx->chunk_row, ctx->chunk_cap,
           tokens, p.pad_id, batches,
           batch_begin, batch_end, summary, batches_cap, out_tokens, out_mask, out_capacity,
           summary);
  ++ctx->launches;
  return cudaGetLastError();
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
  // bulk-staged pack: 16 warps x 2 slots (~168 KB, one CTA per SM) or 8 warps (two per SM)
  const bool w8 = ctx->pack_bulk_warps == 8;
  const size_t bsm = w8 ? bulk_smem<8>() : bulk_smem<16>();
  e = w8 ? cudaFuncSetAttribute(k_pack_bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm)
         : cudaFuncSetAttribute(k_pack_bulk<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm);
  if (e != cudaSuccess) return e;
  per_sm = 0;
  e = w8 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pack_bulk<8>, 8 * 32, bsm)
         : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pack_bulk<16>, 16 * 32, bsm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  ctx->pack_bulk_blocks = per_sm * ctx->num_sms;
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
      summary, ctx->piece_tok, (int32_t)ctx->pack_reverse);
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
      summary, ctx->piece_tok, (int32_t)ctx->pack_reverse);
  ++ctx->launches;
  return cudaGetLastError();
}

// K6 kernel for a pack call: 1 = bulk-staged, 5 = TMA-staged, 21 = register stream.
// Default: the bulk-staged pack (windows in flight: C2 0.724 vs 0.79 ms, C3 12.18 vs
// 12.70 ms, C4 6.33 vs 6.50 ms per window; it leaves SM room for the scheduling kernels
// of the other windows).  BS_PACK_VARIANT forces one.  The bulk-staged pack stores 16-byte
// mask words and whole 16-byte chunk images, so it needs 16-byte aligned outputs.
static int pack_kernel_choice(const bs_ctx* ctx, const bs_window_params& p,
                              const int32_t* out_tokens, const uint8_t* out_mask) {
  const bool bulk_ok =
      ((reinterpret_cast<uintptr_t>(out_tokens) | reinterpret_cast<uintptr_t>(out_mask)) & 15) == 0;
  int v = ctx->pack_variant;
  if (v != 1 && v != 5 && v != 21)
    v = bulk_ok ? 1 : (p.l_max > 16384 ? 5 : 21);
  if (v == 1 && !bulk_ok) v = p.l_max > 16384 ? 5 : 21;
  return v;
}

bool pack_uses_bulk(const bs_ctx* ctx, const bs_window_params& p, const int32_t* out_tokens,
                    const uint8_t* out_mask) {
  return pack_kernel_choice(ctx, p, out_tokens, out_mask) == 1;
}

cudaError_t launch_pack(bs_ctx* ctx, const int32_t* len, const int32_t* perm,
                        const int64_t* tok_off, const int32_t* tokens, const bs_window_params& p,
                        const bs_batch* batches, int64_t batch_begin, int64_t batch_end,
                        int32_t batches_cap, int32_t* out_tokens, uint8_t* out_mask,
                        int64_t out_capacity, bs_summary* summary, cudaStream_t st) {
  // pack_kernel_choice: the bulk-staged kernel whenever both outputs are 16-byte aligned
  // (every config), else the TMA staging kernel for long-context windows or the
  // flattened 128-bit register stream.  ctx->pack_variant (BS_PACK_VARIANT at bs_create)
  // forces one: 1 = bulk, 5 = TMA, 21 = register stream; all are bit-identical.  The
  // K6 launches carry the low launch priority (launch_k) so that the scheduling kernels
  // of the windows in flight get SMs first.  The slower forms measured in rounds 1-2
  // are recorded in DESIGN.md.
  const int v = pack_kernel_choice(ctx, p, out_tokens, out_mask);
  struct PackScope {
    bs_ctx* c;
    explicit PackScope(bs_ctx* x) : c(x) { c->in_pack = true; }
    ~PackScope() { c->in_pack = false; }
  } scope(ctx);
  if (v == 1)
    return ctx->pack_bulk_warps == 8
               ? launch_pack_bulk<8>(ctx, len, perm, tok_off, tokens, p, batches, batch_begin, batch_end,
                                     batches_cap, out_tokens, out_mask, out_capacity, summary, st)
               : launch_pack_bulk<16>(ctx, len, perm, tok_off, tokens, p, batches, batch_begin, batch_end,
                                      batches_cap, out_tokens, out_mask, out_capacity, summary, st);
  if (v == 5)
    return launch_pack_tma(ctx, len, perm, tok_off, tokens, p, batches, batch_begin, batch_end,
                           batches_cap, out_tokens, out_mask, out_capacity, summary, st);
  return launch_pack_stream<4, 4, true>(ctx, len, perm, tok_off, tokens, p, batches, batch_begin,
                                        batch_end, batches_cap, out_tokens, out_mask, out_capacity,
                                        summary, st);
}

}  // namespace bsk
