// K6 design probe (tools/pack_probe.cu): the C2 pack's data movement on synthetic rows,
// comparing the register stream against a bulk-staged form, standalone.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o pack_probe pack_probe.cu
//   ./pack_probe [n_rows=1000000] [pitch_round=32] [src_align_tokens=32]
//
// Rows: lognormal(5.5, 1.1) lengths capped at 4095 (C2), token store in arrival order
// (rows start every src_align tokens), pack order = lengths ascending (SJF) in batches of
// 698 rows (C2's n_max), pitch = round_up(batch max, pitch_round).  Row descriptor (16 B):
// {src | x << 40, dst | pitch << 40}.  The output is [rows, pitch] int32 + u8 mask, rows
// contiguous, batch after batch.
//
// k_reg   — the library's register stream: a warp copies 32 consecutive rows as one
//           flattened stream of 16-byte vectors (kU per lane in flight), mask as 16-byte
//           words, row lookup by a 5-step shuffle search.
// k_bulk  — the output is cut into chunks of kT tokens; a warp owns kS shared-memory
//           slots; per chunk each row's real tokens arrive by one cp.async.bulk into the
//           slot's image of the chunk (mbarrier completion), the lanes add row tails and
//           padding, write the mask straight from registers, and one cp.async.bulk
//           shared -> global stores the token image.  Bytes in flight per SM are bounded
//           by shared memory, not registers.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <random>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

constexpr uint64_t kLo40 = (1ull << 40) - 1;

__device__ __forceinline__ int4 ld_nc(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_cs(int4* p, int4 v) {
  asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint32_t mask_word(int32_t k) {
  return k >= 4 ? 0x01010101u : (k <= 0 ? 0u : (0x01010101u >> (8 * (4 - k))));
}
__device__ __forceinline__ int4 mask16(int32_t k) {
  return make_int4((int)mask_word(k), (int)mask_word(k - 4), (int)mask_word(k - 8),
                   (int)mask_word(k - 12));
}

// ------------------------------------------------------------------ register stream
template <int kU>
__global__ void __launch_bounds__(256, 4)
    k_reg(const ulonglong2* __restrict__ desc, int64_t n_rows, const int32_t* __restrict__ tokens,
          int32_t pad, int32_t* __restrict__ out, uint8_t* __restrict__ mask) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t g = w * 32 + lane;
  if (w * 32 >= n_rows) return;
  int64_t src = 0, dst = 0;
  int32_t x = 0, pitch = 0;
  if (g < n_rows) {
    const ulonglong2 d = desc[g];
    src = (int64_t)(d.x & kLo40);
    x = (int32_t)(d.x >> 40);
    dst = (int64_t)(d.y & kLo40);
    pitch = (int32_t)(d.y >> 40);
  }
  const int64_t d0 = __shfl_sync(FULL, dst, 0);
  const int32_t rel = (int32_t)(dst - d0);  // element offset of the row in the group
  const int32_t end = __shfl_sync(FULL, g < n_rows ? rel + pitch : 0, 31);
  int32_t tot = end;
  {  // rows past n_rows: the last valid lane's end
    const unsigned vm = __ballot_sync(FULL, g < n_rows);
    const int lastv = 31 - __clz(vm);
    tot = __shfl_sync(FULL, rel + pitch, lastv);
  }
  const int32_t relv = g < n_rows ? rel : 0x7fffffff;
  const int32_t tv = tot >> 2;  // vectors
  int4* o4 = reinterpret_cast<int4*>(out + d0);
  for (int32_t q0 = 0; q0 < tv; q0 += 32 * kU) {
    int4 val[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int32_t q = q0 + u * 32 + lane;
      const int32_t e = 4 * q;
      int j = 0;
#pragma unroll
      for (int s = 16; s >= 1; s >>= 1) {
        const int32_t rj = __shfl_sync(FULL, relv, j + s);
        if (rj <= e) j += s;
      }
      const int64_t s_j = __shfl_sync(FULL, src, j);
      const int32_t x_j = __shfl_sync(FULL, x, j);
      const int32_t r_j = __shfl_sync(FULL, rel, j);
      const int32_t v = (e - r_j) >> 2;
      int4 r = make_int4(pad, pad, pad, pad);
      if (q < tv) {
        const int32_t* sp = tokens + s_j;
        if (4 * v + 4 <= x_j) {
          r = ld_nc(reinterpret_cast<const int4*>(sp) + v);
        } else if (4 * v < x_j) {
          const int rem = x_j - 4 * v;
          r.x = sp[4 * v];
          if (rem > 1) r.y = sp[4 * v + 1];
          if (rem > 2) r.z = sp[4 * v + 2];
        }
      }
      val[u] = r;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int32_t q = q0 + u * 32 + lane;
      if (q < tv) st_cs(o4 + q, val[u]);
    }
  }
  // mask: 16-byte words (pitch % 16 == 0 => a word never straddles rows)
  int4* m4 = reinterpret_cast<int4*>(mask + d0);
  for (int32_t m = lane; m < (tot >> 4); m += 32) {
    const int32_t e = 16 * m;
    int j = 0;
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      const int32_t rj = __shfl_sync(FULL, relv, j + s);
      if (rj <= e) j += s;
    }
    const int32_t x_j = __shfl_sync(FULL, x, j);
    const int32_t r_j = __shfl_sync(FULL, rel, j);
    st_cs(m4 + m, mask16(x_j - (e - r_j)));
  }
}

// ------------------------------------------------------------------ bulk staged
__device__ __forceinline__ uint32_t sptr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sptr(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(sptr(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sptr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra W_%=;\n}\n" ::"r"(sptr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* s, const void* g, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          sptr(s)),
      "l"(g), "r"(bytes), "r"(sptr(b))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* g, const void* s, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(sptr(s)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int kT>
struct Slot {
  int32_t tok[kT];                 // token image of the chunk
  ulonglong2 rows[kT / 16 + 1];    // descriptors of the chunk's rows
  uint16_t mark[kT / 16];          // 1 + local row index of the row starting in each 16-token group
};

template <int kT, int kW, int kS>
__global__ void __launch_bounds__(kW * 32, 1)
    k_bulk(const ulonglong2* __restrict__ desc, const int32_t* __restrict__ chunk_row,
           int64_t n_rows, int64_t total, int64_t n_chunks, const int32_t* __restrict__ tokens,
           int32_t pad, int32_t* __restrict__ out, uint8_t* __restrict__ mask) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[kW][kS];
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  Slot<kT>* slots = reinterpret_cast<Slot<kT>*>(smem) + wib * kS;
  if (lane == 0) {
    for (int s = 0; s < kS; ++s) mbar_init(&bars[wib][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int64_t gw = (int64_t)blockIdx.x * kW + wib;
  const int64_t nw = (int64_t)gridDim.x * kW;

  auto issue = [&](int s, int64_t u) {
    Slot<kT>& S = slots[s];
    const int64_t c0 = u * kT, c1 = min(c0 + kT, total);
    for (int i = lane; i < kT / 32; i += 32) reinterpret_cast<uint32_t*>(S.mark)[i] = 0u;
    __syncwarp();
    const int64_t g0 = chunk_row[u];
    for (int64_t base = g0;; base += 32) {
      const int64_t g = base + lane;
      ulonglong2 d = make_ulonglong2(0, 0);
      if (g < n_rows) d = desc[g];
      const int64_t dst = (int64_t)(d.y & kLo40);
      const int32_t pitch = (int32_t)(d.y >> 40);
      const bool in = g < n_rows && dst < c1;
      uint32_t bytes = 0;
      const int li = (int)(base - g0) + lane;
      if (in) {
        S.rows[li] = d;
        const int64_t lo = max(dst, c0);
        S.mark[(lo - c0) >> 4] = (uint16_t)(li + 1);
        const int64_t src = (int64_t)(d.x & kLo40);
        const int32_t x = (int32_t)(d.x >> 40);
        const int64_t hi = min(dst + x, c1);
        if (hi > lo) bytes = (uint32_t)((hi - lo) & ~3ll) * 4u;
      }
      uint32_t tx = bytes;
#pragma unroll
      for (int o = 16; o; o >>= 1) tx += __shfl_xor_sync(FULL, tx, o);
      if (lane == 0 && tx) mbar_expect(&bars[wib][s], tx);
      __syncwarp();
      if (bytes) {
        const int64_t lo = max(dst, c0);
        bulk_g2s(S.tok + (lo - c0), tokens + (int64_t)(d.x & kLo40) + (lo - dst), bytes, &bars[wib][s]);
      }
      const bool more = __shfl_sync(FULL, in && dst + pitch < c1, 31);
      if (!more) break;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars[wib][s]);
  };

  auto finish = [&](int s, int64_t u, uint32_t parity) {
    Slot<kT>& S = slots[s];
    const int64_t c0 = u * kT, c1 = min(c0 + kT, total);
    mbar_wait(&bars[wib][s], parity);
    constexpr int kG = kT >= 512 ? kT / 512 : 1;  // 16-token groups per lane
    uint16_t mk[kG];
    int run = 0;
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      mk[j] = lane * kG + j < kT / 16 ? S.mark[lane * kG + j] : 0;
      run = max(run, (int)mk[j]);
    }
    int incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl = max(incl, y);
    }
    int carry = __shfl_up_sync(FULL, incl, 1);
    if (lane == 0) carry = 1;
    carry = max(carry, 1);
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      carry = max(carry, (int)mk[j]);
      const int m = lane * kG + j;
      const int64_t p = c0 + 16 * (int64_t)m;
      if (m >= kT / 16 || p >= c1) continue;
      const ulonglong2 d = S.rows[carry - 1];
      const int64_t dst = (int64_t)(d.y & kLo40);
      const int32_t x = (int32_t)(d.x >> 40);
      const int32_t o = (int32_t)(p - dst);
      st_cs(reinterpret_cast<int4*>(mask + p), mask16(x - o));
      const int32_t f4 = x & ~3;
      if (o + 16 > f4) {  // tail / padding vectors of this group
        const int32_t* sp = tokens + (int64_t)(d.x & kLo40);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int32_t q = o + 4 * v;
          if (q + 4 <= f4) continue;
          int4 r = make_int4(pad, pad, pad, pad);
          if (q < x) {
            const int rem = x - q;
            r.x = sp[q];
            if (rem > 1) r.y = sp[q + 1];
            if (rem > 2) r.z = sp[q + 2];
          }
          *reinterpret_cast<int4*>(S.tok + 16 * m + 4 * v) = r;
        }
      }
    }
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      bulk_s2g(out + c0, S.tok, (uint32_t)(c1 - c0) * 4u);
      bulk_commit();
    }
  };

  // chunks of this warp: u_k = gw + k * nw
  int64_t k_issued = 0;
  for (int s = 0; s < kS; ++s) {
    const int64_t u = gw + (int64_t)s * nw;
    if (u < n_chunks) { issue(s, u); ++k_issued; }
  }
  for (int64_t k = 0;; ++k) {
    const int64_t u = gw + k * nw;
    if (u >= n_chunks) break;
    const int s = (int)(k % kS);
    finish(s, u, (uint32_t)((k / kS) & 1));
    // refill this slot with chunk k + kS once its store has read the image
    const int64_t un = gw + (k + kS) * nw;
    if (un < n_chunks) {
      if (lane == 0) bulk_wait_read<0>();
      __syncwarp();
      issue(s, un);
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------------ host
template <typename F>
static float best_ms(F f, int reps = 10) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  CK(cudaGetLastError());
  return best;
}

template <int kT, int kW, int kS>
static void run_bulk(const char* name, const ulonglong2* d_desc, int64_t n_rows, int64_t total,
                     const int32_t* d_tok, int32_t* d_out, uint8_t* d_mask, double bytes,
                     const std::vector<int32_t>& chunk_row_h, int sms, uint64_t ref_sum,
                     uint64_t ref_msum) {
  const int64_t n_chunks = (total + kT - 1) / kT;
  std::vector<int32_t> cr(chunk_row_h.begin(), chunk_row_h.begin() + n_chunks);
  int32_t* d_cr;
  CK(cudaMalloc(&d_cr, n_chunks * 4));
  CK(cudaMemcpy(d_cr, cr.data(), n_chunks * 4, cudaMemcpyHostToDevice));
  const size_t smem = sizeof(Slot<kT>) * kW * kS;
  CK(cudaFuncSetAttribute(k_bulk<kT, kW, kS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bulk<kT, kW, kS>, kW * 32, smem));
  const int grid = sms * std::max(1, per_sm);
  CK(cudaMemset(d_out, 0, total * 4));
  CK(cudaMemset(d_mask, 0, total));
  const float t = best_ms([&] {
    k_bulk<kT, kW, kS><<<grid, kW * 32, smem>>>(d_desc, d_cr, n_rows, total, n_chunks, d_tok, -1,
                                               d_out, d_mask);
  });
  // verify against the reference sums
  std::vector<int32_t> h(total);
  std::vector<uint8_t> hm(total);
  CK(cudaMemcpy(h.data(), d_out, total * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hm.data(), d_mask, total, cudaMemcpyDeviceToHost));
  uint64_t s = 0, ms = 0;
  for (int64_t i = 0; i < total; ++i) { s = s * 1000003ull + (uint32_t)h[i]; ms += hm[i] * (uint64_t)(i % 977 + 1); }
  printf("{\"kernel\": \"%s\", \"T\": %d, \"warps\": %d, \"slots\": %d, \"smem\": %zu, \"ctas_per_sm\": %d, "
         "\"ms\": %.4f, \"gbs\": %.1f, \"ok\": %s}\n",
         name, kT, kW, kS, smem, per_sm, t, bytes / t / 1e6,
         (s == ref_sum && ms == ref_msum) ? "true" : "false");
  CK(cudaFree(d_cr));
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 1000000;
  const int pround = argc > 2 ? atoi(argv[2]) : 32;
  const int salign = argc > 3 ? atoi(argv[3]) : 32;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  std::mt19937_64 rng(1234);
  std::lognormal_distribution<double> ln(5.5, 1.1);
  std::vector<int32_t> len(n);
  for (auto& l : len) l = (int32_t)std::min(4095.0, std::max(1.0, std::round(ln(rng))));
  std::vector<int64_t> off(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) off[i + 1] = off[i] + (len[i] + salign - 1) / salign * salign;
  std::vector<int32_t> tok(off[n]);
  for (int64_t i = 0; i < (int64_t)tok.size(); ++i) tok[i] = (int32_t)((i * 2654435761ull) & 0x7fff);
  std::vector<int64_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return len[a] < len[b]; });
  const int64_t bsz = 698;
  std::vector<ulonglong2> desc(n);
  int64_t dst = 0, sum_len = 0;
  for (int64_t b0 = 0; b0 < n; b0 += bsz) {
    const int64_t b1 = std::min(n, b0 + bsz);
    int32_t mx = 0;
    for (int64_t g = b0; g < b1; ++g) mx = std::max(mx, len[order[g]]);
    const int32_t pitch = (mx + pround - 1) / pround * pround;
    for (int64_t g = b0; g < b1; ++g) {
      const int64_t r = order[g];
      desc[g].x = (uint64_t)off[r] | ((uint64_t)len[r] << 40);
      desc[g].y = (uint64_t)dst | ((uint64_t)pitch << 40);
      dst += pitch;
      sum_len += len[r];
    }
  }
  const int64_t total = dst;
  // host reference image sums
  uint64_t ref_sum = 0, ref_msum = 0;
  {
    int64_t i = 0;
    for (int64_t g = 0; g < n; ++g) {
      const int64_t src = desc[g].x & kLo40;
      const int32_t x = (int32_t)(desc[g].x >> 40), pitch = (int32_t)(desc[g].y >> 40);
      for (int32_t c = 0; c < pitch; ++c, ++i) {
        const int32_t v = c < x ? tok[src + c] : -1;
        ref_sum = ref_sum * 1000003ull + (uint32_t)v;
        ref_msum += (c < x ? 1ull : 0ull) * (uint64_t)(i % 977 + 1);
      }
    }
  }
  // chunk -> first row, for every chunk size used below (chunk_row at the finest grain)
  const double bytes = 4.0 * sum_len + 8.0 * n + 5.0 * total;
  printf("{\"rows\": %lld, \"sum_len\": %lld, \"packed\": %lld, \"pitch_round\": %d, \"bytes\": %.0f}\n",
         (long long)n, (long long)sum_len, (long long)total, pround, bytes);
  ulonglong2* d_desc;
  int32_t *d_tok, *d_out;
  uint8_t* d_mask;
  CK(cudaMalloc(&d_desc, n * 16));
  CK(cudaMalloc(&d_tok, tok.size() * 4));
  CK(cudaMalloc(&d_out, total * 4 + 64));
  CK(cudaMalloc(&d_mask, total + 64));
  CK(cudaMemcpy(d_desc, desc.data(), n * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_tok, tok.data(), tok.size() * 4, cudaMemcpyHostToDevice));
  {
    const int64_t groups = (n + 31) / 32;
    const int grid = (int)((groups + 7) / 8);
    CK(cudaMemset(d_out, 0, total * 4));
    CK(cudaMemset(d_mask, 0, total));
    const float t = best_ms([&] { k_reg<4><<<grid, 256>>>(d_desc, n, d_tok, -1, d_out, d_mask); });
    std::vector<int32_t> h(total);
    std::vector<uint8_t> hm(total);
    CK(cudaMemcpy(h.data(), d_out, total * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hm.data(), d_mask, total, cudaMemcpyDeviceToHost));
    uint64_t s = 0, ms = 0;
    for (int64_t i = 0; i < total; ++i) { s = s * 1000003ull + (uint32_t)h[i]; ms += hm[i] * (uint64_t)(i % 977 + 1); }
    printf("{\"kernel\": \"reg4\", \"ms\": %.4f, \"gbs\": %.1f, \"ok\": %s}\n", t, bytes / t / 1e6,
           (s == ref_sum && ms == ref_msum) ? "true" : "false");
  }
  auto chunk_rows = [&](int64_t T) {
    std::vector<int32_t> cr((total + T - 1) / T + 1);
    for (int64_t g = 0; g < n; ++g) {
      const int64_t d0 = desc[g].y & kLo40, p = (int64_t)(desc[g].y >> 40);
      for (int64_t u = (d0 + T - 1) / T; u * T < d0 + p; ++u) cr[u] = (int32_t)g;
    }
    return cr;
  };
  {
    auto cr = chunk_rows(2048);
    run_bulk<2048, 8, 2>("bulk", d_desc, n, total, d_tok, d_out, d_mask, bytes, cr, sms, ref_sum, ref_msum);
    run_bulk<2048, 16, 1>("bulk", d_desc, n, total, d_tok, d_out, d_mask, bytes, cr, sms, ref_sum, ref_msum);
  }
  {
    auto cr = chunk_rows(1024);
    run_bulk<1024, 16, 2>("bulk", d_desc, n, total, d_tok, d_out, d_mask, bytes, cr, sms, ref_sum, ref_msum);
    run_bulk<1024, 8, 2>("bulk", d_desc, n, total, d_tok, d_out, d_mask, bytes, cr, sms, ref_sum, ref_msum);
    run_bulk<1024, 12, 2>("bulk", d_desc, n, total, d_tok, d_out, d_mask, bytes, cr, sms, ref_sum, ref_msum);
    run_bulk<1024, 32, 1>("bulk", d_desc, n, total, d_tok, d_out, d_mask, bytes, cr, sms, ref_sum, ref_msum);
  }
  {
    auto cr = chunk_rows(512);
    run_bulk<512, 32, 2>("bulk", d_desc, n, total, d_tok, d_out, d_mask, bytes, cr, sms, ref_sum, ref_msum);
    run_bulk<512, 16, 2>("bulk", d_desc, n, total, d_tok, d_out, d_mask, bytes, cr, sms, ref_sum, ref_msum);
    run_bulk<512, 16, 4>("bulk", d_desc, n, total, d_tok, d_out, d_mask, bytes, cr, sms, ref_sum, ref_msum);
    run_bulk<512, 24, 3>("bulk", d_desc, n, total, d_tok, d_out, d_mask, bytes, cr, sms, ref_sum, ref_msum);
    run_bulk<512, 8, 2>("bulk", d_desc, n, total, d_tok, d_out, d_mask, bytes, cr, sms, ref_sum, ref_msum);
  }
  {
    auto cr = chunk_rows(256);
    run_bulk<256, 32, 2>("bulk", d_desc, n, total, d_tok, d_out, d_mask, bytes, cr, sms, ref_sum, ref_msum);
    run_bulk<256, 16, 2>("bulk", d_desc, n, total, d_tok, d_out, d_mask, bytes, cr, sms, ref_sum, ref_msum);
  }
  return 0;
}
