// C1 over peer memory: the global length histogram of a sharded window without a
// host-driven collective (alternative to the NCCL all-reduce).
//
// Every rank owns an exchange buffer — two histogram slots and an epoch flag — that
// the other ranks map through CUDA IPC (on an HGX B200 node: NVLink / NVSwitch peer
// memory).  Per window, on the window's stream, after K1:
//   k_peer_copy   this rank's histogram -> its slot (epoch + 1) & 1
//   k_peer_flag   epoch counter + 1, system-scope fence, flag := epoch (release)
//   k_peer_reduce every CTA waits (acquire, system scope) until all ranks' flags reach
//                 the epoch, then sums the ranks' slots element-wise straight from peer
//                 memory into hist_global (L1-bypassing loads)
// The epoch lives on the device, so the sequence replays inside a CUDA graph.  Two
// slots suffice: a rank can publish epoch e + 2 (reusing slot e & 1) only after its
// reduce of e + 1 saw every peer's flag e + 1, which each peer posts after it finished
// reading epoch e.  A peer that never arrives latches BS_FLAG_PEER_TIMEOUT after ~5 s
// instead of hanging the GPU.
#include "ctx.cuh"

namespace bsk {

namespace {

constexpr int kFlagWords = 64;  // flag region after the two slots: [0] published, [1] counter

__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t* p) {
  int64_t v;
  asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(int64_t* p, int64_t v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

}  // namespace

__global__ void k_peer_copy(const uint32_t* __restrict__ hist, int64_t words, uint32_t* xbuf,
                            int64_t slot_words, const int64_t* flags) {
  pdl_prologue();
  const int64_t e = flags[1] + 1;  // the epoch this window publishes
  uint32_t* slot = xbuf + (e & 1) * slot_words;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words;
       i += (int64_t)gridDim.x * blockDim.x)
    slot[i] = hist[i];
}

__global__ void k_peer_flag(int64_t* flags) {
  pdl_prologue();
  const int64_t e = flags[1] + 1;
  flags[1] = e;
  __threadfence_system();  // the slot written by k_peer_copy is visible system-wide
  st_release_sys(flags, e);
}

__global__ void __launch_bounds__(256)
    k_peer_reduce(uint32_t* const* __restrict__ peers, int world, int64_t words,
                  int64_t slot_words, const int64_t* own_flags, uint32_t* __restrict__ out,
                  bs_summary* sum) {
  pdl_prologue();
  __shared__ int s_ok;
  const int64_t e = own_flags[1];
  const int64_t slot = (e & 1) * slot_words;
  if (threadIdx.x == 0) {
    int ok = 1;
    const uint64_t t0 = global_ns();
    for (int r = 0; r < world; ++r) {
      const int64_t* f = reinterpret_cast<const int64_t*>(peers[r] + 2 * slot_words);
      while (ld_acquire_sys(f) < e) {
        if (global_ns() - t0 > 5000000000ull) { ok = 0; break; }
        __nanosleep(200);
      }
      if (!ok) break;
    }
    s_ok = ok;
    if (!ok) latch_flags(sum, BS_FLAG_PEER_TIMEOUT);
  }
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t acc = 0;
    for (int r = 0; r < world; ++r) acc += __ldcg(peers[r] + slot + i);
    out[i] = acc;
  }
  (void)s_ok;
}

cudaError_t launch_peer_reduce(bs_ctx* ctx, const uint32_t* hist_local, const bs_window_params& p,
                               uint32_t* hist_global, bs_summary* summary, cudaStream_t st) {
  const int64_t words = (int64_t)p.l_max * p.n_classes;
  const int64_t slot_words = (int64_t)ctx->l_cap * ctx->c_max;
  int64_t* flags = reinterpret_cast<int64_t*>(ctx->xbuf + 2 * slot_words);
  const unsigned blocks = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>((words + 255) / 256, 2LL * ctx->num_sms));
  launch_k(ctx, k_peer_copy, dim3(blocks), dim3(256), 0, st, false, hist_local, words, ctx->xbuf, slot_words, flags);
  launch_k(ctx, k_peer_flag, dim3(1), dim3(1), 0, st, false, flags);
  launch_k(ctx, k_peer_reduce, dim3(blocks), dim3(256), 0, st, false, ctx->peer_ptrs, ctx->peer_world, words, slot_words, flags,
                                        hist_global, summary);
  ctx->launches += 3;
  return cudaGetLastError();
}

int peer_flag_words() { return kFlagWords; }

}  // namespace bsk
