// common.cuh — shared device helpers for the BucketServe sm_100a kernels.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "bucketserve.h"

namespace bsk {

constexpr int kWarp = 32;
constexpr int32_t kEnd = -1;  // chain terminal: the 2^r-th successor lies past the segment

// 30-bit counts + 2 flag bits in the decoupled-lookback status words
constexpr uint32_t kStatAgg = 1u << 30;
constexpr uint32_t kStatPrefix = 2u << 30;
constexpr uint32_t kStatMask = (1u << 30) - 1;

// Programmatic dependent launch (sm_90+).  The window's kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization (ctx.cuh: launch_k), so a kernel may
// be scheduled while its predecessor on the stream is still running.  Every kernel calls
// pdl_prologue() first: griddepcontrol.wait blocks until the predecessor grid has
// completed and its writes are visible (a no-op for a normal launch) — so completion is
// still transitive along the stream — and launch_dependents lets the successor's CTAs be
// scheduled as soon as every CTA of this grid has started, hiding its launch latency
// behind this grid's run time.
__device__ __forceinline__ void pdl_prologue() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Length seen by the scheduler: pd_sim.py:382-383 truncates len >= L to L-1;
// otherwise BucketSet.assign raises ValueError (bucket_manager.py:112-115).
// Out-of-range values are clamped (so every stage stays in bounds) and latched.
__device__ __forceinline__ int32_t eff_len(int32_t x, int32_t L, int truncate, unsigned& fl) {
  if (x < 0) { fl |= BS_FLAG_LEN_RANGE; return 0; }
  if (x >= L) {
    if (!truncate) fl |= BS_FLAG_LEN_RANGE;
    return L - 1;
  }
  return x;
}
__device__ __forceinline__ int32_t eff_cls(uint32_t c, int32_t C, unsigned& fl) {
  if ((int32_t)c >= C) { fl |= BS_FLAG_CLASS_RANGE; return C - 1; }
  return (int32_t)c;
}

// CPython float floor division (Objects/floatobject.c, _float_div_mod): the operation
// behind `self.token_budget() // mean_len` in current_n_max (batch_controller.py:104)
__device__ __forceinline__ double py_floordiv(double vx, double wx) {
  double mod = fmod(vx, wx);
  double div = __ddiv_rn(__dsub_rn(vx, mod), wx);
  if (mod != 0.0) {
    if ((wx < 0) != (mod < 0)) { mod = __dadd_rn(mod, wx); div = __dsub_rn(div, 1.0); }
  }
  double fd;
  if (div != 0.0) {
    fd = floor(div);
    if (__dsub_rn(div, fd) > 0.5) fd = __dadd_rn(fd, 1.0);
  } else {
    fd = copysign(0.0, __ddiv_rn(vx, wx));
  }
  return fd;
}

__device__ __forceinline__ void latch_flags(bs_summary* s, unsigned fl) {
  if (fl && s) atomicOr(reinterpret_cast<unsigned long long*>(&s->flags), (unsigned long long)fl);
}

__device__ __forceinline__ void add_i64(int64_t* p, int64_t v) {
  atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}
__device__ __forceinline__ void max_i64(int64_t* p, int64_t v) {
  atomicMax(reinterpret_cast<long long*>(p), (long long)v);
}

// relaxed gpu-scope load/store for lookback status words (never cached in L1)
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// streaming 128-bit load (read once) / store (write once, evict first)
__device__ __forceinline__ int4 ld_stream_v4(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream_v4(int4* p, int4 v) {
  asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_stream_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(0xffffffffu, v, o);
    if ((int)lane_id() >= o) v += t;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_incl_max(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(0xffffffffu, v, o);
    if ((int)lane_id() >= o && t > v) v = t;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T t = __shfl_xor_sync(0xffffffffu, v, o);
    v = t > v ? t : v;
  }
  return v;
}

// Block-wide exclusive scan. `scratch` needs 33 elements of T in shared memory.
// Returns the exclusive prefix; *total receives the block sum.  All threads call.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* scratch, T* total) {
  const int lane = lane_id(), wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  T incl = warp_incl_scan(v);
  if (lane == 31) scratch[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    T w = lane < nw ? scratch[lane] : T(0);
    T wi = warp_incl_scan(w);
    if (lane < nw) scratch[lane] = wi - w;
    if (lane == nw - 1) scratch[32] = wi;
  }
  __syncthreads();
  T r = scratch[wid] + incl - v;
  *total = scratch[32];
  __syncthreads();
  return r;
}

// Block-wide exclusive scan of K values per thread with one pair of barriers (instead of
// K separate scans).  `scratch` needs K * 33 elements of T in shared memory.  v[k] is
// replaced by its exclusive prefix; total[k] receives the block sum.  All threads call.
template <int K, typename T>
__device__ __forceinline__ void block_excl_scan_k(T (&v)[K], T (&total)[K], T* scratch) {
  const int lane = lane_id(), wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  T incl[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    incl[k] = warp_incl_scan(v[k]);
    if (lane == 31) scratch[k * 33 + wid] = incl[k];
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      T w = lane < nw ? scratch[k * 33 + lane] : T(0);
      T wi = warp_incl_scan(w);
      if (lane < nw) scratch[k * 33 + lane] = wi - w;
      if (lane == nw - 1) scratch[k * 33 + 32] = wi;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    v[k] = scratch[k * 33 + wid] + incl[k] - v[k];
    total[k] = scratch[k * 33 + 32];
  }
  __syncthreads();
}

}  // namespace bsk
