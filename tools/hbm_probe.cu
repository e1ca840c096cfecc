// HBM ceiling for K6's traffic mix (tools/hbm_probe.cu; nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a -o hbm_probe hbm_probe.cu).
//
// K6 at C2 reads 1.86 GB (token rows) and writes 2.26 GB (int32 rows + u8 mask rows,
// 4:1), i.e. 45 % reads.  The measured copy peak in MEASURED_PEAKS.json is a 1:1
// read/write copy.  This probe times perfectly contiguous streams with the same
// byte counts and mixes, with the same 128-bit streaming loads / evict-first
// stores as k_pack, so the pack's fraction can be read against the ceiling of
// its own mix:
//   read     read R bytes (xor-reduced, one word stored per CTA)
//   write    write W bytes
//   copy     read N, write N (the MEASURED_PEAKS mix)
//   packmix  read R, write 4/5 W to one stream and 1/5 W to a second stream
// Prints one JSON line per probe: GB/s = bytes moved / best-of-10 kernel time.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

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

constexpr int kU = 4;

template <int kU>
__global__ void k_read(const int4* a, int64_t n, int* out) {
  int acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride * kU) {
    int4 t[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) t[u] = i + u * stride < n ? ld_nc(a + i + u * stride) : int4{};
#pragma unroll
    for (int u = 0; u < kU; ++u) acc ^= t[u].x ^ t[u].y ^ t[u].z ^ t[u].w;
  }
  if (acc == 0x7fffffff) out[blockIdx.x] = acc;
}

__global__ void k_write(int4* a, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    st_cs(a + i, make_int4((int)i, 1, 2, 3));
}

template <int kU>
__global__ void k_copy(const int4* a, int4* b, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride * kU) {
    int4 t[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) t[u] = i + u * stride < n ? ld_nc(a + i + u * stride) : int4{};
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (i + u * stride < n) st_cs(b + i + u * stride, t[u]);
  }
}

// read nr vectors, write nw1 vectors (the first nr copied, the rest padding) to b and
// nw2 = nw1 / 4 vectors to m (the mask stream), all contiguous
template <int kU>
__global__ void k_packmix(const int4* a, int64_t nr, int4* b, int64_t nw1, int4* m, int64_t nw2) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw1; i += stride * kU) {
    int4 t[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t j = i + u * stride;
      t[u] = j < nr ? ld_nc(a + j) : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t j = i + u * stride;
      if (j < nw1) st_cs(b + j, t[u]);
      if ((j & 3) == 0 && (j >> 2) < nw2) st_cs(m + (j >> 2), make_int4(0x01010101, 0x01010101, 0, 0));
    }
  }
}

static void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e));
    exit(1);
  }
}

template <typename F>
static float best_ms(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  check(cudaDeviceSynchronize(), "warmup");
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  check(cudaGetLastError(), "probe");
  return best;
}

int main(int argc, char** argv) {
  // defaults: K6's C2 window (bytes from bench.py's roofline block)
  const double read_b = argc > 1 ? atof(argv[1]) : 1.858e9;
  const double write_b = argc > 2 ? atof(argv[2]) : 2.258e9;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t nr = (int64_t)(read_b / 16);
  const int64_t nw = (int64_t)(write_b / 16);
  const int64_t nw1 = nw * 4 / 5, nw2 = nw - nw1;
  const int64_t ncopy = (int64_t)((read_b + write_b) / 32);
  int4 *a, *b, *m;
  int* out;
  check(cudaMalloc(&a, (size_t)std::max(nr, ncopy) * 16 + (size_t)nw * 16), "malloc a");
  check(cudaMalloc(&b, (size_t)std::max(nw1, ncopy) * 16), "malloc b");
  check(cudaMalloc(&m, (size_t)nw2 * 16 + 16), "malloc m");
  check(cudaMalloc(&out, 1 << 20), "malloc out");
  cudaMemset(a, 1, (size_t)std::max(nr, ncopy) * 16);
  for (int per_sm : {2, 4, 8}) {
    const int grid = sms * per_sm, th = 256;
    float t;
    t = best_ms([&] { k_read<4><<<grid, th>>>(a, nr, out); });
    printf("{\"probe\": \"read\", \"ctas_per_sm\": %d, \"bytes\": %.0f, \"ms\": %.4f, \"gbs\": %.1f}\n",
           per_sm, nr * 16.0, t, nr * 16.0 / t / 1e6);
    t = best_ms([&] { k_read<16><<<grid, th>>>(a, nr, out); });
    printf("{\"probe\": \"read16\", \"ctas_per_sm\": %d, \"bytes\": %.0f, \"ms\": %.4f, \"gbs\": %.1f}\n",
           per_sm, nr * 16.0, t, nr * 16.0 / t / 1e6);
    t = best_ms([&] { k_write<<<grid, th>>>(a, nw); });
    printf("{\"probe\": \"write\", \"ctas_per_sm\": %d, \"bytes\": %.0f, \"ms\": %.4f, \"gbs\": %.1f}\n",
           per_sm, nw * 16.0, t, nw * 16.0 / t / 1e6);
    t = best_ms([&] { k_copy<4><<<grid, th>>>(a, b, ncopy); });
    printf("{\"probe\": \"copy\", \"ctas_per_sm\": %d, \"bytes\": %.0f, \"ms\": %.4f, \"gbs\": %.1f}\n",
           per_sm, ncopy * 32.0, t, ncopy * 32.0 / t / 1e6);
    t = best_ms([&] { k_copy<16><<<grid, th>>>(a, b, ncopy); });
    printf("{\"probe\": \"copy16\", \"ctas_per_sm\": %d, \"bytes\": %.0f, \"ms\": %.4f, \"gbs\": %.1f}\n",
           per_sm, ncopy * 32.0, t, ncopy * 32.0 / t / 1e6);
    t = best_ms([&] { k_packmix<4><<<grid, th>>>(a, nr, b, nw1, m, nw2); });
    printf("{\"probe\": \"packmix\", \"ctas_per_sm\": %d, \"bytes\": %.0f, \"ms\": %.4f, \"gbs\": %.1f}\n",
           per_sm, (nr + nw1 + nw2) * 16.0, t, (nr + nw1 + nw2) * 16.0 / t / 1e6);
    t = best_ms([&] { k_packmix<16><<<grid, th>>>(a, nr, b, nw1, m, nw2); });
    printf("{\"probe\": \"packmix16\", \"ctas_per_sm\": %d, \"bytes\": %.0f, \"ms\": %.4f, \"gbs\": %.1f}\n",
           per_sm, (nr + nw1 + nw2) * 16.0, t, (nr + nw1 + nw2) * 16.0 / t / 1e6);
  }
  return 0;
}
