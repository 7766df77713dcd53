// Microbenchmark (diagnostics, not product): HBM read rate of a persistent
// one-CTA-per-SM TMA stream as a function of ring depth and stage size.
// Each CTA streams a contiguous range of 128-row x 128-col bf16 tiles
// (two 64-col 128B-swizzled boxes per tile, like K1's K/V tiles); a consumer
// warp releases each stage as soon as it lands.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2602_05305_b200/csrc tma_stream.cu -o tma_stream -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include "fb_sm100_ptx.cuh"
using namespace fb;

template <int STAGES, int TPS, bool KV = false>  // TPS tiles (32 KB) per stage; KV: tile t from A, t+1 from B
__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm2, long long tiles, int rows_per_slab, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr uint32_t STAGE_BYTES = TPS * 32768;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long per = tiles / TPS;  // stage units
  const long long b = per * blockIdx.x / gridDim.x, e = per * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    ptx::fence_barrier_init();
  }
  __syncthreads();
  if (warp == 0 && lane == 0) {
    const uint64_t pol = ptx::policy_evict_first();
    int j = 0;
    for (long long u = b; u < e; ++u, ++j) {
      const int s = j % STAGES;
      ptx::mbar_wait(&empty[s], ((j / STAGES) & 1) ^ 1);
      ptx::mbar_expect_tx(&full[s], STAGE_BYTES);
      for (int t = 0; t < TPS; ++t) {
        const long long tile = KV ? (u * TPS + t) / 2 : u * TPS + t;
        const int slab = (int)(tile / (rows_per_slab / 128));
        const int row = (int)(tile % (rows_per_slab / 128)) * 128;
        const CUtensorMap* m = (KV && (t & 1)) ? &tm2 : &tm;
        for (int bx = 0; bx < 2; ++bx)
          ptx::tma_load_3d(smem + s * STAGE_BYTES + t * 32768 + bx * 16384, m, &full[s], bx * 64, row, slab, pol);
      }
    }
  } else if (warp == 1 && lane == 0) {
    unsigned long long acc = 0;
    int j = 0;
    for (long long u = b; u < e; ++u, ++j) {
      const int s = j % STAGES;
      ptx::mbar_wait(&full[s], (j / STAGES) & 1);
      acc += smem[s * STAGE_BYTES + 7];
      ptx::mbar_arrive(&empty[s]);
    }
    if (acc == 0xdeadbeef) sink[0] = acc;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return (PFN_cuTensorMapEncodeTiled_v12000)fn;
}

template <int STAGES, int TPS, bool KV = false>
void run(void* buf, int slabs, int rows, int sms, unsigned long long* sink, void* buf2 = nullptr) {
  CUtensorMap tm, tm2;
  cuuint64_t dims[3] = {128, (cuuint64_t)rows, (cuuint64_t)slabs};
  cuuint64_t str[2] = {128 * 2, (cuuint64_t)rows * 128 * 2};
  cuuint32_t box[3] = {64, 128, 1}, es[3] = {1, 1, 1};
  enc()(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  tm2 = tm;
  if (KV) enc()(&tm2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf2, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const size_t smem = STAGES * TPS * 32768 + 2 * STAGES * 8 + 1024;
  auto k = stream_kernel<STAGES, TPS, KV>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const long long tiles = (long long)slabs * rows / 128 * (KV ? 2 : 1);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) k<<<sms, 64, smem>>>(tm, tm2, tiles, rows, sink);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int r = 0; r < reps; ++r) k<<<sms, 64, smem>>>(tm, tm2, tiles, rows, sink);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)tiles * 32768;
  printf("%s stages=%d x %d KB (in flight/SM %d KB): %.1f us/launch, %.0f GB/s  [%s]\n", KV ? "K+V" : "one", STAGES, TPS * 32, STAGES * TPS * 32,
         ms * 1000 / reps, bytes / (ms / reps * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int slabs = 256, rows = 32768;  // 2.15 GB = K1's KV at b=16
  void* buf; cudaMalloc(&buf, (size_t)slabs * rows * 128 * 2);
  cudaMemset(buf, 1, (size_t)slabs * rows * 128 * 2);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  // K1's access pattern: K and V tiles of the same rows from two slabs (half size each)
  void* buf2; cudaMalloc(&buf2, (size_t)slabs * rows * 128 * 2 / 2);
  cudaMemset(buf2, 1, (size_t)slabs * rows * 128 * 2 / 2);
  for (int rep = 0; rep < 2; ++rep) {
    run<3, 2>(buf, slabs, rows, sms, sink);
    run<3, 2, true>(buf, slabs / 2, rows, sms, sink, buf2);
    run<3, 1>(buf, slabs, rows, sms, sink);
  }
  return 0;
}
