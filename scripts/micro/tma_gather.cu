// Microbenchmark (diagnostics, not product): HBM read rate of the K8-style
// gather -- 128-row tiles assembled from 8 random 16-row blocks of a
// [slabs, rows, 128] bf16 cache -- as a function of the TMA box shape:
//   mode 0: two 64-col x 16-row boxes per block (16 ops / 32 KB tile, K1 today)
//   mode 1: one 4-D box {64 cols, 8 rows, 2 halves, 2 atoms} per block (8 ops)
//   mode 2: dense: two 64-col x 128-row boxes per tile at a random 128-row offset
// One CTA per SM, 3-stage ring of 64 KB (K + V-sized: two tiles per stage).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2602_05305_b200/csrc tma_gather.cu -o tma_gather -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "fb_sm100_ptx.cuh"
using namespace fb;

__device__ __forceinline__ void tma_load_4d_raw(void* dst, const void* tmap, uint64_t* bar, int c0, int c1, int c2,
                                                int c3, uint64_t policy) {
  ptx::tma_load_4d(dst, tmap, bar, c0, c1, c2, c3, policy);
}

template <int MODE>
__global__ void __launch_bounds__(64, 1) gather_kernel(const __grid_constant__ CUtensorMap tm, const int* blocks,
                                                       int tiles_per_cta, int slabs, int nblk, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int STAGES = 3;
  constexpr uint32_t STAGE_BYTES = 65536;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    ptx::fence_barrier_init();
  }
  __syncthreads();
  const int* my = blocks + (long long)blockIdx.x * tiles_per_cta * 16;  // 16 blocks (K + V tile) per stage
  if (warp == 0 && lane == 0) {
    const uint64_t pol = ptx::policy_evict_first();
    for (int j = 0; j < tiles_per_cta; ++j) {
      const int s = j % STAGES;
      ptx::mbar_wait(&empty[s], ((j / STAGES) & 1) ^ 1);
      ptx::mbar_expect_tx(&full[s], STAGE_BYTES);
      unsigned char* dst = smem + s * STAGE_BYTES;
      for (int t = 0; t < 2; ++t) {  // K-like and V-like tile
        if (MODE == 2) {
          const int b0 = my[j * 16 + t * 8];
          const int slab = b0 % slabs, row = ((b0 / slabs) * 16) & ~127;
          for (int bx = 0; bx < 2; ++bx)
            ptx::tma_load_3d(dst + t * 32768 + bx * 16384, &tm, &full[s], bx * 64, row, slab, pol);
        } else {
          for (int i = 0; i < 8; ++i) {
            const int b = my[j * 16 + t * 8 + i];
            const int slab = b % slabs, row = (b / slabs) * 16;
            if (MODE == 0) {
              for (int bx = 0; bx < 2; ++bx)
                ptx::tma_load_3d(dst + t * 32768 + bx * 16384 + i * 2048, &tm, &full[s], bx * 64, row, slab, pol);
            } else {
              tma_load_4d_raw(dst + t * 32768 + i * 4096, &tm, &full[s], 0, 0, 0, (slab * (nblk * 2)) + row / 8, pol);
            }
          }
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    unsigned long long acc = 0;
    for (int j = 0; j < tiles_per_cta; ++j) {
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

template <int MODE>
void run(void* buf, int slabs, int rows, int sms, int tiles_per_cta, const int* dblocks, unsigned long long* sink) {
  CUtensorMap tm;
  CUresult r;
  if (MODE == 1) {  // {64 cols, 8 rows, 2 halves, atoms over all slabs}
    cuuint64_t dims[4] = {64, 8, 2, (cuuint64_t)slabs * rows / 8};
    cuuint64_t str[3] = {256, 128, 2048};
    cuuint32_t box[4] = {64, 8, 2, 2}, es[4] = {1, 1, 1, 1};
    r = enc()(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[3] = {128, (cuuint64_t)rows, (cuuint64_t)slabs};
    cuuint64_t str[2] = {256, (cuuint64_t)rows * 256};
    cuuint32_t box[3] = {64, MODE == 2 ? 128u : 16u, 1}, es[3] = {1, 1, 1};
    r = enc()(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return; }
  const size_t smem = 3 * 65536 + 64 + 1024;
  auto k = gather_kernel<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) k<<<sms, 64, smem>>>(tm, dblocks, tiles_per_cta, slabs, rows / 16, sink);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int i = 0; i < reps; ++i) k<<<sms, 64, smem>>>(tm, dblocks, tiles_per_cta, slabs, rows / 16, sink);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)sms * tiles_per_cta * 65536;
  printf("mode %d (%s): tiles/CTA %d: %.1f us/launch, %.0f GB/s  [%s]\n", MODE,
         MODE == 0 ? "2 boxes per 16-row block" : MODE == 1 ? "one 4-D box per block" : "dense 128-row boxes",
         tiles_per_cta, ms * 1000 / reps, bytes / (ms / reps * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int slabs = 32, rows = 65536;  // C4 b=4: 32 kv slabs of 64K rows (537 MB)
  void* buf; cudaMalloc(&buf, (size_t)slabs * rows * 128 * 2);
  cudaMemset(buf, 1, (size_t)slabs * rows * 128 * 2);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  for (int tpc : {6, 12, 24}) {
    const size_t n = (size_t)sms * tpc * 16;
    std::vector<int> h(n);
    srand(7);
    for (auto& x : h) x = rand() % (slabs * (rows / 16));  // block id = slab + slabs * block-in-slab
    int* d; cudaMalloc(&d, n * 4); cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 2; ++rep) {
      run<0>(buf, slabs, rows, sms, tpc, d, sink);
      run<1>(buf, slabs, rows, sms, tpc, d, sink);
      run<2>(buf, slabs, rows, sms, tpc, d, sink);
    }
    cudaFree(d);
  }
  return 0;
}
