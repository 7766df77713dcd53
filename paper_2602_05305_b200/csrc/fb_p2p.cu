// Peer-memory split-KV exchange: the ranks of one node map each
// other's packed (O, LSE) partial buffers through CUDA IPC, so the exchange
// step of the split-KV refresh is a device-side flag handshake followed by
// the K3 merge reading the peers' partials directly over NVLink -- no NCCL
// collective, no staging copy.
//
//   fb_p2p_alloc / fb_p2p_free   device memory (zeroed) + its IPC handle
//   fb_p2p_open / fb_p2p_close   map / unmap a peer's buffer in this process
//   fb_p2p_signal                one thread: system-scope fence, then a
//                                release store of `value` into slot `slot`
//                                of every listed flag array (the peers')
//   fb_p2p_wait                  one warp: acquire-polls n flags until each
//                                is >= value (watchdog: traps after ~4 s)
// Flags only grow (the caller's epoch counter), so they are never reset.
#include "fb_kernels.cuh"
#include "fb_sm100_ptx.cuh"

#include <cstring>
#include <string>

namespace fb {
namespace {

__global__ void p2p_signal_kernel(uint64_t* const* __restrict__ peer_flags, int n, int slot, uint64_t value) {
  ptx::pdl_wait();
  // every write of this stream's earlier kernels (the local K1 partial) is
  // complete at this kernel's start; make it visible at system scope before
  // the peers see the flag
  asm volatile("fence.sc.sys;" ::: "memory");
  for (int p = 0; p < n; ++p) {
    uint64_t* f = peer_flags[p] + slot;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(value) : "memory");
  }
}

__global__ void p2p_wait_kernel(const uint64_t* __restrict__ flags, int n, uint64_t value) {
  ptx::pdl_wait();
  const int i = threadIdx.x;
  if (i < n) {
    uint32_t polls = 0;
    while (true) {
      uint64_t x;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(flags + i) : "memory");
      if (x >= value) break;
      if (++polls == (1u << 26)) __trap();  // a peer that never signals must not hang the GPU
      __nanosleep(64);
    }
  }
  __syncwarp();
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}

}  // namespace
}  // namespace fb

using namespace fb;

int fb_p2p_alloc(size_t bytes, void** ptr, void* handle) {
  if (ptr == nullptr || handle == nullptr || bytes == 0) return fail(FB_ERR_VALUE, "fb_p2p_alloc: bad arguments");
  *ptr = nullptr;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaSuccess) e = cudaMemset(p, 0, bytes);
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    if (p) cudaFree(p);
    return fail(FB_ERR_CUDA, std::string("fb_p2p_alloc: ") + cudaGetErrorString(e));
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == FB_P2P_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle, &h, sizeof(h));
  *ptr = p;
  return FB_OK;
}

int fb_p2p_free(void* ptr) {
  cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? FB_OK : fail(FB_ERR_CUDA, std::string("fb_p2p_free: ") + cudaGetErrorString(e));
}

int fb_p2p_open(const void* handle, void** ptr) {
  if (ptr == nullptr || handle == nullptr) return fail(FB_ERR_VALUE, "fb_p2p_open: bad arguments");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(FB_ERR_CUDA, std::string("fb_p2p_open: ") + cudaGetErrorString(e));
  *ptr = p;
  return FB_OK;
}

int fb_p2p_close(void* ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(ptr);
  return e == cudaSuccess ? FB_OK : fail(FB_ERR_CUDA, std::string("fb_p2p_close: ") + cudaGetErrorString(e));
}

int fb_p2p_signal(uint64_t* const* peer_flags, int n, int slot, uint64_t value, void* stream) {
  if (peer_flags == nullptr || n < 1 || slot < 0) return fail(FB_ERR_VALUE, "fb_p2p_signal: bad arguments");
  launch_pdl(p2p_signal_kernel, dim3(1), dim3(1), 0, reinterpret_cast<cudaStream_t>(stream), peer_flags, n, slot,
             value);
  count_launch();
  return check_launch("p2p_signal_kernel");
}

int fb_p2p_wait(const uint64_t* flags, int n, uint64_t value, void* stream) {
  if (flags == nullptr || n < 1 || n > 32) return fail(FB_ERR_VALUE, "fb_p2p_wait: 1 <= n <= 32 flags");
  launch_pdl(p2p_wait_kernel, dim3(1), dim3(32), 0, reinterpret_cast<cudaStream_t>(stream), flags, n, value);
  count_launch();
  return check_launch("p2p_wait_kernel");
}
