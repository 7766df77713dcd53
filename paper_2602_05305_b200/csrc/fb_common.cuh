// Shared device/host helpers for the FlashBlock B200 library.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <math.h>
#include <string>
#include <utility>

#include "../../include/flashblock_b200.h"

namespace fb {

// ---------------------------------------------------------------- errors

void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int check_launch(const char* what);
void count_launch(int n = 1);

// ---------------------------------------------------------------- numerics

template <typename T> struct Num;
template <> struct Num<double> {
  static __device__ __forceinline__ double exp_(double x) { return exp(x); }
  static __device__ __forceinline__ double log_(double x) { return log(x); }
  static __device__ __forceinline__ double ninf() { return -INFINITY; }
};
template <> struct Num<float> {
  static __device__ __forceinline__ float exp_(float x) { return expf(x); }
  static __device__ __forceinline__ float log_(float x) { return logf(x); }
  static __device__ __forceinline__ float ninf() { return -INFINITY; }
};

template <typename To, typename Ti> __device__ __forceinline__ To cvt(Ti x) { return (To)x; }
template <> __device__ __forceinline__ float cvt<float, __nv_bfloat16>(__nv_bfloat16 x) {
  return __bfloat162float(x);
}
template <> __device__ __forceinline__ double cvt<double, __nv_bfloat16>(__nv_bfloat16 x) {
  return (double)__bfloat162float(x);
}
template <> __device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16, float>(float x) {
  return __float2bfloat16_rn(x);
}
template <> __device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16, double>(double x) {
  return __float2bfloat16_rn((float)x);
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

inline int num_sms() {
  static int sms = -1;
  if (sms < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) sms = 148;
  }
  return sms;
}

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Launch with programmatic stream serialization (PDL): the kernel may begin
// while the previous kernel on the stream finishes; kernels launched this way
// call griddepcontrol.wait before reading global inputs.  FB_NO_PDL=1 in the
// environment disables it (diagnostics).
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// launch_pdl with a 1-D thread-block cluster of `cluster` CTAs (0 / 1: none)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                      cudaStream_t st, int cluster, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cluster > 1 ? cluster : 1;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = cluster > 1 ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Precision-mode type bundles (see flashblock_b200.h).
struct ModeF64 { using Tin = double; using Ts = double; using Ta = double; using To = double; using Tl = double; };
struct ModeF32 { using Tin = float; using Ts = float; using Ta = double; using To = float; using Tl = double; };
struct ModeBF16 { using Tin = __nv_bfloat16; using Ts = float; using Ta = float; using To = float; using Tl = float; };
// Sparse-mask scoring modes: lognorm in double; scores double for f64/f32 inputs
// (the reference widens q and k before the product, sparse.py:117-118).
struct ModeMaskF64 { using Tin = double; using Ts = double; using Ta = double; using To = double; using Tl = double; };
struct ModeMaskF32 { using Tin = float; using Ts = double; using Ta = double; using To = double; using Tl = double; };
struct ModeMaskBF16 { using Tin = __nv_bfloat16; using Ts = float; using Ta = double; using To = double; using Tl = double; };

inline size_t dtype_size(int dt) { return dt == FB_F64 ? 8 : dt == FB_F32 ? 4 : 2; }

}  // namespace fb
