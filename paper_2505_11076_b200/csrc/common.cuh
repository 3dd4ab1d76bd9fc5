// Shared helpers for the DBF B200 kernels (sm_100a).
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

#include "dbf_b200.h"

namespace dbf {

constexpr int kRowBlock = 16;          // rows per tiled block (MMA M)
constexpr int kChunkCols = 256;        // columns per tiled chunk (8 x MMA K=32)
constexpr int kChunkBytes = 512;       // 16 rows x 256 cols x 1 bit
constexpr int kNumSMs = 148;

// Thread-local record of the last CUDA failure (reported through dbf_last_cuda_error).
void set_cuda_error(cudaError_t e);

inline int check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { set_cuda_error(e); return DBF_ERR_CUDA; }
  return DBF_OK;
}

// Opt a kernel into `bytes` of dynamic shared memory once per DEVICE (the attribute is per device
// context: a process driving two GPUs must set it on each); lock-free, idempotent if raced.
template <auto Kern> inline int ensure_smem_attr(int bytes) {
  static std::atomic<uint64_t> done{0};  // one per kernel (the template argument is the kernel itself)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) { set_cuda_error(e); return DBF_ERR_CUDA; }
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return DBF_OK;
  e = cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) { set_cuda_error(e); return DBF_ERR_CUDA; }
  done.fetch_or(bit, std::memory_order_acq_rel);
  return DBF_OK;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t canonical_pitch(int64_t cols) { return ceil_div(ceil_div(cols, 32), 4) * 4; }
inline int64_t row_blocks(int64_t rows) { return ceil_div(rows, kRowBlock); }
inline int64_t chunks(int64_t cols) { return ceil_div(cols, kChunkCols); }

inline bool valid_float_dtype(int dt) {
  return dt == DBF_F16 || dt == DBF_F32 || dt == DBF_F64 || dt == DBF_BF16;
}
inline size_t dtype_size(int dt) {
  return dt == DBF_F64 ? 8 : (dt == DBF_F32 ? 4 : 2);
}

// ---- typed loads / stores --------------------------------------------------------------
template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<__half>(__half v) { return __half2float(v); }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <> __device__ __forceinline__ float to_f32<double>(double v) { return (float)v; }

template <typename T> __device__ __forceinline__ double to_f64(T v) { return (double)to_f32<T>(v); }
template <> __device__ __forceinline__ double to_f64<double>(double v) { return v; }

template <typename T> __device__ __forceinline__ T from_f64(double v);
template <> __device__ __forceinline__ float from_f64<float>(double v) { return (float)v; }
template <> __device__ __forceinline__ double from_f64<double>(double v) { return v; }
template <> __device__ __forceinline__ __half from_f64<__half>(double v) { return __float2half_rn((float)v); }
template <> __device__ __forceinline__ __nv_bfloat16 from_f64<__nv_bfloat16>(double v) { return __float2bfloat16_rn((float)v); }

// Dispatch helper: calls f(T{}) for the runtime dtype.
template <typename F> inline int dispatch_float(int dt, F&& f) {
  switch (dt) {
    case DBF_F16: return f(__half{});
    case DBF_F32: return f(float{});
    case DBF_F64: return f(double{});
    case DBF_BF16: return f(__nv_bfloat16{});
    default: return DBF_ERR_INVALID_ARGUMENT;
  }
}

}  // namespace dbf
