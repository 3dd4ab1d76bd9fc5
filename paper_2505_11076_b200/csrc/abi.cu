// Library metadata, layout queries and the north_star "XOR + HADD2" ablation decode kernel.
#include "common.cuh"

namespace dbf {

static thread_local cudaError_t g_last_cuda_error = cudaSuccess;
void set_cuda_error(cudaError_t e) { g_last_cuda_error = e; }

// ---- ablation: y[r] = sum_c s[r,c] x[c] on CUDA cores, batch 1, canonical layout.
// Each lane owns 128 columns (one 16-byte load per row) and keeps its x values in registers as
// half2 pairs (x[32w+i], x[32w+16+i]); the packed word puts the two signs at bits i and 16+i, so
// ONE shift moves both to the fp16 sign positions 15/31, one LOP3 applies them ((~w<<s) & mask ^ x)
// and one HADD2 accumulates.  fp16 partial sums are flushed to fp32 every 32 columns.
template <typename XT>
__global__ void __launch_bounds__(256) xor_matvec_kernel(const uint32_t* __restrict__ words,
                                                         int rows, int cols, int64_t pitch,
                                                         const XT* __restrict__ x,
                                                         float* __restrict__ y) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nslices = blockDim.x >> 5;           // warps per row (each covers 4096 columns)
  const int word0 = (warp * 32 + lane) * 4;       // first of this lane's 4 words
  __half2 xp[4][16];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int c0 = (word0 + q) * 32 + i, c1 = c0 + 16;
      const float v0 = c0 < cols ? to_f32<XT>(x[c0]) : 0.f;
      const float v1 = c1 < cols ? to_f32<XT>(x[c1]) : 0.f;
      xp[q][i] = __floats2half2_rn(v0, v1);
    }
  __shared__ float part[8];
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    float acc = 0.f;
    if (word0 < pitch) {
      const uint4 w4 = *(const uint4*)(words + (int64_t)r * pitch + word0);
      const uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t nw = ~wv[q];  // bit 0 (= -1) must set the fp16 sign bit
        __half2 h = __float2half2_rn(0.f);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint32_t sgn = (nw << (15 - i)) & 0x80008000u;
          uint32_t xv = *(const uint32_t*)&xp[q][i];
          xv ^= sgn;
          h = __hadd2(h, *(const __half2*)&xv);
        }
        const float2 f = __half22float2(h);
        acc += f.x + f.y;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (nslices == 1) {
      if (lane == 0) y[r] = acc;
    } else {
      if (lane == 0) part[warp] = acc;
      __syncthreads();
      if (threadIdx.x == 0) {
        float s = 0.f;
        for (int w = 0; w < nslices; ++w) s += part[w];
        y[r] = s;
      }
      __syncthreads();
    }
  }
}

}  // namespace dbf

using namespace dbf;

extern "C" int dbf_abi_version(void) { return DBF_ABI_VERSION; }

extern "C" const char* dbf_status_string(int status) {
  switch (status) {
    case DBF_OK: return "ok";
    case DBF_ERR_INVALID_ARGUMENT: return "invalid argument";
    case DBF_ERR_SHAPE: return "shape mismatch";
    case DBF_ERR_WORKSPACE: return "workspace too small";
    case DBF_ERR_CUDA: return "CUDA error";
    case DBF_ERR_UNSUPPORTED: return "unsupported configuration";
    default: return "unknown status";
  }
}

extern "C" int dbf_last_cuda_error(void) { return (int)g_last_cuda_error; }
extern "C" const char* dbf_last_cuda_error_string(void) { return cudaGetErrorString(g_last_cuda_error); }

extern "C" int64_t dbf_row_bytes(int64_t cols) { return cols < 0 ? 0 : (cols + 7) / 8; }
extern "C" int64_t dbf_canonical_pitch_words(int64_t cols) { return cols < 1 ? 0 : canonical_pitch(cols); }
extern "C" int64_t dbf_tiled_bytes(int64_t rows, int64_t cols) {
  if (rows < 1 || cols < 1) return 0;
  return row_blocks(rows) * chunks(cols) * kChunkBytes;
}

extern "C" int dbf_sign_matvec_xor(const uint32_t* words, int64_t rows, int64_t cols,
                                   int64_t word_pitch, const void* x, int x_dtype, float* y,
                                   void* stream) {
  if (!words || !x || !y || rows < 1 || cols < 1 || word_pitch < canonical_pitch(cols) ||
      rows > INT32_MAX)
    return DBF_ERR_INVALID_ARGUMENT;
  const int64_t slices = ceil_div(cols, 4096);
  if (slices > 8) return DBF_ERR_UNSUPPORTED;
  const int threads = (int)slices * 32;
  const int grid = (int)std::min<int64_t>(rows, 148 * 16);
  cudaStream_t s = (cudaStream_t)stream;
  if (x_dtype == DBF_F16)
    xor_matvec_kernel<__half><<<grid, threads, 0, s>>>(words, (int)rows, (int)cols, word_pitch,
                                                       (const __half*)x, y);
  else if (x_dtype == DBF_F32)
    xor_matvec_kernel<float><<<grid, threads, 0, s>>>(words, (int)rows, (int)cols, word_pitch,
                                                      (const float*)x, y);
  else
    return DBF_ERR_INVALID_ARGUMENT;
  return check_launch();
}
