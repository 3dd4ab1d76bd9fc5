// Microbenchmark: legacy mma.sync throughput on B200 (sm_100a) -- HMMA m16n8k16 (f16 x f16 -> f32)
// vs IMMA m16n8k32 (u8 x s8 -> s32), instructions per clock per SM with 8 independent accumulator
// chains per warp and W warps per SM.  Question: would a fp16 HMMA sign GEMV (no activation
// quantization, 8 tokens per instruction) out-issue the int8 IMMA one at 16 tokens?
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

template <bool HALF>
__global__ void mma_loop(int iters, long long* cycles, float* sink) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float fc[8][4] = {};
  int ic[8][4] = {};
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (HALF) {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(fc[c][0]), "+f"(fc[c][1]), "+f"(fc[c][2]), "+f"(fc[c][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      } else {
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+r"(ic[c][0]), "+r"(ic[c][1]), "+r"(ic[c][2]), "+r"(ic[c][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      }
    }
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int e = 0; e < 4; ++e) s += fc[c][e] + (float)ic[c][e];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

int main() {
  const int iters = 4096;
  long long* cyc;
  float* sink;
  cudaMalloc(&cyc, 148 * 8 * sizeof(long long));
  cudaMalloc(&sink, 148 * 1024 * sizeof(float));
  for (int warps : {4, 8, 16}) {
    for (int half = 0; half < 2; ++half) {
      for (int rep = 0; rep < 2; ++rep) {
        if (half) mma_loop<true><<<148, 32 * warps>>>(iters, cyc, sink);
        else mma_loop<false><<<148, 32 * warps>>>(iters, cyc, sink);
      }
      cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      const double per_sm = (double)iters * 8 * warps / mx;
      printf("%s warps/SM %2d: %.3f mma/clk/SM  (%.0f MAC/clk/SM)\n", half ? "HMMA m16n8k16 f16->f32" : "IMMA m16n8k32 u8.s8 ",
             warps, per_sm, per_sm * (half ? 2048 : 4096));
    }
  }
  return 0;
}
