// Microbenchmark: tcgen05.mma kind::f16 M=128 K=16 at SMALL N (16..256), A from TMEM (TS) or
// shared memory (SS), rotating over R distinct A tiles (4, or 48 = a 12-stage x 4-MMA ring like the
// prefill kernel's small-token tiles), one accumulator, one issuing thread per SM, all 148 SMs.
// Question: is the K loop of the small-token prefill (~620 cycles per 4 MMAs) bound by the MMA when
// its A operand changes every instruction?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2505_11076_b200/csrc umma_small.cu -o umma_small
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace dbf::sm100;

template <int N, bool TS, int R>
__global__ void __launch_bounds__(128, 1) bench(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t done;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 1) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = idesc_f16_f32(128, N);
    // B (activations, N x 16 fp16 per MMA, 128-byte swizzled K-major) from 8 KB boxes; A (SS): 4 KB
    // per MMA tile (128 rows x 16 K) inside 16 KB 64-K blocks
    const uint32_t a_smem = smem_u32(smem), b_smem = smem_u32(smem + 128 * 1024);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int r = i % R, kb = r >> 2, kk = r & 3;
      const uint64_t bd = sdesc_k_sw128(b_smem + (kb % 8) * 8192 + kk * 32);
      if (TS)
        mma_f16_ts(tmem, tmem + 64 + r * 8, bd, idesc, 1);
      else
        mma_f16_ss(tmem, sdesc_k_sw128(a_smem + (kb % 8) * 16384 + kk * 32), bd, idesc, 1);
    }
    mma_commit(&done);
    mbar_wait(&done, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

template <int N, bool TS, int R>
void run() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  const int iters = 4800;
  auto k = bench<N, TS, R>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k<<<148, 128, 200 * 1024>>>(d, iters);
  k<<<148, 128, 200 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("%s N=%-3d A tiles %2d: %s  cycles/mma %6.1f  (math floor %.0f)\n", TS ? "TS" : "SS", N, R,
         cudaGetErrorString(e), avg / iters, 128.0 * N / 256.0);
  cudaFree(d);
}

int main() {
  run<16, true, 4>();
  run<16, true, 48>();
  run<16, false, 4>();
  run<16, false, 48>();
  run<32, true, 48>();
  run<32, false, 48>();
  run<64, true, 48>();
  run<64, false, 48>();
  run<256, true, 4>();
  run<256, true, 48>();
  run<256, false, 48>();
  return 0;
}
