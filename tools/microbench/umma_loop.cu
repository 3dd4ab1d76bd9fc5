// Microbenchmark: the prefill MMA issue loop in isolation (B200).  One issuing thread per SM, 148
// CTAs; per "K block" 4 x tcgen05.mma.kind::f16 M128 K16 (A from TMEM, rotating over 8 slots like
// the prefill's A ring; B from 128B-swizzled smem boxes), followed by C commits to mbarriers and an
// optional tcgen05.fence::after_thread_sync.  Reports cycles per K block.
// Question: why does the prefill's K loop take ~620 (N=256) / ~780 (N=128) cycles per K block when
// the MMAs alone should take 4 x 128 / 4 x 64-80?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2505_11076_b200/csrc umma_loop.cu -o umma_loop
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace dbf::sm100;

template <int N>
__global__ void __launch_bounds__(128, 1) bench(long long* out, int iters, int commits, int fence, int slots, int acc2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bars[4];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 192 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3C003C00u * ((i & 7) == 1);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
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
    constexpr int kBox = N * 128;  // one 64-column box of N rows
    const uint32_t b_smem = smem_u32(smem);
    const int nbox = (192 * 1024) / kBox;
    long long t0 = clock64();
    for (int kb = 0; kb < iters; ++kb) {
      if (fence) tc_fence_after();
      const uint32_t a = tmem + (acc2 ? 2 * N : N) + (kb % slots) * 32;
      const uint32_t d = tmem + (acc2 ? (kb / 64 & 1) * N : 0);
      const uint32_t b = b_smem + (kb % nbox) * kBox;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) mma_f16_ts(d, a + kk * 8, sdesc_k_sw128(b + kk * 32), idesc, 1);
      for (int c = 0; c < commits; ++c) mma_commit(&bars[c]);
    }
    mma_commit(&bars[3]);
    mbar_wait(&bars[3], 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

template <int N>
void run(int commits, int fence, int slots, int acc2) {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  const int iters = 2048;
  cudaFuncSetAttribute(bench<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int r = 0; r < 3; ++r) bench<N><<<148, 128, 200 * 1024>>>(d, iters, commits, fence, slots, acc2);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("N=%-3d commits %d fence %d A slots %2d acc2 %d: %s  cycles/K-block %6.1f  (math %d)\n", N, commits, fence,
         slots, acc2, cudaGetErrorString(e), avg / iters, 4 * 128 * N / 256);
  cudaFree(d);
}

int main() {
  for (int c = 0; c <= 2; ++c) run<256>(c, 0, 6, 0);
  run<256>(1, 1, 6, 0);
  run<256>(2, 1, 6, 0);
  for (int c = 0; c <= 2; ++c) run<128>(c, 0, 8, 1);
  run<128>(2, 1, 8, 1);
  run<128>(0, 0, 1, 1);
  run<64>(0, 0, 12, 1);
  run<64>(2, 1, 12, 1);
  return 0;
}
