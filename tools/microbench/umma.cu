// Microbenchmark: tcgen05.mma issue rate on B200 (kind::f16, M=128), A from TMEM (TS) or smem (SS),
// N = 64/128/256, with and without concurrent tcgen05.st traffic into other TMEM columns.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2505_11076_b200/csrc umma.cu -o umma
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace dbf::sm100;

template <int N, bool TS, bool ST>
__global__ void __launch_bounds__(256, 1) bench(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t done;
  __shared__ uint32_t tbase;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_mbar_init();
    stop = 0;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 1) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  long long t0 = 0, t1 = 0;
  if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = idesc_f16_f32(128, N);
    const uint32_t a_smem = smem_u32(smem), b_smem = smem_u32(smem + 32768);
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (TS)
        mma_f16_ts(tmem, tmem + 256 + (i & 3) * 8, sdesc_k_sw128(b_smem + (i & 3) * 32), idesc, 1);
      else
        mma_f16_ss(tmem, sdesc_k_sw128(a_smem + (i & 3) * 32), sdesc_k_sw128(b_smem + (i & 3) * 32), idesc, 1);
    }
    mma_commit(&done);
    mbar_wait(&done, 0);
    t1 = clock64();
    stop = 1;
    out[blockIdx.x] = t1 - t0;
  }
  if (ST && warp >= 4) {
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = 0;
    const uint32_t la = (uint32_t)((warp & 3) * 32) << 16;
    while (!stop) {
      tmem_st16(tmem + la + 384 + (lane & 1) * 16, v);
      tmem_wait_st();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

template <int N, bool TS, bool ST>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  const int iters = 4096;
  auto k = bench<N, TS, ST>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  k<<<148, 256, 70 * 1024>>>(d, iters);
  k<<<148, 256, 70 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double ideal = 128.0 * N / 256.0;
  printf("%-28s %s  cycles/mma %.1f  (ideal %.0f, %.0f%%)\n", name, cudaGetErrorString(e), avg / iters, ideal,
         100.0 * ideal / (avg / iters));
  cudaFree(d);
}

int main() {
  run<64, true, false>("TS N=64");
  run<128, true, false>("TS N=128");
  run<256, true, false>("TS N=256");
  run<128, false, false>("SS N=128");
  run<256, false, false>("SS N=256");
  run<128, true, true>("TS N=128 + tcgen05.st");
  run<256, true, true>("TS N=256 + tcgen05.st");
  return 0;
}
